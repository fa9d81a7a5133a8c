# Per-role timelines: first conv, L1 (threshold halo), L2 (bn halo, TMA), L4 (blocked).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BTNN_FTC_DBG=1 timeout 300 python scripts/ftc_timeline.py > gpurun_out/tl_ftc.txt 2>&1; echo ftc rc=$?
for L in 1 2 4; do
  BTNN_TC_DBG=16 BTNN_TC_DBG_NTH=$((19 + L - 1)) timeout 300 python scripts/tc_timeline_plan.py > gpurun_out/tl_L$L.txt 2>&1; echo L$L rc=$?
done
