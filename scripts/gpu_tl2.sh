# L1 (threshold halo) timelines under timing-experiment switches.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for F in 16 28 18 30 17; do
  BTNN_TC_DBG=$F BTNN_TC_DBG_NTH=19 timeout 300 python scripts/tc_timeline_plan.py > gpurun_out/tl_L1_$F.txt 2>&1; echo "F=$F rc=$?"
  grep -A7 "halo units" gpurun_out/tl_L1_$F.txt
done
