# Per-role clock64 timelines (timing build) of chosen ResNet-18 b512 layers: LAYERS="2 4 14"
cd $GRAFT_REPO_ROOT; O=gpurun_out/timeline; mkdir -p $O
for L in $LAYERS; do
  BTNN_LIB=$PWD/paper_2006_16578_b200/libbtnn_cuda_timing.so BTNN_TC_DBG=16 BTNN_TC_DBG_NTH=$((L-1)) timeout 300 python scripts/tc_timeline_plan.py > $O/layer$L.txt 2>&1; echo "layer $L rc=$?"; cat $O/layer$L.txt | head -70
done
