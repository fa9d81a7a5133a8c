# One ncu --set full capture (source-correlated) of kernel regex NCU_K at batch NCU_B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-first_conv_tc_kernel}" -c ${NCU_C:-1} -o gpurun_out/prof_${TAG:-x} python bench.py --steps 1 --warmup 0 --batch ${NCU_B:-512} --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"; tail -3 gpurun_out/ncu_full.log
