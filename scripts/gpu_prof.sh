# Profile: ncu --set full (source-correlated) on the first-conv TC kernel and the first
# two bit-conv layers (threshold + bn route) of one bench step, plus the launch list.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-bgemm_tc_kernel|first_conv_tc_kernel}" -c ${NCU_C:-3} -o gpurun_out/prof_${TAG:-x} python bench.py --steps 1 --warmup 0 --batch ${NCU_B:-256} --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"; tail -3 gpurun_out/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_${TAG:-x}.csv python bench.py --steps 1 --warmup 0 --batch 512 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo "ncu-l rc=$?"
