# Round profile: launch list of one b512 step, ncu --set full of the first conv and the
# first three tensor-core conv launches (L1 threshold halo, L2 bn halo, L3), bench line.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_${TAG:-final}.csv python bench.py --steps 1 --warmup 0 --batch 512 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"first_conv_tc_kernel|bgemm_tc_kernel" -c 4 -o gpurun_out/prof_${TAG:-final} python bench.py --steps 1 --warmup 0 --batch 512 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"
timeout 900 python bench.py > gpurun_out/bench_${TAG:-final}.json 2> gpurun_out/bench_${TAG:-final}.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_${TAG:-final}.json
