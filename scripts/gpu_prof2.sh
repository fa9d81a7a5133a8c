cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bgemm_tc_kernel|first_conv_tiled" -c 3 -o gpurun_out/prof2 python bench.py --steps 1 --warmup 1 --batch 256 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; tail -3 gpurun_out/ncu2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 0 --batch 256 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; tail -2 gpurun_out/ncu_l.log
