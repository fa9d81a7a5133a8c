cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --batch 256 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err
head -c 2500 gpurun_out/bench6.json; tail -3 gpurun_out/bench6.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bgemm_tc_kernel -c 3 -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 1 --batch 256 --no-cpu-baseline > gpurun_out/ncu_tc.log 2>&1; tail -3 gpurun_out/ncu_tc.log
