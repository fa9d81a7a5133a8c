cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --batch 256 --no-cpu-baseline > gpurun_out/bench10.json 2> gpurun_out/bench10.err
head -c 3800 gpurun_out/bench10.json; tail -3 gpurun_out/bench10.err
