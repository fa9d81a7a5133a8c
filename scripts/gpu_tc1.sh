cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -q -m gpu -x -k "tc" > gpurun_out/pytest_tc.log 2>&1; tail -30 gpurun_out/pytest_tc.log
timeout 600 python bench.py --steps 10 --warmup 3 --batch 256 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err
head -c 2500 gpurun_out/bench3.json; tail -3 gpurun_out/bench3.err
