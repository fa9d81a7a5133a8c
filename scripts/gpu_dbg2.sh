cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python scripts/debug_tc2.py 2>&1 | tail -40
timeout 600 python bench.py --steps 10 --warmup 3 --batch 256 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err
head -c 3500 gpurun_out/bench8.json; tail -3 gpurun_out/bench8.err
