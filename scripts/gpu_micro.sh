# Engine peaks + tcgen05 layout probe, then a short bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
make -C paper_2006_16578_b200/csrc microbench > gpurun_out/mb_build.log 2>&1
timeout 300 ./build/microbench > gpurun_out/microbench.json 2> gpurun_out/microbench.err
cat gpurun_out/microbench.json gpurun_out/microbench.err
timeout 600 python bench.py --steps 10 --warmup 3 --batch 256 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
head -c 1500 gpurun_out/bench2.json; tail -3 gpurun_out/bench2.err
