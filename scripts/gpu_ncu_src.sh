# One `ncu --set full --import-source on` capture per named kernel launch of a ResNet-18
# b512 forward (first conv, and bgemm layers by launch index), for source-level analysis.
# Usage (under gpurun): TAG=x SKIPS="1 3" bash scripts/gpu_ncu_src.sh
cd $GRAFT_REPO_ROOT; O=gpurun_out/${TAG:-ncusrc}; mkdir -p $O
ARGS="bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernels ${BENCH_ARGS}"
if [ -z "$NOFTC" ]; then
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:first_conv_tc_kernel -c 1 -o $O/ftc python $ARGS > $O/ncu_ftc.log 2>&1; echo "ncu ftc rc=$?"
fi
for s in $SKIPS; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:bgemm_tc_kernel --launch-skip $s -c 1 -o $O/bg$s python $ARGS > $O/ncu_bg$s.log 2>&1; echo "ncu bg$s rc=$?"
done
