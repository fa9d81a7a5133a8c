# A/B of timing-build knobs on the ResNet-18 b512 bench line (per-layer ms). Each entry of
# $KNOBS is a comma-separated env assignment list ("-" = none). Under gpurun.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${TAG:-knobs}; mkdir -p $O
for k in ${KNOBS:--}; do
  envs=$(echo "$k" | tr ',' ' '); [ "$k" = "-" ] && envs=""
  env $envs BTNN_LIB=$PWD/paper_2006_16578_b200/libbtnn_cuda_timing.so timeout 600 python bench.py --model ${MODEL:-resnet18} --no-cpu-baseline --no-kernels > $O/bench_$k.json 2> $O/bench_$k.err
  python -c "
import json; d=json.load(open('$O/bench_$k.json')); print('$k', round(d['value']), d['parity']['bit_exact']); print(' '.join(f'{v:.3f}' for v in d['layer_ms'].values()))"
done
