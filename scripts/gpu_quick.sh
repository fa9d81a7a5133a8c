# Quick A/B: ResNet-18 b512 bench line (parity + per-layer ms), optional extra models.
cd $GRAFT_REPO_ROOT; O=gpurun_out/quick; mkdir -p $O
for m in resnet18 $EXTRA; do
  timeout 600 python bench.py --model $m --no-cpu-baseline --no-kernels > $O/bench_$m.json 2> $O/bench_$m.err; echo "bench $m rc=$?"; tail -2 $O/bench_$m.err
  python -c "
import json; d=json.load(open('$O/bench_$m.json')); print('$m', round(d['value']), 'e2e', round(d['e2e']['value']), d['parity']['bit_exact'], round(d['roofline']['frac'],3)); print({k:v for k,v in d['layer_ms'].items()})"
done
