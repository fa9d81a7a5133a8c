# e2e chunk-size A/B (bench.py e2e key), two runs each.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for C in 128 64 128 64; do
  BTNN_E2E_CHUNK=$C timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b_e2e_$C.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/b_e2e_$C.json').read().strip().splitlines()[-1]);print('chunk $C', round(d['value']), 'e2e', round(d['e2e']['value']))"
done
