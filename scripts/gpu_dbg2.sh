cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for d in 0 64 128 192 2; do
  BTNN_TC_DBG=$d timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/dbg_$d.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/dbg_$d.json').read().strip().splitlines()[-1]); l=d['layer_ms']
print('dbg=$d', ' '.join(f'{k.split(\":\")[0]}:{v:.3f}' for k,v in l.items()))"
done
