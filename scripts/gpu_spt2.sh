cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for E in "BTNN_HALO_WIDE=0" "BTNN_HALO_WIDE=1" "BTNN_HALO_WIDE=0 BTNN_HALO_SPT=1"; do
  env $E timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/spt_x.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/spt_x.json').read().strip().splitlines()[-1]);l=d['layer_ms'];print('$E', round(d['value']), [round(l[k],4) for k in sorted(l, key=lambda x:int(x.split(':')[0]))][:9])"
done
