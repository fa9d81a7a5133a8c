# Halo sites-per-tile sweep (timing experiment): per-layer times at SPT = auto, 16, 8, 4, 2.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for T in 0 16 8 4 2; do
  BTNN_HALO_SPT=$T timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/spt_$T.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/spt_$T.json').read().strip().splitlines()[-1]);l=d['layer_ms'];print('spt=$T', round(d['value']), [round(l[k],4) for k in sorted(l, key=lambda x:int(x.split(':')[0]))][:9])"
done
