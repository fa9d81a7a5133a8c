# A/B of library variants on the bench line (per-layer ms): LIBS="name ..." selects
# paper_2006_16578_b200/libbtnn_cuda_<name>.so ("prod" = the product library), run
# interleaved ROUNDS times. Under gpurun.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${TAG:-ab}; mkdir -p $O
for r in $(seq ${ROUNDS:-2}); do
  for v in ${LIBS:-prod}; do
    lib=$PWD/paper_2006_16578_b200/libbtnn_cuda_$v.so; [ "$v" = "prod" ] && lib=$PWD/paper_2006_16578_b200/libbtnn_cuda.so
    BTNN_LIB=$lib timeout 600 python bench.py --model ${MODEL:-resnet18} --no-cpu-baseline --no-kernels > $O/bench_${v}_$r.json 2> $O/bench_${v}_$r.err
    python -c "
import json; d=json.load(open('$O/bench_${v}_$r.json')); print('$v', round(d['value']), d['parity']['bit_exact']); print(' '.join(f'{v:.3f}' for v in d['layer_ms'].values()))"
  done
done
