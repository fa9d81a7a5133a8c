# A/B of library variants on the bench line's e2e (models in $MODELS), interleaved. Under gpurun.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${TAG:-abe}; mkdir -p $O
for r in $(seq ${ROUNDS:-2}); do
  for m in ${MODELS:-mnist-mlp}; do
    for v in ${LIBS:-prod}; do
      lib=$PWD/paper_2006_16578_b200/libbtnn_cuda_$v.so; [ "$v" = "prod" ] && lib=$PWD/paper_2006_16578_b200/libbtnn_cuda.so
      BTNN_LIB=$lib timeout 600 python bench.py --model $m --no-cpu-baseline --no-kernels > $O/b_${m}_${v}_$r.json 2> $O/b_${m}_${v}_$r.err
      python -c "
import json; d=json.load(open('$O/b_${m}_${v}_$r.json')); e=d['e2e']; print('$m $v', round(d['value']), round(e['value']), e.get('steps'), (e.get('pipeline') or {}).get('chunks'))"
    done
  done
done
