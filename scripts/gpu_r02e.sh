# r02e: first-conv generalization + halo pair mode: kernel tests, model parity, bench lines.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r02e; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "first_conv or halved or bconv" > $O/pytest_fc.log 2>&1; echo "fc rc=$?"; tail -4 $O/pytest_fc.log
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_models.py -q -x > $O/pytest_models.log 2>&1; echo "models rc=$?"; tail -4 $O/pytest_models.log
for m in resnet18 alexnet cifar-vgg; do
  timeout 600 python bench.py --model $m --no-cpu-baseline --no-kernels > $O/bench_$m.json 2> $O/bench_$m.err; echo "bench $m rc=$?"; head -c 250 $O/bench_$m.json; echo; tail -2 $O/bench_$m.err
done
