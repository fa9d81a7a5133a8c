# r02b: GPU parity (incl. scale tests), bench lines for every BASELINE config, ncu of the first conv.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/r02b
O=gpurun_out/r02b
nproc > $O/nproc.txt; lscpu | grep "Model name" >> $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x --durations=30 > $O/pytest_scale.log 2>&1; echo "scale rc=$?"; tail -3 $O/pytest_scale.log
timeout 1500 python -m pytest tests -q -m gpu --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_resnet18.json 2> $O/bench_resnet18.err; echo "bench rc=$?"; head -c 600 $O/bench_resnet18.json; echo
for m in alexnet cifar-vgg mnist-mlp bmm1024; do
  timeout 600 python bench.py --model $m > $O/bench_$m.json 2> $O/bench_$m.err; echo "bench $m rc=$?"; head -c 300 $O/bench_$m.json; echo
done
timeout 600 python bench.py --model cifar-vgg --batch 256 > $O/bench_cifar-vgg_b256.json 2> $O/bench_cifar-vgg_b256.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_resnet18_b512.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernels > $O/ncu_l.log 2>&1; echo "ncu-l rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:first_conv_tc_kernel -c 1 -o $O/ftc python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernels > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?"
