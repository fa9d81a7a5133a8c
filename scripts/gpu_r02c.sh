# r02c: bench lines for every BASELINE config, launch list and ncu --set full of the first conv.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r02c; mkdir -p $O
timeout 900 python bench.py > $O/bench_resnet18.json 2> $O/bench_resnet18.err; echo "bench rc=$?"; head -c 400 $O/bench_resnet18.json; echo
for m in alexnet cifar-vgg mnist-mlp; do
  timeout 600 python bench.py --model $m > $O/bench_$m.json 2> $O/bench_$m.err; echo "bench $m rc=$?"; head -c 300 $O/bench_$m.json; echo; tail -2 $O/bench_$m.err
done
timeout 600 python bench.py --model cifar-vgg --batch 256 > $O/bench_cifar-vgg_b256.json 2> $O/bench_cifar-vgg_b256.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_resnet18_b512.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernels > $O/ncu_l.log 2>&1; echo "ncu-l rc=$?"; tail -3 $O/ncu_l.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:first_conv_tc_kernel -c 1 -o $O/ftc python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernels > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?"; tail -3 $O/ncu_full.log
