# Round measurement on one B200 (run from the repo root under gpurun): smoke, GPU parity
# tests, a bench line per BASELINE config, the reference-schema suite CSVs, the launch list
# of the default bench command and one `ncu --set full` capture of every tensor-core layer of
# a ResNet-18 b512 forward. Output: gpurun_out/$TAG/.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${TAG:-measure}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
(nproc; lscpu | grep "Model name") > $O/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
if [ -z "$NOTESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
fi
timeout 900 python bench.py > $O/bench_resnet18.json 2> $O/bench_resnet18.err; echo "bench resnet18 rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_resnet18_reference.json 2> $O/bench_resnet18_reference.err
for m in alexnet cifar-vgg mnist-mlp bmm1024; do
  timeout 600 python bench.py --model $m > $O/bench_$m.json 2> $O/bench_$m.err; echo "bench $m rc=$?"
done
timeout 600 python bench.py --model cifar-vgg --batch 256 > $O/bench_cifar-vgg_b256.json 2> $O/bench_cifar-vgg_b256.err
if [ -z "$NOSUITES" ]; then
  for s in bmm bmm-bin bconv bconv-bin; do timeout 900 python scripts/bench_suites.py --suite $s --bmm-max-n 16384 --csv $O/suite_$s.csv > /dev/null 2>&1; echo "suite $s rc=$?"; done
  timeout 600 python scripts/bench_suites.py --suite model --model resnet18 --batches 8,64,256,512,1024,2048,4096 --csv $O/suite_model_resnet18.csv > /dev/null 2>&1; echo "suite model rc=$?"
fi
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_resnet18_b512.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernels > $O/ncu_l.log 2>&1; echo "ncu-l rc=$?"
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"first_conv_tc_kernel|bgemm_tc_kernel" -c 17 -o $O/resnet18_b512_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-kernels > $O/ncu_full.log 2>&1; echo "ncu-full rc=$?"
