cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/bench_suites.py --suite bmm --bmm-max-n 16384 --csv gpurun_out/suite_bmm.csv; echo "bmm rc=$?"
python scripts/bench_suites.py --suite bmm-bin --bmm-max-n 16384 --csv gpurun_out/suite_bmm_bin.csv; echo "bmm-bin rc=$?"
python scripts/bench_suites.py --suite bconv --csv gpurun_out/suite_bconv.csv; echo "bconv rc=$?"
python scripts/bench_suites.py --suite bconv-bin --csv gpurun_out/suite_bconv_bin.csv; echo "bconv-bin rc=$?"
python scripts/bench_suites.py --suite model --model resnet18 --batches 8,16,32,64,128,256,512,1024,2048,4096 --csv gpurun_out/suite_model_resnet18.csv; echo "model rc=$?"
for f in gpurun_out/suite_*.csv; do echo "== $f"; cat $f; done
