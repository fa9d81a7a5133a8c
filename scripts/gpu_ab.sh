# A/B: bench with the default path and with an env toggle (AB_ENV), then GPU tests.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python - "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"], 3))
    print("layers", d.get("layer_ms"))
except Exception as e:
    print("bench parse failed", e)
PY
}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench A rc=$?"; summ gpurun_out/bench.json; tail -3 gpurun_out/bench.err
env ${AB_ENV:-BTNN_TC_NOTMA=1} timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench B rc=$?"; summ gpurun_out/bench_b.json
timeout 1500 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
