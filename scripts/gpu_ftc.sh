# First-conv iteration: exactness tests, timeline, bench A/B.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "first or resnet or smoke or model" > gpurun_out/pytest_ftc.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_ftc.log
BTNN_FTC_DBG=1 timeout 300 python scripts/ftc_timeline.py > gpurun_out/tl_ftc.txt 2>&1; echo ftc rc=$?; head -14 gpurun_out/tl_ftc.txt; tail -9 gpurun_out/tl_ftc.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"]), "e2e", round(d["e2e"]["value"]), "ms", round(d["ms_per_step"], 3))
print("layers", d.get("layer_ms"))
PY
