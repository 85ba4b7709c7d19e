# session-4 check: GPU suite, then config 4 / 2 / 3 bench lines (no CPU baseline)
mkdir -p gpurun_out
TAG=${TAG:-s4}
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 3 gpurun_out/pytest_gpu_$TAG.log
for c in 4 2 3; do
  timeout 900 python bench.py --config $c --no-cpu > gpurun_out/bench${c}_$TAG.json 2> gpurun_out/bench${c}_$TAG.err; echo "bench$c rc $?"
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/bench${c}_$TAG.json").read().strip().splitlines()[-1])
    print("config $c", d["metric"], round(d["value"]), "ms/step", round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"]), d["clocks"]["sm_mhz"])
    print("   ", {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items() if v["ms_per_step"] > 0.3})
except Exception as e:
    print("config $c failed", e)
PY
done
