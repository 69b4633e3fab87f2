# quick GPU check: parity tests + config-4 bench (F2, F1); extra args -> pytest -k
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > gpurun_out/q_f2.json 2>&1; echo f2=$?
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form F1 > gpurun_out/q_f1.json 2>&1; echo f1=$?
python - <<'PY'
import json
for f in ("gpurun_out/q_f2.json", "gpurun_out/q_f1.json"):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f, "%.4g inst-it/s  frac %.3f  ms/step %.4f" % (d["value"], d["roofline"]["frac"], d["ms_per_step"]), d["clocks"])
PY
