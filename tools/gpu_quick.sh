# quick GPU check: parity tests + config-4 bench (F2, F1, KVL); PYTEST_K -> pytest -k
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for f in F2 F1 KVL; do python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form $f > gpurun_out/q_$f.json 2>&1; echo $f=$?; done
python - <<'PY'
import json
for f in ("F2", "F1", "KVL"):
    for l in open(f"gpurun_out/q_{f}.json"):
        if l.startswith("{"):
            d = json.loads(l)
            print(f, "%.4g inst-it/s  frac %.3f  ms/step %.4f" % (d["value"], d["roofline"]["frac"], d["ms_per_step"]), d["config"]["kernel"]["chunk"], d["config"]["kernel"]["smem"])
PY
