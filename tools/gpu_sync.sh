set -x
for f in F2 F1; do for m in hard soft; do DCOPF_SYNC=$m python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form $f > gpurun_out/s_${f}_$m.json 2>&1; done; done
python - <<'PY'
import json
for f in ("F2","F1"):
  for m in ("hard","soft"):
    for l in open(f"gpurun_out/s_{f}_{m}.json"):
        if l.startswith("{"):
            d = json.loads(l); print(f, m, "%.4g" % d["value"], "ms/step %.4f" % d["ms_per_step"], d["config"]["kernel"]["chunk"], d["config"]["kernel"]["smem"])
PY
