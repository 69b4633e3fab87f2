set -x
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -x -q -k optimizer 2>&1 | tail -2
for f in KVL F2; do python bench.py --workload config4b --form $f --opt adam --alpha 0.1 --steps 30 --warmup 3 --no-cpu-baseline ${NOGAP} > gpurun_out/final/bench_config4b_${f}_adam.json 2>&1; echo $f=$?; done
python bench.py --workload config4b --form KVL --steps 30 --warmup 3 --no-cpu-baseline --no-gap > gpurun_out/final/bench_config4b_KVL.json 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/final/bench_config4b_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); t = d.get("time_to_gap") or {}
            print(f, "%.4g" % d["value"], "frac %.3f" % d["roofline"]["frac"], "ttg", t.get("seconds"), t.get("max_hit_iteration"), t.get("true_gap_at_K"), t.get("reached"))
PY
