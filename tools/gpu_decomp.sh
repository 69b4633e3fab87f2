# decomposition of the batched kernel: normal / data movement only / compute only, + ncu full capture
set -x
for m in 0 1 2; do DCOPF_DEBUG_MODE=$m python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap ${BENCH_ARGS} > gpurun_out/dm$m.json 2>&1; done
python - <<'PY'
import json
for m in (0,1,2):
    for l in open(f"gpurun_out/dm{m}.json"):
        if l.startswith("{"):
            d = json.loads(l); print("mode", m, "ms/step %.4f" % d["ms_per_step"], "%.4g" % d["value"])
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/ncu_${TAG:-x} python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap ${BENCH_ARGS} > gpurun_out/ncu_${TAG:-x}.log 2>&1; echo ncu=$?
