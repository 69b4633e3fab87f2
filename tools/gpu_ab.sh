# A/B: the reference build (lib/libdcopf_dual_ref.so) vs the current one, same box, interleaved
set -x
for r in 1 2; do for v in ref cur; do
  L=""; [ $v = ref ] && L=paper_2406_13191_b200/lib/libdcopf_dual_ref.so
  for f in ${FORMS:-F2 F1}; do DCOPF_LIB=$L python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form $f > gpurun_out/ab_${v}_${f}_$r.json 2>&1; done
done; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/ab_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l); print(f, "%.4g" % d["value"], "ms/step %.4f" % d["ms_per_step"], d["config"]["kernel"]["chunk"], d["config"]["kernel"]["smem"])
PY
