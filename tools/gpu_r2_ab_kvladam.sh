# A/B of a library variant against the current build on the KVL / F2 optimiser lines (3 reps, K = 100)
O=gpurun_out/ab_kvladam
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=paper_2406_13191_b200/lib/variants
for rep in 1 2 3; do
  for v in cur "$@"; do
    if [ $v = cur ]; then unset DCOPF_LIB; else export DCOPF_LIB=$V/$v.so; fi
    timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 100 --warmup 5 --workload config4b --form KVL --opt adam > $O/${v}_kvl_adam_$rep.json 2>/dev/null
    timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 100 --warmup 5 --workload config4b --form F1 --opt adam > $O/${v}_f1_adam_$rep.json 2>/dev/null
    timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 20 --warmup 5 --form KVL > $O/${v}_kvl_k20_$rep.json 2>/dev/null
  done
done
for f in $O/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']))"; done
