O=gpurun_out/ab_kvlp2
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V=paper_2406_13191_b200/lib/variants
for rep in 1 2; do
  for v in cur kvlp2; do
    if [ $v = cur ]; then unset DCOPF_LIB; else export DCOPF_LIB=$V/$v.so; fi
    timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 100 --warmup 5 --workload config4b --form KVL --opt adam > $O/${v}_kvl_adam_$rep.json 2>/dev/null
    timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 100 --warmup 5 --workload config4b --form KVL --opt adagrad > $O/${v}_kvl_adagrad_$rep.json 2>/dev/null
  done
done
for f in $O/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['config']['kernel']['chunk'], d['config']['kernel']['smem'])"; done
