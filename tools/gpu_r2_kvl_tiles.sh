O=gpurun_out/kvl42
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 100 --warmup 5 "$@" > $O/$name.json 2>/dev/null; }
for rep in 1 2; do
  B kvl_auto_$rep --form KVL
  B kvl_42_$rep --form KVL --tile 4,2
  B kvl_adam_auto_$rep --workload config4b --form KVL --opt adam
  B kvl_adam_42_$rep --workload config4b --form KVL --opt adam --tile 4,2
  B f2_42_$rep --tile 4,2
done
B kvl_44_4096 --form KVL --tile 4,4 --batch 4096
B kvl_auto_4096 --form KVL --batch 4096
for f in $O/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], round(d['value']), d['config']['kernel']['chunk'], d['config']['tile']['steps_per_sweep'])"; done
