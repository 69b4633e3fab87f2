# one instance, dense PTDF + Adam: time to a TRUE 1e-3 gap (exact optimum) under several step schedules
O=gpurun_out/single_gap
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
B() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 200 --warmup 10 "$@" > $O/$name.json 2> $O/$name.err; echo $name=$?; }
for s in "5 inv:200" "48 step:0.5:40" "32 step:0.5:50" "16 step:0.5:60" "64 step:0.5:30" "24 step:0.5:40" "16 step:0.5:100" "8 step:0.5:150"; do
  set -- $s
  B c3_$1_${2//:/_} --workload config3 --form PTDF --opt adam --alpha $1 --decay $2
done
for w in config1 config2 config3q; do
  B ${w}_48_step --workload $w --form PTDF --opt adam --alpha 48 --decay step:0.5:40
  B ${w}_5_inv --workload $w --form PTDF --opt adam --alpha 5 --decay inv:200
done
for f in $O/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); t=d.get('time_to_true_gap_single') or {}; print('$f'.split('/')[-1], round(d['ms_per_step']*1e3,1), 'us/it', 'hit', t.get('hit_iteration'), 's', t.get('seconds'), 'gap', t.get('true_gap_at_stop'))"; done
