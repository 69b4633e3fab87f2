# dense path, one instance, Adam / AdaGrad on the single-read step (fast division / sqrt) vs the two-pass kernels
O=gpurun_out/ptdf_adam
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests/test_gpu_ptdf.py -x -q > $O/tests_ptdf.log 2>&1; echo tests=$?; tail -1 $O/tests_ptdf.log
V=paper_2406_13191_b200/lib/variants
B() { lib=$1; name=$2; shift 2; if [ -n "$lib" ]; then export DCOPF_LIB=$lib; else unset DCOPF_LIB; fi
      timeout 900 python bench.py --no-cpu-baseline "$@" > $O/$name.json 2> $O/$name.err; echo $name=$?; }
for v in cur twopass; do
  L=""; [ $v = cur ] || L=$V/$v.so
  B "$L" ${v}_c3_adam --workload config3 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100
  B "$L" ${v}_c3_adagrad --workload config3 --form PTDF --opt adagrad --alpha 5 --steps 2000 --warmup 100 --no-gap
  B "$L" ${v}_c1_adam --workload config1 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100 --no-gap
done
unset DCOPF_LIB
B "" c3_plain --workload config3 --form PTDF --steps 1000 --warmup 20 --no-gap
for f in $O/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); t=d.get('time_to_gap') or {}; print('$f', round(d['ms_per_step']*1000,2), 'us/it', 'ttg', t.get('seconds'), t.get('max_hit_iteration'))"; done
