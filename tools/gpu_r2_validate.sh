# final validation of the build: smoke, the whole GPU suite, the driver's bench command and the default bench
O=gpurun_out/validate
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke=$?
timeout 3000 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo tests=$?; tail -1 $O/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_driver.json 2> $O/bench_driver.err; echo driver=$?
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo default=$?
timeout 900 python bench.py --workload config3 --form PTDF --opt adam --alpha 64 --decay step:0.5:30 --steps 2000 --warmup 100 --no-cpu-baseline > $O/bench_config3_PTDF_adam_step.json 2> $O/e3.err; echo c3=$?
B() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B config4_KVL --form KVL --no-gap
B config4_KVL_K20 --form KVL --no-gap --steps 20 --warmup 5
B config4b_KVL_adam --workload config4b --form KVL --opt adam --no-gap
B config4b_F2_adam --workload config4b --form F2 --opt adam --no-gap
B shard1024_KVL --batch 1024 --form KVL --no-gap --no-e2e --steps 50 --warmup 5
for f in $O/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.4g'%d['value'], 'frac', round(d['roofline']['frac'],3), 'e2e', d.get('e2e') and '%.3g'%d['e2e']['value'], 'ttg-b', (d.get('time_to_true_gap_batched') or {}).get('seconds'), 'ttg-s', (d.get('time_to_true_gap_single') or {}).get('seconds'))"; done
