# round 2: the whole GPU suite + smoke, the default bench line, an A/B of a variant build
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/full_tests.log 2>&1; echo tests=$?
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/full_bench_default.json 2> gpurun_out/full_bench_default.err; echo bench=$?
for rep in 1 2; do
  for v in base fma; do
    if [ $v = base ]; then L=""; else L="DCOPF_LIB=paper_2406_13191_b200/lib/variants/$v.so"; fi
    env $L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e > gpurun_out/full_ab_${v}_$rep.json 2>&1
    env $L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e --form KVL > gpurun_out/full_ab_${v}_kvl_$rep.json 2>&1
  done
done
echo done
