# the whole GPU suite, smoke and the default bench on the current build
O=gpurun_out/suite
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke=$?
timeout 3000 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo tests=$?
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_driver.json 2> $O/bench_driver.err; echo bench=$?
timeout 900 python bench.py --workload config1 --form PTDF --steps 1000 --warmup 20 --no-cpu-baseline --no-gap > $O/bench_c1_ptdf.json 2> $O/e1.err; echo c1=$?
DCOPF_PTDF_FUSED=0 timeout 900 python bench.py --workload config1 --form PTDF --steps 1000 --warmup 20 --no-cpu-baseline --no-gap > $O/bench_c1_ptdf_2pass.json 2> $O/e2.err; echo c12=$?
timeout 900 python bench.py --workload config3 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > $O/bench_c3_kvl_adam.json 2> $O/e3.err; echo c3kvl=$?
echo done
