# the bench lines with their e2e (set_instance_batch from pinned host memory + iterate + get_bound)
O=gpurun_out/e2e
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
B() { name=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B default
B driver --steps 20 --warmup 5
B config4_KVL --form KVL --no-cpu-baseline --no-gap
B config4_F1 --form F1 --no-cpu-baseline --no-gap
B config4b_KVL_adam --workload config4b --form KVL --opt adam --no-cpu-baseline
B config4b_F2_adam --workload config4b --form F2 --opt adam --no-cpu-baseline
B config4b_KVL_adagrad --workload config4b --form KVL --opt adagrad --no-cpu-baseline --no-gap
timeout 1800 python -m pytest tests/test_gpu_compact.py tests/test_gpu_parity.py -x -q -k "compaction or strong_scaling or forced" > $O/tests.log 2>&1; echo tests=$?; tail -1 $O/tests.log
