# the cluster path's single-instance lines (config 3) and its parity tests
O=gpurun_out/cluster
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B c3_f2 --workload config3 --steps 2000 --warmup 100 --no-gap
B c3_kvl --workload config3 --form KVL --steps 2000 --warmup 100 --no-gap
B c3_f1 --workload config3 --form F1 --steps 2000 --warmup 100 --no-gap
B c3_kvl_adam --workload config3 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-gap
B c3_f2_adam --workload config3 --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-gap
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster or config3 or config1 or config2 or optimizer or adam" > $O/tests.log 2>&1; echo tests=$?
