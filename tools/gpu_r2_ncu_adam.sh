# batched path, Adam: bench lines + one ncu --set full capture of the sweep (config 4b, KVL + Adam)
O=gpurun_out/adam
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B kvl_adam --workload config4b --form KVL --opt adam --steps 20 --warmup 5
B f2_adam --workload config4b --form F2 --opt adam --steps 20 --warmup 5
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ptdf.py -x -q -k "optimizer or adam or adagrad or decay or skinny" > $O/tests.log 2>&1; echo tests=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o $O/ncu_kvl_adam python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --workload config4b --form KVL --opt adam > $O/ncu.log 2>&1; echo ncu=$?
