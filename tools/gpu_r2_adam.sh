# batched path, optimiser variants: bench lines (config 4b, KVL / F2 + Adam) and the OPT parity subset
set -x
O=gpurun_out/adam
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B kvl_adam --workload config4b --form KVL --opt adam --steps 20 --warmup 5
B f2_adam --workload config4b --form F2 --opt adam --steps 20 --warmup 5
B kvl_gdm --workload config4b --form KVL --opt gdm --alpha 1e-3 --steps 20 --warmup 5
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ptdf.py tests/test_gpu_compact.py -x -q -k "optimizer or adam or gdm or adagrad or decay or skinny or single_read" > $O/tests.log 2>&1; echo tests=$?
echo done
