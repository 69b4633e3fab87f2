# branch-free fp64 division / square root in the adaptive optimisers: the
# fast-path bit check, the optimiser parity subset, the Adam / AdaGrad bench lines
O=gpurun_out/fastdiv
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -Ipaper_2406_13191_b200/csrc tools/fp64_fastpath_check.cu -o /tmp/fp64_fastpath_check > $O/check_build.log 2>&1
timeout 300 /tmp/fp64_fastpath_check 64 > $O/fp64_fastpath_check.json 2>&1; echo check=$?
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B kvl_adam --workload config4b --form KVL --opt adam --steps 20 --warmup 5
B f2_adam --workload config4b --form F2 --opt adam --steps 20 --warmup 5
B kvl_adagrad --workload config4b --form KVL --opt adagrad --steps 20 --warmup 5
B c3_kvl_adam --workload config3 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100
B c3_f2_adam --workload config3 --form F2 --opt adam --alpha 0.1 --steps 2000 --warmup 100
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "optimizer or adam or gdm or adagrad or decay" > $O/tests.log 2>&1; echo tests=$?
echo done
