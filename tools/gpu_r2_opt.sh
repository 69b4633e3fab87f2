# round 2: optimiser-variant sweep (Adam: 15 warps / 128 registers, state rows prefetched into L2); F1 split tiles
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "split or strong_scaling or optimizer or compaction or kvl" > gpurun_out/opt_tests.log 2>&1; echo tests=$?
B() { timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@"; }
B --workload config4b --form KVL --opt adam --steps 20 --warmup 5 > gpurun_out/opt_kvl_adam.json 2>&1
B --workload config4b --form F2 --opt adam --steps 20 --warmup 5 > gpurun_out/opt_f2_adam.json 2>&1
B --workload config4b --form KVL --opt adam --steps 20 --warmup 5 --tile 4,2 > gpurun_out/opt_kvl_adam_42.json 2>&1
B --workload config4 --steps 20 --warmup 5 > gpurun_out/opt_f2.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/opt_ncu_kvl_adam python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --workload config4b --form KVL --opt adam > gpurun_out/opt_ncu.log 2>&1; echo ncu=$?
echo done
