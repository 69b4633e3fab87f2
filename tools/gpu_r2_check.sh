# round 2: parity subset + bench lines + ncu of the split sweep (after a kernel change)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "split or strong_scaling or sharding or config4 or kvl_batched or more_tiles or compaction or evaluate or outages" > gpurun_out/chk_tests.log 2>&1; echo tests=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
B --tile 4,2 > gpurun_out/chk_42.json 2>&1
B --tile 2,1 > gpurun_out/chk_21.json 2>&1
B --form KVL > gpurun_out/chk_kvl.json 2>&1
B --batch 1024 > gpurun_out/chk_1024.json 2>&1
B --batch 1024 --form KVL > gpurun_out/chk_1024_kvl.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/ncu_chk_42 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --tile 4,2 > gpurun_out/ncu_chk_42.log 2>&1; echo ncu=$?
echo done
