# round 2: parity subset + the main bench lines (after a kernel change)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "split or strong_scaling or optimizer or compaction or kvl or config4 or evaluate" > gpurun_out/q_tests.log 2>&1; echo tests=$?
B() { timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 20 --warmup 5 "$@"; }
for rep in 1 2; do
B > gpurun_out/q_f2_$rep.json 2>&1
B --form KVL > gpurun_out/q_kvl_$rep.json 2>&1
done
B --form F1 > gpurun_out/q_f1.json 2>&1
B --batch 1024 > gpurun_out/q_f2_1024.json 2>&1
B --batch 1024 --form KVL > gpurun_out/q_kvl_1024.json 2>&1
B --workload config4b --form KVL --opt adam > gpurun_out/q_kvl_adam.json 2>&1
echo done
