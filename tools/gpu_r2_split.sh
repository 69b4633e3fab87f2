# round 2: split tiles / 4 instances per lane -- parity first, then the batch sweep
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or strong_scaling or sharding or config4_full or kvl_batched or more_tiles" > gpurun_out/r2_split_tests.log 2>&1; echo tests=$?
for B in 8192 4096 2048 1024; do
  timeout 300 python bench.py --batch $B --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e > gpurun_out/r2s_F2_$B.json 2> gpurun_out/r2s_F2_$B.err; echo B$B=$?
done
for B in 8192 1024; do
  timeout 300 python bench.py --batch $B --form KVL --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e > gpurun_out/r2s_KVL_$B.json 2> gpurun_out/r2s_KVL_$B.err; echo K$B=$?
done
