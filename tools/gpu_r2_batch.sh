# round 2: per-shard-size baseline of the batched path on one GPU (the literal
# config-4 split: 8192 / 4096 / 2048 / 1024 instances per GPU at N = 1 / 2 / 4 / 8)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
for B in 8192 4096 2048 1024; do
  python bench.py --batch $B --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e > gpurun_out/r2_batch_F2_$B.json 2> gpurun_out/r2_batch_F2_$B.err; echo B$B=$?
done
for B in 8192 1024; do
  python bench.py --batch $B --form KVL --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e > gpurun_out/r2_batch_KVL_$B.json 2> gpurun_out/r2_batch_KVL_$B.err; echo K$B=$?
done
