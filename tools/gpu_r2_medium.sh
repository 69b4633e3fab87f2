# round 2: medium batches (branch-and-bound sized) on config-4 instances of the
# 10k-bus network: cluster path (one 16-CTA cluster per instance) vs batched
# path (split tiles), F2 and KVL -> the AUTO threshold
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@"; }
for f in F2 KVL; do
for b in 4 16 64 128 256; do
  B --form $f --batch $b --path cluster --steps 200 --warmup 20 > gpurun_out/med_${f}_cl_$b.json 2>&1
  B --form $f --batch $b --path batched --steps 100 --warmup 10 > gpurun_out/med_${f}_ba_$b.json 2>&1
done
done
echo done
