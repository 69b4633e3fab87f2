# the chunk-aware tiling choice: per-shard-size lines (F2 / KVL / F1) and the split / compaction parity subset
O=gpurun_out/tiles2
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "split or strong_scaling or compaction or config4 or batch" > $O/tests.log 2>&1; echo tests=$?; tail -1 $O/tests.log
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 50 --warmup 5 "$@" > $O/$name.json 2> $O/$name.err; }
for b in 8192 4096 2048 1024; do
  B f2_$b --batch $b; B kvl_$b --batch $b --form KVL; B f1_$b --batch $b --form F1
done
for f in $O/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['config']['kernel']; t=d['config']['tile']; print('$f', round(d['value']), 'V', t['lane_instances'], 'C', t['parts'], 'W', k['tile_width'], 'ch', k['chunk'])"; done
