# F1 on the per-GPU shards of the literal config-4 split: parts per tile (--tile 2,C) at 1024 / 2048 instances
O=gpurun_out/f1_tiles
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "optimizer or adam or adagrad" > $O/tests.log 2>&1; echo tests=$?; tail -1 $O/tests.log
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 50 --warmup 5 --form F1 "$@" > $O/$name.json 2> $O/$name.err; }
B auto1024 --batch 1024
for c in 2 4 6 12 16; do B b1024_c$c --batch 1024 --tile 2,$c; done
B auto2048 --batch 2048
for c in 2 4 8; do B b2048_c$c --batch 2048 --tile 2,$c; done
for f in $O/*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['config']['kernel']; t=d['config']['tile']; print('$f', round(d['value']), t['parts'], k['tile_width'], k['chunk'], k['grid'])"; done
