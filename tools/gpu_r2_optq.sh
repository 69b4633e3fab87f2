# after a change to the optimiser kernels: the batched Adam / AdaGrad bench lines and the optimiser parity subset
O=gpurun_out/optq
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B kvl_adam --workload config4b --form KVL --opt adam --steps 20 --warmup 5
B f2_adam --workload config4b --form F2 --opt adam --steps 20 --warmup 5
B kvl_adagrad --workload config4b --form KVL --opt adagrad --steps 20 --warmup 5
B f2 --steps 20 --warmup 5
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "optimizer or adam or gdm or adagrad or decay or split" > $O/tests.log 2>&1; echo tests=$?
for f in $O/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['roofline']['frac'],3))"; done
tail -1 $O/tests.log
