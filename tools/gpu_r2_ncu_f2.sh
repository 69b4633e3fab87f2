# ncu --set full capture (with source) of the plain batched sweep (config 4, F2: the headline kernel) + the optimiser parity subset
O=gpurun_out/ncu_f2
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "optimizer or adam or gdm or adagrad or decay or split" > $O/tests.log 2>&1; echo tests=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > $O/plain_run.json 2>&1; echo run=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o $O/ncu_f2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > $O/ncu_f2.log 2>&1; echo ncu=$?
tail -1 $O/tests.log
