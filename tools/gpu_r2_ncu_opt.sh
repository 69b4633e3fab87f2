# one ncu --set full capture (with source) of the batched sweep: config 4b KVL + Adam (and F2 + Adam)
O=gpurun_out/ncu_opt
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --workload config4b --form KVL --opt adam > $O/plain_run.json 2>&1; echo run=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o $O/ncu_kvl_adam python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --workload config4b --form KVL --opt adam > $O/ncu_kvl.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o $O/ncu_f2_adam python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --workload config4b --form F2 --opt adam > $O/ncu_f2.log 2>&1; echo ncu2=$?
