set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
B --tile 2,1 > gpurun_out/ab3_cur21.json 2>&1; echo cur=$?
B --tile 4,2 > gpurun_out/ab3_cur42.json 2>&1; echo cur42=$?
B --batch 1024 > gpurun_out/ab3_1024.json 2>&1; echo b1024=$?
B --form KVL > gpurun_out/ab3_kvl.json 2>&1; echo kvl=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/ncu_ab3_21 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --tile 2,1 > gpurun_out/ncu_ab3_21.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/ncu_ab3_42 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --tile 4,2 > gpurun_out/ncu_ab3_42.log 2>&1; echo ncu=$?
