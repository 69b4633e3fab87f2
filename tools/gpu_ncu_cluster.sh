set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cluster -c 1 -o gpurun_out/ncu_cluster_c3_steady python bench.py --workload config3 --steps 100 --warmup 400 --no-cpu-baseline --no-e2e --no-gap > gpurun_out/ncu_cl.log 2>&1; echo ncu=$?
for f in F2 KVL; do python bench.py --workload config3 --form $f --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/bench_c3_${f}_adam.json 2>&1; echo $f=$?; done
python bench.py --workload config1 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/bench_c1_KVL_adam.json 2>&1
python bench.py --workload config3 --form KVL --steps 2000 --warmup 100 --no-cpu-baseline --no-gap > gpurun_out/bench_c3_KVL.json 2>&1
