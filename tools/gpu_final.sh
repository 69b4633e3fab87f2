# round-end evidence: benches (JSON lines), launch list, ncu captures of the top kernels
set -x
mkdir -p gpurun_out/final
python bench.py > gpurun_out/final/bench_config4_F2.json 2> gpurun_out/final/bench_config4_F2.err; echo b1=$?
python bench.py --form F1 --no-cpu-baseline > gpurun_out/final/bench_config4_F1.json 2>&1; echo b2=$?
python bench.py --form KVL --no-cpu-baseline > gpurun_out/final/bench_config4_KVL.json 2>&1; echo b3=$?
python bench.py --workload config3 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final/bench_config3_F2.json 2>&1
python bench.py --workload config3 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final/bench_config3_KVL_adam.json 2>&1
python bench.py --workload config3 --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final/bench_config3_F2_adam.json 2>&1
python bench.py --workload config1 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final/bench_config1_KVL_adam.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_reference.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/final/launches_config4_F2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gap > /dev/null 2>&1; echo l=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/final/ncu_k_sweep_config4_F2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > /dev/null 2>&1; echo n1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/final/ncu_k_sweep_config4_KVL python bench.py --form KVL --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > /dev/null 2>&1; echo n2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cluster -c 1 -o gpurun_out/final/ncu_k_cluster_config3_F2 python bench.py --workload config3 --steps 100 --warmup 400 --no-cpu-baseline --no-e2e --no-gap > /dev/null 2>&1; echo n3=$?
python bench.py --workload config4b --form PTDF --steps 30 --warmup 3 --no-gap > gpurun_out/final/bench_config4b_PTDF.json 2> gpurun_out/final/bench_config4b_PTDF.err; echo b_ptdf=$?
python bench.py --workload config4b --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/final/bench_config4b_F2.json 2>&1; echo b4b=$?
