# the remaining bench lines of profiles/bench_r1_final on the final build
mkdir -p gpurun_out/final7
python bench.py --workload config4b --form KVL --no-cpu-baseline > gpurun_out/final7/bench_config4b_KVL.json 2>/dev/null
python bench.py --workload config4b --form KVL --opt adam --alpha 0.1 --no-cpu-baseline > gpurun_out/final7/bench_config4b_KVL_adam.json 2>/dev/null
python bench.py --workload config4b --opt adam --alpha 0.1 --no-cpu-baseline > gpurun_out/final7/bench_config4b_F2_adam.json 2>/dev/null
python bench.py --workload config4b --no-cpu-baseline > gpurun_out/final7/bench_config4b_F2.json 2>/dev/null
python bench.py --workload config3 --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final7/bench_config3_F2_adam.json 2>/dev/null
python bench.py --workload config1 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final7/bench_config1_KVL_adam.json 2>/dev/null
echo done
