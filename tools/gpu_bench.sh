set -x
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python bench.py --form F1 --no-cpu-baseline > gpurun_out/bench_F1.json 2>&1; echo f1=$?
python bench.py --workload config3 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1; echo c3=$?
python bench.py --workload config3 --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/bench_c3_adam.json 2>&1; echo c3a=$?
python bench.py --workload config1 --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/bench_c1_adam.json 2>&1; echo c1a=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-gap > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
