# round-end evidence (no ncu): smoke, the GPU suite, the bench lines of every form / path
set -x
mkdir -p gpurun_out/final2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final2/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/final2/pytest_gpu.log
python bench.py > gpurun_out/final2/bench_config4_F2.json 2> gpurun_out/final2/bench_config4_F2.err; echo b1=$?
python bench.py --form F1 --no-cpu-baseline > gpurun_out/final2/bench_config4_F1.json 2>&1; echo b2=$?
python bench.py --form KVL --no-cpu-baseline > gpurun_out/final2/bench_config4_KVL.json 2>&1; echo b3=$?
python bench.py --workload config3 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final2/bench_config3_F2.json 2>&1
python bench.py --workload config3 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline > gpurun_out/final2/bench_config3_KVL_adam.json 2>&1
python bench.py --workload config3 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100 > gpurun_out/final2/bench_config3_PTDF_adam_inv200.json 2>&1
python bench.py --workload config4b --form PTDF --steps 30 --warmup 3 > gpurun_out/final2/bench_config4b_PTDF.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final2/bench_reference.json 2>&1
python bench.py --workload config4b --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/final2/bench_config4b_PTDF_adam_inv200.json 2>&1
