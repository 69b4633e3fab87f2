set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/ncu_sweep_f2_v9 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > gpurun_out/ncu_full1.log 2>&1; echo ncu1=$?
