# PTDF dense path: launch list + ncu --set full of the two fused GEMMs (measurement only)
set -x
mkdir -p gpurun_out/ptdf
B="python bench.py --workload config4b --form PTDF --steps 3 --warmup 3 --no-cpu-baseline --no-gap --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 40 --csv --log-file gpurun_out/ptdf/launches.csv $B > /dev/null 2>&1; echo l=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dgemm -s 12 -c 2 -o gpurun_out/ptdf/ncu_dgemm $B > /dev/null 2>&1; echo n=$?
ls -la gpurun_out/ptdf
