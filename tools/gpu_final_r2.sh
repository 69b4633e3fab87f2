# round-2 evidence on a B200: smoke, the GPU suite, every bench line, the
# launch list of the default bench and ncu --set full captures of the sweep
set -x
O=${O:-gpurun_out/final}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo smoke=$?
timeout 3000 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo tests=$?
B() { name=$1; shift; timeout 1200 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B default
B driver --steps 20 --warmup 5
B reference --impl reference --steps 3 --warmup 1
B config4_KVL --form KVL --no-cpu-baseline --no-gap
B config4_F1 --form F1 --no-cpu-baseline --no-gap
for b in 4096 2048 1024; do
  B shard${b}_F2 --batch $b --no-cpu-baseline --no-gap --no-e2e --steps 50 --warmup 5
  B shard${b}_KVL --batch $b --form KVL --no-cpu-baseline --no-gap --no-e2e --steps 50 --warmup 5
  B shard${b}_F1 --batch $b --form F1 --no-cpu-baseline --no-gap --no-e2e --steps 50 --warmup 5
done
B config4b_KVL_adam --workload config4b --form KVL --opt adam --no-cpu-baseline
B config4b_F2_adam --workload config4b --form F2 --opt adam --no-cpu-baseline
B config4b_KVL_adagrad --workload config4b --form KVL --opt adagrad --no-cpu-baseline --no-gap
B config4_F2_K100 --steps 100 --warmup 5 --no-cpu-baseline --no-gap --no-e2e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -Ipaper_2406_13191_b200/csrc tools/fp64_fastpath_check.cu -o /tmp/fp64_fastpath_check > $O/check_build.log 2>&1
timeout 300 /tmp/fp64_fastpath_check 64 > $O/fp64_fastpath_check.json 2>&1; echo fastpath=$?
B config4b_PTDF --workload config4b --form PTDF --no-cpu-baseline --steps 20 --warmup 3
B config3_F2 --workload config3 --steps 2000 --warmup 100 --no-cpu-baseline
B config3_KVL_adam --workload config3 --form KVL --opt adam --alpha 0.1 --steps 2000 --warmup 100 --no-cpu-baseline
B config3_PTDF_adam --workload config3 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100 --no-cpu-baseline
B config3_PTDF --workload config3 --form PTDF --steps 1000 --warmup 20 --no-cpu-baseline --no-gap
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config4_F2.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e > $O/ncu_launch.log 2>&1; echo launches=$?
# each capture is summarised here (tools/ncu_hotlines.py: throughputs, stalls,
# hot source lines; the raw page as csv) and the .ncu-rep removed: gpurun
# copies back at most 64 MiB
OBJ=paper_2406_13191_b200/lib/obj/dcopf_dual.cu.o
N() { tag=$1; kern=$2; shift 2; timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o $O/ncu_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap "$@" > $O/ncu_$tag.log 2>&1; echo ncu_$tag=$?
      python tools/ncu_hotlines.py $O/ncu_$tag.ncu-rep $kern $OBJ 40 > $O/ncu_${tag}_summary.txt 2>&1
      ncu -i $O/ncu_$tag.ncu-rep --page raw --csv > $O/ncu_${tag}_raw.csv 2>/dev/null
      rm -f $O/ncu_$tag.ncu-rep; }
K2=_ZN5dcopf7k_sweepILi0ELb0ELi19ELb1ELb0ELi2EEEvNS_9SweepArgsE
N config4_F2 $K2
N config4_KVL _ZN5dcopf7k_sweepILi2ELb0ELi19ELb1ELb0ELi2EEEvNS_9SweepArgsE --form KVL
N shard1024_F2 $K2 --batch 1024
N config4b_KVL_adam _ZN5dcopf7k_sweepILi2ELb0ELi19ELb1ELb1ELi2EEEvNS_9SweepArgsE --workload config4b --form KVL --opt adam
N config4b_F2_adam _ZN5dcopf7k_sweepILi0ELb0ELi19ELb1ELb1ELi2EEEvNS_9SweepArgsE --workload config4b --form F2 --opt adam
N shard1024_F1 _ZN5dcopf7k_sweepILi1ELb0ELi19ELb1ELb0ELi2EEEvNS_9SweepArgsE --batch 1024 --form F1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_config3_PTDF.csv python bench.py --workload config3 --form PTDF --steps 20 --warmup 3 --no-cpu-baseline --no-gap --no-e2e > $O/ncu_launch_ptdf.log 2>&1; echo launches_ptdf=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 2 -o $O/ncu_k_fused_config3 python bench.py --workload config3 --form PTDF --steps 5 --warmup 3 --no-cpu-baseline --no-gap --no-e2e > $O/ncu_fused.log 2>&1; echo ncu_fused=$?
ncu -i $O/ncu_k_fused_config3.ncu-rep --page raw --csv > $O/ncu_k_fused_config3_raw.csv 2>/dev/null; rm -f $O/ncu_k_fused_config3.ncu-rep
du -sh $O
echo done
