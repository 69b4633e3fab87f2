# ncu --set full captures of the kernels changed after the final evidence run (KVL plain, F2 + Adam), summarised on the box
O=gpurun_out/ncu_refresh
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
OBJ=paper_2406_13191_b200/lib/obj/dcopf_dual.cu.o
N() { tag=$1; kern=$2; shift 2; timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o $O/ncu_$tag python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap "$@" > $O/ncu_$tag.log 2>&1; echo ncu_$tag=$?
      python tools/ncu_hotlines.py $O/ncu_$tag.ncu-rep $kern $OBJ 40 > $O/ncu_${tag}_summary.txt 2>&1
      ncu -i $O/ncu_$tag.ncu-rep --page raw --csv > $O/ncu_${tag}_raw.csv 2>/dev/null
      rm -f $O/ncu_$tag.ncu-rep; }
N config4_KVL _ZN5dcopf7k_sweepILi2ELb0ELi19ELb1ELb0ELi2EEEvNS_9SweepArgsE --form KVL
N config4b_F2_adam _ZN5dcopf7k_sweepILi0ELb0ELi19ELb1ELb1ELi2EEEvNS_9SweepArgsE --workload config4b --form F2 --opt adam
