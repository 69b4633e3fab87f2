# round 2: F2 prefetch depth P = 1 vs 2 (P = 1 frees shared memory for larger chunks)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
V=paper_2406_13191_b200/lib/variants
for t in 4,2 2,1; do
B --tile $t > gpurun_out/ab6_main_$t.json 2>&1
DCOPF_LIB=$V/p1.so B --tile $t > gpurun_out/ab6_p1_$t.json 2>&1
done
B --batch 1024 > gpurun_out/ab6_main_1024.json 2>&1
DCOPF_LIB=$V/p1.so B --batch 1024 > gpurun_out/ab6_p1_1024.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/ncu_ab6_42 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --tile 4,2 > gpurun_out/ncu_ab6_42.log 2>&1; echo ncu=$?
echo done
