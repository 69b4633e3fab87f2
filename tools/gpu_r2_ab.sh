# round 2: A/B of library builds on the config-4 F2 bench (DCOPF_LIB = variant .so)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
for rep in 1 2; do
DCOPF_LIB=paper_2406_13191_b200/lib/variants/r1.so B > gpurun_out/ab_r1_$rep.json 2>&1; echo r1=$?
B --tile 2,1 > gpurun_out/ab_cur21_$rep.json 2>&1; echo cur=$?
DCOPF_LIB=paper_2406_13191_b200/lib/variants/susp.so B --tile 2,1 > gpurun_out/ab_susp21_$rep.json 2>&1; echo susp=$?
DCOPF_LIB=paper_2406_13191_b200/lib/variants/susp.so B --tile 4,2 > gpurun_out/ab_susp42_$rep.json 2>&1; echo susp42=$?
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/ncu_r1 env DCOPF_LIB=paper_2406_13191_b200/lib/variants/r1.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > gpurun_out/ncu_r1.log 2>&1; echo ncu=$?
