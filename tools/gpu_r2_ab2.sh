set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
for rep in 1 2; do
DCOPF_LIB=paper_2406_13191_b200/lib/variants/r1.so B > gpurun_out/ab2_r1_$rep.json 2>&1; echo r1=$?
B --tile 2,1 > gpurun_out/ab2_cur21_$rep.json 2>&1; echo cur=$?
DCOPF_LIB=paper_2406_13191_b200/lib/variants/unsplit.so B --tile 2,1 > gpurun_out/ab2_unsplit21_$rep.json 2>&1; echo unsplit=$?
B --tile 4,2 > gpurun_out/ab2_cur42_$rep.json 2>&1; echo cur42=$?
done
