# A/B: optimiser-state L2 prefetch (variant nopf without it); the B = 1 dense path with Adam on the
# single-read step against the two-pass kernels
set -x
O=gpurun_out/ab_adam
mkdir -p $O
V=paper_2406_13191_b200/lib/variants
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
for rep in 1 2; do
B kvl_adam_pf$rep --workload config4b --form KVL --opt adam --steps 20 --warmup 5
DCOPF_LIB=$V/nopf.so B kvl_adam_nopf$rep --workload config4b --form KVL --opt adam --steps 20 --warmup 5
B f2_adam_pf$rep --workload config4b --form F2 --opt adam --steps 20 --warmup 5
DCOPF_LIB=$V/nopf.so B f2_adam_nopf$rep --workload config4b --form F2 --opt adam --steps 20 --warmup 5
done
timeout 600 python bench.py --workload config3 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100 --no-cpu-baseline > $O/bench_c3_adam_fused.json 2>$O/e1.err; echo c3f=$?
DCOPF_PTDF_FUSED=0 timeout 600 python bench.py --workload config3 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100 --no-cpu-baseline > $O/bench_c3_adam_2pass.json 2>$O/e2.err; echo c32=$?
timeout 900 python -m pytest tests/test_gpu_ptdf.py -x -q > $O/tests_ptdf.log 2>&1; echo tests=$?
echo done
