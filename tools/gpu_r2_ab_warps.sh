# A/B: consumer warps of the V = 2 sweep (19 default; variants 15 and 17) on the Adam lines
O=gpurun_out/ab_warps
mkdir -p $O
V=paper_2406_13191_b200/lib/variants
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
for rep in 1 2; do
B kvl_adam_w19_$rep --workload config4b --form KVL --opt adam --steps 20 --warmup 5
DCOPF_LIB=$V/w15.so B kvl_adam_w15_$rep --workload config4b --form KVL --opt adam --steps 20 --warmup 5
DCOPF_LIB=$V/w17.so B kvl_adam_w17_$rep --workload config4b --form KVL --opt adam --steps 20 --warmup 5
B f2_adam_w19_$rep --workload config4b --form F2 --opt adam --steps 20 --warmup 5
DCOPF_LIB=$V/w15.so B f2_adam_w15_$rep --workload config4b --form F2 --opt adam --steps 20 --warmup 5
DCOPF_LIB=$V/w17.so B f2_adam_w17_$rep --workload config4b --form F2 --opt adam --steps 20 --warmup 5
done
