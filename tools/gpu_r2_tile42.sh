O=gpurun_out/adam42
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
B() { name=$1; shift; timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B kvl_adam_42 --workload config4b --form KVL --opt adam --steps 20 --warmup 5 --tile 4,2
B f2_adam_42 --workload config4b --form F2 --opt adam --steps 20 --warmup 5 --tile 4,2
B kvl_adam_21 --workload config4b --form KVL --opt adam --steps 20 --warmup 5 --tile 2,1
B kvl_42 --workload config4b --form KVL --steps 20 --warmup 5 --tile 4,2
B f2_42 --workload config4 --steps 20 --warmup 5 --tile 4,2
