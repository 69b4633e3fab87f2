# round 2: ncu of the default sweep (V2C1) and of the optimiser (Adam) sweep; Adam bench lines
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e "$@"; }
B --workload config4b --form KVL --opt adam --steps 20 --warmup 5 > gpurun_out/prof_kvl_adam.json 2>&1
B --workload config4b --form F2 --opt adam --steps 20 --warmup 5 > gpurun_out/prof_f2_adam.json 2>&1
B --workload config4 --form F1 --steps 20 --warmup 5 > gpurun_out/prof_f1.json 2>&1
N() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/$1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap "${@:2}" > gpurun_out/$1.log 2>&1; echo $1=$?; }
N prof_ncu_f2 
N prof_ncu_kvl_adam --workload config4b --form KVL --opt adam
echo done
