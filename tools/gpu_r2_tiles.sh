# round 2: tiling A/B (instances per lane V, parts per tile C) + ncu of the sweep kernel
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
B --batch 8192 --tile 2,1 > gpurun_out/t_8192_21.json 2>&1; echo a=$?
B --batch 8192 --tile 4,2 > gpurun_out/t_8192_42.json 2>&1; echo b=$?
B --batch 8192 --tile 4,1 > gpurun_out/t_8192_41.json 2>&1; echo c=$?
B --batch 1024 --tile 2,8 > gpurun_out/t_1024_28.json 2>&1; echo d=$?
B --batch 1024 --tile 4,16 > gpurun_out/t_1024_416.json 2>&1; echo e=$?
B --batch 1024 --tile 2,16 > gpurun_out/t_1024_216.json 2>&1; echo f=$?
B --batch 2048 --tile 2,4 > gpurun_out/t_2048_24.json 2>&1; echo g=$?
B --batch 4096 --tile 2,2 > gpurun_out/t_4096_22.json 2>&1; echo h=$?
N() { timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 -o gpurun_out/$1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-gap "${@:2}" > gpurun_out/$1.log 2>&1; echo $1=$?; }
N ncu_t21 --tile 2,1
N ncu_t42 --tile 4,2
