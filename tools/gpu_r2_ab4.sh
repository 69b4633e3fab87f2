# round 2: consumer-warp count A/B (register budget vs warps) for V = 2 and V = 4
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
V=paper_2406_13191_b200/lib/variants
B --tile 2,1 > gpurun_out/ab5_main21.json 2>&1
B --tile 4,2 > gpurun_out/ab5_main42.json 2>&1
DCOPF_LIB=$V/w2n17.so B --tile 2,1 > gpurun_out/ab5_n17_21.json 2>&1
DCOPF_LIB=$V/w4n14.so B --tile 4,2 > gpurun_out/ab5_n14_42.json 2>&1
DCOPF_LIB=$V/w4n13.so B --tile 4,2 > gpurun_out/ab5_n13_42.json 2>&1
B --tile 4,2 --form KVL > gpurun_out/ab5_main42_kvl.json 2>&1
B --tile 2,1 --form KVL > gpurun_out/ab5_main21_kvl.json 2>&1
DCOPF_LIB=$V/w4n14.so B --tile 4,2 --form KVL > gpurun_out/ab5_n14_42_kvl.json 2>&1
B --batch 1024 --tile 4,16 > gpurun_out/ab5_main_1024_416.json 2>&1
B --batch 1024 --tile 2,8 > gpurun_out/ab5_main_1024_28.json 2>&1
echo done
