# B = 1 dense path: the single-read step against the two-pass kernels
# (agreement at small K, parity subset, config-3 bench lines, launch list, one ncu --set full capture)
set -x
O=gpurun_out/fused
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
timeout 600 python tools/dbg_fused.py > $O/dbg.log 2>&1; echo dbg=$?
timeout 1200 python -m pytest tests/test_gpu_ptdf.py -q -x > $O/pytest.log 2>&1; echo tests=$?
B() { name=$1; shift; timeout 900 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo $name=$?; }
B c3_plain --workload config3 --form PTDF --steps 1000 --warmup 20 --no-cpu-baseline --no-gap
DCOPF_PTDF_FUSED=0 B c3_plain_2pass --workload config3 --form PTDF --steps 1000 --warmup 20 --no-cpu-baseline --no-gap
B c3_gdm --workload config3 --form PTDF --opt gdm --alpha 1e-3 --steps 1000 --warmup 20 --no-cpu-baseline --no-gap
B c1_plain --workload config1 --form PTDF --steps 1000 --warmup 20 --no-cpu-baseline --no-gap
DCOPF_PTDF_FUSED=0 B c1_plain_2pass --workload config1 --form PTDF --steps 1000 --warmup 20 --no-cpu-baseline --no-gap
B c3_adam --workload config3 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100 --no-cpu-baseline
DCOPF_PTDF_FUSED=0 B c3_adam_2pass --workload config3 --form PTDF --opt adam --alpha 5 --decay inv:200 --steps 2000 --warmup 100 --no-cpu-baseline
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3_ptdf.csv python bench.py --workload config3 --form PTDF --steps 20 --warmup 3 --no-cpu-baseline --no-gap --no-e2e > $O/ncu_launch.log 2>&1; echo launches=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -c 1 -o $O/ncu_fused python bench.py --workload config3 --form PTDF --steps 5 --warmup 3 --no-cpu-baseline --no-gap --no-e2e > $O/ncu_full.log 2>&1; echo ncu=$?
echo done
