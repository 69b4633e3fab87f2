# A/B of library builds (paper_2406_13191_b200/lib/variants/NAME.so vs the current build) on bench lines,
# alternating builds, K = 100:  bash tools/gpu_r2_ab_lib.sh NAME [NAME...]
O=gpurun_out/ab_lib
rm -rf $O
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo build=$?
V=paper_2406_13191_b200/lib/variants
B() { lib=$1; shift; if [ -n "$lib" ]; then export DCOPF_LIB=$lib; else unset DCOPF_LIB; fi
      timeout 600 python bench.py --no-cpu-baseline --no-gap --no-e2e --steps 100 --warmup 5 "$@"; }
for rep in 1 2; do
  for v in cur "$@"; do
    if [ $v = cur ]; then L=""; else L="$V/$v.so"; fi
    B "$L" --workload config4b --form KVL --opt adam > $O/${v}_kvl_adam_$rep.json 2>/dev/null
    B "$L" --workload config4b --form F2 --opt adam > $O/${v}_f2_adam_$rep.json 2>/dev/null
    B "$L" > $O/${v}_f2_$rep.json 2>/dev/null
    B "$L" --form KVL > $O/${v}_kvl_$rep.json 2>/dev/null
    B "$L" --form F1 > $O/${v}_f1_$rep.json 2>/dev/null
    B "$L" --steps 20 > $O/${v}_f2k20_$rep.json 2>/dev/null
  done
done
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compact.py -x -q -k "split or strong_scaling or compaction or config4 or batch or optimizer or kvl or f1" > $O/tests.log 2>&1; echo tests=$?; tail -1 $O/tests.log
for f in $O/*_[12].json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['roofline']['frac'],3), 'ch', d['config']['kernel']['chunk'])"; done
