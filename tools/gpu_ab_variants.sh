# A/B of library builds on a bench line: build variants with extra nvcc flags,
# e.g.  bash /path/mkvar  (see tools/README.md), then on the GPU box:
#   bash tools/gpu_ab_variants.sh "--tile 4,2" base variantA variantB ...
# (base = the in-tree library; a variant NAME = paper_2406_13191_b200/lib/variants/NAME.so)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
args=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib="DCOPF_LIB=paper_2406_13191_b200/lib/variants/$v.so"; fi
    env $lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e $args \
      > gpurun_out/ab_${v}_$rep.json 2>&1; echo $v=$?
  done
done
