set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
B() { timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e "$@"; }
V=paper_2406_13191_b200/lib/variants
for v in base l2a3 l2a5 l2a8; do
  if [ $v = base ]; then L=""; else L="DCOPF_LIB=$V/$v.so"; fi
  env $L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e --tile 2,1 > gpurun_out/ab8_${v}_21.json 2>&1
  env $L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e --tile 4,2 > gpurun_out/ab8_${v}_42.json 2>&1
  env $L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-gap --no-e2e --form KVL --tile 2,1 > gpurun_out/ab8_${v}_kvl21.json 2>&1
done
for t in "1024 2,8" "1024 4,16" "1024 2,16" "2048 2,4" "2048 4,8" "4096 2,2" "4096 4,4" "8192 4,2"; do
  set -- $t
  B --batch $1 --tile $2 > gpurun_out/ab8_b$1_${2/,/_}.json 2>&1
  B --batch $1 --tile $2 --form KVL > gpurun_out/ab8_kvl_b$1_${2/,/_}.json 2>&1
done
echo done
