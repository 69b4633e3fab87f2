# A/B of PTDF GEMM-path builds, plain and Adam (measurement only)
for opt in "" "--opt adam --alpha 5 --decay inv:200"; do
B="python bench.py --workload config4b --form PTDF $opt --steps 20 --warmup 3 --no-cpu-baseline --no-gap --no-e2e"
for v in default paper_2406_13191_b200/lib/variants/*.so; do
  if [ "$v" = default ]; then out=$($B 2>/dev/null); else out=$(DCOPF_LIB=$v $B 2>/dev/null); fi
  echo "[$opt] $(basename $v) $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],2), round(d["roofline"]["frac"],3))')"
done
done
