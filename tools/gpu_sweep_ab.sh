# A/B of sweep-kernel builds on the default bench (measurement only), interleaved
B="python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-gap --no-e2e"
for rep in 1 2; do
for v in default paper_2406_13191_b200/lib/variants/*.so; do
  if [ "$v" = default ]; then out=$($B 2>/dev/null); else out=$(DCOPF_LIB=$v $B 2>/dev/null); fi
  echo "$(basename $v) $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],4))')"
done
done
