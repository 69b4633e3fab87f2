# A/B of PTDF launch options (measurement only): env settings in turn
B="python bench.py --workload config4b --form PTDF --steps 20 --warmup 3 --no-cpu-baseline --no-gap --no-e2e"
for v in "DCOPF_PTDF_SPLIT=1" "DCOPF_PTDF_SPLIT=2" "DCOPF_PTDF_GROUP=4" "DCOPF_PTDF_GROUP=16" "DCOPF_PTDF_GROUP=40"; do
  out=$(env $v $B 2>/dev/null)
  echo "$v $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],2), round(d["roofline"]["achieved"],2), round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])')"
done
