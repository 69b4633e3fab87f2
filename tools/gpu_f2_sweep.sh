# measurement only: F2 chunk / ring life near the chosen point
run() { out=$(env "$@" python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-gap --no-e2e 2>/dev/null); echo "F2 $* :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["config"]["kernel"]["chunk"], d["config"]["kernel"]["ring_life"], d["config"]["kernel"]["smem"])' 2>/dev/null)"; }
run DCOPF_X=default
run DCOPF_CHUNK=26 DCOPF_RING_LIFE=3
run DCOPF_CHUNK=27 DCOPF_RING_LIFE=2
run DCOPF_CHUNK=28 DCOPF_RING_LIFE=1
run DCOPF_CHUNK=30 DCOPF_RING_LIFE=1
run DCOPF_CHUNK=25 DCOPF_RING_LIFE=3
run DCOPF_X=default
