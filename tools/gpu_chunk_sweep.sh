# measurement only: schedule chunk / ring-life choices on the default bench (config 4, F2)
B="python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-gap --no-e2e"
run() { out=$(env "$@" $B 2>/dev/null); echo "$* :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["config"]["kernel"]["chunk"], d["config"]["kernel"]["ring_life"], d["config"]["kernel"]["smem"])' 2>/dev/null)"; }
run DCOPF_X=default
for ch in 22 24 26 28 30; do for life in 2 4 6; do run DCOPF_CHUNK=$ch DCOPF_RING_LIFE=$life; done; done
run DCOPF_X=default
