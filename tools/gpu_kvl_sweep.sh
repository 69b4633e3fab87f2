# measurement only: KVL with one program-block stage, larger chunks
run() { out=$(env "$@" python bench.py --form KVL --steps 100 --warmup 10 --no-cpu-baseline --no-gap --no-e2e 2>/dev/null); echo "KVL $* :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["config"]["kernel"]["chunk"], d["config"]["kernel"]["ring_life"], d["config"]["kernel"]["smem"])' 2>/dev/null)"; }
run DCOPF_PREFETCH=1
for ch in 44 48 52 56; do for life in 2 4; do run DCOPF_PREFETCH=1 DCOPF_CHUNK=$ch DCOPF_RING_LIFE=$life; done; done
