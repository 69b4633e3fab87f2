# measurement only: chunk choices for F1 and KVL on config 4
run() { form=$1; shift; out=$(env "$@" python bench.py --form $form --steps 100 --warmup 10 --no-cpu-baseline --no-gap --no-e2e 2>/dev/null); echo "$form $* :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["config"]["kernel"]["chunk"], d["config"]["kernel"]["ring_life"], d["config"]["kernel"]["smem"])' 2>/dev/null)"; }
run F1 DCOPF_X=default
for ch in 17 18 19 20; do run F1 DCOPF_CHUNK=$ch DCOPF_RING_LIFE=2; done
run KVL DCOPF_X=default
for ch in 34 36 40 44; do for life in 2 4; do run KVL DCOPF_CHUNK=$ch DCOPF_RING_LIFE=$life; done; done
