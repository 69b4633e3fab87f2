# measurement only: program-block prefetch depth of the sweep producer (DCOPF_PREFETCH) per form
run() { form=$1; shift; out=$(env "$@" python bench.py --form $form --steps 100 --warmup 10 --no-cpu-baseline --no-gap --no-e2e 2>/dev/null); echo "$form $* :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["config"]["kernel"]["chunk"], d["config"]["kernel"]["ring_life"], d["config"]["kernel"]["smem"])' 2>/dev/null)"; }
for form in F2 KVL F1; do
  run $form DCOPF_X=default
  run $form DCOPF_PREFETCH=1
  run $form DCOPF_PREFETCH=3
done
