# measurement only: the three sparse forms on config 4 (chunk / ring life chosen by the library)
for form in F2 F1 KVL; do
  out=$(python bench.py --form $form --steps 100 --warmup 10 --no-cpu-baseline --no-gap --no-e2e 2>/dev/null)
  echo "$form :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), d["config"]["kernel"]["chunk"], d["config"]["kernel"]["ring_life"], d["config"]["kernel"]["smem"], round(d["roofline"]["frac"],4))')"
done
