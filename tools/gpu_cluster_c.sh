# measurement only: cluster size on config 3 (one instance)
for c in 16 8; do
  for form in F2 KVL; do
    out=$(DCOPF_CLUSTER=$c python bench.py --workload config3 --form $form --steps 2000 --warmup 100 --no-cpu-baseline --no-gap --no-e2e 2>/dev/null)
    echo "C=$c $form :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), "us", d["config"]["cluster_size"])' 2>/dev/null)"
  done
done
