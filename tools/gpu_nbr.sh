set -x
DCOPF_CLUSTER_NBR=1 timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or kvl or large_single or optimizer or config0 or stopping or first_hit" 2>&1 | tail -3
run() { env "$@" python bench.py --workload ${W:-config3} --form ${FORM:-F2} --steps 2000 --warmup 100 --no-cpu-baseline --no-e2e --no-gap > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$* ${W:-config3} ${FORM:-F2}', '%.3f us/it' % (1e3*d['ms_per_step']), d['config']['cluster_size'])" || tail -3 /tmp/o.txt; }
for f in F2 KVL F1; do FORM=$f run X=1; FORM=$f run DCOPF_CLUSTER_NBR=1; done
W=config1 run X=1; W=config1 run DCOPF_CLUSTER_NBR=1
