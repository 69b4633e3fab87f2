set -x
run() { env "$@" python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form ${FORM:-F2} > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', '%.4g' % d['value'], d['config']['kernel']['chunk'], d['config']['kernel']['smem'])" || tail -3 /tmp/o.txt; }
run X=1
run DCOPF_COST=30,12,50,35,12,25
run DCOPF_COST=30,12,90,35,12,25
run DCOPF_COST=20,16,70,25,16,25
run DCOPF_COST=40,8,70,45,8,25
run DCOPF_CHUNK=20 DCOPF_RING_LIFE=2
run DCOPF_CHUNK=20 DCOPF_RING_LIFE=4
FORM=F1 run X=1
FORM=F1 run DCOPF_COST=30,12,70,35,12,25
FORM=F1 run DCOPF_COST=30,30,60,35,30,25
FORM=F1 run DCOPF_CHUNK=12 DCOPF_RING_LIFE=2
