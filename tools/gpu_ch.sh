set -x
run() { env "$@" python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form ${FORM:-F2} > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', '%.4g' % d['value'], d['config']['kernel']['chunk'], d['config']['kernel']['smem'])" || tail -3 /tmp/o.txt; }
for ch in 24 20 16 12; do run DCOPF_CHUNK=$ch DCOPF_RING_LIFE=2; done
run DCOPF_CHUNK=20 DCOPF_RING_LIFE=2 DCOPF_PREFETCH=3
run DCOPF_CHUNK=16 DCOPF_RING_LIFE=4
run DCOPF_CHUNK=24 DCOPF_RING_LIFE=2 DCOPF_DEBUG_MODE=1
run DCOPF_CHUNK=24 DCOPF_RING_LIFE=2 DCOPF_DEBUG_MODE=2
run DCOPF_CHUNK=16 DCOPF_RING_LIFE=2 DCOPF_DEBUG_MODE=1
run DCOPF_CHUNK=16 DCOPF_RING_LIFE=2 DCOPF_DEBUG_MODE=2
