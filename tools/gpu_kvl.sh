set -x
run() { env "$@" python bench.py --form KVL --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', '%.4g' % d['value'], d['config']['kernel']['chunk'], d['config']['kernel']['smem'], d['config']['kernel']['ring_life'])" || tail -2 /tmp/o.txt; }
run X=1
for ch in 24 28 36 40; do for life in 2 4; do run DCOPF_CHUNK=$ch DCOPF_RING_LIFE=$life; done; done
run DCOPF_DEBUG_MODE=1
