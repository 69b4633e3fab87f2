set -x
run() { env "$@" python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form ${FORM:-F2} > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', '%.4g' % d['value'])" || tail -3 /tmp/o.txt; }
for f in F2 F1; do for sp in 1.0 1.15 1.25 1.4 1.6; do FORM=$f run DCOPF_SMSP_SPEED=$sp; done; done
