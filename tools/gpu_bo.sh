set -x
run() { env "$@" python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form ${FORM:-F2} > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', '%.4g' % d['value'])" || tail -3 /tmp/o.txt; }
L=paper_2406_13191_b200/lib
for f in F2 F1; do
FORM=$f run X=1
for b in 8 16 64; do FORM=$f run DCOPF_LIB=$L/libdcopf_dual_bo$b.so; done
done
