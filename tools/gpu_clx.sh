set -x
run() { env "$@" python bench.py --workload ${W:-config3} --form ${FORM:-F2} --steps 2000 --warmup 100 --no-cpu-baseline --no-e2e --no-gap > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$* ${W:-config3} ${FORM:-F2}', '%.3f us/it' % (1e3*d['ms_per_step']), d['config']['cluster_size'], d['config']['kernel']['threads'])" || tail -3 /tmp/o.txt; }
L=paper_2406_13191_b200/lib
for f in F2 KVL; do
FORM=$f run X=1
FORM=$f run DCOPF_CLUSTER=8
FORM=$f run DCOPF_LIB=$L/libdcopf_dual_ct512.so
FORM=$f run DCOPF_LIB=$L/libdcopf_dual_ct512.so DCOPF_CLUSTER=8
done
W=config1 run X=1
W=config1 run DCOPF_CLUSTER=2
W=config1 run DCOPF_CLUSTER=8
W=config1 run DCOPF_LIB=$L/libdcopf_dual_ct512.so
