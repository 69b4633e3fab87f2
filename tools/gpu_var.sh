set -x
run() { env "$@" python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --no-gap --form ${FORM:-F2} 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', '%.4g' % d['value'], d['config']['kernel']['smem'])"; }
run X=1
run DCOPF_POOL_PAD=512
run DCOPF_RED_SEPARATE=1
run DCOPF_POOL_PAD=512 DCOPF_RED_SEPARATE=1
run DCOPF_LIB=paper_2406_13191_b200/lib/libdcopf_dual_ref.so
