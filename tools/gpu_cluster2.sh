set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "cluster or kvl or optimizer or first_hit or config0 or divergence" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for w in config1 config3; do for f in F2 KVL; do python bench.py --workload $w --form $f --steps 2000 --warmup 100 --no-cpu-baseline --no-e2e --no-gap > /tmp/o.txt 2>&1; grep '^{' /tmp/o.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $f', '%.4g it/s' % d['value'], '%.3f us/it' % (1e3*d['ms_per_step']))"; done; done
