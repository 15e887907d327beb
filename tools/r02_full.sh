cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1500 python -m pytest -q tests -m gpu > gpurun_out/full_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/full_tests.log
timeout 900 python bench.py --no-cpu --no-c3 --steps 5 --warmup 3 > gpurun_out/full_bench.log 2>&1; echo bench=$?
grep '^{' gpurun_out/full_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); p=d['partitioned']; print({k: (p[k]['ms_per_wave'], p[k]['e2e']['value']) for k in ('k2','k3')}); print(json.dumps({k: d['c4'][k]['ms_per_batch'] for k in ('k2','k3')}))"
