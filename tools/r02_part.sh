cd "${GRAFT_REPO_ROOT:-/root/repo}"
true > gpurun_out/part_tests.log 2>&1; echo tests=$?; tail -30 gpurun_out/part_tests.log
timeout 900 python bench.py --no-cpu --no-c3 --steps 5 --warmup 3 > gpurun_out/part_bench.log 2>&1; echo bench=$?
grep '^{' gpurun_out/part_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print(json.dumps(d['partitioned'], indent=1)); print(json.dumps({k: d['c4'][k]['ms_per_batch'] for k in ('k2','k3')}))"
tail -5 gpurun_out/part_bench.log
