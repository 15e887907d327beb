cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 ${TESTS:-} > gpurun_out/k4r_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/k4r_tests.log
timeout 600 python tools/ab_c4.py "{'k4_mode': 0}" "{'k4_mode': 1}" > gpurun_out/k4r_ab.log 2>&1; echo ab=$?
cat gpurun_out/k4r_ab.log | tail -8
timeout 600 python bench.py --no-cpu --no-c3 --no-c4 --steps 20 --warmup 5 > gpurun_out/k4r_bench.log 2>&1; echo bench=$?
grep '^{' gpurun_out/k4r_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('kernel_ms_per_step'))"
