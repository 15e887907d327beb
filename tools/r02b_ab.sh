#!/bin/bash
# A/B round: fast parity subset, C4 knob A/B, C2 bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_fuzz.py ${EXTRA_TESTS} > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/ab_tests.log
timeout 900 python tools/ab_c4.py "$@" > gpurun_out/ab.log 2>&1; echo ab=$?
cat gpurun_out/ab.log | tail -12
if [ -z "$NO_C2" ]; then
timeout 600 python bench.py --no-cpu --no-c3 --no-c4 --steps 20 --warmup 5 > gpurun_out/ab_bench.log 2>&1; echo bench=$?
grep '^{' gpurun_out/ab_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('kernel_ms_per_step'))"
fi
