#!/bin/bash
# N=2 bench path exercised on one GPU (both ranks on cuda:0, gloo): checks the
# torchrun path of bench.py still completes; its timings are not measurements
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TH_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu \
  > gpurun_out/two_rank.log 2>&1; echo two_rank=$?
grep '^{' gpurun_out/two_rank.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['e2e']['value'], d['partitioned']['k3']['interconnect']['bytes_per_hop'])"
tail -3 gpurun_out/two_rank.log | cut -c1-300
