#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k nccl > gpurun_out/nccl_test.log 2>&1; echo "rc=$?" >> gpurun_out/nccl_test.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun.log 2>&1; echo "rc=$?" >> gpurun_out/torchrun.log
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 --ref-sample 64 > gpurun_out/ref_arm.log 2>&1; echo "rc=$?" >> gpurun_out/ref_arm.log
