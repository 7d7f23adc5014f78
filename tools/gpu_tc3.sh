#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -s > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
for p in ${PRECS:-fp32}; do timeout 300 python bench.py --steps 5 --warmup 3 --precision $p --no-cpu-baseline > gpurun_out/bench_$p.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$p.log; done
