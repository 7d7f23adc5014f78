#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
python tools/diag_acc.py > gpurun_out/diag.log 2>&1
timeout 300 python -m pytest tests/test_gpu_gemm.py -q > gpurun_out/pytest_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemm.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s > gpurun_out/pytest_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_parity.log
