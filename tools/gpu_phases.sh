#!/bin/bash
# Per-phase clock profile of the per-centre kernels (library built with make PHASES=1 into
# ab/phases.so): prints the forward / backward phase shares.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
cp ab/phases.so paper_2604_07276_b200/libnnmd_b200.so
NNMD_PROFILE_PHASES=1 timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/phases.log 2>&1
grep "nnmd phases" gpurun_out/phases.log | tail -2
tail -5 gpurun_out/phases.log
