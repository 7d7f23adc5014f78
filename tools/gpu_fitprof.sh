#!/bin/bash
# Clock breakdown of the TMA-fed fitting-net GEMMs (TG_PROF build of this box's copy).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
make -C paper_2604_07276_b200/csrc -B -j8 EXTRA=-DTG_PROF > /dev/null 2>&1
timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2>&1 | grep fit_tma | tail -6 > gpurun_out/fitprof.log
