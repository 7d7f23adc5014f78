#!/bin/bash
# Stress of the TMA-fed fitting net: repeated GPU suites and long benches at rc 4 / 6 / 8
# (every step runs the TMA fit GEMMs); any fault shows up as a non-zero rc.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_pytest_$i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest_$i.log; done
for rc in 6 4 6 8 6; do
  timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --rc $rc > gpurun_out/t_bench_rc$rc.log 2>&1; echo "bench rc=$?" >> gpurun_out/t_bench_rc$rc.log
  tail -n 1 gpurun_out/t_bench_rc$rc.log >> gpurun_out/t_summary.log
done
grep -h "pytest rc" gpurun_out/t_pytest_*.log >> gpurun_out/t_summary.log
