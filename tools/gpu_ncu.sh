#!/bin/bash
# ncu evidence: launch list (all kernels of a short bench) + full capture of the top kernels.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${TAG:-r01}
PREC=${PREC:-fp32}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --precision $PREC > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_centre_backward -c 1 \
  -o gpurun_out/${TAG}_bwd python bench.py --steps 1 --warmup 0 --no-cpu-baseline --precision $PREC > gpurun_out/${TAG}_ncu_bwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_neighbors|k_force_gather|k_centre_forward" -c 3 \
  -o gpurun_out/${TAG}_misc python bench.py --steps 1 --warmup 0 --no-cpu-baseline --precision $PREC > gpurun_out/${TAG}_ncu_misc.log 2>&1
ls -la gpurun_out
