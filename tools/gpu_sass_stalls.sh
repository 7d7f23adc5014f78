#!/bin/bash
# Per-SASS-instruction stall samples of one k_centre_backward launch (source page, CSV).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
K=${KERNEL:-k_centre_backward}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 \
  -o gpurun_out/sass_stalls python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/sass_stalls_ncu.log 2>&1
ncu -i gpurun_out/sass_stalls.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_stalls.csv 2>&1
gzip -f gpurun_out/sass_stalls.csv
rm -f gpurun_out/sass_stalls.ncu-rep
ls -la gpurun_out | head
