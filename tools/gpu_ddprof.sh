# Line-level ncu profile of the DD-side kernels (neighbour lists, force gather) at C1
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_neighbors|k_force_gather" -c 3 \
  -o gpurun_out/dd_lines python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/dd_ncu.log 2>&1
python tools/ncu_lines.py gpurun_out/dd_lines.ncu-rep 40 "k_neighbors" > gpurun_out/nbr1_lines.txt 2>&1
python tools/ncu_lines.py gpurun_out/dd_lines.ncu-rep 40 "k_force_gather" > gpurun_out/gather_lines.txt 2>&1
ncu -i gpurun_out/dd_lines.ncu-rep --page details --csv > gpurun_out/dd_details.csv 2>&1
rm -f gpurun_out/*.ncu-rep
