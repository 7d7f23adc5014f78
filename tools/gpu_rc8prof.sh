cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
make -C paper_2604_07276_b200/csrc PHASES=1 -B -j8 > /dev/null 2>&1
NNMD_PROFILE_PHASES=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --rc 8 2>&1 | grep phases > gpurun_out/rc8_phases.log
make -C paper_2604_07276_b200/csrc -B -j8 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_centre_(forward|backward)" -c 2 \
  -o gpurun_out/rc8_centre python bench.py --steps 1 --warmup 0 --no-cpu-baseline --rc 8 > gpurun_out/rc8_ncu.log 2>&1
python tools/ncu_lines.py gpurun_out/rc8_centre.ncu-rep 40 k_centre_forward > gpurun_out/rc8_fwd_lines.txt 2>&1
python tools/ncu_lines.py gpurun_out/rc8_centre.ncu-rep 40 k_centre_backward > gpurun_out/rc8_bwd_lines.txt 2>&1
rm -f gpurun_out/*.ncu-rep
