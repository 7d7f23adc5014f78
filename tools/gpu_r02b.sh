#!/bin/bash
# Round-2 evidence trip: GPU suite, smoke, bench (rc 6 headline + rc 4 / rc 8 lines), the
# reference arm, virtual-rank strong-scaling estimate, sweep harness, ncu launch list and
# --set full captures of the HBM-bound / route / fitting kernels and of both per-centre
# kernels.  Everything lands in gpurun_out/ with the $TAG prefix.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${TAG:-r02b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/${T}_bench_reference.log 2>&1
for rc in 4 8; do
  timeout 600 python bench.py --steps 10 --warmup 3 --rc $rc --no-cpu-baseline > gpurun_out/${T}_bench_rc$rc.log 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --precision tf32 --no-cpu-baseline > gpurun_out/${T}_bench_tf32.log 2>&1
timeout 300 python tools/virtual_ranks.py > gpurun_out/${T}_virtual_ranks.json 2> gpurun_out/${T}_virtual_ranks.err
if [ -z "${NO_SWEEP:-}" ]; then
timeout 900 python -m paper_2604_07276_b200.sweep --mode strong --ranks 1 2 4 8 --out gpurun_out/${T}_sweep_strong > gpurun_out/${T}_sweep_strong.log 2>&1
timeout 900 python -m paper_2604_07276_b200.sweep --mode weak --ranks 1 2 4 8 --out gpurun_out/${T}_sweep_weak > gpurun_out/${T}_sweep_weak.log 2>&1
for rc in 4 8; do
timeout 900 python -m paper_2604_07276_b200.sweep --mode strong --ranks 1 8 --rc $rc --out gpurun_out/${T}_sweep_rc$rc > gpurun_out/${T}_sweep_rc$rc.log 2>&1
done
fi
if [ -z "${NO_NCU:-}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_neighbors|k_force_gather|k_route|k_merge|k_energy_virial|k_fit_tma|k_fit_out|k_fit_splitk|k_dd_members|k_cell_fill|k_finalize" -c 26 \
  -o gpurun_out/${T}_hbm python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${T}_ncu_hbm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_centre_(forward|backward)" -c 2 \
  -o gpurun_out/${T}_centre python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${T}_ncu_centre.log 2>&1
fi
# summarise on the box (reports exceed the 64 MiB copy-back limit): launch list, key
# metrics per captured kernel, per-line stalls of the backward; then drop the reports
python tools/summarize_ncu.py ${T} > gpurun_out/${T}_summarize.log 2>&1
cp profiles/${T}_launches.txt profiles/${T}_ncu.txt profiles/${T}_ncu.json profiles/ncu_latest.json gpurun_out/ 2>/dev/null
[ -f gpurun_out/${T}_centre.ncu-rep ] && python tools/ncu_lines.py gpurun_out/${T}_centre.ncu-rep 60 k_centre_backward > gpurun_out/${T}_bwd_lines.txt 2>&1
[ -f gpurun_out/${T}_centre.ncu-rep ] && python tools/ncu_lines.py gpurun_out/${T}_centre.ncu-rep 40 k_centre_forward > gpurun_out/${T}_fwd_lines.txt 2>&1
rm -f gpurun_out/*.ncu-rep gpurun_out/${T}_launches.csv
du -sh gpurun_out; ls gpurun_out | head -80
