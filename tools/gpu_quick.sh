#!/bin/bash
# Quick GPU iteration: parity tests, a short bench (no CPU baseline) and the per-phase
# cycle profile of the centre kernels.  Logs under gpurun_out/.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/q_bench.log
if [ -n "${PHASES:-}" ]; then
  # phase counters are compiled out of production builds: rebuild this box's copy with them
  make -C paper_2604_07276_b200/csrc PHASES=1 -B -j8 > /dev/null 2>&1
  NNMD_PROFILE_PHASES=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline ${BENCH_ARGS:-} 2>&1 | grep phases | tail -2 > gpurun_out/q_phases.log
fi
tail -3 gpurun_out/q_pytest.log
python - <<'PY'
import json
for ln in open("gpurun_out/q_bench.log"):
    if ln.startswith("{"):
        d = json.loads(ln)
        print("ms/step %.3f  e2e %.2f steps/s  kernels %s" % (d["ms_per_step"], d["e2e"]["value"],
              {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}))
PY
[ -n "${PHASES:-}" ] && cat gpurun_out/q_phases.log
