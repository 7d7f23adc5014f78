#!/bin/bash
# compute-sanitizer racecheck + memcheck of smoke() (300 atoms, 2 DD ranks, every product
# kernel of a step) and of one rc = 4 multi-centre-unit evaluation.  Logs under gpurun_out/.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${TAG:-r02c}
mkdir -p gpurun_out
cat > /tmp/pack_case.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2604_07276_b200 as nb
box, pos, sp = nb.synth_system(300, 0.1, 0.9, 3)
m = nb.init_model(nb.paper_spec(4.0), 1)
r = nb.DeviceEvaluator(m, n_ranks=2).compute(pos, sp, box)
print("pack case E", r["energy"])
PY
for tool in racecheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py > gpurun_out/${T}_${tool}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_${tool}_smoke.log
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python /tmp/pack_case.py > gpurun_out/${T}_${tool}_pack.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_${tool}_pack.log
done
tail -n 4 gpurun_out/${T}_*check_*.log
