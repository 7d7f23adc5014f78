#!/bin/bash
# A/B timing of experiment switches: bench (no CPU baseline) once per NNMD_FLAGS value.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for f in ${FLAGS_LIST:-0 1 2 3}; do
  NNMD_FLAGS=$f timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); k = d['kernel_ms_per_step']
        print('flags=$f ms/step %.3f fwd %.3f bwd %.3f fit %.3f' % (d['ms_per_step'], k['centre_forward'], k['centre_backward'], k['fit']))
"
done
