#!/bin/bash
# Interleaved A/B timing of prebuilt library variants (ab/lib*.so, git-ignored): each
# round installs every variant in turn and runs a short bench, so box-to-box and
# run-to-run drift hits all variants alike.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
LIB=paper_2604_07276_b200/libnnmd_b200.so
cp $LIB ab/.orig.so
for round in $(seq ${ROUNDS:-3}); do
  for v in ab/lib*.so; do
    cp $v $LIB
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); k = d['kernel_ms_per_step']
        fit = sum(v for n, v in k.items() if 'fit' in n)
        nbr = sum(v for n, v in k.items() if 'neighbo' in n or 'nbr' in n)
        print('$v round $round ms/step %.3f fwd %.3f bwd %.3f fit %.3f nbr %.3f gather %.3f' % (d['ms_per_step'], k['centre_forward'], k['centre_backward'], fit, nbr, k.get('force_gather', 0)))
"
  done
done
cp ab/.orig.so $LIB
