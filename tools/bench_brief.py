#!/usr/bin/env python
"""Run bench.py (extra args passed through) and print ms/step and the per-centre kernel times."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = os.environ.get("TAG", "")
p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", *sys.argv[1:]],
                   capture_output=True, text=True)
line = [l for l in p.stdout.splitlines() if l.startswith("{") and '"metric"' in l]
if not line:
    print(tag, "bench failed:", (p.stdout + p.stderr)[-1500:])
    sys.exit(1)
d = json.loads(line[-1])
k = d["kernel_ms_per_step"]
print(f"{tag} ms/step {d['ms_per_step']:.3f} fwd {k['centre_forward']:.3f} bwd {k['centre_backward']:.3f} "
      f"fit {k['fit']:.3f} e2e {d['e2e']['value']:.2f} steps/s")
