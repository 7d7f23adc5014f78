"""Drop-in check on the GPU: the reference's own run_md (engine.cpp:143-211) driven by the
reference DpProvider and by GpuDpProvider (include/nnmd_b200_provider.hpp), both through
the unmodified reference engine (oracle/_ref/provider_md, built by make -C oracle
integration).  Trajectories must agree."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "provider_md")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("decomposed", [0, 1])
def test_reference_run_md_with_gpu_provider(decomposed):
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, "5", str(decomposed)], capture_output=True, text=True, timeout=600)
    line = r.stdout.strip().splitlines()[-1]
    d = json.loads(line)
    print(d)
    assert r.returncode == 0, r.stdout + r.stderr
    assert d["max_rel_energy_diff"] < 1e-5 and d["max_position_diff"] < 1e-6
