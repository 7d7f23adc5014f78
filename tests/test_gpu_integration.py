"""Drop-in check on the GPU: the reference's own run_md (engine.cpp:143-211) driven by the
reference DpProvider and by GpuDpProvider (include/nnmd_b200_provider.hpp), both through
the unmodified reference engine (oracle/_ref/provider_md, built by make -C oracle
integration).  Trajectories must agree; the device-resident GpuDpProvider::run_md must
reproduce the provider's run_md trajectory bit for bit; the TraceSink spans and
CollectiveLedger records must match the reference's."""
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
    lines = [json.loads(x) for x in r.stdout.strip().splitlines() if x.startswith("{")]
    tr = [x["trace"] for x in lines if "trace" in x][0]
    d = [x for x in lines if "provider" in x][0]
    print(tr, d)
    assert r.returncode == 0, r.stdout + r.stderr
    assert d["max_rel_energy_diff"] < 1e-5 and d["max_position_diff"] < 1e-6
    # device-resident loop (GpuDpProvider::run_md) == reference run_md with the provider
    assert d["device_loop_position_diff"] == 0.0 and d["device_loop_potential_diff"] == 0.0
    # TraceSink / CollectiveLedger records identical in kind, rank, step and bytes
    assert tr["ledger_match"] and tr["span_keys_match"] and tr["chrome_roundtrip"]
