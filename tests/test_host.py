"""Host-side checks of the product library that need no GPU: the C ABI loads and exports
every declared symbol, model init/IO is bit-identical to the reference, DD planning
matches the reference, error paths map to the reference exception classes."""
import hashlib
import os

import numpy as np
import pytest

import paper_2604_07276_b200 as nb
from conftest import load_golden


def test_library_exports_every_header_symbol():
    L = nb.lib()
    names = nb.header_functions()
    assert len(names) >= 20
    missing = [f for f in names if not hasattr(L, f)]
    assert not missing, missing
    assert b"sm_100a" in L.nnmd_b200_version()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", nb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_init_model_bitidentical_to_reference(tmp_path):
    g = load_golden("paper_small")
    m = nb.init_model(nb.paper_spec(6.0), 1)
    assert m.n_params() == 1584945
    p = str(tmp_path / "m.nmdp")
    m.save(p)
    assert hashlib.sha256(open(p, "rb").read()).hexdigest() == str(g["model_sha256"])
    m2 = nb.load_model(p)
    p2 = str(tmp_path / "m2.nmdp")
    m2.save(p2)
    assert open(p, "rb").read() == open(p2, "rb").read()
    s = m2.spec()
    assert (s.n_feat, s.n_reduced, s.attn_dim, tuple(s.embed_hidden), tuple(s.fit_hidden)) == (
        128, 32, 256, (32, 64), (256, 256, 256))


def test_load_model_errors(tmp_path):
    p = tmp_path / "bad.nmdp"
    p.write_bytes(b"XXXX1234")
    with pytest.raises(nb.Error, match="bad magic"):
        nb.load_model(str(p))
    m = nb.init_model(nb.test_spec(1.5), 3)
    good = tmp_path / "good.nmdp"
    m.save(str(good))
    data = good.read_bytes()
    (tmp_path / "trunc.nmdp").write_bytes(data[:-5])
    with pytest.raises(nb.Error, match="truncated"):
        nb.load_model(str(tmp_path / "trunc.nmdp"))
    (tmp_path / "trail.nmdp").write_bytes(data + b"\0")
    with pytest.raises(nb.Error, match="trailing"):
        nb.load_model(str(tmp_path / "trail.nmdp"))


@pytest.mark.parametrize("case", ["dd_case_0", "dd_case_1", "dd_case_2"])
def test_partition_ranks_matches_reference(case):
    g = load_golden(case)
    rc = float(g["rc"])
    for nr in (1, 2, 4, 8):
        assert np.array_equal(nb.partition_ranks(g["box"], nr, rc), g[f"dd_masked_R{nr}_dims"])
        assert np.array_equal(nb.partition_ranks(g["box"], nr, 2 * rc), g[f"dd_wide_R{nr}_dims"])


def test_partition_ranks_known_answers():
    # test_decomp.cpp:61-93
    assert list(nb.partition_ranks([10, 10, 10], 8)) == [2, 2, 2]
    assert list(nb.partition_ranks([10, 10, 10], 1)) == [1, 1, 1]
    assert list(nb.partition_ranks([10, 10, 10], 2)) == [2, 1, 1]
    assert list(nb.partition_ranks([2, 1, 1], 4)) == [2, 2, 1]
    with pytest.raises(nb.Error):
        nb.partition_ranks([10, 10, 10], 64, 6.0)
    d = nb.partition_ranks([10, 10, 10], 4, 5.0)
    assert min(10 / d[0], 10 / d[1], 10 / d[2]) >= 5.0
    # 1HCI-sized box: 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2
    L = (15668 / 0.1) ** (1 / 3)
    assert [list(nb.partition_ranks([L] * 3, r, 6.0)) for r in (2, 4, 8)] == [[2, 1, 1], [2, 2, 1], [2, 2, 2]]


def test_synth_system_deterministic_and_physical():
    box, pos, sp = nb.synth_system(4000, 0.1, 0.9, 3)
    box2, pos2, sp2 = nb.synth_system(4000, 0.1, 0.9, 3)
    assert np.array_equal(pos, pos2) and np.array_equal(sp, sp2)
    assert box[0] == pytest.approx((4000 / 0.1) ** (1 / 3))
    assert pos.min() >= 0 and (pos < box[0]).all()
    assert set(np.unique(sp)) <= set(range(6)) and len(np.unique(sp)) == 6
    from scipy.spatial import cKDTree
    d, _ = cKDTree(pos, boxsize=box[0]).query(pos, k=2)
    assert d[:, 1].min() >= 0.9


def test_evaluator_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    m = nb.init_model(nb.test_spec(1.5), 3)
    with pytest.raises(nb.CudaError):
        nb.DeviceEvaluator(m)
