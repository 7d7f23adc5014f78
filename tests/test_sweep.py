"""Sweep harness (paper_2604_07276_b200/sweep.py): the Eq. 8 throughput fit, the scaling
efficiencies and throughput_per_day against the compiled reference (analysis.cpp:148-208,
engine.cpp:213-216), the weak-scaling replication (cli.cpp:654-669) and the fit-scaling
CSV/JSON outputs (cli.cpp:739-800).  CPU only."""
import json
import os

import numpy as np
import pytest

from paper_2604_07276_b200 import sweep as S

POINT_SETS = [
    [(1, 7.3), (2, 13.9), (4, 25.1), (8, 40.2)],
    [(1, 0.61), (2, 1.1), (4, 1.6), (8, 1.9), (16, 2.1)],
    [(2, 5.0), (8, 5.0)],                       # flat: alpha clamps to 0
    [(1, 1.0), (2, 2.0), (4, 4.0)],             # ideal: beta 0, r^2 1
]


@pytest.mark.parametrize("pts", POINT_SETS)
def test_fit_matches_reference(ref, pts):
    a = S.fit_throughput(pts)
    b = ref.fit_throughput(pts)
    for k in ("alpha", "beta", "r_squared"):
        assert a[k] == pytest.approx(b[k], rel=1e-14, abs=1e-14), k
    assert np.allclose(a["residuals"], b["residuals"], rtol=1e-12, atol=1e-15)
    for n_p in (1, 3, 8, 32):
        if a["alpha"] > 0 or a["beta"] > 0:
            assert S.predict_throughput(a["alpha"], a["beta"], n_p) == pytest.approx(
                ref.predict_throughput(b["alpha"], b["beta"], n_p), rel=1e-14)


@pytest.mark.parametrize("weak", [False, True])
def test_efficiency_matches_reference(ref, weak):
    tr = {1: 42.5, 2: 80.1, 4: 147.0, 8: 233.3}
    for reference in (1, 2):
        a = S.scaling_efficiency(tr, reference, weak)
        b = ref.scaling_efficiency(tr, reference, weak)
        for k in tr:
            assert a[k] == pytest.approx(b[k], rel=1e-15)
    assert ref.throughput_per_day(3, 0.002, 0.0235) == pytest.approx(S.throughput_per_day(3, 0.002, 0.0235), rel=1e-15)


def test_fit_rejects_degenerate():
    with pytest.raises(ValueError):
        S.fit_throughput([(2, 1.0), (2, 3.0)])
    with pytest.raises(ValueError):
        S.fit_throughput([(1, 1.0)])


def test_weak_replication_layout():
    box = np.array([10.0, 11.0, 12.0])
    pos = np.array([[1.0, 2.0, 3.0], [9.5, 0.5, 0.25]])
    sp = np.array([1, 4], dtype=np.int32)
    B, P, Sp, G = S.replicate(box, pos, sp, np.arange(2), 3)
    assert np.array_equal(B, [30.0, 11.0, 12.0])
    assert np.array_equal(G, [0, 1, 2, 3, 4, 5])
    assert np.array_equal(P[2:4, 0], pos[:, 0] + 10.0) and np.array_equal(P[4:, 1:], pos[:, 1:])
    assert np.array_equal(Sp, [1, 4, 1, 4, 1, 4])


def test_fit_scaling_outputs(tmp_path):
    pts = os.path.join(tmp_path, "sweep.csv")
    with open(pts, "w") as f:
        f.write("mode,n_ranks,n_atoms,step_seconds,throughput\n")
        for n, t in POINT_SETS[0]:
            f.write(f"strong,{n},15668,{0.002 * 86400 / t!r},{t!r}\n")
    res = S.fit_scaling(pts, str(tmp_path))
    js = json.load(open(os.path.join(tmp_path, "scaling_fit.json")))
    assert js["reference"] == 1 and not js["weak"]
    rows = open(os.path.join(tmp_path, "efficiency.csv")).read().strip().splitlines()
    assert rows[0] == "n_ranks,throughput,efficiency,model_throughput" and len(rows) == 5
    assert res["efficiency"][8] == pytest.approx(40.2 / 7.3 / 8)
