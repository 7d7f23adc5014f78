"""Pin the CPU oracle (oracle/dp_oracle.cpp) against the reference's golden vectors.

The golden vectors (tests/golden/*.npz) were produced by the compiled, unmodified reference
(tests/golden/make_golden.py).  Where oracle/_ref is present the restatement is also
cross-checked live against the reference library.
"""
import numpy as np
import pytest

import oracle as O
from conftest import load_golden

CASES = ["dd_case_0", "dd_case_1", "dd_case_2"]


def _model(port, g):
    return port.model_init(O.test_spec(float(g["rc"])), int(g["model_seed"]))


@pytest.mark.parametrize("case", CASES)
def test_oracle_rows_bitexact(port, case):
    g = load_golden(case)
    h = _model(port, g)
    counts, mem, img, d = port.neighbor_rows(h, g["pos"], g["species"], g["box"])
    assert np.array_equal(counts, g["row_counts"])
    assert np.array_equal(mem, g["row_member"])
    assert np.array_equal(img, g["row_image"])
    assert np.array_equal(d, g["row_d"])  # FP64 displacements bit for bit
    port.model_free(h)


@pytest.mark.parametrize("case", CASES)
def test_oracle_energy_forces_virial(port, case):
    g = load_golden(case)
    h = _model(port, g)
    r = port.evaluate(h, g["pos"], g["species"], g["box"])
    assert r["energy"] == pytest.approx(float(g["energy"]), rel=1e-13, abs=1e-13)
    assert np.abs(r["atom_energy"] - g["atom_energy"]).max() <= 1e-13
    fs = np.abs(g["forces"]).max()
    assert np.abs(r["forces"] - g["forces"]).max() <= 1e-12 * fs
    assert np.abs(r["virial"] - g["virial"]).max() <= 1e-12 * np.abs(g["virial"]).max()
    port.model_free(h)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("scheme,tag", [(0, "masked"), (1, "wide")])
@pytest.mark.parametrize("nr", [1, 2, 4, 8])
def test_oracle_dd_and_halo(port, case, scheme, tag, nr):
    g = load_golden(case)
    h = _model(port, g)
    rc = float(g["rc"])
    thick = rc if scheme == 0 else 2 * rc
    dims = port.partition_ranks(g["box"], nr, thick)
    assert np.array_equal(dims, g[f"dd_{tag}_R{nr}_dims"])
    assert np.array_equal(port.owner_ranks(g["pos"], g["box"], dims), g[f"owner_R{nr}_{tag}"])
    F = np.zeros_like(g["forces"])
    E = 0.0
    for r in range(nr):
        a, o, s = port.build_halo(g["pos"], g["box"], dims, r, thick)
        assert np.array_equal(a, g[f"halo_{tag}_R{nr}_r{r}_atom"])
        assert np.array_equal(o, g[f"halo_{tag}_R{nr}_r{r}_owner"])
        assert np.array_equal(s, g[f"halo_{tag}_R{nr}_r{r}_shift"])
        out = port.dd_rank(h, g["pos"], g["species"], g["box"], nr, scheme, r)
        st = g[f"dd_{tag}_R{nr}_stats"][r]
        assert list(out["stats"]) == list(st[:3])
        F += out["forces"]
        E += out["energy"]
    assert E == pytest.approx(float(g[f"dd_{tag}_R{nr}_energy"]), rel=1e-12, abs=1e-12)
    assert np.abs(F - g[f"dd_{tag}_R{nr}_forces"]).max() <= 1e-12 * np.abs(g["forces"]).max()
    port.model_free(h)


def test_oracle_paper_model(port):
    g = load_golden("paper_small")
    h = port.model_init(O.PAPER_SPEC, 1)
    assert port.nparams(h) == int(g["nparams"]) == 1584945
    counts, mem, img, _ = port.neighbor_rows(h, g["pos"], g["species"], g["box"])
    assert np.array_equal(counts, g["row_counts"])
    assert np.array_equal(mem, g["row_member"]) and np.array_equal(img, g["row_image"])
    port.model_free(h)


def test_oracle_paper_model_energy_subset(port):
    """Per-centre energies of the paper model on a few centres (full eval is slow on CPU)."""
    g = load_golden("paper_small")
    h = port.model_init(O.PAPER_SPEC, 1)
    counts, mem, img, d = port.neighbor_rows(h, g["pos"], g["species"], g["box"])
    off = np.concatenate([[0], np.cumsum(counts)])
    for c in (0, 57, 399):
        rows = slice(off[c], off[c + 1])
        e, _ = port.evaluate_center(h, int(g["species"][c]), d[rows], g["species"][mem[rows]])
        assert e == pytest.approx(float(g["atom_energy"][c]), rel=1e-12, abs=1e-14)
    port.model_free(h)


def test_oracle_overflow_names_atom(port):
    g = load_golden("overflow_atom7")
    spec = O.test_spec(1.5, 2, 0)
    spec["n_max"] = 2
    h = port.model_init(spec, 12345)
    with pytest.raises(O.CapacityError, match="atom id 7"):
        port.evaluate(h, g["pos"], g["species"], g["box"], gids=g["gids"])
    assert "atom id 7" in str(g["message"])
    port.model_free(h)


def test_oracle_model_file_bitidentical(port, tmp_path):
    g = load_golden("paper_small")
    import hashlib
    h = port.model_init(O.PAPER_SPEC, 1)
    p = str(tmp_path / "m.nmdp")
    port.model_save(h, p)
    assert hashlib.sha256(open(p, "rb").read()).hexdigest() == str(g["model_sha256"])
    h2 = port.model_load(p)
    assert np.array_equal(port.flat(h), port.flat(h2))
    port.model_free(h)
    port.model_free(h2)


def test_oracle_matches_live_reference(port, ref):
    """Live cross-check against the compiled reference (dev container / GPU box)."""
    box, pos, sp, rc = ref.make_dd_case(424242)
    spec = O.test_spec(rc)
    hr, hp = ref.model_init(spec, 5), port.model_init(spec, 5)
    a, b = ref.evaluate(hr, pos, sp, box), port.evaluate(hp, pos, sp, box)
    assert a["energy"] == b["energy"]
    assert np.abs(a["forces"] - b["forces"]).max() <= 1e-12 * np.abs(a["forces"]).max()
    ref.model_free(hr)
    port.model_free(hp)


HEADLINE = ["c0_1500", "c1_15668", "rc4_2000", "rc8_4200"]


def test_oracle_synth_matches_product_generator(port):
    """The oracle's synthetic generator (used by the goldens and bench.py's reference arm,
    which must not map the product library) is bitwise the product's nnmd_synth_system."""
    import paper_2604_07276_b200 as nb
    for n, seed in ((15668, 1), (1500, 2), (400, 7), (37, 3)):
        a = port.synth_system(n, 0.1, 0.9, seed)
        b = nb.synth_system(n, 0.1, 0.9, seed)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("name", HEADLINE)
def test_headline_golden_rows_and_sampled_centres(port, name):
    """Headline-config goldens (compiled reference): the oracle reproduces the input
    digest, the canonical rows (sha256 + counts) and, for sampled centres, the reference's
    per-centre energies (bitwise-level)."""
    import hashlib
    g = load_golden(name)
    box, pos, sp = port.synth_system(int(g["n"]), 0.1, 0.9, int(g["seed"]))
    sha = hashlib.sha256(box.tobytes() + pos.tobytes() + sp.astype(np.int32).tobytes()).hexdigest()
    assert sha == str(g["input_sha256"])
    rc = float(g["rc"])
    h = port.model_init(dict(O.PAPER_SPEC, rc=rc, rcs=0.55 * rc, n_max=int(g["n_max"])), 1)
    counts, mem, img, d = port.neighbor_rows(h, pos, sp, box)
    assert np.array_equal(counts, g["row_counts"])
    rows = np.concatenate([mem.reshape(-1, 1), img], 1).astype(np.int32)
    assert hashlib.sha256(counts.astype(np.int32).tobytes() + rows.tobytes()).hexdigest() == str(g["rows_sha256"])
    off = np.concatenate([[0], np.cumsum(counts)])
    for c in (0, len(pos) // 3, len(pos) - 1):
        r = slice(off[c], off[c + 1])
        e, _ = port.evaluate_center(h, int(sp[c]), d[r], sp[mem[r]])
        assert abs(e - g["atom_energy"][c]) <= 1e-13 * max(1.0, abs(e)), (c, e, g["atom_energy"][c])
    # golden self-consistency: E = sum e_i, net force ~ 0, W symmetric (A19)
    assert abs(g["atom_energy"].sum() - float(g["energy"])) <= 1e-9 * abs(float(g["energy"]))
    fmax = np.abs(g["forces"]).max()
    assert np.abs(g["forces"].sum(axis=0)).max() <= 1e-9 * fmax * len(pos)
    W = g["virial"]
    assert np.abs(W - W.T).max() <= 1e-9 * np.abs(W).max()
    port.model_free(h)


def _strain(pos, a, b, h):
    p = pos.copy()
    p[:, a] += h * pos[:, b]
    return p


def test_virial_is_strain_derivative(port):
    """the virial convention W_ab = -sum_k g_{k,a} d_{k,b} (the reference has
    none) is -dE/d(eps_ab) under the homogeneous strain x_a -> x_a + eps_ab x_b.  Checked in
    FP64 on the oracle by central differences, all nine components, on a non-periodic
    cluster (any strain is admissible there) and along the axes of a periodic box."""
    g = load_golden("dd_case_0")
    h = _model(port, g)
    pos, sp, box = g["pos"], g["species"], g["box"]
    free = np.array([0, 0, 0], dtype=np.uint8)
    w = port.evaluate(h, pos, sp, box, periodic=free)["virial"]
    step = 1e-6
    fd = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            ep = port.evaluate(h, _strain(pos, a, b, step), sp, box, periodic=free)["energy"]
            em = port.evaluate(h, _strain(pos, a, b, -step), sp, box, periodic=free)["energy"]
            fd[a, b] = -(ep - em) / (2 * step)
    assert np.abs(w - fd).max() <= 1e-6 * np.abs(w).max(), (w, fd)
    # periodic: scaling one axis of positions and box together
    w = port.evaluate(h, pos, sp, box)["virial"]
    for a in range(3):
        s = np.ones(3)
        s[a] = 1 + step
        ep = port.evaluate(h, pos * s, sp, box * s)["energy"]
        s[a] = 1 - step
        em = port.evaluate(h, pos * s, sp, box * s)["energy"]
        assert abs(w[a, a] + (ep - em) / (2 * step)) <= 1e-6 * np.abs(w).max()
    port.model_free(h)
