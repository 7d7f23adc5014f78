"""Edge cases against the compiled reference (oracle/_ref, run on the GPU box as a prebuilt
library): non-periodic axes (SimBox::periodic, neighbor.cpp:22-30, decomp.cpp:96-131),
non-identity global ids (the canonical row key's last component, deeppot.cpp:141-148),
and empty / one- / two-atom systems."""
import numpy as np
import pytest

import oracle as O
import paper_2604_07276_b200 as nb

pytestmark = pytest.mark.gpu
TOL = 1e-5


def rel_err(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)) if a.size else 0.0


def rows_by_centre(counts, mem, img):
    off = np.concatenate([[0], np.cumsum(counts)])
    return [(mem[off[i]:off[i + 1]], img[off[i]:off[i + 1]]) for i in range(len(counts))]


def check_rows(ev, n_max, rows):
    ca, idx, img, cnt = ev.debug_nlist(0, n_max)
    for c, atom in enumerate(ca):
        gm, gi = rows[atom]
        assert cnt[c] == len(gm)
        assert np.array_equal(idx[c, : cnt[c]], gm)
        assert np.array_equal(img[c, : cnt[c]], gi)


@pytest.fixture(scope="module")
def models(ref):
    h = ref.model_init(O.test_spec(4.0, n_species=6), 5)
    yield h, nb.init_model(nb.test_spec(4.0, n_species=6), 5)
    ref.model_free(h)


@pytest.mark.parametrize("per", [(1, 0, 1), (0, 0, 0), (0, 1, 1)])
def test_nonperiodic_axes_rows_and_forces(ref, models, per):
    h, m = models
    box, pos, sp = nb.synth_system(700, 0.1, 0.9, 21)  # L = 19.1 A: 2 ranks fit the 2 rc wide halo
    rows = rows_by_centre(*ref.center_rows(h, pos, sp, box, periodic=per)[:3])
    want = ref.evaluate(h, pos, sp, box, periodic=per)
    ev = nb.DeviceEvaluator(m, n_ranks=1)
    ev.set_debug(True)
    r = ev.compute(pos, sp, box, periodic=per)
    check_rows(ev, 64, rows)
    assert abs(r["energy"] - want["energy"]) <= TOL * abs(want["energy"])
    assert rel_err(r["forces"], want["forces"]) <= TOL
    assert rel_err(r["virial"], want["virial"]) <= TOL
    for scheme in (nb.MASKED_REDUCTION, nb.WIDE_HALO):
        dd = ref.dd_evaluate(h, pos, sp, box, 2, scheme=scheme, periodic=per)
        g = nb.DeviceEvaluator(m, n_ranks=2, scheme=scheme).compute(pos, sp, box, periodic=per)
        assert abs(g["energy"] - dd["energy"]) <= TOL * abs(dd["energy"])
        assert rel_err(g["forces"], dd["forces"]) <= TOL
        assert rel_err(g["atom_energy"], dd["atom_energy"]) <= TOL


def test_shuffled_global_ids(ref, models):
    h, m = models
    box, pos, sp = nb.synth_system(300, 0.1, 0.9, 23)
    gids = (np.random.default_rng(3).permutation(len(pos)) * 7 + 11).astype(np.int64)
    rows = rows_by_centre(*ref.center_rows(h, pos, sp, box, gids=gids)[:3])
    want = ref.evaluate(h, pos, sp, box, gids=gids)
    ev = nb.DeviceEvaluator(m, n_ranks=1)
    ev.set_debug(True)
    r = ev.compute(pos, sp, box, gids=gids)
    check_rows(ev, 64, rows)
    assert abs(r["energy"] - want["energy"]) <= TOL * abs(want["energy"])
    assert rel_err(r["forces"], want["forces"]) <= TOL


def test_empty_one_and_two_atom_systems(ref, models):
    h, m = models
    box = np.array([20.0, 20.0, 20.0])
    ev = nb.DeviceEvaluator(m, n_ranks=1)
    r0 = ev.compute(np.zeros((0, 3)), np.zeros(0, dtype=np.int32), box)
    assert r0["energy"] == 0.0 and r0["forces"].shape == (0, 3)
    for pos, sp in [(np.array([[5.0, 5.0, 5.0]]), np.array([2], dtype=np.int32)),
                    (np.array([[5.0, 5.0, 5.0], [6.1, 5.4, 4.7]]), np.array([0, 3], dtype=np.int32))]:
        want = ref.evaluate(h, pos, sp, box)
        r = ev.compute(pos, sp, box)
        assert abs(r["energy"] - want["energy"]) <= TOL * abs(want["energy"])
        assert np.abs(r["forces"] - want["forces"]).max() <= TOL * max(np.abs(want["forces"]).max(), 1e-12) + 1e-12


@pytest.mark.parametrize("half_jitter", [False, True])
@pytest.mark.parametrize("n_species", [1, 2])
def test_exact_key_ties_on_a_lattice(ref, models, half_jitter, n_species):
    """Simple cubic lattice (spacing 2.5 A, exactly representable): every centre sees its 6
    first and 12 second neighbours at bitwise-equal r^2, so rows hinge on the gid tie-break
    of the canonical key (deeppot.cpp:141-148).  The centre-list build ranks on a packed
    (species, r^2) key and must detect these ties and fall back to the full comparison.
    Half-jittered: ties remain only around unjittered centres."""
    h, m = models
    g = np.arange(6) * 2.5
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + 0.25
    rng = np.random.default_rng(17)
    if half_jitter:
        pos[1::2] += rng.uniform(-0.1, 0.1, size=pos[1::2].shape)
    sp = (np.arange(len(pos)) % n_species).astype(np.int32)
    box = np.array([15.0, 15.0, 15.0])
    gids = (rng.permutation(len(pos)) * 3 + 5).astype(np.int64)
    rows = rows_by_centre(*ref.center_rows(h, pos, sp, box, gids=gids)[:3])
    want = ref.evaluate(h, pos, sp, box, gids=gids)
    ev = nb.DeviceEvaluator(m, n_ranks=1)
    ev.set_debug(True)
    r = ev.compute(pos, sp, box, gids=gids)
    check_rows(ev, 64, rows)
    assert abs(r["energy"] - want["energy"]) <= TOL * abs(want["energy"])
    if half_jitter:  # (the perfect lattice's forces cancel to rounding noise)
        assert rel_err(r["forces"], want["forces"]) <= TOL
