"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors and
the CPU oracle.  Bit-exact for neighbour rows and halo sets; FP32 network tolerance 1e-5
relative for energy (|dE|/|E|), forces (max|dF| / max|F|) and virial (max|dW| / max|W|)."""
import numpy as np
import pytest

import paper_2604_07276_b200 as nb
import oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu
CASES = ["dd_case_0", "dd_case_1", "dd_case_2"]
TOL = 1e-5  # FP32 contractions vs the FP64 reference


def rel_err(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def make_test_model(case_g):
    return nb.init_model(nb.test_spec(float(case_g["rc"])), int(case_g["model_seed"]))


def rows_by_centre(g):
    off = np.concatenate([[0], np.cumsum(g["row_counts"])])
    return [(g["row_member"][off[i]:off[i + 1]], g["row_image"][off[i]:off[i + 1]]) for i in range(len(g["row_counts"]))]


def check_rows(ev, rank, n_max, golden_rows):
    ca, idx, img, cnt = ev.debug_nlist(rank, n_max)
    for c, atom in enumerate(ca):
        gm, gi = golden_rows[atom]
        assert cnt[c] == len(gm), (rank, atom)
        assert np.array_equal(idx[c, : cnt[c]], gm), (rank, atom)
        assert np.array_equal(img[c, : cnt[c]], gi), (rank, atom)
    return ca


PRECS = [nb.PREC_FP32, nb.PREC_TF32, nb.PREC_FP32_SIMT]


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("case", CASES)
def test_single_domain_rows_bitexact_and_energy(case, prec):
    TOL = nb.TOLERANCE[prec]
    g = load_golden(case)
    m = make_test_model(g)
    ev = nb.DeviceEvaluator(m, n_ranks=1, precision=prec)
    ev.set_debug(True)
    r = ev.compute(g["pos"], g["species"], g["box"])
    ca = check_rows(ev, 0, 64, rows_by_centre(g))
    assert np.array_equal(ca, np.arange(len(g["pos"])))
    assert abs(r["energy"] - g["energy"]) / abs(g["energy"]) <= TOL
    assert rel_err(r["forces"], g["forces"]) <= TOL
    assert rel_err(r["virial"], g["virial"]) <= TOL
    assert rel_err(r["atom_energy"], g["atom_energy"]) <= TOL


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("scheme,tag", [(nb.MASKED_REDUCTION, "masked"), (nb.WIDE_HALO, "wide")])
@pytest.mark.parametrize("nr", [1, 2, 4, 8])
def test_dd_rows_halo_forces(case, scheme, tag, nr):
    g = load_golden(case)
    m = make_test_model(g)
    ev = nb.DeviceEvaluator(m, n_ranks=nr, scheme=scheme)
    ev.set_debug(True)
    r = ev.compute(g["pos"], g["species"], g["box"])
    grows = rows_by_centre(g)
    for rank in range(nr):
        atom, own, sh = ev.debug_ghosts(rank)
        assert np.array_equal(atom, g[f"halo_{tag}_R{nr}_r{rank}_atom"])
        assert np.array_equal(own, g[f"halo_{tag}_R{nr}_r{rank}_owner"])
        assert np.array_equal(sh, g[f"halo_{tag}_R{nr}_r{rank}_shift"])
        check_rows(ev, rank, 64, grows)
        st = ev.rank_stats(rank)
        gs = g[f"dd_{tag}_R{nr}_stats"][rank]
        assert (st["locals"], st["ghosts"], st["centers"]) == tuple(gs[:3])
    e_ref = float(g[f"dd_{tag}_R{nr}_energy"])
    assert abs(r["energy"] - e_ref) / abs(e_ref) <= TOL
    assert rel_err(r["forces"], g[f"dd_{tag}_R{nr}_forces"]) <= TOL
    assert rel_err(r["atom_energy"], g[f"dd_{tag}_R{nr}_atom_energy"]) <= TOL
    assert rel_err(r["virial"], g["virial"]) <= TOL


@pytest.mark.parametrize("prec", PRECS)
def test_paper_model_small_system(prec):
    TOL = nb.TOLERANCE[prec]
    g = load_golden("paper_small")
    m = nb.init_model(nb.paper_spec(6.0), 1)
    ev = nb.DeviceEvaluator(m, n_ranks=1, precision=prec)
    ev.set_debug(True)
    r = ev.compute(g["pos"], g["species"], g["box"])
    check_rows(ev, 0, 160, rows_by_centre(g))
    print("paper_small prec", prec, "dE/E", abs(r["energy"] - g["energy"]) / abs(g["energy"]),
          "dF", rel_err(r["forces"], g["forces"]), "dW", rel_err(r["virial"], g["virial"]))
    assert abs(r["energy"] - g["energy"]) / abs(g["energy"]) <= TOL
    assert rel_err(r["forces"], g["forces"]) <= TOL
    assert rel_err(r["virial"], g["virial"]) <= TOL
    ev2 = nb.DeviceEvaluator(m, n_ranks=2, precision=prec)
    r2 = ev2.compute(g["pos"], g["species"], g["box"])
    assert abs(r2["energy"] - g["dd_masked_R2_energy"]) / abs(g["energy"]) <= TOL
    assert rel_err(r2["forces"], g["dd_masked_R2_forces"]) <= TOL
    # per-centre energies are rank-count invariant bit for bit (same rows, same kernel)
    assert np.array_equal(r2["atom_energy"], r["atom_energy"])


def test_overflow_names_atom_id():
    g = load_golden("overflow_atom7")
    m = nb.init_model(nb.test_spec(1.5, 2, 0), 12345)
    m.set_n_max(2)
    ev = nb.DeviceEvaluator(m)
    with pytest.raises(nb.CapacityError, match="atom id 7"):
        ev.compute(g["pos"], g["species"], g["box"], gids=g["gids"])


def test_unwrapped_and_bad_species_rejected():
    g = load_golden("dd_case_0")
    m = make_test_model(g)
    ev = nb.DeviceEvaluator(m)
    pos = g["pos"].copy()
    pos[3, 1] = -0.1
    with pytest.raises(nb.Error, match="wrapped"):
        ev.compute(pos, g["species"], g["box"])
    sp = g["species"].copy()
    sp[5] = 9
    with pytest.raises(nb.Error, match="species"):
        ev.compute(g["pos"], sp, g["box"])
    # the context stays usable after an input error
    r = ev.compute(g["pos"], g["species"], g["box"])
    assert abs(r["energy"] - g["energy"]) / abs(g["energy"]) <= TOL


def test_isolated_atom_energy_is_fit_of_zero():
    m = nb.init_model(nb.test_spec(1.5, 2, 1), 99)
    port = O.Port()
    h = port.model_init(O.test_spec(1.5, 2, 1), 99)
    box = np.array([12.0, 12.0, 12.0])
    pos = np.array([[6.0, 6.0, 6.0]])
    sp = np.array([0], dtype=np.int32)
    r = nb.DeviceEvaluator(m).compute(pos, sp, box)
    o = port.evaluate(h, pos, sp, box)
    assert r["energy"] == pytest.approx(o["energy"], rel=1e-6)
    assert np.all(r["forces"] == 0.0)


def test_translation_invariance_and_momentum():
    g = load_golden("paper_small")
    m = nb.init_model(nb.paper_spec(6.0), 1)
    ev = nb.DeviceEvaluator(m)
    r0 = ev.compute(g["pos"], g["species"], g["box"])
    L = g["box"][0]
    moved = np.mod(g["pos"] + np.array([0.37, -0.21, 0.11]), L)
    r1 = ev.compute(moved, g["species"], g["box"])
    assert abs(r1["energy"] - r0["energy"]) / abs(r0["energy"]) <= TOL
    assert rel_err(r1["forces"], r0["forces"]) <= TOL
    assert np.abs(r0["forces"].sum(axis=0)).max() <= 1e-6 * np.abs(r0["forces"]).max() * len(g["pos"]) ** 0.5
    W = r0["virial"]
    assert np.abs(W - W.T).max() <= 1e-5 * np.abs(W).max()


def test_provider_species_map_and_group_mask():
    g = load_golden("dd_case_1")
    m = make_test_model(g)
    n = len(g["pos"])
    atoms = nb.AtomSet(np.arange(n), g["species"], g["pos"])
    box = nb.SimBox(g["box"])
    p = nb.DpProvider(m, nb.DpProvider.Options(decomposed=True, scheme=nb.WIDE_HALO, n_ranks=2))
    res = p.evaluate(atoms, box)
    assert abs(res.energy - g["energy"]) / abs(g["energy"]) <= TOL
    assert rel_err(res.forces, g["forces"]) <= TOL
    mask = np.zeros(n, dtype=bool)
    mask[: n // 2] = True
    pm = nb.DpProvider(m, nb.DpProvider.Options(), group_mask=mask)
    rm = pm.evaluate(atoms, box)
    assert np.all(rm.forces[n // 2:] == 0.0)
    with pytest.raises(nb.Error, match="species map"):
        nb.DpProvider(m, nb.DpProvider.Options(species_map=[0, 1])).evaluate(atoms, box)


def test_full_size_1hci_properties():
    """15,668-atom C1 system: rank-count invariance of per-centre energies (bitwise), force
    sum, virial symmetry, and oracle spot checks of per-centre energies."""
    box, pos, sp = nb.synth_system(15668, 0.1, 0.9, 1)
    m = nb.init_model(nb.paper_spec(6.0), 1)
    r1 = nb.DeviceEvaluator(m, n_ranks=1).compute(pos, sp, box)
    r8 = nb.DeviceEvaluator(m, n_ranks=8).compute(pos, sp, box)
    assert np.array_equal(r1["atom_energy"], r8["atom_energy"])
    assert rel_err(r8["forces"], r1["forces"]) <= 1e-9
    fmax = np.abs(r1["forces"]).max()
    assert np.abs(r1["forces"].sum(axis=0)).max() <= 1e-6 * fmax * len(pos) ** 0.5
    W = r1["virial"]
    assert np.abs(W - W.T).max() <= 1e-5 * np.abs(W).max()
    port = O.Port()
    h = port.model_init(O.PAPER_SPEC, 1)
    counts, mem, img, d = port.neighbor_rows(h, pos, sp, box)
    off = np.concatenate([[0], np.cumsum(counts)])
    for c in (0, 4321, 15667):
        rows = slice(off[c], off[c + 1])
        e, _ = port.evaluate_center(h, int(sp[c]), d[rows], sp[mem[rows]])
        assert abs(r1["atom_energy"][c] - e) <= TOL * max(abs(e), 1e-3)
    port.model_free(h)


def test_nccl_collective_path_single_gpu(monkeypatch):
    """The NCCL collective-2 path (dlopen libnccl, ncclCommInitRank, in-place f64
    ncclAllReduce of [E, W, F, e_i]) on one GPU gives the same result as without it."""
    g = load_golden("dd_case_1")
    m = make_test_model(g)
    r0 = nb.DeviceEvaluator(m, n_ranks=2).compute(g["pos"], g["species"], g["box"])
    monkeypatch.setenv("NNMD_FORCE_NCCL", "1")
    ev = nb.DeviceEvaluator(m, n_ranks=2)
    r1 = ev.compute(g["pos"], g["species"], g["box"])
    assert r1["energy"] == r0["energy"]
    assert np.array_equal(r1["forces"], r0["forces"])
    names = [name for name, _ in ev.kernel_times()]
    assert "nccl_allreduce" in names and "nccl_broadcast" in names  # collectives 2 and 1
    # the step flags travel through the int32 max all-reduce: overflow still names the atom
    go = load_golden("overflow_atom7")
    mo = nb.init_model(nb.test_spec(1.5, 2, 0), 12345)
    mo.set_n_max(2)
    evo = nb.DeviceEvaluator(mo, n_ranks=2)
    with pytest.raises(nb.CapacityError, match="atom id 7"):
        evo.compute(go["pos"], go["species"], go["box"], gids=go["gids"])
    # the ledger's ghost-route bytes are the total over all DD ranks (decomp.cpp:463-468)
    ev.set_trace(spans=False, ledger=True)
    ev.compute(g["pos"], g["species"], g["box"])
    routes = sum(ev.rank_stats(k)["route_entries"] for k in range(2))
    led = {kind: b for _, kind, b, _ in ev.ledger()}
    assert led["ghost_force_route"] == 20 * routes and routes > 0


@pytest.mark.parametrize("prec", [nb.PREC_FP32, nb.PREC_FP32_SIMT])
def test_large_neighbour_counts_multi_tile(prec):
    """n > 128 rows per centre (rc = 8 territory): multi-tile per-centre GEMMs, the
    unfused softmax path and n_max = 320, against the CPU oracle."""
    import oracle as O
    port = O.Port()
    box, pos, sp = nb.synth_system(700, 0.42, 0.7, 21)
    rc = 5.2
    spec = nb.test_spec(rc, n_species=6)
    spec.n_max = 320
    m = nb.init_model(spec, 8)
    ospec = O.test_spec(rc, n_species=6)
    ospec["n_max"] = 320
    h = port.model_init(ospec, 8)
    ev = nb.DeviceEvaluator(m, n_ranks=1, precision=prec)
    ev.set_debug(True)
    r = ev.compute(pos, sp, box)
    _, _, _, cnt = ev.debug_nlist(0, 320)
    assert cnt.max() > 160, cnt.max()
    o = port.evaluate(h, pos, sp, box)
    tol = nb.TOLERANCE[prec]
    assert abs(r["energy"] - o["energy"]) / abs(o["energy"]) <= tol
    assert rel_err(r["forces"], o["forces"]) <= tol
    assert rel_err(r["virial"], o["virial"]) <= tol
    port.model_free(h)


@pytest.mark.parametrize("rc", [4.0, 8.0])
def test_paper_model_cutoff_sweep_spotcheck(rc):
    """Paper-sized DPA-1 at rc = 4 (n_max 64) and rc = 8 (n_max 320): per-centre energies
    of sampled centres against the CPU oracle, and rank invariance (1 vs 8 DD ranks)."""
    import oracle as O
    box, pos, sp = nb.synth_system(2000 if rc == 4.0 else 4200, 0.1, 0.9, 5)
    m = nb.init_model(nb.paper_spec(rc), 1)
    r1 = nb.DeviceEvaluator(m, n_ranks=1).compute(pos, sp, box)
    r8 = nb.DeviceEvaluator(m, n_ranks=8 if rc == 4.0 else 1).compute(pos, sp, box)
    if rc == 4.0:
        # n_max 64: centres run as multi-centre 128-row units whose composition follows the
        # rank's centre order, so FP32 accumulation order (not the arithmetic) varies with
        # the rank count
        assert rel_err(r8["atom_energy"], r1["atom_energy"]) <= 1e-6
    else:
        assert np.array_equal(r1["atom_energy"], r8["atom_energy"])
    port = O.Port()
    h = port.model_init(dict(O.PAPER_SPEC, rc=rc, rcs=0.55 * rc, n_max=O.nmax_for_rc(rc)), 1)
    counts, mem, img, d = port.neighbor_rows(h, pos, sp, box)
    off = np.concatenate([[0], np.cumsum(counts)])
    for c in (0, 777, len(pos) - 1):
        rows = slice(off[c], off[c + 1])
        e, _ = port.evaluate_center(h, int(sp[c]), d[rows], sp[mem[rows]])
        assert abs(r1["atom_energy"][c] - e) <= 1e-5 * max(abs(e), 1e-2), (c, r1["atom_energy"][c], e)
    port.model_free(h)



def test_multi_centre_units_match_single_centre_path(monkeypatch):
    """rc = 4 (n_max 64): multi-centre 128-row units (up to four centres per tile, block-
    diagonal attention) against the one-centre-per-tile path (NNMD_FLAGS bit 3) on the
    same inputs: energies, forces, virial and per-atom energies within 1e-6, rows equal."""
    box, pos, sp = nb.synth_system(1200, 0.1, 0.9, 9)
    m = nb.init_model(nb.paper_spec(4.0), 3)
    monkeypatch.setenv("NNMD_FLAGS", "8")
    single = nb.DeviceEvaluator(m, n_ranks=2).compute(pos, sp, box)
    monkeypatch.delenv("NNMD_FLAGS")
    packed = nb.DeviceEvaluator(m, n_ranks=2).compute(pos, sp, box)
    assert abs(packed["energy"] - single["energy"]) <= 1e-6 * abs(single["energy"])
    for k in ("forces", "virial", "atom_energy"):
        assert rel_err(packed[k], single[k]) <= 1e-6, k


def test_virial_is_strain_derivative_on_gpu():
    """The product's virial against -dE/d(eps_ab) of the product's own energy under the
    homogeneous strain x_a -> x_a + eps_ab x_b (non-periodic cluster, all nine components;
    FP32 FMA network so that central differences resolve it)."""
    g = load_golden("dd_case_0")
    m = nb.init_model(nb.test_spec(float(g["rc"])), int(g["model_seed"]))
    ev = nb.DeviceEvaluator(m, n_ranks=1, precision=nb.PREC_FP32_SIMT)
    pos, sp, box = g["pos"], g["species"], g["box"]
    free = np.array([0, 0, 0], dtype=np.uint8)
    w = ev.compute(pos, sp, box, periodic=free)["virial"]
    step = 1e-3
    fd = np.zeros((3, 3))
    for a in range(3):
        for b in range(3):
            pp, pm = pos.copy(), pos.copy()
            pp[:, a] += step * pos[:, b]
            pm[:, a] -= step * pos[:, b]
            fd[a, b] = -(ev.compute(pp, sp, box, periodic=free)["energy"] -
                         ev.compute(pm, sp, box, periodic=free)["energy"]) / (2 * step)
    assert np.abs(w - fd).max() <= 2e-3 * np.abs(w).max(), (w, fd)


@pytest.mark.parametrize("scheme", [nb.MASKED_REDUCTION, nb.WIDE_HALO])
@pytest.mark.parametrize("which", ["NNMD_GHOST_CAP", "NNMD_LOCAL_CAP"])
def test_ghost_capacity_overflow_redo(monkeypatch, scheme, which):
    """The DD build has no host read-back: buffers are sized by per-rank local and ghost
    capacities and an overflow is flagged on the device, then the step is redone with
    grown capacities.  A capacity of 16 forces that path; the result must equal, bit for
    bit, a run whose first estimate fits."""
    g = load_golden("dd_case_0")
    m = nb.init_model(nb.test_spec(float(g["rc"])), int(g["model_seed"]))
    ref = nb.DeviceEvaluator(m, n_ranks=4, scheme=scheme).compute(g["pos"], g["species"], g["box"])
    monkeypatch.setenv(which, "16")
    ev = nb.DeviceEvaluator(m, n_ranks=4, scheme=scheme)
    r = ev.compute(g["pos"], g["species"], g["box"])
    for k in ("forces", "virial", "atom_energy"):
        assert np.array_equal(r[k], ref[k]), k
    assert r["energy"] == ref["energy"]
    st = [ev.rank_stats(q) for q in range(4)]
    assert all(s["ghosts"] > 16 and s["locals"] > 16 for s in st)
    r2 = ev.compute(g["pos"], g["species"], g["box"])  # grown capacities are kept
    assert np.array_equal(r2["forces"], ref["forces"])


def test_route_as_several_processes(monkeypatch):
    """The point-to-point ghost-force route as W processes would run it (NNMD_EMULATE_WORLD:
    each emulated process's plan, its receives as device copies into the receive buffers,
    its merge over the atoms it owns) must give the single-process result bit for bit --
    this checks the receive-buffer layout and the remote segment offsets of the merge on
    one GPU; only the NCCL transport itself is left to a multi-GPU box."""
    import subprocess, sys, json, os
    g = "dd_case_0"
    code = (
        "import sys, json, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_2604_07276_b200 as nb\nfrom conftest import load_golden\n"
        "g = load_golden(%r)\n"
        "m = nb.init_model(nb.test_spec(float(g['rc'])), int(g['model_seed']))\n"
        "out = {}\n"
        "for R in (2, 4, 8):\n"
        "    r = nb.DeviceEvaluator(m, n_ranks=R).compute(g['pos'], g['species'], g['box'])\n"
        "    out[R] = [r['energy'], r['forces'].tolist(), r['atom_energy'].tolist()]\n"
        "print(json.dumps(out))\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)), g)
    def run(env):
        e = dict(os.environ)
        e.update(env)
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        return json.loads(p.stdout.strip().splitlines()[-1])
    base = run({})
    for w in ("2", "3"):
        emu = run({"NNMD_EMULATE_WORLD": w})
        for R in base:
            assert emu[R][0] == base[R][0]
            assert emu[R][1] == base[R][1]
            assert emu[R][2] == base[R][2]
