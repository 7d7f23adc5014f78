"""Generate the committed golden vectors from the COMPILED REFERENCE (oracle/_ref).

Run in the dev container (needs /root/reference to build oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py

Every output number comes from the unmodified reference library through its public API
(oracle/ref_capi.cpp): init_model/save_model, build_neighbor_list+center_rows,
evaluate_dp, dd_evaluate, partition_ranks/owner_rank_of/build_halo.  The virial is the
SURVEY A19 definition assembled from the reference's public row gradients.

Inputs:
* dd_case_{0,1,2}: acceptance.cpp:36-43 make_dd_case (seeds 9000+i), test_model(rc, 3, 3,
  seed 9000+i) -- 160-256 atoms, rc = L/6.2.
* paper_small: the paper-sized DPA-1 (1,584,945 params, seed 1, rc 6, n_max 160) on a
  400-atom synthetic solvated system (nnmd_synth_system, rho 0.1, min-sep 0.9, seed 7).
* overflow_atom7: test_deeppot.cpp:94-103 (n_max 2, "atom id 7").
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def dd_case(R, i):
    seed = 9000 + i
    box, pos, sp, rc = R.make_dd_case(seed)
    spec = O.test_spec(rc)
    h = R.model_init(spec, seed)
    res = R.evaluate(h, pos, sp, box)
    counts, mem, img, d = R.center_rows(h, pos, sp, box)
    g = dict(box=box, pos=pos, species=sp, rc=rc, model_seed=seed, energy=res["energy"], forces=res["forces"],
             atom_energy=res["atom_energy"], virial=res["virial"], row_counts=counts, row_member=mem,
             row_image=img, row_d=d)
    for nr in (1, 2, 4, 8):
        for scheme, tag in ((0, "masked"), (1, "wide")):
            dd = R.dd_evaluate(h, pos, sp, box, nr, scheme, workers=4)
            g[f"dd_{tag}_R{nr}_energy"] = dd["energy"]
            g[f"dd_{tag}_R{nr}_forces"] = dd["forces"]
            g[f"dd_{tag}_R{nr}_atom_energy"] = dd["atom_energy"]
            g[f"dd_{tag}_R{nr}_dims"] = dd["dims"]
            g[f"dd_{tag}_R{nr}_stats"] = dd["stats"]
            thick = rc if scheme == 0 else 2 * rc
            dims = dd["dims"]
            for r in range(nr):
                a, o, s = R.build_halo(pos, box, dims, r, thick)
                g[f"halo_{tag}_R{nr}_r{r}_atom"] = a
                g[f"halo_{tag}_R{nr}_r{r}_owner"] = o
                g[f"halo_{tag}_R{nr}_r{r}_shift"] = s
            g[f"owner_R{nr}_{tag}"] = R.owner_ranks(pos, box, dims)
    R.model_free(h)
    np.savez_compressed(os.path.join(OUT, f"dd_case_{i}.npz"), **g)
    print("dd_case", i, len(pos), "atoms, E =", res["energy"])


def paper_small(R):
    import paper_2604_07276_b200 as nb
    box, pos, sp = nb.synth_system(400, 0.1, 0.9, 7)
    h = R.model_init(O.PAPER_SPEC, 1)
    path = "/tmp/paper_rc6_seed1.nmdp"
    R.model_save(h, path)
    sha = hashlib.sha256(open(path, "rb").read()).hexdigest()
    res = R.evaluate(h, pos, sp, box)
    counts, mem, img, d = R.center_rows(h, pos, sp, box)
    dd2 = R.dd_evaluate(h, pos, sp, box, 2, 0, workers=8)
    np.savez_compressed(os.path.join(OUT, "paper_small.npz"), box=box, pos=pos, species=sp, model_sha256=sha,
                        nparams=R.nparams(h), energy=res["energy"], forces=res["forces"],
                        atom_energy=res["atom_energy"], virial=res["virial"], row_counts=counts, row_member=mem,
                        row_image=img, dd_masked_R2_energy=dd2["energy"], dd_masked_R2_forces=dd2["forces"])
    R.model_free(h)
    print("paper_small E =", res["energy"], "sha", sha[:16])


def overflow_case(R):
    box = np.array([10.0, 10.0, 10.0])
    pos = np.array([[5.0, 5.0, 5.0], [5.5, 5.0, 5.0], [4.5, 5.0, 5.0], [5.0, 5.5, 5.0]])
    sp = np.zeros(4, dtype=np.int32)
    gids = np.array([7, 1, 2, 3])
    h = R.model_init(O.test_spec(1.5, 2, 0), 12345)
    R.set_nmax(h, 2)
    msg = ""
    try:
        R.evaluate(h, pos, sp, box, gids=gids)
    except O.CapacityError as e:
        msg = str(e)
    R.model_free(h)
    np.savez_compressed(os.path.join(OUT, "overflow_atom7.npz"), box=box, pos=pos, species=sp, gids=gids,
                        message=np.array(msg))
    print("overflow:", msg)


if __name__ == "__main__":
    R = O.Ref()
    for i in range(3):
        dd_case(R, i)
    paper_small(R)
    overflow_case(R)
