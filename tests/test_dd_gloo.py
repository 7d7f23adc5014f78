"""World-size-2 multi-process test of the DD decomposition on CPU (gloo).

Mirrors the product's N > 1 layout: DD rank r is evaluated by process r % world_size
(context.cpp run loop), each process contributes its ranks' global-indexed partial forces,
owned energies and virial, and one all-reduce (the NCCL collective 2 on GPUs; gloo here)
yields the replicated result of dd_evaluate (decomp.cpp:471-538).  The grid comes from the
product's host planner (nnmd_partition_ranks); the per-rank arithmetic from the CPU oracle.
Checked against the compiled reference's golden dd_evaluate outputs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, n_ranks, scheme, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_2604_07276_b200 as nb
        from conftest import load_golden
        g = load_golden(case)
        rc = float(g["rc"])
        dims = nb.partition_ranks(g["box"], n_ranks, rc if scheme == 0 else 2 * rc)
        port_ = O.Port()
        h = port_.model_init(O.test_spec(rc), int(g["model_seed"]))
        n = len(g["pos"])
        buf = np.zeros(10 + 4 * n)  # [E, W9, F(3n), ae(n)] -- the product's d_out layout
        for r in range(n_ranks):
            if r % world != rank:
                continue
            out = port_.dd_rank(h, g["pos"], g["species"], g["box"], n_ranks, scheme, r)
            buf[0] += out["energy"]
            buf[1:10] += out["virial"].ravel()
            buf[10:10 + 3 * n] += out["forces"].ravel()
            buf[10 + 3 * n:] += out["atom_energy"]
        t = torch.from_numpy(buf)
        dist.all_reduce(t)
        if rank == 0:
            q.put((dims.tolist(), t.numpy().copy()))
        port_.model_free(h)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["dd_case_0", "dd_case_2"])
@pytest.mark.parametrize("scheme,tag", [(0, "masked"), (1, "wide")])
@pytest.mark.parametrize("n_ranks", [2, 4])
def test_two_process_dd_matches_reference(case, scheme, tag, n_ranks):
    from conftest import load_golden
    g = load_golden(case)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, case, n_ranks, scheme, q), nprocs=2, join=True, start_method="spawn")
    dims, buf = q.get(timeout=60)
    n = len(g["pos"])
    assert dims == list(g[f"dd_{tag}_R{n_ranks}_dims"])
    e_ref = float(g[f"dd_{tag}_R{n_ranks}_energy"])
    assert abs(buf[0] - e_ref) <= 1e-12 * abs(e_ref)
    F = buf[10:10 + 3 * n].reshape(n, 3)
    assert np.abs(F - g[f"dd_{tag}_R{n_ranks}_forces"]).max() <= 1e-12 * np.abs(g["forces"]).max()
    assert np.abs(buf[10 + 3 * n:] - g[f"dd_{tag}_R{n_ranks}_atom_energy"]).max() <= 1e-13
    assert np.abs(buf[1:10].reshape(3, 3) - g["virial"]).max() <= 1e-12 * np.abs(g["virial"]).max()
