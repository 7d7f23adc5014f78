"""Product NCCL path across processes: one process per GPU (world_size 2), DD rank r in
process r % 2, collective 1 (ncclBroadcast of rank 0's positions) and collective 2
(ncclAllReduce of [E, W, F, e_i] plus the step flags) -- decomp.cpp:157-204, 471-538.

Needs two visible GPUs (skipped otherwise; the gpurun boxes expose one).  The host-side
layout is covered on CPU by tests/test_dd_gloo.py.  Checked against the compiled
reference's dd_evaluate golden vectors at R = 2 (both schemes), and the overflow case: a
CapacityError raised on one process's DD rank must surface on BOTH processes (the step
flags are all-reduced before either process decides to throw).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, job, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_07276_b200 as nb
        from conftest import load_golden
        uid = nb.DeviceEvaluator.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
        dist.broadcast(t, src=0)
        uid = bytes(t.numpy().tobytes())
        kind, case, scheme = job
        g = load_golden(case)
        if kind == "dd":
            m = nb.init_model(nb.test_spec(float(g["rc"])), int(g["model_seed"]))
            ev = nb.DeviceEvaluator(m, n_ranks=2, scheme=scheme, device=rank, world_size=world, world_rank=rank,
                                    nccl_id=uid)
            # only world rank 0's coordinates are read (collective 1 broadcasts them)
            pos = g["pos"] if rank == 0 else None
            r = ev.compute(pos if pos is not None else np.zeros_like(g["pos"]), g["species"], g["box"])
            names = [k for k, _ in ev.kernel_times()]
            q.put((rank, r["energy"], r["forces"], r["atom_energy"], r["virial"], names))
        else:  # overflow: n_max 2 around atom id 7 -- only the rank owning it detects it
            m = nb.init_model(nb.test_spec(1.5, 2, 0), 12345)
            m.set_n_max(2)
            ev = nb.DeviceEvaluator(m, n_ranks=2, device=rank, world_size=world, world_rank=rank, nccl_id=uid)
            try:
                ev.compute(g["pos"], g["species"], g["box"], gids=g["gids"])
                q.put((rank, "no error"))
            except nb.CapacityError as e:
                q.put((rank, str(e)))
        ev.close()
    finally:
        dist.destroy_process_group()


def _run(job):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(2, _free_port(), job, q), nprocs=2, join=True, start_method="spawn")
    return sorted([q.get(timeout=120) for _ in range(2)], key=lambda x: x[0])


@pytest.mark.skipif(_n_gpus() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("scheme,tag", [(0, "masked"), (1, "wide")])
def test_two_gpu_nccl_matches_reference(scheme, tag):
    from conftest import load_golden
    g = load_golden("dd_case_1")
    out = _run(("dd", "dd_case_1", scheme))
    e_ref = float(g[f"dd_{tag}_R2_energy"])
    for rank, e, f, ae, w, names in out:
        assert "nccl_broadcast" in names and "nccl_allreduce" in names
        assert abs(e - e_ref) / abs(e_ref) <= 1e-5
        assert np.abs(f - g[f"dd_{tag}_R2_forces"]).max() <= 1e-5 * np.abs(g["forces"]).max()
        assert np.abs(ae - g[f"dd_{tag}_R2_atom_energy"]).max() <= 1e-5 * np.abs(g["atom_energy"]).max()
    # replicated result: both processes hold the same bits
    assert out[0][1] == out[1][1] and np.array_equal(out[0][2], out[1][2])


@pytest.mark.skipif(_n_gpus() < 2, reason="needs two GPUs")
def test_two_gpu_overflow_raises_on_every_process():
    out = _run(("overflow", "overflow_atom7", 0))
    for rank, msg in out:
        assert "atom id 7" in msg, (rank, msg)
