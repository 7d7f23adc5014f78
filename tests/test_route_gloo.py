"""Ghost-force route across processes on CPU (gloo): the product's point-to-point plan.

On GPUs the masked scheme routes each ghost image's force partial to the atom's owner rank
with ncclSend/ncclRecv (context.cpp route_and_reduce; reference decomp.cpp:445-469), using
the plan of ``nnmd_route_schedule`` (host code, no GPU).  One gpurun box has a single GPU,
so this test runs that exact plan over gloo with world_size 2 and 3: every process packs
synthetic routed entries of its DD ranks grouped by destination (in a scrambled order
inside each group, as the device's atomic fill does), all-reduces the (source,
destination) counts, posts the plan's sends and receives, and merges what its ranks own in
the reference order (owner's zero-image partial first, then routed partials by (zero
image first, image, rank); decomp.cpp:502-536).  The result must equal, bit for bit, a
single-process merge of all entries, and the plan must satisfy its own invariants.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ZERO = 13  # packed zero shift


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entries(n_atoms, R, s):
    """Routed entries of DD rank s: (atom, img, src, fx, fy, fz); owner(atom) = atom % R.
    A zero-image entry of an atom s owns is its base partial, never routed."""
    rng = np.random.default_rng(1000 + s)
    out = []
    for atom in rng.choice(n_atoms, size=n_atoms // 2, replace=False):
        for img in rng.choice(27, size=rng.integers(1, 4), replace=False):
            if img == ZERO and atom % R == s:
                continue
            out.append((atom, img, s, *rng.normal(size=3)))
    return np.array(out, dtype=np.float64).reshape(-1, 6)


def _base(n_atoms):
    return np.random.default_rng(7).normal(size=(n_atoms, 3))


def _merge(n_atoms, R, owned, base, entries):
    f = np.zeros((n_atoms, 3))
    key = lambda e: (0 if int(e[1]) == ZERO else 1, int(e[1]), int(e[2]))
    by_atom = {}
    for e in entries:
        by_atom.setdefault(int(e[0]), []).append(e)
    for t in range(n_atoms):
        if not owned(t % R):
            continue
        acc = base[t].copy()
        for e in sorted(by_atom.get(t, []), key=key):
            acc = acc + e[3:6]
        f[t] = acc
    return f


def _worker(rank, world, port, R, n_atoms, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_07276_b200 as nb
        local = lambda r: r % world == rank
        rng = np.random.default_rng(rank)
        send = {}
        cnt = np.zeros((R, R), dtype=np.int32)
        for s in range(R):
            if not local(s):
                continue
            e = _entries(n_atoms, R, s)
            groups = []
            for o in range(R):
                g = e[(e[:, 0].astype(int) % R) == o]
                groups.append(g[rng.permutation(len(g))])  # arrival order inside a group is arbitrary
                cnt[s, o] = len(g)
            send[s] = np.concatenate(groups) if groups else np.zeros((0, 6))
        tc = torch.from_numpy(cnt.copy())
        dist.all_reduce(tc)
        cnt = tc.numpy()
        plan = nb.route_schedule(R, world, rank, cnt)
        # invariants: every transfer crosses processes, counts match, offsets are the
        # group starts of the sender's / receiver's buffers
        for op in plan:
            assert op["count"] == cnt[op["src"], op["dst"]] > 0
            if op["kind"] == "send":
                assert local(op["src"]) and not local(op["dst"]) and op["peer"] == op["dst"] % world
                assert op["offset"] == cnt[op["src"], :op["dst"]].sum()
            else:
                assert local(op["dst"]) and not local(op["src"]) and op["peer"] == op["src"] % world
                assert op["offset"] == sum(cnt[op["src"], o] for o in range(op["dst"]) if local(o))
        recv = {s: np.zeros((sum(cnt[s, o] for o in range(R) if local(o)), 6)) for s in range(R) if not local(s)}
        seq = {}
        reqs = []
        for op in plan:  # posting order; the k-th transfer of a process pair gets tag k on both sides
            k = seq.get(op["peer"], 0)
            seq[op["peer"]] = k + 1
            if op["kind"] == "send":
                buf = torch.from_numpy(np.ascontiguousarray(send[op["src"]][op["offset"]:op["offset"] + op["count"]]))
                reqs.append(dist.isend(buf, dst=op["peer"], tag=k))
            else:
                buf = torch.zeros((op["count"], 6), dtype=torch.float64)
                reqs.append((dist.irecv(buf, src=op["peer"], tag=k), op, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                recv[r[1]["src"]][r[1]["offset"]:r[1]["offset"] + r[1]["count"]] = r[2].numpy()
            else:
                r.wait()
        # incoming stream of this process: local sources' groups for local owners + receives
        inc = [send[s][cnt[s, :o].sum():cnt[s, :o].sum() + cnt[s, o]] for s in send for o in range(R) if local(o)]
        inc += list(recv.values())
        inc = np.concatenate(inc) if inc else np.zeros((0, 6))
        f = _merge(n_atoms, R, local, _base(n_atoms), inc)
        t = torch.from_numpy(f)
        dist.all_reduce(t)  # one writer per atom: exact
        if rank == 0:
            q.put((t.numpy().copy(), len(plan)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,R", [(2, 2), (2, 4), (3, 5), (2, 8), (3, 8)])
def test_route_plan_over_gloo_matches_single_process_merge(world, R):
    n_atoms = 60
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, n_atoms, q)) for r in range(world)]
    for p in procs:
        p.start()
    f, nops = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    all_entries = np.concatenate([_entries(n_atoms, R, s) for s in range(R)])
    ref = _merge(n_atoms, R, lambda r: True, _base(n_atoms), all_entries)
    assert nops > 0
    np.testing.assert_array_equal(f, ref)  # bitwise: same per-atom order on every layout


def test_route_plan_single_process_is_empty():
    import paper_2604_07276_b200 as nb
    cnt = np.arange(16, dtype=np.int32).reshape(4, 4)
    assert nb.route_schedule(4, 1, 0, cnt) == []


def test_route_plan_rejects_bad_counts():
    import paper_2604_07276_b200 as nb
    with pytest.raises(nb.Error):
        nb.route_schedule(2, 2, 0, np.array([[0, -1], [0, 0]]))
