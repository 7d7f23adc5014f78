"""Scaling harness on B200 -- the reference's ``cmd_sweep`` / ``cmd_fit_scaling``
(cli.cpp:619-800) and its analysis formulas (analysis.cpp:148-208), over the CUDA path.

``sweep`` runs ``dd_evaluate`` (this package's ``DeviceEvaluator``) for each rank count and
writes the reference's CSVs:

* ``sweep.csv``              mode,n_ranks,n_atoms,step_seconds,throughput
* ``sweep_rank_phases.csv``  step,rank,locals,ghosts,phase,seconds,bytes (per-rank phases
                             dd_build / neighbor_build / inference / force_assembly, then
                             one row per ledger record on rank -1 with its bytes)
* ``ledger.csv``             step,kind,bytes,participants (CollectiveLedger records)

Step time follows cmd_sweep's virtual parallel machine (cli.cpp:672-717): the minimum over
steps of the step-global (collective) time plus the slowest rank's minimum-over-steps busy
time.  With one process all DD ranks run back to back on one GPU and each rank's busy
time is its own CUDA-event-timed phases, so on one GPU this is an ESTIMATE of an R-GPU run
that leaves out the NCCL time of collective 2 (which it cannot measure); with one process
per GPU (torchrun, world_size == n_ranks) the spans are that rank's own and the NCCL
collectives are measured.  Weak mode replicates the box along x, one replica per
``ranks_per_replica`` ranks (cli.cpp:654-669).

``fit_scaling`` is cmd_fit_scaling: the Eq. 8 fit 1/tr = alpha/n_p + beta
(``fit_throughput``, analysis.cpp:156-192) and the strong / weak efficiencies
(``scaling_efficiency``, analysis.cpp:194-208) -> ``scaling_fit.json``, ``efficiency.csv``.
The formulas are pinned against the compiled reference in tests/test_sweep.py.

    python -m paper_2604_07276_b200.sweep --mode strong --ranks 1 2 4 8 --out sweep_out
"""
from __future__ import annotations

import argparse
import json
import os
from typing import Dict, Iterable, List, Sequence, Tuple

import numpy as np

PHASE_CSV = ("dd_build", "neighbor_build", "inference", "force_assembly")


# ------------------------------------------------------------------ analysis.cpp / engine.cpp
def throughput_per_day(n_steps: int, dt: float, elapsed_seconds: float) -> float:
    """engine.cpp:213-216: simulated time per day of wall time."""
    if not elapsed_seconds > 0.0:
        raise ValueError("throughput: elapsed must be > 0")
    return float(n_steps) * dt / elapsed_seconds * 86400.0


def predict_throughput(alpha: float, beta: float, n_p: float) -> float:
    """analysis.cpp:148-154 (Eq. 8): tr(n_p) = 1 / (alpha / n_p + beta)."""
    if n_p < 1.0:
        raise ValueError("predict_throughput: n_p must be >= 1")
    if not (alpha > 0.0 or beta > 0.0):
        raise ValueError("predict_throughput: alpha = beta = 0 is undefined")
    return 1.0 / (alpha / n_p + beta)


def fit_throughput(points: Sequence[Tuple[float, float]]) -> dict:
    """analysis.cpp:156-192: least squares of 1/tr = alpha * (1/n_p) + beta, both clamped
    at zero; r^2 of the linearised fit."""
    if len(points) < 2:
        raise ValueError("fit_throughput: need at least two points")
    if all(p[0] == points[0][0] for p in points[1:]):
        raise ValueError("fit_throughput: degenerate design matrix (one n_p)")
    sx = sy = sxx = sxy = 0.0
    n = float(len(points))
    for np_, tr in points:
        if not (np_ >= 1.0 and tr > 0.0):
            raise ValueError("fit_throughput: bad point")
        x, y = 1.0 / np_, 1.0 / tr
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
    denom = n * sxx - sx * sx
    alpha = (n * sxy - sx * sy) / denom
    beta = (sy - alpha * sx) / n
    alpha = max(alpha, 0.0)
    beta = max(beta, 0.0)
    ss_res = ss_tot = 0.0
    y_mean = sy / n
    res = []
    for np_, tr in points:
        y = 1.0 / tr
        y_hat = alpha / np_ + beta
        res.append(y - y_hat)
        ss_res += (y - y_hat) * (y - y_hat)
        ss_tot += (y - y_mean) * (y - y_mean)
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0.0 else (1.0 if ss_res < 1e-24 else 0.0)
    return {"alpha": alpha, "beta": beta, "r_squared": r2, "residuals": res}


def scaling_efficiency(tr: Dict[int, float], reference: int, weak: bool = False) -> Dict[int, float]:
    """analysis.cpp:194-208: strong eff(n) = (tr(n)/tr(ref)) * (ref/n); weak tr(n)/tr(ref)."""
    if reference not in tr:
        raise ValueError("scaling_efficiency: reference rank count missing")
    t_ref = tr[reference]
    if not t_ref > 0.0:
        raise ValueError("scaling_efficiency: non-positive reference")
    return {n: (t / t_ref if weak else (t / t_ref) * (reference / n)) for n, t in sorted(tr.items())}


def replicate(box, pos, species, gids, replicas: int):
    """cmd_sweep's weak replication along x (cli.cpp:654-669): gid + rep * n, x + rep * Lx."""
    n = len(pos)
    reps = max(1, replicas)
    P = np.concatenate([pos + np.array([r * box[0], 0.0, 0.0]) for r in range(reps)])
    S = np.concatenate([species] * reps)
    G = np.concatenate([np.asarray(gids, dtype=np.int64) + r * n for r in range(reps)])
    B = np.array([box[0] * reps, box[1], box[2]], dtype=np.float64)
    return B, np.ascontiguousarray(P), np.ascontiguousarray(S, dtype=np.int32), G


def _csv(v: float) -> str:
    return repr(float(v))


# ------------------------------------------------------------------ cmd_sweep on the device
def sweep(model, box, pos, species, mode: str = "strong", ranks: Iterable[int] = (1, 2, 4, 8), steps: int = 3,
          scheme: int = 0, ranks_per_replica: int = 1, dt: float = 0.002, out: str = "sweep_out", device: int = 0,
          precision: int = 0, warmup: int = 1, world_size: int = 1, world_rank: int = 0, nccl_id=None) -> List[dict]:
    """cmd_sweep (cli.cpp:619-733) over DeviceEvaluator; returns the sweep.csv points."""
    import torch

    from . import DeviceEvaluator

    if mode not in ("strong", "weak"):
        raise ValueError("sweep: mode must be strong or weak")
    os.makedirs(out, exist_ok=True)
    points_rows = ["mode,n_ranks,n_atoms,step_seconds,throughput"]
    rank_rows = ["step,rank,locals,ghosts,phase,seconds,bytes"]
    ledger_rows = ["n_ranks,step,kind,bytes,participants"]
    points = []
    gids0 = np.arange(len(pos), dtype=np.int64)
    dev = torch.device("cuda", device)
    for npr in ranks:
        B, P, S, G = (box, pos, species, gids0)
        if mode == "weak":
            B, P, S, G = replicate(box, pos, species, gids0, max(1, npr // ranks_per_replica))
        n = len(P)
        ev = DeviceEvaluator(model, n_ranks=npr, scheme=scheme, device=device, precision=precision,
                             world_size=world_size, world_rank=world_rank, nccl_id=nccl_id)
        d_pos = torch.from_numpy(P).to(dev)
        d_sp = torch.from_numpy(S).to(dev)
        d_gid = torch.from_numpy(G).to(dev)
        d_out = torch.zeros(10 + 4 * n, dtype=torch.float64, device=dev)
        for _ in range(warmup):
            ev.compute_device(n, d_pos.data_ptr(), d_sp.data_ptr(), d_gid.data_ptr(), B, d_out.data_ptr())
        ev.set_trace(spans=False, ledger=True)
        busy: Dict[int, List[float]] = {}
        coll: List[float] = []
        for s in range(steps):
            ev.clear_trace()
            ev.set_step(s)
            ev.compute_device(n, d_pos.data_ptr(), d_sp.data_ptr(), d_gid.data_ptr(), B, d_out.data_ptr())
            kt = dict()
            for name, ms in ev.kernel_times():
                kt[name] = kt.get(name, 0.0) + ms
            nccl_ms = sum(v for k, v in kt.items() if k.startswith("nccl_"))
            # step-global phases: gather_positions (ownership kernel) + the NCCL collectives
            coll.append(1e-3 * (kt.get("owner", 0.0) + nccl_ms))
            for r in range(npr):
                if r % world_size != world_rank:
                    continue
                st = ev.rank_stats(r)
                secs = (1e-3 * st["dd_ms"], 1e-3 * st["neighbor_ms"], 1e-3 * st["inference_ms"],
                        1e-3 * max(0.0, st["comm_ms"] - nccl_ms))
                busy.setdefault(r, []).append(sum(secs))
                for ph, t in zip(PHASE_CSV, secs):
                    rank_rows.append(f"{s},{r},{st['locals']},{st['ghosts']},{ph},{_csv(t)},0")
            for (step, kind, nbytes, parts) in ev.ledger():
                rank_rows.append(f"{step},-1,,,{kind},,{nbytes}")
                ledger_rows.append(f"{npr},{step},{kind},{nbytes},{parts}")
        slowest = max(min(v) for v in busy.values())
        step_est = min(coll) + slowest
        tr = throughput_per_day(1, dt, step_est)
        points_rows.append(f"{mode},{npr},{n},{_csv(step_est)},{_csv(tr)}")
        points.append({"mode": mode, "n_ranks": npr, "n_atoms": n, "step_seconds": step_est, "throughput": tr,
                       "slowest_rank_busy_s": slowest, "collective_s": min(coll)})
        print(f"sweep {mode}: n_ranks {npr} atoms {n} step {step_est:.6g} s, throughput {tr:.6g}", flush=True)
        ev.close()
        del d_pos, d_sp, d_gid, d_out
        torch.cuda.empty_cache()
    if world_rank == 0:
        for name, rows in (("sweep.csv", points_rows), ("sweep_rank_phases.csv", rank_rows),
                           ("ledger.csv", ledger_rows)):
            with open(os.path.join(out, name), "w") as f:
                f.write("\n".join(rows) + "\n")
    return points


def read_points(points_csv: str) -> List[Tuple[float, float]]:
    pts = []
    with open(points_csv) as f:
        next(f)
        for line in f:
            if not line.strip():
                continue
            cells = line.strip().split(",")
            if len(cells) < 5:
                raise ValueError(f"fit-scaling: bad row '{line.strip()}'")
            pts.append((float(cells[1]), float(cells[4])))
    return pts


def fit_scaling(points_csv: str, out: str, reference: int = 0, weak: bool = False) -> dict:
    """cmd_fit_scaling (cli.cpp:739-800): scaling_fit.json and efficiency.csv."""
    pts = read_points(points_csv)
    fit = fit_throughput(pts)
    tr_by_rank = {int(n): t for n, t in pts}
    ref = reference if reference > 0 else min(tr_by_rank)
    eff = scaling_efficiency(tr_by_rank, ref, weak)
    os.makedirs(out, exist_ok=True)
    res = dict(fit, reference=ref, weak=weak)
    with open(os.path.join(out, "scaling_fit.json"), "w") as f:
        json.dump(res, f, indent=2)
    rows = ["n_ranks,throughput,efficiency,model_throughput"]
    for n_, t in sorted(tr_by_rank.items()):
        rows.append(f"{n_},{_csv(t)},{_csv(eff[n_])},{_csv(predict_throughput(fit['alpha'], fit['beta'], n_))}")
    with open(os.path.join(out, "efficiency.csv"), "w") as f:
        f.write("\n".join(rows) + "\n")
    res["efficiency"] = eff
    return res


def main(argv=None):
    ap = argparse.ArgumentParser(description="cmd_sweep + cmd_fit_scaling on B200")
    ap.add_argument("--mode", choices=["strong", "weak"], default="strong")
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--atoms", type=int, default=15668)
    ap.add_argument("--rc", type=float, default=6.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--scheme", choices=["masked", "wide"], default="masked")
    ap.add_argument("--ranks-per-replica", type=int, default=1)
    ap.add_argument("--dt", type=float, default=0.002, help="ps per step (2 fs, PAPER.md:305)")
    ap.add_argument("--out", default="sweep_out")
    args = ap.parse_args(argv)
    from . import init_model, paper_spec, synth_system
    box, pos, sp = synth_system(args.atoms, 0.1, 0.9, 1)
    model = init_model(paper_spec(args.rc), 1)
    sweep(model, box, pos, sp, mode=args.mode, ranks=args.ranks, steps=args.steps,
          scheme=0 if args.scheme == "masked" else 1, ranks_per_replica=args.ranks_per_replica, dt=args.dt,
          out=args.out)
    res = fit_scaling(os.path.join(args.out, "sweep.csv"), args.out, weak=args.mode == "weak")
    print(json.dumps({k: v for k, v in res.items() if k != "residuals"}, default=str))


if __name__ == "__main__":
    main()
