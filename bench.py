#!/usr/bin/env python
"""Benchmark: one DPA-1 force evaluation per MD step (BASELINE.json north star).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--rc 6]
                  [--weak] [--scheme masked|wide]

* step     = one DpProvider::evaluate of the whole system: DD build, canonical neighbour
             rows, DPA-1 forward + exact backward, force/virial assembly and (N > 1) the
             NCCL force reduction -- the reference's dd_evaluate (decomp.cpp:265-542).
* workload = configs[1]: 1HCI-sized synthetic solvated protein, 15,668 atoms, rho 0.1/A^3,
             paper-sized DPA-1 (1,584,945 random-init params, seed 1), rc 6 A, n_max 160.
             N > 1: the same system strong-scaled over N DD ranks (one per GPU); --weak
             replicates it N times along x (cli.cpp:654-669).
* value    = steps/s of the whole job, inputs resident in HBM, CUDA events on the
             library's stream, max over ranks, L2 flushed (256 MB write) between steps.
* e2e      = steps/s through the C-ABI host entry point (nnmd_b200_compute) from pinned
             host buffers: H2D of coords/types/gids and D2H of energy/virial/forces/
             per-atom energies inside the timed region (wall clock, max over ranks).
* reference arm (--impl reference) = the compiled reference (oracle/_ref, built from the
             unmodified sources) on this box's host cores, rank 0 only, inputs from the
             oracle's own generator (no product library in that process).  One FULL
             force evaluation is timed, tiled over the K timed steps: step i runs the
             reference's per-step work for centres [i*n/K, (i+1)*n/K) --
             build_neighbor_list + the stock evaluate_dp with a LocalMask, split over all
             host threads.  value = 1 / (mean list build + sum of the K slice
             evaluations), i.e. full steps/s; the whole timed region is one full step.
* --gpus N without WORLD_SIZE in the environment re-launches itself under
             torch.distributed.run (N ranks, 127.0.0.1); NCCL_DEBUG=INFO goes to stderr.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DT_FS = 2.0
N_ATOMS = 15668
RHO = 0.1


def ns_per_day(steps_per_s):
    return steps_per_s * 86400.0 * DT_FS * 1e-6


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def make_system(n_gpus, weak, seed=1, replicas=0, oracle_gen=False):
    """configs[1] system (replicated along x for weak scaling, cli.cpp:654-669).  The
    reference arm uses the oracle's generator (bitwise equal, tests/test_oracle.py) so
    that its process never maps the product library."""
    if oracle_gen:
        import oracle as O
        box, pos, sp = O.Port().synth_system(N_ATOMS, RHO, 0.9, seed)
    else:
        import paper_2604_07276_b200 as nb
        box, pos, sp = nb.synth_system(N_ATOMS, RHO, 0.9, seed)
    reps = replicas if replicas > 0 else (n_gpus if weak else 1)
    if reps > 1:
        pos = np.concatenate([pos + np.array([k * box[0], 0.0, 0.0]) for k in range(reps)])
        sp = np.concatenate([sp] * reps)
        box = np.array([box[0] * reps, box[1], box[2]])
    return box, np.ascontiguousarray(pos), np.ascontiguousarray(sp, dtype=np.int32)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return ws, rank, local


def allmax(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def bcast_bytes(b, ws):
    if ws == 1:
        return b
    import torch
    import torch.distributed as dist
    t = torch.frombuffer(bytearray(b if b is not None else bytes(128)), dtype=torch.uint8).clone()
    dist.broadcast(t, src=0)
    return bytes(t.numpy().tobytes())


# ---------------------------------------------------------------------------------------
def cpu_reference_sample(box, pos, sp, rc, n_sample, seed=0):
    """cpu_baseline leg of our arm: compiled reference on host cores, neighbour list +
    n_sample random centres (center_rows + evaluate_center, fwd+bwd), extrapolated."""
    import oracle as O
    R = O.Ref()
    spec = dict(O.PAPER_SPEC, rc=rc, rcs=0.55 * rc, n_max=O.nmax_for_rc(rc))
    h = R.model_init(spec, 1)
    rng = np.random.default_rng(seed)
    centres = np.sort(rng.choice(len(pos), size=min(n_sample, len(pos)), replace=False)).astype(np.int32)
    threads = host_threads()
    t_list, t_cent, _ = R.time_centers(h, pos, sp, box, centres, threads)
    R.model_free(h)
    t_step = t_list + t_cent * len(pos) / len(centres)
    return dict(value=1.0 / t_step, t_step=t_step, t_list=t_list, t_centres=t_cent, cores=threads,
                sample=f"build_neighbor_list({len(pos)} atoms) + {len(centres)} random centres "
                       f"(center_rows+evaluate_center, fwd+bwd) on {threads} threads, extrapolated x{len(pos)/len(centres):.1f}")


def workload_config(args, n, ws):
    """The config dict both arms print (the driver compares them)."""
    return {"workload": f"1HCI-sized synthetic solvated protein, {n} atoms, DPA-1 1.58M params, rc={args.rc} A, "
                        f"{'weak' if args.weak else 'strong'} DD over {args.gpus} GPU(s)",
            "n_atoms": n, "rc": args.rc, "n_max": {4.0: 64, 6.0: 160, 8.0: 320}.get(float(args.rc), 160),
            "dd_ranks": args.gpus, "scheme": args.scheme, "model_seed": 1, "system_seed": 1,
            "l2": "flushed between steps (256 MB write)"}


def run_reference(args, ws, rank):
    """The reference's own CPU implementation on this box's host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle as O
    box, pos, sp = make_system(args.gpus, args.weak, replicas=args.replicas, oracle_gen=True)
    n = len(pos)
    R = O.Ref()
    spec = dict(O.PAPER_SPEC, rc=args.rc, rcs=0.55 * args.rc, n_max=O.nmax_for_rc(args.rc))
    h = R.model_init(spec, 1)
    threads = host_threads()
    for i in range(args.warmup):  # untimed: a few centres to fault in code, weights and pages
        R.step_slice(h, pos, sp, box, (i * 97) % (n - 8), (i * 97) % (n - 8) + 8, threads)
    K = max(1, args.steps)
    bounds = [n * i // K for i in range(K + 1)]
    t_list, t_eval, e_sum = [], [], 0.0
    for i in range(K):
        if bounds[i + 1] <= bounds[i]:
            continue
        tl, te, e = R.step_slice(h, pos, sp, box, bounds[i], bounds[i + 1], threads)
        t_list.append(tl)
        t_eval.append(te)
        e_sum += e
    R.model_free(h)
    t_step = float(np.mean(t_list)) + float(np.sum(t_eval))
    v = 1.0 / t_step
    sample = (f"one full force evaluation of all {n} centres, tiled over the {K} timed steps (step i = "
              f"build_neighbor_list + stock evaluate_dp with a LocalMask over centres [i*n/K, (i+1)*n/K) on "
              f"{threads} host threads); value = 1 / (mean list build + sum of slice evaluations)")
    line = {"impl": "reference", "metric": "MD steps/s (DPA-1 force evaluation per step)", "value": v,
            "unit": "steps/s", "higher_is_better": True, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * t_step, "ns_per_day": ns_per_day(v),
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic solvated protein (oracle synth_system seed 1 == nnmd_synth_system), "
                    "random-init DPA-1 weights (reference init_model seed 1)",
            "config": workload_config(args, n, ws),
            "timed_region_s": float(np.sum(t_list) + np.sum(t_eval)),
            "full_steps_timed": 1,
            "t_list_s_mean": float(np.mean(t_list)), "t_eval_s_sum": float(np.sum(t_eval)),
            "energy": e_sum,
            "cpu_baseline": {"value": v, "unit": "steps/s", "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
def algorithmic_flops(counts):
    """SURVEY 8(d) per-centre work of the reference algorithm (MACs -> x2 FLOP).
    centre_backward (dominant kernel): B(n) minus the fitting net, run in k_fit."""
    n = counts.astype(np.float64)
    fwd = 2.0 * (404640 * n + 1548 * n * n + 1196288 - 1179904)
    bwd = 2.0 * (405280 * n + 3084 * n * n + 1212672 - 1179904)
    return fwd.sum(), bwd.sum()


def executed_flops(counts, M=128, E=(32, 64), na=3):
    """FLOPs the folded kernels execute (attention re-associated; SIMT, no padding)."""
    n = counts.astype(np.float64)
    emb = n * (E[0] * E[1] + E[1] * M)
    att_f = na * (n * M * 2 * M + 2 * n * n * M)
    att_b = na * (n * M * 2 * M + 2 * n * n * M) + na * (4 * n * n * M + n * 2 * M * M)
    return 2 * (emb + att_f).sum(), 2 * (2 * emb + att_b).sum()


def run_ours(args, ws, rank, local):
    import torch
    import paper_2604_07276_b200 as nb
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    box, pos, sp = make_system(args.gpus, args.weak, replicas=args.replicas)
    n = len(pos)
    model = nb.init_model(nb.paper_spec(args.rc), 1)
    uid = nb.DeviceEvaluator.nccl_unique_id() if (ws > 1 and rank == 0) else None
    uid = bcast_bytes(uid, ws) if ws > 1 else None
    scheme = nb.WIDE_HALO if args.scheme == "wide" else nb.MASKED_REDUCTION
    prec = {"fp32": nb.PREC_FP32, "tf32": nb.PREC_TF32, "simt": nb.PREC_FP32_SIMT}[args.precision]
    ev = nb.DeviceEvaluator(model, n_ranks=ws, scheme=scheme, device=local, world_size=ws, world_rank=rank,
                            nccl_id=uid, precision=prec)
    stream = torch.cuda.ExternalStream(ev.stream(), device=dev)
    d_pos = torch.from_numpy(pos).to(dev)
    d_sp = torch.from_numpy(sp).to(dev)
    d_gid = torch.arange(n, dtype=torch.int64, device=dev)
    d_out = torch.zeros(10 + 4 * n, dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    torch.cuda.synchronize()

    def step():
        ev.compute_device(n, d_pos.data_ptr(), d_sp.data_ptr(), d_gid.data_ptr(), box, d_out.data_ptr())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = nb.lib().nnmd_b200_launch_count()
    ev_times = []
    kernel_acc = {}
    with ClockSampler(local) as clk:
        barrier(ws)
        torch.cuda.synchronize()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
            step()
            b.record(stream)
            b.synchronize()
            ev_times.append(a.elapsed_time(b))
            for name, ms in ev.kernel_times():
                kernel_acc[name] = kernel_acc.get(name, 0.0) + ms
        torch.cuda.synchronize()
        barrier(ws)
    launches = nb.lib().nnmd_b200_launch_count() - launches0
    ms_step = allmax(float(np.mean(ev_times)), ws)
    ms_median = allmax(float(np.median(ev_times)), ws)  # SURVEY 8(d) quotes the median step
    value = 1000.0 / ms_step
    stats = ev.rank_stats(rank)
    clocks = clk.summary()

    # ---- roofline of the dominant kernel (centre_backward), per launch
    res = d_out[10:10 + 3 * n].cpu()
    ev.set_debug(True)
    step()
    _, _, _, cnt = ev.debug_nlist(rank, nb.paper_spec(args.rc).n_max)
    ev.set_debug(False)
    f_fwd, f_bwd = algorithmic_flops(cnt)
    x_fwd, x_bwd = executed_flops(cnt)
    npass = {"fp32": 3, "tf32": 1, "simt": 1}[args.precision]
    k_bwd = kernel_acc.get("centre_backward", 0.0) / args.steps
    k_fwd = kernel_acc.get("centre_forward", 0.0) / args.steps
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    # the kernel is timed per launch at full clock (no power cap seen): burst peak
    peak = peaks.get("bf16_tflops", 1622.5)
    traffic, traffic_src = None, None
    try:  # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
        nc = json.load(open(os.path.join(ROOT, "profiles", "ncu_latest.json")))
        traffic = nc["k_centre_backward"]["dram_bytes"]
        traffic_src = ("profiles/ncu_latest.json: dram__bytes_read.sum + dram__bytes_write.sum of one "
                       f"ncu --set full capture ({nc.get('_source', 'earlier run')}), not this run")
    except Exception:
        pass
    achieved = f_bwd / (k_bwd * 1e-3) / 1e12 if k_bwd > 0 else 0.0

    # ---- HBM-bound kernels: SURVEY 8(d) algorithmic bytes per launch / event time
    hbm_peak = peaks.get("hbm_gbs", 6552.3)
    sum_n = float(cnt.sum())
    n_c = float(len(cnt))
    members = float(stats["locals"] + stats["ghosts"])
    n_max = nb.paper_spec(args.rc).n_max
    # the environment matrix is built inside the centre-list kernel (k_neighbors writes
    # R, Z, sigma), so its bytes are counted with that launch
    alg = {
        "neighbors_env": (members * 36 + n_c * n_max * 4                  # pos f64x3 + species + gid; nlist
                          + sum_n * (4 + 8 + 24 + 4 + 16 + 4) + n_c * 40),  # env: nlist, member, pos, species -> R, Z
        "force_gather": sum_n * (24 + 4) + members * 24,                  # f64 row grads + index; f64 member forces
    }
    timer_of = {"neighbors_env": "neighbors", "force_gather": "force_gather"}
    hbm = {}
    for k, b in alg.items():
        ms = kernel_acc.get(timer_of[k], 0.0) / args.steps
        if ms > 0:
            gbs = b / (ms * 1e-3) / 1e9
            hbm[k] = {"algorithmic_bytes": b, "ms_per_launch": ms, "achieved_gbs": gbs, "peak_gbs": hbm_peak,
                      "frac": gbs / hbm_peak}

    # ---- e2e through the host C-ABI entry point (pinned host buffers)
    h_pos = torch.from_numpy(pos).pin_memory().numpy()
    h_sp = torch.from_numpy(sp).pin_memory().numpy()
    h_gid = torch.arange(n, dtype=torch.int64).pin_memory().numpy()
    for _ in range(max(1, args.warmup)):
        ev.compute(h_pos, h_sp, box, gids=h_gid)
    barrier(ws)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = ev.compute(h_pos, h_sp, box, gids=h_gid)
    t_e2e = allmax((time.perf_counter() - t0) / args.steps, ws)
    e2e = 1.0 / t_e2e
    h2d = ws * n * (24 + 4 + 8)
    d2h = ws * (8 * 10 + n * 24 + n * 8)

    # ---- full MD steps through the device-resident loop (nnmd_b200_run_md_device): force
    # evaluation + leap-frog + energies per step, positions/velocities resident in HBM
    rng = np.random.default_rng(7)
    masses = np.where(sp == 0, 1.008, 12.0).astype(np.float64)
    d_mpos = torch.from_numpy(pos.copy()).to(dev)
    d_vel = torch.from_numpy(rng.normal(0.0, 0.01, size=(n, 3))).to(dev)
    d_mass = torch.from_numpy(masses).to(dev)
    d_en = torch.zeros(2 * max(args.steps, args.warmup, 1), dtype=torch.float64, device=dev)
    md_dt = 0.0005  # reduced units of the reference CLI; ns/day below uses the paper's 2 fs

    def md(k):
        ev.run_md_device(n, d_mpos.data_ptr(), d_vel.data_ptr(), d_mass.data_ptr(), d_sp.data_ptr(),
                         d_gid.data_ptr(), box, md_dt, k, d_en.data_ptr())

    md(args.warmup)
    torch.cuda.synchronize()
    barrier(ws)
    t0 = time.perf_counter()
    md(args.steps)
    torch.cuda.synchronize()
    t_md = allmax((time.perf_counter() - t0) / args.steps, ws)
    md_loop = {"value": 1.0 / t_md, "unit": "MD steps/s", "ns_per_day": ns_per_day(1.0 / t_md),
               "api": "nnmd_b200_run_md_device (DPA-1 forces + leap-frog, state resident in HBM)",
               "e_total_first_last": [float(d_en[1].item()), float(d_en[2 * args.steps - 1].item())]}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        c = cpu_reference_sample(box, pos, sp, args.rc, args.ref_sample)
        cpu = {"value": c["value"], "unit": "steps/s", "cores": c["cores"], "kind": "reference", "sample": c["sample"]}

    if rank == 0:
        line = {
            "metric": "MD steps/s (DPA-1 force evaluation per step)", "value": value, "unit": "steps/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_median": ms_median,
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
            "dtype": {"fp32": "f32 (3xTF32 tcgen05)", "tf32": "tf32", "simt": "f32 (SIMT)"}[args.precision], "data": "synthetic solvated protein (nnmd_synth_system seed 1), random-init DPA-1 weights (init_model seed 1)",
            "nccl": nccl_info(ws),
            "ns_per_day": ns_per_day(value),
            "config": dict(workload_config(args, n, ws),
                           precision={"fp32": "3xTF32 tcgen05 (FP32-grade, tol 1e-5)", "tf32": "1xTF32 tcgen05 (tol 5e-3)",
                                      "simt": "FP32 SIMT (tol 1e-5)"}[args.precision] + "; fp64 geometry/forces"),
            "e2e": {"value": e2e, "unit": "steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ns_per_day": ns_per_day(e2e)},
            "roofline": {"bound": "tensor", "kernel": "k_centre_backward", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_flop_per_launch": f_bwd, "ms_per_launch": k_bwd,
                         "executed_tflops": npass * x_bwd / (k_bwd * 1e-3) / 1e12 if k_bwd > 0 else 0.0,
                         "mma_passes": npass,
                         "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst; kernel timed per launch)",
                         "forward": {"ms_per_launch": k_fwd, "algorithmic_flop": f_fwd,
                                     "achieved_tflops": f_fwd / (k_fwd * 1e-3) / 1e12 if k_fwd > 0 else 0.0}},
            "hbm_kernels": hbm,
            "md_loop": md_loop,
            "kernel_ms_per_step": {k: v / args.steps for k, v in sorted(kernel_acc.items(), key=lambda x: -x[1])},
            "rank0_stats": stats,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cpu_baseline": cpu,
            "energy": float(d_out[0].item()),
        }
        print(json.dumps(line), flush=True)
    ev.close()


def nccl_info(ws):
    """What NCCL reported at communicator init (NCCL_DEBUG=INFO), for the rank count check."""
    return {"world_size": ws, "NCCL_DEBUG": os.environ.get("NCCL_DEBUG"),
            "debug_file": os.environ.get("NCCL_DEBUG_FILE"), "backend": "nccl" if ws > 1 else "none (1 process)"}


def respawn_under_torchrun(n):
    """`bench.py --gpus N` outside torchrun: launch N ranks (one per GPU) ourselves."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--rc", type=float, default=6.0)
    ap.add_argument("--weak", action="store_true")
    ap.add_argument("--replicas", type=int, default=0,
                    help="replicate the 15,668-atom box this many times along x (cli.cpp:654-669) on the given "
                         "GPUs; default: --gpus with --weak, else 1")
    ap.add_argument("--scheme", choices=["masked", "wide"], default="masked")
    ap.add_argument("--ref-sample", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", choices=["fp32", "tf32", "simt"], default="fp32",
                    help="fp32 = 3xTF32 tcgen05 (FP32-grade, default); tf32 = 1xTF32 tcgen05; simt = CUDA-core FP32")
    args = ap.parse_args()
    # NCCL init lines ("... rank r nranks N ... Init COMPLETE") to stderr; stdout keeps the
    # one JSON line
    os.environ["NCCL_DEBUG"] = "INFO"  # (the boxes preset VERSION)
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(respawn_under_torchrun(args.gpus))
    ws, rank, local = dist_setup()
    if ws != args.gpus and args.impl == "ours":
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {ws}")
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
