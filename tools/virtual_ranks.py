"""Per-rank cost of the DD decomposition on ONE GPU: the 15,668-atom system evaluated with
R = 1, 2, 4, 8 DD ranks run back to back on the same device (SURVEY 8(e) grids).  Each
rank's kernels see ~N/R centres, so sum-over-ranks time minus the R = 1 time exposes the
fixed per-rank overheads that bound strong scaling across GPUs.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07276_b200 as nb  # noqa: E402

box, pos, sp = nb.synth_system(15668, 0.1, 0.9, 1)
m = nb.init_model(nb.paper_spec(6.0), 1)
out = {}
for R in (1, 2, 4, 8):
    ev = nb.DeviceEvaluator(m, n_ranks=R)
    d_pos = torch.from_numpy(pos).cuda()
    d_sp = torch.from_numpy(sp).cuda()
    d_gid = torch.arange(len(pos), dtype=torch.int64, device="cuda")
    d_out = torch.zeros(10 + 4 * len(pos), dtype=torch.float64, device="cuda")
    for _ in range(3):
        ev.compute_device(len(pos), d_pos.data_ptr(), d_sp.data_ptr(), d_gid.data_ptr(), box, d_out.data_ptr())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        ev.compute_device(len(pos), d_pos.data_ptr(), d_sp.data_ptr(), d_gid.data_ptr(), box, d_out.data_ptr())
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    st = [ev.rank_stats(r) for r in range(R)]
    out[R] = {"ms_all_ranks": ms, "max_rank_inference_ms": max(s["inference_ms"] for s in st),
              "max_rank_dd_nbr_ms": max(s["dd_ms"] + s["neighbor_ms"] for s in st),
              "centres": [s["centers"] for s in st]}
    ev.close()
t1 = out[1]["ms_all_ranks"]
for R in (2, 4, 8):
    # on R GPUs each rank would run alone: estimate = slowest rank's share of the sequential run
    est = out[R]["ms_all_ranks"] / R * (max(out[R]["centres"]) / (sum(out[R]["centres"]) / R))
    out[R]["est_ms_per_step_on_R_gpus"] = est
    out[R]["est_strong_efficiency"] = t1 / (R * est)
print(json.dumps(out))
