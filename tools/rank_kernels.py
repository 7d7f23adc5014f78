#!/usr/bin/env python
"""Per-kernel time per step, summed over DD ranks, at R = 1 and R = 8 DD ranks on one GPU:
where the strong-scaling overhead (sum over ranks minus the one-rank time) goes."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_07276_b200 as nb  # noqa: E402

box, pos, sp = nb.synth_system(15668, 0.1, 0.9, 1)
m = nb.init_model(nb.paper_spec(6.0), 1)
res = {}
for R in [int(x) for x in (sys.argv[1:] or ["1", "8"])]:
    ev = nb.DeviceEvaluator(m, n_ranks=R)
    d_pos = torch.from_numpy(pos).cuda()
    d_sp = torch.from_numpy(sp).cuda()
    d_gid = torch.arange(len(pos), dtype=torch.int64, device="cuda")
    d_out = torch.zeros(10 + 4 * len(pos), dtype=torch.float64, device="cuda")
    acc = {}
    for it in range(8):
        ev.compute_device(len(pos), d_pos.data_ptr(), d_sp.data_ptr(), d_gid.data_ptr(), box, d_out.data_ptr())
        torch.cuda.synchronize()
        if it >= 3:
            for k, v in ev.kernel_times():
                acc[k] = acc.get(k, 0.0) + v / 5
    res[R] = acc
    ev.close()
keys = sorted(res[max(res)], key=lambda k: -res[max(res)][k])
print(f"{'kernel':28s} " + " ".join(f"R={R:<8d}" for R in res))
for k in keys:
    print(f"{k:28s} " + " ".join(f"{res[R].get(k, 0.0):9.3f}" for R in res))
print(f"{'total':28s} " + " ".join(f"{sum(res[R].values()):9.3f}" for R in res))
print(json.dumps(res))
