#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (text + json).

  python tools/summarize_ncu.py TAG    # reads gpurun_out/TAG_launches.csv, TAG_*.ncu-rep

Writes profiles/TAG_launches.txt (per-kernel share of the step from the launch list) and
profiles/TAG_ncu.txt / profiles/TAG_ncu.json (key metrics per captured kernel: duration,
DRAM bytes, L2 / DRAM throughput, tensor-pipe activity, occupancy, stall ratios).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_tf32_dst_fp32.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "sm__inst_executed.avg.per_cycle_active", "lts__t_sector_hit_rate.pct",
]


def launches(tag):
    path = os.path.join(OUT, f"{tag}_launches.csv")
    if not os.path.exists(path):
        return None
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    agg = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {tag}: ncu launch list (gpu__time_duration, --clock-control none, cold-cache/serialised)",
             f"# total {tot/1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches", ""]
    for k, (c, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{100*ns/tot:6.2f}%  {ns/1e6:10.3f} ms  {c:5d} launches  {k}")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    return agg


def reports(tag):
    res = {}
    for fn in sorted(os.listdir(OUT)):
        if not (fn.startswith(tag + "_") and fn.endswith(".ncu-rep")):
            continue
        raw = subprocess.run(["ncu", "-i", os.path.join(OUT, fn), "--page", "raw", "--csv"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
            ent = {}
            for k in KEYS:
                if k in d:
                    u = units[hdr.index(k)]
                    try:
                        ent[k] = [float(d[k].replace(",", "")), u]
                    except ValueError:
                        pass
            res.setdefault(name, []).append(ent)
    lines = [f"# {tag}: ncu --set full captures (one line per captured launch)", ""]
    for name, ents in res.items():
        for e in ents:
            lines.append(name)
            for k, (v, u) in e.items():
                lines.append(f"    {k:80s} {v:16.4f} {u}")
    open(os.path.join(PROF, f"{tag}_ncu.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(res, open(os.path.join(PROF, f"{tag}_ncu.json"), "w"), indent=1)
    # per-kernel DRAM traffic per launch of the latest capture (read by bench.py roofline)
    latest = {}
    for name, ents in res.items():
        e = ents[0]
        rd = e.get("dram__bytes_read.sum", [0, "byte"])
        wr = e.get("dram__bytes_write.sum", [0, "byte"])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        latest[name.split("<")[0]] = {"tag": tag, "dram_bytes": rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1),
                                      "duration_ms": e.get("gpu__time_duration.sum", [0])[0]}
    json.dump(latest, open(os.path.join(PROF, "ncu_latest.json"), "w"), indent=1)
    return res


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    a = launches(tag)
    r = reports(tag)
    print("launch kernels:", 0 if a is None else len(a), "captured kernels:", list(r))
