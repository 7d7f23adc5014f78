#!/usr/bin/env python
"""Top SASS instructions by stall samples, with the dominant stall reasons (from
tools/gpu_sass_stalls.sh's CSV).  python tools/sass_stalls.py gpurun_out/sass_stalls.csv.gz [top]"""
import csv, gzip, io, sys
rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]), encoding="utf-8")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for i, r in enumerate(rows[2:]):
    if len(r) != len(hdr):
        continue
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    data.append((s, i, r))
tot = sum(d[0] for d in data)
agg = {h: sum(int(d[2][ix[h]] or 0) for d in data) for h in stalls}
print("total", tot, " ".join(f"{h[6:]}:{100*v/tot:.1f}%" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for s, i, r in sorted(data, key=lambda x: -x[0])[:top]:
    rs = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{100*s/tot:5.2f}% #{i:5d} {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{100*v/max(s,1):.0f}" for v, n in rs if v))
