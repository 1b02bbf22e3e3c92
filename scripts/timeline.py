"""Busy warps over time from a PMS8G_TIMELINE dump (diagnostics).
usage: PMS8G_TIMELINE=/tmp/tl.bin python scripts/profile_run.py L D 0 1 stride; python scripts/timeline.py /tmp/tl.bin [bins]"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 2)
bins = int(sys.argv[2]) if len(sys.argv) > 2 else 25
start = a[:, 0].astype(np.int64)
kind = (a[:, 1] >> np.uint64(62)).astype(np.int64)
end = (a[:, 1] & np.uint64((1 << 62) - 1)).astype(np.int64)
t0, t1 = start.min(), end.max()
span = t1 - t0
print(f"{len(a)} tasks over {span / 1e6:.1f} ms; by kind (0 static, 1 donated range, 2 donated nodes): "
      + ", ".join(f"{k}: {int((kind == k).sum())} tasks {float((end - start)[kind == k].sum()) / 1e6:.0f} warp-ms" for k in range(3)))
edges = np.linspace(t0, t1, bins + 1)
for b in range(bins):
    lo, hi = edges[b], edges[b + 1]
    row = []
    for k in range(3):
        m = kind == k
        ov = np.clip(np.minimum(end[m], hi) - np.maximum(start[m], lo), 0, None).sum()
        row.append(ov / (hi - lo))
    print(f"  {(lo - t0) / 1e6:7.1f} ms  busy warps: static {row[0]:7.1f}  range {row[1]:7.1f}  nodes {row[2]:7.1f}  total {sum(row):7.1f}")
