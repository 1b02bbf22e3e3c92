"""Active warps over time from a PMS8G_TIMELINE dump (diagnostics).
usage: python scripts/timeline.py dump.bin total_warps [bins]"""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 2)
W = int(sys.argv[2])
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 40
st = a[:, 0].astype(np.int64)
en = (a[:, 1] & np.uint64((1 << 62) - 1)).astype(np.int64)
kind = (a[:, 1] >> np.uint64(62)).astype(np.int64)
t0, t1 = st.min(), en.max()
T = t1 - t0
print(f"{len(a)} tasks over {T / 1e6:.2f} ms; static {np.sum(kind == 0)} ranges {np.sum(kind == 1)} nodes {np.sum(kind == 2)}")
edges = np.linspace(t0, t1, nb + 1)
busy = np.zeros((3, nb))
for k in range(3):
    s, e = st[kind == k], en[kind == k]
    for b in range(nb):
        lo, hi = edges[b], edges[b + 1]
        busy[k, b] = np.clip(np.minimum(e, hi) - np.maximum(s, lo), 0, None).sum() / (hi - lo)
last_static_claim = st[kind == 0].max() - t0
print(f"last static task claimed at {last_static_claim / 1e6:.2f} ms")
for b in range(nb):
    tot = busy[:, b].sum()
    print(f"{(edges[b] - t0) / 1e6:7.2f} ms  busy warps {tot:7.1f} ({tot / W:5.1%})  static {busy[0, b]:7.1f} "
          f"ranges {busy[1, b]:6.1f} nodes {busy[2, b]:6.1f}")
