"""Print the fused-MLP per-CTA item timeline saved by bench.py (CB_TRACE_SEL=200 CB_TRACE_OUT=x.npy)."""
import sys

import numpy as np

a = np.load(sys.argv[1])[:148 * 12].reshape(148, 12)
t0 = a[a > 0].min()
for c in range(0, 148, int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    row = a[c]
    print(f"{c:3d} | " + " | ".join(f"{(row[2 * i] - t0) / 1e3:6.1f}->{(row[2 * i + 1] - t0) / 1e3:6.1f}"
                                    for i in range(5) if row[2 * i] > 0) + f" || merge {(row[10] - t0) / 1e3:6.1f}->{(row[11] - t0) / 1e3:6.1f}")
