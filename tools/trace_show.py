"""Print a CTA-pair GEMM event trace saved by bench.py (CB_TRACE_SEL=100+kind CB_TRACE_OUT=x.npy).
python tools/trace_show.py x.npy [max_ctas]"""
import sys

import numpy as np

EV = ["start", "tma_done", "mma_done", "tfull", "flag_ok", "epi_done", "end", "exit"]
a = np.load(sys.argv[1])
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 128
t, ch = a[:1024].reshape(128, 8), a[1024:].reshape(128, 8)
used = np.where(t[:, 0] > 0)[0][:lim]
t0 = t[used, 0].min()
f = lambda x: np.where(x > 0, (x - t0) / 1000.0, np.nan)
print("cta  " + " ".join(f"{e:>9s}" for e in EV) + "   | epilogue chunk ends (warp 2)")
for i in used:
    print(f"{i:4d} " + " ".join(f"{x:9.2f}" for x in f(t[i])) + "   | " + " ".join(f"{x:6.2f}" for x in f(ch[i])))
