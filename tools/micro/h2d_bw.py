"""Pinned host -> device copy bandwidth: one stream vs two streams (K and V halves), 12.6 MB pieces like the
request path's per-layer fetch, and one large copy."""
import torch
import time
n_layers, piece = 32, 6 * 1024 * 1024 * 2  # one layer's K (or V): 3072 x 1024 bf16 = 6.3 MB
hk = torch.empty(n_layers * piece, dtype=torch.uint8).pin_memory()
hv = torch.empty(n_layers * piece, dtype=torch.uint8).pin_memory()
dk = torch.empty_like(hk, device="cuda")
dv = torch.empty_like(hv, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(two):
    for i in range(n_layers):
        sl = slice(i * piece, (i + 1) * piece)
        with torch.cuda.stream(s1):
            dk[sl].copy_(hk[sl], non_blocking=True)
        with torch.cuda.stream(s2 if two else s1):
            dv[sl].copy_(hv[sl], non_blocking=True)
for two in (False, True, False, True):
    torch.cuda.synchronize()
    t = time.perf_counter()
    run(two)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{'two streams' if two else 'one stream '}: {2 * n_layers * piece / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms)")
torch.cuda.synchronize(); t = time.perf_counter(); dk.copy_(hk, non_blocking=True); torch.cuda.synchronize()
print(f"one 400 MB copy: {hk.numel() / (time.perf_counter() - t) / 1e9:.1f} GB/s")
