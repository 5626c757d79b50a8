"""HBM direction probe: write-only (fill), read-only (sum), copy; best of 20, CUDA events."""
import torch
n = 1 << 30  # 1 Gi fp32 = 4 GiB
a = torch.empty(n, dtype=torch.float32, device="cuda")
b = torch.empty(n, dtype=torch.float32, device="cuda")
a.fill_(1.0); b.fill_(2.0)
def best(fn, nbytes):
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return nbytes / min(ts) / 1e9
print("write-only fill GB/s", best(lambda: a.fill_(3.0), 4 * n))
print("read-only sum GB/s", best(lambda: a.sum(), 4 * n))
print("copy (r+w) GB/s", best(lambda: b.copy_(a), 8 * n))
# strided 128-B line writes like the K2 epilogue: rows of 1225 floats, 32-float pieces
m = 65536 * 8
out = torch.empty(m, 1225, dtype=torch.float32, device="cuda")
print("fill 321MB-class buffer GB/s", best(lambda: out.fill_(1.0), out.numel() * 4))
