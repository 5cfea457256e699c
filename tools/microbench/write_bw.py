"""HBM write-only and read-only bandwidth on one B200 (torch kernels), for the QKVU roofline."""
import torch
x = torch.empty(2 * 1024**3, dtype=torch.bfloat16, device="cuda")   # 4 GiB
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def t(fn, nbytes, n=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / best / 1e6
print("write-only fill GB/s", round(t(lambda: x.fill_(1.0), x.numel() * 2)))
print("copy (r+w) GB/s", round(t(lambda: y.copy_(x), 2 * x.numel() * 2)))
print("read-only sum GB/s", round(t(lambda: x.sum(dtype=torch.float32), x.numel() * 2)))
