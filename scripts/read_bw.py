"""Read-only HBM bandwidth probes (torch reductions over 8 GB) vs copy."""
import torch
x = torch.empty(4 << 30, dtype=torch.bfloat16, device="cuda").uniform_()
y = torch.empty_like(x)
for name, fn, nbytes in [("sum (read)", lambda: x.sum(dtype=torch.float32), x.numel() * 2),
                         ("amax (read)", lambda: x.amax(), x.numel() * 2),
                         ("copy (r+w)", lambda: y.copy_(x), 2 * x.numel() * 2)]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name:12s} {nbytes / ms / 1e6:8.0f} GB/s")
