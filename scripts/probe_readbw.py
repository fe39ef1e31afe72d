"""Read-only HBM bandwidth reference (developer tool): torch min/max reductions over a
buffer far larger than L2, CUDA events, best of 10.  The strict metric's ceiling for a
two-read design is half of this."""
import torch
x = torch.randn(1 << 30, device="cuda")          # 4 GiB
for name, fn in (("amax", lambda: torch.amax(x)), ("aminmax", lambda: torch.aminmax(x)),
                 ("sum", lambda: x.sum())):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {x.numel() * 4 / best / 1e6:.0f} GB/s read ({best:.3f} ms)")
