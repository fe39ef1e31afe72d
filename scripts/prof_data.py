"""Developer probe (SEL_BATCH_PROF=1 builds): tile_consume cycles per value inside k_batch<3>
on synthetic 512^3 data of known code spread (ramp: all codes 0; ramp + noise of +-s codes)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1806_08901_b200 as sel

n = 512
g = torch.arange(n, device="cuda", dtype=torch.float32)
ramp = (g[:, None, None] + 2 * g[None, :, None] + 3 * g[None, None, :]) / (6 * n)   # VR ~ 1
torch.manual_seed(0)
for label, spread in (("ramp", 0.0), ("ramp + noise +-3 codes", 3.0), ("ramp + noise +-100 codes", 100.0),
                      ("ramp + noise +-3000 codes", 3000.0)):
    eb = 1e-4
    fields = []
    for i in range(3):
        x = ramp.clone()
        if spread:
            x += (torch.rand(n, n, n, device="cuda") - 0.5) * (2 * eb * spread / 4)   # Lorenzo of 8 terms
        fields.append(x)
    for rw in (0, 1):
        p = sel.Plan((n, n, n), eb, "rel")
        p.set_option("range_warps", rw)
        buf = torch.zeros(148 * 8 + 16, dtype=torch.int64, device="cuda")
        p.estimate_batch(fields); torch.cuda.synchronize()
        sel.lib().sel_dev_batch_profile(ctypes.c_void_p(buf.data_ptr()))
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); r = p.estimate_batch(fields); e1.record(); torch.cuda.synchronize()
        v = buf[:148 * 8].view(148, 8).double().cpu().numpy()
        print(f"{label} rw={rw}: {e0.elapsed_time(e1):.3f} ms, tile_consume {v[:, 6].mean() * 148 / (3 * n ** 3):.3f} cycles/value/SM, "
              f"all consumer buckets {v[:, :6].sum(1).mean() * 148 / (3 * n ** 3):.3f}; H={r[0]['sz_entropy']:.2f} zfp_bpv={r[0]['zfp_bits_per_value']:.2f}", flush=True)
        sel.lib().sel_dev_batch_profile(None)
        p.close()
