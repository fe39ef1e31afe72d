"""Single small-field latency (developer tool): device time of sel_estimate on one C1
field (256x256) through k_batch and through the per-field kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel
x = torch.from_numpy(synth.c1_field()).cuda()
for shape_scale in (1, 4):
    t = x if shape_scale == 1 else torch.from_numpy(synth.c1_field((1024, 1024))).cuda()
    for bk in (1, 0):
        sk = bk  # batch_kernel=1 routes one small field to k_small
        p = sel.Plan(tuple(t.shape), 1e-4)
        p.set_option("batch_kernel", bk)
        for _ in range(5):
            p.estimate(t)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        buf = p.results_buffer(1, "pinned")
        e0.record()
        for _ in range(200):
            p.estimate_batch_async([t], buf)
        e1.record(); torch.cuda.synchronize()
        print(f"{tuple(t.shape)} batch_kernel={bk}: {e0.elapsed_time(e1) / 200 * 1000:.1f} us per estimate (stream-ordered)")
        p.close()
