"""Time sampled-block estimation (stride) on C2 / C4 fields (developer tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel
for cfg, nf, st in ((2, 20, (1, 10)), (2, 20, (1, 1)), (4, 2, (4, 4, 4)), (4, 6, (4, 4, 4))):
    fs = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
    p = sel.Plan(tuple(fs[0].shape), synth.CONFIGS[cfg]["eb_rel"][0], "rel", st)
    if os.environ.get("SEL_G"):
        p.set_option("groups", int(os.environ["SEL_G"]))
    buf = p.results_buffer(nf)
    for _ in range(2):
        p.estimate_batch_async(fs, buf)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.estimate_batch_async(fs, buf)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    p.set_option("kernel_timing", 1); p.kernel_times(reset=True)
    p.estimate_batch(fs)
    kms, kn = p.kernel_times(reset=True)
    print(f"C{cfg} stride {st} nf={nf}: {ms / nf * 1000:.1f} us/field, {nf * fs[0].numel() * 4 / ms / 1e6:.0f} GB/s; "
          f"per-kernel avg us {[round(m / max(c, 1) * 1000, 1) for m, c in zip(kms, kn)]} launches {kn}", flush=True)
    p.close(); del fs
