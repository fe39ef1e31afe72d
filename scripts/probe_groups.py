"""k_batch CTA-group sweep (developer tool): time per field for G = 1..4 per config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08901_b200 as sel
import synth

for cfg, nf in (((2, 100), (3, 10), (1, 256)) if len(sys.argv) < 2 else [tuple(map(int, a.split(":"))) for a in sys.argv[1:]]):
    shape = synth.CONFIGS[cfg]["shape"]
    fields = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
    eb = synth.CONFIGS[cfg]["eb_rel"][0]
    p = sel.Plan(shape, eb, "rel")
    buf = p.results_buffer(nf)
    ref = None
    lags = [int(v) for v in os.environ.get("SWEEP_LAG", "1").split(",")]
    Gs = ((0, 1, 2, 3, 4) if cfg != 1 else (0, 4, 8, 12, 16, 24)) if os.environ.get("SWEEP_G") else (0,)
    if os.environ.get("SWEEP_GS"):
        Gs = tuple(int(v) for v in os.environ["SWEEP_GS"].split(","))
    for lag, G in [(l, g) for l in lags for g in Gs]:
        if G > nf:
            continue
        p.set_option("groups", G)
        p.set_option("lag", lag)
        for _ in range(2):
            p.estimate_batch_async(fields, buf)
        torch.cuda.synchronize()
        res = p.decode_results(buf, nf)
        if ref is None:
            ref = res
        same = all(a == b for a, b in zip(res, ref))
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            p.estimate_batch_async(fields, buf)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gbs = nf * fields[0].numel() * 4 / ms / 1e6
        print(f"C{cfg} nf={nf} lag={lag} G={G}: {ms/nf*1000:.1f} us/field {gbs:.0f} GB/s identical={same}", flush=True)
    p.close()
    del fields
