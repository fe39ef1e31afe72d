"""Developer probe: k_batch<3> with the value range on the range warps (option
range_warps = 1) against the R-task path (= 0): results must be identical, time both.

    python scripts/exp_rw.py [c3,c4,big]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel


def timed(fields, eb, opts, reps=5):
    p = sel.Plan(tuple(fields[0].shape), eb, "rel")
    for k, v in opts.items():
        p.set_option(k, v)
    buf = p.results_buffer(len(fields))
    for _ in range(2):
        p.estimate_batch_async(fields, buf)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        p.estimate_batch_async(fields, buf)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res = p.decode_results(buf, len(fields))
    p.close()
    return ms, res


def compare(label, fields, eb, variants):
    base = None
    for name, opts in variants:
        ms, res = timed(fields, eb, opts)
        gbs = len(fields) * fields[0].numel() * 4 / ms / 1e6
        same = "-"
        if base is None:
            base = res
        else:
            same = all(a == b or (a != a and b != b) for ra, rb in zip(base, res) for a, b in
                       ((ra[k], rb[k]) for k in ra))
        print(f"{label} eb={eb:g} {name}: {ms:.3f} ms  {gbs:.0f} GB/s  identical={same}", flush=True)


SEL = set((sys.argv[1] if len(sys.argv) > 1 else "c3,c4,big").split(","))
V = [("rw=0", {"range_warps": 0}), ("rw=1", {"range_warps": 1})]
if "c4" in SEL:
    f = [torch.from_numpy(synth.make_field(4, i)).cuda() for i in range(6)]
    compare("C4", f, 1e-4, V)
    compare("C4[:1]", f[:1], 1e-4, V)
    compare("C4[:2]", f[:2], 1e-4, V)
    del f
if "c3" in SEL:
    f = [torch.from_numpy(synth.make_field(3, i)).cuda() for i in range(13)]
    for eb in (1e-3, 1e-5):
        compare("C3", f, eb, V)
    del f
if "big" in SEL:
    torch.manual_seed(1)
    x = torch.randn(1024, 1024, 1024, device="cuda")
    x += torch.linspace(-4, 4, 1024, device="cuda")[:, None, None]
    compare("1024^3 noise+ramp", [x], 1e-2, V)
    compare("1024^3 noise+ramp", [x], 1e-4, V)
