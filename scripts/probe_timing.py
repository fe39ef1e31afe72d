"""Timing probe: batch pipeline on/off, per-kernel attribution (developer tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08901_b200 as sel
import synth

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nf = int(sys.argv[2]) if len(sys.argv) > 2 else 20
shape = synth.CONFIGS[cfg]["shape"]
fields = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
eb = synth.CONFIGS[cfg]["eb_rel"][0]
p = sel.Plan(shape, eb, "rel")

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for pipe in (1, 0):
    p.set_option("pipeline", pipe)
    ms = timeit(lambda: p.estimate_batch(fields))
    print(f"pipeline={pipe}: {ms:.3f} ms / {nf} fields = {ms/nf*1000:.1f} us/field, "
          f"{nf*fields[0].numel()*4/ms/1e6:.1f} GB/s")
p.set_option("pipeline", 1)
p.set_option("kernel_timing", 1)
p.kernel_times(reset=True)
p.estimate_batch(fields)
ms, n = p.kernel_times(reset=True)
print("per-kernel (sequential, events):", [f"{m/max(c,1)*1000:.1f}us" for m, c in zip(ms, n)])
p.set_option("kernel_timing", 0)
# single-field estimate latency
t = fields[0]
ms1 = timeit(lambda: p.estimate(t), reps=20)
print(f"single estimate(): {ms1*1000:.1f} us")
# per-field kernel times (sequential, events)
p.set_option("kernel_timing", 1)
rows = []
for i, f in enumerate(fields[:10]):
    p.kernel_times(reset=True)
    for _ in range(3):
        r = p.estimate(f)
    ms, n = p.kernel_times(reset=True)
    rows.append((i, [round(m / c * 1000, 1) for m, c in zip(ms, n)], round(r["sz_entropy"], 2), r["choice"]))
for row in rows:
    print("field", *row)
