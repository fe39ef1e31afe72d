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
if os.environ.get("SEL_G"):
    p.set_option("groups", int(os.environ["SEL_G"]))

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
    rows.append((i, [round(m / max(c, 1) * 1000, 1) for m, c in zip(ms, n)], round(r["sz_entropy"], 2), r["choice"]))
for row in rows:
    print("field", *row)
# k_batch per-phase cycle breakdown (warp 0 of each CTA)
import ctypes
buf = torch.zeros(148 * 8 + 16, dtype=torch.int64, device="cuda")
sel.lib().sel_dev_batch_profile(ctypes.c_void_p(buf.data_ptr()))
p.set_option("kernel_timing", 0)
p.estimate_batch(fields)
torch.cuda.synchronize()
v = buf[:148 * 8].view(148, 8).double().cpu().numpy()
q = buf[148 * 8:].double().cpu().numpy() / 148
print("flush parts per CTA (ovf, bar1, hist, bar2):", [f"{x/1e3:.1f}k" for x in q[:4]])
print("data wait per CTA before (T, R, F/other):", [f"{x/1e3:.1f}k" for x in q[4:7]])
names = ["wait", "flush+publish", "T", "R", "F", "release"]
tot = v[:, :6].sum(1)
print("k_batch warp-0 cycles per CTA (mean):", {n: f"{v[:, k].mean()/1e3:.1f}k ({v[:, k].mean()/tot.mean()*100:.0f}%)" for k, n in enumerate(names)})
print("flushes per CTA %.1f, publishes per warp0 %.1f" % (v[:, 6].mean(), v[:, 7].mean()))
print("CTA total spread: min %.1fk max %.1fk" % (tot.min()/1e3, tot.max()/1e3))
pr = buf[148 * 8 + 8:148 * 8 + 12].double().cpu().numpy() / 148
print("producer per CTA: total %.1fk, empty-wait %.1fk, decode %.1fk, tasks %.0f -> %.0f cycles/task decode, %.0f cycles/task total"
      % (pr[0] / 1e3, pr[1] / 1e3, pr[2] / 1e3, pr[3], pr[2] / max(pr[3], 1), pr[0] / max(pr[3], 1)))
sel.lib().sel_dev_batch_profile(None)
