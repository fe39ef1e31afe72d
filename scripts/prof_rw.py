"""Developer probe (SEL_BATCH_PROF=1 builds): k_batch per-CTA cycle counters on C4."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nfs = [int(a) for a in (sys.argv[2] if len(sys.argv) > 2 else "1,6").split(",")]
fields = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(max(nfs))]
eb = synth.CONFIGS[cfg]["eb_rel"][0]
for nf in nfs:
  for rw in (0, 1):
    p = sel.Plan(tuple(fields[0].shape), eb, "rel")
    p.set_option("range_warps", rw)
    buf = torch.zeros(148 * 8 + 16, dtype=torch.int64, device="cuda")
    p.estimate_batch(fields[:nf]); torch.cuda.synchronize()
    sel.lib().sel_dev_batch_profile(ctypes.c_void_p(buf.data_ptr()))
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); p.estimate_batch(fields[:nf]); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    v = buf[:148 * 8].view(148, 8).double().cpu().numpy()
    q = buf[148 * 8:].double().cpu().numpy() / 148
    names = ["wait", "flush+publish", "T", "R", "F", "release"]
    tot = v[:, :6].sum(1)
    print(f"nf={nf} rw={rw}: {ms:.3f} ms;", {n: f"{v[:, k].mean()/1e3:.0f}k ({v[:, k].mean()/tot.mean()*100:.0f}%)" for k, n in enumerate(names)},
          "tot %.0fk" % (tot.mean() / 1e3))
    print("   tile_consume alone per CTA: %.0fk cycles = %.3f cycles/value/SM" % (v[:, 6].mean() / 1e3, v[:, 6].mean() * 148 / (nf * fields[0].numel())))
    print("   data wait per CTA before (T, R, F/other):", [f"{x/1e3:.0f}k" for x in q[4:7]])
    pr = buf[148 * 8 + 8:148 * 8 + 12].double().cpu().numpy() / 148
    print("   producer per CTA: total %.0fk, empty-wait %.0fk, decode %.0fk, tasks %.0f" % (pr[0] / 1e3, pr[1] / 1e3, pr[2] / 1e3, pr[3]))
    sel.lib().sel_dev_batch_profile(None)
    p.close()
