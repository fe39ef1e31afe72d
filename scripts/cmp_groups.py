"""Compare k_batch results across CTA-group counts (developer tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel
cfg, nf = int(sys.argv[1]), int(sys.argv[2])
fs = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
p = sel.Plan(tuple(fs[0].shape), synth.CONFIGS[cfg]["eb_rel"][0])
res = {}
for G in (1, 2, 3, 1):
    p.set_option("groups", G)
    out = p.estimate_batch(fs)
    if G in res:
        ref = res[G]
        nd = sum(1 for a, b in zip(out, ref) if a != b)
        print(f"G={G} repeat: {nd} fields differ")
    res[G] = out
for G in (2, 3):
    for i, (a, b) in enumerate(zip(res[1], res[G])):
        d = {k: (a[k], b[k]) for k in a if a[k] != b[k]}
        if d:
            print(f"G={G} field {i}: {d}")
            break
