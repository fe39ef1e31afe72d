"""k_batch vs the per-field kernels on a stack of full-size fields (developer check)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel
cfg, nf = int(sys.argv[1]), int(sys.argv[2])
fs = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
p = sel.Plan(tuple(fs[0].shape), synth.CONFIGS[cfg]["eb_rel"][0])
p.set_option("batch_kernel", 0)
ref = [p.estimate(f) for f in fs]
p.set_option("batch_kernel", 1)
bad = 0
for rep in range(3):
    out = p.estimate_batch(fs)
    for i, (a, b) in enumerate(zip(out, ref)):
        d = {k: (a[k], b[k]) for k in a if a[k] != b[k] and not (isinstance(a[k], float) and abs(a[k] - b[k]) <= 1e-9 * max(abs(a[k]), abs(b[k])))}
        if d:
            bad += 1
            if bad <= 2:
                print(f"rep {rep} field {i}: {list(d.items())[:3]}")
print(f"C{cfg} nf={nf}: {bad} mismatching (field, rep) of {3 * nf}")
