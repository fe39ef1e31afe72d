"""Run k_batch on N fields of config C a few times (for ncu): one_batch.py C N [G]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel
cfg, nf = int(sys.argv[1]), int(sys.argv[2])
fs = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
p = sel.Plan(tuple(fs[0].shape), synth.CONFIGS[cfg]["eb_rel"][0])
if len(sys.argv) > 3:
    p.set_option("groups", int(sys.argv[3]))
for _ in range(3):
    p.estimate_batch(fs)
torch.cuda.synchronize()
print("ok")
