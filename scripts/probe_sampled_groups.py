"""k_batch CTA-group sweep at a sampling stride (developer tool):
    python scripts/probe_sampled_groups.py CFG NF S0,S1[,S2] G [G ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1806_08901_b200 as sel

cfg, nf = int(sys.argv[1]), int(sys.argv[2])
stride = tuple(int(v) for v in sys.argv[3].split(","))
fs = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
for G in [int(v) for v in sys.argv[4:]]:
    p = sel.Plan(tuple(fs[0].shape), synth.CONFIGS[cfg]["eb_rel"][0], "rel", stride)
    p.set_option("groups", G)
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
    print(f"C{cfg} stride {stride} G={G}: {nf * fs[0].numel() * 4 / ms / 1e6:.0f} GB/s", flush=True)
    p.close()
