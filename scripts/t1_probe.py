import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1806_08901_b200 as sel, synth
x = synth.c1_field()
t = torch.from_numpy(x).cuda()
mode = sys.argv[1]
with sel.Plan(x.shape, 1e-4) as p:
    if mode == "seq": p.set_option("batch_kernel", 0)
    if mode == "dbg": p.set_option("debug", 1)
    r = p.estimate(t)
    print(mode, r["sz_bits_per_value"], r["zfp_bits_per_value"])
