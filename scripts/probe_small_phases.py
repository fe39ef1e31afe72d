"""k_small phase times (developer tool; build with SEL_EXTRA_NVCC_FLAGS=-DSEL_SMALL_PROF=1):
range, barrier 1, blocks, histogram flush, barrier 2 (CTA 0), phase 3 + result (the last
CTA), in ns."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_1806_08901_b200 as sel
for shape in ((256, 256), (1024, 1024)):
    x = torch.from_numpy(synth.c1_field(shape)).cuda()
    p = sel.Plan(shape, 1e-4)
    for _ in range(20):
        p.estimate(x)
    buf = np.zeros(7, np.uint64)
    rc = sel.lib().sel_debug_copy(p._h, b"small_prof", buf.ctypes.data_as(ctypes.c_void_p), 56)
    names = ["range", "barrier1", "blocks", "flush", "barrier2", "phase3+result", "last_cta"]
    print(shape, rc, dict(zip(names, [int(v) for v in buf])))
    p.close()
