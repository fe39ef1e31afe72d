"""Developer probe: N1 calls (sel_estimate_multi) on the C3 fields (3 ebs) and one C4 / C5 field
(6 ebs), tile pipeline vs the one-thread-per-block pass; device time per call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel

def run(xs, ebs, label):
    for tile in (1, 0):
        p = sel.Plan(tuple(xs[0].shape), ebs[0], "rel")
        p.set_option("multi_tile", tile)
        p.estimate_multi(xs[0], ebs)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for x in xs:
            p.estimate_multi(x, ebs)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / len(xs)
        print(f"{label} k={len(ebs)} tile={tile}: {ms * 1e3:.1f} us / call, {xs[0].numel() * 4 / ms / 1e6:.0f} GB/s x {len(ebs)}", flush=True)
        p.close()

which = sys.argv[1] if len(sys.argv) > 1 else "c3,c4,c5"
if "c3" in which:
    run([torch.from_numpy(synth.make_field(3, i)).cuda() for i in range(13)], [1e-3, 1e-4, 1e-5], "C3 x13")
if "c4" in which:
    for i in (0, 1, 4):
        run([torch.from_numpy(synth.make_field(4, i)).cuda()], [1e-3, 1e-4, 1e-5], f"C4[{i}]")
if "c5" in which:
    for m in (0, 1):
        run([torch.from_numpy(synth.make_field(5, m, shape=(512, 512, 512))).cuda()], [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7], f"C5-512 mix {m}")
