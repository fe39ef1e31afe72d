"""Time k_batch for (lag, G) settings on one config (developer tool): probe_lag.py C NF lag:G ..."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel
cfg, nf = int(sys.argv[1]), int(sys.argv[2])
fs = [torch.from_numpy(synth.make_field(cfg, i)).cuda() for i in range(nf)]
p = sel.Plan(tuple(fs[0].shape), synth.CONFIGS[cfg]["eb_rel"][0])
buf = p.results_buffer(nf)
ref = None
for spec in sys.argv[3:]:
    lag, G = map(int, spec.split(":"))
    p.set_option("lag", lag).set_option("groups", G)
    for _ in range(2):
        p.estimate_batch_async(fs, buf)
    torch.cuda.synchronize()
    res = p.decode_results(buf, nf)
    ref = ref or res
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.estimate_batch_async(fs, buf)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"C{cfg} nf={nf} lag={lag} G={G}: {ms / nf * 1000:.1f} us/field "
          f"{nf * fs[0].numel() * 4 / ms / 1e6:.0f} GB/s identical={res == ref}", flush=True)
