"""Throughput of k_batch on every BASELINE config (developer tool; writes a markdown table).

    python scripts/measure_all.py [c1,c2,c3,c4,c5] > gpurun_out/throughput.md
Fields already in HBM, steps = one sel_estimate_batch_async of the whole stack + D2H of
the results, CUDA events, 2 warm-up + 5 timed steps; GB/s = float32 input bytes / time.
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1806_08901_b200 as sel

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]


def run(fields, eb, stride, label):
    shape = tuple(fields[0].shape)
    p = sel.Plan(shape, eb, "rel", stride)
    for kv in os.environ.get("SEL_OPTS", "").split(","):      # e.g. SEL_OPTS=range_warps=0,groups=2
        if kv:
            p.set_option(kv.split("=")[0], float(kv.split("=")[1]))
    buf = p.results_buffer(len(fields))
    nfields, fields = len(fields), p.field_stack(fields)      # pointers marshalled once
    for _ in range(2):
        p.estimate_batch_async(fields, buf)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.estimate_batch_async(fields, buf)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res = p.decode_results(buf, len(fields))
    nsz = sum(1 for r in res if r["choice"] == 0)
    gbs = len(fields) * fields.fields[0].numel() * 4 / ms / 1e6
    print(f"| {label} | {len(fields)} | {eb:g} | {stride or 'all'} | {ms / len(fields) * 1e3:.1f} | "
          f"{gbs:.0f} | {100 * gbs / PEAK:.1f} | {nsz} / {len(fields) - nsz} |", flush=True)
    p.close()


def run_multi(fields, ebs, label):
    """N1: every eb of the sweep from one read per field (sel_estimate_multi)."""
    shape = tuple(fields[0].shape)
    p = sel.Plan(shape, ebs[0], "rel")
    p.estimate_multi(fields[0], ebs)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for f in fields:
        p.estimate_multi(f, ebs)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    gbs = len(fields) * fields[0].numel() * 4 / ms / 1e6
    print(f"| {label} (N1: {len(ebs)} ebs, one read) | {len(fields)} | {','.join(f'{e:g}' for e in ebs)} | all | "
          f"{ms / len(fields) * 1e3:.1f} | {gbs:.0f} (x{len(ebs)} = {gbs * len(ebs):.0f}) | {100 * gbs / PEAK:.1f} | - |",
          flush=True)
    p.close()


SEL = set((sys.argv[1] if len(sys.argv) > 1 else "c1,c2,c3,c4,c5").split(","))
print(f"| workload | fields | eb_rel | stride | us / field | GB/s | % of HBM ({PEAK:g} GB/s) | SZ / ZFP chosen |")
print("|---|---:|---:|---|---:|---:|---:|---|")
if "c1" in SEL:
  f1 = [torch.from_numpy(synth.c1_field(seed=i)).cuda() for i in range(256)]
  run(f1, 1e-4, None, "C1 256x256 (x256 seeds)")
  del f1
if "c2" in SEL:
  f2 = [torch.from_numpy(synth.make_field(2, i)).cuda() for i in range(100)]
  run(f2, 1e-4, None, "C2 1800x3600")
  run(f2, 1e-4, (1, 10), "C2 1800x3600")
  del f2
if "c3" in SEL:
  f3 = [torch.from_numpy(synth.make_field(3, i)).cuda() for i in range(13)]
  for eb in (1e-3, 1e-4, 1e-5):
    run(f3, eb, None, "C3 100x500x500")
  run_multi(f3, [1e-3, 1e-4, 1e-5], "C3 100x500x500")
  del f3
if "c4" in SEL:
  f4 = [torch.from_numpy(synth.make_field(4, i)).cuda() for i in range(6)]
  run(f4, 1e-4, None, "C4 512^3")
  run(f4, 1e-4, (4, 4, 4), "C4 512^3")
  del f4
  torch.cuda.empty_cache()
for mix in ((0, 1, 2) if "c5" in SEL else ()):
    t0 = time.time()
    x = torch.from_numpy(synth.make_field(5, mix)).cuda()
    for eb in (1e-2, 1e-4, 1e-6):
        run([x], eb, None, f"C5 1024^3 w={(0, 0.5, 1)[mix]}")
    run_multi([x], [1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7], f"C5 1024^3 w={(0, 0.5, 1)[mix]}")
    del x
    torch.cuda.empty_cache()
