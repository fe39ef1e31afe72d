"""Summarise an ncu --set full report as markdown (key metrics, stall reasons, hot lines).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep "title" > profiles/rNN_x.md
"""
import csv, io, subprocess, sys, collections

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
KEYS = [("gpu__time_duration.sum", "kernel duration"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
        ("smsp__inst_executed.sum", "warp instructions"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes / warp instr"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA")]
print(f"# {title}\n\nSource: `{rep.split('/')[-1]}` (ncu --set full --clock-control none --import-source on)\n")
for r in rows[2:]:
    name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    print(f"## {name}\n\n| metric | value | unit |\n|---|---:|---|")
    for k, d in KEYS:
        if k in h:
            i = h.index(k)
            print(f"| {d} (`{k}`) | {r[i]} | {u[i]} |")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(r[i]), n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("\nWarp stall reasons (warps stalled per issue):\n")
    print(", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True) if v >= 0.05))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fname = {}, None
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] in ("Line No", "Function Name", ""):
        continue
    if r[2] == "-":
        try:
            agg[(fname, int(r[0]))] = (int(r[7]), int(r[4]), r[1][:90])
        except ValueError:
            pass
if agg:
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    byf = collections.Counter()
    for (f, _), v in agg.items():
        byf[f] += v[0]
    print("\nInstructions by file: " + ", ".join(f"{f} {n / ti * 100:.1f}%" for f, n in byf.most_common(8)))
    print("\nHottest source lines by stall samples:\n\n| % stall samples | % instr | line | source |\n|---:|---:|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        s = v[2].replace("|", "\\|")
        print(f"| {v[1] / ts * 100:.1f} | {v[0] / ti * 100:.1f} | {k[0]}:{k[1]} | `{s}` |")
