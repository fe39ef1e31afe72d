"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
fname, agg, order = None, {}, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 9 or r[0] in ("Line No", "Function Name"):
        continue
    if r[0] != "-" and r[2] == "-":          # a CUDA line row (aggregated)
        try:
            key = (fname, int(r[0]))
            agg[key] = [int(r[7]), int(r[4]), r[1][:100], int(r[8])]
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print("total warp inst", tot, "stall samples", ts)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][int(sys.argv[3]) if len(sys.argv) > 3 else 1])[:n]:
    print(f"{v[0]/tot*100:5.1f}%i {v[1]/ts*100:5.1f}%s {v[3]/max(v[0],1):4.1f}thr {k[0]}:{k[1]}  {v[2]}")
