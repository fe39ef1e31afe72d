"""List SASS branch/sync instructions of an ncu cuda,sass source page by executed count."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
fname = line = None
c, cs, txt = collections.Counter(), collections.Counter(), {}
tot = 0
ops = sys.argv[2].split(",") if len(sys.argv) > 2 else ["BRA", "BSSY", "BSYNC", "WARPSYNC", "NANOSLEEP", "SYNCS"]
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] in ("Line No", "Function Name"):
        continue
    if r[0] not in ("", "-") and r[2] == "-":
        line = (fname, int(r[0])); txt[line] = r[1][:80]; continue
    if r[0] == "" and r[2].startswith("0x"):
        try:
            n = int(r[7]); s = int(r[4])
        except ValueError:
            continue
        tot += n
        ins = r[3].strip()
        toks = ins.split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
        if any(op.startswith(o) for o in ops):
            c[(line, op)] += n; cs[(line, op)] += s
for k, n in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{n/tot*100:5.2f}% st{cs[k]:5d} {k[1]:14s} {k[0][0]}:{k[0][1]} {txt.get(k[0], '')}")
