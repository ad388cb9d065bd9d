"""Summarise an ncu --page source --csv --print-source sass dump: top stall instructions, shared-memory excess
wavefronts, opcode mix.  Usage: python tools/ncu_src_summary.py dump.csv [kernel-substring]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
sel = sys.argv[2] if len(sys.argv) > 2 else None
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and r:
        cur["rows"].append(r)
for b in blocks:
    if sel and sel not in b["name"]:
        continue
    h = b["hdr"]
    ix = {k: h.index(k) for k in h}
    print("==", b["name"][:120])
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in b["rows"])
    print("total stall samples", tot)
    top = sorted(b["rows"], key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:25]
    for r in top:
        print(f'{int(r[ix["Warp Stall Sampling (All Samples)"]]):8d} {r[ix["Instructions Executed"]]:>12} exc_wf={r[ix["L1 Wavefronts Shared Excessive"]]:>10}  {r[ix["Source"]].strip()[:90]}')
    ops = collections.Counter()
    for r in b["rows"]:
        op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
        if op.startswith("@"):
            op = r[ix["Source"]].split()[1]
        ops[op.split(".")[0]] += int(float(r[ix["Instructions Executed"]] or 0))
    print("opcode mix:", ops.most_common(14))
    exc = [(int(float(r[ix["L1 Wavefronts Shared Excessive"]] or 0)), r[ix["Source"]].strip()[:70]) for r in b["rows"]]
    print("excessive shared wavefronts:", sorted(exc, reverse=True)[:6])
