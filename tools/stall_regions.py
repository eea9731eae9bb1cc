"""Stall reasons per code region of one kernel from an ncu source page
(--page source --csv): windows of W SASS lines holding >= 1 % of the samples.
Usage: python tools/stall_regions.py page.csv [W]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 100
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i]
ci, cs, cn = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
sc = [(k, h[6:]) for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
L = []
for r in rows[i + 1:]:
    try:
        L.append((int(float(r[ci])), int(float(r[cn] or 0)), r[cs].strip(), [float(r[k] or 0) for k, _ in sc]))
    except (ValueError, IndexError):
        continue
tot = sum(x[1] for x in L)
for k in range(0, len(L), W):
    seg = L[k:k + W]
    sm = sum(x[1] for x in seg)
    if sm < 0.01 * tot:
        continue
    st = [sum(x[3][j] for x in seg) for j in range(len(sc))]
    s = sum(st) or 1
    top = sorted(zip(st, [h for _, h in sc]), reverse=True)[:4]
    ops = {}
    for n, _, src, _ in seg:
        o = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
        ops[o] = ops.get(o, 0) + n
    print(f"{k:5d} {100*sm/tot:5.1f}%  " + " ".join(f"{h}={100*v/s:.0f}" for v, h in top)
          + "  | " + " ".join(f"{o}" for o, _ in sorted(ops.items(), key=lambda x: -x[1])[:3]))
