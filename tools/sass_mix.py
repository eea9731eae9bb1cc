"""Instruction mix of one kernel from an ncu source page (--page source --csv):
executed warp-instructions per opcode, stall samples per opcode, and shared
wavefronts. Usage: ncu -i rep --page source --csv -k regex:NAME > x.csv;
python tools/sass_mix.py x.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[i]
ci, cs, cn = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
cw = hdr.index("L1 Wavefronts Shared")
cnt, smp, wf = collections.Counter(), collections.Counter(), collections.Counter()
for r in rows[i + 1:]:
    if len(r) <= ci or not r[ci]:
        continue
    try:
        float(r[ci])
    except ValueError:
        continue
    op = r[cs].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    cnt[o] += int(float(r[ci])); smp[o] += int(float(r[cn] or 0)); wf[o] += int(float(r[cw] or 0))
tot = sum(cnt.values()); ts = sum(smp.values())
print(f"total warp-instr {tot:.4g}, samples {ts}")
for o, c in cnt.most_common(25):
    print(f"{o:10s} {c:12d} {100*c/tot:5.1f}%  stall-samples {100*smp[o]/max(ts,1):5.1f}%  smem-wavefronts {wf[o]}")
