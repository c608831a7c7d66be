# hot SASS regions of an ncu report (tuning only): python scratch/sass_hot.py rep [addr...]
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iSrc = h.index("Source"); iA = h.index("Address"); iE = h.index("Instructions Executed")
tot = sum(float(r[iS] or 0) for r in data)
A = [int(r[iA], 16) for r in data]; base = A[0]
b = collections.OrderedDict()
for r, a in zip(data, A):
    k = (a - base) // 0x200
    b.setdefault(k, [0, 0, collections.Counter()])
    b[k][0] += float(r[iS] or 0); b[k][1] += int(r[iE] or 0)
    t = r[iSrc].split(); op = t[1] if t and t[0].startswith('@') else (t[0] if t else '')
    b[k][2][op] += int(r[iE] or 0)
for k, (s, e, c) in b.items():
    if s / tot > 0.004: print(f"{(k*0x200):6x} {s/tot*100:5.1f}% inst {e:>11} {c.most_common(5)}")
te = sum(int(r[iE] or 0) for r in data)
dm = sum(int(r[iE] or 0) for r in data if 'DMMA' in r[iSrc])
print("total warp inst", te, "DMMA", dm)
for a0 in sys.argv[2:]:
    a0 = int(a0, 16)
    idx = min(range(len(A)), key=lambda i: abs(A[i] - base - a0))
    for r in data[max(0, idx - 30): idx + 30]:
        print(f"{float(r[iS] or 0)/tot*100:5.1f}% {int(r[iA],16)-base:6x} {r[iE]:>10} {r[iSrc][:100]}")
