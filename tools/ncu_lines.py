#!/usr/bin/env python3
"""Per-source-line totals from an ncu report (needs -lineinfo and --import-source):
instructions executed, warp-stall samples and the top stall reasons per line.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, cur_file, header = [], None, None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        cur_file = next(csv.reader([line]))[1].split("/")[-1]
        continue
    if line.startswith('"Line No"'):
        header = next(csv.reader([line]))
        continue
    if header is None or not line.startswith('"') or line.startswith('"Function Name"'):
        continue
    r = next(csv.reader([line]))
    if r[0] and r[2] == "-":  # source line summary row
        d = dict(zip(header, r))
        rows.append((cur_file, r[0], r[1], d))
def num(d, k):
    try:
        return float(d.get(k, 0) or 0)
    except ValueError:
        return 0.0
tot_s = sum(num(d, "Warp Stall Sampling (All Samples)") for *_, d in rows) or 1
tot_i = sum(num(d, "Instructions Executed") for *_, d in rows) or 1
stalls = [k for k in header if k.startswith("stall_") and "Not Issued" not in k] if header else []
rows.sort(key=lambda t: -num(t[3], "Warp Stall Sampling (All Samples)"))
print(f"{'file:line':32s} {'samp%':>6s} {'inst%':>6s}  top stalls  | source")
for f, ln, src, d in rows[:top]:
    s = num(d, "Warp Stall Sampling (All Samples)")
    i = num(d, "Instructions Executed")
    st = sorted(((num(d, k), k[6:]) for k in stalls), reverse=True)[:3]
    sts = " ".join(f"{n}:{v / max(s, 1) * 100:.0f}" for v, n in st if v > 0)
    print(f"{f + ':' + ln:32s} {s / tot_s * 100:6.2f} {i / tot_i * 100:6.2f}  {sts:34s} | {src.strip()[:70]}")
