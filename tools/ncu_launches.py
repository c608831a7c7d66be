#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/ncu_launches.py gpurun_out/launches.csv [bench.json] > profiles/rNN_ncu_launches.md

Per-launch times under ncu are cold-cache and serialised: compare shares, not
absolute times. With a bench JSON line, the CUDA-event share of the same kernels
is printed beside the ncu share.
"""
import csv
import io
import json
import sys
from collections import OrderedDict


def main():
    lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("qrmc_dev::", "")
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
                 "nsecond": 1e-9}.get(unit, 1e-9)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    ev, dim = {}, None
    if len(sys.argv) > 2:
        line = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
        ks = line.get("kernel_seconds_per_solve", {})
        et = sum(ks.values()) or 1.0
        ev = {k: v / et for k, v in ks.items()}
        dim = line.get("config", {}).get("d")
    # the headline workload's kernels (template dimension = its d): their ncu share among
    # themselves, beside the bench's CUDA-event share
    def headline(k):
        base = k.split("<")[0]
        if base not in ev:
            return False
        return "<" not in k or dim is None or k.split("<")[1].split(",")[0].split(">")[0].strip() == str(dim)
    hl = sum(t for k, (n, t) in agg.items() if headline(k)) or 1.0
    print("| kernel | launches | total s (ncu) | share of all (ncu) | share of the headline solve (ncu) | share in bench (CUDA events) |")
    print("|---|---|---|---|---|---|")
    for k, (n, t) in agg.items():
        base = k.split("<")[0]
        h = headline(k)
        e = f"{100 * ev[base]:.1f}%" if h else "-"
        hs = f"{100 * t / hl:.1f}%" if h else "-"
        print(f"| {k} | {n} | {t:.3f} | {100 * t / tot:.1f}% | {hs} | {e} |")


if __name__ == "__main__":
    main()
