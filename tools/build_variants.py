#!/usr/bin/env python3
"""Timing-experiment builds (responses_ws.cu recompiled, the rest linked from the main build) of libqrmc_gpu.so (compile-time switches; results of the
experimental switches are NOT valid solves):  python tools/build_variants.py NAME=DEF[,DEF] ...
-> paper_2407_21084_b200/_lib/variants/libqrmc_gpu_NAME.so (run with QRMC_GPU_LIB=...)."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2407_21084_b200 import build  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    out = ROOT / "paper_2407_21084_b200" / "_lib" / "variants" / f"libqrmc_gpu_{name}.so"
    build.build(out=out, defines=[d for d in defs.split(",") if d], only=ONLY)
    return out


ONLY = {"responses_ws.cu"}
args = sys.argv[1:]
if args and args[0].startswith("--only="):
    ONLY = set(args.pop(0)[len("--only="):].split(","))
build.build()  # the main objects the variants link against
with ThreadPoolExecutor(max_workers=4) as ex:
    for p in ex.map(one, args):
        print(p)
