#!/usr/bin/env python3
"""Generate tests/golden/golden_v1.json from the REFERENCE itself.

Runs the unmodified reference sources compiled by oracle/Makefile
(oracle/_ref/libqrmc_ref.so = /root/reference/proj/src/*.cpp + the Boost
shim) through their public API and records their outputs bit-exactly
(doubles as float.hex). Run in the build container, where /root/reference
exists:  make -C oracle ref && python tests/golden/make_golden.py
The fixture is committed; tests compare the C restatement (oracle/) and the
GPU library against it without needing the reference at run time.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracles  # noqa: E402
from golden_cases import CASES, DRAW_STREAMS, PATH_CASES, build_case  # noqa: E402

from paper_2407_21084_b200 import _abi  # noqa: E402


def hexs(a) -> list:
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def main() -> None:
    R = oracles.ref()
    out: dict = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref/libqrmc_ref.so "
                 "(unmodified /root/reference/proj/src + oracle/shim)"}
    # Random123 known answers as published in proj/tests/test_rng.cpp:14-40
    kat_in = [([0, 0, 0, 0], [0, 0]),
              ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2),
              ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0])]
    out["philox_kat"] = [{"ctr": c, "key": k, "out": R.philox(c, k)[0].tolist()} for c, k in kat_in]
    rng = np.random.default_rng(2407)
    ctr = rng.integers(0, 2**32, size=(32, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(32, 2), dtype=np.uint64).astype(np.uint32)
    out["philox_random"] = {"ctr": ctr.tolist(), "key": key.tolist(), "out": R.philox(ctr, key).tolist()}
    sids = np.array([s for _, s in DRAW_STREAMS], dtype=np.uint64)
    out["draws"] = {"seed": 42, "stream_ids": [int(s) for s in sids],
                    "u64": [[int(v) for v in row] for row in R.stream_draws(42, sids, 12, 0)],
                    "uniform": [hexs(r) for r in R.stream_draws(42, sids, 12, 1)],
                    "normal": [hexs(r) for r in R.stream_draws(42, sids, 12, 2)]}
    ps = [0.5, 0.975, 0.995, 0.0013498980316301, 1e-10, 1 - 1e-10, 0.3, 0.02, 2.0**-53]
    out["normal_quantile"] = {"p": hexs(ps), "z": hexs([R.normal_quantile(p) for p in ps])}
    gam = []
    for kind, dim, deg in [(0, 1, [40]), (0, 3, [2, 5, 3]), (1, 3, [6]), (1, 4, [5]), (1, 2, [20]),
                           (2, 3, [4]), (2, 4, [2]), (2, 2, [19]), (2, 4, [100]), (2, 6, [16]),
                           (0, 2, [31, 31])]:
        rows, kmax = R.gamma(kind, dim, deg)
        gam.append({"kind": kind, "dim": dim, "degrees": deg, "size": int(rows.shape[0]),
                    "kmax": kmax.tolist(), "sha256": hashlib.sha256(rows.astype("<i4").tobytes()).hexdigest(),
                    "head": rows[:6].tolist(), "tail": rows[-3:].tolist()})
    out["gamma"] = gam
    paths = []
    for pc in PATH_CASES:
        prob, cfg = build_case(pc)
        p = R.cloud_paths(prob, cfg, pc["step"], pc["first"], pc["n"])
        paths.append({"case": pc, "paths": hexs(p)})
    out["paths"] = paths
    solves = []
    for case in CASES:
        prob, cfg = build_case(case)
        k = R.gamma(cfg.c.gamma_kind, prob.dim, list(case["degrees"]))[0].shape[0]
        coeffs, stats = R.backward_solve(prob, cfg, k)
        origin = np.zeros(prob.dim)
        u00 = R.evaluate(cfg, prob.dim, coeffs[0], origin)[0]
        entry = {"case": case, "basis_size": int(k), "coeffs": hexs(coeffs),
                 "applications": int(stats.applications), "clipped": int(stats.clipped),
                 "u00": float(u00).hex()}
        if case.get("mse"):
            m, step_sq = R.mse_metrics(cfg, prob.dim, case.get("kappa", 0.6), prob.terminal_params[1],
                                       prob.horizon, coeffs, 555, 300)
            entry["mse"] = hexs(m[:4])
        solves.append(entry)
    out["solves"] = solves
    dst = Path(__file__).resolve().parent / "golden_v1.json"
    dst.write_text(json.dumps(out, separators=(",", ":")))
    print(f"wrote {dst} ({dst.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
