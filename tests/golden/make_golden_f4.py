#!/usr/bin/env python3
"""Generate tests/golden/f4_v1.json from the REFERENCE build.

The unmodified reference sources (oracle/_ref/libqrmc_ref.so) reach Boost's students_t for
a Student measure with mu not in {1, 2} (proj/src/student.cpp:60, 73); the shim defines it
with include/qrmc_student_t.h (Boost itself is not vendored: parity with real Boost is
unpinned). Per-coordinate affine drift and diagonal diffusion are ProblemSpec std::function
members built by oracle/ref_capi.cpp exactly as include/qrmc_gpu.h specifies them. Records
full coefficient tables, truncation counters and u(0, x0) per case, and measure values.

    make -C oracle ref && python tests/golden/make_golden_f4.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracles  # noqa: E402
from golden_cases import F4_CASES, build_case  # noqa: E402


def hexs(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def main() -> None:
    R = oracles.ref()
    out = {"generator": "tests/golden/make_golden_f4.py", "source": "oracle/_ref/libqrmc_ref.so (reference + shim)"}
    meas = []
    for mu in (0.7, 3.5, 6.0, 30.0):
        u = np.array([1e-15, 1e-9, 1e-3, 0.1, 0.37, 0.5, 0.8, 0.999, 1 - 1e-9])
        x = np.array([-1e6, -30.0, -2.5, -0.3, 0.0, 1e-5, 0.1, 1.7, 40.0, 1e8])
        meas.append({"mu": mu, "u": hexs(u), "inv_cdf": hexs(R.measure(mu, 1, 2, u)), "x": hexs(x),
                     "cdf": hexs(R.measure(mu, 1, 1, x)), "pdf": hexs(R.measure(mu, 1, 0, x))})
    out["measure"] = meas
    solves = []
    for case in F4_CASES:
        prob, cfg = build_case(case)
        k = R.gamma(cfg.c.gamma_kind, prob.dim, list(case["degrees"]))[0].shape[0]
        coeffs, stats = R.backward_solve(prob, cfg, k)
        u00 = R.evaluate(cfg, prob.dim, coeffs[0], np.zeros(prob.dim))[0]
        solves.append({"case": case, "basis_size": int(k), "coeffs": hexs(coeffs),
                       "applications": int(stats.applications), "clipped": int(stats.clipped),
                       "u00": float(u00).hex()})
    out["solves"] = solves
    dst = Path(__file__).resolve().parent / "f4_v1.json"
    dst.write_text(json.dumps(out, separators=(",", ":")))
    print(f"wrote {dst} ({dst.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
