#!/usr/bin/env python3
"""Generate tests/golden/bases_v1.npz from the REFERENCE itself.

Coefficient goldens for the index sets the BASELINE.json configs are restated
on: Gamma_H(6,16) and Gamma_H(2,19) (config 5), Gamma_H(6,64)
(config 4) and Gamma_H(4,100) at the real N = 20 (config 2). Each solve runs the
unmodified reference sources (oracle/_ref/libqrmc_ref.so, proj/src/solver.cpp:109-226)
at an M the reference finishes in seconds. Tables of 10^4-10^5 coefficients per
step are too large to commit whole, so every step keeps a deterministic sample of
coefficient indices (always including k = 0 and k = K - 1) bit-exactly, plus the
row's sum of |alpha| and max |alpha|, u(0, 0) (solver.cpp:228-237) and the
truncation counters. Run in the build container:

    make -C oracle ref && python tests/golden/make_golden_bases.py
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracles  # noqa: E402

from paper_2407_21084_b200 import _abi  # noqa: E402

# name, d, Gamma_H degree, N, M, q, seed
BASES = [
    ("c5_d6_hyp16_N10", 6, 16, 10, 2048, 5.1, 42),
    ("c5_d2_hyp19_N20", 2, 19, 20, 8192, 2.1, 42),
    ("c5_d2_hyp19_N10", 2, 19, 10, 5000, 0.0, 7),
    ("c4_d6_hyp64_N3", 6, 64, 3, 1024, 5.1, 42),
    ("c2_d4_hyp100_N20", 4, 100, 20, 1024, 5.1, 42),
]
SAMPLE = 1024


def sample_indices(k: int, seed: int) -> np.ndarray:
    if k <= SAMPLE:
        return np.arange(k)
    rng = np.random.default_rng(seed)
    idx = rng.choice(np.arange(1, k - 1), size=SAMPLE - 2, replace=False)
    return np.sort(np.concatenate([[0, k - 1], idx]))


def main() -> None:
    R = oracles.ref()
    out = {}
    for name, d, deg, n, m, q, seed in BASES:
        prob = _abi.sin_bench_problem(d)
        cfg = _abi.ConfigHolder(steps=n, paths=m, damping=q, seed=seed, gamma_kind=_abi.GAMMA_HYPERBOLIC,
                                degrees=[deg])
        k = R.gamma(_abi.GAMMA_HYPERBOLIC, d, [deg])[0].shape[0]
        t0 = time.time()
        coeffs, stats = R.backward_solve(prob, cfg, k)
        idx = sample_indices(k, 2407 + d * 1000 + deg)
        u00 = R.evaluate(cfg, d, coeffs[0], np.zeros(d))[0]
        out[f"{name}/meta"] = np.array([d, deg, n, m, seed, k, stats.applications, stats.clipped], dtype=np.int64)
        out[f"{name}/damping"] = np.array([q])
        out[f"{name}/idx"] = idx.astype(np.int64)
        out[f"{name}/sample"] = coeffs[:, idx]
        out[f"{name}/l1"] = np.abs(coeffs).sum(axis=1)
        out[f"{name}/maxabs"] = np.abs(coeffs).max(axis=1)
        out[f"{name}/u00"] = np.array([u00])
        print(f"{name}: K={k} {time.time() - t0:.1f}s u00={u00:.6f} clipped={stats.clipped}")
    dst = Path(__file__).resolve().parent / "bases_v1.npz"
    np.savez_compressed(dst, **out)
    print(f"wrote {dst} ({dst.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
