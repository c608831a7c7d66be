"""Shared pytest setup: markers, import paths, oracle builds.

`-m "not gpu"` runs everywhere (oracle vs reference bit-parity, golden
vectors, host logic, the C ABI's host-only entry points, multi-rank host
tests over gloo); `-m gpu` needs a B200 and calls the CUDA library through
the C ABI.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the CUDA library")
    port = ROOT / "oracle" / "lib" / "libqrmc_oracle.so"
    if not port.exists() or port.stat().st_mtime < (ROOT / "oracle" / "qrmc_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "port"], check=True)
    lib = ROOT / "paper_2407_21084_b200" / "_lib" / "libqrmc_gpu.so"
    if not lib.exists():
        from paper_2407_21084_b200 import build
        build.build()


@pytest.fixture(scope="session")
def port():
    import oracles
    return oracles.port()


@pytest.fixture(scope="session")
def ref():
    import oracles
    if not oracles.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracles.ref()
