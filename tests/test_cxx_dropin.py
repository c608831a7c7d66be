"""The header-only C++ drop-in (include/qrmc_gpu.hpp) compiles and links:
against the C ABI alone, and -- where the reference headers exist -- against
the reference's own types, as a reference call site would use it
(INTEGRATION.md). No device call is made."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2407_21084_b200" / "_lib"
REF_INC = Path("/root/reference/proj/include")

PLAIN = r'''
#include "qrmc_gpu.hpp"
#include <cstdio>
int main(int argc, char**) {
    qrmc_gpu::Config c;
    c.steps = 0;  // invalid: rejected host-side before any device work
    c.gamma_kind = QRMC_GAMMA_HYPERBOLIC;
    c.degrees = {6};
    try {
        qrmc_gpu::backward_solve(qrmc_gpu::sin_benchmark(2), c);
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument: %s\n", e.what());
        return 0;
    }
    return 1;
}
'''

WITH_REF = r'''
#include "qrmc/errors.hpp"
#include "qrmc/solver.hpp"
#define QRMC_GPU_WITH_REFERENCE_TYPES
#include "qrmc_gpu.hpp"
qrmc::CoefficientTable call_site(const qrmc::RunConfig& cfg) {
    return qrmc_gpu::backward_solve(qrmc_gpu::sin_benchmark(2), cfg);
}
'''


def _gxx():
    g = shutil.which("g++")
    if not g:
        pytest.skip("g++ unavailable")
    return g


def test_cxx_wrapper_links_and_validates(tmp_path):
    src = tmp_path / "plain.cpp"
    src.write_text(PLAIN)
    exe = tmp_path / "plain"
    subprocess.run([_gxx(), "-std=c++20", f"-I{ROOT / 'include'}", str(src), f"-L{LIB}", "-lqrmc_gpu",
                    f"-Wl,-rpath,{LIB}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "steps must be >= 1" in out.stdout


def test_cxx_wrapper_accepts_reference_types(tmp_path):
    if not REF_INC.exists():
        pytest.skip("reference headers absent")
    src = tmp_path / "with_ref.cpp"
    src.write_text(WITH_REF)
    subprocess.run([_gxx(), "-std=gnu++20", "-fsyntax-only", f"-I{ROOT / 'include'}", f"-I{REF_INC}",
                    str(src)], check=True)


DROPIN = ROOT / "oracle" / "_ref" / "dropin_check"


@pytest.mark.gpu
def test_reference_call_site_runs_the_dropin_on_the_device():
    """oracle/dropin_check.cpp: a reference call site compiled against the reference's own
    headers and sources (oracle/Makefile, in the build container) with include/qrmc_gpu.hpp
    (QRMC_GPU_WITH_REFERENCE_TYPES), linked against libqrmc_gpu.so: the acceptance
    determinism criterion (acceptance_main.cpp:369-395) through the drop-in, its
    CoefficientTable against qrmc::backward_solve on the same inputs (1e-10, TruncationStats
    equal) and the same exception types/messages/steps as the reference."""
    import torch
    assert torch.cuda.is_available()
    if not DROPIN.exists():
        pytest.skip("oracle/_ref/dropin_check not built (needs /root/reference at build time)")
    out = subprocess.run([str(DROPIN)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "DROPIN OK" in out.stdout
    assert out.stdout.count("PASS") >= 10 and "FAIL" not in out.stdout
