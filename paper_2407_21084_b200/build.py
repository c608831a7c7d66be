"""Build the in-tree CUDA library ``_lib/libqrmc_gpu.so`` for sm_100a.

    python -m paper_2407_21084_b200.build

nvcc cross-compiles here without a GPU; the .so is git-ignored but travels
to the GPU box with the repo snapshot. One shared object holds the kernels
(csrc/kernels.cu), the host runtime (csrc/host.cpp) and the C ABI
(include/qrmc_gpu.h); CUDA runtime is linked statically, NCCL is dlopen'ed
only for multi-GPU sessions.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "_lib" / "libqrmc_gpu.so"
SOURCES = [CSRC / "kernels.cu", CSRC / "responses_mma.cu", CSRC / "responses_ws.cu", CSRC / "project_mma.cu", CSRC / "host.cpp",
           CSRC / "table_io.cpp"]
HEADERS = [CSRC / "kernels.cuh", CSRC / "qrmc_device.cuh", CSRC / "qrmc_types.h", CSRC / "series_block.cuh", CSRC / "mma_common.cuh", ROOT / "include" / "qrmc_gpu.h",
           ROOT / "include" / "qrmc_normal_quantile.h", ROOT / "include" / "qrmc_student_t.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def json_include() -> str:
    """nlohmann/json.hpp (the JSON library the reference builds against): the
    coefficient artifact writer (csrc/table_io.cpp) serialises with it."""
    import site
    cands = [os.environ.get("QRMC_JSON_DIR", "")]
    for p in site.getsitepackages():
        cands.append(os.path.join(p, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
    for c in cands:
        if c and Path(c, "json.hpp").exists():
            return c
    raise RuntimeError("nlohmann json.hpp not found (set QRMC_JSON_DIR)")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS + [Path(__file__)])


SRMC_OUT = PKG / "_lib" / "libqrmc_srmc.so"
SRMC_SOURCES = [CSRC / "srmc.cu", CSRC / "srmc_host.cpp"]
SRMC_HEADERS = [CSRC / "qrmc_device.cuh", CSRC / "qrmc_types.h", CSRC / "srmc_types.h", ROOT / "include" / "qrmc_srmc.h",
                ROOT / "include" / "qrmc_gpu.h", ROOT / "include" / "qrmc_normal_quantile.h",
                ROOT / "include" / "qrmc_student_t.h"]


def build_srmc(force: bool = False, verbose: bool = False) -> Path:
    """Second in-tree library: the SRMC solver (include/qrmc_srmc.h)."""
    if not force and SRMC_OUT.exists():
        t = SRMC_OUT.stat().st_mtime
        if all(p.stat().st_mtime <= t for p in SRMC_SOURCES + SRMC_HEADERS + [Path(__file__)]):
            return SRMC_OUT
    SRMC_OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = SRMC_OUT.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-shared", "-Xcompiler",
           "-fPIC", "-Xptxas", "-warn-spills", f"-I{ROOT / 'include'}", f"-I{CSRC}", *map(str, SRMC_SOURCES), "-o",
           str(tmp), "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    tmp.replace(SRMC_OUT)
    return SRMC_OUT


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines=(), only=None) -> Path:
    """libqrmc_gpu.so: every translation unit compiled for sm_100a in parallel
    (one nvcc per source), then linked into one shared library in-tree."""
    if out is None:
        build_srmc(force=force, verbose=verbose)
    target = out or OUT
    if out is None and not force and not needs_build():
        return OUT
    target.parent.mkdir(parents=True, exist_ok=True)
    objdir = target.parent / ("obj_" + target.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    common = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
              "-Xptxas", "-warn-spills", f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{json_include()}",
              *[f"-D{d}" for d in defines]]
    if verbose:
        common.insert(0, "-Xptxas=-v")

    newest_dep = max(p.stat().st_mtime for p in HEADERS + [Path(__file__)])

    def compile_one(src: Path) -> Path:
        if only is not None and src.name not in only:
            # a variant build recompiles only `only`; the rest come from the main build
            build(verbose=verbose)
            return OUT.parent / ("obj_" + OUT.stem) / (src.name + ".o")
        obj = objdir / (src.name + ".o")
        if not force and not defines and obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, newest_dep):
            return obj
        r = subprocess.run([nvcc(), *common, "-c", str(src), "-o", str(obj)], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name} ({r.returncode}):\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = target.with_suffix(".so.tmp")
    r = subprocess.run([nvcc(), *ARCH, "-shared", *map(str, objs), "-o", str(tmp), "-ldl"], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({r.returncode}):\n{r.stderr}")
    tmp.replace(target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
