"""The C-ABI library without a GPU: it loads, exports every symbol
include/qrmc_gpu.h declares, and its host-only logic (index-set
enumeration, validation and error mapping, multi-GPU lane sharding) agrees
with the reference. No compute call is made here."""
import ctypes as C
import hashlib
import json
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2407_21084_b200 import _abi, api

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden_v1.json").read_text())


def declared_symbols():
    text = (ROOT / "include" / "qrmc_gpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qrmc_(?:gpu|problem)_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _abi.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(_abi.EXPORTED_SYMBOLS) <= set(syms)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("g", GOLDEN["gamma"], ids=lambda g: f"{g['kind']}-{g['dim']}-{g['degrees']}")
def test_gamma_enumeration_matches_reference(g):
    kind = {0: "full", 1: "total", 2: "hyperbolic"}[g["kind"]]
    s = api.MultiIndexSet(kind, g["dim"], tuple(g["degrees"]))
    rows = s.indices()
    assert rows.shape == (g["size"], g["dim"])
    assert hashlib.sha256(rows.astype("<i4").tobytes()).hexdigest() == g["sha256"]


def test_gamma_against_reference_live(ref):
    for kind, dim, deg in [(1, 5, [7]), (2, 5, [20]), (2, 7, [10]), (0, 4, [3, 1, 4, 2]), (1, 1, [0]), (2, 1, [1])]:
        a = api.MultiIndexSet({0: "full", 1: "total", 2: "hyperbolic"}[kind], dim, tuple(deg)).indices()
        b, _ = ref.gamma(kind, dim, deg)
        np.testing.assert_array_equal(a, b)


def test_gamma_errors():
    with pytest.raises(api.CapacityError):
        len(api.MultiIndexSet.full([400, 400, 400]))  # multi_index.cpp:102-104
    with pytest.raises(api.CapacityError):
        len(api.MultiIndexSet.total(12, 40))
    with pytest.raises(ValueError):
        len(api.MultiIndexSet.hyperbolic(3, 0))
    with pytest.raises(ValueError):
        len(api.MultiIndexSet.full([-1]))


def _solve_status(prob, cfg):
    L = _abi.lib()
    co = np.zeros(1 << 16)
    st = _abi.Stats()
    err = C.create_string_buffer(512)
    rc = L.qrmc_gpu_backward_solve(None, C.byref(prob), cfg.ref(), co.ctypes.data_as(C.POINTER(C.c_double)),
                                   co.size, None, C.byref(st), err, 512)
    return rc, err.value.decode()


@pytest.mark.parametrize("bad,status,msg", [
    (dict(steps=0), _abi.EINVAL, "steps must be >= 1"),
    (dict(paths=0), _abi.EINVAL, "paths must be >= 1"),
    (dict(damping=-1.0), _abi.EINVAL, "damping must be finite"),
    (dict(paths=1 << 40), _abi.EINVAL, "stream-id layout"),
    (dict(mu=-1.0), _abi.EINVAL, "mu must be positive"),
    (dict(mu=float("inf")), _abi.EINVAL, "mu must be positive"),
])
def test_config_validation_before_device(bad, status, msg):
    """RunConfig::validate / SamplingMeasure rules (solver.cpp:23-35, student.cpp:21-44)
    are enforced host-side, before any device is touched."""
    kw = dict(steps=2, paths=10, seed=1, gamma_kind=0, degrees=[2], mu=2.0)
    kw.update(bad)
    rc, err = _solve_status(_abi.sin_bench_problem(1), _abi.ConfigHolder(**kw))
    assert rc == status and msg in err


def test_problem_validation_before_device():
    p = _abi.sin_bench_problem(2)
    p.horizon = 0.0
    rc, err = _solve_status(p, _abi.ConfigHolder(steps=2, paths=10, gamma_kind=0, degrees=[2, 2]))
    assert rc == _abi.EINVAL and "horizon" in err
    p = _abi.sin_bench_problem(2)
    p.moment_ratio = 0.5
    rc, err = _solve_status(p, _abi.ConfigHolder(steps=2, paths=10, gamma_kind=0, degrees=[2, 2]))
    assert rc == _abi.EINVAL and "moment_ratio" in err
    p = _abi.sin_bench_problem(2)
    p.driver_kind = 99
    rc, _ = _solve_status(p, _abi.ConfigHolder(steps=2, paths=10, gamma_kind=0, degrees=[2, 2]))
    assert rc == _abi.ENOTIMPL  # no device functor, no CPU fallback
    # dims of gamma and problem disagree (test_solver.cpp:435-442)
    rc, _ = _solve_status(_abi.sin_bench_problem(1), _abi.ConfigHolder(steps=2, paths=10, gamma_kind=1, degrees=[2]))
    # 1-d total(2) is valid; a 2-d full set on a 1-d problem is not
    rc, err = _solve_status(_abi.sin_bench_problem(1), _abi.ConfigHolder(steps=2, paths=10, gamma_kind=0, degrees=[2, 2]))
    assert rc == _abi.EINVAL


@pytest.mark.parametrize("paths", [1, 1000, 1024, 1025, 262144, 262145, 1_000_003, 20_000_000])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_lane_sharding_partitions_paths(paths, world):
    """Ranks own disjoint lane ranges; their paths (via the kernels' owned-index
    map) partition [0, M) and follow the reference's chunk->lane rule
    (parallel.hpp:20-36)."""
    L = _abi.lib()
    total = 0
    seen = []
    for rank in range(world):
        lo, hi, n = C.c_int32(), C.c_int32(), C.c_int64()
        assert L.qrmc_gpu_lane_ownership(paths, rank, world, C.byref(lo), C.byref(hi), C.byref(n)) == 0
        total += n.value
        if paths <= 262145:
            ms = [L.qrmc_gpu_owned_path(q, lo.value, hi.value - lo.value) for q in range(n.value)]
            assert all(0 <= m < paths for m in ms)
            assert all(lo.value <= (m // 1024) % 256 < hi.value for m in ms)
            seen.extend(ms)
    assert total == paths
    if paths <= 262145:
        assert sorted(seen) == list(range(paths))


# ---------------------------------------------------------------- tensor-core layout
# host.cpp build_mma_layout: the fragment streams of the FP64 tensor-core kernels.
# qrmc_gpu_mma_layout_check replays both kernels' data flow on the host (units,
# step alignment, mma lane order, term/group table rows, K2 rectangles and output
# map) for a random point and checks it against the direct sum over Gamma.
MMA_CASES = [
    (_abi.GAMMA_HYPERBOLIC, 4, [100]),   # the bench workload (K = 12,752)
    (_abi.GAMMA_HYPERBOLIC, 4, [16]),
    (_abi.GAMMA_HYPERBOLIC, 3, [8]),
    (_abi.GAMMA_HYPERBOLIC, 3, [40]),
    (_abi.GAMMA_HYPERBOLIC, 5, [20]),
    (_abi.GAMMA_HYPERBOLIC, 6, [8]),
    (_abi.GAMMA_HYPERBOLIC, 8, [6]),
    (_abi.GAMMA_TOTAL, 3, [9]),
    (_abi.GAMMA_TOTAL, 4, [6]),
    (_abi.GAMMA_TOTAL, 6, [4]),
    (_abi.GAMMA_FULL, 3, [3]),
    (_abi.GAMMA_FULL, 4, [3]),
    (_abi.GAMMA_FULL, 3, [5, 2, 7]),
    (_abi.GAMMA_FULL, 5, [1]),
    (_abi.GAMMA_FULL, 3, [3, 3, 0]),    # single-term leaf level
    (_abi.GAMMA_FULL, 3, [0, 0, 5]),    # one group
    (_abi.GAMMA_HYPERBOLIC, 3, [1]),
    (_abi.GAMMA_TOTAL, 4, [1]),
    (_abi.GAMMA_TOTAL, 7, [3]),
]


def _layout_check(kind, dim, degrees, seed=7):
    L = _abi.lib()
    deg = (C.c_int32 * len(degrees))(*degrees)
    info = (C.c_int64 * 8)()
    rel = C.c_double()
    err = C.create_string_buffer(512)
    st = L.qrmc_gpu_mma_layout_check(kind, dim, deg, len(degrees), seed, info, C.byref(rel), err, 512)
    assert st == 0, err.value.decode()
    return list(info), rel.value


@pytest.mark.parametrize("kind,dim,degrees", MMA_CASES, ids=lambda v: str(v))
def test_mma_layout_replays_the_series(kind, dim, degrees):
    info, rel = _layout_check(kind, dim, degrees)
    K = _abi.lib().qrmc_gpu_gamma_size(kind, dim, (C.c_int32 * len(degrees))(*degrees), len(degrees))
    assert info[0] == 1, "chain index sets with d >= 3 take the tensor-core kernels"
    assert info[1] == K
    assert info[4] == info[3], "the replay reads every fragment of the stream exactly once"
    assert info[3] * 32 >= K and info[5] >= info[3]
    assert rel < 1e-13, rel


def test_mma_layout_bench_useful_fraction():
    # 12,752 useful MACs of 32 per fragment: 83% at the bench configuration
    info, _ = _layout_check(_abi.GAMMA_HYPERBOLIC, 4, [100])
    assert 0.80 < 12752 / (32 * info[3]) <= 1.0


@pytest.mark.parametrize("kind,dim,degrees", [(_abi.GAMMA_HYPERBOLIC, 2, [10]), (_abi.GAMMA_FULL, 1, [20]),
                                               (_abi.GAMMA_TOTAL, 2, [7])])
def test_mma_layout_not_used_below_three_coordinates(kind, dim, degrees):
    info, rel = _layout_check(kind, dim, degrees)
    assert info[0] == 0 and rel == 0.0
