"""Multi-GPU correctness of the library's own sharded path, on one device.

qrmc_gpu_replay_ranks_solve runs a world-G solve's kernels for every rank on the
current device: each rank with its own lane ownership (lane_lo > 0 and
owned_lanes < 256 for G > 1, exactly as on a real rank), its own response and
cloud buffers, and writing only its own lanes' partial rows -- the rows the
per-step ncclAllGather assembles on G GPUs (host.cpp enqueue_solve). The
reference's contract that `workers` never changes results (solver.hpp:29,
test_solver.cpp:238-262) makes every G bitwise equal to the world-1 solve,
truncation counters and error status included (solver.cpp:220-223,
parallel.cpp:22-43)."""
import ctypes as C

import numpy as np
import pytest

from paper_2407_21084_b200 import _abi, api


def replay(prob, cfg, world):
    L = _abi.lib()
    K = L.qrmc_gpu_gamma_size(cfg.c.gamma_kind, prob.dim, cfg.c.degrees, cfg.c.n_degrees)
    coeffs = np.zeros((cfg.c.steps, K))
    stats = _abi.Stats()
    err = C.create_string_buffer(1024)
    st = L.qrmc_gpu_replay_ranks_solve(C.byref(prob), cfg.ref(), world, coeffs.ctypes.data_as(C.POINTER(C.c_double)),
                                       coeffs.size, C.byref(stats), err, 1024)
    return st, coeffs, stats, err.value.decode()


def test_replay_validates_world_before_touching_a_device():
    prob = _abi.sin_bench_problem(2)
    cfg = _abi.ConfigHolder(steps=2, paths=100, seed=1, gamma_kind=0, degrees=[3, 3])
    for bad in (0, -1, 257):
        st, _, _, msg = replay(prob, cfg, bad)
        assert st == _abi.EINVAL and "world" in msg


CASES = [
    # tensor-core kernels (d >= 3); M spans several chunk rounds per lane and is ragged
    dict(dim=4, kind=2, degrees=[16], steps=5, paths=300_001, damping=5.1),
    dict(dim=6, kind=2, degrees=[8], steps=3, paths=50_000, damping=5.1),
    # series-program kernels (d <= 2)
    dict(dim=2, kind=2, degrees=[19], steps=6, paths=270_000, damping=2.1),
    # fewer chunks than lanes: most ranks own no paths at all for G = 8
    dict(dim=3, kind=1, degrees=[6], steps=4, paths=5_000, damping=0.0),
]


@pytest.mark.gpu
@pytest.mark.parametrize("c", CASES, ids=lambda c: f"d{c['dim']}_k{c['kind']}_M{c['paths']}")
@pytest.mark.parametrize("world", [2, 3, 8])
def test_every_world_is_bitwise_equal_to_the_single_rank_solve(c, world):
    import torch
    assert torch.cuda.is_available()
    prob = _abi.sin_bench_problem(c["dim"])
    cfg = _abi.ConfigHolder(steps=c["steps"], paths=c["paths"], damping=c["damping"], seed=2407,
                            gamma_kind=c["kind"], degrees=c["degrees"])
    ref, rs, _ = api.backward_solve(prob, cfg)
    st, got, gs, msg = replay(prob, cfg, world)
    assert st == _abi.OK, msg
    np.testing.assert_array_equal(got, ref)
    assert (gs.applications, gs.clipped) == (rs.applications, rs.clipped)
    n = c["steps"]
    assert gs.applications == c["paths"] * n * (n + 1) // 2
    assert gs.kernel_launches == (2 * world + 1) * n


@pytest.mark.gpu
@pytest.mark.parametrize("split", ["1", "2"])
@pytest.mark.parametrize("world", [2, 8])
def test_k2_lane_split_keeps_worlds_bitwise_equal(monkeypatch, split, world):
    # K2 may split each lane's chunks over two CTAs (QRMC_K2_SPLIT; host.cpp decides on the
    # 256-lane grid whatever the world size), so both settings must stay G-independent
    monkeypatch.setenv("QRMC_K2_SPLIT", split)
    prob = _abi.sin_bench_problem(4)
    cfg = _abi.ConfigHolder(steps=4, paths=400_003, damping=5.1, seed=77, gamma_kind=2, degrees=[40])
    ref, rs, _ = api.backward_solve(prob, cfg)
    st, got, gs, msg = replay(prob, cfg, world)
    assert st == _abi.OK, msg
    np.testing.assert_array_equal(got, ref)
    assert (gs.applications, gs.clipped) == (rs.applications, rs.clipped)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 3])
def test_errors_are_global_across_ranks(world):
    """A SimulationError on any path fails the whole solve with the smallest step,
    whichever rank owns the path; a NumericError likewise."""
    blow = _abi.custom_problem(3, _abi.TERMINAL_CONST, _abi.DRIVER_ZERO, terminal_params=(1.0,),
                               drift=_abi.DRIFT_CONST, drift_params=(1e30,), growth_g=1.0)
    cfg = _abi.ConfigHolder(steps=3, paths=40_000, seed=1, gamma_kind=2, degrees=[4])
    st, _, _, msg = replay(blow, cfg, world)
    assert st == _abi.ESIM and "step" in msg
    nan = _abi.custom_problem(3, _abi.TERMINAL_NAN, _abi.DRIVER_ZERO, growth_g=1.0)
    st, _, _, _ = replay(nan, cfg, world)
    assert st == _abi.ENUMERIC
