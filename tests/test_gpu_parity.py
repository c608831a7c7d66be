"""GPU parity: the sm_100a library, called through the C ABI, against the
reference (golden fixtures from oracle/_ref) and the C restatement (live).

Tolerances: integer and replay work is bit-exact
(Philox words, stream ids, uniforms, Gamma order, truncation counters);
Gaussians, Euler paths and mu=2 starts are bit-exact except where CUDA's
log() differs from glibc by an ulp; coefficient tables satisfy
max_k |alpha_gpu - alpha_ref| <= 1e-10 * max(1, max_k |alpha_ref|) and
|u_gpu(0, x0) - u_ref(0, x0)| <= 1e-10."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from golden_cases import CASES, build_case
from paper_2407_21084_b200 import _abi, api

pytestmark = pytest.mark.gpu
GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden_v1.json").read_text())
ALPHA_TOL = 1e-10


def unhex(a):
    return np.array([float.fromhex(x) for x in a])


def alpha_close(a, b):
    scale = max(1.0, float(np.abs(b).max()))
    return float(np.abs(a - b).max()) / scale


@pytest.fixture(scope="module")
def L():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return _abi.lib()


def test_philox_on_device(L):
    g = GOLDEN["philox_random"]
    ctr = np.ascontiguousarray(g["ctr"], dtype=np.uint32)
    key = np.ascontiguousarray(g["key"], dtype=np.uint32)
    out = np.zeros_like(ctr)
    err = C.create_string_buffer(256)
    P = C.POINTER(C.c_uint32)
    assert L.qrmc_gpu_philox(ctr.ctypes.data_as(P), key.ctypes.data_as(P), len(ctr), out.ctypes.data_as(P), err, 256) == 0
    assert out.tolist() == g["out"]
    for kat in GOLDEN["philox_kat"]:
        c = np.array([kat["ctr"]], dtype=np.uint32)
        k = np.array([kat["key"]], dtype=np.uint32)
        o = np.zeros_like(c)
        assert L.qrmc_gpu_philox(c.ctypes.data_as(P), k.ctypes.data_as(P), 1, o.ctypes.data_as(P), err, 256) == 0
        assert o[0].tolist() == kat["out"]


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_stream_draws_on_device(L, kind):
    g = GOLDEN["draws"]
    sids = np.array(g["stream_ids"], dtype=np.uint64)
    out = np.zeros((len(sids), 12), dtype=np.uint64 if kind == 0 else np.float64)
    err = C.create_string_buffer(256)
    assert L.qrmc_gpu_stream_draws(g["seed"], sids.ctypes.data_as(C.POINTER(C.c_uint64)), len(sids), 12, kind,
                                   out.ctypes.data_as(C.c_void_p), err, 256) == 0
    if kind == 0:
        assert out.tolist() == g["u64"]
    elif kind == 1:
        np.testing.assert_array_equal(out.ravel(), unhex(sum(g["uniform"], [])))
    else:
        ref = unhex(sum(g["normal"], []))
        np.testing.assert_allclose(out.ravel(), ref, rtol=4e-16, atol=0)


def test_stream_draws_many_vs_port(L, port):
    sids = (np.arange(4096, dtype=np.uint64) * np.uint64(2654435761)) | (np.uint64(7) << np.uint64(40))
    out = np.zeros((4096, 8))
    err = C.create_string_buffer(256)
    assert L.qrmc_gpu_stream_draws(123, sids.ctypes.data_as(C.POINTER(C.c_uint64)), 4096, 8, 2,
                                   out.ctypes.data_as(C.c_void_p), err, 256) == 0
    ref = port.stream_draws(123, sids, 8, 2)
    ulps = np.abs(out - ref) / np.spacing(np.abs(ref))
    assert ulps.max() <= 4
    assert (out == ref).mean() > 0.99


@pytest.mark.parametrize("pc", GOLDEN["paths"], ids=lambda p: p["case"]["name"])
def test_cloud_paths_on_device(L, pc):
    case = pc["case"]
    prob, cfg = build_case(case)
    n = case["n"]
    out = np.zeros((n, case["steps"] - case["step"] + 1, prob.dim))
    err = C.create_string_buffer(256)
    assert L.qrmc_gpu_cloud_paths(C.byref(prob), cfg.ref(), case["step"], case["first"], n,
                                  out.ctypes.data_as(C.POINTER(C.c_double)), err, 256) == 0, err.value
    ref = unhex(pc["paths"]).reshape(out.shape)
    if case.get("mu", 2.0) == 2.0:
        np.testing.assert_array_equal(out[:, 0, :], ref[:, 0, :])  # mu=2 starts: correctly rounded ops, bit-exact
    np.testing.assert_allclose(out, ref, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("entry", GOLDEN["solves"], ids=lambda e: e["case"]["name"])
def test_backward_solve_matches_reference(L, entry):
    case = entry["case"]
    prob, cfg = build_case(case)
    coeffs, stats, _ = api.backward_solve(prob, cfg)
    ref = unhex(entry["coeffs"]).reshape(coeffs.shape)
    assert alpha_close(coeffs, ref) <= ALPHA_TOL
    assert stats.applications == entry["applications"]
    assert stats.clipped == entry["clipped"]
    mu = case.get("mu", 2.0)
    gam = api.MultiIndexSet({0: "full", 1: "total", 2: "hyperbolic"}[case["kind"]], prob.dim, tuple(case["degrees"]))
    table = api.CoefficientTable(case["steps"], case["paths"], case["damping"], case["seed"], 1.0,
                                 api.Measure(mu, prob.dim, tuple(case.get("center", ()))), gam, coeffs)
    assert abs(table.evaluate(0, np.zeros(prob.dim)) - float.fromhex(entry["u00"])) <= 1e-10
    if "mse" in entry:
        bench = api.SinBenchmark(prob.dim)
        rep = api.mse_metrics(table, bench, 555, 300)
        np.testing.assert_allclose([rep.mse_max, rep.mse_av, rep.mse_max_undamped, rep.mse_av_undamped],
                                   unhex(entry["mse"]), rtol=1e-9)


def test_constant_terminal_recovered_exactly(L):
    prob, cfg = build_case(next(c for c in CASES if c["name"] == "const_terminal_driverless"))
    coeffs, _, _ = api.backward_solve(prob, cfg)
    assert (coeffs[:, 0] == 1.0).all()  # test_solver.cpp:227-236 (bitwise)


@pytest.mark.parametrize("cfgkw", [
    dict(dim=4, kind=2, degrees=[16], steps=6, paths=20_000, damping=5.1, mu=2.0),
    dict(dim=6, kind=2, degrees=[8], steps=4, paths=8_000, damping=5.1, mu=2.0),
    dict(dim=2, kind=0, degrees=[31, 31], steps=10, paths=102_400, damping=0.0, mu=2.0),  # BASELINE configs[0]
    dict(dim=3, kind=1, degrees=[9], steps=5, paths=30_000, damping=2.1, mu=1.0),
    dict(dim=1, kind=0, degrees=[100], steps=20, paths=20_000, damping=2.1, mu=2.0),
    dict(dim=5, kind=2, degrees=[12], steps=3, paths=5_000, damping=5.1, mu=2.0),
    dict(dim=8, kind=2, degrees=[4], steps=3, paths=3_000, damping=5.1, mu=2.0),
    # tensor-core layout edge shapes: a zero-degree coordinate, a single-term leaf
    # level, one group, tiny sets, ragged last chunks of 1024 paths
    dict(dim=3, kind=0, degrees=[2, 0, 3], steps=4, paths=5_000, damping=0.0, mu=2.0),
    dict(dim=3, kind=0, degrees=[3, 3, 0], steps=3, paths=4_097, damping=2.1, mu=2.0),
    dict(dim=3, kind=0, degrees=[0, 0, 5], steps=3, paths=3_000, damping=0.0, mu=2.0),
    dict(dim=3, kind=2, degrees=[1], steps=3, paths=2_049, damping=5.1, mu=2.0),
    dict(dim=4, kind=1, degrees=[1], steps=4, paths=1_000, damping=0.0, mu=1.0),
    dict(dim=7, kind=1, degrees=[3], steps=3, paths=3_333, damping=5.1, mu=2.0),
    dict(dim=4, kind=2, degrees=[100], steps=3, paths=1_025, damping=5.1, mu=2.0),
])
def test_backward_solve_matches_port_live(L, port, cfgkw):
    prob = _abi.sin_bench_problem(cfgkw["dim"])
    cfg = _abi.ConfigHolder(steps=cfgkw["steps"], paths=cfgkw["paths"], damping=cfgkw["damping"], seed=2407,
                            gamma_kind=cfgkw["kind"], degrees=cfgkw["degrees"], mu=cfgkw["mu"])
    coeffs, stats, _ = api.backward_solve(prob, cfg)
    ref, rs = port.backward_solve(prob, cfg, coeffs.shape[1])
    assert alpha_close(coeffs, ref) <= ALPHA_TOL
    n, m = cfgkw["steps"], cfgkw["paths"]
    assert stats.applications == rs.applications == m * n * (n + 1) // 2
    assert abs(int(stats.clipped) - int(rs.clipped)) <= max(1, rs.clipped // 100000)


def test_determinism_and_memory_modes(L):
    prob = _abi.sin_bench_problem(3)
    kw = dict(steps=5, paths=50_000, damping=2.1, seed=99, gamma_kind=2, degrees=[10])
    a, _, _ = api.backward_solve(prob, _abi.ConfigHolder(**kw))
    b, _, _ = api.backward_solve(prob, _abi.ConfigHolder(**kw))
    c, _, _ = api.backward_solve(prob, _abi.ConfigHolder(memory_mode=_abi.MEMORY_RECOMPUTE, **kw))
    d, _, _ = api.backward_solve(prob, _abi.ConfigHolder(workers=1, **kw))
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(a, c)  # store == recompute (test_solver.cpp:254)
    np.testing.assert_array_equal(a, d)  # workers never change results
    kw["seed"] = 100
    e, _, _ = api.backward_solve(prob, _abi.ConfigHolder(**kw))
    assert not np.array_equal(a, e)


def test_errors_surface_as_reference_exceptions(L):
    nan = _abi.custom_problem(1, _abi.TERMINAL_NAN, _abi.DRIVER_ZERO, growth_g=1.0)
    with pytest.raises(api.NumericError):
        api.backward_solve(nan, _abi.ConfigHolder(steps=2, paths=50, seed=1, gamma_kind=0, degrees=[3]))
    blow = _abi.custom_problem(1, _abi.TERMINAL_CONST, _abi.DRIVER_ZERO, terminal_params=(1.0,),
                               drift=_abi.DRIFT_CONST, drift_params=(1e30,), growth_g=1.0)
    with pytest.raises(api.SimulationError) as ei:
        api.backward_solve(blow, _abi.ConfigHolder(steps=3, paths=50, seed=1, gamma_kind=0, degrees=[3]))
    assert ei.value.step >= 1


def test_evaluate_matches_reference(L, port):
    prob, cfg = build_case(CASES[1])
    coeffs, _, _ = api.backward_solve(prob, cfg)
    rng = np.random.default_rng(3)
    x = rng.standard_t(2, size=(500, 2))
    gam = api.MultiIndexSet.hyperbolic(2, 6)
    table = api.CoefficientTable(5, 4000, 2.1, 4242, 1.0, api.Measure(2.0, 2), gam, coeffs)
    got = table.evaluate(2, x)
    ref = port.evaluate(cfg, 2, coeffs[2], x)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-13)


def test_full_size_properties_config2(L):
    """BASELINE configs[1] workload at M = 2e6 (one tenth of the bench's M):
    size-independent properties -- exact application count, bitwise repeat,
    finite table, clip fraction in the reference's range (test_solver.cpp:219-224)."""
    prob = _abi.sin_bench_problem(4)
    kw = dict(steps=20, paths=2_000_000, damping=5.1, seed=42, gamma_kind=2, degrees=[100])
    a, sa, _ = api.backward_solve(prob, _abi.ConfigHolder(**kw))
    b, sb, _ = api.backward_solve(prob, _abi.ConfigHolder(**kw))
    np.testing.assert_array_equal(a, b)
    assert sa.applications == 2_000_000 * 20 * 21 // 2
    assert sa.clipped == sb.clipped
    assert np.isfinite(a).all()
    assert sa.clipped / sa.applications < 0.15  # q=5.1 re-amplifies tail noise (test_solver.cpp:216-224)
    # alpha_0 approximates the damped solution's leading coefficient: u(0, 0) ~ 1.6
    gam = api.MultiIndexSet.hyperbolic(4, 100)
    t = api.CoefficientTable(20, 2_000_000, 5.1, 42, 1.0, api.Measure(2.0, 4), gam, a)
    assert abs(t.evaluate(0, np.zeros(4)) - 1.6) < 0.25  # M / Christoffel number ~ 17 here: coarse


def test_statistical_table1_and_table2(L):
    """Statistical agreement with the closed form, the reference's acceptance
    criteria (acceptance_main.cpp:277-328; PAPER Table 1 row 1, Table 2)."""
    bench = api.SinBenchmark(1)
    gam = api.MultiIndexSet.full([100])
    meas = api.Measure(2.0, 1)
    q0_max, q0_av, q21_max, q21_av, origin = [], [], [], [], []
    for r in range(50):
        t = api.solve(bench, gam, meas, steps=20, paths=20000, damping=0.0, seed=20000 + r)
        rep = api.mse_metrics(t, bench, 555, 1000)
        q0_max.append(rep.mse_max)
        q0_av.append(rep.mse_av)
        origin.append(t.evaluate(0, np.zeros(1)))
    for r in range(20):
        t = api.solve(bench, gam, meas, steps=20, paths=20000, damping=2.1, seed=20000 + r)
        rep = api.mse_metrics(t, bench, 555, 1000)
        q21_max.append(rep.mse_max)
        q21_av.append(rep.mse_av)
    assert abs(np.mean(q0_max[:20]) - (-3.658)) <= 0.5
    assert abs(np.mean(q0_av[:20]) - (-3.868)) <= 0.5
    assert abs(np.mean(q21_max) - (-4.615)) <= 0.5
    assert sum(q21_av[r] < q0_av[r] for r in range(20)) >= 18
    lo, hi = api.confidence_interval(origin, 0.99)
    assert lo <= 1.6 <= hi and hi - lo <= 0.15


# ---------------------------------------------------------------- kernel families
# d >= 3 plans run the FP64 tensor-core kernels (responses_mma.cu, project_mma.cu);
# QRMC_K1=series / QRMC_K2=series force the series-program kernels. Both families
# must reproduce the reference's goldens.
def _kernel_names(prob, cfg):
    L = _abi.lib()
    plan = C.c_void_p()
    err = C.create_string_buffer(512)
    assert L.qrmc_gpu_plan_create(None, C.byref(prob), cfg.ref(), C.byref(plan), err, 512) == 0, err.value
    try:
        return [L.qrmc_gpu_plan_kernel_name(plan, w).decode() for w in range(3)]
    finally:
        L.qrmc_gpu_plan_destroy(plan)


@pytest.mark.parametrize("entry", GOLDEN["solves"],
                         ids=lambda e: e["case"]["name"])
def test_series_program_kernels_match_reference(L, entry, monkeypatch):
    case = entry["case"]
    prob, cfg = build_case(case)
    monkeypatch.setenv("QRMC_K1", "series")
    monkeypatch.setenv("QRMC_K2", "series")
    assert _kernel_names(prob, cfg)[:2] == ["k_responses", "k_project"]
    coeffs, stats, _ = api.backward_solve(prob, cfg)
    ref = unhex(entry["coeffs"]).reshape(coeffs.shape)
    assert alpha_close(coeffs, ref) <= ALPHA_TOL
    assert stats.applications == entry["applications"]
    assert stats.clipped == entry["clipped"]


@pytest.mark.parametrize("dim,kind,deg", [(3, 2, [8]), (4, 2, [100]), (6, 2, [8]), (4, 1, [6]), (5, 0, [2])])
def test_tensor_core_kernels_selected(L, dim, kind, deg):
    prob = _abi.sin_bench_problem(dim)
    cfg = _abi.ConfigHolder(steps=3, paths=2048, damping=5.1, seed=1, gamma_kind=kind, degrees=deg)
    k1 = "k_responses_ws" if dim <= 4 else "k_responses_mma"  # host.cpp make_plan policy
    assert _kernel_names(prob, cfg) == [k1, "k_project_mma", "k_finish_step"]


@pytest.mark.parametrize("entry", [e for e in GOLDEN["solves"] if e["case"]["dim"] >= 3],
                         ids=lambda e: e["case"]["name"])
def test_ring_tensor_core_k1_matches_reference(L, entry, monkeypatch):
    # QRMC_K1=mma keeps the single-buffered k_responses_mma (cp.async fragment
    # rings) that the warp-specialised K1 replaced; both must reproduce the goldens
    case = entry["case"]
    prob, cfg = build_case(case)
    monkeypatch.setenv("QRMC_K1", "mma")
    assert _kernel_names(prob, cfg)[0] == "k_responses_mma"
    coeffs, stats, _ = api.backward_solve(prob, cfg)
    ref = unhex(entry["coeffs"]).reshape(coeffs.shape)
    assert alpha_close(coeffs, ref) <= ALPHA_TOL
    assert (stats.applications, stats.clipped) == (entry["applications"], entry["clipped"])


@pytest.mark.parametrize("split", ["1", "2"])
def test_k2_lane_split_matches_port(L, port, monkeypatch, split):
    # K2's two-CTA lane split (half 0 + half 1, combined by the later CTA) and the single
    # CTA per lane both reproduce the restatement; M gives lanes of 1 and 2 chunks
    monkeypatch.setenv("QRMC_K2_SPLIT", split)
    prob = _abi.sin_bench_problem(4)
    cfg = _abi.ConfigHolder(steps=3, paths=300_000, damping=5.1, seed=19, gamma_kind=2, degrees=[20])
    coeffs, stats, _ = api.backward_solve(prob, cfg)
    ref, rs = port.backward_solve(prob, cfg, coeffs.shape[1])
    assert float(np.abs(coeffs - ref).max()) / max(1.0, float(np.abs(ref).max())) <= ALPHA_TOL
    assert (stats.applications, stats.clipped) == (rs.applications, rs.clipped)


@pytest.mark.parametrize("dim,deg,paths", [(3, 8, 5000), (4, 100, 3000), (6, 16, 2051)])
def test_k2_batch_width_does_not_change_bits(L, monkeypatch, dim, deg, paths):
    # K2 stages 24 or 16 paths per shared-memory batch (host.cpp picks by d and fit);
    # a chunk's short last batch adds exact zeros, so the tensor-core sum over paths
    # runs in the same order either way and the coefficients agree bit for bit
    prob = _abi.sin_bench_problem(dim)
    cfg = _abi.ConfigHolder(steps=3, paths=paths, damping=5.1, seed=5, gamma_kind=2, degrees=[deg])
    monkeypatch.setenv("QRMC_K2_BATCH", "24")
    wide, sw, _ = api.backward_solve(prob, cfg)
    monkeypatch.setenv("QRMC_K2_BATCH", "16")
    assert _kernel_names(prob, cfg)[1] == "k_project_mma"
    narrow, sn, _ = api.backward_solve(prob, cfg)
    np.testing.assert_array_equal(wide, narrow)
    assert (sw.applications, sw.clipped) == (sn.applications, sn.clipped)


@pytest.mark.parametrize("dim,deg", [(5, 12), (6, 8)])
def test_forced_ws_k1_matches_port_for_more_coordinates(L, port, monkeypatch, dim, deg):
    # the warp-specialised K1 stays correct where the plan prefers k_responses_mma
    monkeypatch.setenv("QRMC_K1", "ws")
    prob = _abi.sin_bench_problem(dim)
    cfg = _abi.ConfigHolder(steps=3, paths=4000, damping=5.1, seed=21, gamma_kind=2, degrees=[deg])
    assert _kernel_names(prob, cfg)[0] == "k_responses_ws"
    coeffs, stats, _ = api.backward_solve(prob, cfg)
    ref, rs = port.backward_solve(prob, cfg, coeffs.shape[1])
    assert alpha_close(coeffs, ref) <= ALPHA_TOL
    assert stats.applications == rs.applications


def test_ws_and_ring_k1_agree_at_config2_shape(L, monkeypatch):
    prob = _abi.sin_bench_problem(4)
    cfg = _abi.ConfigHolder(steps=6, paths=40_000, damping=5.1, seed=3, gamma_kind=2, degrees=[100])
    a, sa, _ = api.backward_solve(prob, cfg)
    monkeypatch.setenv("QRMC_K1", "mma")
    b, sb, _ = api.backward_solve(prob, cfg)
    assert alpha_close(a, b) <= ALPHA_TOL
    assert (sa.applications, sa.clipped) == (sb.applications, sb.clipped)


def test_tensor_core_and_series_kernels_agree(L):
    # same solve through both kernel families: agreement to rounding
    prob = _abi.sin_bench_problem(4)
    cfg = _abi.ConfigHolder(steps=6, paths=30000, damping=5.1, seed=11, gamma_kind=2, degrees=[24])
    a, sa, _ = api.backward_solve(prob, cfg)
    import os
    os.environ["QRMC_K1"] = "series"
    os.environ["QRMC_K2"] = "series"
    try:
        b, sb, _ = api.backward_solve(prob, cfg)
    finally:
        del os.environ["QRMC_K1"]
        del os.environ["QRMC_K2"]
    assert alpha_close(a, b) <= ALPHA_TOL
    assert (sa.applications, sa.clipped) == (sb.applications, sb.clipped)


def test_tensor_core_kernels_fall_back_when_tables_exceed_smem(L):
    # per-path cosine tables of 2 x 601 + 3 entries do not fit shared memory with 32
    # paths: the plan takes the series-program kernels (still no CPU fallback)
    prob = _abi.sin_bench_problem(3)
    cfg = _abi.ConfigHolder(steps=2, paths=1024, damping=0.0, seed=1, gamma_kind=_abi.GAMMA_FULL,
                            degrees=[600, 600, 2])
    assert _kernel_names(prob, cfg)[:2] == ["k_responses", "k_project"]
