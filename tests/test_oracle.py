"""The CPU oracle, pinned: the C restatement (oracle/qrmc_oracle.c) against the
reference's own outputs (golden fixtures from oracle/_ref) and, where the
reference build is present, against the reference live, bit for bit.
Also the reference's published known answers (proj/tests/test_rng.cpp) and
exactness fixtures (proj/tests/test_solver.cpp)."""
import json
import hashlib
from pathlib import Path

import numpy as np
import pytest

from golden_cases import CASES, DRAW_STREAMS, PATH_CASES, build_case
from paper_2407_21084_b200 import _abi

GOLDEN = json.loads((Path(__file__).parent / "golden" / "golden_v1.json").read_text())


def unhex(a):
    return np.array([float.fromhex(x) for x in a])


def test_philox_known_answers(port):
    # Random123 KATs, proj/tests/test_rng.cpp:14-40
    expected = [[0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8],
                [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD],
                [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]]
    for kat, exp in zip(GOLDEN["philox_kat"], expected):
        assert kat["out"] == exp
        assert port.philox(kat["ctr"], kat["key"])[0].tolist() == exp
    g = GOLDEN["philox_random"]
    assert port.philox(np.array(g["ctr"]), np.array(g["key"])).tolist() == g["out"]


def test_stream_draws_bitwise(port):
    g = GOLDEN["draws"]
    sids = np.array(g["stream_ids"], dtype=np.uint64)
    assert port.stream_draws(g["seed"], sids, 12, 0).tolist() == g["u64"]
    np.testing.assert_array_equal(port.stream_draws(g["seed"], sids, 12, 1).ravel(), unhex(sum(g["uniform"], [])))
    np.testing.assert_array_equal(port.stream_draws(g["seed"], sids, 12, 2).ravel(), unhex(sum(g["normal"], [])))


def test_uniforms_open_interval(port):
    u = port.stream_draws(1, np.arange(2000, dtype=np.uint64), 100, 1)
    assert (u > 0).all() and (u < 1).all()  # test_rng.cpp:58-70


def test_normal_quantile_standard_values(port):
    # proj/tests/test_rng.cpp:72-78 tolerances
    assert abs(port.normal_quantile(0.5)) <= 1e-14
    assert port.normal_quantile(0.975) == pytest.approx(1.959963985, rel=1e-8)
    assert port.normal_quantile(0.995) == pytest.approx(2.5758293035, rel=1e-8)
    assert port.normal_quantile(0.0013498980316301) == pytest.approx(-3.0, rel=1e-10)
    g = GOLDEN["normal_quantile"]
    for p, z in zip(unhex(g["p"]), unhex(g["z"])):
        assert port.normal_quantile(p) == z


def test_normal_moments(port):
    z = port.stream_draws(2024, np.array([5], dtype=np.uint64), 200000, 2).ravel()
    assert abs(z.mean()) < 4.0 / np.sqrt(z.size)   # test_rng.cpp:80-93
    assert z.var() == pytest.approx(1.0, rel=0.02)


@pytest.mark.parametrize("g", GOLDEN["gamma"], ids=lambda g: f"{g['kind']}-{g['dim']}-{g['degrees']}")
def test_gamma_enumeration(port, g):
    rows, kmax = port.gamma(g["kind"], g["dim"], g["degrees"])
    assert rows.shape[0] == g["size"]
    assert kmax.tolist() == g["kmax"]
    assert hashlib.sha256(rows.astype("<i4").tobytes()).hexdigest() == g["sha256"]


def test_pinned_cardinalities(port):
    # proj/tests/test_multi_index.cpp:66-77, acceptance_main.cpp:103-107
    assert port.gamma(1, 3, [6])[0].shape[0] == 84
    assert port.gamma(1, 4, [5])[0].shape[0] == 126
    assert port.gamma(2, 3, [4])[0].shape[0] == 50
    assert port.gamma(2, 4, [2])[0].shape[0] == 48
    assert port.gamma(1, 2, [20])[0].shape[0] == 231
    assert port.gamma(2, 2, [19])[0].shape[0] == 99


@pytest.mark.parametrize("pc", GOLDEN["paths"], ids=lambda p: p["case"]["name"])
def test_cloud_paths_bitwise(port, pc):
    case = pc["case"]
    prob, cfg = build_case(case)
    p = port.cloud_paths(prob, cfg, case["step"], case["first"], case["n"])
    np.testing.assert_array_equal(p.ravel(), unhex(pc["paths"]))


@pytest.mark.parametrize("entry", GOLDEN["solves"], ids=lambda e: e["case"]["name"])
def test_backward_solve_bitwise_vs_reference_golden(port, entry):
    case = entry["case"]
    prob, cfg = build_case(case)
    coeffs, stats = port.backward_solve(prob, cfg, entry["basis_size"])
    np.testing.assert_array_equal(coeffs.ravel(), unhex(entry["coeffs"]))
    assert stats.applications == entry["applications"]
    assert stats.clipped == entry["clipped"]
    u00 = port.evaluate(cfg, prob.dim, coeffs[0], np.zeros(prob.dim))[0]
    assert u00 == float.fromhex(entry["u00"])
    if "mse" in entry:
        m, _ = port.mse_metrics(cfg, prob.dim, 0.6, prob.terminal_params[1], prob.horizon, coeffs, 555, 300)
        np.testing.assert_array_equal(m[:4], unhex(entry["mse"]))


def test_exactness_fixtures(port):
    # constant terminal, no driver: alpha_0 == 1.0 bitwise (test_solver.cpp:227-236)
    e = next(e for e in GOLDEN["solves"] if e["case"]["name"] == "const_terminal_driverless")
    c = unhex(e["coeffs"]).reshape(e["case"]["steps"], -1)
    assert (c[:, 0] == 1.0).all()
    assert (np.abs(c[:, 1:]) <= 3.0 / np.sqrt(400.0)).all()
    # every value clips: applications == clipped == M N (N+1)/2 (test_solver.cpp:291-303)
    e = next(e for e in GOLDEN["solves"] if e["case"]["name"] == "truncation_every_value")
    assert e["applications"] == e["clipped"] == 100 * 4 * 5 // 2
    # store == recompute bitwise (test_solver.cpp:238-262)
    a = next(e for e in GOLDEN["solves"] if e["case"]["name"] == "sin_d2_hyp6_q2.1")
    b = next(e for e in GOLDEN["solves"] if e["case"]["name"] == "sin_d2_hyp6_q2.1_recompute")
    assert a["coeffs"] == b["coeffs"]


def test_errors_match_reference(port):
    prob = _abi.custom_problem(1, _abi.TERMINAL_NAN, _abi.DRIVER_ZERO, growth_g=1.0)
    cfg = _abi.ConfigHolder(steps=2, paths=50, seed=1, gamma_kind=0, degrees=[3])
    rc, _, _ = port.backward_solve_status(prob, cfg, 4)
    assert rc == _abi.ENUMERIC  # test_solver.cpp:285-289
    prob = _abi.custom_problem(1, _abi.TERMINAL_CONST, _abi.DRIVER_ZERO, terminal_params=(1.0,),
                               drift=_abi.DRIFT_CONST, drift_params=(1e30,), growth_g=1.0)
    rc, stats, _ = port.backward_solve_status(prob, cfg, 4)
    assert rc == _abi.ESIM and stats.error_step >= 1  # test_sde.cpp:143-158
    for bad in (dict(steps=0), dict(paths=0), dict(damping=-1.0)):
        kw = dict(steps=2, paths=10, seed=1, gamma_kind=0, degrees=[2])
        kw.update(bad)
        rc, _, _ = port.backward_solve_status(_abi.sin_bench_problem(1), _abi.ConfigHolder(**kw), 3)
        assert rc == _abi.EINVAL  # test_solver.cpp:425-443


def test_port_matches_reference_live(port, ref):
    """Random small configurations: the restatement reproduces the reference bit for bit."""
    rng = np.random.default_rng(11)
    for trial in range(6):
        d = int(rng.integers(1, 4))
        kind = int(rng.integers(0, 3))
        degrees = [int(rng.integers(1, 5)) for _ in range(d)] if kind == 0 else [int(rng.integers(2, 8))]
        prob = _abi.sin_bench_problem(d)
        cfg = _abi.ConfigHolder(steps=int(rng.integers(1, 5)), paths=int(rng.integers(1, 2500)),
                                damping=float(rng.choice([0.0, 2.1, 5.1])), seed=int(rng.integers(0, 2**63)),
                                gamma_kind=kind, degrees=degrees, mu=float(rng.choice([1.0, 2.0])))
        k = ref.gamma(kind, d, degrees)[0].shape[0]
        a, sa = port.backward_solve(prob, cfg, k)
        b, sb = ref.backward_solve(prob, cfg, k)
        np.testing.assert_array_equal(a, b)
        assert (sa.applications, sa.clipped) == (sb.applications, sb.clipped)
