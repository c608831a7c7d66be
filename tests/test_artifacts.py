"""Coefficient artifacts: the library's `qrmc.coefficients.v1`
writer against the reference's own table_to_json (proj/src/table_io.cpp:45-73, run
from oracle/_ref), byte for byte, and the Python load path (table_from_json,
table_io.cpp:83-125). Host-only."""
import ctypes as C

import numpy as np
import pytest

from paper_2407_21084_b200 import _abi, api

CASES = [
    dict(kind=_abi.GAMMA_HYPERBOLIC, dim=4, degrees=[12], steps=3, damping=5.1, mu=2.0, center=None),
    dict(kind=_abi.GAMMA_TOTAL, dim=3, degrees=[5], steps=2, damping=0.0, mu=1.0, center=[0.5, -1.25, 3.0]),
    dict(kind=_abi.GAMMA_FULL, dim=2, degrees=[4], steps=4, damping=2.1, mu=2.0, center=None),
    dict(kind=_abi.GAMMA_FULL, dim=3, degrees=[2, 0, 3], steps=1, damping=0.0, mu=2.0, center=[1e-5, 0.0, -7.0]),
    dict(kind=_abi.GAMMA_HYPERBOLIC, dim=1, degrees=[7], steps=5, damping=0.0, mu=2.0, center=None),
]


def _cfg(case, paths=123457, seed=2 ** 63 + 5):
    return _abi.ConfigHolder(steps=case["steps"], paths=paths, damping=case["damping"], seed=seed,
                             gamma_kind=case["kind"], degrees=case["degrees"], mu=case["mu"],
                             center=case["center"])


def _coeffs(case, rng):
    K = _abi.lib().qrmc_gpu_gamma_size(case["kind"], case["dim"], (C.c_int32 * len(case["degrees"]))(*case["degrees"]),
                                       len(case["degrees"]))
    c = rng.standard_normal((case["steps"], K)) * 10.0 ** rng.integers(-12, 12, (case["steps"], K))
    # formatting corner cases: integral values, signed zero, tiny/huge, short decimals
    specials = [0.0, -0.0, 1.0, -3.0, 0.1, 1e-5, 1.5e-7, 123456789.0, 1e21, 2.5e-300, 5e-324,
                1.7976931348623157e308, 0.30000000000000004]
    flat = c.reshape(-1)
    flat[: min(len(specials), flat.size)] = specials[: flat.size]
    return c


def _ours(cfg, dim, horizon, coeffs):
    L = _abi.lib()
    err = C.create_string_buffer(512)
    p = coeffs.ctypes.data_as(C.POINTER(C.c_double))
    n = L.qrmc_gpu_table_json(cfg.ref(), dim, horizon, p, None, 0, err, 512)
    assert n > 0, err.value
    buf = C.create_string_buffer(int(n))
    assert L.qrmc_gpu_table_json(cfg.ref(), dim, horizon, p, buf, int(n), err, 512) == n
    return buf.value


def _theirs(ref, cfg, dim, horizon, coeffs):
    f = ref.L.qrmc_ref_table_json
    f.argtypes = [C.POINTER(_abi.Config), C.c_int32, C.c_double, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]
    f.restype = C.c_int64
    p = coeffs.ctypes.data_as(C.POINTER(C.c_double))
    n = f(cfg.ref(), dim, horizon, p, None, 0)
    assert n > 0
    buf = C.create_string_buffer(int(n))
    f(cfg.ref(), dim, horizon, p, buf, int(n))
    return buf.value


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['kind']}-{c['dim']}-{c['degrees']}")
def test_table_json_bytes_match_reference(ref, case):
    rng = np.random.default_rng(case["dim"] * 7 + case["steps"])
    cfg = _cfg(case)
    coeffs = np.ascontiguousarray(_coeffs(case, rng))
    for horizon in (1.0, 0.75, 2.0 / 3.0):
        assert _ours(cfg, case["dim"], horizon, coeffs) == _theirs(ref, cfg, case["dim"], horizon, coeffs)


def test_table_json_round_trip(tmp_path):
    case = CASES[0]
    rng = np.random.default_rng(3)
    coeffs = _coeffs(case, rng)
    gamma = api.MultiIndexSet("hyperbolic", 4, (12,))
    t = api.CoefficientTable(case["steps"], 123457, 5.1, 2 ** 63 + 5, 1.0, api.Measure(2.0, 4), gamma, coeffs)
    f = tmp_path / "table.json"
    t.save_json(f)
    raw = f.read_bytes()
    assert raw.endswith(b"\n") and raw[:-1].decode() == t.to_json()
    back = api.CoefficientTable.load_json(f)
    assert (back.steps, back.paths, back.damping, back.seed, back.horizon) == (t.steps, t.paths, t.damping, t.seed, 1.0)
    np.testing.assert_array_equal(back.table, coeffs)  # shortest round-trip formatting: exact
    assert back.to_json() == t.to_json()


@pytest.mark.parametrize("mutate,msg", [
    (lambda d: d.replace('"qrmc.coefficients.v1"', '"qrmc.coefficients.v0"'), "unknown schema"),
    (lambda d: d.replace('"step":0', '"step":9'), "out of range"),
    (lambda d: d.replace('[[0,0,0,0],', '[[0,0,0,1],', 1), "index order"),
    (lambda d: d[: len(d) // 2], "parse error"),
])
def test_table_json_load_rejects_bad_documents(mutate, msg):
    case = CASES[0]
    coeffs = _coeffs(case, np.random.default_rng(4))
    t = api.CoefficientTable(case["steps"], 10, 5.1, 1, 1.0, api.Measure(2.0, 4),
                             api.MultiIndexSet("hyperbolic", 4, (12,)), coeffs)
    with pytest.raises(ValueError, match=msg):
        api.CoefficientTable.from_json(mutate(t.to_json()))
