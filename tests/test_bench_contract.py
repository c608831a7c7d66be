"""bench.py's JSON contract: the committed run of record (CPU) and a small live run (GPU).

The keys and relations the driver reads: metric/value/unit, ms_per_step, roofline (achieved /
peak = frac, traffic), e2e (value, unit, h2d/d2h bytes), gpu_launches, clocks, cpu_baseline,
and the SRMC / config-4 objects."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"]


def check_line(d: dict, srmc: bool, config4: bool):
    for k in REQUIRED:
        assert k in d, k
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT and d["higher_is_better"] is True
    n = d["config"]["N"]
    m = d["config"]["paths_total"]
    assert abs(d["value"] - bench.path_steps(m, n) / (d["ms_per_step"] / 1e3)) <= 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "fp64" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert 0 < r["frac"] < 1 and "builder-measured" in r["peak_source"]
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 3 * n * d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    if srmc:
        assert set(d["srmc"]) == {"config2", "config3", "config4"}
        for v in d["srmc"].values():
            assert abs(v["roofline"]["frac"] - v["roofline"]["achieved"] / v["roofline"]["peak"]) < 1e-12
    if config4:
        c = d["gqrmdp_config4"]
        assert c["basis_size"] == 76433 and c["N"] == 10 and c["value"] > 0


def test_run_of_record_keeps_the_contract():
    d = json.loads((ROOT / "profiles" / "r02_bench.json").read_text())
    check_line(d, srmc=True, config4=True)
    assert d["n_gpus"] == 1 and d["config"]["paths_per_gpu"] == bench.DEFAULT_PATHS_PER_GPU
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["extrapolated"] is True
    ref = json.loads((ROOT / "profiles" / "r02_bench_reference.json").read_text())
    assert ref["impl"] == "reference" and ref["metric"] == d["metric"] and ref["unit"] == d["unit"]
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["e2e"]["value"] == ref["value"]


def test_flop_counts_are_the_stated_formulas():
    assert bench.srmc_flops_per_path_step(4, 5) == 267
    assert bench.srmc_flops_per_path_step(6, 1) == 327
    assert bench.path_steps(10, 20) == 10 * 20 * 21 // 2


@pytest.mark.gpu
def test_small_live_bench_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "3", "--paths",
                          "200000", "--no-cpu-baseline", "--no-srmc", "--no-config4", "--e2e-steps", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    check_line(d, srmc=False, config4=False)
    assert d["config"]["paths_per_gpu"] == 200000
