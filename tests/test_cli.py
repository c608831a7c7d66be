"""The reference CLI's subcommands on the B200 library (paper_2407_21084_b200/cli.py;
proj/tools/qrmc_main.cpp). Host-only parts run on CPU; solve/bench need the device."""
import json

import numpy as np
import pytest

from paper_2407_21084_b200 import api, cli


@pytest.mark.parametrize("dim,kind,deg,expect", [(6, "hyperbolic", 64, 76433), (4, "hyperbolic", 100, 12752),
                                                 (2, "full", 31, 1024), (3, "total", 5, 56)])
def test_mindex_card(capsys, dim, kind, deg, expect):
    assert cli.main(["mindex-card", "--dim", str(dim), "--kind", kind, "--deg", str(deg)]) == 0
    assert capsys.readouterr().out.strip() == str(expect)


def test_solve_dry_run(capsys):
    # christoffel number of Gamma_H(4,100) = L_Gamma = 116,641
    rc = cli.main(["solve", "--dim", "4", "--kind", "hyperbolic", "--deg", "100", "--steps", "20",
                   "--paths", "20000000", "--q", "5.1", "--dry-run"])
    out = capsys.readouterr().out
    assert rc == 0
    assert "basis size 12752, christoffel 116641" in out
    assert "dry run: memory estimate" in out


@pytest.mark.parametrize("argv", [
    ["solve", "--dim", "2", "--kind", "total", "--degrees", "3", "3", "--steps", "2", "--paths", "10"],
    ["solve", "--dim", "2", "--kind", "full", "--degrees", "3", "--steps", "2", "--paths", "10"],
    ["solve", "--dim", "0", "--steps", "2", "--paths", "10"],
    ["solve", "--dim", "2", "--steps", "2"],
])
def test_usage_errors_exit_1(argv, capsys):
    assert cli.main(argv) == 1


def test_bench_table_io_error_exit_3(tmp_path, capsys):
    bad = tmp_path / "bad.json"
    bad.write_text('{"schema": "nope"}')
    assert cli.main(["bench", "--dim", "2", "--steps", "2", "--paths", "10", "--table", str(bad)]) == 3


@pytest.mark.gpu
def test_solve_writes_artifact_and_bench_scores_it(tmp_path, capsys):
    out = tmp_path / "t.json"
    argv = ["--dim", "2", "--kind", "hyperbolic", "--deg", "6", "--steps", "5", "--paths", "20000",
            "--q", "2.1", "--seed", "7"]
    assert cli.main(["solve", *argv, "--out", str(out)]) == 0
    text = capsys.readouterr().out
    assert "wrote" in text and "value at origin, t=0:" in text
    table = api.CoefficientTable.load_json(out)
    assert table.to_json() == out.read_text()[:-1]
    meta = json.loads((tmp_path / "t.json.meta.json").read_text())
    assert meta["truncation"]["applications"] == 20000 * 5 * 6 // 2
    # the same solve through the Python API gives the same artifact bytes
    ref = api.solve(api.SinBenchmark(2, lambda_=1 / np.sqrt(2)), api.MultiIndexSet("hyperbolic", 2, (6,)),
                    api.Measure(2.0, 2), 5, 20000, 2.1, 7)
    assert ref.to_json() == table.to_json()
    rep = tmp_path / "r.csv"
    assert cli.main(["bench", *argv, "--table", str(out), "--out", str(rep), "--format", "csv"]) == 0
    lines = rep.read_text().splitlines()
    assert lines[0] == "d,delta,q,kind,degree,basis_size,paths,seed,mse_max,mse_av,wall_seconds"
    assert lines[1].startswith("2,0.2,2.1,hyperbolic,6,")
