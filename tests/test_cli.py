"""CLI surface (paper_2304_14969_b200/cli.py, mirroring the reference's
cli.py): argument handling and exit codes on CPU; the subcommands end to end
on the GPU with the reference's CSV schemas."""
from __future__ import annotations

import pytest

from paper_2304_14969_b200 import cli


def test_usage_errors_exit_2(capsys):
    assert cli.main(["min-sdrp", "--width", "54", "--depths", "7", "--circuits", "1"]) == 2
    assert cli.main(["no-such-command"]) == 2


def test_span_and_grid_parsing():
    assert cli._parse_span("3:5") == [3, 4, 5] and cli._parse_span("7,9") == [7, 9]
    assert cli._parse_grid("6x6, 12x4") == [(6, 6), (12, 4)]


def test_closed_forms():
    import numpy as np
    idx = np.arange(8)
    assert np.allclose(cli._qft_expected(3, "zero", idx), 8 ** -0.5)
    assert abs(cli._qft_expected(3, "ghz", idx)[0] - 2 / 4) < 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["hybrid", "fused"])
def test_qft_bench_csv(tmp_path, engine):
    out = tmp_path / "q.csv"
    rc = cli.main(["qft-bench", "--n-min", "6", "--n-max", "12", "--init", "ghz", "--repeats", "1",
                   "--engine", engine, "--out", str(out)])
    assert rc == 0
    lines = out.read_text().splitlines()
    assert lines[0].startswith("# engine=paper_2304_14969_b200") and "rng=pcg64" in lines[0]
    assert lines[2] == "n,init,wall_ms,peak_amplitudes,verified,engine,sweeps,hbm_gbs,hbm_frac"
    rows = [r.split(",") for r in lines[3:]]
    assert [int(r[0]) for r in rows] == list(range(6, 13)) and all(r[4] == "1" for r in rows)


@pytest.mark.gpu
def test_min_sdrp_and_validate_csv(tmp_path):
    out = tmp_path / "m.csv"
    assert cli.main(["min-sdrp", "--width", "10", "--depths", "4:5", "--circuits", "2", "--mem-budget", "4096",
                     "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[2] == "width,depth,seed,p_min,f_model,peak_amplitudes,wall_ms" and len(lines) == 3 + 4
    out = tmp_path / "v.csv"
    assert cli.main(["validate", "--grid", "6x4", "--circuits", "2", "--p-grid", "0,0.5,1", "--out", str(out)]) == 0
    rows = out.read_text().splitlines()[3:]
    assert len(rows) == 6
    for r in rows:  # p = 0 is exact: model and overlap fidelity both 1
        w, d, seed, p, fm, fe = r.split(",")[:6]
        if float(p) == 0:
            assert abs(float(fm) - 1) < 1e-12 and abs(float(fe) - 1) < 1e-9
    assert cli.main(["qft-bench", "--n-min", "8", "--n-max", "8", "--engine", "fused", "--mem-budget", "16",
                     "--out", str(tmp_path / "x.csv")]) == 4
