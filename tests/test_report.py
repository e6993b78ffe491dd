"""CPU: result rows in the reference wire format (cli.py:62-65, 378-437):
golden byte-exact row (reference tests/test_cli.py:158-168), CSV / JSON round
trips, and cross-loading with the reference's own load_rows / speedup_report."""

import json

import pytest

from paper_1907_01252_b200.report import CSV_COLUMNS, ResultRow, emit_csv, emit_json, load_rows
from refimport import pintbench

HEADER = ",".join(CSV_COLUMNS)


def test_golden_row_byte_exact(tmp_path):
    row = ResultRow("heat1d", 0.05, 0.005, "classic", 2, 7, 0.001953125, 0.75)
    p = tmp_path / "one.csv"
    emit_csv([row], str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == HEADER
    assert lines[1] == "heat1d,0.050000000000000003,0.0050000000000000001,classic,2,7,0.001953125,0.75,,,,"


def test_round_trips(tmp_path):
    rows = [ResultRow("c1", 0.02, 0.002, "classic", 2, 7, 0.001953125, 0.75),
            ResultRow("c1", 0.02, 0.002, "classic", 3, None, 1e-9, None, t_seq_s=10.0, t_par_s=5.0,
                      speedup_meas=2.0, speedup_theory=4.0)]
    emit_csv(rows, str(tmp_path / "r.csv"))
    emit_json(rows, str(tmp_path / "r.json"), {"gpu": "B200"})
    assert load_rows(str(tmp_path / "r.csv")) == rows
    assert load_rows(str(tmp_path / "r.json")) == rows
    assert json.loads((tmp_path / "r.json").read_text())["metadata"]["gpu"] == "B200"


@pytest.mark.skipif(pintbench() is None, reason="reference package not available")
def test_reference_reads_our_rows(tmp_path):
    from pintbench.cli import load_rows as ref_load, speedup_report
    rows = [ResultRow("c1", 0.0, 0.002, "discretization", 0, 10, 1e-4, None),
            ResultRow("c1", 0.02, 0.002, "classic", 3, None, 5e-5, None, t_seq_s=10.0, t_par_s=2.0,
                      speedup_meas=5.0, speedup_theory=5.78)]
    emit_csv(rows, str(tmp_path / "r.csv"))
    ref_rows = ref_load(str(tmp_path / "r.csv"))
    assert [r.as_tuple() for r in ref_rows] == [r.as_tuple() for r in rows]
    assert "best K: 0.02 (classic)" in speedup_report(ref_rows)
