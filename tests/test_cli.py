"""CLI drop-in: subcommands, output lines, exit codes and
record.csv, following the reference's tests/test_driver_cli.py:75-150."""

import csv
import json
import os

import pytest

import oracle
import outio_oracle
from paper_1304_7654_b200 import case_text, load_case, tc_tiny
from paper_1304_7654_b200.cli import main
from paper_1304_7654_b200.records import (RECORD_COLUMNS, DEVICE_COLUMNS, ReportRecord,
                                          efficiency_mpi, emit_report, power_per_iteration)

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "host.json")) as fh:
    HOST = json.load(fh)


@pytest.fixture()
def tiny_cfg(tmp_path):
    path = tmp_path / "tc-tiny.cfg"
    path.write_text(case_text(tc_tiny()))
    return str(path)


@pytest.mark.parametrize("name", ["tc-tiny", "C1", "C3", "ring5", "stacked"])
@pytest.mark.parametrize("exchange,k", [("aggregated", 0), ("per-element", 2)])
def test_predict_matches_reference_forecasts(name, exchange, k, tmp_path, capsys):
    entry = HOST["cases"][name]
    cfg = tmp_path / f"{name}.cfg"
    cfg.write_text(entry["case_text"])
    for ranks, fc in entry["forecast"].items():
        assert main(["predict", "--case", str(cfg), "--machine", "xe6", "--exchange", exchange,
                     "--ranks", ranks]) == 0
        out = capsys.readouterr().out.splitlines()
        assert out[1] == f"messages_per_direction={fc[k]} bytes_per_direction={fc[k + 1]}"
        assert out[2].startswith("predicted_seconds_per_direction=")


def test_predict_tiny_per_element(tiny_cfg, capsys):
    assert main(["predict", "--case", tiny_cfg, "--machine", "xe6", "--exchange", "per-element"]) == 0
    out = capsys.readouterr().out
    assert "messages_per_direction=8" in out and "bytes_per_direction=384" in out


def test_verify_ok_mismatch_missing(tmp_path, capsys):
    case = tc_tiny()
    res = oracle.run(case, 2, record_norms=False)
    a, b = tmp_path / "a", tmp_path / "b"
    outio_oracle.write_files(a, case.blocks, case.planes, res.fields)
    outio_oracle.write_files(b, case.blocks, case.planes, res.fields)
    assert main(["verify", "--out", str(b), "--golden", str(a)]) == 0
    assert "OK       restart.bin" in capsys.readouterr().out
    blob = bytearray((b / "restart.bin").read_bytes())
    blob[10] ^= 0xFF
    (b / "restart.bin").write_bytes(bytes(blob))
    os.remove(b / "flowtec_0.bin")
    assert main(["verify", "--out", str(b), "--golden", str(a)]) == 1
    out = capsys.readouterr().out
    assert "MISMATCH restart.bin" in out and "MISSING  flowtec_0.bin" in out


def test_config_errors_exit_2(tmp_path, tiny_cfg):
    assert main(["run", "--case", str(tmp_path / "nope.cfg"), "--ranks", "1", "--out", str(tmp_path / "o")]) == 2
    bad = tmp_path / "bad.cfg"
    bad.write_text("[case]\nnharms = banana\n")
    assert main(["run", "--case", str(bad), "--ranks", "1", "--out", str(tmp_path / "o")]) == 2
    # capacity: more ranks than blocks, refused before any device work
    assert main(["run", "--case", tiny_cfg, "--ranks", "3", "--out", str(tmp_path / "o")]) == 2
    assert main(["run", "--case", tiny_cfg, "--ranks", "1", "--iterations", "0",
                 "--out", str(tmp_path / "o")]) == 2


def test_report_efficiency_and_energy(tmp_path, capsys):
    rows = [["tiny", "", "1", "1", "5", "2.000", "0", "0", "5", "36", "6", "", ""],
            ["tiny", "", "2", "1", "5", "1.250", "340", "16320", "5", "36", "6", "", ""]]
    path = tmp_path / "r.csv"
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(RECORD_COLUMNS)
        w.writerows(rows)
    assert main(["report", "--records", str(path), "--machine", "bgq"]) == 0
    cap = capsys.readouterr()
    lines = cap.out.splitlines()
    assert lines[0] == ",".join(RECORD_COLUMNS)
    eff = efficiency_mpi(2.0, 1.25, 1, 2)
    wh = power_per_iteration(1.25, 80.0, 1, 5)
    assert lines[2].endswith(f",{eff:.4f},{wh:.3f}")
    assert "efficiency" in cap.err
    recs = [ReportRecord("c", "", 1, 1, 1, 1.0, 0, 0, 0, 0, 1)]
    assert emit_report(recs)[0].splitlines()[1].endswith(",1.0000,")


@pytest.mark.gpu
def test_cli_run_verify_roundtrip(tiny_cfg, tmp_path, capsys, cuda):
    out_a, out_b, out_c = (str(tmp_path / x) for x in "abc")
    args = ["--case", tiny_cfg, "--iterations", "5"]
    assert main(["run", *args, "--ranks", "1", "--io", "per-value", "--out", out_a]) == 0
    assert main(["run", *args, "--ranks", "2", "--threads", "2", "--exchange-threads", "tagged",
                 "--out", out_b]) == 0
    assert main(["run", *args, "--ranks", "2", "--transport", "loopback", "--reduce", "per-item",
                 "--exchange", "per-element", "--out", out_c]) == 0
    for d in (out_a, out_b, out_c):
        assert os.path.exists(os.path.join(d, "flowtec_2.bin"))
    assert main(["verify", "--out", out_b, "--golden", out_a]) == 0
    assert main(["verify", "--out", out_c, "--golden", out_a]) == 0
    case = load_case(tiny_cfg)
    want = tmp_path / "oracle"
    res = oracle.run(case, 5, record_norms=False)
    outio_oracle.write_files(want, case.blocks, case.planes, res.fields)
    assert main(["verify", "--out", out_a, "--golden", str(want)]) == 0
    with open(os.path.join(out_c, "record.csv")) as fh:
        rows = list(csv.DictReader(fh))
    assert list(rows[0]) == list(RECORD_COLUMNS + DEVICE_COLUMNS)
    r = rows[0]
    # counters as the reference: 17 exchanges x 2 directions, per-element
    # messages 2 per cut cell; per-item reduce: planes * nbody collectives per iteration
    assert int(r["iterations"]) == 5 and int(r["activations"]) == 6
    assert int(r["collectives"]) == 5 * case.planes * case.nbody
    assert float(r["units_per_s"]) > 0 and 0 < float(r["roofline_frac"])
