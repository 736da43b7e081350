"""CLI (`python -m paper_2408_11417_b200.cli`) mirroring the reference's gemmsched CLI."""

import json
import os
import subprocess
import sys

import pytest

import paper_2408_11417_b200 as sk
from paper_2408_11417_b200 import cli

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_report_matches_reference_build_report(tmp_path):
    path = tmp_path / "records.csv"
    path.write_text(GOLD["report_case"]["records_csv"])
    out = tmp_path / "report.json"
    assert cli.main(["report", "--records", str(path), "--out", str(out)]) == 0
    assert json.loads(out.read_text()) == GOLD["report_case"]["report"]
    assert cli.main(["report", "--records", str(path), "--tolerances", "0,30", "--out", str(out)]) == 0
    assert json.loads(out.read_text()) == GOLD["report_case"]["report_tol"]


def test_report_errors(tmp_path, capsys):
    assert cli.main(["report", "--records", str(tmp_path / "missing.csv")]) == 1
    bad = tmp_path / "bad.csv"
    bad.write_text("nope\n")
    assert cli.main(["report", "--records", str(bad)]) == 1
    assert "bad header" in capsys.readouterr().err


def test_query_against_reference_bank(tmp_path, capsys):
    path = tmp_path / "bank.sieve"
    path.write_bytes(bytes.fromhex(GOLD["small_bank"]["hex"]))
    (m, n, k), want = GOLD["small_bank"]["queries"][0]
    assert cli.main(["query", "--sieve", str(path), "--size", f"{m}x{n}x{k}", "--repeat", "1000"]) == 0
    out = capsys.readouterr().out
    labels = [sk.canonical_policies()[o].label for o in want]
    assert f"candidates for {m}x{n}x{k}: " + (", ".join(labels) if labels else "(none)") in out
    assert "median" in out


def test_query_rejects_corrupt_bank(tmp_path, capsys):
    data = bytearray.fromhex(GOLD["small_bank"]["hex"])
    data[50] ^= 1
    path = tmp_path / "bad.sieve"
    path.write_bytes(bytes(data))
    assert cli.main(["query", "--sieve", str(path), "--size", "1x2x3"]) == 1
    assert "ChecksumError" in capsys.readouterr().err


def test_argument_parsing():
    assert cli.parse_tile("128x256x64") == sk.TileShape(128, 256, 64)
    assert cli.parse_size("1x2x3") == sk.ProblemSize(1, 2, 3)
    assert cli.parse_range("64:8192").values()[0] == 64
    assert cli.parse_tolerances("0,5,20") == [0.0, 0.05, 0.2]
    with pytest.raises(SystemExit):
        cli.main(["tune", "--tile", "128x", "--out-sieve", "a", "--out-records", "b"])


def test_module_entry_point_help():
    res = subprocess.run([sys.executable, "-m", "paper_2408_11417_b200.cli", "--help"], capture_output=True,
                         text=True, cwd=ROOT)
    assert res.returncode == 0 and "tune" in res.stdout and "verify" in res.stdout


@pytest.mark.gpu
def test_tune_tiny_grid_and_verify_on_gpu(tmp_path):
    sieve, records = tmp_path / "b.sieve", tmp_path / "r.csv"
    assert cli.main(["tune", "--m", "64:256", "--n", "64:128", "--k", "32:64", "--out-sieve", str(sieve),
                     "--out-records", str(records), "--reps", "3"]) == 0
    bank = sk.SieveBank.load(str(sieve))
    rows = sk.read_records_csv(str(records))
    assert len(rows) == 3 * 2 * 2 * 7
    for row in rows:
        if row.is_winner:
            assert row.policy in bank.query(row.size)
    assert cli.main(["verify", "--cases", "35", "--seed", "3"]) == 0
    assert cli.main(["verify", "--cases", "8", "--seed", "3", "--inject-fault"]) == 1


def test_query_tile_bank_with_cost_model_prior(capsys):
    import os

    bank_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "round1", "tilebank5")
    assert cli.main(["query", "--sieve", bank_dir, "--size", "3000x5000x7000", "--repeat", "10"]) == 0
    out = capsys.readouterr().out
    assert "cost-model prior:" in out and "candidates for 3000x5000x7000:" in out
    assert cli.main(["query", "--sieve", bank_dir, "--size", "512x512x16384", "--nearest", "none", "--repeat", "10"]) == 0
    assert "128x128x128/" in capsys.readouterr().out
