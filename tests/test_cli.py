"""CLI (cli.py) mirroring the reference's m/cli.py for the gpu strategy:
argument handling and exit codes on CPU, full runs on the GPU."""

from __future__ import annotations

import json

import pytest

from conftest import hexrows
from paper_1603_06757_b200 import BitMatrix, parse_report, read_matrix_file, write_matrix_file
from paper_1603_06757_b200 import cli


def test_random_roundtrip(tmp_path, capsys):
    out = tmp_path / "g.txt"
    assert cli.main(["random", "--k", "6", "--n", "14", "--seed", "3", "--out", str(out),
                     "--quiet"]) == cli.EXIT_OK
    M = read_matrix_file(str(out))
    assert (M.num_rows, M.num_cols) == (6, 14)
    assert cli.main(["random", "--k", "6", "--n", "14", "--seed", "3"]) == cli.EXIT_OK
    assert "random systematic code k=6 n=14 seed=3" in capsys.readouterr().out


def test_missing_input_and_bad_args(tmp_path):
    assert cli.main(["mindist"]) == cli.EXIT_INVALID
    assert cli.main(["mindist", "--in", str(tmp_path / "nope.txt")]) == cli.EXIT_PARSE
    bad = tmp_path / "bad.txt"
    bad.write_text("01x\n")
    assert cli.main(["mindist", "--in", str(bad)]) == cli.EXIT_PARSE
    ok = tmp_path / "ok.txt"
    write_matrix_file(str(ok), BitMatrix([0b101, 0b011], 3))
    # the reference's CPU strategies are not part of this build
    assert cli.main(["mindist", "--in", str(ok), "--algorithm", "saved"]) == cli.EXIT_INVALID
    # reference-only knobs are accepted
    ns = cli.build_parser().parse_args(["mindist", "--in", "x", "--s", "4", "--threads", "8",
                                        "--budget-mb", "64"])
    assert ns.algorithm == "gpu" and ns.gpus == 1


@pytest.mark.gpu
def test_mindist_golden(goldens, tmp_path, capsys):
    fx = [c for c in goldens["configs"] if c["name"] == "cfg2"][0]
    path = tmp_path / "cfg2.txt"
    write_matrix_file(str(path), BitMatrix(hexrows(fx["rows"]), fx["n"]))
    rep_path = tmp_path / "rep.txt"
    assert cli.main(["mindist", "--in", str(path), "--out", str(rep_path),
                     "--quiet"]) == cli.EXIT_OK
    rep = parse_report(rep_path.read_text())
    assert rep["distance"] == fx["distance"]
    assert rep["bounds_trace"] == [tuple(t) for t in fx["bounds_trace"]]
    assert rep["combinations"] == fx["combinations"]
    capsys.readouterr()
    assert cli.main(["bench", "--in", str(path), "--json", "--quiet"]) == cli.EXIT_OK
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["distance"] == fx["distance"] and line["value"] > 0


@pytest.mark.gpu
def test_max_g_and_resume(goldens, tmp_path):
    fx = [c for c in goldens["configs"] if c["name"] == "cfg2"][0]
    path = tmp_path / "cfg2.txt"
    write_matrix_file(str(path), BitMatrix(hexrows(fx["rows"]), fx["n"]))
    part = tmp_path / "part.txt"
    assert cli.main(["mindist", "--in", str(path), "--out", str(part), "--max-g", "2",
                     "--quiet"]) == cli.EXIT_MAX_G
    assert parse_report(part.read_text())["g_reached"] == 2
    full = tmp_path / "full.txt"
    assert cli.main(["mindist", "--in", str(path), "--resume", str(part), "--out",
                     str(full), "--quiet"]) == cli.EXIT_OK
    assert parse_report(full.read_text())["distance"] == fx["distance"]


@pytest.mark.gpu
def test_brute(goldens, tmp_path, capsys):
    fx = [c for c in goldens["configs"] if c["name"] == "cfg1"][0]
    path = tmp_path / "cfg1.txt"
    write_matrix_file(str(path), BitMatrix(hexrows(fx["rows"]), fx["n"]))
    assert cli.main(["brute", "--in", str(path)]) == cli.EXIT_OK
    assert f"distance={fx['distance']}" in capsys.readouterr().out
    assert cli.main(["brute", "--in", str(path), "--max-k", "10"]) == cli.EXIT_TOO_LARGE
