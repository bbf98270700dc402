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


def test_construct_script(tmp_path, section6):
    """`construct` builds C3 = extend([234,51]) from a script with the
    paper's polynomials, bit-identical to the reference's matrix; script
    errors map to the reference's exit codes."""
    from conftest import hexrows
    from paper_1603_06757_b200 import cli
    from paper_1603_06757_b200.gf2 import read_matrix_file

    m = section6["m"]
    f2 = "116," + ",".join(str(e) for e in range(115, -1, -1))  # (x^117-1)/(x+1) = all ones
    script = tmp_path / "c3.txt"
    script.write_text("# section 6, C3\n"
                      f"m = {m}\n"
                      f"f1 = {','.join(map(str, section6['f1_exps']))}\n"
                      f"f2 = {f2}\n"
                      f"p = {','.join(map(str, section6['p1_exps']))}\n"
                      "extend\n")
    out = tmp_path / "c3.mat"
    assert cli.main(["construct", "--in", str(script), "--out", str(out), "--quiet"]) == 0
    G = read_matrix_file(str(out))
    fx = [c for c in section6["codes"] if c["name"] == "C3"][0]
    assert (G.num_cols, G.num_rows) == (fx["n"], fx["k"])
    assert list(G.rows) == hexrows(fx["rows"])
    bad = tmp_path / "bad.txt"
    bad.write_text("m = 7\nf1 = 2,1,0\nf2 = 0\np = 0\n")
    assert cli.main(["construct", "--in", str(bad), "--quiet"]) == cli.EXIT_NOT_A_DIVISOR
    bad.write_text("m = 7\nbogus = 1\n")
    assert cli.main(["construct", "--in", str(bad), "--quiet"]) == cli.EXIT_SCRIPT


def test_device_errors_exit_codes(tmp_path):
    """No usable device maps to EXIT_DEVICE (14) -- never a silent CPU run;
    on a GPU box, more stored columns than the kernels hold maps to
    EXIT_TOO_LARGE (11), not EXIT_INVALID."""
    import random

    from paper_1603_06757_b200 import _native

    try:
        have_gpu = _native.device_count() > 0
    except Exception:
        have_gpu = False
    small = tmp_path / "small.txt"
    write_matrix_file(str(small), BitMatrix([0b1011, 0b0110], 4))
    wide = tmp_path / "wide.txt"
    rng = random.Random(5)
    write_matrix_file(str(wide), BitMatrix([rng.getrandbits(290) for _ in range(28)], 290))
    if have_gpu:
        assert cli.main(["mindist", "--in", str(wide), "--quiet"]) == cli.EXIT_TOO_LARGE
    else:
        assert cli.main(["mindist", "--in", str(small), "--quiet"]) == cli.EXIT_DEVICE
        assert cli.main(["brute", "--in", str(small)]) == cli.EXIT_DEVICE
