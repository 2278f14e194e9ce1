"""The CLI front end against the reference's golden CLI outputs
(proj/tests/test_formats.cpp:67-153, proj/docs/golden/*)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
ARCH = "input 4x4x1; conv 3x3x2 s1 p1; relu; dense 3"


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2007_10868_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=300)


def test_gen_reproduces_golden(tmp_path):
    """test_formats.cpp:67-73: gen --seed 202608 --inputs 3 -> model.json + inputs.csv."""
    m, x = tmp_path / "m.json", tmp_path / "x.csv"
    r = cli("gen", "--seed", "202608", "--arch", ARCH, "--out", str(m), "--inputs-out", str(x), "--inputs", "3")
    assert r.returncode == 0, r.stderr
    assert json.loads(m.read_text()) == json.load(open(os.path.join(GOLDEN, "model.json")))
    assert x.read_text() == open(os.path.join(GOLDEN, "inputs.csv")).read()


def test_usage_errors_exit_2(tmp_path):
    r = cli("verify", "--model", str(tmp_path / "missing.json"), "--inputs", "x", "--epsilon", "0.1")
    assert r.returncode == 2 and r.stderr.startswith("error:")


@pytest.mark.gpu
def test_verify_matches_golden_report():
    """test_formats.cpp:75-85: verify --epsilon 0.03 == report.jsonl modulo runtime_ns."""
    r = cli("verify", "--model", os.path.join(GOLDEN, "model.json"), "--inputs",
            os.path.join(GOLDEN, "inputs.csv"), "--epsilon", "0.03")
    assert r.returncode == 0, r.stderr
    got = [json.loads(l) for l in r.stdout.splitlines()]
    want = [json.loads(l) for l in open(os.path.join(GOLDEN, "report.jsonl"))]
    for g, w in zip(got, want):
        g.pop("runtime_ns"), w.pop("runtime_ns")
        assert g == w
        assert list(g) == list(w)  # field order (test_formats.cpp:114-123)
    assert len(got) == len(want)


@pytest.mark.gpu
def test_bench_matches_golden_csv():
    """test_formats.cpp:125-143: header and early_term_fraction of bench.csv."""
    r = cli("bench", "--model", os.path.join(GOLDEN, "model.json"), "--inputs",
            os.path.join(GOLDEN, "inputs.csv"), "--epsilon", "0.03")
    assert r.returncode == 0, r.stderr
    got = r.stdout.splitlines()
    want = open(os.path.join(GOLDEN, "bench.csv")).read().splitlines()
    assert got[0] == want[0] == "index,runtime_ns,early_term_fraction"
    for g, w in zip(got[1:], want[1:]):
        gi, _, gf = g.split(",")
        wi, _, wf = w.split(",")
        assert (gi, gf) == (wi, wf)


def test_load_inputs_keeps_strings(tmp_path):
    """model_io.cpp:331-353: cells stay strings, trimmed; a trailing comma
    makes no empty cell (std::getline); an inner empty cell throws."""
    from paper_2007_10868_b200.model_io import load_inputs, parse_decimal
    p = tmp_path / "x.csv"
    p.write_text("0.5, 0.25 ,\r\n\n1,x\n")
    assert load_inputs(str(p)) == [["0.5", "0.25"], ["1", "x"]]
    p.write_text("0.5,,1\n")
    with pytest.raises(RuntimeError, match="empty cell on line 1"):
        load_inputs(str(p))
    assert parse_decimal("0.25") == 0.25
    for bad in ("1.", ".5", "1e3", "x"):
        with pytest.raises(ValueError, match="bad decimal: "):
            parse_decimal(bad)


@pytest.mark.gpu
def test_bad_row_is_a_per_input_error(tmp_path):
    """main.cpp:117-184: a malformed or short row yields {index, error}, the
    other rows still verify, and the exit code is 1."""
    rows = open(os.path.join(GOLDEN, "inputs.csv")).read().splitlines()
    x = tmp_path / "x.csv"
    x.write_text("\n".join([rows[0], "0.5,0.5", rows[1].replace(",", ",abc,", 1)]) + "\n")
    r = cli("verify", "--model", os.path.join(GOLDEN, "model.json"), "--inputs", str(x),
            "--epsilon", "0.03")
    assert r.returncode == 1, r.stderr
    got = [json.loads(l) for l in r.stdout.splitlines()]
    assert got[0]["verdict"] == "verified"
    assert got[1] == {"index": 1, "error": "input size mismatch"}
    assert got[2]["index"] == 2 and "error" in got[2]
