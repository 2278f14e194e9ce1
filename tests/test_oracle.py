"""CPU-only: pin the oracle. The plain-C restatement (oracle/polycert_port.c)
must equal the UNMODIFIED reference (oracle/_ref) bit-for-bit, and both must
reproduce the reference's golden vectors (proj/docs/golden, copied to
tests/golden). Also pins the generator port (paper_2007_10868_b200/gen.py)."""
import json
import os

import numpy as np
import pytest

from cases import BACKSUB_ARCHS, EXTRA_ARCHS

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden_inputs():
    return np.array([[float(t) for t in l.split(",")]
                     for l in open(os.path.join(GOLDEN, "inputs.csv")).read().split()])


def test_port_reproduces_golden_report(port):
    from paper_2007_10868_b200 import generate
    net = generate(202608, "input 4x4x1; conv 3x3x2 s1 p1; relu; dense 3")
    for line, x in zip(open(os.path.join(GOLDEN, "report.jsonl")), golden_inputs()):
        rec = json.loads(line)
        lo, hi = port.input_box(x, 0.03)
        r = port.analyze(net.layers, lo, hi, label=rec["candidate"])
        assert r["margins"].tolist() == [m["lower"] for m in rec["margins"]]
        assert r["verified"] == (rec["verdict"] == "verified")
        assert r["stats"]["rows_terminated_early"] == rec["rows_terminated"]


def test_bench_csv_fraction(port):
    """docs/golden/bench.csv early_term_fraction = rows_terminated / rows_total."""
    from paper_2007_10868_b200 import generate
    net = generate(202608, "input 4x4x1; conv 3x3x2 s1 p1; relu; dense 3")
    rows = [l.split(",") for l in open(os.path.join(GOLDEN, "bench.csv")).read().split()[1:]]
    for (idx, _, frac), x in zip(rows, golden_inputs()):
        lo, hi = port.input_box(x, 0.03)
        s = port.analyze(net.layers, lo, hi, label=1)["stats"]
        assert "%.6f" % (s["rows_terminated_early"] / s["rows_total"]) == frac


def test_generator_matches_golden_model():
    """test_formats.cpp:67-73: gen --seed 202608 reproduces docs/golden/model.json and inputs.csv."""
    from paper_2007_10868_b200 import generate, random_inputs
    from paper_2007_10868_b200.model_io import model_to_json_obj
    net = generate(202608, "input 4x4x1; conv 3x3x2 s1 p1; relu; dense 3")
    assert model_to_json_obj(net) == json.load(open(os.path.join(GOLDEN, "model.json")))
    assert np.array_equal(random_inputs(202609, 3, 16), golden_inputs())


@pytest.mark.parametrize("arch", BACKSUB_ARCHS + EXTRA_ARCHS)
def test_generator_matches_reference(ref, arch):
    from paper_2007_10868_b200 import generate
    net = generate(77, arch)
    h = ref.generate(77, arch)
    try:
        rl = ref.layers(h)
        assert len(rl) == len(net.layers)
        for a, b in zip(net.layers, rl):
            assert a.kind == b.kind and tuple(a.out_shape) == tuple(b.out_shape)
            assert list(a.preds) == list(b.preds)
            if a.weights is not None:
                assert np.array_equal(np.asarray(a.weights).reshape(-1), b.weights.reshape(-1))
                assert np.array_equal(a.bias, b.bias)
    finally:
        ref.free(h)


@pytest.mark.parametrize("arch", BACKSUB_ARCHS + EXTRA_ARCHS)
@pytest.mark.parametrize("early_term", [True, False])
def test_port_equals_reference(ref, port, arch, early_term):
    from paper_2007_10868_b200 import generate, random_inputs
    net = generate(900, arch)
    h = ref.generate(900, arch)
    try:
        X = random_inputs(901, 2, int(np.prod(net.input_shape)))
        for x, eps in zip(X, [1.0 / 16, 0.25]):
            lab = ref.candidate(h, x)
            lab = lab if lab >= 0 else 0
            r = ref.verify(h, x, eps, label=lab, early_term=early_term)
            lo, hi = port.input_box(x, eps)
            p = port.analyze(net.layers, lo, hi, label=lab, early_term=early_term)
            for k in ("b_lo", "b_hi", "r_lo", "r_hi", "margins"):
                assert np.array_equal(r[k].view(np.int64), p[k].view(np.int64)), k
            assert r["stats"] == p["stats"] and r["verified"] == p["verified"]
    finally:
        ref.free(h)


def test_port_chunk_invariance(port):
    from paper_2007_10868_b200 import generate
    net = generate(40, BACKSUB_ARCHS[2])
    x = np.full(32, 0.5)
    lo, hi = port.input_box(x, 0.06)
    a = port.analyze(net.layers, lo, hi, label=0, chunk_rows=1)
    b = port.analyze(net.layers, lo, hi, label=0, chunk_rows=7)
    c = port.analyze(net.layers, lo, hi, label=0, memory_budget=1 << 16)
    for k in ("b_lo", "b_hi", "margins"):
        assert np.array_equal(a[k], b[k]) and np.array_equal(a[k], c[k])


def test_scalar_kats(port):
    """test_interval.cpp:121-149 exact-op non-widening KATs."""
    f = lambda op, a, b: float(port.scalar_ops(op, np.array([a]), np.array([b]))[0])
    assert f(0, 0.5, 0.25) == 0.75 and f(1, 0.5, 0.25) == 0.75
    assert f(0, 1.0, -1.0) == 0.0
    assert f(2, 1.5, 2.5) == 3.75 and f(3, -1.5, 2.5) == -3.75
    assert f(4, 3.0, 2.0) == 1.5 and f(5, 3.0, -2.0) == -1.5
    assert f(4, 1.0, 3.0) < f(5, 1.0, 3.0)
    assert f(2, 0.1, 0.1) < f(3, 0.1, 0.1)
    assert f(0, 1.0, 2.0 ** -80) < 1.0 < f(1, 1.0, 2.0 ** -80)
    assert f(2, 2.0 ** -400, 2.0 ** -200) < 2.0 ** -600 < f(3, 2.0 ** -400, 2.0 ** -200)
    assert f(0, np.inf, 1.0) == np.finfo(np.float64).max  # step_down(inf)
