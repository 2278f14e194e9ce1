"""GPU parity: the CUDA engine (through the C-ABI) against the CPU oracle on
the same seeded inputs — bounds (padded and raw twins), margins, verdicts and
PassStats must be bit-identical (== on every double, and the same bit
pattern). Reference behaviour pinned: proj/tests/test_backsub.cpp,
test_analyzer.cpp, test_formats.cpp."""
import json
import os

import numpy as np
import pytest

from cases import BACKSUB_ARCHS, EXTRA_ARCHS

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def pc():
    import paper_2007_10868_b200 as pc
    return pc


def _flat(bounds):
    return np.concatenate([b[0] for b in bounds]), np.concatenate([b[1] for b in bounds])


def check_same(got, ref, what):
    assert got.shape == ref.shape, what
    eq = got == ref
    assert eq.all(), f"{what}: {int((~eq).sum())} mismatches, first at {int(np.argmin(eq))}: {got[~eq][:3]} vs {ref[~eq][:3]}"
    # bit patterns too (the reference never produces -0.0 where we produce +0.0)
    assert np.array_equal(got.view(np.int64), ref.view(np.int64)), f"{what}: signed-zero difference"


def run_case(pc, port, net, center, eps, label=None, early_term=True, chunk_rows=0, clamp=True):
    v = pc.Verifier(net, pc.AnalysisOptions(early_term=early_term, chunk_rows=chunk_rows))
    box = pc.input_box(center, eps, clamp)
    lo, hi = port.input_box(center, eps, clamp)
    check_same(box.lo, lo, "input_box lo")
    check_same(box.hi, hi, "input_box hi")
    if label is None:
        label = int(np.argmax(np.random.default_rng(0).random(net.output_size)))
    g = v.test(box.lo, box.hi, label, want_bounds=True)
    r = port.analyze(net.layers, lo, hi, label=label, early_term=early_term, chunk_rows=chunk_rows)
    blo, bhi = _flat(g.bounds)
    rlo, rhi = _flat(g.raw)
    check_same(blo, r["b_lo"], "bounds.lo")
    check_same(bhi, r["b_hi"], "bounds.hi")
    check_same(rlo, r["r_lo"], "raw.lo")
    check_same(rhi, r["r_hi"], "raw.hi")
    check_same(g.margins, r["margins"], "margins")
    assert g.verified == r["verified"]
    assert g.stats == r["stats"], (g.stats, r["stats"])
    return g, r


def test_golden_report(pc, port):
    """proj/docs/golden/report.jsonl: margins and rows_terminated, eps 0.03."""
    net = pc.generate(202608, "input 4x4x1; conv 3x3x2 s1 p1; relu; dense 3")
    X = np.array([[float(t) for t in l.split(",")] for l in open(os.path.join(GOLDEN, "inputs.csv")).read().split()])
    v = pc.Verifier(net)
    for line, x in zip(open(os.path.join(GOLDEN, "report.jsonl")), X):
        rec = json.loads(line)
        box = pc.input_box(x, 0.03, True)
        verdict = v.verify_robustness(box, rec["candidate"])
        assert [m for _, m in verdict.margins] == [m["lower"] for m in rec["margins"]]
        assert verdict.verified == (rec["verdict"] == "verified")
        assert verdict.stats["rows_terminated_early"] == rec["rows_terminated"]


def test_identity_margins(pc):
    """test_analyzer.cpp:61-76: widened identity net, margins ~0.4 / ~-0.2."""
    L = pc.Layer
    net = pc.Network([L("input", [], (1, 1, 2)),
                      L("dense", [0], weights=np.array([[1.0, 0.0], [0.0, 1.0]]), bias=np.zeros(2))])
    net.validate()
    v = pc.Verifier(net)
    v1 = v.verify_robustness(pc.input_box([0.7, 0.1], 0.1, True), 0)
    assert v1.verified and abs(v1.margins[0][1] - 0.4) <= 1e-12 * 0.4
    v2 = v.verify_robustness(pc.input_box([0.7, 0.1], 0.4, True), 0)
    assert not v2.verified and abs(v2.margins[0][1] + 0.2) <= 1e-12 * 0.2


@pytest.mark.parametrize("arch", BACKSUB_ARCHS + EXTRA_ARCHS)
@pytest.mark.parametrize("seed", [900, 41])
def test_random_nets(pc, port, arch, seed):
    net = pc.generate(seed, arch)
    X = pc.random_inputs(seed + 1, 2, int(np.prod(net.input_shape)))
    for i, eps in enumerate([1.0 / 16, 0.25]):
        run_case(pc, port, net, X[i], eps, label=i % net.output_size)


@pytest.mark.parametrize("arch", BACKSUB_ARCHS[1:3] + EXTRA_ARCHS[2:4])
def test_early_term_and_chunking(pc, port, arch):
    """Early termination and chunk size never change results (test_backsub.cpp:74-157)."""
    net = pc.generate(500, arch)
    x = np.full(int(np.prod(net.input_shape)), 0.5)
    g1, _ = run_case(pc, port, net, x, 0.06, label=0, early_term=True)
    g2, _ = run_case(pc, port, net, x, 0.06, label=0, early_term=False)
    g3, _ = run_case(pc, port, net, x, 0.06, label=0, early_term=True, chunk_rows=1)
    for a, b in zip(g1.bounds, g2.bounds):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for a, b in zip(g1.bounds, g3.bounds):
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert g2.stats["rows_terminated_early"] == 0


def test_gain_scaled_mlp(pc, port):
    """R2 'gain init': He-scaled dyadic weights, mixed verdicts, live rows."""
    net = pc.generate(7, "input 28x28x1; dense 100; relu; dense 100; relu; dense 100; relu; dense 10")
    for L in net.layers:
        if L.kind == "dense":
            fan_in = L.weights.shape[1]
            L.weights = L.weights * 2.0 ** round(np.log2(np.sqrt(fan_in)))
    X = pc.random_inputs(8, 2, 784)
    for x in X:
        run_case(pc, port, net, x, 0.012, label=0)


@pytest.mark.parametrize("width", [20, 120])
def test_out_of_band_magnitudes(pc, port, width):
    """Layers scaled by 2^-560 / 2^+560: products leave [2^-499, 2^999], so the
    forward and back-substitution kernels must take their checked paths (the
    reference's 2^-500 residual floor, subnormal sums) and stay bit-exact."""
    net = pc.generate(31, f"input 4x4x1; dense {width}; relu; dense {width}; relu; dense {width}; relu; dense 10")
    scales = iter([1.0, 2.0 ** -560, 2.0 ** 560, 1.0])
    for L in net.layers:
        if L.kind == "dense":
            f = next(scales)
            L.weights = L.weights * f
            L.bias = L.bias * f
    X = pc.random_inputs(32, 2, 16)
    for x in X:
        run_case(pc, port, net, x, 0.05, label=0)


@pytest.mark.parametrize("width", [20, 120])
def test_signed_zero_parameters(pc, port, width):
    """-0 biases (an accumulator that starts at -0 must see every exact-zero
    term, as the reference adds them) and +-0 weights next to stably-negative
    inputs: the skipped-term shortcuts of the dense kernels stay exact."""
    net = pc.generate(21, f"input 4x4x1; dense {width}; relu; dense {width}; relu; dense {width}; relu; dense 10")
    for k, L in enumerate(net.layers):
        if L.kind == "dense":
            L.bias = L.bias.copy()
            L.bias[::3] = -0.0
            L.weights = L.weights.copy()
            L.weights[:, 1::5] = 0.0
            L.weights[:, 3::7] = -0.0
    X = pc.random_inputs(22, 2, 16)
    for x in X:
        run_case(pc, port, net, x, 0.05, label=0)
    v = pc.Verifier(net)
    X = pc.random_inputs(23, 9, 16)
    boxes = [pc.input_box(x, 0.05) for x in X]
    lo, hi = np.stack([b.lo for b in boxes]), np.stack([b.hi for b in boxes])
    labels = np.zeros(len(X), dtype=np.int32)
    ver, mar, st, _ = v.test_batch(lo, hi, labels, concurrency=1)
    for i in range(len(X)):
        r = v.test(lo[i], hi[i], 0)
        assert np.array_equal(r.margins.view(np.int64), mar[i].view(np.int64))
        assert bool(ver[i]) == r.verified and st[i] == r.stats


@pytest.mark.parametrize("name,n_img", [("mnist_6x100", 3), ("mnist_9x500", 1), ("cifar_convbig", 1)])
def test_baseline_configs(pc, port, name, n_img):
    """BASELINE.json configs: generator weights seed 7, inputs seed 8,
    label = candidate of the concrete forward pass; verdicts, margins, bounds, stats."""
    from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED
    arch, eps_s = CONFIGS[name]
    net = pc.generate(MODEL_SEED, arch)
    X = pc.random_inputs(INPUT_SEED, n_img, int(np.prod(net.input_shape)))
    v = pc.Verifier(net)
    for x in X:
        lab = v.candidate(x)
        assert lab >= 0
        run_case(pc, port, net, x, float(eps_s), label=lab)


@pytest.mark.parametrize("arch", [EXTRA_ARCHS[3], EXTRA_ARCHS[8], BACKSUB_ARCHS[1], EXTRA_ARCHS[9]])
@pytest.mark.parametrize("concurrency", [1, 5, 12])
def test_batch_matches_sequential(pc, arch, concurrency):
    _batch_vs_sequential(pc, arch, concurrency, 12)


@pytest.mark.parametrize("arch", [EXTRA_ARCHS[8], EXTRA_ARCHS[1]])
def test_large_image_batch(pc, arch):
    """One schedule over 40 images (> 128 margin rows, more rows than one block)."""
    _batch_vs_sequential(pc, arch, 1, 40)


def _batch_vs_sequential(pc, arch, concurrency, n_img):
    """pc_net_test_batch == one-at-a-time pc_net_test, bit for bit (margins,
    verdicts, PassStats). 12 images over `concurrency` workers: image-batched
    schedules of 12 and 3 images per walk, and one image per walk."""
    net = pc.generate(11, arch)
    v = pc.Verifier(net)
    X = pc.random_inputs(12, n_img, int(np.prod(net.input_shape)))
    boxes = [pc.input_box(x, 0.05) for x in X]
    labels = np.array([max(v.candidate(x), 0) for x in X], dtype=np.int32)
    lo = np.stack([b.lo for b in boxes])
    hi = np.stack([b.hi for b in boxes])
    ver, mar, st, ms = v.test_batch(lo, hi, labels, concurrency=concurrency)
    assert ms > 0
    for i in range(len(X)):
        r = v.test(lo[i], hi[i], int(labels[i]))
        assert np.array_equal(r.margins.view(np.int64), mar[i].view(np.int64))
        assert bool(ver[i]) == r.verified and st[i] == r.stats


def test_batch_device_inputs_match_host(pc):
    """pc_net_test_batch with device-resident boxes == with host boxes (bench's value leg)."""
    import torch
    net = pc.generate(11, EXTRA_ARCHS[8])
    v = pc.Verifier(net)
    X = pc.random_inputs(13, 24, int(np.prod(net.input_shape)))
    boxes = [pc.input_box(x, 0.05) for x in X]
    labels = np.array([max(v.candidate(x), 0) for x in X], dtype=np.int32)
    lo = np.stack([b.lo for b in boxes])
    hi = np.stack([b.hi for b in boxes])
    vh, mh, sh, _ = v.test_batch(lo, hi, labels, concurrency=3)
    dlo, dhi = torch.from_numpy(lo).cuda(), torch.from_numpy(hi).cuda()
    torch.cuda.synchronize()
    vd, md_, sd, _ = v.test_batch(dlo.data_ptr(), dhi.data_ptr(), labels, 3, device_inputs=True)
    assert np.array_equal(mh.view(np.int64), md_.view(np.int64))
    assert np.array_equal(vh, vd) and sh == sd
