"""GPU parity directly against the UNMODIFIED reference (oracle/_ref, built from
/root/reference/proj by oracle/build_ref.sh and shipped with the snapshot).

* BASELINE configs (6x100, 9x500, ConvBig) on 8 images each: verdicts, margin
  bit patterns, every padded/raw per-neuron bound, PassStats.
* R2 "gain init" 6x100 at eps 0.012 / 0.013: mixed verdicts.
* The image-batched schedule (pc_net_test_batch, 64 images in one schedule)
  against the reference image by image.
* The residual configs (ResNet-18, the 34-layer headline): the committed
  fixtures tests/golden/ref_<config>_img<i>.json, written by
  scripts/ref_fixtures.py from oracle/_ref (verify_robustness,
  analyzer.hpp:256-276): label, verdict, margin bits, PassStats and a SHA-256
  per layer of the padded and raw bound bit patterns.

Reference calls run on a host thread pool (ctypes releases the GIL), one image
per thread, like the CLI's worker pool (tools/main.cpp:117).
"""
import glob
import hashlib
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
STAT_KEYS = ["rows_total", "rows_terminated_early", "gbc_madds", "gbc_dense_equiv", "dense_madds",
             "checkpoints"]


@pytest.fixture(scope="module")
def pc():
    import paper_2007_10868_b200 as pc
    return pc


def _bits_equal(a, b, what):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, what
    bad = a.view(np.int64) != b.view(np.int64)
    assert not bad.any(), f"{what}: {int(bad.sum())} mismatches, first at {int(np.argmax(bad))}: {a[bad][:3]} vs {b[bad][:3]}"


def _ref_model(ref, net):
    """The reference's own parse of this net (model_to_json -> model_from_json_text)."""
    from paper_2007_10868_b200.model_io import model_to_json_obj
    return ref.from_json(json.dumps(model_to_json_obj(net)))


def _compare(g, r, label, what):
    assert g.verified == r["verified"], what
    _bits_equal(g.margins, r["margins"], f"{what} margins")
    assert g.stats == r["stats"], (what, g.stats, r["stats"])
    if r.get("b_lo") is not None and g.bounds:
        blo = np.concatenate([b[0] for b in g.bounds])
        bhi = np.concatenate([b[1] for b in g.bounds])
        rlo = np.concatenate([b[0] for b in g.raw])
        rhi = np.concatenate([b[1] for b in g.raw])
        _bits_equal(blo, r["b_lo"], f"{what} bounds.lo")
        _bits_equal(bhi, r["b_hi"], f"{what} bounds.hi")
        _bits_equal(rlo, r["r_lo"], f"{what} raw.lo")
        _bits_equal(rhi, r["r_hi"], f"{what} raw.hi")


def _run_vs_ref(pc, ref, net, X, eps, want_bounds=True, labels=None):
    h = _ref_model(ref, net)
    v = pc.Verifier(net)
    if labels is None:
        labels = [v.candidate(x) for x in X]
    ref_labels = [ref.candidate(h, x) for x in X]
    assert labels == ref_labels  # forward_eval + unique_argmax (eval.hpp:39-102)
    with ThreadPoolExecutor(max_workers=min(len(X), os.cpu_count() or 1)) as ex:
        futs = [ex.submit(ref.verify, h, x, eps, True, lab, True, 0, 0, 1, want_bounds)
                for x, lab in zip(X, labels)]
        gpu = []
        for x, lab in zip(X, labels):
            box = pc.input_box(x, eps)
            gpu.append(v.test(box.lo, box.hi, lab, want_bounds=want_bounds))
        refs = [f.result() for f in futs]
    for i, (g, r) in enumerate(zip(gpu, refs)):
        _compare(g, r, labels[i], f"image {i}")
    ref.free(h)
    return gpu, refs


@pytest.mark.parametrize("name", ["mnist_6x100", "mnist_9x500", "cifar_convbig"])
def test_baseline_configs_vs_reference(pc, ref, name):
    """SURVEY.md §8d configs, model seed 7, inputs seed 8, 8 images, eps as a decimal
    string parsed by the reference (double_from_decimal, decimal.cpp:63-76)."""
    from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED
    arch, eps_s = CONFIGS[name]
    net = pc.generate(MODEL_SEED, arch)
    eps = ref.double_from_decimal(eps_s)
    assert eps == float(eps_s)
    X = pc.random_inputs(INPUT_SEED, 8, int(np.prod(net.input_shape)))
    _bits_equal(X, ref.random_inputs(INPUT_SEED, 8, X.shape[1]), "random_inputs")
    gpu, _ = _run_vs_ref(pc, ref, net, X, eps)
    assert all(g.verified for g in gpu)  # R1 init: every image verifies


def _gain_scaled(pc, arch):
    """R2 'gain init': every affine layer's weights x 2^round(log2 sqrt(fan_in)) (exact)."""
    net = pc.generate(7, arch)
    for L in net.layers:
        if L.kind == "dense":
            fan_in = L.weights.shape[1]
            L.weights = L.weights * 2.0 ** round(np.log2(np.sqrt(fan_in)))
    return net


@pytest.mark.parametrize("eps", ["0.012", "0.013"])
def test_gain_scaled_6x100_mixed_verdicts(pc, ref, eps):
    from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED
    net = _gain_scaled(pc, CONFIGS["mnist_6x100"][0])
    X = pc.random_inputs(INPUT_SEED, 12, 784)
    gpu, refs = _run_vs_ref(pc, ref, net, X, float(eps))
    verdicts = [g.verified for g in gpu]
    assert any(verdicts) and not all(verdicts), verdicts  # meaningful verdict parity


def test_image_batched_schedule_vs_reference(pc, ref):
    """pc_net_test_batch with 64 images in ONE image-batched schedule (the bench's
    throughput kernels, k_dense_coef3) == the reference, image by image."""
    from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED
    net = _gain_scaled(pc, CONFIGS["mnist_6x100"][0])  # live rows in every pass
    X = pc.random_inputs(INPUT_SEED + 1, 64, 784)
    v = pc.Verifier(net)
    labels = np.array([max(v.candidate(x), 0) for x in X], dtype=np.int32)
    eps = 0.012
    boxes = [pc.input_box(x, eps) for x in X]
    lo, hi = np.stack([b.lo for b in boxes]), np.stack([b.hi for b in boxes])
    ver, mar, st, _ = v.test_batch(lo, hi, labels, concurrency=1)
    h = _ref_model(ref, net)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        refs = list(ex.map(lambda a: ref.verify(h, a[0], eps, True, int(a[1]), True, 0, 0, 1, False),
                           zip(X, labels)))
    for i, r in enumerate(refs):
        assert bool(ver[i]) == r["verified"], i
        _bits_equal(mar[i], r["margins"], f"image {i} margins")
        assert st[i] == r["stats"], (i, st[i], r["stats"])
    assert 0 < int(np.sum(ver)) < len(X)
    ref.free(h)


def _fixtures():
    return sorted(glob.glob(os.path.join(GOLDEN, "ref_*.json")))


def layer_hashes(arrs, offsets):
    out = []
    for k in range(len(offsets) - 1):
        a, b = offsets[k], offsets[k + 1]
        out.append({n: hashlib.sha256(np.ascontiguousarray(x[a:b]).tobytes()).hexdigest()
                    for n, x in arrs.items()})
    return out


@pytest.mark.parametrize("path", _fixtures(), ids=lambda p: os.path.basename(p)[4:-5])
def test_residual_config_fixture(pc, path):
    """The residual configs against the reference's own results (fixtures made by
    scripts/ref_fixtures.py): bit-identical verdict, margins, PassStats, and
    every layer's padded and raw bounds (SHA-256 of the bit patterns)."""
    fx = json.load(open(path))
    from paper_2007_10868_b200.configs import CONFIGS
    arch, eps_s = CONFIGS[fx["config"]]
    assert arch == fx["arch"] and eps_s == fx["eps"]
    net = pc.generate(fx["model_seed"], arch)
    X = pc.random_inputs(fx["input_seed"], fx["image"] + 1, int(np.prod(net.input_shape)))
    x = X[fx["image"]]
    v = pc.Verifier(net, pc.AnalysisOptions(early_term=fx["early_term"]))
    assert v.candidate(x) == fx["label"]
    box = pc.input_box(x, float(eps_s), fx["clamp01"])
    g = v.test(box.lo, box.hi, fx["label"], want_bounds=True)
    assert g.verified == fx["verified"]
    assert [m.hex() for m in g.margins] == fx["margins_hex"]
    assert g.stats == fx["stats"], (g.stats, fx["stats"])
    arrs = {"b_lo": np.concatenate([b[0] for b in g.bounds]),
            "b_hi": np.concatenate([b[1] for b in g.bounds]),
            "r_lo": np.concatenate([b[0] for b in g.raw]),
            "r_hi": np.concatenate([b[1] for b in g.raw])}
    got = layer_hashes(arrs, v.offsets)
    bad = [k for k, (a, b) in enumerate(zip(got, fx["layer_sha256"])) if a != b]
    assert len(got) == len(fx["layer_sha256"]) and not bad, f"layers with different bounds: {bad}"
    n_last = len(fx["last_layer"]["b_lo"])
    for k, arr in arrs.items():
        assert [float(t).hex() for t in arr[-n_last:]] == fx["last_layer"][k]
