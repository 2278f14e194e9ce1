"""Soundness against the exact-rational engine and candidate parity.

* Every GPU bound (padded per-neuron bounds) and margin must CONTAIN the
  reference's exact-rational result for the same network and box
  (ExactRational analyze + run_margin_pass, analyzer.hpp:198-276 over mpq,
  exposed by oracle/ref_driver.cpp ref_rational_contains), and a GPU
  "verified" must imply the exact verdict. Radii are dyadic (exact in
  double) so the widened and the exact input boxes are the same set.
  Nets stay small (the reference's oracle is meant for <= ~4000 neurons,
  oracle.hpp:85-86).
* The GPU candidate label (pc_net_candidate) equals forward_eval +
  unique_argmax of the reference (eval.hpp:39-102, tools/main.cpp:86-100) on
  the BASELINE configs' inputs.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SOUND_ARCHS = [
    "input 6x6x1; dense 20; relu; dense 20; relu; dense 5",
    "input 8x8x1; conv 3x3x4 s1 p1; relu; conv 4x4x4 s2 p1; relu; dense 5",
    "input 6x6x2; conv 3x3x4 s1 p1; relu; block(conv 3x3x4 s1 p1; relu; conv 3x3x4 s1 p1 | skip); relu; dense 4",
    "input 8x8x2; conv 3x3x4 s1 p1; relu; block(conv 4x4x6 s2 p1; relu; conv 3x3x6 s1 p1 | conv 2x2x6 s2 p0); relu; dense 3",
    "input 28x28x1; dense 100; relu; dense 100; relu; dense 10",
]


@pytest.fixture(scope="module")
def pc():
    import paper_2007_10868_b200 as pc
    return pc


def _ref_model(ref, net):
    from paper_2007_10868_b200.model_io import model_to_json_obj
    return ref.from_json(json.dumps(model_to_json_obj(net)))


def _gain(net):
    for L in net.layers:
        if L.kind in ("dense", "conv"):
            fan_in = L.weights.shape[1] if L.kind == "dense" else L.fw * L.fh * L.cin
            L.weights = L.weights * 2.0 ** round(np.log2(np.sqrt(fan_in)))
    return net


@pytest.mark.parametrize("gain", [False, True], ids=["R1", "R2"])
@pytest.mark.parametrize("arch", SOUND_ARCHS)
def test_bounds_contain_exact_rational(pc, ref, arch, gain):
    if gain and arch.startswith("input 28x28"):
        pytest.skip("exact rationals of the gain-scaled 784-100-100 net take minutes per image")
    net = pc.generate(11, arch)
    if gain:
        net = _gain(net)
    h = _ref_model(ref, net)
    v = pc.Verifier(net)
    X = pc.random_inputs(12, 3, int(np.prod(net.input_shape)))
    for num, den in [(1, 32), (3, 256)]:
        for x in X:
            lab = max(v.candidate(x), 0)
            box = pc.input_box(x, num / den, True)
            g = v.test(box.lo, box.hi, lab, want_bounds=True)
            blo = np.concatenate([b[0] for b in g.bounds])
            bhi = np.concatenate([b[1] for b in g.bounds])
            bad, exact_verified = ref.rational_contains(h, x, num, den, True, lab, blo, bhi, g.margins)
            assert bad == 0, f"{bad} widened values do not contain the exact ones"
            assert not g.verified or exact_verified  # widened verdict is sound
    ref.free(h)


@pytest.mark.parametrize("name", ["mnist_6x100", "mnist_9x500", "cifar_convbig"])
def test_candidate_matches_reference(pc, ref, name):
    from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED
    arch, _ = CONFIGS[name]
    net = pc.generate(MODEL_SEED, arch)
    h = _ref_model(ref, net)
    X = pc.random_inputs(INPUT_SEED, 100, int(np.prod(net.input_shape)))
    v = pc.Verifier(net)
    assert [v.candidate(x) for x in X] == [ref.candidate(h, x) for x in X]
    ref.free(h)
