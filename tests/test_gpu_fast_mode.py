"""The fast numeric mode (pc_options.numeric_mode = 1): the conv
coefficients, constant chains and concretisations of long rows use native
directed rounding (RD / RU FMAs and adds) instead of the reference's
round-to-nearest-then-step rule. It is sound but not bit-identical, so its
parity is reported separately from the bit-exact mode:

* soundness: every bound and margin contains the exact-rational result of the
  reference's rational engine (oracle.hpp / ExactRational analyze), and a
  fast-mode "verified" implies the exact verdict;
* verdict parity and closeness on the residual configs' reference fixtures:
  the same verdict as the unmodified reference, margins within a relative
  1e-5 (the tolerance BASELINE.json's north star states for floating point).
"""
import glob
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

# >= 32 channels and >= 256-cell rows, so the fast conv kernel and the fast
# long-row chains run (smaller layers take the exact kernels, also sound)
FAST_ARCHS = [
    "input 6x6x2; conv 3x3x32 s1 p1; relu; conv 3x3x32 s1 p1; relu; dense 4",
    "input 6x6x1; conv 3x3x32 s1 p1; relu; block(conv 3x3x32 s1 p1; relu; conv 3x3x32 s1 p1 | skip); relu; dense 3",
    "input 8x8x1; conv 3x3x32 s1 p1; relu; block(conv 4x4x32 s2 p1; relu; conv 3x3x32 s1 p1 | conv 2x2x32 s2 p0); relu; dense 3",
]


@pytest.fixture(scope="module")
def pc():
    import paper_2007_10868_b200 as pc
    return pc


def _ref_model(ref, net):
    from paper_2007_10868_b200.model_io import model_to_json_obj
    return ref.from_json(json.dumps(model_to_json_obj(net)))


@pytest.mark.parametrize("arch", FAST_ARCHS)
def test_fast_mode_contains_exact_rational(pc, ref, arch):
    net = pc.generate(31, arch)
    h = _ref_model(ref, net)
    v = pc.Verifier(net, pc.AnalysisOptions(numeric_mode=1, early_term=False))
    X = pc.random_inputs(32, 1, int(np.prod(net.input_shape)))  # exact rationals: ~5-30 s per box
    for num, den in [(1, 64), (1, 16)]:
        for x in X:
            lab = max(v.candidate(x), 0)
            box = pc.input_box(x, num / den, True)
            g = v.test(box.lo, box.hi, lab, want_bounds=True)
            blo = np.concatenate([b[0] for b in g.bounds])
            bhi = np.concatenate([b[1] for b in g.bounds])
            bad, exact_verified = ref.rational_contains(h, x, num, den, True, lab, blo, bhi, g.margins)
            assert bad == 0, f"{bad} fast-mode values do not contain the exact ones"
            assert not g.verified or exact_verified
    ref.free(h)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "ref_cifar_resnet*_img*.json"))),
                         ids=lambda p: os.path.basename(p)[4:-5])
def test_fast_mode_residual_verdicts(pc, path):
    fx = json.load(open(path))
    from paper_2007_10868_b200.configs import CONFIGS
    arch, eps_s = CONFIGS[fx["config"]]
    net = pc.generate(fx["model_seed"], arch)
    x = pc.random_inputs(fx["input_seed"], fx["image"] + 1, int(np.prod(net.input_shape)))[fx["image"]]
    v = pc.Verifier(net, pc.AnalysisOptions(numeric_mode=1, early_term=fx["early_term"]))
    box = pc.input_box(x, float(eps_s), fx["clamp01"])
    g = v.test(box.lo, box.hi, fx["label"])
    ref = np.array([float.fromhex(m) for m in fx["margins_hex"]])
    assert g.verified == fx["verified"]
    rel = np.abs(g.margins - ref) / np.maximum(1.0, np.abs(ref))
    assert rel.max() <= 1e-5, rel.max()
