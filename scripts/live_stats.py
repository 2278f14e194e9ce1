"""Liveness structure of the ReLU layers of one verified image (which conv
outputs k_gbc_live computes): per ReLU layer, the fraction of live cells,
of channels live at any position, and the spread of live channels per
position. usage: python scripts/live_stats.py CONFIG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_10868_b200 as pc  # noqa: E402
from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cifar_resnet34"
arch, eps_s = CONFIGS[name]
net = pc.generate(MODEL_SEED, arch)
v = pc.Verifier(net)
x = pc.random_inputs(INPUT_SEED, 1, int(np.prod(net.input_shape)))[0]
box = pc.input_box(x, float(eps_s))
r = v.test(box.lo, box.hi, max(v.candidate(x), 0), want_bounds=True)
for k, L in enumerate(net.layers):
    if L.kind != "relu":
        continue
    p = L.preds[0]
    lo, hi = r.bounds[p]
    rlo, rhi = r.raw[p]
    w, h, c = net.layers[p].out_shape
    dead = (lo < 0) & ~(hi > 0) & ~(rhi > 0)
    live = ~dead.reshape(h * w, c)
    nl = live.sum(1)
    print(f"relu {k:3d} grid {w}x{h}x{c}: live {live.mean():.3f}, channels live anywhere "
          f"{live.any(0).mean():.3f}, live everywhere {live.all(0).mean():.3f}, "
          f"nl/pos min {nl.min()} p25 {np.percentile(nl, 25):.0f} med {np.median(nl):.0f} max {nl.max()}, "
          f"unstable {int(((lo < 0) & (hi > 0)).sum())}")
