"""Verify images of a named config (for ncu / sanitizer captures): image 0 as
a warm-up, then images 1..n. usage: python scripts/one_image.py CONFIG [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_10868_b200 as pc  # noqa: E402
from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
arch, eps_s = CONFIGS[name]
net = pc.generate(MODEL_SEED, arch)
v = pc.Verifier(net)
X = pc.random_inputs(INPUT_SEED, n + 1, int(np.prod(net.input_shape)))
first = int(os.environ.get("ONE_IMAGE_FIRST", "0"))  # 1: no warm-up image (targeted ncu skips)
for i, x in enumerate(X):
    if i < first:
        continue
    box = pc.input_box(x, float(eps_s))
    t0 = time.perf_counter()
    r = v.verify_robustness(box, max(v.candidate(x), 0))
    print(i, r.verified, f"{1000 * (time.perf_counter() - t0):.1f} ms", v.last_timing()["launches"], flush=True)
