"""Median single-image latency of a config (one image at a time through
pc_net_test, device-resident boxes): n images after one warm-up image.
usage: python scripts/latency.py CONFIG [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_10868_b200 as pc  # noqa: E402
from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
arch, eps_s = CONFIGS[name]
net = pc.generate(MODEL_SEED, arch)
v = pc.Verifier(net)
X = pc.random_inputs(INPUT_SEED, n + 1, int(np.prod(net.input_shape)))
boxes = [pc.input_box(x, float(eps_s)) for x in X]
labels = [max(v.candidate(x), 0) for x in X]
wall, dev, launches, ok = [], [], [], 0
for i, (b, lab) in enumerate(zip(boxes, labels)):
    t0 = time.perf_counter()
    r = v.verify_robustness(b, lab)
    w = 1000 * (time.perf_counter() - t0)
    if i == 0:
        continue
    t = v.last_timing()
    wall.append(w)
    dev.append(t["total_ms"])
    launches.append(t["launches"])
    ok += bool(r.verified)
print(f"{name} n={n} verified={ok} wall_ms_median={np.median(wall):.3f} device_ms_median={np.median(dev):.3f} "
      f"launches_median={int(np.median(launches))}", flush=True)
