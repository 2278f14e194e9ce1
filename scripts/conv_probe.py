"""Conv-kernel work and time on one image of a config, walks serialised
(pc_net_set_serial: per-launch CUDA events time each kernel alone):
executed interval madds (live cells) vs the reference's gbc_madds, conv
kernel ms, whole-verification ms. usage: python scripts/conv_probe.py CONFIG"""
import json
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
X = pc.random_inputs(INPUT_SEED, 2, int(np.prod(net.input_shape)))
modes = (True,) if os.environ.get("PROBE_SERIAL_ONLY") else (False,) if os.environ.get("PROBE_CONC_ONLY") else (False, True)
for serial in modes:
    v.set_serial(serial)
    for i, x in enumerate(X):
        box = pc.input_box(x, float(eps_s))
        r = v.verify_robustness(box, max(v.candidate(x), 0))
        t = v.last_timing()
        k = v.last_kernel_timing("conv")
        print(json.dumps({"config": name, "image": i, "serial": serial, "verified": r.verified,
                          "total_ms": round(t["total_ms"], 2), "conv_ms": round(k["ms"], 2),
                          "conv_launches": k["launches"], "executed_madds": k["executed_madds"],
                          "ref_gbc_madds": r.stats["gbc_madds"],
                          "executed_per_s": k["executed_madds"] / (k["ms"] / 1e3) if k["ms"] else None}),
              flush=True)
