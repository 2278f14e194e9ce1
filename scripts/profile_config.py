"""Per-kernel-class device time per image (PC_PROFILE=1) for a named config."""
import json
import os
import sys
import time

os.environ["PC_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_10868_b200 as pc  # noqa: E402
from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED  # noqa: E402

name = sys.argv[1]
n_img = int(sys.argv[2]) if len(sys.argv) > 2 else 2
et = not (len(sys.argv) > 3 and sys.argv[3] == "noet")
arch, eps_s = CONFIGS[name]
net = pc.generate(MODEL_SEED, arch)
v = pc.Verifier(net, pc.AnalysisOptions(early_term=et))
if os.environ.get("PROFILE_SERIAL"):  # one stream, one pipeline: class times are exclusive
    v.set_serial(True)
X = pc.random_inputs(INPUT_SEED, n_img + 1, int(np.prod(net.input_shape)))
for i, x in enumerate(X):
    lab = v.candidate(x)
    box = pc.input_box(x, float(eps_s))
    t0 = time.perf_counter()
    verdict = v.verify_robustness(box, max(lab, 0))
    wall = (time.perf_counter() - t0) * 1000
    if i == 0:
        continue  # warm-up
    t = v.last_timing()
    prof = v.last_profile()
    win = prof.pop("gbc_window_madds", [0, 0])[1]
    passes = prof.pop("passes", [])
    prof.pop("timeline", None)
    prof.pop("host_arena_alloc", None)
    tot = sum(ms for k, (_, ms) in prof.items() if not k.startswith("gap:"))
    print(json.dumps({"config": name, "image": i, "verified": verdict.verified, "wall_ms": round(wall, 2),
                      "device_ms": round(t["total_ms"], 2), "launches": t["launches"],
                      "stats": verdict.stats,
                      "gbc_nonzero_fraction": (verdict.stats["gbc_madds"] / win) if win else None,
                      "passes": passes,
                      "classes": {k: [c, round(ms, 3), round(100 * ms / max(tot, 1e-9), 1)]
                                  for k, (c, ms) in sorted(prof.items(), key=lambda kv: -kv[1][1]) if c or ms > 0.05}}))
