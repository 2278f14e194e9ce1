"""Chain-fold diagnostics over one verified image (pc_scan_stats): scan steps,
links committed by scans, scalar fallbacks. usage: python scripts/scan_stats.py CONFIG"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_10868_b200 as pc  # noqa: E402
from paper_2007_10868_b200 import _lib  # noqa: E402
from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cifar_resnet34"
arch, eps_s = CONFIGS[name]
net = pc.generate(MODEL_SEED, arch)
v = pc.Verifier(net)
x = pc.random_inputs(INPUT_SEED, 1, int(np.prod(net.input_shape)))[0]
box = pc.input_box(x, float(eps_s))
lab = max(v.candidate(x), 0)
v.verify_robustness(box, lab)
out = (ctypes.c_ulonglong * 8)()
_lib.check(_lib.lib.pc_scan_stats(1, out))
v.verify_robustness(box, lab)
_lib.check(_lib.lib.pc_scan_stats(0, out))
steps, links, fails, frameless, ties, huge, grew, shrank = list(out)
print({"config": name, "scan_steps": steps, "scanned_links": links, "fallbacks_after_scan": fails,
       "frameless_scalar": frameless, "ties": ties, "huge_terms": huge, "fail_grew": grew,
       "fail_shrank_or_flipped": shrank, "links_per_step": links / max(steps, 1),
       "fallback_per_link": fails / max(links, 1)})
