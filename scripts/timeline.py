"""Where the time of one verification goes, from the PC_PROFILE timeline
(one walk pipeline, its two streams): busy time of each kernel class, of the
coefficient stream (s), the constants stream (s2), the exact checkpoint
stream (s3) and the prediction stream (s4), the overlap of s and s2 and the
time neither runs (host round trips, launch gaps).
usage: PC_PIPES=1 python scripts/timeline.py CONFIG"""
import json
import os
import sys

os.environ["PC_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2007_10868_b200 as pc  # noqa: E402
from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED  # noqa: E402

NAMES = None


def union(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        tot += cur[1] - cur[0]
    return tot


def intersect(a_iv, b_iv, grid=0.005):
    # busy-both time on a fine grid (ms)
    end = max([b for _, b in a_iv + b_iv] + [0])
    n = int(end / grid) + 2
    A = np.zeros(n, bool)
    B = np.zeros(n, bool)
    for s, e in a_iv:
        A[int(s / grid):int(e / grid) + 1] = True
    for s, e in b_iv:
        B[int(s / grid):int(e / grid) + 1] = True
    return float((A & B).sum() * grid), float((~A & ~B).sum() * grid)


name = sys.argv[1] if len(sys.argv) > 1 else "cifar_resnet34"
arch, eps_s = CONFIGS[name]
net = pc.generate(MODEL_SEED, arch)
v = pc.Verifier(net)
X = pc.random_inputs(INPUT_SEED, 2, int(np.prod(net.input_shape)))
for i, x in enumerate(X):
    v.verify_robustness(pc.input_box(x, float(eps_s)), max(v.candidate(x), 0))
prof = v.last_profile()
t = v.last_timing()
tl = prof["timeline"]
classes = [k for k in prof if not k.startswith("gap:") and k not in ("timeline", "passes", "gbc_window_madds", "host_arena_alloc")]
s0 = [(a, b) for c, st, a, b in tl if st == 0]
s1 = [(a, b) for c, st, a, b in tl if st == 1]
s3 = [(a, b) for c, st, a, b in tl if st == 2]
s4 = [(a, b) for c, st, a, b in tl if st == 3]
both, idle = intersect(s0, s1)
out = {"config": name, "total_ms": t["total_ms"], "s_busy_ms": union(s0), "s2_busy_ms": union(s1),
       "s3_busy_ms": union(s3), "s4_busy_ms": union(s4),
       "both_busy_ms": both, "neither_busy_ms": idle, "s_idle_ms": t["total_ms"] - union(s0),
       "class_busy_ms": {}}
for ci, cname in enumerate(classes):
    iv = [(a, b) for c, st, a, b in tl if c == ci]
    if iv:
        out["class_busy_ms"][cname] = round(union(iv), 2)
# per pass: the seed launch opens each pass (on s)
seed_cls = classes.index("seed") if "seed" in classes else -1
starts = sorted(a for c, st, a, b in tl if c == seed_cls)
per = []
for k, t0 in enumerate(starts):
    t1 = starts[k + 1] if k + 1 < len(starts) else max(b for _, _, _, b in tl)
    seg = [(c, st, max(a, t0), min(b, t1)) for c, st, a, b in tl if b > t0 and a < t1]
    busy = [round(union([(a, b) for c, st, a, b in seg if st == j]), 2) for j in range(4)]
    per.append({"ms": round(t1 - t0, 2), "s": busy[0], "s2": busy[1], "s3": busy[2], "s4": busy[3]})
out["passes"] = per
print(json.dumps(out))
