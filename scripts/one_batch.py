"""One image-batched schedule (64 images, one worker context) of the 9x500 bench
workload — a fixed unit of work for ncu metric totals per image."""
import sys
import numpy as np
import paper_2007_10868_b200 as pc
from paper_2007_10868_b200.configs import CONFIGS, INPUT_SEED, MODEL_SEED

name = sys.argv[1] if len(sys.argv) > 1 else "mnist_9x500"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
arch, eps = CONFIGS[name]
net = pc.generate(MODEL_SEED, arch)
v = pc.Verifier(net)
X = pc.random_inputs(INPUT_SEED, n, int(np.prod(net.input_shape)))
boxes = [pc.input_box(x, float(eps)) for x in X]
labels = np.array([max(v.candidate(x), 0) for x in X], dtype=np.int32)
lo, hi = np.stack([b.lo for b in boxes]), np.stack([b.hi for b in boxes])
ver, _, _, ms = v.test_batch(lo, hi, labels, concurrency=1)
print(f"{name}: {n} images, {int(ver.sum())} verified, {ms:.3f} ms")
