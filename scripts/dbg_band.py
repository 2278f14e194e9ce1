import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
from test_gpu_numeric import operands, gpu_ops
from oracle.pyoracle import Port
port = Port()
a, b = operands()
fin = np.isfinite(a) & np.isfinite(b); a, b = a[fin], b[fin]
with np.errstate(all="ignore"):
    p = np.abs(a * b)
pm = (p == 0) | ((p >= 2.0 ** -499) & (p <= 2.0 ** 999))
for op, ref in ((11, 2), (12, 3)):
    g, r = gpu_ops(op, a[pm], b[pm]), port.scalar_ops(ref, a[pm], b[pm])
    bad = np.flatnonzero(g != r)
    print(op, len(bad), [(a[pm][k].hex(), b[pm][k].hex(), g[k].hex(), r[k].hex()) for k in bad[:5]])
