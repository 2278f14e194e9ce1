"""ctypes wrappers for the two CPU oracles. TEST INFRASTRUCTURE ONLY.

* ``Port``  — oracle/build/libpolycert_port.so, the plain-C restatement of the
  reference's widened engine (oracle/polycert_port.c). Always buildable
  (gcc only); travels to the GPU box.
* ``Ref``   — oracle/_ref/libpolycert_ref.so, the UNMODIFIED reference compiled
  from /root/reference by oracle/build_ref.sh (git-ignored; built here and
  shipped with the gpurun snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker or the CPU baseline.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libpolycert_port.so")
REF_SO = os.path.join(HERE, "_ref", "libpolycert_ref.so")
KIND = {"input": 0, "dense": 1, "conv": 2, "relu": 3, "residual_join": 4}
KIND_NAME = {v: k for k, v in KIND.items()}

vp, ci, ll, cd = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double


def _p(a):
    return a.ctypes.data_as(vp) if a is not None else None


def build_port():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return PORT_SO


class Port:
    """The plain-C restatement (oracle/polycert_port.c)."""

    def __init__(self):
        if not os.path.exists(PORT_SO):
            build_port()
        self.lib = ctypes.CDLL(PORT_SO)
        self.lib.port_analyze.restype = ci
        self.lib.port_input_box.restype = ci

    def input_box(self, center, eps, clamp01=True):
        c = np.ascontiguousarray(center, dtype=np.float64)
        lo, hi = np.empty_like(c), np.empty_like(c)
        rc = self.lib.port_input_box(_p(c), ci(len(c)), cd(eps), ci(int(clamp01)), _p(lo), _p(hi))
        if rc:
            raise ValueError("input_box: clamped center outside [0,1]")
        return lo, hi

    def scalar_ops(self, op, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty_like(a)
        self.lib.port_scalar_ops(ci(op), _p(a), _p(b), _p(out), ll(len(a)))
        return out

    def chain_fold(self, acc0, terms, up):
        acc0 = np.ascontiguousarray(acc0, dtype=np.float64)
        terms = np.ascontiguousarray(terms, dtype=np.float64)
        upa = np.ascontiguousarray(up, dtype=np.int32)
        out = np.empty_like(acc0)
        self.lib.port_chain_fold(ci(terms.shape[0]), ci(terms.shape[1]), _p(acc0), _p(terms), _p(upa), _p(out))
        return out

    def analyze(self, layers, box_lo, box_hi, label=-1, early_term=True, chunk_rows=0,
                memory_budget=0):
        """layers: list of objects with kind, preds, out_shape, fw.., weights, bias."""
        n = len(layers)
        info = np.zeros((n, 16), dtype=np.int32)
        wptr = (vp * n)()
        bptr = (vp * n)()
        keep = []
        total = 0
        for k, L in enumerate(layers):
            w, h, c = L.out_shape
            total += w * h * c
            p = list(L.preds) + [-1, -1]
            info[k, :15] = [KIND[L.kind], len(L.preds), p[0], p[1], w, h, c, L.fw, L.fh, L.sw,
                            L.sh, L.pw, L.ph, L.cin, L.cout]
            if L.weights is not None:
                wa = np.ascontiguousarray(L.weights, dtype=np.float64).reshape(-1)
                ba = np.ascontiguousarray(L.bias, dtype=np.float64)
                keep += [wa, ba]
                wptr[k], bptr[k] = wa.ctypes.data, ba.ctypes.data
        n_out = int(np.prod(layers[-1].out_shape))
        margins = np.zeros(max(n_out - 1, 1))
        verified = ci(0)
        stats = np.zeros(6, dtype=np.int64)
        bl, bh, rl, rh = (np.empty(total) for _ in range(4))
        lo = np.ascontiguousarray(box_lo, dtype=np.float64)
        hi = np.ascontiguousarray(box_hi, dtype=np.float64)
        rc = self.lib.port_analyze(_p(info), ci(n), wptr, bptr, _p(lo), _p(hi), ci(label),
                                   ci(int(early_term)), ll(chunk_rows), ll(memory_budget),
                                   ctypes.byref(verified), _p(margins), _p(stats), _p(bl), _p(bh),
                                   _p(rl), _p(rh))
        if rc:
            raise RuntimeError(f"port_analyze failed ({rc})")
        return {"verified": bool(verified.value) if label >= 0 else None,
                "margins": margins[: n_out - 1] if label >= 0 else None,
                "stats": dict(zip(["rows_total", "rows_terminated_early", "gbc_madds",
                                   "gbc_dense_equiv", "dense_madds", "checkpoints"],
                                  stats.tolist())),
                "b_lo": bl, "b_hi": bh, "r_lo": rl, "r_hi": rh}


class RefLayer:
    def __init__(self, **kw):
        self.__dict__.update(kw)


class Ref:
    """The unmodified reference (compiled by oracle/build_ref.sh)."""

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        self.lib = ctypes.CDLL(REF_SO)
        L = self.lib
        L.ref_generate.restype = vp
        L.ref_generate.argtypes = [ctypes.c_uint64, ctypes.c_char_p]
        L.ref_from_json.restype = vp
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_double_from_decimal.restype = cd
        L.ref_total_neurons.restype = ll
        L.ref_to_json.restype = vp
        L.ref_free.argtypes = [vp]

    def generate(self, seed, arch):
        h = self.lib.ref_generate(ctypes.c_uint64(seed), arch.encode())
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return vp(h)

    def from_json(self, text):
        h = self.lib.ref_from_json(text.encode())
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        return vp(h)

    def to_json(self, h):
        p = self.lib.ref_to_json(h)
        s = ctypes.cast(p, ctypes.c_char_p).value.decode()
        self.lib.ref_free_str(vp(p))
        return s

    def free(self, h):
        self.lib.ref_free(h)

    def layers(self, h):
        n = self.lib.ref_num_layers(h)
        out = []
        for k in range(n):
            info = (ci * 16)()
            nw, nb = ll(), ll()
            self.lib.ref_layer_info(h, ci(k), info, ctypes.byref(nw), ctypes.byref(nb))
            w = np.empty(nw.value) if nw.value else None
            b = np.empty(nb.value) if nb.value else None
            self.lib.ref_layer_params(h, ci(k), _p(w), _p(b))
            preds = [info[2], info[3]][: info[1]]
            kind = KIND_NAME[info[0]]
            if kind == "dense" and w is not None:
                w = w.reshape(info[6], -1)
            out.append(RefLayer(kind=kind, preds=preds, out_shape=(info[4], info[5], info[6]),
                                fw=info[7], fh=info[8], sw=info[9], sh=info[10], pw=info[11],
                                ph=info[12], cin=info[13], cout=info[14], head=info[15],
                                weights=w, bias=b))
        return out

    def random_inputs(self, seed, count, dim):
        out = np.empty((count, dim))
        self.lib.ref_random_inputs(ctypes.c_uint64(seed), ci(count), ci(dim), _p(out))
        return out

    def double_from_decimal(self, s):
        return self.lib.ref_double_from_decimal(s.encode())

    def candidate(self, h, center):
        c = np.ascontiguousarray(center, dtype=np.float64)
        return self.lib.ref_candidate(h, _p(c))

    def verify(self, h, center, eps, clamp01=True, label=-1, early_term=True, chunk_rows=0,
               memory_budget=0, workers=1, want_bounds=True):
        c = np.ascontiguousarray(center, dtype=np.float64)
        total = self.lib.ref_total_neurons(h)
        bl = bh = rl = rh = None
        if want_bounds:
            bl, bh, rl, rh = (np.empty(total) for _ in range(4))
        margins = np.zeros(64)
        verified = ci(0)
        stats = np.zeros(6, dtype=np.int64)
        sec = cd(0)
        rc = self.lib.ref_verify(h, _p(c), cd(eps), ci(int(clamp01)), ci(label), ci(int(early_term)),
                                 ll(chunk_rows), ll(memory_budget), ci(workers),
                                 ctypes.byref(verified), _p(margins), _p(stats), _p(bl), _p(bh),
                                 _p(rl), _p(rh), ctypes.byref(sec))
        if rc:
            raise RuntimeError(self.lib.ref_last_error().decode())
        layers_n = self.lib.ref_num_layers(h)
        info = (ci * 16)()
        nw, nb = ll(), ll()
        self.lib.ref_layer_info(h, ci(layers_n - 1), info, ctypes.byref(nw), ctypes.byref(nb))
        n_out = info[4] * info[5] * info[6]
        return {"verified": bool(verified.value) if label >= 0 else None,
                "margins": margins[: n_out - 1].copy() if label >= 0 else None,
                "stats": dict(zip(["rows_total", "rows_terminated_early", "gbc_madds",
                                   "gbc_dense_equiv", "dense_madds", "checkpoints"],
                                  stats.tolist())),
                "b_lo": bl, "b_hi": bh, "r_lo": rl, "r_hi": rh, "seconds": sec.value}

    def rational_contains(self, h, center, eps_num, eps_den, clamp01, label, b_lo, b_hi, margins):
        """Exact-rational soundness check (oracle.hpp / the ExactRational engine,
        analyzer.hpp:198-276 over mpq): the number of given widened bounds and
        margins that fail to contain the exact ones, and the exact verdict."""
        c = np.ascontiguousarray(center, dtype=np.float64)
        bl = np.ascontiguousarray(b_lo, dtype=np.float64)
        bh = np.ascontiguousarray(b_hi, dtype=np.float64)
        m = np.ascontiguousarray(margins if margins is not None else np.zeros(1), dtype=np.float64)
        ver = ci(0)
        bad = self.lib.ref_rational_contains(h, _p(c), ctypes.c_long(eps_num), ctypes.c_long(eps_den),
                                             ci(int(clamp01)), ci(label), _p(bl), _p(bh), _p(m),
                                             ctypes.byref(ver))
        if bad < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return bad, bool(ver.value)

    def verify_batch(self, h, centers, eps, clamp01=True, threads=1, early_term=True):
        X = np.ascontiguousarray(centers, dtype=np.float64)
        n = X.shape[0]
        verdicts = np.zeros(n, dtype=np.int32)
        per = np.zeros(n)
        wall = cd(0)
        rc = self.lib.ref_verify_batch(h, _p(X), ci(n), cd(eps), ci(int(clamp01)), ci(threads),
                                       ci(int(early_term)), _p(verdicts), ctypes.byref(wall), _p(per))
        if rc < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return verdicts, wall.value, per
