"""The drop-in verifier surface (proj/include/polycert/analyzer.hpp:164-276,
network.hpp:150-177), backed by the GPU engine through the C-ABI.

    net = generate(7, arch)                       # or model_io.load_model(path)
    v = Verifier(net)                             # pc_net_create: upload to the GPU
    box = input_box(center, eps, clamp01=True)    # InputBox<WidenedFloat64>
    verdict = v.verify_robustness(box, label)     # verify_robustness(net, box, label, opt)
    result = v.analyze(box)                       # analyze(...).state.bounds / .raw

Results are bit-identical to the reference's WidenedFloat64 analysis.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .network import Network


@dataclass
class AnalysisOptions:  # analyzer.hpp:164-169
    early_term: bool = True
    chunk_rows: int = 0
    memory_budget: int = 0  # 0: engine default (16 GiB of device workspace)
    device: int = -1
    exec_mode: int = 0  # 0 auto, 1 host-driven schedule, 2 device-driven (CUDA graph)
    numeric_mode: int = 0  # 0 WidenedFloat64 bit for bit; 1 fast native directed rounding (sound)


@dataclass
class InputBox:  # network.hpp:155-158
    lo: np.ndarray
    hi: np.ndarray


@dataclass
class Verdict:  # analyzer.hpp:247-254
    verified: bool
    label: int
    margins: list  # [(class j, certified lower bound of out_label - out_j)], ascending j
    stats: dict = field(default_factory=dict)


@dataclass
class AnalysisResult:  # analyzer.hpp:171-175
    bounds: list  # per layer: (lo, hi) arrays, padded
    raw: list     # per layer: (lo, hi) arrays, unpadded freeze-test twin
    stats: dict = field(default_factory=dict)
    margins: np.ndarray | None = None
    verified: bool | None = None


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def fp64_peak(device: int = -1) -> float:
    """Measured FP64 FMA throughput of the device (FMA/s; pc_fp64_peak)."""
    v = ctypes.c_double(0)
    _lib.check(_lib.lib.pc_fp64_peak(int(device), ctypes.byref(v)))
    return v.value


def input_box(center, eps: float, clamp01: bool = True) -> InputBox:
    """input_box<WidenedFloat64> (network.hpp:160-177), computed on the GPU."""
    c = np.ascontiguousarray(center, dtype=np.float64).reshape(-1)
    lo = np.empty_like(c)
    hi = np.empty_like(c)
    _lib.check(_lib.lib.pc_input_box(_ptr(c), len(c), float(eps), int(bool(clamp01)), _ptr(lo), _ptr(hi)))
    return InputBox(lo, hi)


class Verifier:
    """A network instantiated on the GPU (Network<WidenedFloat64> analogue)."""

    def __init__(self, net: Network, options: AnalysisOptions | None = None):
        if net.layers[0].out_shape is None:
            raise ValueError("network has no input shape")
        self.net = net
        self.options = options or AnalysisOptions()
        o = _lib.PcOptions()
        _lib.lib.pc_default_options(ctypes.byref(o))
        o.early_term = int(bool(self.options.early_term))
        o.chunk_rows = int(self.options.chunk_rows)
        o.memory_budget = int(self.options.memory_budget)
        o.device = int(self.options.device)
        o.exec_mode = int(self.options.exec_mode)
        o.numeric_mode = int(self.options.numeric_mode)
        descs = net.descs()
        h = ctypes.c_void_p()
        w, hh, c = net.input_shape
        _lib.check(_lib.lib.pc_net_create(descs, len(net.layers), w, hh, c, ctypes.byref(o),
                                          ctypes.byref(h)))
        self._h = h
        if net.layers[-1].out_shape is None:
            net.validate()
        self.offsets = net.offsets()
        self.n_out = _lib.lib.pc_net_output_size(h)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib.pc_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # test(lo, up, label) — the reference-facing entry point
    def test(self, lo, up, label: int, want_bounds: bool = False):
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        up = np.ascontiguousarray(up, dtype=np.float64)
        nm = max(self.n_out - 1, 1)
        margins = np.zeros(nm)
        verified = ctypes.c_int(0)
        st = _lib.PcStats()
        T = self.offsets[-1]
        bl = bh = rl = rh = None
        if want_bounds:
            bl, bh, rl, rh = (np.empty(T) for _ in range(4))
        _lib.check(_lib.lib.pc_net_test(self._h, _ptr(lo), _ptr(up), int(label), ctypes.byref(verified),
                                        _ptr(margins), _ptr(bl), _ptr(bh), _ptr(rl), _ptr(rh),
                                        ctypes.byref(st)))
        res = AnalysisResult(bounds=[], raw=[], stats=st.as_dict())
        if want_bounds:
            for k in range(len(self.offsets) - 1):
                a, b = self.offsets[k], self.offsets[k + 1]
                res.bounds.append((bl[a:b], bh[a:b]))
                res.raw.append((rl[a:b], rh[a:b]))
        if label >= 0:
            res.margins = margins[: self.n_out - 1]
            res.verified = bool(verified.value)
        return res

    def verify_robustness(self, box: InputBox, label: int, want_bounds: bool = False) -> Verdict:
        """verify_robustness (analyzer.hpp:256-276)."""
        if label < 0 or label >= self.n_out:
            raise _lib.InvalidArgument(_lib.PC_ERR_INVALID_ARGUMENT, "margin: label out of range")
        r = self.test(box.lo, box.hi, label, want_bounds)
        classes = [j for j in range(self.n_out) if j != label]
        v = Verdict(verified=r.verified, label=label,
                    margins=[(j, float(m)) for j, m in zip(classes, r.margins)], stats=r.stats)
        if want_bounds:
            v.analysis = r
        return v

    def analyze(self, box: InputBox) -> AnalysisResult:
        """analyze (analyzer.hpp:198-242): refined per-neuron bounds."""
        return self.test(box.lo, box.hi, -1, want_bounds=True)

    def test_batch(self, lo, up, labels, concurrency: int = 8, device_inputs: bool = False):
        """Verify many boxes concurrently (one stream per worker). lo/up: (n, input numel)
        host arrays, or device pointers (ints) when device_inputs. Returns
        (verified[n], margins[n, n_out-1], stats list, device_ms)."""
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        n = len(labels)
        nm = max(self.n_out - 1, 1)
        verified = np.zeros(n, dtype=np.int32)
        margins = np.zeros((n, nm))
        stats = (_lib.PcStats * max(n, 1))()
        ms = ctypes.c_double(0)
        if device_inputs:
            plo, pup = ctypes.c_void_p(lo), ctypes.c_void_p(up)
        else:
            lo = np.ascontiguousarray(lo, dtype=np.float64)
            up = np.ascontiguousarray(up, dtype=np.float64)
            plo, pup = _ptr(lo), _ptr(up)
        _lib.check(_lib.lib.pc_net_test_batch(self._h, n, plo, pup, int(bool(device_inputs)),
                                              _ptr(labels), int(concurrency), _ptr(verified),
                                              _ptr(margins), stats, ctypes.byref(ms)))
        return verified.astype(bool), margins[:, : self.n_out - 1], [s.as_dict() for s in stats[:n]], ms.value

    def candidate(self, center) -> int:
        """Unique argmax of the concrete forward pass (-1 on ties), on the GPU."""
        c = np.ascontiguousarray(center, dtype=np.float64)
        lab = ctypes.c_int(-1)
        _lib.check(_lib.lib.pc_net_candidate(self._h, _ptr(c), ctypes.byref(lab), None))
        return lab.value

    @property
    def stream_handle(self) -> int:
        """cudaStream_t of the engine (for CUDA-event timing by callers)."""
        return int(_lib.lib.pc_net_stream(self._h) or 0)

    def test_device(self, d_lo: int, d_up: int, label: int):
        """test(lo, up, label) with the box already in device memory (pointers)."""
        nm = max(self.n_out - 1, 1)
        margins = np.zeros(nm)
        verified = ctypes.c_int(0)
        st = _lib.PcStats()
        _lib.check(_lib.lib.pc_net_test_device(self._h, ctypes.c_void_p(d_lo), ctypes.c_void_p(d_up),
                                               int(label), ctypes.byref(verified), _ptr(margins),
                                               ctypes.byref(st)))
        return bool(verified.value), margins[: self.n_out - 1], st.as_dict()

    def enable_sharding(self, group=None, transport: str = "auto"):
        """Row-shard every pass across the ranks of a torch.distributed group
        (one process per GPU; results identical to unsharded). Returns (rank, world).
        transport: "auto" (native NCCL on an NCCL group), "native", "callback"."""
        from . import sharding
        return sharding.enable(self, group, transport)

    def disable_sharding(self):
        from . import sharding
        sharding.disable(self)

    @staticmethod
    def last_profile() -> dict:
        """Per-kernel-class {class: [launches, ms]} of the last call (PC_PROFILE=1)."""
        import json
        n = _lib.lib.pc_last_profile(None, 0) + 1
        buf = ctypes.create_string_buffer(n)
        _lib.lib.pc_last_profile(buf, n)
        return json.loads(buf.value.decode())

    @staticmethod
    def last_kernel_timing(kernel: str = "conv"):
        """CUDA-event ms, algorithmic bytes and launches of one coefficient kernel
        ("dense" = k_dense_coef*, "conv" = k_gbc_sparse2 / k_gbc_coef) in the last call."""
        ms, by, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
        _lib.lib.pc_last_kernel_timing(1 if kernel == "conv" else 0, ctypes.byref(ms), ctypes.byref(by),
                                       ctypes.byref(n))
        return {"ms": ms.value, "bytes": by.value, "launches": n.value,
                "executed_madds": float(_lib.lib.pc_last_conv_executed_madds()) if kernel == "conv" else None}

    def set_serial(self, serial: bool = True):
        """One stream, one pipeline per walk, so per-launch CUDA events time
        each kernel alone (roofline measurement); results are identical."""
        _lib.check(_lib.lib.pc_net_set_serial(self._h, int(bool(serial))))

    def last_timing(self):
        t, dm, db, dl = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
        _lib.lib.pc_last_timing(ctypes.byref(t), ctypes.byref(dm), ctypes.byref(db), ctypes.byref(dl))
        return {"total_ms": t.value, "dense_ms": dm.value, "dense_bytes": db.value,
                "dense_launches": dl.value, "dense_madds": float(_lib.lib.pc_last_dense_madds()),
                "launches": int(_lib.lib.pc_last_launch_count())}
