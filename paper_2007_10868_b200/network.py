"""Network model: the mode-neutral layer list (the reference's ModelDoc /
LayerDoc, proj/include/polycert/network.hpp:16-55) with FP64 parameters in the
reference's flat layouts, lowered to the C-ABI's pc_layer_desc array.
Validation (shape inference + structural rules, model_io.cpp:49-135) is done
by the native library so messages match the reference's.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass
class Layer:
    kind: str                      # input | dense | conv | relu | residual_join
    preds: list = field(default_factory=list)
    out_shape: tuple | None = None  # (w, h, c); filled by validation
    weights: np.ndarray | None = None  # dense [out][in]; conv flat ((fy*fw+fx)*cin+ci)*cout+co
    bias: np.ndarray | None = None
    fw: int = 0
    fh: int = 0
    sw: int = 1
    sh: int = 1
    pw: int = 0
    ph: int = 0
    cin: int = 0
    cout: int = 0


class Network:
    """Immutable layer DAG in topological id order; layers[0] is the input."""

    def __init__(self, layers: list[Layer]):
        self.layers = layers
        self._keep = []

    @property
    def input_shape(self):
        return self.layers[0].out_shape

    def descs(self):
        """pc_layer_desc array (the arrays it points at are kept alive on self)."""
        arr = (_lib.PcLayerDesc * len(self.layers))()
        self._keep = []
        for k, L in enumerate(self.layers):
            d = arr[k]
            d.kind = _lib.KIND[L.kind]
            d.n_preds = len(L.preds)
            for i, p in enumerate(L.preds[:2]):
                d.preds[i] = int(p)
            if L.kind == "dense":
                w = np.ascontiguousarray(L.weights, dtype=np.float64)
                d.n_out = int(w.shape[0]) if w.ndim == 2 else int(len(L.bias))
                b = np.ascontiguousarray(L.bias, dtype=np.float64)
                self._keep += [w, b]
                d.weights, d.bias = w.ctypes.data, b.ctypes.data
            elif L.kind == "conv":
                w = np.ascontiguousarray(L.weights, dtype=np.float64).reshape(-1)
                b = np.ascontiguousarray(L.bias, dtype=np.float64)
                self._keep += [w, b]
                d.weights, d.bias = w.ctypes.data, b.ctypes.data
                d.fw, d.fh, d.sw, d.sh = L.fw, L.fh, L.sw, L.sh
                d.pw, d.ph, d.cin, d.cout = L.pw, L.ph, L.cin, L.cout
        return arr

    def validate(self):
        """Shape inference + validate_model's rules; raises ModelError."""
        arr = self.descs()
        shapes = (ctypes.c_int * (3 * len(self.layers)))()
        w, h, c = self.input_shape
        _lib.check(_lib.lib.pc_validate(arr, len(self.layers), w, h, c, shapes))
        for k, L in enumerate(self.layers):
            L.out_shape = (shapes[3 * k], shapes[3 * k + 1], shapes[3 * k + 2])
        return self

    def numel(self, k: int) -> int:
        w, h, c = self.layers[k].out_shape
        return w * h * c

    def offsets(self):
        off = [0]
        for k in range(len(self.layers)):
            off.append(off[-1] + self.numel(k))
        return off

    @property
    def output_size(self) -> int:
        return self.numel(len(self.layers) - 1)

    def total_neurons(self) -> int:
        return self.offsets()[-1]
