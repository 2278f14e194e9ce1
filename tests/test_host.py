"""CPU-only checks of the product library: it loads (every symbol resolves),
exports every entry point include/polycert_b200.h declares, validates models
with the reference's messages (model_io.cpp:49-135), and has no CPU fallback."""
import ctypes

import numpy as np
import pytest


def test_library_loads_and_exports_header_symbols():
    from paper_2007_10868_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH, mode=ctypes.RTLD_GLOBAL | 2)  # RTLD_NOW: all symbols resolve
    syms = _lib.header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name


def _net(layers):
    import paper_2007_10868_b200 as pc
    return pc.Network(layers)


def test_validation_messages():
    import paper_2007_10868_b200 as pc
    L = pc.Layer
    with pytest.raises(pc._lib.ModelError, match="model: layer 1: in_channels 2 != predecessor channels 1"):
        _net([L("input", [], (4, 4, 1)), L("conv", [0], weights=np.zeros(3 * 3 * 2 * 2), bias=np.zeros(2),
                                               fw=3, fh=3, cin=2, cout=2)]).validate()
    with pytest.raises(pc._lib.ModelError, match="model: layer 1: stride does not tile the padded input"):
        _net([L("input", [], (5, 5, 1)), L("conv", [0], weights=np.zeros(4), bias=np.zeros(1),
                                               fw=2, fh=2, sw=2, sh=2, cin=1, cout=1)]).validate()
    with pytest.raises(pc._lib.ModelError, match="model: layer 2: relu fed by relu"):
        _net([L("input", [], (1, 1, 2)), L("relu", [0]), L("relu", [1])]).validate()
    with pytest.raises(pc._lib.ModelError, match="model: layer 1: predecessor 3 is not an earlier layer"):
        _net([L("input", [], (1, 1, 2)), L("relu", [3])]).validate()
    with pytest.raises(pc._lib.ModelError, match="residual_join needs 2 predecessor"):
        _net([L("input", [], (1, 1, 2)), L("residual_join", [0])]).validate()
    with pytest.raises(pc._lib.ModelError, match="model: no layers"):
        _net([L("input", [], (1, 1, 2))]).validate()


def test_validation_shapes():
    import paper_2007_10868_b200 as pc
    net = pc.generate(7, "input 8x8x2; conv 4x4x3 s2 p1; relu; block(conv 3x3x3 s1 p1 | skip); relu; dense 5")
    assert [L.out_shape for L in net.layers] == [(8, 8, 2), (4, 4, 3), (4, 4, 3), (4, 4, 3), (4, 4, 3),
                                                 (4, 4, 3), (1, 1, 5)]


def test_no_cpu_fallback():
    """Without a CUDA device the engine refuses to run (PC_ERR_CUDA), never computes on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2007_10868_b200 as pc
    net = pc.generate(7, "input 1x1x4; dense 3; relu; dense 2")
    with pytest.raises(pc._lib.CudaError):
        pc.Verifier(net)
    with pytest.raises(pc._lib.CudaError):
        pc.input_box([0.5] * 4, 0.1)


def test_model_json_roundtrip(tmp_path):
    import paper_2007_10868_b200 as pc
    from paper_2007_10868_b200 import model_io
    net = pc.generate(202608, "input 4x4x1; conv 3x3x2 s1 p1; relu; dense 3")
    p = tmp_path / "m.json"
    model_io.save_model(net, str(p))
    back = model_io.load_model(str(p))
    for a, b in zip(net.layers, back.layers):
        assert a.kind == b.kind and a.out_shape == b.out_shape
        if a.weights is not None:
            assert np.array_equal(np.asarray(a.weights).reshape(-1), np.asarray(b.weights).reshape(-1))
    with pytest.raises(ValueError, match="malformed number"):
        model_io.model_from_json_obj({"format": "polycert-model-v1", "input_shape": [1, 1, 1],
                                      "layers": [{"id": 1, "kind": "dense", "predecessors": [0],
                                                  "weights": [["1e3"]], "bias": ["0"]}]})
