"""polycert-model-v1 JSON and inputs CSV (proj/src/model_io.cpp:196-353,
proj/docs/model_format.md). Numbers are decimal strings; they are parsed with
one correct rounding (float() == strtod, decimal.cpp:63-76)."""
from __future__ import annotations

import json
import re

import numpy as np

from .gen import decimal_from_double
from .network import Layer, Network

_DEC = re.compile(r"^[+-]?[0-9]+(\.[0-9]+)?$")  # decimal.cpp:14-44
FORMAT = "polycert-model-v1"


def _num(t, lid):
    if not isinstance(t, str):
        raise ValueError(f"model: layer {lid}: numbers must be decimal strings")
    if not _DEC.match(t):
        raise ValueError(f"model: layer {lid}: malformed number '{t}'")
    return float(t)


def parse_decimal(t: str) -> float:
    """double_from_decimal (decimal.cpp:63-76): grammar check, one correct rounding."""
    if not _DEC.match(t):
        raise ValueError(f"bad decimal: {t}")
    return float(t)


def model_from_json_obj(j) -> Network:
    if j.get("format") != FORMAT:
        raise ValueError("model: missing or unsupported format tag")
    w, h, c = (int(v) for v in j["input_shape"])
    layers = [Layer("input", [], (w, h, c))]
    for lj in j["layers"]:
        lid = int(lj["id"])
        kind = lj["kind"]
        if kind not in ("dense", "conv", "relu", "residual_join"):
            raise ValueError(f"model: layer {lid}: unknown kind '{kind}'")
        L = Layer(kind, [int(p) for p in lj["predecessors"]])
        if kind == "dense":
            L.weights = np.array([[_num(t, lid) for t in row] for row in lj["weights"]], dtype=np.float64)
            L.bias = np.array([_num(t, lid) for t in lj["bias"]], dtype=np.float64)
        elif kind == "conv":
            L.fw, L.fh = (int(v) for v in lj["filter_size"])
            L.sw, L.sh = (int(v) for v in lj["stride"])
            L.pw, L.ph = (int(v) for v in lj["padding"])
            L.cin, L.cout = int(lj["in_channels"]), int(lj["out_channels"])
            flat = [_num(co, lid) for fy in lj["filter"] for fx in fy for ci in fx for co in ci]
            L.weights = np.array(flat, dtype=np.float64)
            L.bias = np.array([_num(t, lid) for t in lj["bias"]], dtype=np.float64)
        layers.append(L)
    return Network(layers).validate()


def load_model(path: str) -> Network:
    with open(path) as f:
        return model_from_json_obj(json.load(f))


def model_to_json_obj(net: Network) -> dict:
    """model_to_json_text (model_io.cpp:265-310); values as exact decimals."""
    out = {"format": FORMAT, "input_shape": list(net.input_shape), "layers": []}
    for k, L in enumerate(net.layers[1:], start=1):
        lj = {"id": k, "kind": L.kind, "predecessors": list(L.preds)}
        if L.kind == "dense":
            lj["weights"] = [[decimal_from_double(v) for v in row] for row in np.asarray(L.weights)]
            lj["bias"] = [decimal_from_double(v) for v in L.bias]
        elif L.kind == "conv":
            f = np.asarray(L.weights).reshape(L.fh, L.fw, L.cin, L.cout)
            lj["filter_size"] = [L.fw, L.fh]
            lj["stride"] = [L.sw, L.sh]
            lj["padding"] = [L.pw, L.ph]
            lj["in_channels"] = L.cin
            lj["out_channels"] = L.cout
            lj["filter"] = [[[[decimal_from_double(v) for v in ci] for ci in fx] for fx in fy] for fy in f]
            lj["bias"] = [decimal_from_double(v) for v in L.bias]
        out["layers"].append(lj)
    return out


def save_model(net: Network, path: str):
    with open(path, "w") as f:
        f.write(json.dumps(model_to_json_obj(net), indent=1, sort_keys=True) + "\n")


def load_inputs(path: str) -> list[list[str]]:
    """load_inputs (model_io.cpp:331-353): rows of trimmed decimal strings.

    Cells stay strings, as in the reference; they are parsed (and the row
    length checked) per input inside the CLI's per-input try, so one bad row
    becomes an {index, error} line instead of aborting the run
    (tools/main.cpp:117-184). Split like std::getline(ss, cell, ','): a
    trailing comma does not make an empty last cell.
    """
    rows = []
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"cannot open inputs file: {path}")
    with f:
        for line in f:
            line = line[:-1] if line.endswith("\n") else line
            if not line:
                continue
            parts = line.split(",")
            if parts and parts[-1] == "":
                parts.pop()  # getline yields no cell after a final delimiter
            row = []
            for cell in parts:
                t = cell.strip(" \t\r")
                if not t:
                    raise RuntimeError(f"inputs {path}: empty cell on line {len(rows) + 1}")
                row.append(t)
            if row:
                rows.append(row)
    return rows
