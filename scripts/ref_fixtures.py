"""Generate golden fixtures for the residual configs from the UNMODIFIED reference.

TEST INFRASTRUCTURE ONLY. Runs oracle/_ref/libpolycert_ref.so (the reference
compiled from /root/reference/proj by oracle/build_ref.sh) on one image of a
named BASELINE config and writes tests/golden/ref_<config>_img<i>.json:

* the candidate label (forward_eval + unique_argmax, tools/main.cpp:86-100),
* the verdict and the margin bit patterns (verify_robustness,
  analyzer.hpp:256-276 = analyze + run_margin_pass, backsub.hpp:1070-1096),
* PassStats (backsub.hpp:119-125),
* per layer: SHA-256 of the padded and raw bound bit patterns
  (AnalysisState.bounds / .raw, backsub.hpp:71-80) and the bounds of the
  last layer verbatim.

The full bound arrays are kept (uncommitted) under oracle/_ref/fixtures/ for
debugging. Results are chunk- and worker-invariant (test_backsub.cpp:74-157),
so `workers` only changes the wall time.

    python scripts/ref_fixtures.py cifar_resnet34 0 --workers 2
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Ref  # noqa: E402


def _load_configs():
    # by file path: never import the product package from a checker
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "pc_configs", os.path.join(ROOT, "paper_2007_10868_b200", "configs.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def layer_hashes(layers, arrs):
    out = []
    off = 0
    for L in layers:
        n = int(np.prod(L.out_shape))
        out.append({k: hashlib.sha256(np.ascontiguousarray(a[off:off + n]).tobytes()).hexdigest()
                    for k, a in arrs.items()})
        off += n
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("image", type=int)
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--no-early-term", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    cfg = _load_configs()
    arch, eps_s = cfg.CONFIGS[a.config]
    ref = Ref()
    t0 = time.time()
    h = ref.generate(cfg.MODEL_SEED, arch)
    layers = ref.layers(h)
    dim = int(np.prod(layers[0].out_shape))
    X = ref.random_inputs(cfg.INPUT_SEED, a.image + 1, dim)
    x = X[a.image]
    eps = ref.double_from_decimal(eps_s)
    label = ref.candidate(h, x)
    t1 = time.time()
    print(f"[{a.config} img{a.image}] generated in {t1 - t0:.1f}s, label {label}", flush=True)
    r = ref.verify(h, x, eps, clamp01=True, label=label, early_term=not a.no_early_term,
                   workers=a.workers)
    t2 = time.time()
    arrs = {"b_lo": r["b_lo"], "b_hi": r["b_hi"], "r_lo": r["r_lo"], "r_hi": r["r_hi"]}
    n_last = int(np.prod(layers[-1].out_shape))
    doc = {
        "generator": "scripts/ref_fixtures.py over oracle/_ref (unmodified reference, -O3 -DNDEBUG)",
        "config": a.config, "arch": arch, "eps": eps_s, "model_seed": cfg.MODEL_SEED,
        "input_seed": cfg.INPUT_SEED, "image": a.image, "clamp01": True,
        "early_term": not a.no_early_term, "label": int(label),
        "verified": bool(r["verified"]),
        "margins_hex": [float(m).hex() for m in r["margins"]],
        "stats": {k: int(v) for k, v in r["stats"].items()},
        "layer_sha256": layer_hashes(layers, arrs),
        "last_layer": {k: [float(v).hex() for v in arr[-n_last:]] for k, arr in arrs.items()},
        "ref_seconds": r["seconds"], "workers": a.workers,
    }
    os.makedirs(a.out, exist_ok=True)
    tag = "" if not a.no_early_term else "_noet"
    path = os.path.join(a.out, f"ref_{a.config}_img{a.image}{tag}.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    dbg = os.path.join(ROOT, "oracle", "_ref", "fixtures")
    os.makedirs(dbg, exist_ok=True)
    np.savez(os.path.join(dbg, f"{a.config}_img{a.image}{tag}.npz"), **arrs,
             margins=r["margins"])
    print(f"[{a.config} img{a.image}] verified={doc['verified']} analyze {r['seconds']:.1f}s "
          f"(wall {t2 - t1:.1f}s) stats {doc['stats']} -> {path}", flush=True)


if __name__ == "__main__":
    main()
