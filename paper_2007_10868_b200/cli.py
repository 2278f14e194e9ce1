"""Command-line front end with the reference CLI's subcommands, flags, output
schemas and exit codes (proj/tools/main.cpp:38-320, proj/docs/report_formats.md):

  python -m paper_2007_10868_b200 verify --model M --inputs X --epsilon E [--out F]
      JSONL per input: {"index","candidate","verdict","margins":[{"class","lower"}],
      "runtime_ns","rows_terminated"} (main.cpp:162-176); skipped (tied argmax)
      and per-input error lines as in main.cpp:129-140, 178-184
  python -m paper_2007_10868_b200 bench  ... -> CSV index,runtime_ns,early_term_fraction
  python -m paper_2007_10868_b200 gen --seed S --arch A --out M [--inputs-out X --inputs N]

Exit codes: 0 ok, 1 some input failed, 2 usage / model error (main.cpp:305-320).
Only the widened mode exists here (the reference's rational mode is its exact
CPU oracle). The analysis runs on the GPU; runtime_ns is the wall time of
verify_robustness as in main.cpp:146-150.
"""
from __future__ import annotations

import argparse
import json
import sys
import time


def _run_flags(p):
    p.add_argument("--model", required=True)
    p.add_argument("--inputs", required=True)
    p.add_argument("--epsilon", required=True)
    p.add_argument("--mode", default="widened", choices=["widened"])
    p.add_argument("--no-early-term", action="store_true")
    p.add_argument("--chunk-rows", type=int, default=0)
    p.add_argument("--memory-budget", type=int, default=0)
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--out", default="")
    p.add_argument("--no-clamp", action="store_true")
    p.add_argument("--device", type=int, default=-1)


def _verify_or_bench(a, bench: bool) -> int:
    from . import AnalysisOptions, Verifier, input_box
    from .model_io import load_inputs, load_model, parse_decimal
    net = load_model(a.model)
    rows = load_inputs(a.inputs)
    eps = parse_decimal(a.epsilon)  # decimal string, one correct rounding (decimal.cpp:63-76)
    v = Verifier(net, AnalysisOptions(early_term=not a.no_early_term, chunk_rows=a.chunk_rows,
                                      memory_budget=a.memory_budget, device=a.device))
    n_in = v.net.numel(0)
    lines, failed = [], False
    for i, cells in enumerate(rows):
        try:
            if len(cells) != n_in:
                raise ValueError("input size mismatch")
            x = [parse_decimal(t) for t in cells]  # scalar_from_decimal per cell (main.cpp:122-124)
            label = v.candidate(x)
            if label < 0:  # tied argmax: not a candidate (main.cpp:129-140)
                lines.append(f"{i},0,0.000000" if bench else json.dumps(
                    {"index": i, "candidate": None, "verdict": "skipped", "margins": [], "runtime_ns": 0,
                     "rows_terminated": 0}, separators=(",", ":")))
                continue
            box = input_box(x, eps, not a.no_clamp)
            t0 = time.perf_counter_ns()
            verdict = v.verify_robustness(box, label)
            ns = time.perf_counter_ns() - t0
            st = verdict.stats
            if bench:
                frac = st["rows_terminated_early"] / st["rows_total"] if st["rows_total"] > 0 else 0.0
                lines.append("%d,%d,%.6f" % (i, ns, frac))
            else:
                lines.append(json.dumps(
                    {"index": i, "candidate": label, "verdict": "verified" if verdict.verified else "unknown",
                     "margins": [{"class": c, "lower": m} for c, m in verdict.margins], "runtime_ns": ns,
                     "rows_terminated": st["rows_terminated_early"]}, separators=(",", ":")))
        except Exception as e:  # per-input failure (main.cpp:178-184)
            lines.append(json.dumps({"index": i, "error": str(e)}, separators=(",", ":")))
            failed = True
    out = open(a.out, "w") if a.out else sys.stdout
    try:
        if bench:
            out.write("index,runtime_ns,early_term_fraction\n")
        for line in lines:
            out.write(line + "\n")
    finally:
        if a.out:
            out.close()
    return 1 if failed else 0


def _gen(a) -> int:
    from .gen import decimal_from_double, generate, random_inputs
    from .model_io import save_model
    net = generate(a.seed, a.arch)
    save_model(net, a.out)
    if a.inputs_out:
        import numpy as np
        X = random_inputs(a.seed + 1, a.inputs, int(np.prod(net.input_shape)))
        with open(a.inputs_out, "w") as f:
            for row in X:
                f.write(",".join(decimal_from_double(v) for v in row) + "\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="polycert-b200",
                                 description="polyhedral robustness certifier for relu networks (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    _run_flags(sub.add_parser("verify", help="verify a batch of inputs (JSONL)"))
    _run_flags(sub.add_parser("bench", help="runtime statistics per input (CSV)"))
    g = sub.add_parser("gen", help="generate a seeded model")
    g.add_argument("--seed", type=int, required=True)
    g.add_argument("--arch", required=True)
    g.add_argument("--out", required=True)
    g.add_argument("--inputs-out", default="")
    g.add_argument("--inputs", type=int, default=20)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "gen":
            return _gen(a)
        return _verify_or_bench(a, a.cmd == "bench")
    except Exception as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
