#!/usr/bin/env python
"""Benchmark: ms/image to verify one image (BASELINE.json metric) on 1/2/4/8
B200, GPU engine vs the reference's own CPU verifier.

A "step" verifies one image: analyze + margin pass (verify_robustness,
analyzer.hpp:256-276) on a generator-built network (random-init dyadic
weights of the named architecture, gen.cpp) and generator inputs (seed 8,
image s of the pool). Default workload: the paper's headline 34-layer
residual net (BASELINE.json configs[4], `cifar_resnet34`, eps 2/255, early
termination on).

  value  per-image latency (ms/image): the image's box already in HBM
         (pc_net_test_device), CUDA events on the engine stream around the
         whole verification; N > 1: the same image row-sharded over all ranks
         (native NCCL all-gather), max over ranks. L2 flushed between steps.
  e2e    the same through the reference-facing C-ABI call with HOST buffers
         (pc_net_test: box H2D + margins D2H inside the timed region), host
         clock around the synchronous call, max over ranks.
  throughput_ms_per_image  replicas: images verified concurrently
         (pc_net_test_batch) on every rank, whole-job ms/image.
  parity  the timed images that have reference fixtures
         (tests/golden/ref_<config>_img<i>.json, made by
         scripts/ref_fixtures.py from the unmodified reference) are compared
         bit for bit: verdict, margins, PassStats.
  roofline  the conv back-substitution kernel (k_gbc_flat), the dominant
         kernel of the residual configs: FLOPs (4 per interval multiply-add it
         executes, device-counted) per second of its CUDA-event time with the
         walks serialised (each launch alone on the GPU) vs the FP64 FMA peak
         measured live (pc_fp64_peak); its HBM fraction and the reference-
         equivalent rate (the reference's gbc_madds, which also counts cells
         no result reads) beside it.
  cpu_baseline / --impl reference: the unmodified reference (oracle/_ref)
         on the host's cores, one image with AnalysisOptions.workers = all
         host threads (the reference's latency mode). When one image cannot
         finish in the time allowed (the ResNets take hours), the line
         reports the elapsed time as a lower bound (`value_is_lower_bound`).

`python bench.py --gpus N` (N > 1) relaunches itself under torch.distributed.run
with N ranks; under torchrun the ranks come from the environment.
"""
from __future__ import annotations

import argparse
import glob
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms/image to verify (1/2/4/8 B200) + certified count == CPU ref; HBM GB/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cifar_resnet34")
    ap.add_argument("--no-early-term", action="store_true")
    ap.add_argument("--cpu-sample-seconds", type=float, default=30.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--throughput-images", type=int, default=16, help="images per replica batch")
    ap.add_argument("--concurrency", type=int, default=4, help="worker contexts of the replica batch")
    ap.add_argument("--pool", type=int, default=8, help="distinct images cycled through by the steps")
    ap.add_argument("--fast-steps", type=int, default=4, help="steps of the fast numeric mode (0: skip)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def load_configs():
    """configs.py by file path: the reference arm never imports the product package."""
    spec = importlib.util.spec_from_file_location(
        "pc_configs", os.path.join(ROOT, "paper_2007_10868_b200", "configs.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def workload(name):
    cfg = load_configs()
    arch, eps = cfg.CONFIGS[name]
    return arch, eps, cfg.MODEL_SEED, cfg.INPUT_SEED


def config_dict(args, arch, eps_s, mseed, iseed, world):
    return {"workload": args.config, "arch": arch, "eps": eps_s, "model_seed": mseed,
            "input_seed": iseed, "images": f"pool of {args.pool} generator images, step s verifies image s mod {args.pool}",
            "early_term": not args.no_early_term,
            "parallelism": (f"row sharding x{world} (every pass's live rows split across ranks, "
                            "candidate bounds all-gathered over NCCL)") if world > 1 else "1 GPU",
            "l2": "flushed between steps (256 MB write, outside the timed region)"}


def fixtures(config):
    out = {}
    for p in glob.glob(os.path.join(ROOT, "tests", "golden", f"ref_{config}_img*.json")):
        fx = json.load(open(p))
        if fx.get("early_term", True):
            out[int(fx["image"])] = fx
    return out


def offline_reference_seconds(config):
    """Full-image reference times recorded when the fixtures were made (this
    repo's container CPU, not the bench host)."""
    fx = fixtures(config)
    return {i: {"seconds": f["ref_seconds"], "workers": f["workers"]} for i, f in sorted(fx.items())}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([t.strip() for t in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        busy = [float(s[6]) for s in self.samples if len(s) > 6 and s[6].replace(".", "").isdigit()]
        loaded = [v for v, b in zip(sm, busy) if b > 0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# The reference (CPU): oracle/_ref, the unmodified reference verifier.

_REF_CHILD = r"""
import json, sys, time
sys.path.insert(0, sys.argv[1])
from oracle.pyoracle import Ref
arch, eps_s, mseed, iseed, image, workers, et = json.loads(sys.argv[2])
ref = Ref()
h = ref.generate(mseed, arch)
dim = 1
for v in ref.layers(h)[0].out_shape: dim *= v
x = ref.random_inputs(iseed, image + 1, dim)[image]
lab = ref.candidate(h, x)
print(json.dumps({"phase": "ready", "label": lab}), flush=True)
r = ref.verify(h, x, ref.double_from_decimal(eps_s), True, max(lab, 0), et, 0, 0, workers, False)
print(json.dumps({"phase": "done", "seconds": r["seconds"], "verified": r["verified"],
                  "margins": [m.hex() for m in r["margins"]], "stats": r["stats"]}), flush=True)
"""


def reference_image(arch, eps_s, mseed, iseed, image, workers, et, limit_s):
    """verify_robustness of one image by the unmodified reference in a child
    process with `workers` threads (AnalysisOptions.workers, the reference's
    intra-call row parallelism). Returns (seconds, finished, result). The
    network build / model generation is outside the timed region (as in
    tools/main.cpp:146-150); a run still going after `limit_s` is stopped and
    its elapsed time returned as a lower bound."""
    p = subprocess.Popen([sys.executable, "-c", _REF_CHILD, ROOT,
                          json.dumps([arch, eps_s, mseed, iseed, image, workers, et])],
                         stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    ready = p.stdout.readline()
    if not ready:
        raise RuntimeError("reference child failed: " + p.stderr.read()[-500:])
    t0 = time.perf_counter()
    try:
        out, _ = p.communicate(timeout=limit_s)
        r = json.loads(out.strip().splitlines()[-1])
        return r["seconds"], True, r
    except subprocess.TimeoutExpired:
        elapsed = time.perf_counter() - t0
        p.kill()
        p.communicate()
        return elapsed, False, None


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    arch, eps_s, mseed, iseed = workload(args.config)
    threads = os.cpu_count() or 1
    et = not args.no_early_term
    from oracle.pyoracle import Ref
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
        return
    # the same images as our arm: step s verifies image s mod pool; latency mode
    # (one image, all host threads as the reference's row workers)
    budget = max(30.0, args.cpu_sample_seconds * 4)
    times, lower, verified, done = [], False, 0, 0
    t_start = time.perf_counter()
    for s in range(args.warmup + args.steps):
        left = budget - (time.perf_counter() - t_start)
        if left <= 1.0:
            break
        sec, finished, r = reference_image(arch, eps_s, mseed, iseed, s % args.pool, threads, et, left)
        if not finished:
            times.append(sec)
            lower = True
            break
        if s >= args.warmup or args.warmup + args.steps == 1:
            times.append(sec)
            done += 1
            verified += int(bool(r["verified"]))
    val = 1000.0 * (statistics.mean(times) if times else float("nan"))
    sample = (f"{done} images verified in full (image s mod {args.pool}), workers={threads}"
              if not lower else
              f"one image (image 0) of {args.config} did not finish within {times[-1]:.0f} s with "
              f"workers={threads}; value = elapsed time, a LOWER BOUND on the reference's ms/image")
    line = {"metric": METRIC, "value": val, "unit": "ms/image", "n_gpus": 0, "steps": len(times),
            "warmup": args.warmup, "ms_per_step": val, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "value_is_lower_bound": lower,
            "config": config_dict(args, arch, eps_s, mseed, iseed, 1),
            "cpu_baseline": {"value": val, "unit": "ms/image", "cores": threads, "kind": "reference",
                             "sample": sample},
            "offline_full_image_reference": offline_reference_seconds(args.config),
            "e2e": {"value": val, "unit": "ms/image", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------


def relaunch_distributed(args):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def ncu_traffic(config):
    """DRAM bytes per launch of the conv kernel from a committed ncu --set full
    capture of this config (profiles/*_ncu_gbc_*<config>*.json), or None."""
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*ncu_gbc*{config}*.json"))):
        try:
            best = (json.load(open(p)), os.path.relpath(p, ROOT))
        except Exception:
            pass
    return best


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    rank, world, local = dist_env()
    if args.gpus > 1 and "RANK" not in os.environ:
        relaunch_distributed(args)
    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2007_10868_b200 as pc

    arch, eps_s, mseed, iseed = workload(args.config)
    eps = float(eps_s)  # correctly rounded, == strtod (decimal.cpp:63-76)
    et = not args.no_early_term
    net = pc.generate(mseed, arch)
    v = pc.Verifier(net, pc.AnalysisOptions(early_term=et, device=local))
    n_in = int(np.prod(net.input_shape))
    steps, warm = args.steps, args.warmup
    X = pc.random_inputs(iseed, args.pool, n_in)
    boxes = [pc.input_box(x, eps, True) for x in X]
    labels = [max(v.candidate(x), 0) for x in X]
    dev = torch.device("cuda", local)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    dboxes = [(torch.from_numpy(b.lo).to(dev), torch.from_numpy(b.hi).to(dev)) for b in boxes]
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return t.tolist()

    # roofline of the conv kernel: one unsharded verification per rank with the
    # walks serialised (one stream, one pipeline), so the CUDA events around
    # each conv launch time that kernel alone; the kernel counts the interval
    # multiply-adds it executes (live cells only)
    flush.fill_(1)
    torch.cuda.synchronize()
    v.set_serial(True)
    r0 = v.test_device(dboxes[0][0].data_ptr(), dboxes[0][1].data_ptr(), labels[0])
    kt = v.last_kernel_timing("conv")
    v.set_serial(False)
    ref_madds = r0[2]["gbc_madds"]
    roof_madds = kt["executed_madds"] or ref_madds
    fma_peak = pc.verifier.fp64_peak(local)

    transport = None
    if world > 1:
        v.enable_sharding()  # native NCCL communicator on an NCCL group
        transport = v.shard_transport

    results = {}
    lat, e2e, launches = [], [], 0
    with ClockSampler(local) as clk:
        for s in range(warm + steps):
            i = s % args.pool
            flush.fill_(s & 0xFF)
            torch.cuda.synchronize()
            barrier()
            ver, mar, st = v.test_device(dboxes[i][0].data_ptr(), dboxes[i][1].data_ptr(), labels[i])
            ms = v.last_timing()["total_ms"]
            if s >= warm:
                lat.append(ms)
                launches += v.last_timing()["launches"]
            results.setdefault(i, (ver, mar, st))
    for s in range(warm + steps):  # e2e: host buffers through pc_net_test
        i = s % args.pool
        flush.fill_(s & 0xFF)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        r = v.test(boxes[i].lo, boxes[i].hi, labels[i])
        t1 = time.perf_counter()
        if s >= warm:
            e2e.append(1000.0 * (t1 - t0))
        assert np.array_equal(r.margins.view(np.int64), results[i][1].view(np.int64))
    lat = max_over_ranks(lat)
    e2e = max_over_ranks(e2e)
    if world > 1:
        v.disable_sharding()

    # replicas: images verified concurrently on every rank (no collective)
    thr = None
    if args.throughput_images > 0:
        n_t = args.throughput_images
        idx = [(rank * n_t + j) % args.pool for j in range(n_t)]
        lo = torch.stack([dboxes[j][0] for j in idx])
        hi = torch.stack([dboxes[j][1] for j in idx])
        lab = np.array([labels[j] for j in idx], dtype=np.int32)
        torch.cuda.synchronize()
        v.test_batch(lo.data_ptr(), hi.data_ptr(), lab, args.concurrency, device_inputs=True)  # warm
        barrier()
        _, _, _, bms = v.test_batch(lo.data_ptr(), hi.data_ptr(), lab, args.concurrency, device_inputs=True)
        bms = max_over_ranks([bms])[0]
        thr = {"value": bms / (n_t * world), "unit": "ms/image", "images": n_t * world,
               "concurrency_per_gpu": args.concurrency, "scaling": "weak"}

    # the fast numeric mode (native directed rounding, sound, not bit-identical;
    # SURVEY.md §8f.3): latency on the same images, verdicts and margins
    # against the reference fixtures reported separately
    fast = None
    if world == 1 and args.fast_steps > 0:
        vf = pc.Verifier(net, pc.AnalysisOptions(early_term=et, device=local, numeric_mode=1))
        fl, fres = [], {}
        for s in range(warm + args.fast_steps):
            i = s % args.pool
            flush.fill_(s & 0xFF)
            torch.cuda.synchronize()
            ver, mar, st = vf.test_device(dboxes[i][0].data_ptr(), dboxes[i][1].data_ptr(), labels[i])
            if s >= warm:
                fl.append(vf.last_timing()["total_ms"])
            fres.setdefault(i, (ver, mar))
        fxs = fixtures(args.config)
        cmp = {}
        for i, (ver, mar) in sorted(fres.items()):
            if i in fxs:
                ref_m = np.array([float.fromhex(h) for h in fxs[i]["margins_hex"]])
                cmp[i] = {"verdict_equal": bool(ver) == fxs[i]["verified"],
                          "max_rel_margin_diff": float(np.max(np.abs(mar - ref_m) / np.maximum(1.0, np.abs(ref_m))))}
        fast = {"mode": "numeric_mode=1: RD/RU FMAs in the conv coefficients, RD/RU chains and concretisations "
                        "(sound, not bit-identical to the reference)",
                "latency_ms_per_image": statistics.mean(fl) if fl else None, "steps": len(fl),
                "verified": f"{sum(int(bool(r[0])) for r in fres.values())}/{len(fres)} distinct images",
                "vs_reference_fixtures": cmp}
        vf.close()

    # in-bench parity against the reference fixtures of the timed images
    fx = fixtures(args.config)
    checked, mismatches = [], []
    for i, (ver, mar, st) in sorted(results.items()):
        if i in fx:
            f = fx[i]
            ok = (labels[i] == f["label"] and bool(ver) == f["verified"]
                  and [m.hex() for m in mar] == f["margins_hex"] and st == f["stats"])
            checked.append(i)
            if not ok:
                mismatches.append(i)
    n_ver = sum(int(bool(r[0])) for r in results.values())

    value = statistics.mean(lat)
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        pass
    peak_tflops = 2.0 * fma_peak / 1e12
    conv_s = kt["ms"] / 1000.0
    achieved_tflops = 4.0 * roof_madds / conv_s / 1e12 if conv_s > 0 else 0.0
    hbm_achieved = kt["bytes"] / conv_s / 1e9 if conv_s > 0 else 0.0
    traffic = ncu_traffic(args.config)
    line = {
        "metric": METRIC, "value": value, "unit": "ms/image", "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": value, "higher_is_better": False,
        "latency_ms_per_image": {"mean": value, "median": statistics.median(lat), "min": min(lat),
                                 "max": max(lat)},
        "throughput_ms_per_image": thr,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, arch, eps_s, mseed, iseed, world),
        "verified": f"{n_ver}/{len(results)} distinct images",
        "parity": {"fixtures": "tests/golden/ref_<config>_img<i>.json (unmodified reference)",
                   "images_checked": checked, "mismatches": mismatches,
                   "all_equal": bool(checked) and not mismatches},
        "sharding_transport": transport,
        "fast_mode": fast,
        "e2e": {"value": statistics.mean(e2e), "unit": "ms/image",
                "h2d_bytes_per_step": 2 * 8 * n_in, "d2h_bytes_per_step": 8 * (net.output_size - 1) + 4},
        "gpu_launches": int(launches),
        "roofline": {
            "kernel": "k_gbc_flat (conv back-substitution coefficients, live cells)", "bound": "fp64",
            "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": achieved_tflops / peak_tflops if peak_tflops else None,
            "traffic": (traffic[0].get("dram_bytes_per_launch") if traffic else None),
            "traffic_launch": (traffic[0] if traffic else None),
            "traffic_source": (traffic[1] if traffic else "no ncu capture committed for this config"),
            "algorithmic": "4 FLOPs per interval multiply-add (lo and hi FMA pair); madds = the ones the "
                           "kernel executes (device-counted: live cells x nonzero terms); time = CUDA events "
                           "around every conv launch of one image with the walks serialised (each launch "
                           "alone on the GPU)",
            "reference_equivalent_tflops": 4.0 * ref_madds / conv_s / 1e12 if conv_s > 0 else None,
            "reference_madds": ref_madds,
            "peak_source": "pc_fp64_peak: DFMA throughput measured live on this GPU (2 FLOPs per FMA)",
            "emulation_note": "bit-exact WidenedFloat64 costs 16 FP64-pipe instructions per interval "
                              "madd (4 algorithmic FLOPs), so frac <= 0.125 at full FP64-pipe use",
            "fp64_pipe_frac": (16.0 * roof_madds / conv_s / fma_peak) if conv_s > 0 else None,
            "launches": kt["launches"], "kernel_ms": kt["ms"], "interval_madds": roof_madds,
            "hbm": {"achieved_gbs": hbm_achieved, "peak_gbs": hbm_peak,
                    "frac": hbm_achieved / hbm_peak if hbm_peak else None,
                    "algorithmic_bytes": kt["bytes"],
                    "bytes_model": "16 B per interval of the rows in and out + 8 B per filter tap, per launch"}},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            sec, finished, r = reference_image(arch, eps_s, mseed, iseed, 0, threads, et,
                                               args.cpu_sample_seconds)
            line["cpu_baseline"] = {
                "value": 1000.0 * sec, "unit": "ms/image", "cores": threads, "kind": "reference",
                "value_is_lower_bound": not finished,
                "sample": (f"image 0 of {args.config}, verify_robustness with workers={threads}"
                           + ("" if finished else f"; stopped after {sec:.0f} s: a LOWER BOUND")),
                "offline_full_image_reference": offline_reference_seconds(args.config)}
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
