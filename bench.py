"""Benchmark: FP64 direct-summation Gauss linking numbers on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload kusari|e4in1|knit] [--impl ours|reference]

Workload (default) = BASELINE configs[2]: the synthetic Kusari-scale chainmail
tube, 14,112 rings x 64 segments, 18,752 links; one step verifies the
"after" model (Appendix B.2 edits) against the "before" certificate.

  value   = segment pairs evaluated per step / device time of one pass of the
            hot path (PLS -> discretize -> Gauss sum -> rounding) with the
            packed model already resident in HBM (CUDA events on the stream
            the library launches on; L2 flushed between steps).
  e2e     = the same metric through the public API: verify(after, before_cert)
            from host CurveModel to VerificationReport, incl. the model upload,
            the canonical-JSON digest (overlapped), the D2H of the results and
            the host diff.  e2e.verify_ms is that wall time per step.
  roofline= the Gauss-sum kernel: algorithmic FLOPs (F_PAIR per segment pair,
            DESIGN.md §4) / kernel time, against the FP64 DFMA peak measured
            live on this GPU by lc_probe_fp64_peak.
--impl reference times the CPU oracle port of the reference path
(oracle/: numpy PLS + discretization, C Gauss sum on all host threads).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gauss-sum segment-pairs/sec (FP64)"
UNIT = "seg-pairs/s"
# Algorithmic FP64 FLOPs per segment pair of the reference formula (direct.py:19-46):
# dynamic 2*DFMA + DMUL + DADD of the GAUSS_REF kernel measured with ncu
# (profiles/r01/SUMMARY.md): 261.8 -> frozen at 262.
F_PAIR = 262.0
# FP64 FLOPs the phase kernel actually executes per segment pair (same ncu count,
# GAUSS_PHASE): the hardware-side view of the roofline next to the algorithmic one.
EXEC_FLOP_PAIR = {"phase": 78.5, "atan": 133.3, "ref": 260.3}
# DRAM bytes (read + write) of one gauss_items_kernel launch from the committed
# `ncu --set full` capture of this workload (profiles/r01/gauss_phase_kusari_raw.csv).
NCU_TRAFFIC = {("kusari", "phase"): (23055616 + 58368, "profiles/r01/gauss_phase_kusari_raw.csv")}
L2_FLUSH_BYTES = 512 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["kusari", "e4in1", "knit"], default="kusari")
    ap.add_argument("--mode", choices=["phase", "atan", "ref"], default=os.environ.get("LINKCERT_GAUSS_MODE", "phase"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def build_workload(name):
    from paper_2106_12655_b200 import generators as gen

    if name == "kusari":
        return ("kusari_tube 14112 rings x 64 seg, 18752 links (BASELINE configs[2]); verify(after, cert(before))",
                gen.kusari_tube(), gen.kusari_tube(after=True))
    if name == "e4in1":
        return ("european_4in1 32x32 rings x 64 seg (BASELINE configs[1]); verify(ring 165 pulled, cert)",
                gen.european_4in1(32, 32), gen.european_4in1(32, 32, moved={165: 3.0}))
    return ("knit_tube 20 courses x 100k seg, W=100 (BASELINE configs[3], 20 of 200 courses)",
            gen.knit_tube(courses=20, n=100_000), gen.knit_tube(courses=20, n=100_000))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active"

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.result = {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        if self.proc is None:
            return False
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 3]
        if not rows:
            return False
        sm = [float(r[0]) for r in rows]
        mx = max(float(r[1]) for r in rows)
        masks = [int(r[3].strip(), 16) for r in rows]
        reasons = set()
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}
        for mk in masks:
            for bit, nm in names.items():
                if mk & bit:
                    reasons.add(nm)
        busy = [s for s, mk in zip(sm, masks) if not mk & 0x1] or sm
        self.result = {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": sorted(reasons),
                       "samples": len(rows)}
        return False


def seg_pairs(pairs, vert_off):
    n = np.diff(vert_off)
    return int(np.sum(n[pairs[:, 0]].astype(np.int64) * n[pairs[:, 1]]))


def cpu_reference_step(model, threads):
    """The oracle port of the reference path on the host: returns (seg_pairs, seconds)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import linkcert_oracle as orc

    coeffs, t, off = model.packed()
    t0 = time.perf_counter()
    pairs = orc.pls(coeffs, t, off)
    verts, voff = orc.discretize(coeffs, t, off, model.xi, pairs)
    orc.evaluate_pairs(verts, voff, pairs, threads)
    return seg_pairs(pairs, voff), time.perf_counter() - t0


def run_reference(args, rank, world):
    if rank != 0:
        return
    desc, _, after = build_workload(args.workload)
    threads = os.cpu_count()
    vals = []
    for k in range(args.warmup + args.steps):
        sp, dt = cpu_reference_step(after, threads)
        if k >= args.warmup:
            vals.append((sp, dt))
    tot = sum(dt for _, dt in vals)
    value = sum(sp for sp, _ in vals) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(vals), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "per step: the full workload; oracle PLS (numpy sweep) + discretize (numpy) + "
                                   f"Gauss sum (C, {threads} threads); the reference itself is numba on 1 effective "
                                   "core (GIL)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ["LINKCERT_GAUSS_MODE"] = args.mode
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_12655_b200 as lc
    from paper_2106_12655_b200 import _native
    from paper_2106_12655_b200.certify import device_step, excluded_keys

    desc, before, after = build_workload(args.workload)
    stream = torch.cuda.current_stream()
    ctx = _native.context(local)
    ctx.set_stream(stream.cuda_stream)
    params = lc.DiscretizationParams()
    cert = lc.compute_linking_matrix(before)          # untimed: the certificate being verified against

    # ---- value: device-resident hot path ------------------------------------
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    from paper_2106_12655_b200.pls import upload
    upload(after, ctx)                                  # what verify() uploads (compact polylines here)
    poly = after.polyline_vertices()
    h2d = sum(a.nbytes for a in (poly if poly is not None else after.packed()))
    ex = excluded_keys(())
    step_ms, gauss_ms, launches = [], [], []
    n_sp = None
    with ClockSampler(local) as clk:
        for k in range(args.warmup + args.steps):
            n0 = _native.launch_count()
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pairs, raw, lk, flags = device_step(ctx, after.xi, ex, params)
            e1.record(stream)
            torch.cuda.synchronize()
            if k >= args.warmup:
                launches.append(_native.launch_count() - n0)
                step_ms.append(e0.elapsed_time(e1))
                gauss_ms.append(ctx.stage_times()["gauss"] if (world == 1 or ctx.last_run_fused())
                                else ctx.gauss_event_ms())
            if n_sp is None:
                _, voff = ctx.get_polylines()
                n_sp = seg_pairs(pairs, voff)
                n_closed = int(voff[-1]) + len(voff) - 1     # closed SoA vertices read by the kernel
    clocks = clk.result
    ms = statistics.mean(step_ms)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = n_sp / (ms * 1e-3)

    # ---- e2e: public API, host model in / report out --------------------------
    e2e_ms = []
    report = None
    for k in range(args.warmup + args.steps):
        flush.zero_()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            report = lc.verify(after, cert)
        torch.cuda.synchronize()
        if k >= args.warmup:
            e2e_ms.append(1e3 * (time.perf_counter() - t0))
    e2e = statistics.mean(e2e_ms)
    # the same call path without the model digest ("with and without the digest")
    from paper_2106_12655_b200.certify import diff_arrays, run_device_pipeline
    nd_ms = []
    for k in range(args.warmup + min(args.steps, 10)):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        snap = after.snapshot()
        p_, r_, l_, f_, _ = run_device_pipeline(after, (), params, snapshot=snap)
        diff_arrays(cert.array, p_, r_, l_, f_, False)
        torch.cuda.synchronize()
        if k >= args.warmup:
            nd_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_nd = statistics.mean(nd_ms)
    if world > 1:
        tt = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = float(tt.item())
    d2h = pairs.nbytes + raw.nbytes + lk.nbytes + flags.nbytes

    if rank != 0:
        dist.destroy_process_group()
        return
    peak, _ = ctx.probe_fp64_peak()
    gk = statistics.mean(gauss_ms)
    achieved = F_PAIR * n_sp / (gk * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": desc, "seg_pairs_per_step": n_sp, "pairs": int(len(pairs)),
                   "gauss_mode": args.mode, "device_path": ["staged", "fused", "fused (CUDA graph replay)"][ctx.last_run_fused()], "l2": f"flushed ({L2_FLUSH_BYTES >> 20} MiB write) between steps",
                   "parallelism": f"items sharded over {world} GPU(s), partials all-gathered" if world > 1 else "1 GPU"},
        "e2e": {"value": n_sp / (e2e * 1e-3), "unit": UNIT, "verify_ms": e2e,
                "verify_ms_without_digest": e2e_nd, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "report": {"status": report.status, "destroyed": report.destroyed,
                                                           "created": report.created, "changed": report.changed}},
        "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                     "frac": achieved / peak,
                     "traffic": NCU_TRAFFIC.get((args.workload, args.mode), (None, None))[0],
                     "kernel": f"gauss_items_kernel<{args.mode.upper()}>",
                     "kernel_ms": gk, "f_pair": F_PAIR,
                     "executed": {"flop_per_pair": EXEC_FLOP_PAIR[args.mode],
                                  "tflops": EXEC_FLOP_PAIR[args.mode] * n_sp / (gk * 1e-3) / 1e12,
                                  "frac": EXEC_FLOP_PAIR[args.mode] * n_sp / (gk * 1e-3) / peak},
                     "algorithmic_bytes": 24 * n_closed,
                     "traffic_source": NCU_TRAFFIC.get((args.workload, args.mode), (None, None))[1],
                     "peak_source": "FP64 DFMA-chain probe measured live on this GPU (MEASURED_PEAKS.json has no FP64)"},
        "stage_ms": ctx.stage_times(),
        "clocks": clocks,
        "gpu_launches": int(sum(launches)),
    }
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count()
        sp, dt = cpu_reference_step(after, threads)
        line["cpu_baseline"] = {"value": sp / dt, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": "one full workload pass: oracle PLS + discretize (numpy) + Gauss sum (C, "
                                          f"{threads} threads) = {dt:.2f} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
