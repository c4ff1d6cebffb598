"""Benchmark: FP64 direct-summation Gauss linking numbers on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload kusari|e4in1|knit] [--impl ours|reference]

Workload (default) = BASELINE configs[2]: the synthetic Kusari-scale chainmail
tube, 14,112 rings x 64 segments, 18,752 links; one step verifies the
"after" model (Appendix B.2 edits) against the "before" certificate.

  value   = segment pairs evaluated per step / device time of one pass of the
            hot path (PLS -> discretize -> Gauss sum -> rounding) with the
            model already resident in HBM (CUDA events on the stream the
            library launches on; L2 flushed between steps); N GPUs: the item
            list is split by cost over the ranks, max over ranks.
  e2e     = the same metric through the public API: verify(model, cert) on a
            FRESH CurveModel every step (built outside the timer from loops
            constructed one by one with LoopGeometry.from_polyline), so the
            model snapshot, the host->device upload, the canonical-JSON digest
            (overlapped), the results' D2H and the host diff are inside.
  roofline= the Gauss-sum kernel: FP64 FLOPs it executes per segment pair
            (ncu count, EXEC_FLOP_PAIR) x pairs / kernel time, against the FP64
            peak measured live on this GPU (max of the DFMA-chain and the FP64
            tensor-core probes).  frac_algorithmic uses the reference formula's
            F_PAIR instead (algebraic sharing pushes it above 1).

--gpus N without torchrun re-launches itself under torch.distributed.run
(one process per GPU, NCCL).
--impl reference runs on the host only and never loads the product library:
the CPU oracle port of the reference path (oracle/: numpy PLS +
discretization, C Gauss sum on all host threads) per step, plus one
as-shipped timing of the reference package itself (baseline/_ref, numba).
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import time
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent

METRIC = "Gauss-sum segment-pairs/sec (FP64)"
UNIT = "seg-pairs/s"
# Algorithmic FP64 FLOPs per segment pair of the reference formula (direct.py:19-46):
# dynamic 2*DFMA + DMUL + DADD of the GAUSS_REF kernel measured with ncu
# (profiles/r01/SUMMARY.md): 261.8 -> frozen at 262.
F_PAIR = 262.0
# FP64 FLOPs the kernels actually execute per segment pair (ncu
# smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on, 2*DFMA+DMUL+DADD;
# profiles/r01/counts_*.csv): the numerator of roofline.frac.
EXEC_FLOP_PAIR = {"phase": 73.54, "atan": 128.28, "ref": 260.25}   # profiles/r02/counts_torus_*.csv
# Hardware counters of the committed `ncu --set full` capture of the fused Gauss kernel on
# this workload: DRAM bytes per launch and FP64-pipe activity.
NCU = {("kusari", "phase"): {"traffic": 22983680, "fp64_pipe_active_pct": 71.1,
                             "source": "profiles/r02/gauss_pairs_kusari_raw.csv"}}
L2_FLUSH_BYTES = 512 << 20
DESC = {
    "kusari": "kusari_tube 14112 rings x 64 seg, 18752 links (BASELINE configs[2]); verify(after, cert(before))",
    "e4in1": "european_4in1 32x32 rings x 64 seg (BASELINE configs[1]); verify(ring 165 pulled, cert)",
    "knit": "knit_tube 20 courses x 100k seg, W=100 (BASELINE configs[3], 20 of 200 courses)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["kusari", "e4in1", "knit"], default="kusari")
    ap.add_argument("--mode", choices=["phase", "atan", "ref"], default=os.environ.get("LINKCERT_GAUSS_MODE", "phase"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-as-shipped", action="store_true", help="reference arm: skip the numba reference timing")
    return ap.parse_args()


def load_workloads():
    """paper_2106_12655_b200/workloads.py by path: numpy only, no package import
    (the reference arm must not load the product library)."""
    spec = importlib.util.spec_from_file_location("lc_workloads", ROOT / "paper_2106_12655_b200" / "workloads.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def workload_arrays(name):
    """(before, after) as (verts, loop_off) pairs of closed polylines."""
    w = load_workloads()
    if name == "kusari":
        return w.kusari_tube_vertices(), w.kusari_tube_vertices(after=True)
    if name == "e4in1":
        return w.european_4in1_vertices(32, 32), w.european_4in1_vertices(32, 32, moved={165: 3.0})
    k = w.knit_tube_vertices(courses=20, n=100_000)
    return k, k


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


def oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import linkcert_oracle as orc

    return orc


def cpu_reference_step(verts, off, threads):
    """The oracle port of the reference path on the host: returns (pairs, seg_pairs, seconds)."""
    orc = oracle()
    coeffs, t, off, xi = orc.polyline_model(verts, off)
    t0 = time.perf_counter()
    pairs = orc.pls(coeffs, t, off)
    v, voff = orc.discretize(coeffs, t, off, xi, pairs)
    orc.evaluate_pairs(v, voff, pairs, threads)
    return pairs, seg_pairs(pairs, voff), time.perf_counter() - t0


def as_shipped_reference(before, after, budget_s=150.0):
    """The reference package itself (baseline/_ref, numba) through its public API
    (SURVEY §8(d) "as shipped"): compute_linking_matrix(before) warms the JIT and
    gives the certificate; then verify(after, cert, threads=cpu_count), best of
    up to 3 within `budget_s`.  None when the install is missing."""
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "linkcert").exists():
        return {"unavailable": "baseline/_ref not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/linkcert_numba_cache")
    sys.path.insert(0, str(ref_dir))
    try:
        import linkcert as ref
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"import failed: {type(exc).__name__}: {exc}"}

    def model(arrs):
        v, off = arrs
        return ref.CurveModel([ref.LoopGeometry.from_polyline(v[off[k]:off[k + 1]]) for k in range(len(off) - 1)])

    threads = os.cpu_count()
    t0 = time.perf_counter()
    mb, ma = model(before), model(after)
    t1 = time.perf_counter()
    cert = ref.compute_linking_matrix(mb, threads=threads)
    t2 = time.perf_counter()
    times, rep = [], None
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        while len(times) < 3 and (not times or time.perf_counter() - t0 + times[-1] < budget_s):
            ts = time.perf_counter()
            rep = ref.verify(ma, cert, threads=threads)
            times.append(time.perf_counter() - ts)
    return {"verify_ms_best": 1e3 * min(times), "verify_ms_all": [1e3 * x for x in times],
            "compute_linking_matrix_ms_first_call": 1e3 * (t2 - t1), "model_build_s": t1 - t0,
            "cores": threads, "effective_cores": 1,
            "note": f"reference package as shipped (numba JIT, warmed by compute_linking_matrix), threads={threads}; "
                    "numba holds the GIL so 1 core is effective",
            "report": {"status": rep.status, "destroyed": rep.destroyed, "created": rep.created,
                       "changed": rep.changed}}


def run_reference(args, rank, world):
    """CPU reference arm (rank 0 only): never imports paper_2106_12655_b200."""
    if rank != 0:
        return
    before, after = workload_arrays(args.workload)
    threads = os.cpu_count()
    orc = oracle()
    orc.lib()
    # warm-up (untimed): page in the arrays and the C library on a sample
    for _ in range(args.warmup):
        coeffs, t, off, xi = orc.polyline_model(*after)
        orc.evaluate_pairs(after[0], after[1], orc.pls(coeffs, t, off)[:64], threads)
    vals, pairs = [], None
    for _ in range(args.steps):
        pairs, sp, dt = cpu_reference_step(*after, threads)
        vals.append((sp, dt))
    tot = sum(dt for _, dt in vals)
    n_sp = vals[0][0]
    value = sum(sp for sp, _ in vals) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(vals), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": DESC[args.workload], "seg_pairs_per_step": n_sp, "pairs": int(len(pairs))},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": "per step: the full workload (one verify's PLS + discretize + Gauss sums); oracle "
                                   f"PLS (numpy sweep) + discretize (numpy) + Gauss sum (C, {threads} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_as_shipped:
        ship = as_shipped_reference(before, after)
        line["as_shipped"] = ship
        if "verify_ms_best" in ship:
            line["as_shipped"]["value"] = n_sp / (ship["verify_ms_best"] * 1e-3)
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args):
    """--gpus N (N > 1) without WORLD_SIZE: one process per GPU via torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    if os.environ.get("LINKCERT_BENCH_DRY_RUN") == "1":     # tests: show the command only
        print(json.dumps({"relaunch": cmd}))
        return 0
    return subprocess.call(cmd)


def fresh_loops(arrs):
    """Loops built one by one (separate arrays), as a user's loader would."""
    import paper_2106_12655_b200 as lc

    v, off = arrs
    return [lc.LoopGeometry.from_polyline(v[off[k]:off[k + 1]]) for k in range(len(off) - 1)]


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_under_torchrun(args)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    os.environ["LINKCERT_GAUSS_MODE"] = args.mode

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2106_12655_b200 as lc
    from paper_2106_12655_b200 import _native
    from paper_2106_12655_b200.certify import device_step, diff_arrays, excluded_keys, run_device_pipeline

    before_a, after_a = workload_arrays(args.workload)
    before = lc.CurveModel.from_polyline_arrays(*before_a)
    after = lc.CurveModel.from_polyline_arrays(*after_a)
    stream = torch.cuda.current_stream()
    ctx = _native.context(local)
    ctx.set_stream(stream.cuda_stream)
    params = lc.DiscretizationParams()
    cert = lc.compute_linking_matrix(before)          # untimed: the certificate being verified against

    # ---- value: device-resident hot path ------------------------------------
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    from paper_2106_12655_b200.pls import upload
    upload(after, ctx)                                  # resident model (what verify uploads)
    ex = excluded_keys(())
    step_ms, gauss_ms, launches, stages = [], [], [], []
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
                st = ctx.stage_times()
                stages.append(st)
                gauss_ms.append(st["gauss"] if (world == 1 or ctx.last_run_fused())
                                else ctx.gauss_event_ms())
            if n_sp is None:
                _, voff = ctx.get_polylines()
                n_sp = seg_pairs(pairs, voff)
                n_closed = int(voff[-1]) + len(voff) - 1     # closed SoA vertices read by the kernel
    clocks = clk.result
    # stage breakdown (diagnostic, after the timed region): a few more steps with every
    # stage event recorded (the timed steps record only the Gauss stage's two events)
    detail = []
    for k in range(6):
        flush.zero_()
        torch.cuda.synchronize()
        device_step(ctx, after.xi, ex, params, timings={})   # (a timings request turns stage detail on)
        if k >= 2:
            detail.append(ctx.stage_times())
    ms = statistics.mean(step_ms)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = n_sp / (ms * 1e-3)

    # ---- e2e: public API, a fresh host model in / report out every step --------
    loops = fresh_loops(after_a)                        # separately built loops (outside the timer)

    def timed_verify(model_of_step, steps):
        out, rep = [], None
        for k in range(args.warmup + steps):
            m = model_of_step()                         # fresh CurveModel: nothing cached
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                rep = lc.verify(m, cert)
            torch.cuda.synchronize()
            if k >= args.warmup:
                out.append(1e3 * (time.perf_counter() - t0))
        return statistics.mean(out), rep

    e2e, report = timed_verify(lambda: lc.CurveModel(list(loops), xi=after.xi), args.steps)
    e2e_warm, _ = timed_verify(lambda: after, min(args.steps, 10))
    # the same call path without the model digest ("with and without the digest")
    nd_ms = []
    for k in range(args.warmup + min(args.steps, 10)):
        m = lc.CurveModel(list(loops), xi=after.xi)
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p_, r_, l_, f_, _ = run_device_pipeline(m, (), params, snapshot=m.snapshot())
        diff_arrays(cert.array, p_, r_, l_, f_, False)
        torch.cuda.synchronize()
        if k >= args.warmup:
            nd_ms.append(1e3 * (time.perf_counter() - t0))
    e2e_nd = statistics.mean(nd_ms)
    if world > 1:
        tt = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = float(tt.item())
    h2d = 24 * int(after_a[1][-1]) + 8 * len(after_a[1])         # vertices + loop offsets
    d2h = pairs.nbytes + raw.nbytes + lk.nbytes + flags.nbytes

    if rank != 0:
        dist.destroy_process_group()
        return 0
    # the same arithmetic kernel alone on this workload's work items (no concurrent branches)
    ctx_mode = _native.GAUSS_MODES[args.mode]
    n_items = ctx.prepare_gauss(ctx_mode)
    solo = []
    for _ in range(5):
        ctx.gauss_run(ctx_mode, 0, n_items)
        solo.append(ctx.gauss_event_ms())
    gk_solo = min(solo[1:])
    peak_dfma, _ = ctx.probe_fp64_peak()
    peak_dmma, _ = ctx.probe_fp64_peak(dmma=True)
    peak = max(peak_dfma, peak_dmma)
    gk = statistics.mean(gauss_ms)
    rate = n_sp / (gk * 1e-3)
    executed = EXEC_FLOP_PAIR[args.mode] * rate
    ncu = NCU.get((args.workload, args.mode), {})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": DESC[args.workload], "seg_pairs_per_step": n_sp, "pairs": int(len(pairs))},
        "run": {"gauss_mode": args.mode,
                "device_path": ["staged", "fused", "fused (CUDA graph replay)"][ctx.last_run_fused()],
                "l2": f"flushed ({L2_FLUSH_BYTES >> 20} MiB write) between steps",
                "parallelism": (f"{world} GPUs: work items split by cost, partials exchanged with NCCL" if world > 1
                                else "1 GPU")},
        "e2e": {"value": n_sp / (e2e * 1e-3), "unit": UNIT, "verify_ms": e2e,
                "model": "fresh CurveModel every step over loops built one by one with LoopGeometry.from_polyline "
                         "(outside the timer); verify() snapshots, uploads and hashes it",
                "verify_ms_warm_model": e2e_warm,
                "verify_ms_without_digest": e2e_nd, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "report": {"status": report.status, "destroyed": report.destroyed,
                                                           "created": report.created, "changed": report.changed}},
        "roofline": {"bound": "fp64", "achieved": executed / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                     "frac": executed / peak, "traffic": ncu.get("traffic"),
                     "kernel": f"gauss_pairs_kernel<{args.mode.upper()}> (fused step, beside the checks branch)",
                     "kernel_ms": gk,
                     "flop_per_pair_executed": EXEC_FLOP_PAIR[args.mode],
                     "fp64_pipe_active_pct_ncu": ncu.get("fp64_pipe_active_pct"),
                     "ncu_source": ncu.get("source"),
                     "frac_algorithmic": F_PAIR * rate / peak, "f_pair_algorithmic": F_PAIR,
                     "standalone": {"kernel": f"gauss_items_kernel<{args.mode.upper()}> alone on the same items",
                                    "kernel_ms": gk_solo, "seg_pairs_per_s": n_sp / (gk_solo * 1e-3),
                                    "frac": EXEC_FLOP_PAIR[args.mode] * n_sp / (gk_solo * 1e-3) / peak},
                     "algorithmic_bytes": 24 * n_closed,
                     "peak_probes_tflops": {"dfma": peak_dfma / 1e12, "dmma": peak_dmma / 1e12},
                     "peak_source": "max(FP64 DFMA-chain, FP64 tensor-core MMA) probes measured live on this GPU "
                                    "(MEASURED_PEAKS.json has no FP64 entry)"},
        # the library's stage events (median per stage) of 4 steps run after the timed
        # region with every stage event on; the timed steps time the Gauss stage only
        "stage_ms": {k: (round(statistics.median(x[k] for x in detail), 4) if detail[0][k] is not None else None)
                     for k in detail[0]},
        "stage_ms_gauss_timed": round(statistics.median(x["gauss"] for x in stages), 4),
        "clocks": clocks,
        "gpu_launches": int(sum(launches)),
    }
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count()
        _, sp, dt = cpu_reference_step(*after_a, threads)
        line["cpu_baseline"] = {"value": sp / dt, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": "one full workload pass: oracle PLS + discretize (numpy) + Gauss sum (C, "
                                          f"{threads} threads) = {dt:.2f} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
