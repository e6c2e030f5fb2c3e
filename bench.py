#!/usr/bin/env python
"""BSGD-TV epoch throughput on B200 (BASELINE.json metric; headline workload configs[3]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one BSGD-TV epoch (Algorithm 1, `bsgd_tv_iteration`,
`solvers.py:259-341`, alpha = gamma = 1, monitor off) of configs[3]: 2-D
parallel-beam CT, 1024 x 1024 image, 1440 angles x 1449 bins, Siddon float32
CSR (1.92e9 nonzeros, int32 indices), M = N = 8 blocks, lambda = 0.01, TV prox
by dual FGP with at most 20 iterations (tol 1e-5), mu = 0.9 / (2 u_max) read
from tests/golden/config_mu.json (computed once, identical in both arms).  The
largest configuration that fits one GPU and the one BASELINE.json scales over
1/2/4/8 GPUs.  Inputs are seeded synthetic data of exactly that definition
(problems.py); A and A^T (15.4 GB each) exceed the 126 MB L2, so every epoch
streams from HBM with no explicit flush.

Arms:
  ours       value: K epochs with the state resident in HBM (CUDA-graph replay),
             device time from CUDA events, max over ranks.
             phases / roofline: K eager epochs with CUDA events recorded between
             the epoch's kernels on the launching stream (bsgd_plan_timing): the
             in-epoch K1 / K2 / prox times, the dominant kernel's achieved GB/s.
             e2e: K epochs through the drop-in `bsgd_tv_iteration` with HOST numpy
             state (x, r uploaded before and downloaded after every epoch).
             cpu_baseline: the CPU oracle port (C + OpenMP, all host threads) on a
             bounded sample of epochs of the same configs[3] system.
             secondary: configs[1], [2], [4] (device-resident epochs/s, products).
  reference  the reference package itself (baseline/_ref, `bsgdtv`, unmodified)
             through its own bsgd_tv_iteration with a ThreadPoolExecutor over all
             host cores, on the same A, y, mu; falls back to the oracle port when
             baseline/_ref is absent.  Rank 0 only.
Multi-GPU (torchrun, N > 1): configs[3] row slabs generated on each rank's GPU,
see paper_1812_01307_b200/parallel.py.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "BSGD-TV epochs/s + achieved HBM GB/s (SpMV, TV-prox) at 1/2/4/8 B200"
HEADLINE = 3
MU_TABLE = os.path.join(REPO, "tests", "golden", "config_mu.json")
REF_DIR = os.path.join(REPO, "baseline", "_ref")

WORKLOADS = {
    1: "configs[1]: pure BSGD least squares (lambda=0), A 2,000,000 x 500,000, 32 nnz/row, float32 values, "
       "M=N=8, monitor off",
    2: "configs[2]: 2D parallel-beam CT 512x512, 720 angles x 727 bins, Siddon float32 CSR, lambda=0.01, "
       "FGP<=20 (tol 1e-5), M=N=8, monitor off",
    3: "configs[3]: 2D parallel-beam CT 1024x1024, 1440 angles x 1449 bins, Siddon float32 CSR (int32 indices), "
       "lambda=0.01, FGP<=20 (tol 1e-5), M=N=8, monitor off",
    4: "configs[4]: 3D slice-stacked parallel-beam CT 256^3, 360 angles x 256 rows x 363 bins, block-diagonal "
       "A = A2 (x) I_256 (only the 2-D slice matrix A2 is stored), isotropic 3D TV FGP<=10, lambda=0.01, "
       "M=N=16, monitor off",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def mu_for(index):
    """(mu, u_max) recorded once for configs[index] (tools/make_mu.py)."""
    with open(MU_TABLE) as fh:
        e = json.load(fh)[f"configs[{index}]"]
    return float(e["mu"]), float(e["u_max"])


def config_dict(index, nnz, mu, u_max):
    """The workload definition: identical in both arms (execution details live outside)."""
    d = {"workload": WORKLOADS[index], "nnz": int(nnz), "mu": mu, "u_max": u_max,
         "mu_source": "tests/golden/config_mu.json (50 power iterations, computed once, shared by both arms)",
         "monitor_decrease": False, "alpha": 1.0, "gamma": 1.0,
         "matrix_dtype": "f32 values, int32 indices, int64 row pointers", "vector_dtype": "f64",
         "seeds": {"phantom": 0, "noise": 1, "solver": 0} if index != 1 else
                  {"matrix": 2, "x_true": 0, "solver": 0}}
    if index == 3:
        d.update({"image": "1024x1024", "rays": 1440 * 1449, "blocks": "8x8", "lam": 0.01, "fgp_max_iters": 20,
                  "fgp_tol": 1e-5, "l2": "no flush needed: A and A^T (15.4 GB each) exceed the 126 MB L2 every epoch"})
    return d


# --- CPU (oracle port) ---------------------------------------------------------

def oracle_epochs(csr, y, blocks, mu, lam, max_inner, tol, hw, warmup, steps, budget_s):
    """Time oracle epochs (C restatement + numpy, all host threads). Returns (epochs/s, info)."""
    from oracle import oracle as orc
    threads = orc.default_threads()
    oop = orc.OracleOperator(csr, blocks, blocks, threads=threads)
    prm = orc.Params(mu=mu, lam=lam, epochs=10 ** 9, max_inner_iters=max_inner, tol=tol, monitor_decrease=False)
    st = orc.init_state(oop, y, prm)
    perm = np.arange(csr.shape[1]) if lam > 0 else None
    for _ in range(warmup):
        orc.epoch(st, oop, y, prm, perm, hw)
    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        orc.epoch(st, oop, y, prm, perm, hw)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    total = sum(times)
    return len(times) / total, {"cores": threads, "epochs_timed": len(times), "seconds": round(total, 3)}


# --- clocks ------------------------------------------------------------------------

class Clocks:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path or not os.path.exists(self.path):
            return None
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --- GPU arm ---------------------------------------------------------------------------

def dist_info():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def csr_bytes(nnz, rows, cols):
    """SURVEY.md §8(d) byte model of the two products inside an epoch (float32
    values + int32 indices, int64 row pointers, float64 vectors):
    K1 (lookahead, EpiResid): A stream, pointers, x once, y in, r out;
    K2 (EpiStep with the prox on): A^T stream, pointers, r once, x_k in, g and
    the prox input image b = x_k + mu g out."""
    k1 = nnz * 8 + (rows + 1) * 8 + cols * 8 + 2 * rows * 8
    k2 = nnz * 8 + (cols + 1) * 8 + rows * 8 + 3 * cols * 8
    return k1, k2


def prox_bytes(npx, dim, iters):
    """Fused-schedule prox bytes: per FGP iteration the candidate
    (read q, b; write c) and the dual value + momentum commit (read c, p, b;
    write q): (5 dim + 2) fields of 8 bytes, plus ~10 fields of setup/finalize."""
    return 8 * npx * ((5 * dim + 2) * iters + 10)


def time_events(fn, reps):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_ours(args):
    import torch
    from paper_1812_01307_b200 import problems, solvers, tv

    world, rank, local = dist_info()
    if world > 1 or args.force_dist:
        return run_multi(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    t0 = time.time()
    d = problems.config_device(HEADLINE)
    op = d.op
    torch.cuda.synchronize()
    rows, cols = op.shape
    nnz = int(op.nnz)
    log(f"[bench] configs[3] on device in {time.time() - t0:.1f}s: {op.shape}, nnz={nnz}, "
        f"kernels {op.kernel_info()}")
    mu, u_max = mu_for(HEADLINE)
    lay = d.layout()
    cfg = solvers.SolverConfig(mu=mu, lam=d.lam, epochs=10 ** 9, prox=tv.ProxSettings(d.max_inner_iters, 1e-5),
                               monitor_decrease=False)
    steps = max(2, args.steps // 2 * 2)

    # ---- standalone prox at the FGP cap (non-converging tolerance): a kernel timed alone,
    #      before the long product kernels put the GPU under its power cap (the same
    #      kernel measures ~14% slower right after them) ----
    img = torch.rand(d.height, d.width, dtype=torch.float64, device=dev)
    pst = tv.ProxSettings(d.max_inner_iters, 1e-300)
    for _ in range(5):   # a sub-millisecond kernel: warm the clocks before the timed repetitions
        tv.tv_prox(img, 0.05, pst)
    pms = time_events(lambda: tv.tv_prox(img, 0.05, pst), 20)
    pb = prox_bytes(d.height * d.width, 2, d.max_inner_iters)
    peak0, _ = peaks()
    prox_alone = {"image": f"{d.height}x{d.width}", "iterations": d.max_inner_iters, "ms": round(pms, 4),
                  "algorithmic_bytes": pb, "gbs": round(pb / (pms * 1e6), 1),
                  "frac": round(pb / (pms * 1e6) / peak0, 4),
                  "note": "fields are L2-resident at 1024^2 (8 MB each); timed alone before the epochs"}
    del img

    # ---- value: resident state, graph replay ----
    st = solvers.init_bsgd_state(op, d.y, cfg)
    st._ensure_history(4 * steps + args.warmup + 16)
    for _ in range(args.warmup):
        solvers.bsgd_tv_iteration(st, op, d.y, cfg, layout=lay)
    runner = solvers._GraphRunner(st, cfg, lay, st._y, 2)
    assert runner.capture(False), "CUDA graph capture failed"
    runner.replay()  # warm the graph itself
    torch.cuda.synchronize()
    row0 = st._rows_used + 2
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        start.record()
        for _ in range(steps // 2):
            runner.replay()
        stop.record()
        torch.cuda.synchronize()
    st._rows_used += 2 + steps
    ms_per_step = start.elapsed_time(stop) / steps
    value = 1000.0 / ms_per_step
    clocks = clk.summary()
    hist = st._hist[row0:row0 + steps].cpu().numpy()
    fgp_iters = float(np.mean(hist[:, 5]))
    log(f"[bench] resident: {ms_per_step:.4f} ms/epoch -> {value:.2f} epochs/s (mean FGP iterations {fgp_iters:.2f})")

    # ---- phases: the same epochs eagerly, CUDA events between the kernels ----
    op.set_phase_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        solvers.bsgd_tv_iteration(st, op, st._y, cfg, layout=lay)
    e1.record()
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / steps
    ph, n_ep = op.phase_timing()
    op.set_phase_timing(False)
    ph = {k: v / max(n_ep, 1) for k, v in ph.items()}
    b1, b2 = csr_bytes(nnz, rows, cols)
    peak, peak_src = peaks()
    kinfo = op.kernel_info()
    kernels = {"k1_forward_lookahead": {"kernel": f"{kinfo['forward']} CSR ({kinfo['forward_lanes']} lanes per ray, gather order "
                                                  f"{kinfo['forward_order']}), EpiResid (r = y - A x)",
                                        "ms": round(ph["k1_lookahead"], 4), "bytes": b1,
                                        "gbs": round(b1 / (ph["k1_lookahead"] * 1e6), 1)},
               "k2_transposed_step": {"kernel": f"{kinfo['transposed']} A^T ({kinfo['transposed_lanes']} lanes per pixel, gather order "
                                                f"{kinfo.get('transposed_order', 'native')}), EpiStep (g = 2 A^T r, b = x + mu g)",
                                      "ms": round(ph["k2_step"], 4), "bytes": b2,
                                      "gbs": round(b2 / (ph["k2_step"] * 1e6), 1)},
               "k3_tv_prox": {"kernel": "fgp2_rows_kernel (row walk, one grid barrier per FGP iteration)",
                              "ms": round(ph["prox"], 4), "mean_fgp_iterations": round(fgp_iters, 2)},
               "tail": {"ms": round(ph["tail"], 4)}}
    for k in kernels.values():
        if "gbs" in k:
            k["frac"] = round(k["gbs"] / peak, 4)
    dom_key = "k1_forward_lookahead" if ph["k1_lookahead"] >= ph["k2_step"] else "k2_transposed_step"
    dom = kernels[dom_key]
    phase_sum = sum(ph.values())
    traffic = None
    prof = os.path.join(REPO, "profiles", "roofline_traffic.json")
    if os.path.exists(prof):
        with open(prof) as fh:
            traffic = json.load(fh).get("configs[3]", {}).get(dom_key, {}).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": f"{dom_key}: {dom['kernel']}", "achieved": dom["gbs"], "peak": peak,
                "unit": "GB/s", "frac": round(dom["gbs"] / peak, 4), "traffic": traffic,
                "algorithmic_bytes": dom["bytes"], "launch_ms": dom["ms"], "peak_source": peak_src,
                "note": "achieved = SURVEY 8(d)'s algorithmic bytes (8 B per float32 nonzero + vectors) / launch time; "
                        "the blocked stream stores 6.125 B per nonzero (16-bit offset indices), so the DRAM traffic "
                        "(ncu, `traffic`) is ~0.78 of the algorithmic bytes and the actual DRAM rate is traffic / "
                        "launch time",
                "timing": "CUDA events between the epoch's kernels on the launching stream, averaged over the "
                          f"{n_ep} eager epochs after the graph-timed ones",
                "kernels": kernels,
                "epoch_eager_ms": round(eager_ms, 4), "phase_sum_ms": round(phase_sum, 4),
                "phase_sum_over_epoch": round(phase_sum / eager_ms, 4),
                "epoch_algorithmic_gbs": round((b1 + b2) / (ms_per_step * 1e6), 1)}
    if traffic:
        roofline["dram_gbs_actual"] = round(traffic / (dom["ms"] * 1e6), 1)
        roofline["dram_frac_actual"] = round(traffic / (dom["ms"] * 1e6) / peak, 4)
    log(f"[bench] phases (ms): " + ", ".join(f"{k} {v:.4f}" for k, v in ph.items()) +
        f" | sum {phase_sum:.4f} vs eager epoch {eager_ms:.4f}")

    roofline["tv_prox_standalone"] = prox_alone

    # ---- e2e: host numpy state through the drop-in API ----
    st2 = solvers.init_bsgd_state(op, d.y, cfg)
    st2._ensure_history(4 * steps + 16)
    hx = np.zeros(cols)
    hr = np.asarray(d.y, dtype=np.float64).copy()
    for _ in range(2):
        st2.x, st2.r_vec = hx, hr
        solvers.bsgd_tv_iteration(st2, op, d.y, cfg, layout=lay)
        hx, hr = st2.x, st2.r_vec
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        st2.x, st2.r_vec = hx, hr
        solvers.bsgd_tv_iteration(st2, op, d.y, cfg, layout=lay)
        hx, hr = st2.x, st2.r_vec
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / steps
    e2e = {"value": round(1.0 / e2e_s, 3), "unit": "epochs/s", "h2d_bytes_per_step": (rows + cols) * 8,
           "d2h_bytes_per_step": (rows + cols) * 8,
           "how": "bsgd_tv_iteration with numpy x and r_vec assigned before and read back after every epoch"}
    log(f"[bench] e2e host-state: {e2e_s * 1e3:.3f} ms/epoch")
    del st2

    # ---- CPU baseline on a bounded sample of the same system: the reference package
    #      itself (baseline/_ref) when installed, and the oracle port beside it ----
    cpu = None
    if not args.no_cpu:
        t0 = time.time()
        csr = op.tocsr()
        op._csr = None
        log(f"[bench] host CSR copy {time.time() - t0:.1f}s")
        v, info = oracle_epochs(csr, d.y, 8, mu, d.lam, d.max_inner_iters, 1e-5, (d.height, d.width),
                                warmup=1, steps=max(2, args.cpu_epochs), budget_s=args.cpu_budget)
        port = {"value": round(v, 4), "unit": "epochs/s", "cores": info["cores"], "kind": "port",
                "sample": f"{info['epochs_timed']} epochs ({info['seconds']} s) of the same configs[3] system "
                          f"(same A, y, mu) after 1 warm-up epoch; oracle/ C restatement of scipy csr/csc_matvec "
                          f"+ numpy epilogue and prox, OpenMP over block pairs"}
        log(f"[bench] cpu oracle port: {v:.4f} epochs/s on {info['cores']} threads")
        ref = None if args.no_ref_baseline else reference_epochs(csr, d.y, mu, {
            "height": d.height, "width": d.width, "lam": d.lam, "max_inner_iters": d.max_inner_iters},
            workers=os.cpu_count() or 1, warmup=1, steps=max(2, args.cpu_epochs), budget=args.cpu_budget)
        del csr
        if ref is not None:
            cpu = {"value": round(ref["value"], 4), "unit": "epochs/s", "cores": ref["workers"], "kind": "reference",
                   "sample": f"{ref['epochs']} epochs ({ref['seconds']:.1f} s) of the same configs[3] system "
                             f"(same A, y, mu) after 1 warm-up epoch through the reference package's own "
                             f"bsgd_tv_iteration (baseline/_ref), ThreadPoolExecutor({ref['workers']}), monitor off",
                   "host": host_info(), "port": port}
            log(f"[bench] cpu reference: {ref['value']:.4f} epochs/s on {ref['workers']} threads")
        else:
            cpu = port

    # the r permute into K2's tiled gather order, K2 (blocked A^T + step), prox (1 cooperative
    # row-walk kernel), the x permute into K1's tiled gather order, K1 lookahead, tail
    ki = op.kernel_info()
    launches = 4 + (ki["forward_order"] != "native") + (ki.get("transposed_order", "native") != "native")
    secondary = None
    del st, runner, op, d
    torch.cuda.empty_cache()
    if not args.no_secondary:
        secondary = {}
        for idx in (1, 2, 4):
            try:
                secondary[f"configs[{idx}]"] = run_secondary(args, idx)
            except Exception as exc:  # keep the headline line even if a secondary run fails
                secondary[f"configs[{idx}]"] = {"error": repr(exc)[:300]}
            torch.cuda.empty_cache()

    out = {"metric": METRIC, "value": round(value, 3), "unit": "epochs/s", "n_gpus": 1, "steps": steps,
           "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded configs[3] phantom, projector and noise; problems.py)",
           "config": config_dict(HEADLINE, nnz, mu, u_max), "parallelism": "single GPU",
           "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
           "gpu_launches": launches * steps, "clocks": clocks, "secondary": secondary}
    print(json.dumps(out), flush=True)


def run_secondary(args, index):
    """configs[index]: device-resident epochs/s (graph replay) and the in-epoch kernel times."""
    import torch
    from paper_1812_01307_b200 import blockops, problems, solvers, tv
    t0 = time.time()
    if index == 1:
        h = problems.config(1)
        op = blockops.BlockOperator(h.matrix, blockops.make_partition(*h.matrix.shape, 8, 8))
        y, lam, lay, inner = h.y, 0.0, None, 20
        shape = None
        del h
    else:
        d = problems.config_device(index)
        op, y, lam, lay, inner = d.op, d.y, d.lam, d.layout(), d.max_inner_iters
        shape = (d.depth, d.height, d.width) if d.depth > 1 else (d.height, d.width)
        del d
    torch.cuda.synchronize()
    log(f"[bench] configs[{index}] ready in {time.time() - t0:.1f}s: {op.shape}, nnz={op.nnz}")
    mu, _ = mu_for(index)
    cfg = solvers.SolverConfig(mu=mu, lam=lam, epochs=10 ** 9, prox=tv.ProxSettings(inner, 1e-5),
                               monitor_decrease=False)
    st = solvers.init_bsgd_state(op, y, cfg)
    steps = max(4, min(args.steps, 20)) // 2 * 2
    st._ensure_history(3 * steps + 16)
    for _ in range(3):
        solvers.bsgd_tv_iteration(st, op, y, cfg, layout=lay)
    runner = solvers._GraphRunner(st, cfg, lay, st._y, 2)
    assert runner.capture(False)
    runner.replay()
    torch.cuda.synchronize()
    row0 = st._rows_used + 2
    ms = time_events(runner.replay, steps // 2) / 2
    st._rows_used += 2 + steps
    hist = st._hist[row0:row0 + steps].cpu().numpy()
    op.set_phase_timing(True)
    for _ in range(steps):
        solvers.bsgd_tv_iteration(st, op, st._y, cfg, layout=lay)
    ph, n = op.phase_timing()
    op.set_phase_timing(False)
    ph = {k: round(v / max(n, 1), 4) for k, v in ph.items()}
    rows, cols = op.shape
    out = {"workload": WORKLOADS[index], "nnz": int(op.nnz), "epochs_per_s": round(1000.0 / ms, 2),
           "ms_per_epoch": round(ms, 4), "phases_ms": ph, "kernels": op.kernel_info(),
           "mean_fgp_iterations": round(float(np.mean(hist[:, 5])), 2) if lam > 0 else 0}
    peak, _ = peaks()
    if op.depth == 1:
        b1, b2 = csr_bytes(int(op.nnz), rows, cols)
        if lam == 0:
            b2 -= cols * 8  # no prox image: g and x_next out
        out["k1_gbs"] = round(b1 / (ph["k1_lookahead"] * 1e6), 1)
        out["k2_gbs"] = round(b2 / (ph["k2_step"] * 1e6), 1)
        out["k1_frac"] = round(out["k1_gbs"] / peak, 4)
        out["k2_frac"] = round(out["k2_gbs"] / peak, 4)
    if index == 1:
        # random 8-byte gathers, one per nonzero: capped by the L1 tag stage at ~1
        # distinct sector per SM per cycle (profiles/r01_gather_microbench.md)
        clk = 1965.0
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
        floor = op.nnz / (sms * clk * 1e6) * 1e3
        out["gather_ceiling"] = {"floor_ms": round(floor, 4), "frac_k1": round(floor / ph["k1_lookahead"], 3),
                                 "frac_k2": round(floor / ph["k2_step"], 3)}
    if shape is not None:
        img = torch.rand(*shape, dtype=torch.float64, device="cuda")
        pst = tv.ProxSettings(inner, 1e-300)
        for _ in range(3):
            tv.tv_prox(img, 0.05, pst)
        pms = time_events(lambda: tv.tv_prox(img, 0.05, pst), 10)
        npx = int(np.prod(shape))
        pb = prox_bytes(npx, len(shape), inner)
        if npx >= (1 << 21):
            pb -= 8 * npx * 2 * len(shape)   # split prox: the first iteration reads p = q = 0 as literals
        out["tv_prox_standalone"] = {"shape": "x".join(map(str, shape)), "iterations": inner, "ms": round(pms, 4),
                                     "gbs": round(pb / (pms * 1e6), 1), "frac": round(pb / (pms * 1e6) / peak, 4)}
    if op.depth > 1:
        # A = A2 (x) I_D (slice-stacked, interleaved order): A2 is stored once, so the
        # CSR byte model does not apply.  Per product the HBM bytes are the stored
        # tile records (8 B per stored entry) plus the vectors (input once, output
        # once, y for K1); every logical nonzero is one float64 multiply and add whose
        # vector operand comes from shared memory (tile-staged) -- the products are
        # issue / shared-memory bound, far from either HBM or L2 bandwidth.
        D = op.depth
        snnz = op.nnz // D
        hbm1 = snnz * 8 + cols * 8 + 2 * rows * 8
        hbm2 = snnz * 8 + rows * 8 + 3 * cols * 8
        out["operator_note"] = (f"A = A2 (x) I_{D}: {snnz} stored nonzeros of the 2-D slice matrix applied to {D} "
                                f"slices each ({op.nnz} logical nonzeros); not the ~1e10-nonzero block-diagonal CSR "
                                f"(that operator runs through the general path, tests/test_gpu_fullsize.py z-slab test)")
        out["byte_model"] = {
            "k1_hbm_bytes": hbm1, "k2_hbm_bytes": hbm2,
            "k1_hbm_gbs": round(hbm1 / (ph["k1_lookahead"] * 1e6), 1),
            "k2_hbm_gbs": round(hbm2 / (ph["k2_step"] * 1e6), 1),
            "k1_hbm_frac": round(hbm1 / (ph["k1_lookahead"] * 1e6) / peak, 4),
            "k2_hbm_frac": round(hbm2 / (ph["k2_step"] * 1e6) / peak, 4),
            "logical_fp64_mul_add_per_product": int(op.nnz),
            "k1_g_mul_add_per_s": round(op.nnz / (ph["k1_lookahead"] * 1e6), 1),
            "k2_g_mul_add_per_s": round(op.nnz / (ph["k2_step"] * 1e6), 1),
            "bound": "issue / shared-memory (tile-staged vector rows), profiles/r01_c5.md"}
    del st, runner, op
    return out


def run_multi(args):
    """N > 1 (torchrun, one rank per GPU): configs[3] by row slabs, each rank
    generating only its own rays on its GPU (parallel.CudaShard.parallel_beam),
    one NCCL all-reduce of g (+ ||r||^2) per epoch.  Same JSON contract as the
    single-GPU line; timing = max over ranks of CUDA-event time."""
    import torch
    import torch.distributed as dist
    from paper_1812_01307_b200 import parallel, tv
    from paper_1812_01307_b200.solvers import SolverConfig

    world, rank, local = dist_info()
    if "RANK" not in os.environ:   # --force-dist outside torchrun: a world of one
        os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"})
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
    # one rank per GPU; the modulo only matters for the functional gloo check of
    # the N > 1 code path with every rank on one GPU (--dist-backend gloo)
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.dist_backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(args.dist_backend)
    if args.multi_config == 4:
        return run_multi_slices(args, world, rank, local, dev)
    shard, y_full, meta = parallel.ct_row_slab_shard(HEADLINE, rank, world, device=dev)
    mu, u_max = mu_for(HEADLINE)
    cfg = SolverConfig(mu=mu, lam=meta["lam"], epochs=10 ** 9, prox=tv.ProxSettings(meta["max_inner_iters"], 1e-5),
                       monitor_decrease=False)
    steps = max(2, args.steps // 2 * 2)
    drv = parallel.DistributedBSGD(shard, y_full, cfg, history_capacity=4 * steps + args.warmup + 64)
    for _ in range(args.warmup):
        drv.epoch_step()
    # CUDA-graph replay with the NCCL all-reduce inside has run at world size 1
    # only (one GPU reachable); across ranks the eager epochs are used unless
    # BSGD_DIST_GRAPH=1 (a rank's epoch at configs[3] is ~0.8 ms of GPU work at 8
    # GPUs, well above the ~0.15 ms of host launches, so eager loses little)
    graphed = (world == 1 or os.environ.get("BSGD_DIST_GRAPH") == "1") and drv.capture(2)
    if graphed:
        drv.replay()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record()
        if graphed:
            for _ in range(steps // 2):
                drv.replay()
        else:
            for _ in range(steps):
                drv.epoch_step()
        e1.record()
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item()) / steps
    clocks = clk.summary()

    # e2e: every step the host state goes in (x, this rank's r slice) and comes back
    r0, r1 = shard.spec.row_range
    cols = shard.cols
    hx = torch.empty(cols, dtype=torch.float64, pin_memory=True)
    hr = torch.empty(r1 - r0, dtype=torch.float64, pin_memory=True)
    hx.copy_(drv.x_current)
    hr.copy_(drv.r_current)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        drv.x_current.copy_(hx, non_blocking=True)
        drv.r_current.copy_(hr, non_blocking=True)
        drv.epoch_step()
        hx.copy_(drv.x_current, non_blocking=True)
        hr.copy_(drv.r_current, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / steps], device=dev)
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_s = float(e2e_s.item())

    # roofline: this rank's forward product (local rays) timed alone
    local_nnz = int(shard.op.nnz)
    rows_l = r1 - r0
    x = drv.x_current.clone()
    rout = torch.empty(rows_l, dtype=torch.float64, device=dev)
    t_k1 = time_events(lambda: shard.matvec(x, rout), 10)
    b1 = local_nnz * 8 + (rows_l + 1) * 8 + cols * 8 + rows_l * 8
    nnz_t = torch.tensor([local_nnz], dtype=torch.int64, device=dev)
    dist.all_reduce(nnz_t)
    pk, pk_src = peaks()
    if rank == 0:
        out = {"metric": METRIC, "value": round(1000.0 / ms_step, 3), "unit": "epochs/s", "n_gpus": world,
               "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded configs[3] phantom, projector and noise; problems.py)",
               "config": config_dict(HEADLINE, int(nnz_t.item()), mu, u_max),
               "parallelism": f"row slabs x{world} (whole row blocks, rays generated on each rank's GPU), "
                              f"NCCL all-reduce of g and ||r||^2 per epoch, prox replicated",
               "roofline": {"bound": "hbm", "kernel": "K1 forward CSR SpMV on rank 0's rays", "achieved":
                            round(b1 / (t_k1 * 1e6), 1), "peak": pk, "unit": "GB/s",
                            "frac": round(b1 / (t_k1 * 1e6) / pk, 4), "traffic": None,
                            "algorithmic_bytes": b1, "launch_ms": round(t_k1, 5), "peak_source": pk_src},
               "cpu_baseline": None,
               "e2e": {"value": round(1.0 / e2e_s, 3), "unit": "epochs/s",
                       "h2d_bytes_per_step": (cols + rows_l) * 8, "d2h_bytes_per_step": (cols + rows_l) * 8,
                       "how": "per rank: x and its r slice from pinned host memory in, epoch, both back out"},
               "gpu_launches": 6 * steps, "clocks": clocks, "graphed": graphed}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def run_multi_slices(args, world, rank, local, dev):
    """configs[4] over N GPUs by SLICES (parallel.CudaSliceShard): each rank owns
    256/N slices of A = A2 (x) I_256 and its local x, g, r -- no product exchange;
    per epoch only the slab prox's one-plane halos and scalar sums (device-side
    FGP decisions, fixed sequence) and two small all-reduces.  CUDA-graph replay."""
    import torch
    import torch.distributed as dist
    from paper_1812_01307_b200 import parallel, tv
    from paper_1812_01307_b200.solvers import SolverConfig
    shard, y_full, meta = parallel.ct_slice_shard(rank, world, device=dev)
    mu, u_max = mu_for(4)
    cfg = SolverConfig(mu=mu, lam=meta["lam"], epochs=10 ** 9, prox=tv.ProxSettings(meta["max_inner_iters"], 1e-5),
                       monitor_decrease=False)
    steps = max(2, args.steps // 2 * 2)
    drv = parallel.DistributedBSGD(shard, y_full, cfg, history_capacity=4 * steps + args.warmup + 64)
    for _ in range(args.warmup):
        drv.epoch_step()
    graphed = (world == 1 or os.environ.get("BSGD_DIST_GRAPH") == "1") and drv.capture(2)
    if graphed:
        drv.replay()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record()
        for _ in range(steps // 2 if graphed else steps):
            drv.replay() if graphed else drv.epoch_step()
        e1.record()
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item()) / steps
    clocks = clk.summary()
    hist = drv.history()
    nnz_t = torch.tensor([int(shard.op.nnz)], dtype=torch.int64, device=dev)
    dist.all_reduce(nnz_t)
    if rank == 0:
        out = {"metric": METRIC, "value": round(1000.0 / ms_step, 3), "unit": "epochs/s", "n_gpus": world,
               "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded configs[4] ellipsoid phantom, projector and noise; problems.py)",
               "config": {"workload": WORKLOADS[4], "nnz": int(nnz_t.item()), "mu": mu, "u_max": u_max,
                          "monitor_decrease": False},
               "parallelism": f"slice ownership x{world} (A2 (x) I_D block diagonal in the slices: no product "
                              f"exchange), slab prox on the slice-major volume with device-side FGP decisions",
               "mean_fgp_iterations": round(float(np.mean(hist[-steps:, 5])), 2),
               "cpu_baseline": None, "e2e": None, "gpu_launches": None, "clocks": clocks, "graphed": graphed}
        print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


# --- reference arm -------------------------------------------------------------------

def reference_inputs():
    """configs[3]'s A (host CSR), y and mu: A from the GPU Siddon generator, which is
    bit-identical to the host generator problems.parallel_beam_matrix
    (tests/test_gpu_generator.py) and takes seconds instead of minutes; y as in
    the GPU arm.  Input generation only -- nothing of the B200 path is timed here."""
    import torch
    from paper_1812_01307_b200 import problems
    t0 = time.time()
    d = problems.config_device(HEADLINE)
    csr = d.op.tocsr()
    y = np.asarray(d.y, dtype=np.float64)
    meta = {"height": d.height, "width": d.width, "lam": d.lam, "max_inner_iters": d.max_inner_iters}
    d.op._csr = None
    del d
    torch.cuda.empty_cache()
    log(f"[ref] inputs ready in {time.time() - t0:.1f}s: {csr.shape}, nnz={csr.nnz}")
    return csr, y, meta


def import_reference():
    if not os.path.isdir(os.path.join(REF_DIR, "bsgdtv")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import bsgdtv.blockops  # noqa: F401
        import bsgdtv.solvers  # noqa: F401
        import bsgdtv.tv  # noqa: F401
        return sys.modules["bsgdtv.solvers"]
    except Exception as exc:
        log(f"[ref] baseline/_ref not importable: {exc!r}")
        return None


def reference_epochs(csr, y, mu, meta, workers, warmup, steps, budget, op=None):
    """Time the reference package's bsgd_tv_iteration (baseline/_ref, unmodified) on
    the given system; None when baseline/_ref is not importable."""
    import concurrent.futures as cf
    if import_reference() is None:
        return None
    from bsgdtv import blockops as rb
    from bsgdtv import solvers as rs
    from bsgdtv import tv as rtv
    t0 = time.time()
    if op is None:
        op = rb.BlockOperator(csr, rb.make_partition(csr.shape[0], csr.shape[1], 8, 8))
    build_s = time.time() - t0
    lay = rtv.PixelLayout(meta["height"], meta["width"], np.arange(meta["height"] * meta["width"]))
    prox = rtv.ProxSettings(max_inner_iters=meta["max_inner_iters"], tol=1e-5)
    cfg = rs.SolverConfig(mu=mu, lam=meta["lam"], prox=prox, monitor_decrease=False)
    st = rs.init_bsgd_state(op, y, cfg)
    with cf.ThreadPoolExecutor(workers) as ex:
        exe = ex if workers > 1 else None
        for _ in range(warmup):
            rs.bsgd_tv_iteration(st, op, y, cfg, layout=lay, executor=exe)
        times = []
        t_start = time.perf_counter()
        for _ in range(steps):
            t1 = time.perf_counter()
            rs.bsgd_tv_iteration(st, op, y, cfg, layout=lay, executor=exe)
            times.append(time.perf_counter() - t1)
            if time.perf_counter() - t_start > budget:
                break
    return {"value": len(times) / sum(times), "epochs": len(times), "seconds": sum(times), "workers": workers,
            "build_s": build_s, "op": op}


def run_reference(args):
    world, rank, _ = dist_info()
    if rank != 0:
        return
    csr, y, meta = reference_inputs()
    mu, u_max = mu_for(HEADLINE)
    nnz = int(csr.nnz)
    cores = os.cpu_count() or 1
    variants = {}
    res = reference_epochs(csr, y, mu, meta, workers=cores, warmup=min(args.warmup, 1), steps=args.steps,
                           budget=args.ref_budget)
    if res is not None:
        del csr
        v, n, secs = res["value"], res["epochs"], res["seconds"]
        kind, how = "reference", (f"the reference package (baseline/_ref bsgdtv, unmodified) bsgd_tv_iteration, "
                                  f"ThreadPoolExecutor({cores}), monitor off")
        log(f"[ref] reference: {v:.4f} epochs/s ({n} epochs, {secs:.1f}s; operator built in {res['build_s']:.1f}s)")
        if not args.no_variants:
            from bsgdtv import solvers as rs
            from bsgdtv import tv as rtv
            op = res["op"]
            r1 = reference_epochs(None, y, mu, meta, workers=1, warmup=0, steps=2, budget=args.ref_budget / 3, op=op)
            variants["workers_1_monitor_off"] = {"value": round(r1["value"], 4), "epochs": r1["epochs"]}
            lay = rtv.PixelLayout(meta["height"], meta["width"], np.arange(meta["height"] * meta["width"]))
            prox = rtv.ProxSettings(max_inner_iters=meta["max_inner_iters"], tol=1e-5)
            # run_solver defaults: monitor on and an objective sample every epoch (sample_every = 1)
            t1 = time.perf_counter()
            rs.run_solver("bsgd", rs.Problem(op, y, None, lay),
                          rs.SolverConfig(mu=mu, lam=meta["lam"], prox=prox, epochs=2), workers=cores)
            variants[f"run_solver_defaults_workers_{cores}"] = {
                "value": round(2.0 / (time.perf_counter() - t1), 4), "epochs": 2,
                "note": "monitor on, sample_every=1; includes the initial objective sample"}
            log(f"[ref] variants: {variants}")
    else:
        v, info = oracle_epochs(csr, y, 8, mu, meta["lam"], meta["max_inner_iters"], 1e-5,
                                (meta["height"], meta["width"]), warmup=min(args.warmup, 1), steps=args.steps,
                                budget_s=args.ref_budget)
        n, secs = info["epochs_timed"], info["seconds"]
        kind, how = "port", "oracle/ C + OpenMP restatement (baseline/_ref absent)"
    cpu = {"value": round(v, 4), "unit": "epochs/s", "cores": cores, "kind": kind,
           "sample": f"{n} full configs[3] epochs ({secs:.1f} s) after {min(args.warmup, 1)} warm-up epoch(s); {how}",
           "host": host_info(), "variants": variants or None}
    out = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "epochs/s", "n_gpus": world,
           "steps": n, "warmup": min(args.warmup, 1), "ms_per_step": round(1000.0 / v, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded configs[3] phantom, projector and noise; problems.py)",
           "config": config_dict(HEADLINE, nnz, mu, u_max), "parallelism": f"{cores} host threads",
           "cpu_baseline": cpu,
           "e2e": {"value": round(v, 4), "unit": "epochs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def host_info():
    info = {"cpu_count": os.cpu_count()}
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                info["model"] = line.split(":", 1)[1].strip()
        with open("/proc/meminfo") as fh:
            info["mem_gb"] = round(int(fh.readline().split()[1]) / 2 ** 20, 1)
    except Exception:
        pass
    return info


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the configs[1], [2], [4] measurements")
    ap.add_argument("--no-variants", action="store_true", help="reference arm: skip the 1-worker / monitor variants")
    ap.add_argument("--no-ref-baseline", action="store_true", help="cpu_baseline: the oracle port only")
    ap.add_argument("--multi-config", type=int, choices=[3, 4], default=3,
                    help="multi-GPU arm: configs[3] row slabs (default) or configs[4] slice ownership")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU (row-slab, NCCL) arm even at world size 1 (under torchrun)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="N > 1: gloo only to exercise the multi-rank path with all ranks on one GPU "
                         "(a functional check, not a measurement)")
    ap.add_argument("--cpu-epochs", type=int, default=8)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=60.0)
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
