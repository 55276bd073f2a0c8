#!/usr/bin/env python
"""bench.py — MAPLE hot path on B200: verified ⊑-minimal directions/sec + MAPLE solve time.

One step = one pass of the whole hot path over the configs[2] workload — the
configuration BASELINE.json's metric is quoted on (C3: n=300, m=20 dense-Q integer QP shape, binary box, 2^20 starts,
T=200, lr=0.01; synthetic): maple_feasible_starts (Eq. 4 initial solutions, part of MA per P:509)
+ maple_extract (starts, descent, harvest, dedupe, exact check, ⊑ filter, sort) [sharded + all-gather + global merge
at N>1] + maple_augment from up to 100 of the Eq. 4 points (100 multi-start augmentations) [sharded at N>1].
The context (A, B, B+ resident in HBM) is created once before timing; its host cost (a0) is reported in solve_time
and in the end-to-end number. The other configs run as secondary measurements in the same invocation (key
"secondary": C2a and C2b = configs[1], C5 = one GPU's 2^19-start share of configs[4], C4 = the configs[3] shared-A
batch), each timed the same way but not the headline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N>1) each rank drives one GPU; timing is CUDA events on the library's stream, barrier +
synchronize on both sides, max over ranks; rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified ⊑-minimal directions/sec + MAPLE solve time"
WORKLOAD = "C3"
N_STARTS, T_STEPS, LR, SEED = 1 << 20, 200, 0.01, 3
K_INCUMBENTS = 100
FEAS_K, FEAS_T, FEAS_LR, FEAS_SEED = 1024, 1000, 0.05, 17   # Eq. 4: starts, steps, step size, seed


def _set_workload(name, n_starts=0):
    """Switch the module-level workload constants to another BASELINE config (secondary measurements)."""
    global WORKLOAD, N_STARTS, T_STEPS, LR, SEED
    from synth import config
    inst = config(name)
    WORKLOAD = name
    N_STARTS = n_starts or inst.n_starts
    T_STEPS, LR, SEED = inst.steps, inst.lr, inst.seed


def _instance():
    from synth import config
    return config(WORKLOAD)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def _traffic(kernel, n_starts):
    """dram read + write bytes per launch of `kernel` from the committed ncu --set full capture (profiles/
    r1_traffic.json) when it was taken on this workload and start count, else None."""
    try:
        t = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_traffic.json")))
        e = t[kernel]
        if e["workload"] == WORKLOAD and e["n_starts"] == n_starts:
            return e["read_bytes"] + e["write_bytes"]
    except (OSError, KeyError, ValueError):
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region: ONE `nvidia-smi -lms 200` process (the
    recipe's clocks line), started before and stopped after, so no per-sample driver initialisation lands
    inside the timed steps."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._p = None

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):   # diagnostics only: the JSON line then reports no clocks
            return self
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)   # first sample before the timed region starts
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        self._p.terminate()   # our own child, by handle
        try:
            out, _ = self._p.communicate(timeout=10)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in (out or "").splitlines():
            if line.strip():
                self.rows.append([x.strip() for x in line.split(",")])

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _oracle_cores(r):
    """Threads the oracle sample actually kept busy: process CPU time / wall time over the sample (most of the oracle
    is single-threaded Python; numpy's BLAS may add threads in the lattice and the matrix products)."""
    return round(max(1.0, r["cpu"] / max(r["wall"], 1e-9)), 2)


def _oracle_step(S, KI, offset, KF=16):
    """One bounded oracle sample of the workload: the lattice step, Eq. 4 from KF of the FEAS_K starts (MA's initial
    solutions), fp64 descent + harvest of S starts [offset, offset + S), the exact ⊑ filter of their pool, KI of
    the K_INCUMBENTS augmentations. The full-step estimate scales Eq. 4 by FEAS_K / KF, the descent by N / S and the
    augmentations by K / KI (each linear in its units) and takes the filter as measured on the sample's pool (the full
    pool is larger: a lower bound on the oracle's time)."""
    from oracle import augment as OA, extraction as OX, feasible as OF, lattice as OL, postprocess as OP
    from synth import feasible_points
    inst = _instance()
    c0 = time.process_time()
    t0 = time.perf_counter()
    B = np.array(OL.lll_reduce(OL.kernel_basis(inst.A)), dtype=np.int64)
    t_lat = time.perf_counter() - t0
    pts, _ = OF.feasible_set(inst.A, inst.b, inst.l, inst.u, KF, FEAS_T, FEAS_LR, FEAS_SEED)
    t_eq4 = time.perf_counter() - t0 - t_lat
    t1 = time.perf_counter()
    pool, _ = OX.extract_pool(B, OL.pinv(B), inst.l, inst.u, N_STARTS, T_STEPS, LR, SEED,
                              starts=np.arange(offset, offset + S) % N_STARTS)
    t_desc = time.perf_counter() - t1
    S_min = OP.minimal_filter(pool)
    t_filt = time.perf_counter() - t1 - t_desc
    X0 = np.array(pts[:KI], dtype=np.int64) if len(pts) >= KI else feasible_points(inst, KI, seed=99)
    t2 = time.perf_counter()
    OA.multi_start(OA.Objective(inst.Q, inst.c, inst.c0), inst.A, inst.b, inst.l, inst.u, X0, S_min)
    t_aug = time.perf_counter() - t2
    t_full = t_lat + t_eq4 * (FEAS_K / KF) + t_desc * (N_STARTS / S) + t_filt + t_aug * (K_INCUMBENTS / KI)
    return {"t_full": t_full, "t_desc": t_desc, "t_filt": t_filt, "t_aug": t_aug, "t_eq4": t_eq4, "KF": KF,
            "n_min": len(S_min), "pool": len(pool), "wall": time.perf_counter() - t0,
            "cpu": time.process_time() - c0}


def _sample_text(S, KI, r, offset_text):
    return (f"Eq. 4 from {r['KF']} of {FEAS_K} starts ({r['t_eq4']:.1f} s, x{FEAS_K // r['KF']}); "
            f"{S} of {N_STARTS} starts ({offset_text}; fp64 descent+harvest {r['t_desc']:.1f} s, x{N_STARTS // S}), "
            f"exact filter of their pool ({r['pool']} rows, {r['t_filt']:.1f} s, as measured: a lower bound), "
            f"{KI} of {K_INCUMBENTS} augmentations ({r['t_aug']:.1f} s, x{K_INCUMBENTS // KI}); {r['n_min']} minimal "
            f"directions; estimated step {r['t_full']:.0f} s")


def run_reference(args):
    """The oracle (oracle/, the CPU reference) on a bounded sample of the same workload, per step."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    S, KI = (256, 10) if _instance().n <= 64 else (16, 2)
    res = []
    for it in range(args.warmup + args.steps):
        r = _oracle_step(S, KI, S * it)
        if it >= args.warmup:
            res.append(r)
    t_full = statistics.mean(r["t_full"] for r in res)
    nset = statistics.mean(r["n_min"] for r in res)
    value = nset / t_full
    line = {"metric": METRIC, "value": value, "unit": "directions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": _instance().n, "m": _instance().m, "n_starts": N_STARTS,
                       "steps": T_STEPS, "incumbents": K_INCUMBENTS},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "directions/s", "cores": _oracle_cores(res[-1]), "kind": "oracle",
                             "sample": "per step: " + _sample_text(S, KI, res[-1], f"starts [{S}k, {S}(k+1)) at step k")},
            "e2e": {"value": value, "unit": "directions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_sample():
    """Oracle timed on the host cores on a bounded sample (rank 0, N=1 only)."""
    S, KI = (1024, 20) if _instance().n <= 64 else (32, 4)
    r = _oracle_step(S, KI, 0)
    return {"value": r["n_min"] / r["t_full"], "unit": "directions/s", "cores": _oracle_cores(r), "kind": "oracle",
            "sample": _sample_text(S, KI, r, "the first ones")}


def _incumbents(ctx, inst, world=1):
    """MA's initial solutions: Eq. 4 from FEAS_K diversified starts on the device; up to K_INCUMBENTS of
    the distinct feasible points found (sorted). The planted point is the fallback only when Eq. 4 finds none."""
    pts, _ = ctx.feasible_starts(inst.b, FEAS_K, FEAS_T, FEAS_LR, seed=FEAS_SEED)
    if len(pts) == 0:
        pts = inst.x_plant[None, :].astype(np.int32)
    return pts[:K_INCUMBENTS]


def _roofline(inst, ctx, desc_ms, n_starts_rank, peaks, src, ms):
    """Roofline of the dominant kernel (the descent) for the line: algorithmic work per start-step x N x T over the
    mean descent time (CUDA events on the library's stream) against the peak of the unit that bounds it."""
    n, d = inst.n, inst.d
    units = n_starts_rank * T_STEPS                               # start-steps per descent launch
    path = ctx.descent_kernel
    nnz_b = int(np.count_nonzero(ctx.B))
    alu_peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
    # Algorithmic fp32 ALU work per start-step: 16 ops per coordinate (λ1 derivative 3, gradient add
    # 1, m 2, v 3, sqrt 1, scale + eps 1, reciprocal 1, step 2, round + change test 2) + 1 sign per row of B; the SIMT
    # path runs both contractions on the fp32 lanes as well (+ 2 nnz(B) FMAs).
    ops_per = 16.0 * d + n + (2.0 * nnz_b if path == "simt" else 0.0)
    achieved = ops_per * units / (desc_ms * 1e-3) / 1e12
    kname = {"tc": "descent_tc_kernel", "tcp": "descent_tcp_kernel"}.get(
        path, "descent_simt_kernel")
    roof = {"kernel": kname, "bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "Tops/s",
            "frac": achieved / alu_peak, "traffic": _traffic(kname, n_starts_rank), "ops_per_start_step": ops_per,
            "note": f"achieved = ({'16d+n+2nnz(B)' if path == 'simt' else '16d+n'}) algorithmic fp32 ops x N x T / "
                    f"mean descent time; peak = 148 SMs x 128 lanes x sm_max_mhz ({src} clocks); descent share of "
                    f"step {desc_ms / ms:.2f}"}
    if path in ("tc", "tcp"):
        # tensor view: SURVEY §8(d)-2's 4nd algorithmic flops per start-step, and the MMA work the kernel issues
        # (tcp: 3 f16 passes of the forward + i8 harvest + i8 backward = 3 x 2nd f16 + 2 x 2nd i8 per start-step)
        bf16_peak = peaks.get("bf16_tflops", 1614.6)
        gemm_tflops = 4.0 * n * d * units / (desc_ms * 1e-3) / 1e12
        view = {"algorithmic_tflops": gemm_tflops, "peak_tflops_bf16_measured": bf16_peak}
        if path == "tcp":
            npad, dpad = 320, 288
            f16_tf = 3 * 2.0 * npad * dpad * units / (desc_ms * 1e-3) / 1e12
            i8_tops = 2 * 2.0 * npad * dpad * units / (desc_ms * 1e-3) / 1e12
            view.update({"issued_f16_tflops": f16_tf, "issued_i8_tops": i8_tops,
                         "tensor_pipe_frac_est": f16_tf / bf16_peak + i8_tops / (2 * bf16_peak)})
        roof["tensor_view"] = view
    return roof


def _measure(args, ctx, inst, stream, flush, world, local, one_step, sync_all, steps, warmup):
    """Warm-up, then `steps` timed steps (L2 flushed before each; CUDA events on the library's stream)."""
    import torch
    out = None
    for _ in range(warmup):   # the same pattern as the timed loop: the previous step's result is alive meanwhile
        flush.fill_(1)
        out = one_step()
    sync_all()
    launches0 = ctx.launches()
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    phase = {"descent": [], "dedupe": [], "check": [], "filter": [], "sort": [], "extract_total": [],
             "augment_total": []}
    for k in range(steps):
        flush.fill_(k & 0xFF)              # L2 flush between timed steps (outside the timed region)
        sync_all()
        ev_s[k].record(stream)
        out = one_step()
        ev_e[k].record(stream)
        sync_all()
        t = ctx.timings()
        for key in phase:
            phase[key].append(t[key])
        if os.environ.get("BENCH_VERBOSE"):
            print(f"[bench] step {k}: {ev_s[k].elapsed_time(ev_e[k]):.2f} ms " +
                  " ".join(f"{key} {t[key]:.2f}" for key in phase), file=sys.stderr)
    step_ms = [ev_s[k].elapsed_time(ev_e[k]) for k in range(steps)]
    return float(np.mean(step_ms)), phase, ctx.launches() - launches0, out


def _secondary(args, stream, flush, sync_all, local):
    """The other configs as secondary lines (one GPU, 3 warm-up + 2 timed steps each)."""
    from paper_2412_13576_b200 import maple
    from synth import c4_batch
    global WORKLOAD, N_STARTS, T_STEPS, LR, SEED
    saved = (WORKLOAD, N_STARTS, T_STEPS, LR, SEED)
    res = {}
    for name, ns in (("C2a", 0), ("C2b", 0), ("C5", 1 << 19)):
        _set_workload(name, ns)
        inst = _instance()
        ctx = maple.Context(inst.A, inst.l, inst.u, device=local)
        ctx.set_stream(stream.cuda_stream)
        X0 = _incumbents(ctx, inst)

        def step():
            ds = ctx.extract(N_STARTS, T_STEPS, LR, SEED)
            xb, fb, _, _ = ctx.augment(ds, inst.Q, inst.c, inst.c0, inst.b, _incumbents(ctx, inst))
            return ds, fb
        ms, phase, launches, (ds, fb) = _measure(args, ctx, inst, stream, flush, 1, local, step, sync_all, 2, 3)
        res[name] = {"n": inst.n, "m": inst.m, "n_starts": N_STARTS, "steps": T_STEPS, "ms_per_step": ms,
                     "directions": ds.size, "pool": ds.pool_size, "directions_per_s": ds.size / (ms * 1e-3),
                     "descent_kernel": ctx.descent_kernel, "f_best": fb, "incumbents": int(len(X0)),
                     "phase_ms": {k: float(np.mean(v)) for k, v in phase.items()},
                     "start_steps_per_s": N_STARTS * T_STEPS / (float(np.mean(phase["descent"])) * 1e-3)}
        ds.free()
        ctx.close()
    # configs[3]: one create + one extraction of the C2a matrix reused for 1,000 (f, b) instances x 256
    # incumbents; solve time = create + extract + the batched augmentation
    _set_workload("C2a")
    base, insts = c4_batch(1000, 256)
    t0 = time.perf_counter()
    ctx = maple.Context(base.A, base.l, base.u, device=local)
    ctx.set_stream(stream.cuda_stream)
    create_ms = (time.perf_counter() - t0) * 1e3
    e0 = torch_event()
    e1 = torch_event()
    e2 = torch_event()
    sync_all()
    e0.record(stream)
    ds = ctx.extract(N_STARTS, T_STEPS, LR, SEED)
    e1.record(stream)
    xb, fb = ctx.augment_many(ds, [q for q, _, _, _ in insts], [c for _, c, _, _ in insts], [0.0] * len(insts),
                              [b for _, _, b, _ in insts], [x for _, _, _, x in insts])
    e2.record(stream)
    sync_all()
    ext_ms, aug_ms = e0.elapsed_time(e1), e1.elapsed_time(e2)
    res["C4"] = {"instances": len(insts), "incumbents_each": 256, "create_ms": create_ms, "extract_ms": ext_ms,
                 "augment_many_ms": aug_ms, "solve_ms": create_ms + ext_ms + aug_ms,
                 "ms_per_instance": (ext_ms + aug_ms) / len(insts), "directions": ds.size,
                 "f_best_mean": float(np.mean(fb))}
    ds.free()
    ctx.close()
    WORKLOAD, N_STARTS, T_STEPS, LR, SEED = saved
    return res


def torch_event():
    import torch
    return torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--descent-kernel", type=int, default=0)
    ap.add_argument("--workload", default="C3", choices=["C1", "C2a", "C2b", "C3", "C5"],
                    help="configs[2] (C3) is the headline line; the others are secondary measurements")
    ap.add_argument("--n-starts", type=int, default=0, help="override the workload's start count")
    args = ap.parse_args()
    _set_workload(args.workload, args.n_starts)
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    import __graft_entry__
    if rank == 0 or world == 1:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    from paper_2412_13576_b200 import maple
    from paper_2412_13576_b200 import distributed as D

    maple.load()
    inst = _instance()
    stream = torch.cuda.Stream()
    t_c0 = time.perf_counter()
    ctx = maple.Context(inst.A, inst.l, inst.u, device=local)
    create_ms = (time.perf_counter() - t_c0) * 1e3
    ctx.set_stream(stream.cuda_stream)
    ctx.set_descent_kernel(args.descent_kernel)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")   # > 126 MB L2

    def one_step(c=ctx):
        X0 = _incumbents(c, inst)                       # Eq. 4 initial solutions (MA)
        if world > 1:
            ds, _ = D.sharded_extract(c, N_STARTS, T_STEPS, LR, SEED)
            xb, fb = D.sharded_augment(c, ds, inst.Q, inst.c, inst.c0, inst.b, X0)
        else:
            ds = c.extract(N_STARTS, T_STEPS, LR, SEED)
            xb, fb, _, _ = c.augment(ds, inst.Q, inst.c, inst.c0, inst.b, X0)
        return ds, xb, fb, X0

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        ms, phase, launches, (ds, xb, fb, X0) = _measure(args, ctx, inst, stream, flush, world, local, one_step,
                                                         sync_all, args.steps, args.warmup)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    n_dirs = ds.size
    # all verified: every output row passed the device exact check (C1-C3); assert it here on the host too
    rows = ds.rows_pinned()
    assert rows.shape[0] == 0 or np.all(rows.astype(np.int64) @ inst.A.T == 0)

    # ---- end-to-end through the public API with host buffers (create + Eq. 4 starts + extract + D2H set + augment)
    e2e_ms, e2e_host = [], []
    h2d = inst.A.size * 4 + inst.l.size * 4 + inst.u.size * 4 + inst.Q.size * 8 + inst.c.size * 8 + 2 * inst.b.size * 4
    d2h = 0
    # W untimed end-to-end solves first (like the device-timed steps): a second context's first allocations grow the
    # stream-ordered pool (physical pages, ~1 s at C3) and the first solves after it still ran ~100 ms slow; later
    # solves reuse everything, as in a serving process
    for k in range(-max(1, args.warmup), max(3, args.steps)):
        flush.fill_(3)
        sync_all()
        e0, e1 = torch_event(), torch_event()
        e0.record(stream)
        th = [time.perf_counter()]
        c2 = maple.Context(inst.A, inst.l, inst.u, device=local)
        c2.set_stream(stream.cuda_stream)
        th.append(time.perf_counter())
        X0e = _incumbents(c2, inst)
        th.append(time.perf_counter())
        if world > 1:
            d2, _ = D.sharded_extract(c2, N_STARTS, T_STEPS, LR, SEED)
        else:
            d2 = c2.extract(N_STARTS, T_STEPS, LR, SEED)
        th.append(time.perf_counter())
        hrows = d2.rows_pinned()
        th.append(time.perf_counter())
        if world > 1:
            xb2, fb2 = D.sharded_augment(c2, d2, inst.Q, inst.c, inst.c0, inst.b, X0e)
        else:
            xb2, fb2, _, _ = c2.augment(d2, inst.Q, inst.c, inst.c0, inst.b, X0e)
        e1.record(stream)
        sync_all()
        th.append(time.perf_counter())
        if k >= 0:
            e2e_ms.append(e0.elapsed_time(e1))
            e2e_host.append(np.diff(th) * 1e3)
        h2d_k = h2d + X0e.size * 4
        d2h = hrows.shape[0] * d2.stride + xb2.size * 4 + 8 + X0e.size * 4
        d2.free()
        c2.close()
    e2e = float(np.mean(e2e_ms))
    if world > 1:
        tt = torch.tensor([e2e], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = float(tt.item())

    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary and WORKLOAD == "C3":
        secondary = _secondary(args, stream, flush, sync_all, local)

    if rank == 0:
        peaks, src = _peaks()
        desc_ms = float(np.mean(phase["descent"]))
        roof = _roofline(inst, ctx, desc_ms, N_STARTS / world, peaks, src, ms)
        line = {"metric": METRIC, "value": n_dirs / (ms * 1e-3), "unit": "directions/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": WORKLOAD, "n": inst.n, "m": inst.m, "d": inst.d, "n_starts": N_STARTS,
                           "steps": T_STEPS, "lr": LR, "incumbents": int(len(X0)), "eq4_starts": FEAS_K,
                           "l2": "flushed (256 MB write) between timed steps",
                           "parallelism": f"starts sharded over {world} GPU(s), 1 all-gather"},
                "directions": n_dirs, "pool": ds.pool_size, "f_best": fb, "descent_kernel": ctx.descent_kernel,
                "solve_time_ms": {"create": float(np.median(np.array(e2e_host), axis=0)[0]),
                                  "create_first_in_process": create_ms,
                                  "extract": float(np.mean(phase["extract_total"])),
                                  "augment": float(np.mean(phase["augment_total"])),
                                  "ma_incl_eq4": ms - float(np.mean(phase["extract_total"]))},
                "phase_ms": {k: float(np.mean(v)) for k, v in phase.items()},
                "start_steps_per_s": N_STARTS * T_STEPS / (float(np.mean(phase["descent"])) * 1e-3),
                "e2e": {"value": n_dirs / (e2e * 1e-3), "unit": "directions/s", "h2d_bytes_per_step": int(h2d_k),
                        "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e, "ms_all": [round(x, 3) for x in e2e_ms],
                        "host_ms": dict(zip(["create", "eq4", "extract", "rows", "augment"],
                                            [round(float(x), 3) for x in np.median(np.array(e2e_host), axis=0)]))},
                "gpu_launches": int(launches // max(args.steps, 1)) * args.steps,
                "gpu_launches_per_step": launches / max(args.steps, 1),
                "roofline": roof,
                "clocks": clk.summary()}
        if secondary is not None:
            line["secondary"] = secondary
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline_sample()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
