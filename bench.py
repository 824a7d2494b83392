#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the multilevel NMF hot path.

Workload (N=1): BASELINE.json config 4, the largest single-GPU configuration:
256x256-pixel images (m = 65536), n = 262144 columns (64 GiB fp32 M), r = 64,
HALS.  A "step" is one HALS sweep at the finest level (both M-streaming
products, both Gram matrices, both sweeps) on seeded synthetic data of that
shape generated on the device.  For N > 1 the columns of
M are sharded over the ranks (strong scaling: the total problem is fixed) with
one NCCL allreduce of [M W^T | W W^T] per step.

Arms:
  default           the B200 engine.  value: device-timed iterations/s (CUDA
                    events on the engine's stream, max over ranks); e2e: the
                    same metric through the C-ABI with pinned host buffers.
  --impl reference  the reference's own CPU implementation (oracle/_ref: the
                    unmodified mlnmf sources, OpenMP on all host cores) on
                    bounded column slices of the same workload, extrapolated
                    linearly in n (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "NMF iterations/sec + time-to-rel-error; HBM GB/s vs roofline, 1/2/4/8 GPU"
UNIT = "iterations/s"
CFG = 4
M_ROWS, N_TOTAL, RANK, LEVELS = 65536, 262144, 64, 5
WORKLOAD = "config4: 256x256 px (m=65536), n=262144, r=64, HALS, one finest-level sweep per step"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


TRAFFIC_SRC = "profiles/r02_traffic_config4.json (ncu dram__bytes_read+write per launch, 1 GPU)"


def traffic_for(kernel, world):
    """DRAM bytes per launch of `kernel` from the committed ncu capture of this
    workload (profiles/); None if absent or not the 1-GPU configuration."""
    p = os.path.join(REPO, "profiles", "r02_traffic_config4.json")
    if world != 1 or not os.path.exists(p):
        return None
    with open(p) as f:
        k = json.load(f)["kernels"].get(kernel)
    return k["traffic_bytes"] if k else None


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled (every 20 ms) during the timed region: only the samples
    whose timestamps fall between mark_start() and mark_end() are summarised (all of them if never marked)."""

    def __init__(self, index=0):
        self.index, self.proc = index, None
        self.path = f"/tmp/mlb_clocks_{os.getpid()}.csv"
        self.t0 = self.t1 = None

    def __enter__(self):
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    @staticmethod
    def _stamp(text):
        import datetime
        try:
            return datetime.datetime.strptime(text.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except Exception:
            return None

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            rows = [l.strip().split(", ") for l in open(self.path) if l.strip()]
        except Exception:
            return out
        sm, mx, reasons, power, total = [], [], set(), [], 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                total += 1
                ts = self._stamp(r[0])
                if self.t0 is not None and self.t1 is not None and ts is not None and not (self.t0 <= ts <= self.t1):
                    continue
                sm.append(float(r[1]))
                mx.append(float(r[2]))
                power.append(float(r[3]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        if sm:
            out.update(sm_mhz=float(np.median(sm)), sm_max_mhz=float(max(mx)), samples=len(sm),
                       power_w_max=float(max(power)) if power else None)
        out["samples_total"] = total
        out["reasons"] = sorted(reasons)
        return out


# ---------------------------------------------------------------------------
# torch.distributed plumbing (gloo: id broadcast, barriers, max of timings)
# ---------------------------------------------------------------------------
def dist_setup():
    world, rank, local = env_int("WORLD_SIZE", 1), env_int("RANK", 0), env_int("LOCAL_RANK", 0)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bcast_obj(b, world):
    if world == 1:
        return b
    import torch.distributed as dist
    obj = [b]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


# ---------------------------------------------------------------------------
# reference arm (CPU): oracle/_ref on column slices of config 4
# ---------------------------------------------------------------------------
REF_SLICES = (128, 512, 4096)


def reference_steps(steps, warmup, slices=REF_SLICES):
    """The reference's hals_step (oracle/_ref: the unmodified mlnmf sources,
    fp64, OpenMP) on column slices of config 4, median of `steps` timed steps
    each after `warmup`; a least-squares line t = a + b n through the slice
    medians, evaluated at n = 262144.  Returns (t_full, info) with the slice
    times, the fit and its largest relative residual at the slices."""
    import oracle
    ref, restated = oracle.Reference(), oracle.Restated()
    data = {}
    for ns in slices:
        M = oracle.generate_config(CFG, n=N_TOTAL, col0=0, n_cols=ns, restated=restated)
        V, W = ref.random_init(M_ROWS, ns, RANK, 0)
        data[ns] = [M, V, W]
    times = {ns: [] for ns in slices}
    for it in range(warmup + steps):
        for ns in slices:
            M, V, W = data[ns]
            t0 = time.perf_counter()
            V, W, _ = ref.hals_step(M, V, W)
            dt = time.perf_counter() - t0
            data[ns][1], data[ns][2] = V, W
            if it >= warmup:
                times[ns].append(dt)
    x = np.array(slices, dtype=np.float64)
    y = np.array([float(np.median(times[ns])) for ns in slices])
    b, a = np.polyfit(x, y, 1)
    resid = float(np.max(np.abs((a + b * x) - y) / y))
    return a + b * N_TOTAL, dict(t_slices_s={str(k): float(v) for k, v in zip(slices, y)},
                                 fit_a_s=float(a), fit_b_s_per_col=float(b), fit_max_rel_residual=resid)


def ref_sample_text(steps, info):
    pts = ", ".join(f"n={k}: {v:.4f} s" for k, v in info["t_slices_s"].items())
    return (f"reference hals_step (oracle/_ref = unmodified mlnmf sources, fp64, OpenMP) on column slices of "
            f"config 4 (m=65536, r=64), median of {steps} steps each ({pts}); least-squares line "
            f"t = {info['fit_a_s']:.4f} s + {info['fit_b_s_per_col'] * 1e3:.4f} ms/column through the three points "
            f"(max relative residual {info['fit_max_rel_residual'] * 100:.2f} %), evaluated at n=262144")


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    t0 = time.perf_counter()
    t_full, info = reference_steps(args.steps, args.warmup)
    value = 1.0 / t_full
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_full * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config-4 generator, column slices)",
        "config": {"workload": WORKLOAD, "global_batch": N_TOTAL, "seq_len": M_ROWS,
                   "parallelism": f"cpu{threads}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": ref_sample_text(args.steps, info)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0, **info,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline():
    """The reference arm's measurement on a bounded sample, in a fresh process: inside this one the
    reference's OpenMP team shares the host with torch's thread pools (r02: the in-process 3-step medians
    fitted with 3-13 % residual against < 1 % for the stand-alone reference arm)."""
    threads = os.cpu_count() or 1
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT", "OMP_NUM_THREADS")}
    try:
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference", "--steps", "3",
                              "--warmup", "1"], env=env, capture_output=True, text=True, timeout=600, check=True)
        line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
        cb = line["cpu_baseline"]
        cb["sample"] += " (fresh process)"
        for k in ("t_slices_s", "fit_a_s", "fit_b_s_per_col", "fit_max_rel_residual"):
            cb[k] = line.get(k)
        return cb
    except Exception:
        os.environ.setdefault("OMP_NUM_THREADS", str(threads))
        t_full, info = reference_steps(steps=3, warmup=1)
        return {"value": 1.0 / t_full, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": ref_sample_text(3, info) + " (in process)", **info}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args):
    world, rank, local = dist_setup()
    import torch
    import paper_1009_0881_b200 as P

    torch.cuda.set_device(local)
    nid = bcast_obj(P.nccl_unique_id() if (world > 1 and rank == 0) else None, world)
    col0, n_loc = P.shard_columns(N_TOTAL, world, rank)
    gemm = {"auto": P.GEMM_AUTO, "simt": P.GEMM_SIMT, "tc": P.GEMM_TCGEN05}[args.gemm]
    s = P.Session(device=local, dtype=P.F32, gemm_path=gemm, world=world, rank=rank, nccl_id=nid)
    t_gen = time.perf_counter()
    s.generate(CFG, seed=0, n_total=N_TOTAL, col0=col0, n_local=n_loc)
    norm = float(np.sqrt(s.norm2(0)))
    t_gen = time.perf_counter() - t_gen
    # random_init(seed 0) on this shard + the start sample; zero budget => no step
    tr0 = s.run_configuration(1, "hals", "none", RANK, 0, 0.0, 0)
    ext = torch.cuda.ExternalStream(s.stream, device=local)

    s.steps("hals", args.warmup)
    s.sync()
    barrier(world)
    launches0 = s.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.mark_start()
        ev0.record(ext)
        s.steps("hals", args.steps)
        ev1.record(ext)
        ev1.synchronize()
        clk.mark_end()
    ms = ev0.elapsed_time(ev1)
    launches = s.launches - launches0
    ms_max = allreduce_max(ms, world)
    value = args.steps / (ms_max / 1e3)

    # per-product durations: a separate profiled pass (CUDA events bracketing
    # each M-streaming product on the engine stream)
    s.set_profiling(True)
    s.steps("hals", 3)
    kt = s.kernel_times()
    phases = s.phase_times()
    s.set_profiling(False)
    mwt_ms = kt["mwt_ms"] / max(kt["mwt_n"], 1)
    vtm_ms = kt["vtm_ms"] / max(kt["vtm_n"], 1)
    bytes_per_pass = M_ROWS * n_loc * 4
    dom_ms, dom = (vtm_ms, "C = V^T M") if vtm_ms >= mwt_ms else (mwt_ms, "A = M W^T")
    achieved = bytes_per_pass / (dom_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    err_end = s.error()
    tc = s.tc_active

    e2e = None
    if args.e2e:
        host = torch.empty((M_ROWS, n_loc), dtype=torch.float32, pin_memory=True)
        s.export_data(host.data_ptr())
        s.close()
        # a fresh communicator for the e2e session (one NCCL id per communicator)
        nid2 = bcast_obj(P.nccl_unique_id() if (world > 1 and rank == 0) else None, world)
        e2e = run_e2e(P, host, local, gemm, args.e2e_iters, norm, world, rank, nid2, col0)
        del host
    else:
        s.close()

    ttt = time_to_target(P, local, gemm) if (args.ttt and world == 1) else None
    small = small_configs(P, local, args.cpu_baseline) if (args.small and world == 1) else None
    ttts = ttt_small(P, local, args.cpu_baseline) if (args.ttt and args.small and world == 1) else None

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if tc else "f32 storage / f64 accumulate",
        "data": "synthetic (BASELINE config-4 generator on the device, seed 0)",
        "config": {"workload": WORKLOAD, "global_batch": N_TOTAL, "seq_len": M_ROWS,
                   "parallelism": f"column-shard x{world}", "l2": "inputs larger than L2 (M = 64 GiB fp32)",
                   "gemm_path": "tcgen05 kind::i8 digit products (fp32 M and fp64 factors on per-row 31-bit fixed-point grids, four int8 digits each, exact int32 accumulation)" if tc else "SIMT fp64-accumulate"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_for(dom, world), "kernel": dom,
                     "peak_source": peak_src, "traffic_source": TRAFFIC_SRC,
                     "algorithmic_bytes_per_launch": bytes_per_pass,
                     "avg_ms": {"A = M W^T": mwt_ms, "C = V^T M": vtm_ms,
                                "allreduce [A|B]": kt["comm_ms"] / max(kt["comm_n"], 1) if kt["comm_n"] else 0.0},
                     "step_frac_in_products": (mwt_ms + vtm_ms) / (ms_max / args.steps),
                     "step_phases_ms": phases},
        "rel_error": {"start": float(tr0.error[0]) / norm, "after_bench": err_end / norm},
        "gen_s": t_gen,
    }
    if e2e:
        line["e2e"] = e2e
    if ttt:
        line["time_to_target"] = ttt
    if small:
        line["small_configs"] = small
    if ttts:
        line["time_to_target_small"] = ttts
    if args.cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)


def run_e2e(P, host, local, gemm, iters, norm, world=1, rank=0, nccl_id=None, col0=0):
    """One reference-facing solve through the C-ABI from pinned host memory:
    set_data (H2D of this rank's columns of M) + run_configuration(levels=1,
    HALS, none, r=64, work:iters) + get_factors (D2H of V and this rank's W
    columns), wall-clock timed between barriers, max over ranks.  Byte counts
    are whole-job (all ranks)."""
    import torch
    m, nl = host.shape
    Vh = torch.empty((m, RANK), dtype=torch.float32, pin_memory=True)
    Wh = torch.empty((RANK, nl), dtype=torch.float32, pin_memory=True)
    torch.cuda.synchronize()
    se = P.Session(device=local, dtype=P.F32, gemm_path=gemm, world=world, rank=rank, nccl_id=nccl_id)
    barrier(world)
    t0 = time.perf_counter()
    se.set_data_ptr(host.data_ptr(), P.F32, m, nl, P.ImageGrid(256, 256), n_total=N_TOTAL, col0=col0)
    tr = se.run_configuration(1, "hals", "none", RANK, 0, float(iters), 0)
    se.get_factors_ptr(Vh.data_ptr(), Wh.data_ptr(), P.F32)
    wall = allreduce_max(time.perf_counter() - t0, world)
    se.close()
    steps = int(tr.phase_steps.sum())
    return {"value": steps / wall, "unit": UNIT, "h2d_bytes_per_step": m * N_TOTAL * 4 / steps,
            "d2h_bytes_per_step": (world * m * RANK + RANK * N_TOTAL) * 4 / steps,
            "call": f"mlnmf_session_set_data + mlnmf_session_run_configuration(levels=1, hals, none, r=64, "
                    f"work:{iters}, trace_every=0) + mlnmf_session_get_factors; pinned host fp32, "
                    f"{world} rank(s), wall time max over ranks",
            "iters_per_call": steps, "wall_s": wall, "final_rel_error": float(tr.error[-1]) / norm}


# solver kinds BASELINE.json names per config (configs[0..3])
SMALL_KINDS = {0: ("hals",), 1: ("mu", "hals"), 2: ("anls", "hals"), 3: ("hals", "mu", "anls")}


def small_configs(P, local, with_cpu):
    """BASELINE configs 0-3 (L2-resident, launch/latency bound):
    single-level sweeps/s on the device for every solver kind BASELINE.json
    names for the config (fp32 storage, SIMT fp64-accumulate products, data
    generated on the device, trace_every=0; HALS/MU 100 sweeps, ANLS 20),
    next to the reference's own step (oracle/_ref, fp64, OpenMP on all host
    cores) from the same random init, median of 2 steps."""
    out = {}
    ref = None
    if with_cpu:
        import oracle
        if oracle.Reference.available():
            ref, restated = oracle.Reference(), oracle.Restated()
    for cfg in (0, 1, 2, 3):
        c = P.GEN_CONFIGS[cfg]
        M = oracle.generate_config(cfg, restated=restated) if ref is not None else None
        for kind in SMALL_KINDS[cfg]:
            work = 20.0 if kind == "anls" else 100.0
            with P.Session(device=local, dtype=P.F32) as s:
                s.generate(cfg, seed=0)
                s.run_configuration(1, kind, "none", c["r"], 0, 5.0, 0)  # warm-up (graphs, buffers)
                s.sync()
                t0 = time.perf_counter()
                tr = s.run_configuration(1, kind, "none", c["r"], 0, work, 0)
                s.sync()
                wall = time.perf_counter() - t0
            steps = int(tr.phase_steps.sum())
            e = {"shape": f"{c['h']}x{c['w']} (m={c['h'] * c['w']}) x n={c['n']}, r={c['r']}", "kind": kind,
                 "sweeps": steps, "gpu_it_s": steps / wall, "gpu_ms_per_step": wall / steps * 1e3}
            if ref is not None:
                V, W = ref.random_init(M.shape[0], M.shape[1], c["r"], 0)
                step = {"mu": ref.mu_step, "hals": ref.hals_step, "anls": ref.anls_step}[kind]
                ts = []
                for _ in range(2):
                    t1 = time.perf_counter()
                    res = step(M, V, W)
                    ts.append(time.perf_counter() - t1)
                    V, W = res[0], res[1]
                e["cpu_ref_ms_per_step"] = float(np.median(ts)) * 1e3
                e["cpu_ref_note"] = "first two steps from random init (ANLS: cold active sets, slowest sweeps)"
                e["cpu_cores"] = os.cpu_count() or 1
                e["speedup"] = e["cpu_ref_ms_per_step"] / e["gpu_ms_per_step"]
            out[f"config{cfg}_{kind}"] = e
    return out


def ttt_small(P, local, with_cpu):
    """BASELINE.md section 2 for configs 0-3 at their BASELINE budgets
    (config 0 work:100, 1 work:500, 2-3 work:100; each config's first solver
    kind in BASELINE.json): target = the reference's single-level final
    relative error; for none / NI / VC / FMG the time to the first finest-
    level sample at or below it, on the reference CPU (oracle/_ref, fp64,
    OpenMP on all host cores) and on the GPU (fp32 M storage, fp64 factors),
    both including the pyramid build and random_init (setup = the run's wall
    time minus its last sample's elapsed time, added to the hit time), plus
    the GPU trajectory's largest relative deviation from the reference's on
    the same fp32-rounded M (every sample, trace_every = 1)."""
    import oracle
    ref = oracle.Reference() if (with_cpu and oracle.Reference.available()) else None
    restated = oracle.Restated()
    out = {}
    for cfg in (0, 1, 2, 3):
        c, oc = P.GEN_CONFIGS[cfg], oracle.CONFIGS[cfg]
        kind, budget = SMALL_KINDS[cfg][0], float(oc["budget"])
        M32 = oracle.generate_config(cfg, restated=restated).astype(np.float32)
        M64 = M32.astype(np.float64)
        norm = float(np.sqrt((M64 * M64).sum()))
        e = {"shape": f"{c['h']}x{c['w']} x n={c['n']}, r={c['r']}, {c['levels']} levels", "kind": kind,
             "budget": f"work:{budget:g}"}
        cpu, gpu = {}, {}
        if ref is not None:
            for cyc in ("none", "ni", "vc", "fmg"):
                L = 1 if cyc == "none" else c["levels"]
                t0 = time.perf_counter()
                _, _, tr = ref.run_configuration(M64, c["h"], c["w"], L, kind, cyc, c["r"], 0, budget, 1)
                wall = time.perf_counter() - t0
                cpu[cyc] = (tr, wall)
            target = float(cpu["none"][0].error[-1]) / norm
        with P.Session(device=local, dtype=P.F32) as s:
            s.set_data(M32, P.ImageGrid(c["h"], c["w"]))
            s.run_configuration(c["levels"], kind, "fmg", c["r"], 0, 4.0, 1)  # warm-up (buffers, graphs)
            for cyc in ("none", "ni", "vc", "fmg"):
                L = 1 if cyc == "none" else c["levels"]
                with P.Session(device=local, dtype=P.F32) as s2:  # fresh pyramid: its build is timed
                    s2.set_data(M32, P.ImageGrid(c["h"], c["w"]))
                    s2.sync()
                    t0 = time.perf_counter()
                    tr = s2.run_configuration(L, kind, cyc, c["r"], 0, budget, 1)
                    wall = time.perf_counter() - t0
                gpu[cyc] = (tr, wall)
        if ref is None:
            target = float(gpu["none"][0].error[-1]) / norm
        e["target_rel_error"] = target

        def hit(tr, wall):
            rel = tr.error / norm
            el = tr.elapsed_s if hasattr(tr, "elapsed_s") else tr.elapsed  # product / oracle trace
            k = np.nonzero((tr.level == 1) & (rel <= target * (1 + 1e-9)))[0]
            setup = wall - float(el[-1])
            return (setup + float(el[k[0]])) if len(k) else None, wall

        for cyc in ("none", "ni", "vc", "fmg"):
            g_t, g_wall = hit(*gpu[cyc])
            row = {"gpu_time_to_target_s": g_t, "gpu_wall_s": g_wall,
                   "gpu_final_rel_error": float(gpu[cyc][0].error[-1]) / norm}
            if ref is not None:
                c_t, c_wall = hit(*cpu[cyc])
                tg, tc = gpu[cyc][0], cpu[cyc][0]
                same = len(tg.error) == len(tc.error) and np.array_equal(tg.level, tc.level)
                row.update(cpu_time_to_target_s=c_t, cpu_wall_s=c_wall,
                           cpu_final_rel_error=float(tc.error[-1]) / norm,
                           same_schedule=bool(same and np.allclose(tg.work_units, tc.work)),
                           max_rel_dev=float(np.max(np.abs(tg.error - tc.error) / tc.error)) if same else None)
                if c_t and g_t:
                    row["speedup_time_to_target"] = c_t / g_t
            e[cyc] = row
        if ref is not None:
            e["cpu_cores"] = os.cpu_count() or 1
        out[f"config{cfg}_{kind}"] = e
    return out


def time_to_target(P, local, gemm):
    """Time-to-target relative error: target = the
    single-level (cycle none) final relative error at work:20; report the
    elapsed time of the first finest-level sample at or below it for none and
    NI / VC / FMG (5 levels), traced every 2 steps."""
    out = {}
    with P.Session(device=local, dtype=P.F32, gemm_path=gemm) as s:
        s.generate(CFG, seed=0)
        norm = float(np.sqrt(s.norm2(0)))
        runs = {"none": s.run_configuration(1, "hals", "none", RANK, 0, 20.0, 2)}
        # the R(M) pyramid (GridHierarchy::build, transfer.cpp:155-174), timed
        # once; the multilevel runs below reuse it, so it is added to their
        # time-to-target (pyramid_s)
        s.sync()
        t0 = time.perf_counter()
        s.build_levels(LEVELS)
        s.sync()
        out["pyramid_s"] = time.perf_counter() - t0
        target = float(runs["none"].error[-1]) / norm
        for cyc in ("ni", "vc", "fmg"):
            runs[cyc] = s.run_configuration(LEVELS, "hals", cyc, RANK, 0, 20.0, 2)
        out["target_rel_error"] = target
        for cyc, tr in runs.items():
            rel = tr.error / norm
            hit = np.nonzero((tr.level == 1) & (rel <= target * (1 + 1e-12)))[0]
            t_hit = float(tr.elapsed_s[hit[0]]) if len(hit) else None
            out[cyc] = {"time_s": t_hit,
                        "time_s_incl_pyramid": (t_hit + (out["pyramid_s"] if cyc != "none" else 0.0))
                        if t_hit is not None else None,
                        "final_rel_error": float(rel[-1]), "total_s": float(tr.elapsed_s[-1]),
                        "phase_steps": tr.phase_steps.tolist()}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--gemm", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--e2e-iters", type=int, default=20)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-ttt", dest="ttt", action="store_false")
    ap.add_argument("--no-small", dest="small", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
