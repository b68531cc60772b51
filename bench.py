#!/usr/bin/env python
"""Benchmark of the Hilbert-reordered SEM leapfrog step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

One "step" = one leapfrog time step of the whole hot path (stiffness apply with
gather + conflict-free scatter, M^-1 scaling, Ricker source, update) over the
configured mesh.  Workload: BASELINE.json configs[3] (C4, 2048 x 2048 cells per
GPU, P3) -- the weak-scaling configuration the metric's 1/2/4/8-GPU numbers and
the >= 60 % HBM roofline target are quoted on; its per-step working set
(~1.75 GB) is far larger than the 126 MB L2, so no flush is needed between
steps.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "element-updates/sec per time step and achieved HBM GB/s fraction, 1/2/4/8 B200"
UNIT = "element-updates/s"


def load_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)", {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def problem_for(name: str, world: int):
    from paper_2104_08416_b200 import meshgen as mg
    return mg.config(name, 1, gpus=world) if name == "C4" else mg.config(name, 1)


def ncu_traffic(config, kernel):
    """DRAM bytes (read + write) of one launch of `kernel` on `config`, from the
    committed `ncu --set full` capture summarised in profiles/traffic_<config>.json
    (None if there is none).  Not measured in this run: ncu perturbs timing."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_%s.json" % config)) as f:
            d = json.load(f)[kernel]
        return float(d["traffic_bytes"]) / 1e9
    except Exception:
        return None


def graph_split(steps):
    """sem_step_n's one-rank graph replays (api.cu) after the warm-up's sem_step_n(0) captured
    them all: (size, replays) for the graphs of 32, 16, 8, 4, 2 and 1 steps."""
    out, left = [], steps
    for sz in (32, 16, 8, 4, 2, 1):
        if left // sz:
            out.append((sz, left // sz))
            left -= (left // sz) * sz
    return out


def gpu_launches(steps, info, world):
    """Kernels of this library launched in the timed region: per step K7 + K8
    (+ the interface kernels with several ranks); the one-rank graph loop adds a
    step-counter kernel per captured step and one counter reset per graph size used."""
    if world == 1 and os.environ.get("SEM_GRAPH", "1") != "0":
        return int(steps * 3 + len(graph_split(steps)))
    return int(steps * info["launches_per_step"])


def k7_bytes(info):
    """Algorithmic bytes per launch of K7 / K8."""
    E, Np, N = info["n_elements"], info["nodes_per_elem"], info["n_nodes"]
    Nint, Nsh = info["n_interior_nodes"], info["n_shared_nodes"]
    k7 = E * (4 * Np + 24) + 8 * N + 24 * Nint
    k8 = 24 * Nsh
    return float(k7), float(k8)


def _make_ctx(S, local, rank, world, stream, dist):
    nccl_id = None
    if world > 1:
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    return S.SemContext(local, rank, world, nccl_id=nccl_id, stream=stream.cuda_stream)


def _max_over_ranks(dist, x):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch
    from paper_2104_08416_b200 import sem as S

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # a real (non-default) stream shared by libsem and the torch events
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    peak, peak_src, peaks = load_peak()

    # weak scaling: the global C4 mesh grows with the GPU count (2048^2 cells per GPU)
    pb = problem_for(args.config, world)
    m = pb.mesh
    ctx = _make_ctx(S, local, rank, world, stream, dist)
    ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH)
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, pb.amplitude, pb.dt)
    info = ctx.sem_get_info()
    E_glob = info["n_elements_global"]

    # sem_step_n(0) captures the step loop's CUDA graphs outside the timed region; the clock
    # sampler starts next, and the W warm-up steps run right before the timed region (after the
    # sampler's start-up pause, so the timed steps do not begin on an idle GPU)
    ctx.sem_step_n(0)
    ctx.sem_sync()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ctx.sem_step_n(args.warmup)
    ctx.sem_sync()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0.record(stream)
    ctx.sem_step_n(args.steps)  # the product path (one rank: CUDA-graph step loop)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    # per-kernel CUDA events for the roofline: a second pass through the same CUDA-graph step
    # loop, captured with event-record nodes around every K7 and K8 (whole replays of 32 steps)
    ctx.sem_set_kernel_timing(True)
    ctx.sem_step_n(max(32, min(args.steps, 400) // 32 * 32))
    kt = ctx.sem_kernel_times()
    ctx.sem_set_kernel_timing(False)
    clk = clocks.stop()
    ms = _max_over_ranks(dist, ms)
    U, nstep = ctx.sem_read_field()
    finite = bool(np.isfinite(U[~np.isnan(U)]).all()) if world > 1 else bool(np.isfinite(U).all())

    ms_step = ms / args.steps
    value = E_glob * args.steps / (ms / 1e3)
    b7, b8 = k7_bytes(info)
    if kt["k8_launches"] == 0:  # K8 fused into K7: shared nodes are finalised there too
        b7, b8 = b7 + b8, 0.0
    k7_avg = kt["k7_ms"] / max(kt["k7_launches"], 1)
    k8_avg = kt["k8_ms"] / max(kt["k8_launches"], 1)
    achieved = b7 / (k7_avg * 1e-3) / 1e9
    step_gbs = info["bytes_alg_per_step"] / (ms_step * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if args.config == "C4" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded meshgen recipe, DESIGN.md)",
        "config": {"workload": "%s: %s" % (args.config, WORKLOADS.get(args.config, "")),
                   "elements_global": E_glob, "elements_per_gpu": info["n_elements"],
                   "nodes_global": info["n_nodes_global"], "nodes_rank0": info["n_nodes"], "degree": pb.P,
                   "ordering": "hilbert elements + first-touch nodes",
                   "parallelism": ("contiguous Hilbert-range partition, NCCL interface exchange (%d ranks)" % world
                                   if world > 1 else "1 GPU"),
                   "interface_nodes_rank0": info["n_interface_nodes"], "neighbors_rank0": info["n_neighbors"],
                   "l2": "no flush: per-step working set %.2f GB per GPU > 126 MB L2" % (info["bytes_alg_per_step"] / 1e9),
                   "chunk_elems": info["chunk_elems"], "shared_node_frac": info["n_shared_nodes"] / info["n_nodes"],
                   "step_loop": step_loop_label(args.steps, world),
                   "dt": pb.dt},
        "roofline": {"bound": "hbm", "kernel": "k7_step (stiffness apply + fused leapfrog)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": peak_src, "traffic": ncu_traffic(args.config, "k7_step"),
                     "traffic_unit": "GB per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum, profiles/)",
                     "bytes_per_launch": b7, "avg_launch_ms": k7_avg,
                     "k7_share_of_step": kt["k7_ms"] / max(kt["k7_ms"] + kt["k8_ms"], 1e-9),
                     "timing_pass_steps": kt["k7_launches"],
                     "k8_avg_launch_ms": k8_avg, "k8_bytes_per_launch": b8},
        "step_alg_gbs": step_gbs, "step_alg_frac": step_gbs / peak,
        "step_alg_frac_of_8tbs": step_gbs / 8000.0,
        "gpu_launches": gpu_launches(args.steps, info, world),
        "clocks": clk,
        "prep_ms": {"mesh_reorder": info["prep_reorder_ms"], "build_operators": info["prep_build_ms"]},
        "field_finite": finite,
    }
    ctx.close()
    # the end-to-end leg right after the main measurement, before the other legs
    # churn host and device memory
    if args.e2e:
        out["e2e"] = e2e(pb, args, S, local, rank, world, stream, dist)
    if rank == 0 and world == 1 and (args.orderings or args.heun or args.orders or args.configs):
        ctx = S.SemContext(local, stream=stream.cuda_stream)
        if args.configs:
            out["configs"] = configs_leg(ctx, args, S, peak)
        if args.orderings:
            out["orderings"] = orderings(ctx, pb, args, S)
            out["scatter_ablation"] = scatter_ablation(ctx, pb, args, S)
        if args.heun:
            out["heun"] = heun_leg(ctx, pb, args, S, peak)
        if args.orders:
            out["orders_5_7"] = orders_leg(ctx, args, S, peak, peaks)
        ctx.close()
    if rank == 0 and world == 1 and args.cpu:
        out["cpu_baseline"] = cpu_baseline(pb)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def step_loop_label(steps, world):
    """How sem_step_n(steps) launches (api.cu: sem_step_n): one rank replays captured CUDA
    graphs of 32 steps for each whole block of 32, then one of 16, 8, 4, 2, 1 steps each as
    needed for the rest."""
    if world > 1 or os.environ.get("SEM_GRAPH", "1") == "0":
        return "stream launches (%d steps)" % steps
    parts = ["%d replay%s of a %d-step CUDA graph" % (n, "s" if n > 1 else "", sz) for sz, n in graph_split(steps)]
    return " + ".join(parts) or "none"


WORKLOADS = {
    "C1": "32x32 cells [0,1]^2 +-0.2h jitter, P2, c=1, Ricker 10 Hz",
    "C2": "512x512 cells [0,4000]^2 m +-0.25h jitter, P3, c=2000 m/s, Ricker 15 Hz",
    "C3": "graded 2000x1000 cells over [0,8000]x[0,4000] m, 3 layers, P3, Ricker 10 Hz",
    "C4": "2048x2048 cells per GPU (h=7.8125 m) +-0.25h jitter, P3, c=2000 m/s, Ricker 15 Hz",
    "C5": "graded 16384x8192 cells, 10 random layers, P2, Ricker 10 Hz",
}


def orderings(ctx, pb, args, S):
    """Hilbert vs random vs natural, same physical mesh (1 GPU)."""
    import torch
    res = {}
    K = max(50, min(args.steps, 400))
    variants = [
        ("hilbert", pb.mesh, pb.c, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH),
        ("hilbert_canonical_nodes", pb.mesh, pb.c, S.SEM_ORDER_HILBERT, S.SEM_NODES_CANONICAL),
        ("natural", pb.natural, pb.c_natural, S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
        ("random", pb.mesh, pb.c, S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
        # the paper's other strategies (reading R20) and the
        # degree-sorted node renumbering (reading R12)
        ("conn", pb.mesh, pb.c, S.SEM_ORDER_CONN, S.SEM_NODES_VISIT),
        ("dist", pb.mesh, pb.c, S.SEM_ORDER_DIST, S.SEM_NODES_VISIT),
        ("hilbert_degree_sorted_nodes", pb.mesh, pb.c, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH_DEGREE),
    ]
    stream = torch.cuda.current_stream()
    assert stream.cuda_stream != 0
    for name, m, c, eo, no in variants:
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, eo, no)
        src = pb.src_vertex if m is pb.mesh else int(pb.mesh.vert_perm[pb.src_vertex])
        ctx.sem_build_operators(c, src, pb.f0, pb.t0, pb.amplitude, pb.dt)
        ctx.sem_step_n(5)
        ctx.sem_set_kernel_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.sem_step_n(K)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        kt = ctx.sem_kernel_times()
        ctx.sem_set_kernel_timing(False)
        info = ctx.sem_get_info()
        res[name] = {"element_updates_per_s": info["n_elements"] / (ms * 1e-3), "ms_per_step": ms,
                     "alg_gbs": info["bytes_alg_per_step"] / (ms * 1e-3) / 1e9,
                     "k7_ms": kt["k7_ms"] / max(kt["k7_launches"], 1),
                     "k8_ms": kt["k8_ms"] / max(kt["k8_launches"], 1),
                     "shared_node_frac": info["n_shared_nodes"] / info["n_nodes"],
                     "max_chunk_nodes": info["max_chunk_nodes"], "steps": K,
                     "prep_reorder_ms": info["prep_reorder_ms"]}
    return res


def scatter_ablation(ctx, pb, args, S):
    """NEXT-4: the product's chunk-owned scatter vs fp64 atomics vs the paper's
    global element colouring, same mesh, Hilbert order."""
    import torch
    res = {}
    K = max(50, min(args.steps, 200))
    stream = torch.cuda.current_stream()
    m = pb.mesh
    for name, mode in [("chunk", S.SEM_SCATTER_CHUNK), ("atomic", S.SEM_SCATTER_ATOMIC),
                       ("color", S.SEM_SCATTER_COLOR)]:
        ctx.sem_set_scatter(mode)
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, pb.amplitude, pb.dt)
        ctx.sem_step_n(5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.sem_step_n(K)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        info = ctx.sem_get_info()
        res[name] = {"element_updates_per_s": info["n_elements"] / (ms * 1e-3), "ms_per_step": ms,
                     "alg_gbs": info["bytes_alg_per_step"] / (ms * 1e-3) / 1e9,
                     "launches_per_step": info["launches_per_step"], "global_colors": info["n_global_colors"],
                     "steps": K}
    ctx.sem_set_scatter(S.SEM_SCATTER_CHUNK)
    return res


def fp64_peak():
    """Measured FP64 FMA throughput (tools/dfma_peak.cu -> profiles/dfma_peak.json),
    else the nominal 148 SMs x 64 DFMA/clk x 2 flop x 1.965 GHz."""
    try:
        with open(os.path.join(ROOT, "profiles", "dfma_peak.json")) as f:
            return float(json.load(f)["fp64_fma_tflops"]), "measured (profiles/dfma_peak.json)"
    except Exception:
        return 148 * 64 * 2 * 1.965e9 / 1e12, "nominal 148 x 64 DFMA/clk x 1.965 GHz"


FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE = fp64_peak()


# The other BASELINE.json configurations at one GPU, each with its own roofline line (SURVEY
# §8(d): quote C3 and C5 beside the headline C4).  C5 runs at 1/4 linear size here (16.8 M P2
# elements of the same graded, 10-layer recipe; about half its per-GPU share at 8 GPUs): the
# full 268 M-element mesh takes minutes of host-side generation alone.
CONFIG_LEG = [("C2", 1), ("C3", 1), ("C5", 4)]


def configs_leg(ctx, args, S, peak):
    import torch
    from paper_2104_08416_b200 import meshgen as mg
    res = {}
    stream = torch.cuda.current_stream()
    for name, scale in CONFIG_LEG:
        pb = mg.config(name, scale)
        m = pb.mesh
        ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, pb.amplitude, pb.dt)
        ctx.sem_step_n(max(3, args.warmup))
        ctx.sem_step_n(0)  # capture the graph step loop outside the timed region
        K = max(64, min(args.steps, 1024)) // 32 * 32
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.sem_step_n(K)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        ctx.sem_set_kernel_timing(True)
        ctx.sem_step_n(min(K, 256))
        kt = ctx.sem_kernel_times()
        ctx.sem_set_kernel_timing(False)
        info = ctx.sem_get_info()
        b7, b8 = k7_bytes(info)
        k7 = kt["k7_ms"] / max(kt["k7_launches"], 1)
        k8 = kt["k8_ms"] / max(kt["k8_launches"], 1)
        ach = b7 / (k7 * 1e-3) / 1e9
        step_gbs = info["bytes_alg_per_step"] / (ms * 1e-3) / 1e9
        res[name if scale == 1 else "%s/%d" % (name, scale)] = {
            "workload": WORKLOADS[name] + ("" if scale == 1 else " (1/%d linear size)" % scale),
            "elements": info["n_elements"], "degree": pb.P, "steps": K,
            "element_updates_per_s": info["n_elements"] / (ms * 1e-3), "ms_per_step": ms,
            "roofline": {"bound": "hbm", "kernel": "k7_step", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": ncu_traffic(name, "k7_step"), "bytes_per_launch": b7,
                         "avg_launch_ms": k7},
            "k8_avg_launch_ms": k8, "k8_bytes_per_launch": b8,
            "step_alg_gbs": step_gbs, "step_alg_frac": step_gbs / peak,
            "shared_node_frac": info["n_shared_nodes"] / info["n_nodes"],
            "l2": "C2's 109 MB per step fits the 126 MB L2 (no flush: quoted as is)" if name == "C2" else
                  "working set > L2"}
    return res


def orders_leg(ctx, args, S, peak, peaks):
    """NEXT-2: the paper's Benchmark 1 shape (2000 x 1000 units, 1M elements,
    PAPER.md:572) at its orders 5-7 and 4 (readings R21,
    R21b), Hilbert vs the shuffled file order ("None").  FP64-bound from P5 on
    (DESIGN.md)."""
    import torch
    from paper_2104_08416_b200 import meshgen as mg
    res = {}
    stream = torch.cuda.current_stream()
    for P in (4, 5, 6, 7):
        pb = mg.config("B1", 1, degree=P)
        Np = (P + 1) * (P + 2) // 2
        flop_elem = 2.0 * (3 * Np * (Np + 1) / 2 + Np * Np)  # K^e entries (2 FMA + MUL) + symmetric mat-vec
        for name, eo, no in [("hilbert", S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH),
                             ("none", S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL)]:
            ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, P, eo, no)
            ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, pb.amplitude, pb.dt)
            ctx.sem_step_n(5)
            K = max(50, min(args.steps, 300))
            ctx.sem_set_kernel_timing(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            ctx.sem_step_n(K)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
            kt = ctx.sem_kernel_times()
            ctx.sem_set_kernel_timing(False)
            info = ctx.sem_get_info()
            k7 = kt["k7_ms"] / max(kt["k7_launches"], 1)
            b7, _ = k7_bytes(info)
            tf = info["n_elements"] * flop_elem / (k7 * 1e-3) / 1e12
            res["P%d_%s" % (P, name)] = {
                "elements": info["n_elements"], "element_updates_per_s": info["n_elements"] / (ms * 1e-3),
                "ms_per_step": ms, "k7_ms": k7, "k8_ms": kt["k8_ms"] / max(kt["k8_launches"], 1),
                "alg_gbs": info["bytes_alg_per_step"] / (ms * 1e-3) / 1e9,
                "k7_hbm_frac": b7 / (k7 * 1e-3) / 1e9 / peak,
                "k7_fp64_tflops": tf, "k7_fp64_frac": tf / FP64_PEAK_TFLOPS,
                "fp64_peak_tflops": FP64_PEAK_TFLOPS, "fp64_peak_source": FP64_PEAK_SOURCE, "steps": K}
    # the paper's own Benchmark 1 workload: Heun, orders 5 and 7, 1M elements
    # (Table avg_cpu_time_orders_exp_1)
    for P, name, eo, no in [(5, "hilbert", S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH),
                            (5, "none", S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL),
                            (7, "hilbert", S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH),
                            (7, "none", S.SEM_ORDER_INPUT, S.SEM_NODES_CANONICAL)]:
        pb = mg.config("B1", 1, degree=P)
        ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
        ctx.sem_mesh_reorder(pb.mesh.vxy, pb.mesh.tri, P, eo, no)
        ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, pb.amplitude, pb.dt * 0.2)
        ctx.sem_step_n(5)
        K = max(50, min(args.steps, 300))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        ctx.sem_step_n(K)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        info = ctx.sem_get_info()
        ctx.sem_set_integrator(S.SEM_INTEGRATOR_LEAPFROG)
        # PAPER.md:764-770 (1M elements, 32 threads): order 5 SFC 1.465 s / None 1.736 s, order 7 3.414 / 4.010
        paper_s = {(5, "hilbert"): 1.465, (5, "none"): 1.736, (7, "hilbert"): 3.414, (7, "none"): 4.010}[(P, name)]
        res["P%d_heun_%s" % (P, name)] = {
            "elements": info["n_elements"], "element_updates_per_s": info["n_elements"] / (ms * 1e-3),
            "ms_per_step": ms, "alg_gbs": info["bytes_alg_per_step"] / (ms * 1e-3) / 1e9, "steps": K,
            "paper_context": {"s_per_step": paper_s, "machine": "Xeon E5-2698 v3, 32 threads",
                              "source": "PAPER.md:764-770 (Table avg_cpu_time_orders_exp_1, SFC / None)",
                              "ratio_to_paper": paper_s / (ms * 1e-3)}}
    return res


def heun_bytes(info):
    """Algorithmic bytes per launch of the Heun element pass KH7 / fix-up KH8
    (DESIGN.md "Heun"): per element mu (4 Np) + F, sd (40) + V read and write
    (32 Np); per node U, W read (16) in KH7, and (h/2)/M read + U, W write (24)
    where the node is finalised (KH7 interior, KH8 shared)."""
    E, Np, N = info["n_elements"], info["nodes_per_elem"], info["n_nodes"]
    Nint, Nsh = info["n_interior_nodes"], info["n_shared_nodes"]
    return float(E * (36 * Np + 40) + 16 * N + 24 * Nint), float(24 * Nsh)


def heun_leg(ctx, pb, args, S, peak):
    """The paper's own integrator (Heun on (U, V), NEXT-1) on the same mesh:
    one step = both RHS evaluations of PAPER.md:269-291, fused in one pass."""
    import torch
    m = pb.mesh
    K = max(50, min(args.steps, 500))
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_HEUN)
    ctx.sem_mesh_reorder(m.vxy, m.tri, pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH)
    h = pb.dt * 0.2  # reading R19 (meshgen.heun_h)
    ctx.sem_build_operators(pb.c, pb.src_vertex, pb.f0, pb.t0, pb.amplitude, h)
    ctx.sem_step_n(5)
    stream = torch.cuda.current_stream()
    ctx.sem_set_kernel_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    ctx.sem_step_n(K)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    kt = ctx.sem_kernel_times()
    ctx.sem_set_kernel_timing(False)
    info = ctx.sem_get_info()
    U, _ = ctx.sem_read_field()
    ctx.sem_set_integrator(S.SEM_INTEGRATOR_LEAPFROG)
    b7, b8 = heun_bytes(info)
    k7 = kt["k7_ms"] / max(kt["k7_launches"], 1)
    achieved = b7 / (k7 * 1e-3) / 1e9
    return {"element_updates_per_s": info["n_elements"] / (ms * 1e-3), "ms_per_step": ms, "steps": K, "h": h,
            "alg_bytes_per_step": info["bytes_alg_per_step"],
            "alg_gbs": info["bytes_alg_per_step"] / (ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": "k_heun (lagged V update + Alg. 2 + K u + fused Heun update)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "bytes_per_launch": b7, "avg_launch_ms": k7,
                         "fix_avg_launch_ms": kt["k8_ms"] / max(kt["k8_launches"], 1), "fix_bytes_per_launch": b8},
            "field_finite": bool(np.isfinite(U).all())}


def e2e(pb, args, S, device, rank, world, stream, dist):
    """The whole job through the public C ABI from pinned host buffers:
    mesh H2D + reorder + operators + K steps + field D2H, timed on the host
    around synchronising calls (inputs start in host memory); max over ranks."""
    import torch
    m = pb.mesh
    vxy = torch.from_numpy(m.vxy).pin_memory()
    tri = torch.from_numpy(m.tri).pin_memory()
    c = torch.from_numpy(pb.c).pin_memory()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    nmax = pb.mesh.nv + 3 * m.ne * (pb.P - 1) + m.ne * max(0, (pb.P - 1) * (pb.P - 2) // 2)  # >= N
    # every host buffer of the job is pinned before the timed region
    out = torch.zeros(nmax, dtype=torch.float64).pin_memory()
    reorder_out = {"keys": torch.zeros(m.ne, dtype=torch.int32).pin_memory().numpy().view(np.uint32),
                   "elem_perm": torch.zeros(m.ne, dtype=torch.int32).pin_memory().numpy(),
                   "node_perm": torch.zeros(nmax, dtype=torch.int32).pin_memory().numpy()}
    t0 = time.perf_counter()
    ctx = _make_ctx(S, device, rank, world, stream, dist)
    t_create = time.perf_counter()
    r = ctx.sem_mesh_reorder(vxy.numpy(), tri.numpy(), pb.P, S.SEM_ORDER_HILBERT, S.SEM_NODES_FIRST_TOUCH,
                             out=reorder_out)
    t_reorder = time.perf_counter()
    ctx.sem_build_operators(c.numpy(), pb.src_vertex, pb.f0, pb.t0, pb.amplitude, pb.dt)
    t_build = time.perf_counter()
    ctx.sem_step_n(args.steps)
    ctx.sem_sync()
    t_steps = time.perf_counter()
    ctx.sem_read_field(out=out.numpy()[: r["n_nodes"]])
    t1 = time.perf_counter()
    ctx.close()
    secs = _max_over_ranks(dist, t1 - t0)
    E = m.ne
    h2d = m.vxy.nbytes + m.tri.nbytes + pb.c.nbytes + (r["n_nodes"] * 8 if world > 1 else 0)
    d2h = r["n_nodes"] * 8 + E * 8 + r["n_nodes"] * 4
    phases = {"create": t_create - t0, "mesh_reorder": t_reorder - t_create, "build_operators": t_build - t_reorder,
              "steps": t_steps - t_build, "read_field": t1 - t_steps}
    return {"value": E * args.steps / secs, "unit": UNIT, "seconds": secs, "phases_s_rank0": phases,
            "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
            "includes": "sem_mesh_reorder + sem_build_operators + sem_step_n(K) + sem_read_field"}


def cpu_baseline(pb, steps=2):
    """The oracle, as it stands, on this host's cores: a bounded sample of the
    same workload (a few leapfrog steps of the full mesh)."""
    from oracle import core
    from oracle.core import OracleSEM
    m = pb.mesh
    t0 = time.perf_counter()
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    setup = time.perf_counter() - t0
    o.leapfrog(pb.dt, 1, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0)  # warm-up
    t0 = time.perf_counter()
    o.leapfrog(pb.dt, steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0)
    dt = time.perf_counter() - t0
    cores = core.num_threads()
    # also one thread on C1-C2 (C2 recipe, 2 steps)
    from paper_2104_08416_b200 import meshgen as mg
    c2 = mg.config("C2", 1)
    o2 = OracleSEM(c2.mesh.vxy, c2.mesh.tri, c2.P, c2.c)
    core.set_num_threads(1)
    try:
        o2.leapfrog(c2.dt, 1, src=c2.src_vertex, A=1.0, f0=c2.f0, t0=c2.t0)
        t1 = time.perf_counter()
        o2.leapfrog(c2.dt, 2, src=c2.src_vertex, A=1.0, f0=c2.f0, t0=c2.t0)
        one = c2.mesh.ne * 2 / (time.perf_counter() - t1)
    finally:
        core.set_num_threads(cores)
    return {"value": m.ne * steps / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": "%d leapfrog steps of the full %s mesh (%d elements), oracle setup %.1f s excluded"
                      % (steps, pb.name, m.ne, setup),
            "cpu": _cpu_model(),
            "one_thread_C2": {"value": one, "unit": UNIT, "cores": 1,
                              "sample": "2 leapfrog steps of the full C2 mesh (524288 elements, P3)"}}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    """--impl reference: the oracle (the reference arm of this tier), timed as it
    stands on the host cores, on a bounded sample of the same workload recipe.

    The sample is the same recipe at a reduced cell count per axis, chosen from
    a short calibration so that the W + K oracle steps take about a minute."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import core
    from oracle.core import OracleSEM
    from paper_2104_08416_b200 import meshgen as mg
    budget_s = 60.0
    # torchrun exports OMP_NUM_THREADS=1 to every rank; rank 0 is the only one that works here,
    # so it takes the host's cores as the N=1 launch (plain `python bench.py`) does
    if "TORCHELASTIC_RUN_ID" in os.environ and os.environ.get("OMP_NUM_THREADS") == "1":
        core.set_num_threads(len(os.sched_getaffinity(0)))
    nthr = core.num_threads()
    # calibrate the oracle's element-update rate on a small sample of the recipe
    cal = mg.config(args.config, 16)
    oc = OracleSEM(cal.mesh.vxy, cal.mesh.tri, cal.P, cal.c)
    oc.leapfrog(cal.dt, 1, src=cal.src_vertex, A=1.0, f0=cal.f0, t0=cal.t0)
    t0 = time.perf_counter()
    oc.leapfrog(cal.dt, 3, src=cal.src_vertex, A=1.0, f0=cal.f0, t0=cal.t0)
    rate = 3 * cal.mesh.ne / (time.perf_counter() - t0)
    full_e = problem_elems(args.config)
    scale = 1
    while full_e / (scale * scale) * (args.steps + args.warmup) / rate > budget_s and scale < 64:
        scale *= 2
    pb = mg.config(args.config, scale)
    m = pb.mesh
    o = OracleSEM(m.vxy, m.tri, pb.P, pb.c)
    U, Up = o.leapfrog(pb.dt, args.warmup, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0)
    t0 = time.perf_counter()
    o.leapfrog(pb.dt, args.steps, src=pb.src_vertex, A=1.0, f0=pb.f0, t0=pb.t0, U=U, Uprev=Up,
               step0=args.warmup)
    dt = time.perf_counter() - t0
    value = m.ne * args.steps / dt
    sample = ("%s recipe at 1/%d cells per axis (%d elements of %d), %d steps on %d host threads"
              % (args.config, scale, m.ne, full_e, args.steps, nthr))
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": "%s: %s" % (args.config, WORKLOADS.get(args.config, "")),
                                           "sample": sample},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthr, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def problem_elems(name):
    return {"C1": 2048, "C2": 524288, "C3": 4000000, "C4": 8388608, "C5": 268435456}[name]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-orderings", dest="orderings", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-heun", dest="heun", action="store_false")
    ap.add_argument("--no-orders", dest="orders", action="store_false")
    ap.add_argument("--no-configs", dest="configs", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
