"""Benchmark: Parallel Evoformer train step (fwd + loss + bwd) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

Workload (BASELINE.json configs[1]): one Parallel Evoformer block at the
AF2 initial-training shape s=128 r=256 c_m=256 c_z=128 h=8 c_opm=32 t=4,
bf16 operands / fp32 accumulation and residual streams, synthetic N(0,1)
inputs (make_batch seed 32), random-init weights (init_params seed 32).
A step = forward + loss + backward with every parameter gradient.

Metric: Evoformer train samples/s (whole job); also fwd+bwd ms per block.
Multi-GPU (torchrun, one rank per GPU): BP=2 x DP=N/2 (N even) with the
branch exchange over NCCL; N=1 is BP=1.  value = samples processed by all
ranks / max-over-ranks device time.

--impl reference times the reference algorithm's CPU implementation (the
pinned numpy oracle port, oracle/evoformer_np.py) on the host cores.

Other SURVEY.md §8(d) configurations (1 GPU): --crop R (C5 crop sweep,
r = 128 / 384), --stack [--blocks K] (C3: the 4-block extra-MSA stack,
s_e=1024 c_e=64, feeding a K-block main stack, default 48).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "af2": dict(s=128, r=256, c_m=256, c_z=128, h=8, c_opm=32, t_factor=4, n_blocks=1),
    "mid": dict(s=32, r=64, c_m=64, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=1),
    "c1": dict(s=16, r=32, c_m=32, c_z=16, h=4, c_opm=8, t_factor=4, n_blocks=2),
}
METRIC = "Evoformer train samples/sec (BP=1 vs BP=2, 1/2/4/8 B200); fwd+bwd ms/block"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port, sampled sub-op by sub-op
# ---------------------------------------------------------------------------

def cpu_sample(kw, budget_s=60.0, reps=1):
    """Fwd+bwd of each of the nine sub-ops at the full shape, fp32 numpy
    on all host cores; block time = sum of the sub-op times (the residual
    adds are negligible).  Returns (seconds per block, details)."""
    import numpy as np
    from oracle import evoformer_np as O
    d = O.Dims(**{**kw, "n_blocks": 1})
    P = O.init_params(d, 32, dtype=np.float32)
    m, z = O.make_batch(d, 32, 1, dtype=np.float32)[0]
    rng = np.random.default_rng(0)
    times = {}
    for name in O.SUBOPS:
        px = f"blk0.{name}"
        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            delta, cache = O.subop_fwd(name, P, px, m, z, d)
            R = rng.standard_normal(delta.shape).astype(np.float32)
            O.subop_vjp(name, R, cache, P, px, d, O.Grads())
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        times[name] = best
    return sum(times.values()), times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    kw = CONFIGS[args.config]
    cores = os.cpu_count()
    # each "step" is one full-block sample (the nine sub-ops, ~10 s on 16
    # cores); bounded to 1 warm-up + 3 timed samples so the run stays short
    warm = min(max(args.warmup, 0), 1)
    for _ in range(warm):
        cpu_sample(kw)
    per = []
    for _ in range(max(1, min(args.steps, 3))):
        t, _ = cpu_sample(kw)
        per.append(t)
    t = min(per)
    value = kw["n_blocks"] / t / kw["n_blocks"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": len(per), "warmup": warm, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"parallel_evoformer_block_{args.config}",
                                        **kw, "precision": "fp32 numpy"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": "fwd+bwd of each of the 9 sub-ops once at full shape "
                                   "(oracle/evoformer_np.py, numpy fp32, all cores); "
                                   "block time = sum"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, 0
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                reasons |= int(parts[3], 16)
            except ValueError:
                continue
        if not sm:
            return None
        sm.sort()
        names = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                 0x100: "display_clock_setting"}
        rs = [v for k, v in names.items() if reasons & k]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": rs,
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# BP=2 prediction from one GPU: the two branches timed separately
# ---------------------------------------------------------------------------

NVLINK_GBS = 750.0   # assumed achievable NVLink 5 bandwidth per direction (900 nominal)


def bp2_prediction(cfg, store, precision, dev, bp1_block_ms, reps=20):
    """Per block: the MSA branch (row / column attention, MSA transition,
    outer product mean; fwd + bwd) and the pair branch (triangle updates,
    triangle attentions, pair transition; fwd + bwd) each replayed as a CUDA
    graph and timed with events, plus the block's four fp32 Z-sized BP
    messages (fwd: o, z''; bwd: dz'', the dz_in allreduce) at NVLINK_GBS.
    BP=2 block time = max(branches) + exchange (src/schedules.py:214-297:
    the exchange is not overlapped)."""
    import torch
    from paper_2211_00235_b200 import distributed as D
    ex = D.CudaExec(cfg, store, precision, dev)
    ex.pack("all")
    s, r = cfg.s, cfg.r
    g = torch.Generator(device=dev).manual_seed(0)
    m = torch.randn(s * r, cfg.c_m, device=dev, generator=g)
    z = torch.randn(r * r, cfg.c_z, device=dev, generator=g)
    dm = torch.randn(s * r, cfg.c_m, device=dev, generator=g) * 1e-3
    dz = torch.randn(r * r, cfg.c_z, device=dev, generator=g) * 1e-3

    def msa():
        _, _, ctx = ex.msa_fwd(0, m, z)
        ex.msa_bwd(0, ctx, dm, dz)

    def pair():
        _, ctx = ex.pair_fwd(0, z)
        ex.pair_bwd(0, ctx, dz)

    out = {}
    for name, fn in (("msa_branch_ms", msa), ("pair_branch_ms", pair)):
        fn()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            fn()
        graph.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
        del graph
    zbytes = r * r * cfg.c_z * 4
    exch_ms = 4 * zbytes / (NVLINK_GBS * 1e9) * 1e3
    bp2 = max(out["msa_branch_ms"], out["pair_branch_ms"]) + exch_ms
    out.update(bp1_block_ms=bp1_block_ms, exchange_bytes_per_block=4 * zbytes,
               exchange_ms_at_assumed_nvlink=exch_ms, assumed_nvlink_gbs=NVLINK_GBS,
               predicted_bp2_block_ms=bp2, predicted_bp2_speedup=bp1_block_ms / bp2,
               paper_bp2_speedup="1.37-1.39x (PAPER.md, UniFold/PPFold on A100)",
               method="each branch's fwd+bwd of one block replayed as a CUDA graph on this "
                      "GPU; BP=2 block = max(branches) + 4 fp32 Z messages at the assumed "
                      "NVLink rate")
    return out


# ---------------------------------------------------------------------------
# native arm
# ---------------------------------------------------------------------------

def run_native(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2211_00235_b200 as pkg
    from paper_2211_00235_b200 import _native, kernels as K, schedules as S
    from oracle import evoformer_np as O

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:   # gloo: ranks may share one GPU (checks the N > 1 code path)
            dist.init_process_group("gloo")
    kw = CONFIGS[args.config]
    if args.blocks:
        kw = {**kw, "n_blocks": args.blocks}
    if args.crop:
        kw = {**kw, "r": args.crop}
    cfg = pkg.EvoConfig(**kw)
    store = pkg.init_params(cfg, 32, device=dev)
    bp = 2 if (world > 1 and world % 2 == 0 and not args.dp_only) else 1
    dp = world // bp
    layout = S.ParallelLayout(dp=dp, bp=bp)
    runner = None
    if world > 1:
        # BP=2 x DP (or DP only): each compute segment between two collectives
        # replays as a CUDA graph (distributed.GraphedExec); the collectives
        # are host-issued NCCL calls
        from paper_2211_00235_b200 import distributed as D
        runner = D.DistributedStep(cfg, store, layout, precision=args.precision,
                                   graphs=args.graph)
    else:
        st = S.StepState(cfg, store, args.precision, dev)
        st.pack()
    dp_i = layout.coords(rank)[0]
    m_h, z_h = S.make_batch(cfg, 32 + dp_i, 1, device="cpu")[0]
    m_h, z_h = m_h.pin_memory(), z_h.pin_memory()
    m_d, z_d = m_h.to(dev), z_h.to(dev)
    loss_h = torch.empty(1, dtype=torch.float32).pin_memory()

    def step_eager(m, z):
        if runner is not None:
            return runner.step(m, z)
        return S.full_step(st, m, z)

    # warm-up (first-touch allocations; for N > 1 the first two steps are the
    # eager warm-up and the segment capture)
    launches_eager_step = None
    for w in range(args.warmup):
        n_w = _native.launch_count()
        step_eager(m_d, z_d)
        if w == 0:   # the first step is eager in every mode: its launch count
            launches_eager_step = _native.launch_count() - n_w
    torch.cuda.synchronize()

    use_graph = args.graph
    gs = None
    if use_graph and runner is None:
        # one train step captured as a CUDA graph by the package
        # (StepState.capture), two slots with their own static inputs for the
        # double-buffered end-to-end input pipeline
        gs = st.capture(m_d, z_d, warmup=0, slots=2)
        step_graph = lambda: gs.step(*gs.inputs(0), slot=0)
    else:
        step_graph = lambda: step_eager(m_d, z_d)

    def timed(fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(k):
            fn()
        a1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = a0.elapsed_time(a1) / k
        if world > 1:
            tt = torch.tensor([t], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    # timed region (device-resident inputs), clocks sampled during it
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    ms = timed(step_graph, args.steps)
    clk = clocks.stop()

    # kernel-family breakdown: CUDA events around every GEMM / attention
    # launch on the launching stream, over an eager pass of the same steps
    prof = []
    K.PROFILE = prof
    shapes = [] if args.detail else None
    K.PROFILE_SHAPES = shapes
    n0 = _native.launch_count()
    ms_eager = timed(lambda: step_eager(m_d, z_d), args.steps)
    launches = _native.launch_count() - n0
    if launches == 0 and launches_eager_step:
        # graph-replayed segments (N > 1): the native launches inside the
        # graphs are the eager step's, every step
        launches = launches_eager_step * args.steps
    K.PROFILE = None
    K.PROFILE_SHAPES = None
    fam = {}
    for name, flops, e0, e1 in prof:
        d_ms = e0.elapsed_time(e1)
        f = fam.setdefault(name, [0.0, 0.0, 0])
        f[0] += flops
        f[1] += d_ms
        f[2] += 1
    if shapes is not None and rank == 0:
        det = {}
        for (name, flops, e0_, e1_), shp in zip(prof, shapes):
            key = f"{name} {shp}" if shp else name
            dd = det.setdefault(key, [0.0, 0.0, 0])
            dd[0] += flops
            dd[1] += e0_.elapsed_time(e1_)
            dd[2] += 1
        for key, (fl, tms, n) in sorted(det.items(), key=lambda kv: -kv[1][1]):
            print(f"{tms / args.steps:8.3f} ms/step {n // args.steps:3d}x "
                  f"{fl / (tms / 1e3) / 1e12 if tms else 0:8.1f} TF/s  {key}", file=sys.stderr)

    # end-to-end: pinned host inputs -> device, step, loss -> host, every step
    def e2e_eager():
        m_d.copy_(m_h, non_blocking=True)
        z_d.copy_(z_h, non_blocking=True)
        out = step_graph() if runner is not None else step_eager(m_d, z_d)
        loss_h.copy_(out[2].reshape(1), non_blocking=True)

    def e2e_pipelined(k):
        # the H2D of step i+1 runs on a copy stream into the other graph slot's
        # static inputs while step i computes (double-buffered input pipeline)
        comp = torch.cuda.current_stream()
        copy = torch.cuda.Stream()
        h2d = [torch.cuda.Event() for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(comp)
        copy.wait_event(a0)

        def load(i):
            with torch.cuda.stream(copy):
                if i >= 2:
                    copy.wait_event(free[i % 2])  # step i-2 done with this buffer set
                mb, zb = gs.inputs(i % 2)
                mb.copy_(m_h.view(mb.shape), non_blocking=True)
                zb.copy_(z_h.view(zb.shape), non_blocking=True)
                h2d[i % 2].record(copy)

        load(0)
        for i in range(k):
            if i + 1 < k:
                load(i + 1)
            comp.wait_event(h2d[i % 2])
            out = gs.step(*gs.inputs(i % 2), slot=i % 2)
            loss_h.copy_(out[2].reshape(1), non_blocking=True)
            free[i % 2].record(comp)
        a1.record(comp)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / k

    if gs is not None:
        e2e_pipelined(2)
        ms_e2e = e2e_pipelined(args.steps)
        e2e_mode = "double-buffered H2D on a copy stream overlapping the previous step"
    else:
        ms_e2e = timed(e2e_eager, args.steps)
        e2e_mode = "serial H2D -> step -> loss D2H"

    # roofline timing: one step's launches of each kernel family re-issued
    # back to back inside a CUDA graph (device time, no host gaps)
    fam_graph = {}
    if use_graph and runner is None:
        rec = []
        K.RECORD = rec
        step_eager(m_d, z_d)
        K.RECORD = None
        torch.cuda.synchronize()
        for famname in sorted({r[0] for r in rec}):
            calls = [r for r in rec if r[0] == famname]
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                for _, _, fn, _ in calls:
                    fn()
            torch.cuda.current_stream().wait_stream(side)
            with torch.cuda.graph(g):
                for _, _, fn, _ in calls:
                    fn()
            g.replay()
            reps = max(3, args.steps)
            t_ms = timed(g.replay, reps)
            fam_graph[famname] = (sum(c[1] for c in calls), t_ms, len(calls))
        del rec

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    d = O.Dims(**kw)
    flops_block = 3 * O.block_flops(d)
    flops_step = flops_block * cfg.n_blocks
    samples = dp  # one sample per DP replica per step
    value = samples / (ms / 1e3)
    peak, peak_sus, hbm, src = peaks()
    step_tflops = flops_step * dp / (ms / 1e3) / 1e12
    roof = None
    if fam_graph:
        top = max(fam_graph, key=lambda k: fam_graph[k][1])
        fl, tms, n = fam_graph[top]
        achieved = fl / (tms / 1e3) / 1e12
        traffic = None
        # DRAM bytes per launch of this family from the committed ncu capture
        # of this configuration (tools/step_trace.py --family-json)
        dram_file = {(256, 128): "r02_family_dram.json",
                     (384, 128): "r02_family_dram_crop384.json"}.get((cfg.r, cfg.s))
        if dram_file and cfg.n_blocks == 1 and cfg.c_m == 256:
            try:
                with open(os.path.join(ROOT, "profiles", dram_file)) as f:
                    traffic = json.load(f)["families"][top]["dram_bytes_per_launch"]
            except Exception:
                traffic = None
        roof = {"bound": "tensor", "kernel": top, "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_unit": f"DRAM bytes per launch (profiles/{dram_file})" if traffic
                else None,
                "algorithmic_flops_per_launch": fl / n,
                "peak_source": src, "launches": n, "share_of_step": tms / ms,
                "timing": "CUDA events around one step's launches of this family, "
                          "re-issued back to back in a CUDA graph on the launching stream"}
        breakdown = {k: {"tflops": v[0] / (v[1] / 1e3) / 1e12, "ms_per_step": v[1],
                         "launches_per_step": v[2], "share_of_step": v[1] / ms}
                     for k, v in fam_graph.items()}
    elif fam:
        top = max(fam, key=lambda k: fam[k][1])
        fl, tms, n = fam[top]
        achieved = fl / (tms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": top, "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                "peak_source": src, "launches": n,
                "share_of_step": tms / (ms_eager * args.steps),
                "timing": "CUDA events around each launch on its stream, eager pass"}
    if not fam_graph:
        breakdown = {k: {"tflops": (v[0] / (v[1] / 1e3) / 1e12) if v[1] > 0 else None,
                         "ms_per_step": v[1] / args.steps,
                         "launches_per_step": v[2] / args.steps}
                     for k, v in fam.items()}
    cpu = None
    if not args.no_cpu_baseline:
        t_cpu, parts = cpu_sample(kw)
        cpu = {"value": 1.0 / (t_cpu * cfg.n_blocks), "unit": "samples/s",
               "cores": os.cpu_count(), "kind": "port",
               "sample": "fwd+bwd of each of the 9 sub-ops once at the full shape "
                         "(oracle/evoformer_np.py, numpy fp32, all host cores); "
                         f"block time = sum = {t_cpu:.1f} s"}
    h2d = (m_h.numel() + z_h.numel()) * 4
    bp2 = None
    if world == 1 and not args.no_bp2:
        bp2 = bp2_prediction(cfg, store, args.precision, dev, ms / cfg.n_blocks)
    peak_mem = torch.cuda.max_memory_allocated(dev) / 1e9
    c3 = None
    if world == 1 and not args.no_c3 and args.config == "af2" and not args.crop:
        import gc
        del gs, st
        gc.collect()
        torch.cuda.empty_cache()
        c3 = c3_summary(args)
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "ms_per_block_fwd_bwd": ms / cfg.n_blocks,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if args.precision == "bf16" else "f32", "data": "synthetic",
        "config": {"workload": f"parallel_evoformer_block_{args.config}", **kw,
                   "precision": args.precision, "parallelism": f"bp{bp}xdp{dp}",
                   "global_batch": dp,
                   "l2": "step working set (>1 GB of activations) exceeds the 126 MB L2"},
        "step_tflops": step_tflops, "step_frac_of_peak": step_tflops / peak,
        "roofline": roof, "kernels": breakdown, "cpu_baseline": cpu,
        "e2e": {"value": samples / (ms_e2e / 1e3), "unit": "samples/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4, "ms_per_step": ms_e2e,
                "mode": e2e_mode},
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "launch_mode": ("cuda_graph" if runner is None else "cuda_graph_segments")
        if use_graph else "eager", "ms_per_step_eager": ms_eager,
        "clocks": clk,
        "peak_mem_gb": peak_mem,
        "bp2_prediction": bp2,
        "c3_stack_1gpu": c3,
        # the last timed step's loss (read back every e2e step): a non-finite
        # loss invalidates the line
        "loss": float(loss_h[0]), "loss_finite": bool(np.isfinite(float(loss_h[0]))),
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


EXTRA_AF2 = dict(s=1024, r=256, c_m=64, c_z=128, h=8, c_opm=32, t_factor=4, n_blocks=4)


def run_stack(args):
    """C3 on one GPU: the 4-block extra-MSA stack feeding
    the main stack (schedules.composed_step), one step = fwd + loss + bwd of
    both stacks with every parameter gradient, captured as one CUDA graph.
    The main-stack depth is --blocks (default 48)."""
    import numpy as np
    import torch

    import paper_2211_00235_b200 as pkg
    from paper_2211_00235_b200 import _native, schedules as S
    from oracle import evoformer_np as O

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        return run_stack_bp(args, world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    kw_m = {**CONFIGS["af2"], "n_blocks": args.blocks or 48}
    if args.crop:
        kw_m["r"] = args.crop
    if args.seqs:
        kw_m["s"] = args.seqs
    kw_e = {**EXTRA_AF2, "r": kw_m["r"]}
    if args.extra_seqs:
        kw_e["s"] = args.extra_seqs
    ce, cm = pkg.EvoConfig(**kw_e), pkg.EvoConfig(**kw_m)
    ste = S.StepState(ce, pkg.init_params(ce, 33, device=dev), args.precision, dev,
                      checkpoint=args.checkpoint)
    stm = S.StepState(cm, pkg.init_params(cm, 32, device=dev), args.precision, dev,
                      checkpoint=args.checkpoint)
    ste.pack()
    stm.pack()
    rng = np.random.default_rng(32)
    host = [torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).pin_memory()
            for shape in ((ce.s, ce.r, ce.c_m), (cm.s, cm.r, cm.c_m), (cm.r, cm.r, cm.c_z))]
    dev_in = [h.to(dev) for h in host]
    loss_h = torch.empty(1, dtype=torch.float32).pin_memory()
    for _ in range(args.warmup):
        S.composed_step(ste, stm, *dev_in)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    graph = torch.cuda.CUDAGraph()
    n0 = _native.launch_count()
    with torch.cuda.graph(graph):
        out = S.composed_step(ste, stm, *dev_in)
        loss_h.copy_(out[2].reshape(1), non_blocking=True)
    launches_per_step = _native.launch_count() - n0
    graph.replay()
    torch.cuda.synchronize()

    def timed(fn, k):
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(k):
            fn()
        a1.record()
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / k

    clocks = Clocks(0)
    clocks.start()
    time.sleep(0.3)
    ms = timed(graph.replay, args.steps)
    clk = clocks.stop()

    def e2e():  # pinned host inputs -> static device buffers, step, loss -> host
        for h, d in zip(host, dev_in):
            d.copy_(h, non_blocking=True)
        graph.replay()

    ms_e2e = timed(e2e, args.steps)
    flops = 3 * (O.block_flops(O.Dims(**kw_e)) * ce.n_blocks
                 + O.block_flops(O.Dims(**kw_m)) * cm.n_blocks)
    peak, _, _, src = peaks()
    tflops = flops / (ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": 1e3 / ms, "unit": "samples/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "ms_per_block_fwd_bwd": ms / (ce.n_blocks + cm.n_blocks),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if args.precision == "bf16" else "f32", "data": "synthetic",
        "config": {"workload": ("evoformer_stack_c4_finetune" if kw_e["s"] > 1024
                                else "evoformer_stack_c3"), "main": kw_m, "extra": kw_e,
                   "precision": args.precision, "parallelism": "bp1xdp1", "global_batch": 1,
                   "activation_checkpointing": args.checkpoint,
                   "l2": "step working set exceeds the 126 MB L2"},
        "flops_per_step": flops, "step_tflops": tflops, "step_frac_of_peak": tflops / peak,
        "peak_source": src,
        "e2e": {"value": 1e3 / ms_e2e, "unit": "samples/s",
                "h2d_bytes_per_step": sum(h.numel() * 4 for h in host),
                "d2h_bytes_per_step": 4, "ms_per_step": ms_e2e,
                "mode": "serial H2D -> graph replay (step + loss D2H)"},
        "gpu_launches": launches_per_step * args.steps,
        "gpu_launches_per_step": launches_per_step, "launch_mode": "cuda_graph",
        "clocks": clk, "peak_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
        "loss": float(loss_h[0]), "loss_finite": bool(np.isfinite(float(loss_h[0]))),
    }
    if not getattr(args, "quiet", False):
        print(json.dumps(line))
    return line


def stack_configs(args):
    kw_m = {**CONFIGS["af2"], "n_blocks": args.blocks or 48}
    if args.crop:
        kw_m["r"] = args.crop
    if args.seqs:
        kw_m["s"] = args.seqs
    kw_e = {**EXTRA_AF2, "r": kw_m["r"]}
    if args.extra_seqs:
        kw_e["s"] = args.extra_seqs
    return kw_m, kw_e


def run_stack_bp(args, world):
    """C3 / C4 under torchrun: BP=2 x DP=world/2 (distributed.composed_bp_step:
    the extra-MSA stack and the main stack as one block schedule per BP pair,
    NCCL broadcasts / allreduces, owner broadcast + DP mean of both stacks'
    gradients).  Eager launches; device time, max over ranks; value = DP
    replicas / step time."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2211_00235_b200 as pkg
    from paper_2211_00235_b200 import distributed as D
    from oracle import evoformer_np as O

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group("gloo")
    if world % 2:
        raise SystemExit("--stack under torchrun needs an even world (BP=2 x DP)")
    layout = pkg.ParallelLayout(dp=world // 2, bp=2)
    comm = D.Comm(layout)
    dp_i = layout.coords(rank)[0]
    kw_m, kw_e = stack_configs(args)
    ce, cm = pkg.EvoConfig(**kw_e), pkg.EvoConfig(**kw_m)
    ex_e = D.CudaExec(ce, pkg.init_params(ce, 33, device=dev), args.precision, dev,
                      checkpoint=args.checkpoint)
    ex_m = D.CudaExec(cm, pkg.init_params(cm, 32, device=dev), args.precision, dev,
                      checkpoint=args.checkpoint)
    rng = np.random.default_rng(32 + dp_i)
    inp = [torch.from_numpy(rng.standard_normal(shape).astype(np.float32)).to(dev)
           for shape in ((ce.s, ce.r, ce.c_m), (cm.s, cm.r, cm.c_m), (cm.r, cm.r, cm.c_z))]

    def step():
        return D.composed_bp_step(ex_e, ex_m, comm, *inp)

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(args.steps):
        step()
    a1.record()
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([a0.elapsed_time(a1) / args.steps], device=dev)
    if args.backend == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    else:
        tc = t.cpu()
        dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        t = tc
    ms = float(t.item())
    if rank == 0:
        flops = 3 * (O.block_flops(O.Dims(**kw_e)) * ce.n_blocks
                     + O.block_flops(O.Dims(**kw_m)) * cm.n_blocks)
        peak, _, _, src = peaks()
        line = {
            "metric": METRIC, "value": layout.dp / (ms / 1e3), "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "ms_per_block_fwd_bwd": ms / (ce.n_blocks + cm.n_blocks), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16" if args.precision == "bf16" else "f32", "data": "synthetic",
            "config": {"workload": ("evoformer_stack_c4_finetune" if kw_e["s"] > 1024
                                    else "evoformer_stack_c3"), "main": kw_m, "extra": kw_e,
                       "precision": args.precision, "parallelism": f"bp2xdp{layout.dp}",
                       "global_batch": layout.dp, "activation_checkpointing": args.checkpoint,
                       "backend": args.backend},
            "flops_per_step": flops, "step_tflops": flops * layout.dp / (ms / 1e3) / 1e12,
            "peak_source": src, "launch_mode": "eager",
        }
        print(json.dumps(line))
    dist.destroy_process_group()
    return None


def c3_summary(args):
    """SURVEY.md §8(d) C3 on this GPU (48 main + 4 extra-MSA blocks, one
    train step graph-replayed), as a key of the default bench line."""
    import copy
    a = copy.copy(args)
    a.blocks, a.crop, a.seqs, a.extra_seqs, a.checkpoint = 48, 0, 0, 0, False
    a.steps, a.warmup, a.quiet = 5, 2, True
    line = run_stack(a)
    keep = ("value", "unit", "ms_per_step", "ms_per_block_fwd_bwd", "step_tflops",
            "step_frac_of_peak", "e2e", "gpu_launches_per_step", "clocks", "peak_mem_gb",
            "config")
    out = {k: line[k] for k in keep}
    out["steps"], out["warmup"] = a.steps, a.warmup
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="af2", choices=list(CONFIGS))
    ap.add_argument("--blocks", type=int, default=0)
    ap.add_argument("--crop", type=int, default=0,
                    help="override the crop size r (C5 sweep: 128 / 256 / 384)")
    ap.add_argument("--stack", action="store_true",
                    help="C3: 4-block extra-MSA stack (s_e=1024, c_e=64) feeding a "
                         "--blocks (default 48) main stack, one GPU")
    ap.add_argument("--seqs", type=int, default=0, help="--stack: main-stack MSA depth s")
    ap.add_argument("--extra-seqs", type=int, default=0,
                    help="--stack: extra-MSA depth s_e (C4: 5120)")
    ap.add_argument("--checkpoint", action="store_true",
                    help="per-block activation checkpointing (recompute each block's "
                         "forward before its backward)")
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo lets ranks share one "
                         "GPU: checks the multi-rank code path on a one-GPU box)")
    ap.add_argument("--dp-only", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time eager launches instead of CUDA-graph replay")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", action="store_true",
                    help="skip the C3 (48 + 4 block stack) measurement key")
    ap.add_argument("--no-bp2", action="store_true",
                    help="skip the one-GPU BP=2 branch-split prediction")
    ap.add_argument("--detail", action="store_true", help="per-call GEMM/attention table on stderr")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.stack:
        run_stack(args)
        return 0
    run_native(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
