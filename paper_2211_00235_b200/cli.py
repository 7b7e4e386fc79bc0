"""Command line front end (src/cli.py:1-254), same subcommands, config files
and exit codes (0 success, 1 a check failed, 2 usage / configuration
error), on the B200 build:

* ``verify <config>``: the configured layout (self-launched world) against
  the one-rank step, field by field.  Layouts without DAP are held to
  bitwise equality (BP and DP reproduce BP=1 exactly on this build, f32
  and bf16), DAP layouts to 1e-5 (f32) / 2e-2 (bf16).
* ``gradcheck <config>``: the native backward of every sub-op and of a
  whole block against central differences of the native forward, on the
  f32 path.  The reference samples single coordinates in f64; an f32
  forward cannot resolve single-coordinate differences, so each parameter
  / input tensor is checked along its own gradient direction (the slope
  of f there must equal the gradient's norm) at a 1e-2 relative bar.
* ``bench <config>``: device time per step (CUDA events, CUDA-graph
  replay) of the one-rank step, and for BP layouts the one-GPU BP=2
  prediction (each branch replayed alone; bench.py --gpus N measures the
  real multi-GPU step under torchrun).
* ``cost <config>``: the step-time model's layout sweep (costmodel.py),
  with the config's device constants (``device.preset = b200`` for the
  measured B200 ones).
"""

from __future__ import annotations

import argparse
import sys

import torch

from . import evoformer as EV
from .config import RunConfig, load_config
from .costmodel import report_csv, speedup_report
from .errors import BranchparError, ConfigError
from .schedules import ParallelLayout, compare_runs

WARMUP_STEPS = 5
GRAD_TOL = 1e-2
SHARD_RTOL = {"f32": 1e-5, "bf16": 2e-2}

COST_SWEEP = (ParallelLayout(), ParallelLayout(bp=2), ParallelLayout(dap=2),
              ParallelLayout(bp=2, dap=2), ParallelLayout(dap=4), ParallelLayout(bp=2, dap=4))


def _tag(layout: ParallelLayout) -> str:
    return f"dp{layout.dp}.bp{layout.bp}.dap{layout.dap}"


def _write_out(path, text: str) -> None:
    if path is not None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)
        print(f"wrote {path}")


def _store(rc: RunConfig):
    if not torch.cuda.is_available():
        raise BranchparError("this build computes on a B200 (CUDA device required)")
    return EV.init_params(rc.model, rc.seed)


def cmd_verify(rc: RunConfig, args) -> int:
    from .distributed import run_distributed
    from .schedules import run_single
    rtol = SHARD_RTOL[rc.precision] if rc.layout.dap > 1 else 0.0
    store = _store(rc)
    single = run_single(rc.model, store, seed=rc.seed, precision=rc.torch_precision)
    dist = run_distributed(rc.model, store, rc.layout, rc.seed, precision=rc.torch_precision)
    report = compare_runs(single, dist, rtol=rtol)
    print(f"layout {_tag(rc.layout)} vs single rank, precision {rc.precision}, rtol {rtol:g}")
    print(report)
    print(f"verify: {'PASS' if report.passed else 'FAIL'}")
    return 0 if report.passed else 1


def _subops(cfg):
    return {
        "row_attn": lambda P, m, z: EV.row_attn(P, "blk0.row_attn", m, z, cfg),
        "col_attn": lambda P, m, z: EV.col_attn(P, "blk0.col_attn", m, cfg),
        "msa_transition": lambda P, m, z: EV.msa_transition(P, "blk0.msa_transition", m, cfg),
        "opm": lambda P, m, z: EV.opm(P, "blk0.opm", m, cfg),
        "tri_mult_out": lambda P, m, z: EV.tri_mult(P, "blk0.tri_mult_out", z, cfg, False),
        "tri_mult_in": lambda P, m, z: EV.tri_mult(P, "blk0.tri_mult_in", z, cfg, True),
        "tri_attn_start": lambda P, m, z: EV.tri_attn(P, "blk0.tri_attn_start", z, cfg, False),
        "tri_attn_end": lambda P, m, z: EV.tri_attn(P, "blk0.tri_attn_end", z, cfg, True),
        "pair_transition": lambda P, m, z: EV.pair_transition(P, "blk0.pair_transition", z, cfg),
    }


def directional_check(f, leaves, rel_change=1e-3, skip=()):
    """Worst relative error, over the leaves, between the analytic slope of
    f along each leaf's own gradient direction (= |g|) and the central
    difference of f along it.  The step moves f by ~rel_change of its value
    (2 h |g| = rel_change |f|): f32 rounding of f is then ~1e-4 of the
    difference, and the curvature terms stay small.  Leaves in `skip`
    (analytic zeros: row_attn.lnz_b shifts every logit of a softmax row
    equally) and leaves with a gradient under 1e-6 of the largest are not
    checked."""
    xs = [x.detach().clone().requires_grad_(True) for x in leaves]
    out = f(*xs)
    f0 = abs(float(out.detach()))
    grads = torch.autograd.grad(out, xs, allow_unused=True)
    gmax = max(float(g.norm()) for g in grads if g is not None)
    worst, where, checked = 0.0, None, 0
    with torch.no_grad():
        for i, g in enumerate(grads):
            if i in skip or g is None or float(g.norm()) < 1e-6 * gmax:
                continue
            gn = float(g.norm())
            v = g / gn
            # step: f moves by ~rel_change of its value, the leaf by <= 1 %
            # (linear regime); a leaf whose 1 % move shifts f by less than
            # 1e-4 of f is below what an f32 forward resolves: not checked
            scale = max(float(xs[i].norm()), 1e-2 * xs[i].numel() ** 0.5)
            h = min(0.5 * rel_change * max(f0, 1e-30) / gn, 1e-2 * scale)
            if 2.0 * h * gn < 1e-4 * f0:
                continue
            checked += 1
            args_p = [x.detach() for x in xs]
            args_m = [x.detach() for x in xs]
            args_p[i] = xs[i].detach() + h * v
            args_m[i] = xs[i].detach() - h * v
            num = (float(f(*args_p)) - float(f(*args_m))) / (2.0 * h)
            rel = abs(num - gn) / gn
            if rel > worst:
                worst, where = rel, (i, gn, num)
    return worst, (where, checked)


def _zeros(names):
    return {i for i, n in enumerate(names) if n.endswith(".lnz_b")}


def cmd_gradcheck(rc: RunConfig, args) -> int:
    cfg = rc.model
    prev = EV.get_precision()
    EV.set_precision("fp32")
    try:
        store = _store(rc)
        m0, z0 = EV.seeded_inputs(cfg, rc.seed + 1)
        ok = True
        for subop, build in _subops(cfg).items():
            names = [n for n in store.names() if n.split(".")[0] == "blk0"
                     and n.split(".")[1] == subop]
            needs_m = subop in EV.MSA_SUBOPS
            needs_z = subop == "row_attn" or subop in EV.PAIR_SUBOPS
            leaves = [store[n] for n in names] + ([m0] if needs_m else []) + \
                ([z0] if needs_z else [])

            def f(*xs, _b=build, _n=names, _m=needs_m, _z=needs_z):
                P = dict(zip(_n, xs))
                rest = list(xs[len(_n):])
                m = rest.pop(0) if _m else None
                z = rest.pop(0) if _z else None
                out = _b(P, m, z)
                return (out * out).mean()

            err, (_, n) = directional_check(f, leaves, skip=_zeros(names))
            passed = err <= GRAD_TOL and n > 0
            ok = ok and passed
            print(f"gradcheck {subop}: max_rel_err={err:.3e} ({n}/{len(leaves)} tensors) "
                  f"{'PASS' if passed else 'FAIL'}")
        names = [n for n in store.names() if n.startswith("blk0.")]
        mb, zb = EV.seeded_inputs(cfg, rc.seed + 2)

        def f_block(*xs):
            # the block's deltas (outputs minus the residual inputs): the
            # outputs themselves are dominated by the inputs, and an f32
            # difference of their squares could not resolve the parameters'
            # contribution
            P = dict(zip(names, xs))
            mo, zo = EV.evoformer_block(P, 0, xs[-2], xs[-1], cfg)
            dmo, dzo = mo - xs[-2], zo - xs[-1]
            return (dmo * dmo).mean() + (dzo * dzo).mean()

        err, (_, n) = directional_check(f_block, [store[n] for n in names] + [mb, zb],
                                        skip=_zeros(names))
        passed = err <= GRAD_TOL and n > 0
        ok = ok and passed
        print(f"gradcheck block ({cfg.variant}): max_rel_err={err:.3e} "
              f"({n}/{len(names) + 2} tensors) {'PASS' if passed else 'FAIL'}")
        print(f"gradcheck: {'PASS' if ok else 'FAIL'}")
        return 0 if ok else 1
    finally:
        EV.set_precision(prev)


def _graph_step_seconds(rc: RunConfig, store, steps: int) -> float:
    from .schedules import StepState, make_batch
    st = StepState(rc.model, store, rc.torch_precision)
    m, z = make_batch(rc.model, rc.seed, 1, store.device)[0]
    gs = st.capture(m, z, warmup=min(WARMUP_STEPS, steps))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, steps - WARMUP_STEPS)
    a.record()
    for _ in range(n):
        gs.step(*gs.inputs(0))
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n / 1e3


def _branch_seconds(rc: RunConfig, store, steps: int):
    """Each branch's fwd+bwd of the whole stack replayed alone as a CUDA
    graph (the BP=2 compute of one rank), plus one forward's exchange."""
    from . import distributed as D
    from .schedules import make_batch
    ex = D.CudaExec(rc.model, store, rc.torch_precision)
    ex.pack("all")
    cfg = rc.model
    m, z = make_batch(cfg, rc.seed, 1, store.device)[0]
    m2, z2 = m.reshape(cfg.s * cfg.r, cfg.c_m), z.reshape(cfg.r * cfg.r, cfg.c_z)

    def msa():
        ctx = []
        cur = m2
        for blk in range(cfg.n_blocks):
            cur, o, c = ex.msa_fwd(blk, cur, z2)
            ctx.append((c, o))
        dm = torch.ones_like(cur)
        for blk in reversed(range(cfg.n_blocks)):
            c, o = ctx[blk]
            dm, _ = ex.msa_bwd(blk, c, dm, torch.ones_like(o))

    def pair():
        ctx = []
        cur = z2
        for blk in range(cfg.n_blocks):
            cur, c = ex.pair_fwd(blk, cur)
            ctx.append(c)
        dz = torch.ones_like(cur)
        for blk in reversed(range(cfg.n_blocks)):
            dz = ex.pair_bwd(blk, ctx[blk], dz)

    out = []
    for fn in (msa, pair):   # eager warm-up, then one capture per branch
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(g):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = max(1, steps - WARMUP_STEPS)
        a.record()
        for _ in range(n):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / n / 1e3)
    return out


def cmd_bench(rc: RunConfig, args) -> int:
    steps = args.repeat if args.repeat is not None else rc.steps
    if steps <= WARMUP_STEPS:
        print(f"error: bench needs more than {WARMUP_STEPS} steps (fixed warmup), got {steps}",
              file=sys.stderr)
        return 2
    store = _store(rc)
    tag = _tag(rc.layout)
    t_single = _graph_step_seconds(rc, store, steps)
    print(f"bench single: {t_single:.6f} s/step ({steps - WARMUP_STEPS} measured after "
          f"{WARMUP_STEPS} warmup; CUDA-graph replay, device time)")
    lines = ["label,seconds_per_step", f"single,{t_single:.6f}"]
    if rc.layout.bp == 2 and rc.layout.dap == 1:
        t_msa, t_pair = _branch_seconds(rc, store, steps)
        cfg = rc.model
        width = 2 if rc.precision == "bf16" else 4
        # per block: o and z'' in the forward, dz'' and the dz_in allreduce
        # in the backward, Z elements each, fp32 on the wire; 750 GB/s NVLink
        xfer = 4 * cfg.n_blocks * cfg.r * cfg.r * cfg.c_z * 4 / 7.5e11
        t_bp = max(t_msa, t_pair) + xfer
        print(f"bench branches: msa {t_msa:.6f} s, pair {t_pair:.6f} s (one GPU, each alone); "
              f"activation width {width} B")
        print(f"bench {tag} (predicted: slower branch + exchange at 750 GB/s): "
              f"{t_bp:.6f} s/step")
        print(f"bench speedup: {t_single / t_bp:.3f}x (predicted)")
        lines.append(f"{tag}_predicted,{t_bp:.6f}")
    elif rc.layout.world_size > 1:
        print(f"bench {tag}: a {rc.layout.world_size}-GPU layout; time it with "
              f"'python -m torch.distributed.run --nproc-per-node {rc.layout.world_size} "
              f"bench.py --gpus {rc.layout.world_size}'")
    _write_out(args.out, "\n".join(lines) + "\n")
    return 0


def cmd_cost(rc: RunConfig, args) -> int:
    layouts = []
    for layout in COST_SWEEP:
        try:
            layout.validate_model(rc.model)
        except ConfigError:
            continue
        layouts.append(layout)
    csv = report_csv(speedup_report(rc.model, rc.device, layouts))
    print(csv, end="")
    _write_out(args.out, csv)
    return 0


COMMANDS = {"verify": cmd_verify, "gradcheck": cmd_gradcheck, "bench": cmd_bench,
            "cost": cmd_cost}


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(
        prog="paper_2211_00235_b200",
        description="equivalence checks, timings and cost reports for the block stack "
                    "under branch, shard and data parallel layouts (B200 build)")
    sub = p.add_subparsers(dest="command", required=True)
    helps = {"verify": "compare the configured layout against a single rank",
             "gradcheck": "finite-difference gradient checks at the configured dims",
             "bench": "device time per step, single rank (and the BP=2 prediction)",
             "cost": "modelled step times for the standard layout sweep"}
    for name, text in helps.items():
        sp = sub.add_parser(name, help=text)
        sp.add_argument("config", help="path to a key-value config file")
        sp.add_argument("--repeat", type=int, default=None,
                        help="bench iterations, including warmup")
        sp.add_argument("--out", default=None, help="write CSV here")
        sp.add_argument("--seed", type=int, default=None, help="override run.seed")
        sp.add_argument("--precision", choices=["f64", "f32", "bf16"], default=None,
                        help="override run.precision (f64 runs as f32 on this build)")
    return p


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code in (0, None) else int(exc.code)
    try:
        rc = load_config(args.config).with_overrides(seed=args.seed, precision=args.precision)
        for note in rc.notes:
            print(f"note: {note}")
        return COMMANDS[args.command](rc, args)
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except BranchparError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
