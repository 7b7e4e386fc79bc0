"""Train-step API (src/schedules.py:43-581) on B200: BP=1 step, branch
parallelism (BP=2) and data parallelism over NCCL, run comparison and the
closed-form communication ledger.

The step is: forward through the stack, loss = mean(m^2) + mean(z^2)
(src/schedules.py:194-195), backward, parameter-gradient sync.  Here the
forward/backward are explicit sequences of native launches
(engine.block_fwd / block_bwd) rather than a tape sweep; the BP=1 path
forms dz_in = dz_pair + dz_row with the same two operands the BP
allreduce sums, so BP=2 reproduces BP=1 bitwise (src/schedules.py:12-15).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine as E
from . import kernels as K
from .errors import ComparisonError, ConfigError
from .evoformer import EvoConfig, ParamStore, act_dtype

F32 = torch.float32


@dataclass(frozen=True)
class ParallelLayout:
    """(dp, bp, dap) layout; rank = ((dp_i*bp)+bp_i)*dap + dap_i
    (src/schedules.py:43-93)."""

    dp: int = 1
    bp: int = 1
    dap: int = 1

    def __post_init__(self):
        if self.dp < 1:
            raise ConfigError(f"layout.dp must be >= 1, got {self.dp}")
        if self.bp not in (1, 2):
            raise ConfigError(
                "layout.bp must be 1 or 2: the block splits into exactly two "
                f"branches (MSA and pair), got bp={self.bp}")
        if self.dap < 1 or (self.dap & (self.dap - 1)) != 0:
            raise ConfigError(f"layout.dap must be a power of two >= 1, got {self.dap}")

    @property
    def world_size(self) -> int:
        return self.dp * self.bp * self.dap

    def rank_of(self, dp_i: int, bp_i: int, dap_i: int = 0) -> int:
        return ((dp_i * self.bp) + bp_i) * self.dap + dap_i

    def coords(self, rank: int):
        dap_i = rank % self.dap
        rest = rank // self.dap
        return rest // self.bp, rest % self.bp, dap_i

    def dap_group(self, rank: int):
        dp_i, bp_i, _ = self.coords(rank)
        return tuple(self.rank_of(dp_i, bp_i, k) for k in range(self.dap))

    def bp_group(self, rank: int):
        dp_i, _, dap_i = self.coords(rank)
        return tuple(self.rank_of(dp_i, b, dap_i) for b in range(self.bp))

    def dp_group(self, rank: int):
        _, bp_i, dap_i = self.coords(rank)
        return tuple(self.rank_of(d, bp_i, dap_i) for d in range(self.dp))

    def validate_model(self, cfg: EvoConfig) -> None:
        if self.dap > 1 and (cfg.s % self.dap or cfg.r % self.dap):
            raise ConfigError(
                f"layout.dap={self.dap} must divide both model.s={cfg.s} "
                f"and model.r={cfg.r}")
        if self.bp == 2 and cfg.variant != "parallel":
            raise ConfigError(
                "branch parallelism needs the parallel block wiring; the "
                f"{cfg.variant!r} variant has a serial dependency between "
                "the tracks inside each block")


@dataclass
class RunResult:
    """Outputs of one training step (src/schedules.py:157-174).  Tensor
    fields are device tensors; ``numpy()`` returns a host copy."""

    m_out: object
    z_out: object
    loss: float
    dm: object
    dz: object
    grads: dict
    trace: object = None
    rank_fwd_seconds: dict | None = None
    wall_seconds: float = 0.0

    def numpy(self) -> "RunResult":
        return RunResult(_np(self.m_out), _np(self.z_out), self.loss, _np(self.dm),
                         _np(self.dz), {k: _np(v) for k, v in self.grads.items()},
                         self.trace, self.rank_fwd_seconds, self.wall_seconds)


def _np(x):
    if isinstance(x, torch.Tensor):
        return x.detach().float().cpu().numpy()
    return np.asarray(x)


def make_batch(cfg: EvoConfig, seed: int, n: int, device="cuda"):
    """n standard-normal (m, z) samples drawn sequentially from one PCG64
    stream, identical to the reference's (src/schedules.py:177-185)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        m = rng.standard_normal((cfg.s, cfg.r, cfg.c_m)).astype(np.float32)
        z = rng.standard_normal((cfg.r, cfg.r, cfg.c_z)).astype(np.float32)
        out.append((torch.as_tensor(m, device=device), torch.as_tensor(z, device=device)))
    return out


# ---------------------------------------------------------------------------
# the BP=1 step
# ---------------------------------------------------------------------------

class StepState:
    """Reusable per-(cfg, precision) state: packed operand weights and the
    per-block gradient banks.  ``pack(store)`` refreshes the operand copies
    after a parameter update."""

    def __init__(self, cfg: EvoConfig, store: ParamStore, precision: str | None = None,
                 device=None, checkpoint: bool = False):
        self.cfg = cfg
        self.act = act_dtype(precision)
        self.dev = device or store.device
        # per-block activation checkpointing: keep only each block's inputs
        # (m, z) through the forward and recompute the block's forward right
        # before its backward (bitwise the same values: every kernel is
        # deterministic), for stacks whose saved activations exceed HBM
        # (C4: 48 blocks at s = 512, r = 384)
        self.checkpoint = checkpoint
        self.P = store.bind()
        self.grads = [E.BlockGrads(b, cfg, self.dev) for b in range(cfg.n_blocks)]
        self.packs = None

    def pack(self, subops=E.MSA_SUBOPS + E.PAIR_SUBOPS):
        self.packs = [E.pack_block(self.P, b, self.cfg, self.act, self.dev, subops)
                      for b in range(self.cfg.n_blocks)]

    def grad_dict(self):
        out = {}
        for bg in self.grads:
            out.update(bg.names)
        return out

    def capture(self, m, z, warmup: int = 1, slots: int = 1) -> "GraphedStep":
        """The step as a CUDA graph (one per slot): `warmup` eager steps
        (first-touch allocations, kernel attributes), then capture on (m, z).
        Replay with the returned object's ``step(m, z, slot)``."""
        if self.packs is None:
            self.pack()
        for _ in range(warmup):
            full_step(self, m, z)
        torch.cuda.synchronize()
        gs = GraphedStep(self)
        for slot in range(slots):
            gs.step(m, z, slot)
        torch.cuda.synchronize()
        return gs


def _tensors_of(x, out=None):
    out = [] if out is None else out
    if isinstance(x, torch.Tensor):
        out.append(x)
    elif isinstance(x, (tuple, list)):
        for v in x:
            _tensors_of(v, out)
    elif isinstance(x, dict):
        for v in x.values():
            _tensors_of(v, out)
    return out


class SegmentGraphs:
    """CUDA graphs of the native launch sequences between two host-side
    events (collectives, or a whole step).  The first call of a key captures
    ``fn`` on static copies of its tensor arguments and replays it; later
    calls copy arguments whose storage changed into those buffers and
    replay.  Segment outputs are static buffers, rewritten by the next replay
    of the same key.  All segments share one memory pool, so a step must
    replay its segments in the order they were captured (the BP / DP
    schedules issue the same sequence every step).  Arguments that are
    outputs of an earlier segment are used in place (no copy)."""

    def __init__(self):
        self.graphs = {}
        self.pool = None
        self.static = set()

    def __call__(self, key, fn, *args):
        tens = [a for a in args if isinstance(a, torch.Tensor)]
        ent = self.graphs.get(key)
        if ent is None:
            sin = [t if t.data_ptr() in self.static else t.clone() for t in tens]
            it = iter(sin)
            cargs = [next(it) if isinstance(a, torch.Tensor) else a for a in args]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self.pool):
                out = fn(*cargs)
            if self.pool is None:
                self.pool = g.pool()
            for t in _tensors_of(out):
                self.static.add(t.data_ptr())
            ent = (g, sin, out)
            self.graphs[key] = ent
        g, sin, out = ent
        for s_, t in zip(sin, tens):
            if s_.data_ptr() != t.data_ptr():
                s_.copy_(t)
        g.replay()
        return out


class GraphedStep:
    """A BP=1 train step replayed as one CUDA graph (StepState.capture):
    ``step(m, z, slot)`` -> (m_out, z_out, loss[1], dm, dz) as static
    buffers (valid until the next call).  Each slot is one captured graph
    with its own static inputs (``inputs(slot)``), so a caller can stage the
    next step's inputs into one slot while the other computes.  Parameter
    gradients land in the StepState's gradient banks as in the eager step."""

    def __init__(self, st: "StepState"):
        self.st = st
        self.seg = SegmentGraphs()

    def step(self, m, z, slot: int = 0):
        return self.seg(("step", slot), lambda a, b: full_step(self.st, a, b), m, z)

    def inputs(self, slot: int = 0):
        """The static (m, z) device buffers of a slot: write inputs there
        and call step() with them to skip the input copy."""
        return tuple(self.seg.graphs[("step", slot)][1])


def _stack_fwd(st: StepState, m_c, z_c):
    """Forward through st's blocks; returns (m, z, per-block saved state):
    the block's ctx, or with st.checkpoint only its inputs (m, z)."""
    cfg, act = st.cfg, st.act
    saved = []
    for blk in range(cfg.n_blocks):
        m_in, z_in = m_c, z_c
        m_c, z_c, c = E.block_fwd(st.P, blk, st.packs[blk], m_c, z_c, cfg, act)
        saved.append((m_in, z_in) if st.checkpoint else c)
        del c
    return m_c, z_c, saved


def _stack_bwd(st: StepState, saved, dm, dz):
    cfg, act = st.cfg, st.act
    for blk in reversed(range(cfg.n_blocks)):
        c = saved[blk]
        saved[blk] = None
        if st.checkpoint:   # recompute the block's forward state
            _, _, c = E.block_fwd(st.P, blk, st.packs[blk], c[0], c[1], cfg, act)
        dm, dz = E.block_bwd(st.P, blk, st.packs[blk], st.grads[blk].packed, c, dm, dz, cfg, act)
        del c
    return dm, dz


def full_step(st: StepState, m, z, fwd_events=None):
    """Forward + loss + backward of the whole stack on one device.
    Returns (m_out, z_out, loss_tensor[1], dm, dz); fwd_events (two CUDA
    events) are recorded around the forward when given."""
    cfg, act = st.cfg, st.act
    s, r = cfg.s, cfg.r
    if st.packs is None:
        st.pack()
    m_c = m.reshape(s * r, cfg.c_m)
    z_c = z.reshape(r * r, cfg.c_z)
    if fwd_events is not None:
        fwd_events[0].record()
    m_c, z_c, ctxs = _stack_fwd(st, m_c, z_c)
    if fwd_events is not None:
        fwd_events[1].record()
    loss = K.zeros(1, F32, m.device)
    dm = torch.empty_like(m_c)
    dz = torch.empty_like(z_c)
    K.sq_mean(m_c, loss, dm)
    K.sq_mean(z_c, loss, dz)
    dm, dz = _stack_bwd(st, ctxs, dm, dz)
    return (m_c.reshape(s, r, cfg.c_m), z_c.reshape(r, r, cfg.c_z), loss,
            dm.reshape(s, r, cfg.c_m), dz.reshape(r, r, cfg.c_z))


def composed_step(extra: StepState, main: StepState, m_e, m, z):
    """an extra-MSA stack (its own EvoConfig: s_e rows,
    c_e channels, c_head = c_e / h) whose pair output feeds the main stack;
    its MSA output m_e' is dropped.  The reference has no extra-MSA module
    (it composes two ``evoformer_stack`` calls, src/evoformer.py:464-467, on
    one tape); the loss is the main stack's (src/schedules.py:194-195), so
    the extra stack's backward is seeded with dm_e' = 0 and the main stack's
    dz_in.  Returns (m_out, z_out, loss[1], dm_e, dm, dz)."""
    ce, cm = extra.cfg, main.cfg
    if (ce.r, ce.c_z) != (cm.r, cm.c_z):
        raise ConfigError(f"extra stack (r={ce.r}, c_z={ce.c_z}) does not feed the main "
                          f"stack (r={cm.r}, c_z={cm.c_z})")
    for st in (extra, main):
        if st.packs is None:
            st.pack()
    me_c = m_e.reshape(ce.s * ce.r, ce.c_m)
    z_c = z.reshape(ce.r * ce.r, ce.c_z)
    me_c, z_c, ctx_e = _stack_fwd(extra, me_c, z_c)
    m_c = m.reshape(cm.s * cm.r, cm.c_m)
    m_c, z_c, ctx_m = _stack_fwd(main, m_c, z_c)
    loss = K.zeros(1, F32, m.device)
    dm = torch.empty_like(m_c)
    dz = torch.empty_like(z_c)
    K.sq_mean(m_c, loss, dm)
    K.sq_mean(z_c, loss, dz)
    dm, dz = _stack_bwd(main, ctx_m, dm, dz)
    dm_e = K.zeros(me_c.shape, F32, m.device)
    dm_e, dz = _stack_bwd(extra, ctx_e, dm_e, dz)
    return (m_c.reshape(cm.s, cm.r, cm.c_m), z_c.reshape(cm.r, cm.r, cm.c_z), loss,
            dm_e.reshape(ce.s, ce.r, ce.c_m), dm.reshape(cm.s, cm.r, cm.c_m),
            dz.reshape(cm.r, cm.r, cm.c_z))


def run_single(cfg: EvoConfig, store: ParamStore, seed: int = 32,
               precision: str | None = None) -> RunResult:
    """Reference step on one GPU (src/schedules.py:387-399), any wiring
    (parallel / af2 / multimer).  rank_fwd_seconds = the forward's device
    time (CUDA events), wall_seconds = the whole step."""
    m, z = make_batch(cfg, seed, 1, store.device)[0]
    st = StepState(cfg, store, precision)
    t0 = time.perf_counter()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    m_out, z_out, loss, dm, dz = full_step(st, m, z, fwd_events=ev)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return RunResult(m_out, z_out, float(loss.item()), dm, dz, st.grad_dict(), None,
                     {0: ev[0].elapsed_time(ev[1]) / 1e3}, wall)


# ---------------------------------------------------------------------------
# comparing runs (src/schedules.py:430-488)
# ---------------------------------------------------------------------------

@dataclass
class FieldComparison:
    field: str
    max_abs: float
    max_rel: float
    bitwise: bool


@dataclass
class ComparisonReport:
    fields: dict
    rtol: float

    @property
    def max_rel(self) -> float:
        return max((f.max_rel for f in self.fields.values()), default=0.0)

    @property
    def bitwise(self) -> bool:
        return all(f.bitwise for f in self.fields.values())

    @property
    def passed(self) -> bool:
        if self.rtol == 0.0:
            return self.bitwise
        return self.max_rel <= self.rtol

    def __str__(self):
        lines = [f"{'field':<12} {'max_abs':>12} {'max_rel':>12} bitwise"]
        for f in self.fields.values():
            lines.append(f"{f.field:<12} {f.max_abs:>12.3e} {f.max_rel:>12.3e} {f.bitwise}")
        lines.append(f"-> {'pass' if self.passed else 'FAIL'} (rtol={self.rtol:g})")
        return "\n".join(lines)


def _rel_diff(a, b):
    a = np.asarray(_np(a), dtype=np.float64)
    b = np.asarray(_np(b), dtype=np.float64)
    diff = np.abs(a - b)
    denom = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return (float(diff.max()) if diff.size else 0.0,
            float((diff / denom).max()) if diff.size else 0.0)


def _equal(a, b):
    if isinstance(a, torch.Tensor) and isinstance(b, torch.Tensor):
        return bool(torch.equal(a, b))
    return bool(np.array_equal(_np(a), _np(b)))


def compare_runs(a: RunResult, b: RunResult, rtol: float = 0.0) -> ComparisonReport:
    """Field-by-field max-abs / max-rel comparison; rtol=0 demands bitwise
    equality (src/schedules.py:464-488)."""
    if set(a.grads) != set(b.grads):
        missing = set(a.grads) ^ set(b.grads)
        raise ComparisonError(f"gradient key sets differ: {sorted(missing)[:5]}")
    fields = {}
    for name in ("loss", "m_out", "z_out", "dm", "dz"):
        xa, xb = getattr(a, name), getattr(b, name)
        if np.shape(_np(xa)) != np.shape(_np(xb)):
            raise ComparisonError(f"{name} shapes differ")
        ma, mr = _rel_diff(xa, xb)
        fields[name] = FieldComparison(name, ma, mr, _equal(xa, xb))
    wa = wr = 0.0
    bit = True
    for key in a.grads:
        ma, mr = _rel_diff(a.grads[key], b.grads[key])
        wa, wr = max(wa, ma), max(wr, mr)
        bit = bit and _equal(a.grads[key], b.grads[key])
    fields["grads"] = FieldComparison("grads", wa, wr, bit)
    return ComparisonReport(fields, rtol)


# ---------------------------------------------------------------------------
# closed-form communication volume, BP and DP parts (src/schedules.py:515-572)
# ---------------------------------------------------------------------------

MSA_PARAM_TENSORS = 35
PAIR_PARAM_TENSORS = 58


def branch_param_elems(cfg: EvoConfig):
    msa = sum(E.subop_grad_numel(n, cfg) for n in E.MSA_SUBOPS)
    pair = sum(E.subop_grad_numel(n, cfg) for n in E.PAIR_SUBOPS)
    return msa, pair


def expected_comm_volume(cfg: EvoConfig, layout: ParallelLayout) -> dict:
    """{(phase, kind): (count, elements)} for one step over the whole world,
    using the reference's accounting (per-tensor parameter collectives,
    src/schedules.py:515-572).  This build buckets the parameter collectives
    per branch and block; the element totals are identical."""
    layout.validate_model(cfg)
    Kb = cfg.n_blocks
    M = cfg.s * cfg.r * cfg.c_m
    Z = cfg.r * cfg.r * cfg.c_z
    O = cfg.r * cfg.r * cfg.c_opm
    B = cfg.r * cfg.r * cfg.h
    msa, pair = branch_param_elems(cfg)
    msa *= Kb
    pair *= Kb
    out = {}

    def bump(phase, kind, count, elements):
        if count:
            c0, e0 = out.get((phase, kind), (0, 0))
            out[(phase, kind)] = (c0 + count, e0 + elements)

    if layout.bp == 2:
        g = layout.dp * layout.dap       # one branch pair per (dp_i, dap_i)
        bump("fwd", "broadcast", 2 * Kb * g, 2 * Kb * Z * g)
        bump("bwd", "broadcast", (Kb + 1) * g, (Kb * Z + M) * g)
        bump("bwd", "allreduce_sum", Kb * g, Kb * Z * g)
        n = (MSA_PARAM_TENSORS + PAIR_PARAM_TENSORS) * Kb
        bump("param", "broadcast", n * g, (msa + pair) * g)
    if layout.dap > 1:
        # per block: gathers of 3 MSA deltas, 5 pair deltas, 3 partner
        # projections (O) and 2 pair-bias row sets (B); the OPM reduce_sum;
        # the enter allreduces of every sub-op input, the gathered partner
        # projections and bias rows; every parameter but opm.out_b
        g = layout.dp
        msa_ar, pair_ar = (MSA_PARAM_TENSORS - 1) * Kb, PAIR_PARAM_TENSORS * Kb
        bump("fwd", "allgather", 3 * Kb * g, 3 * Kb * M * g)
        bump("fwd", "allreduce_sum", Kb * g, Kb * Z * g)
        bump("bwd", "allreduce_sum", 5 * Kb * g, Kb * (4 * M + Z) * g)
        bump("param", "allreduce_sum", msa_ar * g, (msa - Kb * cfg.c_z) * g)
        bump("fwd", "allgather", 10 * Kb * g, Kb * (5 * Z + 3 * O + 2 * B) * g)
        bump("bwd", "allreduce_sum", 10 * Kb * g, Kb * (5 * Z + 3 * O + 2 * B) * g)
        bump("param", "allreduce_sum", pair_ar * g, pair * g)
    if layout.dp > 1:
        g = layout.bp * layout.dap
        n = (MSA_PARAM_TENSORS + PAIR_PARAM_TENSORS) * Kb
        bump("param", "allreduce_sum", n * g, (msa + pair) * g)
    return out


def trace_volume(trace) -> dict:
    """Same shape as expected_comm_volume, read off a recorded CommTrace
    (src/schedules.py:575-581)."""
    out = {}
    for r in trace.records:
        c0, e0 = out.get((r.phase, r.kind), (0, 0))
        out[(r.phase, r.kind)] = (c0 + 1, e0 + r.elements)
    return out
