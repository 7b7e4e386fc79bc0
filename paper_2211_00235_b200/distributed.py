"""Branch Parallelism (BP=2) x data parallelism over torch.distributed:
the schedule of src/schedules.py:214-329 on real processes.

One process per GPU (torchrun); rank = dp_i * bp + bp_i (dap = 1,
src/schedules.py:22, 43-82).  In a BP pair, bp_i = 0 runs the MSA branch
(row/column attention, MSA transition) plus the outer product mean, bp_i = 1
the pair branch (triangle updates, triangle attentions, pair transition).
Per block (the reference's literal order):

  forward   rank0: m' = msa_track(m, z); o = opm(m')        broadcast o  (src 0)
            rank1: z_b = pair_track(z); z'' = z_b + o        broadcast z'' (src 1)
  backward  rank1: broadcast dz'' (src 1); rank0 seeds it into o
            both:  segment backward; allreduce dz_in partials (dz_row + dz_pair)
  end       rank0: broadcast dm (src 0)
  params    owner broadcast of each branch's gradient bucket over the pair,
            then sum / dp over the DP group.

Every cross-rank sum in the BP pair has exactly two operands, and the BP=1
path forms the same sums (dz_in = dz_pair + dz_row, z' = z_pair + o), so
BP=2 reproduces BP=1 bitwise: float addition commutes.

The schedule is written against a small executor interface (`CudaExec`
here: the native kernels; the CPU tests substitute an oracle-backed executor
and run the same schedule under the gloo backend).
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass

import torch
import torch.distributed as dist

from .errors import CollectiveError, ConfigError, WorldError
from .schedules import ParallelLayout, RunResult, make_batch

F32 = torch.float32


@dataclass(frozen=True)
class CommRecord:
    """One completed collective (src/comm.py:41-50)."""

    seq: int
    kind: str
    group: tuple
    src: int | None
    elements: int
    bytes: int
    phase: str


PHASES = ("fwd", "bwd", "param")


class CommTrace:
    """Log of the world's collectives, one record per collective (src/comm.py:52-110):
    ``records``, ``canonical()``, ``totals()``, ``by_phase()``, ``to_csv()``,
    ``csv_text()``.  Built by ``Comm.world_trace()`` from every rank's log
    (each collective counted once, by the lowest rank of its group)."""

    def __init__(self, records=()):
        self.records: list[CommRecord] = []
        self._order: list[int] = []
        for r in records:
            self.add(r.kind, r.group, r.src, r.elements, r.bytes, r.phase)

    def add(self, kind, group, src, elements, nbytes, phase) -> None:
        group = tuple(group)
        idx = sum(1 for r in self.records if r.group == group)
        self.records.append(CommRecord(len(self.records), kind, group, src, int(elements),
                                       int(nbytes), phase))
        self._order.append(idx)

    def canonical(self) -> list:
        """Records ordered by (group, issue order within the group)."""
        pairs = sorted(zip(self.records, self._order), key=lambda p: (p[0].group, p[1]))
        return [r for r, _ in pairs]

    def totals(self, phase: str | None = None, kind: str | None = None):
        """(count, elements, bytes) over matching records."""
        n = el = by = 0
        for r in self.records:
            if (phase is None or r.phase == phase) and (kind is None or r.kind == kind):
                n, el, by = n + 1, el + r.elements, by + r.bytes
        return n, el, by

    def by_phase(self) -> dict:
        return {p: self.totals(phase=p) for p in PHASES}

    def to_csv(self, target) -> None:
        import csv
        own = isinstance(target, (str, os.PathLike))
        fh = open(target, "w", newline="") if own else target
        try:
            w = csv.writer(fh)
            w.writerow(["seq", "kind", "group", "src", "elements", "bytes", "phase"])
            for r in self.canonical():
                w.writerow([r.seq, r.kind, "|".join(map(str, r.group)),
                            "" if r.src is None else r.src, r.elements, r.bytes, r.phase])
        finally:
            if own:
                fh.close()

    def csv_text(self) -> str:
        import io
        buf = io.StringIO()
        self.to_csv(buf)
        return buf.getvalue()


class Comm:
    """Collectives over the BP-pair and DP groups of a layout, with a log of
    every call this rank joined (``trace``; ``world_trace()`` merges the
    ranks' logs into the reference's world-level CommTrace)."""

    def __init__(self, layout: ParallelLayout, rank: int | None = None):
        if not dist.is_initialized():
            raise WorldError("torch.distributed is not initialised (launch with torchrun)")
        self.layout = layout
        self.rank = dist.get_rank() if rank is None else rank
        if dist.get_world_size() != layout.world_size:
            raise ConfigError(f"world size {dist.get_world_size()} != layout world size "
                              f"{layout.world_size}")
        self.groups = {}
        # every rank creates every group, in the same order
        for dp_i in range(layout.dp):
            for k in range(layout.dap):
                g = tuple(layout.rank_of(dp_i, b, k) for b in range(layout.bp))
                self.groups[g] = dist.new_group(list(g)) if layout.bp > 1 else None
        for bp_i in range(layout.bp):
            for k in range(layout.dap):
                g = tuple(layout.rank_of(d, bp_i, k) for d in range(layout.dp))
                self.groups[g] = dist.new_group(list(g)) if layout.dp > 1 else None
        for dp_i in range(layout.dp):
            for bp_i in range(layout.bp):
                g = tuple(layout.rank_of(dp_i, bp_i, k) for k in range(layout.dap))
                self.groups[g] = dist.new_group(list(g)) if layout.dap > 1 else None
        self.pair = layout.bp_group(self.rank)
        self.dpg = layout.dp_group(self.rank)
        self.dapg = layout.dap_group(self.rank)
        self.trace: list[CommRecord] = []

    def _rec(self, kind, group, src, t, phase):
        if phase is None:       # result assembly: not part of the step's ledger
            return
        self.trace.append(CommRecord(len(self.trace), kind, tuple(group), src, int(t.numel()),
                                     int(t.numel() * t.element_size()), phase))

    def broadcast(self, group, src, t, phase):
        if src not in group:
            raise CollectiveError(f"broadcast src {src} not in group {group}")
        dist.broadcast(t, src=src, group=self.groups[tuple(group)])
        self._rec("broadcast", group, src, t, phase)
        return t

    def allreduce_sum(self, group, t, phase):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.groups[tuple(group)])
        self._rec("allreduce_sum", group, None, t, phase)
        return t

    def allgather(self, group, t, out, phase):
        """out = the group's shards t concatenated along axis 0 in rank order
        (src/comm.py:241-243; out has len(group) * t.shape[0] rows)."""
        n = len(group)
        parts = list(out.view(n, *t.shape).unbind(0))
        dist.all_gather(parts, t.contiguous(), group=self.groups[tuple(group)])
        self._rec("allgather", group, None, out, phase)
        return out

    def world_trace(self) -> CommTrace:
        """Every rank's records of the groups it leads (lowest rank), merged
        in rank order: one record per collective of the world."""
        mine = [r for r in self.trace if r.group[0] == self.rank]
        every = [None] * dist.get_world_size()
        dist.all_gather_object(every, mine)
        out = CommTrace()
        for recs in every:
            for r in recs:
                out.add(r.kind, r.group, r.src, r.elements, r.bytes, r.phase)
        return out

    def volume(self, world_reduce=True) -> dict:
        """{(phase, kind): (count, elements)} over the whole world (summed over
        the groups this rank leads, then over ranks)."""
        mine = {}
        for r in self.trace:
            if r.group[0] != self.rank:  # count each group once: by its lowest rank
                continue
            c0, e0 = mine.get((r.phase, r.kind), (0, 0))
            mine[(r.phase, r.kind)] = (c0 + 1, e0 + r.elements)
        if not world_reduce:
            return mine
        keys = [(p, k) for p in PHASES for k in ("broadcast", "allreduce_sum", "allgather")]
        vec = torch.tensor([[mine.get(k, (0, 0))[0], mine.get(k, (0, 0))[1]] for k in keys],
                           dtype=torch.float64)
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        vec = vec.to(dev)
        dist.all_reduce(vec)
        vec = vec.cpu()
        return {k: (int(vec[i, 0]), int(vec[i, 1])) for i, k in enumerate(keys) if vec[i, 0] > 0}


class CudaExec:
    """Branch executor on the native kernels (engine.py)."""

    def __init__(self, cfg, store, precision=None, device=None, checkpoint: bool = False):
        from . import engine as E
        from . import kernels as K
        from .schedules import StepState
        self.E, self.K = E, K
        self.st = StepState(cfg, store, precision, device, checkpoint=checkpoint)
        self.cfg, self.act, self.dev = cfg, self.st.act, self.st.dev
        # activation checkpointing on a BP rank: a branch forward keeps only
        # its inputs; its backward recomputes the branch forward first
        self.checkpoint = checkpoint

    def pack(self, branch):
        """Operand copies of the parameters this rank computes with:
        'msa', 'pair' or 'all'."""
        E = self.E
        subops = {"msa": E.MSA_SUBOPS, "pair": E.PAIR_SUBOPS}.get(branch,
                                                                 E.MSA_SUBOPS + E.PAIR_SUBOPS)
        self.st.pack(subops)

    def grad_bank(self, blk, branch):
        bg = self.st.grads[blk]
        return (bg.msa if branch == "msa" else bg.pair).flat

    def grad_dict(self):
        return self.st.grad_dict()

    def zero_grads(self):
        for bg in self.st.grads:
            bg.msa.flat.zero_()
            bg.pair.flat.zero_()

    def _msa_fwd(self, blk, m, z):
        E, st = self.E, self.st
        m_new, ctxs = E.msa_branch_fwd(st.P, blk, st.packs[blk], m, z, self.cfg, self.act)
        o, co = E.opm_fwd(st.P, f"blk{blk}.opm", st.packs[blk]["opm"], m_new, None, self.cfg,
                          self.act)
        return m_new, o, (ctxs, co)

    def msa_fwd(self, blk, m, z):
        m_new, o, ctx = self._msa_fwd(blk, m, z)
        if self.checkpoint:
            ctx = ("ckpt", m, z)
        return m_new, o, ctx

    def pair_fwd(self, blk, z):
        E, st = self.E, self.st
        z_new, ctx = E.pair_branch_fwd(st.P, blk, st.packs[blk], z, self.cfg, self.act)
        if self.checkpoint:
            ctx = ("ckpt", z)
        return z_new, ctx

    def add(self, a, b):
        out = torch.empty_like(a)
        self.K.add(a, b, out)
        return out

    def div_scalar(self, x, d):
        self.K.div_scalar(x, float(d), x)

    def msa_bwd(self, blk, ctx, dm, d_o):
        E, st = self.E, self.st
        if ctx[0] == "ckpt":          # recompute the branch forward state
            ctx = self._msa_fwd(blk, ctx[1], ctx[2])[2]
        ctxs, co = ctx
        G = st.grads[blk].packed
        e0 = E.msa_emit(G)
        dm3 = E.opm_bwd(st.P, f"blk{blk}.opm", st.packs[blk]["opm"], G["opm"], co, d_o,
                        E.cast_act(d_o, self.act), dm, self.cfg, self.act, emit=e0)
        return E.msa_branch_bwd(st.P, blk, st.packs[blk], G, ctxs, dm3, self.cfg, self.act,
                                handoff=e0)

    def pair_bwd(self, blk, ctx, dz):
        E, st = self.E, self.st
        if isinstance(ctx, tuple) and ctx[0] == "ckpt":
            ctx = E.pair_branch_fwd(st.P, blk, st.packs[blk], ctx[1], self.cfg, self.act)[1]
        return E.pair_branch_bwd(st.P, blk, st.packs[blk], st.grads[blk].packed, ctx, dz,
                                 self.cfg, self.act, dz_act=E.cast_act(dz, self.act))

    def full_step(self, m, z, ev=None):
        from .schedules import full_step
        return full_step(self.st, m, z, fwd_events=ev)

    def sq_mean(self, x):
        loss = self.K.zeros(1, F32, self.dev)
        dx = torch.empty_like(x)
        self.K.sq_mean(x, loss, dx)
        return loss, dx


class DapExec(CudaExec):
    """Branch executor with every sub-op sharded over this rank's DAP group
    (dap.py; src/schedules.py:96-154).  Same interface as CudaExec: the BP
    schedules run on it unchanged, and full_step is the BP=1 step of any
    block wiring (src/evoformer.py:446-458) with the shard hooks."""

    def __init__(self, cfg, store, comm, precision=None, device=None):
        super().__init__(cfg, store, precision, device)
        from . import dap as D
        self.D = D
        self.sh = D.DapShard(comm, comm.dapg)

    def msa_fwd(self, blk, m, z):
        D, st = self.D, self.st
        m_new, c = D.msa_track_fwd(st, self.sh, blk, m, z)
        o, co = D.opm_fwd(st, self.sh, blk, m_new)
        return m_new, o, (c, co)

    def msa_bwd(self, blk, ctx, dm, d_o):
        D, st = self.D, self.st
        c, co = ctx
        dm = self.add(dm, D.opm_bwd(st, self.sh, blk, co, d_o))
        return D.msa_track_bwd(st, self.sh, blk, c, dm)

    def pair_fwd(self, blk, z):
        return self.D.pair_track_fwd(self.st, self.sh, blk, z)

    def pair_bwd(self, blk, ctx, dz):
        return self.D.pair_track_bwd(self.st, self.sh, blk, ctx, dz)

    def replicated(self, blk, branch):
        return self.D.replicated_slices(self.st, blk) if branch == "msa" else []

    def full_step(self, m, z, ev=None):
        D, st, sh, cfg = self.D, self.st, self.sh, self.cfg
        if st.packs is None:
            st.pack()
        s, r = cfg.s, cfg.r
        mc = m.reshape(s * r, cfg.c_m)
        zc = z.reshape(r * r, cfg.c_z)
        _mark(ev, 0)
        ctxs = []
        for blk in range(cfg.n_blocks):
            if cfg.variant == "af2":
                mc, cm = D.msa_track_fwd(st, sh, blk, mc, zc)
                o, co = D.opm_fwd(st, sh, blk, mc)
                zc, cp = D.pair_track_fwd(st, sh, blk, self.add(zc, o))
            elif cfg.variant == "multimer":
                o, co = D.opm_fwd(st, sh, blk, mc)
                zc = self.add(zc, o)
                mc, cm = D.msa_track_fwd(st, sh, blk, mc, zc)
                zc, cp = D.pair_track_fwd(st, sh, blk, zc)
            else:
                m_new, cm = D.msa_track_fwd(st, sh, blk, mc, zc)
                z_b, cp = D.pair_track_fwd(st, sh, blk, zc)
                o, co = D.opm_fwd(st, sh, blk, m_new)
                mc, zc = m_new, self.add(z_b, o)
            ctxs.append((cm, co, cp))
        _mark(ev, 1)
        loss = self.K.zeros(1, F32, mc.device)
        dm, dz = torch.empty_like(mc), torch.empty_like(zc)
        self.K.sq_mean(mc, loss, dm)
        self.K.sq_mean(zc, loss, dz)
        for blk in reversed(range(cfg.n_blocks)):
            cm, co, cp = ctxs[blk]
            ctxs[blk] = None
            if cfg.variant == "af2":
                dz1 = D.pair_track_bwd(st, sh, blk, cp, dz)
                dm = self.add(dm, D.opm_bwd(st, sh, blk, co, dz1))
                dm, dz_row = D.msa_track_bwd(st, sh, blk, cm, dm)
                dz = self.add(dz1, dz_row)
            elif cfg.variant == "multimer":
                dz1 = D.pair_track_bwd(st, sh, blk, cp, dz)
                dm, dz_row = D.msa_track_bwd(st, sh, blk, cm, dm)
                dz1 = self.add(dz1, dz_row)
                dm = self.add(dm, D.opm_bwd(st, sh, blk, co, dz1))
                dz = dz1
            else:
                dz_pair = D.pair_track_bwd(st, sh, blk, cp, dz)
                dm = self.add(dm, D.opm_bwd(st, sh, blk, co, dz))
                dm, dz_row = D.msa_track_bwd(st, sh, blk, cm, dm)
                dz = self.add(dz_pair, dz_row)
        return (mc.reshape(s, r, cfg.c_m), zc.reshape(r, r, cfg.c_z), loss,
                dm.reshape(s, r, cfg.c_m), dz.reshape(r, r, cfg.c_z))


class GraphedExec:
    """Executor wrapper that replays each compute segment of the BP / DP
    schedule (a branch forward, a branch backward, the join add, the loss)
    as a CUDA graph (schedules.SegmentGraphs); the collectives between the
    segments stay host-issued (NCCL / gloo).  The first step runs eagerly
    (warm-up), the second captures, later steps replay."""

    COMPUTE = ("msa_fwd", "pair_fwd", "add", "msa_bwd", "pair_bwd", "sq_mean", "full_step")

    def __init__(self, ex):
        from .schedules import SegmentGraphs
        self.ex = ex
        self.seg = SegmentGraphs()
        self.steps = 0

    def __getattr__(self, name):
        fn = getattr(self.ex, name)
        if name not in self.COMPUTE:
            return fn
        if self.steps == 0:
            return fn
        counter = self._count.setdefault(name, 0)
        self._count[name] = counter + 1

        def call(*args):
            return self.seg((name, counter), fn, *args)
        return call

    def begin_step(self):
        self._count = {}

    def end_step(self):
        self.steps += 1


class ComposedExec:
    """Executor over the C3 composition (schedules.composed_step):
    global block b < K_e is block b of the extra-MSA stack (its own EvoConfig),
    b >= K_e block b - K_e of the main stack.  At the boundary the MSA branch
    drops the extra stack's m_e' and starts the main stack on its own m; in
    the backward the main stack's input gradient dm is kept (``dm_main``) and
    the extra stack's MSA backward is seeded with dm_e' = 0 (the loss reads
    only the main outputs).  The pair stream z runs through both stacks."""

    def __init__(self, ex_extra, ex_main, m_main):
        self.e, self.m, self.m_main = ex_extra, ex_main, m_main
        self.Ke = ex_extra.cfg.n_blocks
        self.dev = ex_main.dev
        self.dm_main = None

    def _pick(self, blk):
        return (self.e, blk) if blk < self.Ke else (self.m, blk - self.Ke)

    def pack(self, branch):
        self.e.pack(branch)
        self.m.pack(branch)

    def grad_bank(self, blk, branch):
        ex, b = self._pick(blk)
        return ex.grad_bank(b, branch)

    def msa_fwd(self, blk, m, z):
        ex, b = self._pick(blk)
        if blk == self.Ke:
            m = self.m_main      # the extra stack's m_e' is dropped
        return ex.msa_fwd(b, m, z)

    def pair_fwd(self, blk, z):
        ex, b = self._pick(blk)
        return ex.pair_fwd(b, z)

    def msa_bwd(self, blk, ctx, dm, d_o):
        ex, b = self._pick(blk)
        dm_in, dz_row = ex.msa_bwd(b, ctx, dm, d_o)
        if blk == self.Ke:
            self.dm_main = dm_in
            cfg = self.e.cfg
            dm_in = self.m.K.zeros((cfg.s * cfg.r, cfg.c_m), F32, self.dev)
        return dm_in, dz_row

    def pair_bwd(self, blk, ctx, dz):
        ex, b = self._pick(blk)
        return ex.pair_bwd(b, ctx, dz)

    def add(self, a, b):
        return self.m.add(a, b)

    def sq_mean(self, x):
        return self.m.sq_mean(x)

    def div_scalar(self, x, d):
        self.m.div_scalar(x, d)


def composed_bp_step(ex_extra, ex_main, comm, m_e, m, z):
    """C3 under branch parallelism (BP=2 in the pair ``comm.pair``): the
    extra-MSA stack feeding the main stack through the same per-block
    schedule as bp_msa_step / bp_pair_step, K_e + K_m blocks.  Call on both
    ranks of the pair; returns (m_out, z_out, loss, dm_e, dm, dz) with the
    fields this rank owns (rank bp 0: m_out, dm_e, dm; rank bp 1: z_out, dz;
    the loss is the rank's half, loss_m or loss_z), and leaves both stacks'
    parameter gradients owner-broadcast over the pair."""
    ce, cm = ex_extra.cfg, ex_main.cfg
    if (ce.r, ce.c_z) != (cm.r, cm.c_z):
        raise ConfigError(f"extra stack (r={ce.r}, c_z={ce.c_z}) does not feed the main "
                          f"stack (r={cm.r}, c_z={cm.c_z})")
    bp_i = comm.layout.coords(comm.rank)[1]
    ex = ComposedExec(ex_extra, ex_main, m.reshape(cm.s * cm.r, cm.c_m))
    if ex_extra.st.packs is None or ex_main.st.packs is None:
        ex.pack("msa" if bp_i == 0 else "pair")
    Kt = ce.n_blocks + cm.n_blocks
    z2 = z.reshape(cm.r * cm.r, cm.c_z)
    if bp_i == 0:
        res = bp_msa_step(ex, comm, m_e.reshape(ce.s * ce.r, ce.c_m), z2, Kt, None)
        out = (res["m_out"].reshape(cm.s, cm.r, cm.c_m), None, res["loss"],
               res["dm"].reshape(ce.s, ce.r, ce.c_m), ex.dm_main.reshape(cm.s, cm.r, cm.c_m),
               None)
    else:
        res = bp_pair_step(ex, comm, z2, Kt, (ce.s * ce.r, ce.c_m))
        out = (None, res["z_out"].reshape(cm.r, cm.r, cm.c_z), res["loss"], None, None,
               res["dz"].reshape(cm.r, cm.r, cm.c_z))
    sync_param_grads(ex, comm, Kt)
    return out


def _mark(ev, i):
    if ev is not None:
        ev[i].record()


def bp_msa_step(ex, comm, m, z, K_blocks, zshape_numel, ev=None):
    """Rank bp_i = 0 (src/schedules.py:214-258).  Returns dict.  ev: two
    CUDA events recorded around the forward (rank_fwd_seconds)."""
    pair = comm.pair
    r0, r1 = pair
    z_cur = z
    ctxs = []
    m_cur = m
    _mark(ev, 0)
    for blk in range(K_blocks):
        m_cur, o, ctx = ex.msa_fwd(blk, m_cur, z_cur)
        ctxs.append(ctx)
        comm.broadcast(pair, r0, o, "fwd")
        z_next = torch.empty_like(z_cur)
        comm.broadcast(pair, r1, z_next, "fwd")
        z_cur = z_next
    _mark(ev, 1)
    loss_m, dm = ex.sq_mean(m_cur)
    for blk in reversed(range(K_blocks)):
        d_o = torch.empty_like(z_cur)
        comm.broadcast(pair, r1, d_o, "bwd")
        dm, dz_row = ex.msa_bwd(blk, ctxs[blk], dm, d_o)
        ctxs[blk] = None
        comm.allreduce_sum(pair, dz_row, "bwd")     # dz_row + dz_pair (rank order)
    comm.broadcast(pair, r0, dm, "bwd")
    return dict(m_out=m_cur, z_out=z_cur, loss=loss_m, dm=dm, dz=dz_row)


def bp_pair_step(ex, comm, z, K_blocks, mshape, ev=None):
    """Rank bp_i = 1 (src/schedules.py:261-297)."""
    pair = comm.pair
    r0, r1 = pair
    z_cur = z
    ctxs = []
    _mark(ev, 0)
    for blk in range(K_blocks):
        z_b, ctx = ex.pair_fwd(blk, z_cur)
        ctxs.append(ctx)
        o = torch.empty_like(z_b)
        comm.broadcast(pair, r0, o, "fwd")
        z_cur = ex.add(z_b, o)                     # z'' = z_pair + o (:276-280)
        comm.broadcast(pair, r1, z_cur, "fwd")
    _mark(ev, 1)
    loss_z, dz = ex.sq_mean(z_cur)
    for blk in reversed(range(K_blocks)):
        comm.broadcast(pair, r1, dz, "bwd")        # dz'' -> seeds o on rank 0
        dz_pair = ex.pair_bwd(blk, ctxs[blk], dz)
        ctxs[blk] = None
        comm.allreduce_sum(pair, dz_pair, "bwd")
        dz = dz_pair
    dm = torch.empty(mshape, dtype=z.dtype, device=z.device)
    comm.broadcast(pair, r0, dm, "bwd")
    return dict(z_out=z_cur, loss=loss_z, dz=dz)


def sync_param_grads(ex, comm, K_blocks):
    """src/schedules.py:300-329: the DAP group's sum of the shard partials
    (every parameter but the replicated ones), owner broadcast over the BP
    pair (one bucket per branch per block), then sum / dp over the DP group."""
    lay = comm.layout
    if lay.dap > 1:
        bp_i = lay.coords(comm.rank)[1]
        mine = ("msa", "pair") if lay.bp == 1 else (("msa",) if bp_i == 0 else ("pair",))
        for blk in range(K_blocks):
            for br in mine:
                g = ex.grad_bank(blk, br)
                pos = 0
                for off, n in sorted(ex.replicated(blk, br)) + [(g.numel(), 0)]:
                    if off > pos:
                        comm.allreduce_sum(comm.dapg, g[pos:off], "param")
                    pos = off + n
    if lay.bp == 2:
        r0, r1 = comm.pair
        for blk in range(K_blocks):
            comm.broadcast(comm.pair, r0, ex.grad_bank(blk, "msa"), "param")
            comm.broadcast(comm.pair, r1, ex.grad_bank(blk, "pair"), "param")
    if lay.dp > 1:
        for blk in range(K_blocks):
            for br in ("msa", "pair"):
                g = ex.grad_bank(blk, br)
                comm.allreduce_sum(comm.dpg, g, "param")
                ex.div_scalar(g, lay.dp)


class DistributedStep:
    """One train step of the (dp, bp) layout on this rank's GPU."""

    def __init__(self, cfg, store, layout: ParallelLayout, precision=None, comm=None,
                 executor=None, graphs: bool = False):
        layout.validate_model(cfg)
        self.cfg, self.layout = cfg, layout
        self.comm = comm or Comm(layout)
        self.rank = self.comm.rank
        self.dp_i, self.bp_i, _ = layout.coords(self.rank)
        if executor is None:
            executor = (DapExec(cfg, store, self.comm, precision) if layout.dap > 1
                        else CudaExec(cfg, store, precision))
        self.ex = executor
        # DAP segments hold collectives: no per-segment graph capture
        if graphs and layout.dap == 1:
            self.ex = GraphedExec(self.ex)
        if layout.bp == 2:
            self.ex.pack("msa" if self.bp_i == 0 else "pair")
        else:
            self.ex.pack("all")

    def step(self, m, z, ev=None):
        """m [s, r, c_m], z [r, r, c_z] on this rank's device.  Returns the
        tuple (m_out, z_out, loss, dm, dz) of fields this rank owns (others
        None); parameter gradients are left synchronised in the executor.
        ev: optional two CUDA events recorded around the forward."""
        cfg, lay, ex = self.cfg, self.layout, self.ex
        s, r = cfg.s, cfg.r
        m2 = m.reshape(s * r, cfg.c_m)
        z2 = z.reshape(r * r, cfg.c_z)
        graphed = isinstance(ex, GraphedExec)
        if graphed:
            ex.begin_step()
            if ex.steps > 0:
                ev = None      # events are not recorded inside the graphs
        try:
            return self._step(ex, cfg, lay, s, r, m, z, m2, z2, ev)
        finally:
            if graphed:
                ex.end_step()

    def _step(self, ex, cfg, lay, s, r, m, z, m2, z2, ev):
        if lay.bp == 1:
            out = ex.full_step(m, z, ev) if ev is not None else ex.full_step(m, z)
            sync_param_grads(ex, self.comm, cfg.n_blocks)
            return out
        if self.bp_i == 0:
            res = bp_msa_step(ex, self.comm, m2, z2, cfg.n_blocks, None, ev)
            out = (res["m_out"].reshape(s, r, cfg.c_m), None, res["loss"],
                   res["dm"].reshape(s, r, cfg.c_m), None)
        else:
            res = bp_pair_step(ex, self.comm, z2, cfg.n_blocks, (s * r, cfg.c_m), ev)
            out = (None, res["z_out"].reshape(r, r, cfg.c_z), res["loss"], None,
                   res["dz"].reshape(r, r, cfg.c_z))
        sync_param_grads(ex, self.comm, cfg.n_blocks)
        return out


def run_distributed(cfg, store, layout: ParallelLayout, seed: int = 32,
                    max_threads: int | None = None, *, precision=None, comm=None,
                    executor=None) -> RunResult:
    """SPMD train step under `layout` (src/schedules.py:332-384).

    Inside an initialised process group (torchrun, one rank per GPU) call it
    on every rank.  Without one it launches the world itself, like the
    reference (src/schedules.py:338-361): layout.world_size processes, rank r
    on cuda:(r % device_count), NCCL when every rank has its own GPU and gloo
    otherwise; the RunResult comes back to the caller.  max_threads is the
    reference's thread cap for its simulated world and has no effect here.

    The RunResult carries the dp_idx = 0 replica's outputs and input
    gradients (gathered within its BP pair), the dp-mean loss, the
    synchronised parameter gradients, the world's CommTrace (one record per
    collective of the step, src/comm.py:52-110) and each rank's forward
    device time in rank_fwd_seconds."""
    layout.validate_model(cfg)
    if comm is None and executor is None and not dist.is_initialized():
        return _spawn_world(cfg, store, layout, seed, precision)
    runner = DistributedStep(cfg, store, layout, precision, comm, executor)
    dev = runner.ex.dev
    samples = make_batch(cfg, seed, layout.dp, device=dev)
    m, z = samples[runner.dp_i]
    ev = ([torch.cuda.Event(enable_timing=True) for _ in range(2)]
          if dev.type == "cuda" else None)
    t0 = time.perf_counter()
    m_out, z_out, loss, dm, dz = runner.step(m, z, ev)
    # replica loss = loss_m + loss_z in the loss dtype (the BP=1 step adds the
    # two means into one fp32 accumulator in the same order: bitwise equal),
    # then the mean over dp
    lt = loss.reshape(1).clone()
    if layout.bp == 2:
        runner.comm.allreduce_sum(runner.comm.pair, lt, None)
    if layout.dp > 1:
        runner.comm.allreduce_sum(runner.comm.dpg, lt, None)
        lt /= layout.dp
    if layout.bp == 2:
        # complete the pair's view: rank0 owns m_out/dm, rank1 z_out/dz
        r0, r1 = runner.comm.pair
        if runner.bp_i == 0:
            z_out_t, dz_t = torch.empty_like(z), torch.empty_like(z)
            m_out_t, dm_t = m_out.contiguous(), dm.contiguous()
        else:
            m_out_t, dm_t = torch.empty_like(m), torch.empty_like(m)
            z_out_t, dz_t = z_out.contiguous(), dz.contiguous()
        for t, src in ((m_out_t, r0), (dm_t, r0), (z_out_t, r1), (dz_t, r1)):
            runner.comm.broadcast(runner.comm.pair, src, t, None)
        m_out, dm, z_out, dz = m_out_t, dm_t, z_out_t, dz_t
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    wall = time.perf_counter() - t0
    fwd = ev[0].elapsed_time(ev[1]) / 1e3 if ev is not None else float("nan")
    every = [None] * dist.get_world_size()
    dist.all_gather_object(every, fwd)
    return RunResult(m_out, z_out, float(lt.item()), dm, dz, runner.ex.grad_dict(),
                     runner.comm.world_trace(), dict(enumerate(every)), wall)


def run_bp(cfg, store, seed: int = 32, max_threads=None, *, precision=None) -> RunResult:
    """Branch parallelism, BP=2 (src/schedules.py:402-403)."""
    return run_distributed(cfg, store, ParallelLayout(bp=2), seed, max_threads,
                           precision=precision)


def run_dp(cfg, store, dp: int, seed: int = 32, max_threads=None, *, precision=None) -> RunResult:
    """Data parallelism over dp replicas (src/schedules.py:410-411)."""
    return run_distributed(cfg, store, ParallelLayout(dp=dp), seed, max_threads,
                           precision=precision)


def run_dap(cfg, store, dap: int, seed: int = 32, max_threads=None, *, precision=None):
    """DAP axial sharding over dap ranks (src/schedules.py:406-407)."""
    return run_distributed(cfg, store, ParallelLayout(dap=dap), seed, max_threads,
                           precision=precision)


# ---------------------------------------------------------------------------
# self-launched world (no process group yet): the reference's World.run
# ---------------------------------------------------------------------------

def _world_main(rank, world, init_file, backend, cfg, store_np, layout, seed, precision, q):
    import traceback
    try:
        ndev = torch.cuda.device_count()
        dev = torch.device("cuda", rank % ndev)
        torch.cuda.set_device(dev)
        kw = dict(backend=backend, init_method=f"file://{init_file}", rank=rank,
                  world_size=world)
        if backend == "nccl":
            kw["device_id"] = dev
        dist.init_process_group(**kw)
        try:
            from .evoformer import ParamStore
            store = ParamStore()
            for name, (arr, branch) in store_np.items():
                store.add(name, torch.as_tensor(arr, device=dev), branch)
            res = run_distributed(cfg, store, layout, seed, precision=precision)
            if rank == 0:
                q.put(("ok", rank, res.numpy()))
            else:
                q.put(("ok", rank, None))
        finally:
            dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        q.put(("err", rank, traceback.format_exc()))


def _spawn_world(cfg, store, layout, seed, precision):
    import tempfile
    import torch.multiprocessing as mp
    world = layout.world_size
    if not torch.cuda.is_available():
        raise WorldError("run_distributed needs CUDA devices (the native kernels)")
    ndev = torch.cuda.device_count()
    backend = "nccl" if ndev >= world else "gloo"
    store_np = {n: (t.detach().cpu().numpy(), store.branch(n)) for n, t in store.items()}
    fd, init_file = tempfile.mkstemp(prefix="evo_world_")
    os.close(fd)
    os.unlink(init_file)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_world_main, args=(r, world, init_file, backend, cfg, store_np,
                                                   layout, seed, precision, q))
             for r in range(world)]
    t0 = time.perf_counter()
    for p in procs:
        p.start()
    result, errors = None, []
    for _ in range(world):
        status, rank, payload = q.get()
        if status == "ok" and rank == 0:
            result = payload
        elif status == "err":
            errors.append(f"rank {rank}:\n{payload}")
    for p in procs:
        p.join(timeout=120)
    if os.path.exists(init_file):
        os.unlink(init_file)
    if errors or result is None:
        raise WorldError("self-launched world failed:\n" + "\n".join(errors))
    dev = store.device

    def back(x):
        return torch.as_tensor(x, device=dev)
    return RunResult(back(result.m_out), back(result.z_out), result.loss, back(result.dm),
                     back(result.dz), {k: back(v) for k, v in result.grads.items()},
                     result.trace, result.rank_fwd_seconds, time.perf_counter() - t0)
