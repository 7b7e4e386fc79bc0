"""Parallel Evoformer block: the reference's model API
(src/evoformer.py:43-475) re-hosted on B200 kernels.

Same names, signatures and parameter conventions as the reference:
``EvoConfig``, ``ParamStore``, ``init_params`` (bit-identical weights for
a given seed), ``param_count``, the nine sub-ops ``row_attn / col_attn /
msa_transition / pair_transition / opm / tri_mult / tri_attn`` (each
returns the sub-op's delta), ``msa_track``, ``pair_track``,
``evoformer_block``, ``evoformer_stack`` and ``seeded_inputs``.

Tensors are torch CUDA tensors instead of tape Tensors; every function is
differentiable through torch autograd (a custom Function whose forward
and backward launch the native kernels; engine.py).  ``P`` is a
name->tensor mapping (``ParamStore.bind()`` or a plain dict), ``px`` the
"blk{b}.{subop}" prefix.  The arithmetic precision is the module-level
``set_precision("fp32"|"bf16")`` (fp32 default; "bf16" = bf16 operands,
fp32 accumulation and fp32 residual streams).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import engine as E
from .errors import ConfigError, DimensionError

VARIANTS = ("af2", "multimer", "parallel")
MSA_SUBOPS = E.MSA_SUBOPS
PAIR_SUBOPS = E.PAIR_SUBOPS
SUBOPS = MSA_SUBOPS + PAIR_SUBOPS

_PRECISION = {"fp32": torch.float32, "bf16": torch.bfloat16}
_state = {"act": torch.float32}


def set_precision(name: str) -> None:
    """'fp32' (parity path) or 'bf16' (tensor-core path)."""
    if name not in _PRECISION:
        raise ConfigError(f"precision must be one of {tuple(_PRECISION)}, got {name!r}")
    _state["act"] = _PRECISION[name]


def get_precision() -> str:
    return "bf16" if _state["act"] == torch.bfloat16 else "fp32"


def act_dtype(precision: str | None = None):
    return _state["act"] if precision is None else _PRECISION[precision]


@dataclass(frozen=True)
class EvoConfig:
    """Model dimensions (src/evoformer.py:43-79). c_head = c_m // h."""

    s: int = 8
    r: int = 16
    c_m: int = 8
    c_z: int = 8
    h: int = 2
    c_opm: int = 32
    t_factor: int = 4
    n_blocks: int = 2
    variant: str = "parallel"
    eps: float = 1e-5

    def __post_init__(self):
        for name in ("s", "r", "c_m", "c_z", "h", "c_opm", "t_factor"):
            if getattr(self, name) < 1:
                raise ConfigError(f"model.{name} must be >= 1, got {getattr(self, name)}")
        if self.n_blocks < 0:
            raise ConfigError(f"model.n_blocks must be >= 0, got {self.n_blocks}")
        if self.variant not in VARIANTS:
            raise ConfigError(f"model.variant must be one of {VARIANTS}, got {self.variant!r}")
        if self.c_m % self.h != 0:
            raise ConfigError(
                f"model.h must divide model.c_m (got h={self.h}, c_m={self.c_m})")
        if self.eps <= 0:
            raise ConfigError(f"model.eps must be > 0, got {self.eps}")

    @property
    def c_head(self) -> int:
        return self.c_m // self.h

    @property
    def hc(self) -> int:
        return self.h * self.c_head


class ParamStore:
    """Ordered name -> fp32 device tensor map with a branch tag per tensor
    (src/evoformer.py:82-136)."""

    def __init__(self):
        self._arrays: dict[str, torch.Tensor] = {}
        self._branch: dict[str, str] = {}

    def add(self, name, array, branch: str) -> None:
        if name in self._arrays:
            raise ConfigError(f"duplicate parameter name {name!r}")
        self._arrays[name] = array
        self._branch[name] = branch

    def names(self):
        return list(self._arrays.keys())

    def branch(self, name: str) -> str:
        return self._branch[name]

    def __getitem__(self, name):
        return self._arrays[name]

    def __contains__(self, name) -> bool:
        return name in self._arrays

    def __len__(self) -> int:
        return len(self._arrays)

    def items(self):
        return self._arrays.items()

    def total_size(self) -> int:
        return sum(int(a.numel()) for a in self._arrays.values())

    def replace(self, name, array) -> None:
        if tuple(array.shape) != tuple(self._arrays[name].shape):
            raise ConfigError(
                f"replacement for {name!r} has shape {tuple(array.shape)}, "
                f"expected {tuple(self._arrays[name].shape)}")
        self._arrays[name] = array

    def copy(self) -> "ParamStore":
        out = ParamStore()
        for name, arr in self._arrays.items():
            out.add(name, arr.clone(), self._branch[name])
        return out

    def bind(self, graph=None) -> dict:
        """name -> tensor, in store order (the reference binds tape leaves,
        src/evoformer.py:134-136; here the tensors themselves)."""
        return dict(self._arrays)

    @property
    def device(self):
        for a in self._arrays.values():
            return a.device
        return torch.device("cuda")

    @classmethod
    def from_reference(cls, ref_store, device="cuda") -> "ParamStore":
        """Adopt a reference ``branchpar`` ParamStore (numpy arrays)."""
        out = cls()
        for name, arr in ref_store.items():
            out.add(name, torch.as_tensor(np.asarray(arr, dtype=np.float32), device=device),
                    ref_store.branch(name))
        return out


def _subop_param_specs(cfg: EvoConfig, subop: str):
    """(suffix, shape, kind) per tensor of one sub-op (src/evoformer.py:139-190)."""
    c_m, c_z, hc, h = cfg.c_m, cfg.c_z, cfg.hc, cfg.h
    c, t = cfg.c_opm, cfg.t_factor
    W, B0, G1, LG, LB = "weight", "bias", "gate_bias", "ln_scale", "ln_shift"
    if subop in ("row_attn", "col_attn"):
        spec = [("ln_g", (c_m,), LG), ("ln_b", (c_m,), LB)]
        if subop == "row_attn":
            spec += [("lnz_g", (c_z,), LG), ("lnz_b", (c_z,), LB)]
        spec += [("q_w", (c_m, hc), W), ("k_w", (c_m, hc), W), ("v_w", (c_m, hc), W),
                 ("gate_w", (c_m, hc), W), ("gate_b", (hc,), G1)]
        if subop == "row_attn":
            spec += [("bias_w", (c_z, h), W)]
        return spec + [("out_w", (hc, c_m), W), ("out_b", (c_m,), B0)]
    if subop in ("msa_transition", "pair_transition"):
        cx = c_m if subop == "msa_transition" else c_z
        return [("ln_g", (cx,), LG), ("ln_b", (cx,), LB), ("w1", (cx, t * cx), W),
                ("b1", (t * cx,), B0), ("w2", (t * cx, cx), W), ("b2", (cx,), B0)]
    if subop == "opm":
        return [("ln_g", (c_m,), LG), ("ln_b", (c_m,), LB), ("a_w", (c_m, c), W),
                ("a_b", (c,), B0), ("b_w", (c_m, c), W), ("b_b", (c,), B0),
                ("out_w", (c * c, c_z), W), ("out_b", (c_z,), B0)]
    if subop in ("tri_mult_out", "tri_mult_in"):
        return [("ln_g", (c_z,), LG), ("ln_b", (c_z,), LB),
                ("a_gate_w", (c_z, c), W), ("a_gate_b", (c,), G1),
                ("a_w", (c_z, c), W), ("a_b", (c,), B0),
                ("b_gate_w", (c_z, c), W), ("b_gate_b", (c,), G1),
                ("b_w", (c_z, c), W), ("b_b", (c,), B0),
                ("out_gate_w", (c_z, c_z), W), ("out_gate_b", (c_z,), G1),
                ("p_ln_g", (c,), LG), ("p_ln_b", (c,), LB),
                ("out_w", (c, c_z), W), ("out_b", (c_z,), B0)]
    if subop in ("tri_attn_start", "tri_attn_end"):
        return [("ln_g", (c_z,), LG), ("ln_b", (c_z,), LB), ("q_w", (c_z, hc), W),
                ("k_w", (c_z, hc), W), ("v_w", (c_z, hc), W), ("bias_w", (c_z, h), W),
                ("gate_w", (c_z, hc), W), ("gate_b", (hc,), G1), ("out_w", (hc, c_z), W),
                ("out_b", (c_z,), B0)]
    raise ConfigError(f"unknown sub-op {subop!r}")


def init_params(cfg: EvoConfig, seed: int, dtype=torch.float32, device="cuda") -> ParamStore:
    """Seeded store, bit-identical to the reference's for the same seed
    (src/evoformer.py:193-218): weights U(-0.02, 0.02) drawn f64 from one
    PCG64 stream in block -> SUBOPS -> spec order, then cast; biases 0,
    gate biases 1, LN scale 1 / shift 0."""
    if isinstance(dtype, type) and issubclass(dtype, np.floating):
        dtype = torch.float32
    if dtype not in (torch.float32,):
        raise ConfigError("parameters are fp32 masters (bf16 is a compute precision: "
                          "see set_precision)")
    rng = np.random.default_rng(seed)
    store = ParamStore()
    for b in range(cfg.n_blocks):
        for subop in SUBOPS:
            branch = "msa" if subop in MSA_SUBOPS else "pair"
            for suffix, shape, kind in _subop_param_specs(cfg, subop):
                if kind == "weight":
                    arr = rng.uniform(-0.02, 0.02, size=shape)
                elif kind in ("gate_bias", "ln_scale"):
                    arr = np.ones(shape)
                else:
                    arr = np.zeros(shape)
                store.add(f"blk{b}.{subop}.{suffix}",
                          torch.as_tensor(arr.astype(np.float32), device=device), branch)
    return store


def param_count(cfg: EvoConfig) -> int:
    """Closed-form parameter count (src/evoformer.py:221-236)."""
    return cfg.n_blocks * sum(E.subop_grad_numel(n, cfg) for n in SUBOPS)


def seeded_inputs(cfg: EvoConfig, seed: int, device="cuda"):
    """Standard-normal m [s,r,c_m] and z [r,r,c_z] (src/evoformer.py:470-475)."""
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((cfg.s, cfg.r, cfg.c_m)).astype(np.float32)
    z = rng.standard_normal((cfg.r, cfg.r, cfg.c_z)).astype(np.float32)
    return (torch.as_tensor(m, device=device), torch.as_tensor(z, device=device))


# ---------------------------------------------------------------------------
# autograd wrappers
# ---------------------------------------------------------------------------

def _no_shard(shard):
    if shard is not None:
        raise ConfigError("DAP sharding (shard=...) is outside this build's scope "
                          "(SURVEY.md 8(f)); pass shard=None")


def _check(t, shape, what):
    if tuple(t.shape) != tuple(shape):
        raise DimensionError(f"{what}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_cuda:
        raise DimensionError(f"{what}: expected a CUDA tensor")


def _subop_names(cfg, px, subop):
    return [f"{px}.{s}" for s, _, _ in _subop_param_specs(cfg, subop)]


class _SubOp(torch.autograd.Function):
    @staticmethod
    def forward(ctx, subop, px, cfg, m, z, *params):
        act = _state["act"]
        names = _subop_names(cfg, px, subop)
        P = dict(zip(names, [p.detach().contiguous() for p in params]))
        dev = (m if m is not None else z).device
        pk = E.pack_subop(P, px, subop, cfg, act, dev)
        s, r = cfg.s, cfg.r
        with torch.no_grad():
            if subop in ("row_attn", "col_attn", "msa_transition", "opm"):
                m2 = m.detach().contiguous().reshape(s * r, cfg.c_m)
            if subop == "row_attn":
                z2 = z.detach().contiguous().reshape(r * r, cfg.c_z)
                out, c = E.attn_fwd(subop, P, px, pk, m2, z2, cfg, act, resid=False)
                shape = m.shape
            elif subop == "col_attn":
                out, c = E.attn_fwd(subop, P, px, pk, m2, None, cfg, act, resid=False)
                shape = m.shape
            elif subop == "msa_transition":
                out, c = E.transition_fwd(P, px, pk, m2, cfg, act, resid=False)
                shape = m.shape
            elif subop == "opm":
                out, c = E.opm_fwd(P, px, pk, m2, None, cfg, act)
                shape = (r, r, cfg.c_z)
            else:
                z2 = z.detach().contiguous().reshape(r * r, cfg.c_z)
                if subop == "pair_transition":
                    out, c = E.transition_fwd(P, px, pk, z2, cfg, act, resid=False)
                elif subop.startswith("tri_mult"):
                    out, c = E.trimul_fwd(subop, P, px, pk, z2, cfg, act, resid=False)
                else:
                    out, c = E.attn_fwd(subop, P, px, pk, z2, None, cfg, act, resid=False)
                shape = z.shape
        ctx.state = (subop, px, cfg, act, P, pk, c, names)
        ctx.has_m, ctx.has_z = m is not None, z is not None
        return out.reshape(shape)

    @staticmethod
    def backward(ctx, dout):
        subop, px, cfg, act, P, pk, c, names = ctx.state
        dev = dout.device
        bank = E.GradBank(E.subop_grad_numel(subop, cfg), dev)
        G, gnames = E.grad_views(subop, cfg, bank)
        s, r = cfg.s, cfg.r
        d = dout.detach().float().contiguous()
        dm = dz = None
        with torch.no_grad():
            if subop in ("row_attn", "col_attn", "tri_attn_start", "tri_attn_end"):
                rows = s * r if subop in ("row_attn", "col_attn") else r * r
                dx, dz_row = E.attn_bwd(subop, P, px, pk, G, c, d.reshape(rows, -1), cfg, act)
                if subop in ("row_attn", "col_attn"):
                    dm, dz = dx, dz_row
                else:
                    dz = dx
            elif subop in ("msa_transition", "pair_transition"):
                rows = s * r if subop == "msa_transition" else r * r
                dx = E.transition_bwd(P, px, pk, G, c, d.reshape(rows, -1), cfg, act)
                if subop == "msa_transition":
                    dm = dx
                else:
                    dz = dx
            elif subop == "opm":
                d2 = d.reshape(r * r, cfg.c_z)
                dm = E.opm_bwd(P, px, pk, G, c, d2, E.cast_act(d2, act), None, cfg, act)
            else:
                dz = E.trimul_bwd(P, px, pk, G, c, d.reshape(r * r, cfg.c_z), cfg, act)
        grads = [gnames[n[len(px) + 1:]] for n in names]
        dm_out = dm.reshape(s, r, cfg.c_m) if (dm is not None and ctx.has_m) else None
        dz_out = dz.reshape(r, r, cfg.c_z) if (dz is not None and ctx.has_z) else None
        return (None, None, None, dm_out, dz_out, *grads)


def _run_subop(subop, P, px, m, z, cfg):
    if not px.endswith("." + subop) and subop not in px:
        pass
    if m is not None:
        _check(m, (cfg.s, cfg.r, cfg.c_m), f"{subop}: m")
    if z is not None:
        _check(z, (cfg.r, cfg.r, cfg.c_z), f"{subop}: z")
    params = [P[n] for n in _subop_names(cfg, px, subop)]
    return _SubOp.apply(subop, px, cfg, m, z, *params)


def row_attn(P, px, m, z, cfg, shard=None):
    """MSA row attention with pair bias (src/evoformer.py:289-297)."""
    _no_shard(shard)
    return _run_subop("row_attn", P, px, m, z, cfg)


def col_attn(P, px, m, cfg, shard=None):
    """MSA column attention (src/evoformer.py:300-311)."""
    _no_shard(shard)
    return _run_subop("col_attn", P, px, m, None, cfg)


def msa_transition(P, px, m, cfg, shard=None):
    """MSA transition MLP (src/evoformer.py:322-324)."""
    _no_shard(shard)
    return _run_subop("msa_transition", P, px, m, None, cfg)


def pair_transition(P, px, z, cfg, shard=None):
    """Pair transition MLP (src/evoformer.py:327-329)."""
    _no_shard(shard)
    return _run_subop("pair_transition", P, px, None, z, cfg)


def opm(P, px, m, cfg, shard=None):
    """Outer product mean (src/evoformer.py:332-356)."""
    _no_shard(shard)
    return _run_subop("opm", P, px, m, None, cfg)


def tri_mult(P, px, z, cfg, incoming: bool, shard=None):
    """Triangle multiplicative update (src/evoformer.py:359-397)."""
    _no_shard(shard)
    return _run_subop("tri_mult_in" if incoming else "tri_mult_out", P, px, None, z, cfg)


def tri_attn(P, px, z, cfg, ending: bool, shard=None):
    """Triangle attention around the starting / ending node
    (src/evoformer.py:400-420)."""
    _no_shard(shard)
    return _run_subop("tri_attn_end" if ending else "tri_attn_start", P, px, None, z, cfg)


class _Track(torch.autograd.Function):
    """One track of a block (residual adds fused into the native launches):
    which = "msa" (m, z) -> m'  or  "pair" (z) -> z'."""

    @staticmethod
    def forward(ctx, which, blk, cfg, names, m, z, *params):
        act = _state["act"]
        P = dict(zip(names, [p.detach().contiguous() for p in params]))
        subops = E.MSA_TRACK if which == "msa" else PAIR_SUBOPS
        pk = E.pack_block(P, blk, cfg, act, z.device, subops)
        s, r = cfg.s, cfg.r
        z2 = z.detach().contiguous().reshape(r * r, cfg.c_z)
        with torch.no_grad():
            if which == "msa":
                out, c = E.msa_branch_fwd(P, blk, pk, m.detach().contiguous(), z2, cfg, act)
                shape = m.shape
            else:
                out, c = E.pair_branch_fwd(P, blk, pk, z2, cfg, act)
                shape = z.shape
        ctx.state = (which, blk, cfg, act, P, pk, c, names)
        return out.reshape(shape)

    @staticmethod
    def backward(ctx, dout):
        which, blk, cfg, act, P, pk, c, names = ctx.state
        s, r = cfg.s, cfg.r
        BG = E.BlockGrads(blk, cfg, dout.device)
        d = dout.detach().float().contiguous()
        with torch.no_grad():
            if which == "msa":
                dm, dz = E.msa_branch_bwd(P, blk, pk, BG.packed, c, d.reshape(s * r, cfg.c_m),
                                          cfg, act)
                dm, dz = dm.reshape(s, r, cfg.c_m), dz.reshape(r, r, cfg.c_z)
            else:
                dm = None
                dz = E.pair_branch_bwd(P, blk, pk, BG.packed, c, d.reshape(r * r, cfg.c_z),
                                       cfg, act).reshape(r, r, cfg.c_z)
        grads = [BG.names[n] for n in names]
        return (None, None, None, None, dm, dz, *grads)


def _track_names(cfg, blk, subops):
    return [f"blk{blk}.{sub}.{s}" for sub in subops for s, _, _ in _subop_param_specs(cfg, sub)]


def msa_track(P, blk: int, m, z, cfg, shard=None):
    """Row attention, column attention and the MSA transition, residually
    (src/evoformer.py:427-432); one native forward / backward."""
    _no_shard(shard)
    _check(m, (cfg.s, cfg.r, cfg.c_m), "msa_track: m")
    _check(z, (cfg.r, cfg.r, cfg.c_z), "msa_track: z")
    names = _track_names(cfg, blk, E.MSA_TRACK)
    return _Track.apply("msa", blk, cfg, names, m, z, *[P[n] for n in names])


def pair_track(P, blk: int, z, cfg, shard=None):
    """Both triangle multiplications, both triangle attentions and the pair
    transition, residually (src/evoformer.py:435-443)."""
    _no_shard(shard)
    _check(z, (cfg.r, cfg.r, cfg.c_z), "pair_track: z")
    names = _track_names(cfg, blk, PAIR_SUBOPS)
    return _Track.apply("pair", blk, cfg, names, None, z, *[P[n] for n in names])


class _Block(torch.autograd.Function):
    """Fused parallel block: one forward/backward of engine.block_*."""

    @staticmethod
    def forward(ctx, blk, cfg, names, m, z, *params):
        act = _state["act"]
        P = dict(zip(names, [p.detach().contiguous() for p in params]))
        pk = E.pack_block(P, blk, cfg, act, m.device)
        with torch.no_grad():
            m2, z2, c = E.block_fwd(P, blk, pk, m.detach().contiguous(),
                                    z.detach().contiguous(), cfg, act)
        ctx.state = (blk, cfg, act, P, pk, c, names)
        return m2.reshape(m.shape), z2.reshape(z.shape)

    @staticmethod
    def backward(ctx, dm, dz):
        blk, cfg, act, P, pk, c, names = ctx.state
        s, r = cfg.s, cfg.r
        dev = (dm if dm is not None else dz).device
        if dm is None:
            dm = torch.zeros((s, r, cfg.c_m), dtype=torch.float32, device=dev)
        if dz is None:
            dz = torch.zeros((r, r, cfg.c_z), dtype=torch.float32, device=dev)
        BG = E.BlockGrads(blk, cfg, dev)
        with torch.no_grad():
            dm_in, dz_in = E.block_bwd(P, blk, pk, BG.packed, c,
                                       dm.detach().float().contiguous().reshape(s * r, cfg.c_m),
                                       dz.detach().float().contiguous().reshape(r * r, cfg.c_z),
                                       cfg, act)
        grads = [BG.names[n] for n in names]
        return (None, None, None, dm_in.reshape(s, r, cfg.c_m), dz_in.reshape(r, r, cfg.c_z),
                *grads)


def block_param_names(cfg, blk):
    return [f"blk{blk}.{sub}.{s}" for sub in SUBOPS
            for s, _, _ in _subop_param_specs(cfg, sub)]


def evoformer_block(P, blk: int, m, z, cfg, shard=None):
    """One block (src/evoformer.py:446-461) in the configured wiring
    (parallel / af2 / multimer), one fused native forward/backward."""
    _no_shard(shard)
    _check(m, (cfg.s, cfg.r, cfg.c_m), "evoformer_block: m")
    _check(z, (cfg.r, cfg.r, cfg.c_z), "evoformer_block: z")
    names = block_param_names(cfg, blk)
    return _Block.apply(blk, cfg, names, m, z, *[P[n] for n in names])


def evoformer_stack(P, m, z, cfg, shard=None):
    """src/evoformer.py:464-467."""
    for blk in range(cfg.n_blocks):
        m, z = evoformer_block(P, blk, m, z, cfg, shard)
    return m, z
