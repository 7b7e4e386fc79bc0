"""Parity of the CUDA path against the reference (golden vectors produced
by the reference itself) and the pinned numpy oracle.

Bars (BASELINE.json north_star): per-tensor rel-L2 <= 1e-5 on the fp32
path and <= 2e-2 on the bf16 path, for the output deltas, dm, dz and
every parameter gradient.
"""

import numpy as np
import pytest
import torch

from helpers import (CONFIGS, golden_as_want, load_golden, normalise_by_reference_f32,
                     rel_l2, step_errors, to_np)

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2


@pytest.fixture(scope="module")
def pkg():
    import paper_2211_00235_b200 as p
    assert torch.cuda.is_available(), "GPU tests need a B200"
    return p


def _worst(errs):
    # NaN sorts as the worst (max() with a NaN key would skip it)
    k = max(errs, key=lambda n: errs[n] if errs[n] == errs[n] else float("inf"))
    v = errs[k]
    return k, (v if v == v else float("inf"))


@pytest.mark.parametrize("tag", ["toy", "odd", "c1"])
def test_step_fp32_matches_reference_golden(pkg, tag):
    cfg = pkg.EvoConfig(**CONFIGS[tag])
    store = pkg.init_params(cfg, 32)
    res = pkg.run_single(cfg, store, seed=32, precision="fp32")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    gold = load_golden(tag)
    want = golden_as_want(gold)
    errs = normalise_by_reference_f32(step_errors(res, want, m_in, z_in, bar=FP32_TOL), want,
                                      FP32_TOL)
    k, v = _worst(errs)
    assert v <= FP32_TOL, f"{tag}: worst {k} rel-L2 {v:.3e}"
    assert abs(res.loss - float(gold["loss"])) <= 1e-5 * abs(float(gold["loss"]))


_ORACLE = {}


def _oracle_step(tag, **over):
    """The pinned oracle's step (float64), cached per configuration."""
    key = (tag, tuple(sorted(over.items())))
    if key not in _ORACLE:
        from oracle import evoformer_np as O
        d = O.Dims(**{**CONFIGS[tag], **over})
        P = O.init_params(d, 32)
        _ORACLE.clear()       # keep at most one large oracle result alive
        _ORACLE[key] = O.run_single(d, P, seed=32)
    return _ORACLE[key]


@pytest.mark.parametrize("precision,tol", [("fp32", FP32_TOL), ("bf16", BF16_TOL)])
def test_step_mid_matches_oracle(pkg, precision, tol):
    cfg = pkg.EvoConfig(**CONFIGS["mid"])
    store = pkg.init_params(cfg, 32)
    res = pkg.run_single(cfg, store, seed=32, precision=precision)
    want = _oracle_step("mid")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, want, m_in, z_in, bar=tol)
    k, v = _worst(errs)
    assert v <= tol, f"{precision}: worst {k} rel-L2 {v:.3e}"


def test_step_wide_bf16_matches_oracle(pkg):
    """AF2 channel widths: the fused LayerNorm paths are the ones running."""
    cfg = pkg.EvoConfig(**CONFIGS["wide"])
    store = pkg.init_params(cfg, 32)
    res = pkg.run_single(cfg, store, seed=32, precision="bf16")
    want = _oracle_step("wide")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, want, m_in, z_in, bar=BF16_TOL)
    k, v = _worst(errs)
    assert v <= BF16_TOL, f"worst {k} rel-L2 {v:.3e}"


def test_step_af2_bf16_matches_oracle(pkg):
    """The headline configuration itself (BASELINE.json configs[1]): one block
    at s=128, r=256, c_m=256, c_z=128 on the bf16 path vs the pinned oracle
    (numpy, ~20 s on the host)."""
    cfg = pkg.EvoConfig(**CONFIGS["af2"])
    store = pkg.init_params(cfg, 32)
    res = pkg.run_single(cfg, store, seed=32, precision="bf16")
    want = _oracle_step("af2")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, want, m_in, z_in, bar=BF16_TOL)
    k, v = _worst(errs)
    assert v <= BF16_TOL, f"worst {k} rel-L2 {v:.3e}"


def test_step_af2_fp32_matches_oracle(pkg):
    """C2 on the fp32 parity path (SIMT FFMA kernels) at the 1e-5 bar; the
    output deltas get the fp32 storage floor rule (helpers.quant_floor)."""
    cfg = pkg.EvoConfig(**CONFIGS["af2"])
    store = pkg.init_params(cfg, 32)
    res = pkg.run_single(cfg, store, seed=32, precision="fp32")
    want = _oracle_step("af2")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, want, m_in, z_in, bar=FP32_TOL)
    k, v = _worst(errs)
    assert v <= FP32_TOL, f"worst {k} rel-L2 {v:.3e}"


def test_step_crop384_bf16_matches_oracle(pkg):
    """C5 r = 384 (s = 128, AF2 widths): the row and triangle attentions
    attend over 384 keys (long-key path), bf16 vs the float64 oracle."""
    from paper_2211_00235_b200 import _native
    cfg = pkg.EvoConfig(**{**CONFIGS["af2"], "r": 384})
    store = pkg.init_params(cfg, 32)
    b0 = _native.backend_counts()
    res = pkg.run_single(cfg, store, seed=32, precision="bf16")
    b1 = _native.backend_counts()
    assert b1["gemm_simt"] == b0["gemm_simt"] and b1["attn_simt"] == b0["attn_simt"]
    want = _oracle_step("af2", r=384)
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, want, m_in, z_in, bar=BF16_TOL)
    k, v = _worst(errs)
    assert v <= BF16_TOL, f"worst {k} rel-L2 {v:.3e}"


@pytest.mark.parametrize("tag", ["toy", "c1"])
@pytest.mark.parametrize("variant", ["af2", "multimer"])
def test_variant_step_fp32_matches_reference_golden(pkg, tag, variant):
    """The af2 and multimer wirings (src/evoformer.py:448-455) on the native
    path vs the reference's own step."""
    cfg = pkg.EvoConfig(**CONFIGS[tag], variant=variant)
    store = pkg.init_params(cfg, 32)
    res = pkg.run_single(cfg, store, seed=32, precision="fp32")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    gold = load_golden(f"{tag}_{variant}")
    want = golden_as_want(gold)
    errs = normalise_by_reference_f32(step_errors(res, want, m_in, z_in, bar=FP32_TOL), want,
                                      FP32_TOL)
    k, v = _worst(errs)
    assert v <= FP32_TOL, f"{tag}/{variant}: worst {k} rel-L2 {v:.3e}"
    assert abs(res.loss - float(gold["loss"])) <= 1e-5 * abs(float(gold["loss"]))


@pytest.mark.parametrize("variant", ["af2", "multimer"])
def test_variant_step_bf16(pkg, variant):
    """bf16 wirings: c1 vs the reference golden, mid vs the oracle."""
    cfg = pkg.EvoConfig(**CONFIGS["c1"], variant=variant)
    res = pkg.run_single(cfg, pkg.init_params(cfg, 32), seed=32, precision="bf16")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, golden_as_want(load_golden(f"c1_{variant}")), m_in, z_in,
                       bar=BF16_TOL)
    k, v = _worst(errs)
    assert v <= BF16_TOL, f"c1/{variant}: worst {k} rel-L2 {v:.3e}"
    cfg = pkg.EvoConfig(**CONFIGS["mid"], variant=variant)
    res = pkg.run_single(cfg, pkg.init_params(cfg, 32), seed=32, precision="bf16")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, _oracle_step("mid", variant=variant), m_in, z_in, bar=BF16_TOL)
    k, v = _worst(errs)
    assert v <= BF16_TOL, f"mid/{variant}: worst {k} rel-L2 {v:.3e}"


def test_bp_rejects_serial_wirings(pkg):
    from paper_2211_00235_b200.schedules import ParallelLayout
    for variant in ("af2", "multimer"):
        cfg = pkg.EvoConfig(**CONFIGS["toy"], variant=variant)
        with pytest.raises(pkg.ConfigError):
            ParallelLayout(bp=2).validate_model(cfg)


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
def test_tracks_autograd_match_oracle(pkg, precision, tol):
    """msa_track / pair_track (src/evoformer.py:427-443) as native autograd
    functions: outputs and the VJP of a random cotangent vs the oracle."""
    import numpy as np
    from oracle import evoformer_np as O
    tag = "toy" if precision == "fp32" else "mid"
    pkg.set_precision(precision)
    try:
        cfg = pkg.EvoConfig(**CONFIGS[tag])
        store = pkg.init_params(cfg, 32)
        d = O.Dims(**CONFIGS[tag])
        Pn = O.init_params(d, 32)
        rng = np.random.default_rng(7)
        m0 = rng.standard_normal((cfg.s, cfg.r, cfg.c_m)).astype(np.float32)
        z0 = rng.standard_normal((cfg.r, cfg.r, cfg.c_z)).astype(np.float32)
        Rm = rng.standard_normal(m0.shape)
        Rz = rng.standard_normal(z0.shape)
        # oracle
        cm, cp = {}, {}
        mo = O._msa_track_fwd(Pn, 0, m0.astype(np.float64), z0.astype(np.float64), d, cm)
        zo = O._pair_track_fwd(Pn, 0, z0.astype(np.float64), d, cp)
        G = O.Grads()
        dm_w, dz_row = O._msa_track_vjp(Rm, cm, Pn, 0, d, G)
        dz_w = O._pair_track_vjp(Rz, cp, Pn, 0, d, G) + dz_row
        # native
        P = {n: t.clone().requires_grad_(True) for n, t in store.items()}
        m = torch.tensor(m0, device="cuda", requires_grad=True)
        z = torch.tensor(z0, device="cuda", requires_grad=True)
        mt = pkg.msa_track(P, 0, m, z, cfg)
        zt = pkg.pair_track(P, 0, z, cfg)
        ((mt * torch.tensor(Rm, device="cuda", dtype=torch.float32)).sum()
         + (zt * torch.tensor(Rz, device="cuda", dtype=torch.float32)).sum()).backward()
        # outputs (the deltas only for bf16: fp32 storage of m + delta floors
        # the delta's rel-L2 near 1e-5 at these dims, helpers.quant_floor)
        if precision == "fp32":
            assert rel_l2(mt, mo) <= tol and rel_l2(zt, zo) <= tol
        else:
            assert rel_l2(mt - m, mo - m0) <= tol
            assert rel_l2(zt - z, zo - z0) <= tol
        assert rel_l2(m.grad, dm_w) <= tol
        assert rel_l2(z.grad, dz_w) <= tol
        for n, g in G.items():
            if n.endswith("lnz_b") or np.linalg.norm(g) < 1e-15:
                continue
            assert rel_l2(P[n].grad, g) <= tol, n
    finally:
        pkg.set_precision("fp32")


def test_step_c1_bf16_matches_reference(pkg):
    cfg = pkg.EvoConfig(**CONFIGS["c1"])
    store = pkg.init_params(cfg, 32)
    res = pkg.run_single(cfg, store, seed=32, precision="bf16")
    m_in, z_in = pkg.make_batch(cfg, 32, 1)[0]
    errs = step_errors(res, golden_as_want(load_golden("c1")), m_in, z_in, bar=BF16_TOL)
    k, v = _worst(errs)
    assert v <= BF16_TOL, f"worst {k} rel-L2 {v:.3e}"


def test_step_is_deterministic(pkg):
    cfg = pkg.EvoConfig(**CONFIGS["mid"])
    store = pkg.init_params(cfg, 32)
    a = pkg.run_single(cfg, store, seed=32, precision="bf16")
    b = pkg.run_single(cfg, store, seed=32, precision="bf16")
    rep = pkg.compare_runs(a, b, rtol=0.0)
    assert rep.bitwise, str(rep)


SUBOP_GOLD = None


def _subop_gold():
    global SUBOP_GOLD
    if SUBOP_GOLD is None:
        import os
        from helpers import GOLD
        SUBOP_GOLD = np.load(os.path.join(GOLD, "subops_toy.npz"))
    return SUBOP_GOLD


@pytest.mark.parametrize("subop", ["row_attn", "col_attn", "msa_transition", "opm",
                                   "tri_mult_out", "tri_mult_in", "tri_attn_start",
                                   "tri_attn_end", "pair_transition"])
def test_subop_api_autograd_matches_reference(pkg, subop):
    """The reference-signature sub-op functions, differentiated by torch
    autograd through the native backward, against the reference tape."""
    pkg.set_precision("fp32")
    cfg = pkg.EvoConfig(**CONFIGS["toy"])
    store = pkg.init_params(cfg, 32)
    gold = _subop_gold()
    P = {n: t.clone().requires_grad_(True) for n, t in store.items()}
    m = torch.tensor(gold["m"], dtype=torch.float32, device="cuda", requires_grad=True)
    z = torch.tensor(gold["z"], dtype=torch.float32, device="cuda", requires_grad=True)
    px = f"blk0.{subop}"
    fn = {
        "row_attn": lambda: pkg.row_attn(P, px, m, z, cfg),
        "col_attn": lambda: pkg.col_attn(P, px, m, cfg),
        "msa_transition": lambda: pkg.msa_transition(P, px, m, cfg),
        "opm": lambda: pkg.opm(P, px, m, cfg),
        "tri_mult_out": lambda: pkg.tri_mult(P, px, z, cfg, incoming=False),
        "tri_mult_in": lambda: pkg.tri_mult(P, px, z, cfg, incoming=True),
        "tri_attn_start": lambda: pkg.tri_attn(P, px, z, cfg, ending=False),
        "tri_attn_end": lambda: pkg.tri_attn(P, px, z, cfg, ending=True),
        "pair_transition": lambda: pkg.pair_transition(P, px, z, cfg),
    }[subop]
    delta = fn()
    assert rel_l2(delta, gold[f"{subop}:delta"]) <= FP32_TOL
    R = torch.tensor(gold[f"{subop}:R"], dtype=torch.float32, device="cuda")
    (delta * R).sum().backward()
    if np.abs(gold[f"{subop}:dm"]).max() > 0:
        assert rel_l2(m.grad, gold[f"{subop}:dm"]) <= FP32_TOL
    if np.abs(gold[f"{subop}:dz"]).max() > 0:
        assert rel_l2(z.grad, gold[f"{subop}:dz"]) <= FP32_TOL
    pre = f"{subop}:grad:"
    for key in gold.files:
        if key.startswith(pre):
            name = f"{px}.{key[len(pre):]}"
            g = gold[key]
            if np.linalg.norm(g) < 1e-15:
                continue
            assert rel_l2(P[name].grad, g) <= FP32_TOL, name


def test_block_autograd_matches_run_single(pkg):
    """evoformer_stack through autograd == the explicit run_single step."""
    pkg.set_precision("fp32")
    cfg = pkg.EvoConfig(**CONFIGS["toy"])
    store = pkg.init_params(cfg, 32)
    ref = pkg.run_single(cfg, store, seed=32, precision="fp32")
    P = {n: t.clone().requires_grad_(True) for n, t in store.items()}
    m, z = pkg.make_batch(cfg, 32, 1)[0]
    m.requires_grad_(True)
    z.requires_grad_(True)
    mo, zo = pkg.evoformer_stack(P, m, z, cfg)
    loss = (mo * mo).mean() + (zo * zo).mean()
    loss.backward()
    assert rel_l2(mo, ref.m_out) <= 1e-6
    assert rel_l2(zo, ref.z_out) <= 1e-6
    assert rel_l2(m.grad, ref.dm) <= 1e-5
    assert rel_l2(z.grad, ref.dz) <= 1e-5
    for n in ref.grads:
        if n.endswith("lnz_b"):
            continue
        assert rel_l2(P[n].grad, ref.grads[n]) <= 1e-5, n
