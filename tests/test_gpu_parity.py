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
    k = max(errs, key=errs.get)
    return k, errs[k]


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


def _oracle_step(tag):
    from oracle import evoformer_np as O
    d = O.Dims(**CONFIGS[tag])
    P = O.init_params(d, 32)
    return O.run_single(d, P, seed=32)


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
