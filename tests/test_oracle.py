"""Pin the numpy oracle (oracle/evoformer_np.py) against golden vectors
produced by the reference itself (tests/golden/make_golden.py).

CPU only.  Tolerances are f64 round-off (the oracle reorders some sums
relative to the reference tape, so bitwise equality is not expected).
"""

import os

import numpy as np
import pytest

from oracle import evoformer_np as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")

CONFIGS = {
    "toy": dict(s=8, r=16, c_m=8, c_z=8, h=2, c_opm=4, t_factor=4, n_blocks=2),
    "odd": dict(s=5, r=6, c_m=4, c_z=6, h=2, c_opm=3, t_factor=4, n_blocks=3),
    "c1": dict(s=16, r=32, c_m=32, c_z=16, h=4, c_opm=8, t_factor=4, n_blocks=2),
}


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    v = np.linalg.norm(a - b) / (den if den > 0 else 1.0)
    return v if np.isfinite(v) else np.inf


def load(name):
    return np.load(os.path.join(GOLD, name))


VARIANT_TAGS = ["toy_af2", "toy_multimer", "c1_af2", "c1_multimer"]


@pytest.mark.parametrize("tag", list(CONFIGS) + VARIANT_TAGS)
def test_step_matches_reference_golden(tag):
    base, _, variant = tag.partition("_")
    d = O.Dims(**CONFIGS[base], variant=variant or "parallel")
    P = O.init_params(d, 32)
    res = O.run_single(d, P, seed=32)
    gold = load(f"step_{tag}.npz")
    for key in ("m_out", "z_out", "dm", "dz"):
        assert rel(res[key], gold[key]) < 1e-12, key
    assert abs(res["loss"] - float(gold["loss"])) < 1e-12 * abs(float(gold["loss"]))
    names = [k[5:] for k in gold.files if k.startswith("grad:")]
    assert sorted(names) == sorted(P)
    for n in names:
        g = gold[f"grad:{n}"]
        if np.linalg.norm(g) < 1e-15:      # analytic zeros (row_attn.lnz_b)
            assert np.abs(res["grads"][n]).max() < 1e-12, n
            continue
        assert rel(res["grads"][n], g) < 1e-10, n


@pytest.mark.parametrize("tag", list(CONFIGS))
def test_block_flops_equal_reference_madds(tag):
    d = O.Dims(**CONFIGS[tag])
    assert O.block_flops(d) == int(load(f"step_{tag}.npz")["madds_block"])


def test_af2_init_flops_match_survey():
    d = O.Dims(s=128, r=256, c_m=256, c_z=128, h=8, c_opm=32, t_factor=4)
    assert 3 * O.block_flops(d) == 696_992_661_504


@pytest.mark.parametrize("subop", O.SUBOPS)
def test_subop_vjp_matches_reference_golden(subop):
    d = O.Dims(**CONFIGS["toy"])
    P = O.init_params(d, 32)
    gold = load("subops_toy.npz")
    m, z = gold["m"], gold["z"]
    px = f"blk0.{subop}"
    delta, cache = O.subop_fwd(subop, P, px, m, z, d)
    assert rel(delta, gold[f"{subop}:delta"]) < 1e-13
    G = O.Grads()
    dm, dz = O.subop_vjp(subop, gold[f"{subop}:R"], cache, P, px, d, G)
    gdm, gdz = gold[f"{subop}:dm"], gold[f"{subop}:dz"]
    if np.abs(gdm).max() > 0:
        assert rel(dm, gdm) < 1e-12
    else:
        assert dm is None
    if np.abs(gdz).max() > 0:
        assert rel(dz, gdz) < 1e-12
    else:
        assert dz is None
    for key in gold.files:
        pre = f"{subop}:grad:"
        if key.startswith(pre):
            g = gold[key]
            name = f"{px}.{key[len(pre):]}"
            if np.linalg.norm(g) < 1e-15:
                assert np.abs(G.get(name, 0.0)).max() < 1e-12
            else:
                assert rel(G[name], g) < 1e-12, name


def test_init_params_match_reference_rng_order():
    # weights are the only RNG consumers; first draw is blk0.row_attn.q_w
    d = O.Dims(**CONFIGS["toy"])
    P = O.init_params(d, 32)
    rng = np.random.default_rng(32)
    q = rng.uniform(-0.02, 0.02, size=(8, 8))
    assert np.array_equal(P["blk0.row_attn.q_w"], q)
    assert len(P) == 93 * d.n_blocks


def test_composed_step_reduces_to_train_step_and_matches_finite_difference():
    """The C3 composition (extra stack -> main stack) is two stacks on one
    tape: with no extra blocks it is the plain step, and its dm_e agrees with
    a central finite difference of the loss along a random direction."""
    dm_ = O.Dims(s=4, r=6, c_m=4, c_z=4, h=2, c_opm=2, n_blocks=1)
    de = O.Dims(s=6, r=6, c_m=2, c_z=4, h=2, c_opm=2, n_blocks=1)
    Pm, Pe = O.init_params(dm_, 32), O.init_params(de, 33)
    rng = np.random.default_rng(5)
    m_e = rng.standard_normal((de.s, de.r, de.c_m))
    m = rng.standard_normal((dm_.s, dm_.r, dm_.c_m))
    z = rng.standard_normal((dm_.r, dm_.r, dm_.c_z))
    d0 = O.Dims(s=6, r=6, c_m=2, c_z=4, h=2, c_opm=2, n_blocks=0)
    plain = O.train_step(Pm, m, z, dm_)
    comp0 = O.composed_step({}, d0, Pm, dm_, m_e, m, z)
    for key in ("m_out", "z_out", "dm", "dz"):
        assert np.array_equal(plain[key], comp0[key])
    out = O.composed_step(Pe, de, Pm, dm_, m_e, m, z)
    v = rng.standard_normal(m_e.shape)
    eps = 1e-6
    lp = O.composed_step(Pe, de, Pm, dm_, m_e + eps * v, m, z)["loss"]
    lm = O.composed_step(Pe, de, Pm, dm_, m_e - eps * v, m, z)["loss"]
    fd = (lp - lm) / (2 * eps)
    an = float(np.sum(out["dm_e"] * v))
    assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (fd, an)
