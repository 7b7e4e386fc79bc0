"""C3 composition: an extra-MSA stack (its own EvoConfig,
more sequences, narrower c_e, c_head = c_e / h) whose pair output feeds the
main stack, fwd+bwd on the native path vs the pinned oracle composition
(oracle.evoformer_np.composed_step).  Bars: rel-L2 <= 1e-5 fp32 and <= 2e-2
bf16 for the outputs, dm, dz, dm_e and every parameter gradient of both
stacks.  (The extra stack's MSA track is trained only through the outer
product mean, so its transition gradients are small, cancellation-heavy
column sums; with plain bf16 operands the ReLU mask flips on near-zero
pre-activations and those gradients sit at 5e-2 -- the same as the oracle
with bf16-rounded matmul operands.  The bf16 path therefore runs the
transitions' first projection as a 3-product bf16 GEMM, engine.transition_fwd.)
"""

import numpy as np
import pytest
import torch

from helpers import ANALYTIC_ZERO, CONFIGS, rel_l2, step_errors, to_np

pytestmark = pytest.mark.gpu

# main = "mid"; extra: 2x the sequences at half the MSA width, c_head = 8
EXTRA = dict(s=64, r=64, c_m=32, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=2)


def _grad_errs(got, want, prefix):
    errs = {}
    for name, g in want.items():
        if name.endswith(ANALYTIC_ZERO):
            continue
        errs[prefix + name] = rel_l2(got[name], g)
    return errs


@pytest.mark.parametrize("precision,tol,tol_extra",
                         [("fp32", 1e-5, 1e-5), ("bf16", 2e-2, 2e-2)])
def test_extra_stack_feeds_main_stack(precision, tol, tol_extra):
    import paper_2211_00235_b200 as pkg
    from paper_2211_00235_b200 import schedules as S
    from oracle import evoformer_np as O

    ce, cm = pkg.EvoConfig(**EXTRA), pkg.EvoConfig(**CONFIGS["mid"])
    se, sm = pkg.init_params(ce, 33), pkg.init_params(cm, 32)
    rng = np.random.default_rng(32)
    m_e = rng.standard_normal((ce.s, ce.r, ce.c_m))
    m = rng.standard_normal((cm.s, cm.r, cm.c_m))
    z = rng.standard_normal((cm.r, cm.r, cm.c_z))
    dev = torch.device("cuda")
    t = [torch.as_tensor(x.astype(np.float32), device=dev) for x in (m_e, m, z)]
    ste = S.StepState(ce, se, precision, dev)
    stm = S.StepState(cm, sm, precision, dev)
    m_out, z_out, loss, dm_e, dm, dz = S.composed_step(ste, stm, *t)
    torch.cuda.synchronize()

    de, dmn = O.Dims(**EXTRA), O.Dims(**CONFIGS["mid"])
    want = O.composed_step(O.init_params(de, 33), de, O.init_params(dmn, 32), dmn,
                           *[to_np(x) for x in t])

    class R:
        pass
    res = R()
    res.m_out, res.z_out, res.dm, res.dz, res.grads = m_out, z_out, dm, dz, stm.grad_dict()
    errs = step_errors(res, dict(want, grads=want["grads_m"]), t[1], t[2], bar=tol)
    errs["dm_e"] = rel_l2(dm_e, want["dm_e"])
    worst = sorted(errs.items(), key=lambda kv: -kv[1])[:8]
    assert worst[0][1] <= tol, f"{precision}: worst rel-L2 {worst}"
    ex = _grad_errs(ste.grad_dict(), want["grads_e"], "extra:")
    worst = sorted(ex.items(), key=lambda kv: -kv[1])[:8]
    assert worst[0][1] <= tol_extra, f"{precision}: worst extra-stack rel-L2 {worst}"
    assert abs(float(loss.item()) - want["loss"]) <= 10 * tol * abs(want["loss"])


def test_extra_stack_rejects_mismatched_pair_shape():
    import paper_2211_00235_b200 as pkg
    from paper_2211_00235_b200 import schedules as S

    ce = pkg.EvoConfig(**{**EXTRA, "c_z": 16})
    cm = pkg.EvoConfig(**CONFIGS["mid"])
    dev = torch.device("cuda")
    ste = S.StepState(ce, pkg.init_params(ce, 33), "fp32", dev)
    stm = S.StepState(cm, pkg.init_params(cm, 32), "fp32", dev)
    z = torch.zeros(cm.r, cm.r, cm.c_z, device=dev)
    with pytest.raises(pkg.ConfigError):
        S.composed_step(ste, stm, torch.zeros(ce.s, ce.r, ce.c_m, device=dev),
                        torch.zeros(cm.s, cm.r, cm.c_m, device=dev), z)
