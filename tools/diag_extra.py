"""Diagnose the C3 extra-stack bf16 gradient errors against the oracle:
per-tensor rel-L2 of the extra stack's parameter gradients, with the
long-key attention keeping P (default) and recomputing it (KEEP_P off).

    python tools/diag_extra.py
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2211_00235_b200 as pkg  # noqa: E402
from paper_2211_00235_b200 import kernels as K, schedules as S  # noqa: E402
from oracle import evoformer_np as O  # noqa: E402
from helpers import CONFIGS, rel_l2, to_np  # noqa: E402

EXTRA = dict(s=64, r=64, c_m=32, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=2)


def run(precision, keep):
    K.KEEP_P_MAX_BYTES = (8 << 30) if keep else 0
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
    out = S.composed_step(ste, stm, *t)
    torch.cuda.synchronize()
    return ste.grad_dict(), stm.grad_dict(), out, t


def main():
    de, dmn = O.Dims(**EXTRA), O.Dims(**CONFIGS["mid"])
    ge, gm, out, t = run("bf16", True)
    want = O.composed_step(O.init_params(de, 33), de, O.init_params(dmn, 32), dmn,
                           *[to_np(x) for x in t])
    for keep in (True, False):
        ge, gm, out, _ = run("bf16", keep)
        errs = {n: rel_l2(ge[n], g) for n, g in want["grads_e"].items()
                if not n.endswith("lnz_b")}
        errs_m = {n: rel_l2(gm[n], g) for n, g in want["grads_m"].items()
                  if not n.endswith("lnz_b")}
        print(f"keep_p={keep}: dm_e {rel_l2(out[3], want['dm_e']):.3e} "
              f"dz {rel_l2(out[5], want['dz']):.3e}")
        for n, e in sorted(errs.items(), key=lambda kv: -kv[1])[:12]:
            print(f"  extra {n:40s} {e:.3e}  |g|={np.linalg.norm(want['grads_e'][n]):.3e}")
        for n, e in sorted(errs_m.items(), key=lambda kv: -kv[1])[:4]:
            print(f"  main  {n:40s} {e:.3e}")


if __name__ == "__main__":
    main()
