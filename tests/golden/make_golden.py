"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
itself (branchpar, /root/reference/pkg/src) in float64.

Run here (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed, small):
  step_<cfg>.npz   run_single(cfg, init_params(cfg, 32), seed=32): m_out,
                   z_out, loss, dm, dz and every parameter gradient
                   (keys "grad:<name>"), plus the tape madds of one block
                   forward ("madds_block") and the reference's own
                   float32-vs-float64 rel-L2 per field ("f32err:<field>").  run_bp is asserted bitwise
                   equal to run_single before saving.
  step_<cfg>_<variant>.npz   the same for the af2 and multimer wirings
                   (toy and c1 dims; no BP check: BP needs the parallel wiring).
  subops_toy.npz   every sub-op of block 0 at the toy dims: forward delta
                   and the VJP of a seeded random cotangent R with respect
                   to m, z and the sub-op's parameters
                   ("<subop>:delta", "<subop>:dm", "<subop>:dz",
                   "<subop>:grad:<suffix>").
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

CONFIGS = {
    # tests/test_schedules.py:15-19 toy dims
    "toy": dict(s=8, r=16, c_m=8, c_z=8, h=2, c_opm=4, t_factor=4, n_blocks=2),
    # tests/test_schedules.py:72-73 odd dims, three blocks
    "odd": dict(s=5, r=6, c_m=4, c_z=6, h=2, c_opm=3, t_factor=4, n_blocks=3),
    # BASELINE.json configs[0] (C1 tiny), h/c_opm/t from SURVEY.md 8(d)
    "c1": dict(s=16, r=32, c_m=32, c_z=16, h=4, c_opm=8, t_factor=4, n_blocks=2),
}


def step_golden(tag, kw, variant="parallel"):
    from branchpar import tensor as T
    from branchpar import evoformer as E
    from branchpar.schedules import compare_runs, run_bp, run_single

    cfg = E.EvoConfig(**kw, variant=variant)
    store = E.init_params(cfg, 32)
    a = run_single(cfg, store, seed=32)
    if variant == "parallel":
        b = run_bp(cfg, store, seed=32)
        assert compare_runs(a, b, rtol=0.0).bitwise, tag
    g = T.Graph()
    P = store.bind(g)
    m, z = E.seeded_inputs(cfg, 32)
    E.evoformer_block(P, 0, g.leaf(m), g.leaf(z), cfg)
    out = dict(m_out=a.m_out, z_out=a.z_out, loss=np.float64(a.loss),
               dm=a.dm, dz=a.dz, madds_block=np.int64(g.madds))
    for name, arr in a.grads.items():
        out[f"grad:{name}"] = arr
    # the reference's OWN float32 deviation from its float64 run, per
    # field: the floor any fp32 implementation is measured against
    f = run_single(cfg, E.init_params(cfg, 32, dtype=np.float32), seed=32)
    m_in, z_in = E.seeded_inputs(cfg, 32)

    def rl(x, y):
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        return np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)

    m32 = m_in.astype(np.float32).astype(np.float64)
    z32 = z_in.astype(np.float32).astype(np.float64)
    out["f32err:m_delta"] = rl(f.m_out.astype(np.float64) - m32, a.m_out - m_in)
    out["f32err:z_delta"] = rl(f.z_out.astype(np.float64) - z32, a.z_out - z_in)
    out["f32err:dm"] = rl(f.dm, a.dm)
    out["f32err:dz"] = rl(f.dz, a.dz)
    for name in a.grads:
        out[f"f32err:grad:{name}"] = rl(f.grads[name], a.grads[name])
    name = f"step_{tag}.npz" if variant == "parallel" else f"step_{tag}_{variant}.npz"
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, "saved", len(out), "arrays; madds/block", g.madds)


def main():
    sys.path.insert(0, REF)
    from branchpar import tensor as T
    from branchpar import evoformer as E

    only = sys.argv[1:]
    for tag, kw in CONFIGS.items():
        if not only or tag in only:
            step_golden(tag, kw)
    # the af2 and multimer wirings (src/evoformer.py:448-455), SURVEY.md 8(f)
    for tag in ("toy", "c1"):
        for variant in ("af2", "multimer"):
            if not only or f"{tag}_{variant}" in only:
                step_golden(tag, CONFIGS[tag], variant)
    if only and "subops" not in only:
        return

    cfg = E.EvoConfig(**CONFIGS["toy"])
    store = E.init_params(cfg, 32)
    m, z = E.seeded_inputs(cfg, 33)
    rng = np.random.default_rng(34)
    out = {}
    for name in E.SUBOPS:
        g = T.Graph()
        P = store.bind(g)
        mt, zt = g.leaf(m), g.leaf(z)
        px = f"blk0.{name}"
        if name == "row_attn":
            delta = E.row_attn(P, px, mt, zt, cfg)
        elif name == "col_attn":
            delta = E.col_attn(P, px, mt, cfg)
        elif name == "msa_transition":
            delta = E.msa_transition(P, px, mt, cfg)
        elif name == "opm":
            delta = E.opm(P, px, mt, cfg)
        elif name == "pair_transition":
            delta = E.pair_transition(P, px, zt, cfg)
        elif name.startswith("tri_mult"):
            delta = E.tri_mult(P, px, zt, cfg, name.endswith("_in"))
        else:
            delta = E.tri_attn(P, px, zt, cfg, name.endswith("_end"))
        R = rng.standard_normal(delta.shape)
        loss = T.reduce_sum(T.mul(delta, g.leaf(R)))
        g.backward(loss)
        out[f"{name}:R"] = R
        out[f"{name}:delta"] = delta.data
        out[f"{name}:dm"] = g.grad(mt)
        out[f"{name}:dz"] = g.grad(zt)
        for pname in store.names():
            if pname.startswith(px + "."):
                out[f"{name}:grad:{pname[len(px) + 1:]}"] = g.grad(P[pname])
    out["m"] = m
    out["z"] = z
    np.savez_compressed(os.path.join(HERE, "subops_toy.npz"), **out)
    print("subops saved", len(out), "arrays")


if __name__ == "__main__":
    main()
