"""Shared test helpers: rel-L2 comparator and golden / oracle access."""

import os

import numpy as np

GOLD = os.path.join(os.path.dirname(__file__), "golden")

CONFIGS = {
    "toy": dict(s=8, r=16, c_m=8, c_z=8, h=2, c_opm=4, t_factor=4, n_blocks=2),
    "odd": dict(s=5, r=6, c_m=4, c_z=6, h=2, c_opm=3, t_factor=4, n_blocks=3),
    "c1": dict(s=16, r=32, c_m=32, c_z=16, h=4, c_opm=8, t_factor=4, n_blocks=2),
    # tensor-core-eligible dims (multiples of 16) that the oracle runs in ~1 s
    "mid": dict(s=32, r=64, c_m=64, c_z=32, h=4, c_opm=16, t_factor=4, n_blocks=1),
    # AF2 channel widths at a small sequence shape: exercises the c_z = 128 /
    # c_m = 256 fused paths (LayerNorm hand-off, fused pair-bias projection)
    "wide": dict(s=64, r=64, c_m=256, c_z=128, h=8, c_opm=32, t_factor=4, n_blocks=1),
    # BASELINE.json configs[1]: AF2 initial-training block
    "af2": dict(s=128, r=256, c_m=256, c_z=128, h=8, c_opm=32, t_factor=4, n_blocks=1),
}

# analytic zeros: softmax shift invariance makes the row-attention pair-bias
# LN shift gradient exactly zero; compare absolutely.
ANALYTIC_ZERO = ("row_attn.lnz_b",)


def to_np(x):
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().double().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(x, dtype=np.float64)


def rel_l2(a, b):
    a, b = to_np(a), to_np(b)
    den = np.linalg.norm(b)
    v = float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))
    return v if np.isfinite(v) else float("inf")    # NaN must never pass a max() / <=


def load_golden(tag):
    return np.load(os.path.join(GOLD, f"step_{tag}.npz"))


def quant_floor(out64, x_in):
    """rel-L2 error that merely storing the exact output in fp32 puts on
    the delta (out - in).  The reference's own float32 run sits at this
    floor (toy: 2.6e-5, odd: 5.6e-5 measured), so deltas are held to
    max(bar, 4 * floor); the activations themselves to the bar."""
    out64 = to_np(out64)
    q = out64.astype(np.float32).astype(np.float64)
    return rel_l2(q - x_in, out64 - x_in)


def step_errors(res, want, m_in, z_in, bar=None):
    """Per-field rel-L2 of a RunResult against a reference dict
    (m_out, z_out, dm, dz, grads{}).  Outputs are compared both directly
    and as deltas; with `bar`, delta errors are normalised by
    max(bar, 4*quant_floor)/bar so one threshold applies to all fields."""
    errs = {}
    m_in, z_in = to_np(m_in), to_np(z_in)
    errs["m_out"] = rel_l2(res.m_out, want["m_out"])
    errs["z_out"] = rel_l2(res.z_out, want["z_out"])
    errs["m_delta"] = rel_l2(to_np(res.m_out) - m_in, to_np(want["m_out"]) - m_in)
    errs["z_delta"] = rel_l2(to_np(res.z_out) - z_in, to_np(want["z_out"]) - z_in)
    if bar is not None:
        for key, out, x in (("m_delta", want["m_out"], m_in), ("z_delta", want["z_out"], z_in)):
            allow = max(bar, 4.0 * quant_floor(out, x))
            errs[key] *= bar / allow
    errs["dm"] = rel_l2(res.dm, want["dm"])
    errs["dz"] = rel_l2(res.dz, want["dz"])
    for name, g in want["grads"].items():
        if name.endswith(ANALYTIC_ZERO):
            scale = max(1e-30, np.abs(to_np(want["grads"][name.replace("lnz_b", "lnz_g")])).max())
            errs["grad:" + name] = float(np.abs(to_np(res.grads[name])).max() / scale)
            continue
        errs["grad:" + name] = rel_l2(res.grads[name], g)
    return errs


def golden_as_want(gold):
    return dict(m_out=gold["m_out"], z_out=gold["z_out"], dm=gold["dm"], dz=gold["dz"],
                grads={k[5:]: gold[k] for k in gold.files if k.startswith("grad:")},
                f32err={k[7:]: float(gold[k]) for k in gold.files if k.startswith("f32err:")})


def normalise_by_reference_f32(errs, want, bar):
    """Hold each field to max(bar, 2 x the reference's own float32 error on
    that field): errs[k] *= bar / allow, so one threshold `bar` applies."""
    ref = want.get("f32err", {})
    for k in list(errs):
        e = ref.get(k)
        if e is not None:
            errs[k] *= bar / max(bar, 2.0 * e)
    return errs
