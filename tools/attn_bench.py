"""Time the fused attention fwd / bwd in isolation (CUDA events), for ncu.

    python tools/attn_bench.py --nb 256 --L 256 --H 8 --D 32 --bias plain
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00235_b200 import kernels as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nb", type=int, default=256)
    ap.add_argument("--L", type=int, default=256)
    ap.add_argument("--H", type=int, default=8)
    ap.add_argument("--D", type=int, default=32)
    ap.add_argument("--bias", default="plain", choices=["plain", "transposed", "none"])
    ap.add_argument("--seq-major", action="store_true")
    ap.add_argument("--what", default="both", choices=["fwd", "bwd", "both"])
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    nb, L, H, D = a.nb, a.L, a.H, a.D
    hc = H * D
    rows = nb * L
    sb, sl = (1, nb) if a.seq_major else (L, 1)
    proj = torch.randn(rows, 4 * hc, device="cuda").to(torch.bfloat16)
    o = torch.empty(rows, hc, device="cuda", dtype=torch.bfloat16)
    gm = torch.empty_like(o)
    lse = torch.empty(nb, H, L, device="cuda")
    bias = None
    bq = bk = 0
    if a.bias != "none":
        bias = torch.randn(H, L * L, device="cuda") * 0.1
        bq, bk = (L, 1) if a.bias == "plain" else (1, L)
    geo = dict(proj=proj, hc=hc, nb=nb, H=H, L=L, D=D, scale=D ** -0.5, sb=sb * 4 * hc,
               sl=sl * 4 * hc, o=o, gm=gm, o_sb=sb * hc, o_sl=sl * hc, lse=lse, bias=bias,
               bh=L * L, bq=bq, bk=bk)
    dgm = torch.randn(rows, hc, device="cuda").to(torch.bfloat16)
    dproj = torch.empty_like(proj)
    dbias = torch.empty(H, L * L, device="cuda") if bias is not None else None

    def fwd():
        K.attention(**geo)

    def bwd():
        K.attention(**geo, dgm=dgm, dproj=dproj, dbias=dbias)

    fwd()
    fl = 4.0 * nb * H * L * L * D
    for name, fn, mult in (("fwd", fwd, 1), ("bwd", bwd, 2)):
        if a.what not in (name, "both"):
            continue
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / a.iters * 1e3
        print(f"{name} nb={nb} L={L} H={H} D={D} bias={a.bias}: {us:.1f} us "
              f"{mult * fl / us / 1e6:.1f} TF/s")


if __name__ == "__main__":
    main()
