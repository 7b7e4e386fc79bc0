"""Time the LayerNorm backward variants at the AF2 pair shape (graph-replayed),
for ncu targeting:  python tools/ln_bench.py [--rows 65536] [--what proj]"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00235_b200 import kernels as K  # noqa: E402
from tools.ew_bench import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=65536)
    ap.add_argument("--what", default="all")
    ap.add_argument("--unused", default=None)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    rows, cols, h = a.rows, 128, 8
    dev, bf = "cuda", torch.bfloat16
    x = torch.randn(rows, cols, device=dev)
    dy = torch.randn(rows, cols, device=dev)
    dres = torch.randn(rows, cols, device=dev)
    g = torch.randn(cols, device=dev)
    b = torch.randn(cols, device=dev)
    y = torch.empty(rows, cols, device=dev)
    mu = torch.empty(rows, device=dev)
    rs = torch.empty(rows, device=dev)
    K.layernorm(x, rows, cols, g, b, y, mu, rs, 1e-5)
    dx = torch.empty(rows, cols, device=dev)
    dxa = torch.empty(rows, cols, device=dev, dtype=bf)
    dg, db, cs = (torch.empty(cols, device=dev) for _ in range(3))
    dbias = torch.randn(h, rows, device=dev)
    Wb = (torch.randn(cols, h, device=dev) * 0.1).to(bf)
    dW = torch.empty(cols, h, device=dev)
    MB = 1e6
    cases = {
        "vec": (lambda: K.layernorm_bwd(dy, x, rows, cols, mu, rs, g, dx, dg, db, dres=dres),
                4 * rows * cols * 4),
        "ex": (lambda: K.layernorm_bwd_ex(dy, x, rows, cols, mu, rs, g, dx, dg, db, dres=dres,
                                          dx_act=dxa, dx_colsum=cs),
               4 * rows * cols * 4 + rows * cols * 2),
        "proj_tri": (lambda: K.layernorm_bwd_proj(dy, x, rows, mu, rs, g, b, dbias, rows, Wb, h,
                                                  dx, dg, db, dW, dres=dres, dx_act=dxa,
                                                  dx_colsum=cs),
                     4 * rows * cols * 4 + rows * cols * 2 + h * rows * 4),
        "proj_row": (lambda: K.layernorm_bwd_proj(None, x, rows, mu, rs, g, b, dbias, rows, Wb, h,
                                                  dx, dg, db, dW, dres=dres),
                     3 * rows * cols * 4 + h * rows * 4),
    }
    yb = torch.empty(rows, cols, device=dev, dtype=bf)
    pb = torch.empty(h, rows, device=dev)
    from paper_2211_00235_b200.kernels import Mat
    cases["fwd_bf16"] = (lambda: K.layernorm(x, rows, cols, g, b, yb, mu, rs, 1e-5),
                         rows * cols * 6 + rows * 8)
    cases["fwd_f32"] = (lambda: K.layernorm(x, rows, cols, g, b, y, mu, rs, 1e-5),
                        rows * cols * 8 + rows * 8)
    cases["fwd_rowdot"] = (lambda: K.gemm(Mat(yb, cols, 1), Mat(Wb, 1, h), Mat(pb, 1, rows), rows, h,
                                          cols),
                           rows * cols * 2 + h * rows * 4)
    for name, (fn, byt) in cases.items():
        if a.what != "all" and not name.startswith(a.what):
            continue
        us = timeit(fn, a.iters)
        print(f"{name:9s} rows={rows}: {us:7.1f} us  {byt / MB:6.1f} MB  {byt / us / 1e3:6.0f} GB/s")


if __name__ == "__main__":
    main()
