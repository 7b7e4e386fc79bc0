"""Time the bandwidth-bound kernels (LayerNorm fwd/bwd, colsum, relu bwd,
casts) at the block's shapes, with achieved GB/s."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00235_b200 import kernels as K  # noqa: E402


def timeit(fn, iters=20):
    """GPU time per call: `iters` calls captured in one CUDA graph, replayed
    (host launch overhead excluded)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    dev = "cuda"
    bf = torch.bfloat16
    for rows, cols in ((32768, 256), (65536, 128)):
        x = torch.randn(rows, cols, device=dev)
        g = torch.randn(cols, device=dev)
        b = torch.randn(cols, device=dev)
        y = torch.empty(rows, cols, device=dev, dtype=bf)
        mu = torch.empty(rows, device=dev)
        rs = torch.empty(rows, device=dev)
        us = timeit(lambda: K.layernorm(x, rows, cols, g, b, y, mu, rs, 1e-5))
        print(f"ln_fwd {rows}x{cols}: {us:.1f} us {rows * cols * 6 / us / 1e3:.0f} GB/s")
        dy = torch.randn(rows, cols, device=dev)
        dx = torch.empty(rows, cols, device=dev)
        dg = torch.empty(cols, device=dev)
        db = torch.empty(cols, device=dev)
        us = timeit(lambda: K.layernorm_bwd(dy, x, rows, cols, mu, rs, g, dx, dg, db, dres=dy))
        print(f"ln_bwd {rows}x{cols}: {us:.1f} us {rows * cols * 16 / us / 1e3:.0f} GB/s")
        us = timeit(lambda: K.colsum(dy, rows, cols, dg))
        print(f"colsum f32 {rows}x{cols}: {us:.1f} us {rows * cols * 4 / us / 1e3:.0f} GB/s")
        yb = dy.to(bf)
        us = timeit(lambda: K.colsum(yb, rows, cols, dg))
        print(f"colsum bf16 {rows}x{cols}: {us:.1f} us {rows * cols * 2 / us / 1e3:.0f} GB/s")
        us = timeit(lambda: K.copy2d(dy, rows, cols, yb, s_rs=cols, d_rs=cols))
        print(f"cast f32->bf16 {rows}x{cols}: {us:.1f} us {rows * cols * 6 / us / 1e3:.0f} GB/s")
    h = torch.randn(32768 * 1024, device=dev).to(bf)
    dh = torch.randn(32768 * 1024, device=dev).to(bf)
    us = timeit(lambda: K.relu_bwd(dh, h, dh, h.numel()))
    print(f"relu_bwd 32768x1024 bf16: {us:.1f} us {h.numel() * 6 / us / 1e3:.0f} GB/s")
    part = torch.randn(9, 8 * 65536, device=dev)
    out = torch.empty(8 * 65536, device=dev)
    us = timeit(lambda: K.reduce_lead(part, 9, 1, 8 * 65536, out, 0, 1))
    print(f"reduce_lead 9x524288: {us:.1f} us {part.numel() * 4 / us / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
