"""Our tcgen05 GEMM against cuBLAS (torch.matmul) on the step's largest GEMM
shapes (the same operand layouts the engine uses), CUDA-event timed."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_00235_b200 import kernels as K  # noqa: E402
from paper_2211_00235_b200.kernels import Mat  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n * 1e3


bf = torch.bfloat16
dev = "cuda"
rows = []
# weight gradients dW[M=c_in, N=c_out] = X^T dY over R rows (X [R, c_in], dY [R, c_out])
for R, cin, cout in ((65536, 128, 1024), (32768, 256, 1024), (65536, 128, 256), (32768, 1024, 256)):
    X = torch.randn(R, cin, device=dev).to(bf)
    dY = torch.randn(R, cout, device=dev).to(bf)
    W = torch.empty(cin, cout, device=dev)
    sk = K.pick_split(R, cin, cout)
    ours = timeit(lambda: K.gemm(Mat(X, 1, cin), Mat(dY, 1, cout), Mat(W, cout, 1), cin, cout, R,
                                 split_k=sk))
    cub = timeit(lambda: torch.matmul(X.t(), dY, out=None))
    rows.append((f"dW [{cin}x{cout}] over {R} rows (split {sk})", ours, cub, 2.0 * R * cin * cout))
# forward projections Y[R, N] = X[R, K] W[K, N], bf16 out
for R, kk, n in ((65536, 128, 1024), (32768, 256, 1024), (32768, 1024, 256)):
    X = torch.randn(R, kk, device=dev).to(bf)
    Wt = torch.randn(n, kk, device=dev).to(bf)
    Y = torch.empty(R, n, device=dev, dtype=bf)
    ours = timeit(lambda: K.gemm(Mat(X, kk, 1), Mat(Wt, kk, 1), Mat(Y, n, 1), R, n, kk))
    cub = timeit(lambda: torch.matmul(X, Wt.t()))
    rows.append((f"Y [{R}x{n}] = X [{R}x{kk}] W (bf16 out)", ours, cub, 2.0 * R * kk * n))
for name, o, c, fl in rows:
    print(f"{name:48s} ours {o:7.1f} us ({fl / o / 1e6:6.0f} TF/s)   cuBLAS {c:7.1f} us "
          f"({fl / c / 1e6:6.0f} TF/s)")
