"""Time one evo_gemm shape in isolation (CUDA events), for ncu targeting.

    python tools/gemm_bench.py --M 65536 --N 1024 --K 128 --b-major mn --epi sigmoid
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2211_00235_b200 import _native as N, kernels as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=65536)
    ap.add_argument("--N", type=int, default=1024)
    ap.add_argument("--K", type=int, default=128)
    ap.add_argument("--a-major", default="k", choices=["k", "mn"])
    ap.add_argument("--b-major", default="mn", choices=["k", "mn"])
    ap.add_argument("--epi", default="none", choices=["none", "relu", "sigmoid", "bias"])
    ap.add_argument("--out", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--opm-map", action="store_true", help="two-level [i,j,p,q] output map")
    ap.add_argument("--split", type=int, default=1)
    ap.add_argument("--residual", action="store_true", help="fp32 residual operand (f32 out)")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    M, Nn, Kd = a.M, a.N, a.K
    bf = torch.bfloat16
    A = torch.randn(M * Kd, device="cuda").to(bf)
    B = torch.randn(Nn * Kd, device="cuda").to(bf)
    Am = K.Mat(A, Kd, 1) if a.a_major == "k" else K.Mat(A, 1, M)
    Bm = K.Mat(B, Kd, 1) if a.b_major == "k" else K.Mat(B, 1, Nn)
    C = torch.empty(M * Nn, device="cuda", dtype=bf if a.out == "bf16" else torch.float32)
    if a.opm_map:
        c = 32
        r = M // c
        Cm = K.Mat(C, r * c * c, c * c, rdiv=c, rs0=c, cdiv=c, cs0=1)
    else:
        Cm = K.Mat(C, Nn, 1)
    bias = torch.randn(Nn, device="cuda") if a.epi != "none" else None
    epi = {"none": N.EPI_NONE, "bias": N.EPI_NONE, "relu": N.EPI_RELU,
           "sigmoid": N.EPI_SIGMOID_FROM}[a.epi]

    R = torch.randn(M * Nn, device="cuda") if a.residual else None

    def run():
        K.gemm(Am, Bm, Cm, M, Nn, Kd, bias=bias, epi=epi, col0=Nn // 4 * 3, split_k=a.split,
               residual=R)

    # graph-replayed (host launch overhead excluded)
    from tools.ew_bench import timeit
    us = timeit(run, a.iters)
    fl = 2.0 * M * Nn * Kd
    byt = (M * Kd + Nn * Kd) * 2 + M * Nn * C.element_size()
    print(f"M={M} N={Nn} K={Kd} a={a.a_major} b={a.b_major} epi={a.epi} out={a.out} "
          f"opm={a.opm_map}: {us:.1f} us  {fl / us / 1e6:.1f} TF/s  {byt / us / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
