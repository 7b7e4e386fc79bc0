"""The strided batched GEMM entry point (evo_gemm) against a plain PyTorch
fp32 reference of the same op, on both the tcgen05/TMA kernel and the
SIMT kernel: every operand-major combination, batching (incl. broadcast
operands), split-K, every epilogue, two-level output maps, ragged sizes.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2211_00235_b200 import kernels
    return kernels


def rel(a, b):
    a, b = a.double(), b.double()
    v = float((a - b).norm() / b.norm().clamp_min(1e-30))
    return v if v == v and v != float("inf") else float("inf")


def make_operand(rows, k, kmajor, batch=1, dtype=torch.bfloat16):
    """Returns (storage tensor, logical [batch, rows, k] fp32 view, rs, cs, bs)."""
    if kmajor:
        t = torch.randn(batch, rows, k, device="cuda").to(dtype)
        return t, t.float(), k, 1, rows * k
    t = torch.randn(batch, k, rows, device="cuda").to(dtype)
    return t, t.float().transpose(1, 2), 1, rows, rows * k


@pytest.mark.parametrize("a_k,b_k", [(True, True), (True, False), (False, True),
                                     (False, False)])
@pytest.mark.parametrize("M,N,Kd", [(128, 128, 64), (200, 72, 100), (300, 520, 256),
                                    (64, 256, 1000)])
@pytest.mark.parametrize("force_simt", [False, True])
@pytest.mark.parametrize("out", [torch.float32, torch.bfloat16])
def test_gemm_majors_and_ragged(K, a_k, b_k, M, N, Kd, force_simt, out):
    from paper_2211_00235_b200 import _native
    A, Af, ars, acs, _ = make_operand(M, Kd, a_k)
    B, Bf, brs, bcs, _ = make_operand(N, Kd, b_k)
    C = torch.empty(M, N, device="cuda", dtype=out)

    def call():
        K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, N, 1), M, N, Kd,
               force_simt=force_simt)

    # the tensor-core kernel takes 16-byte-aligned K-major rows (K % 8 == 0)
    # or MN-major columns (rows % 8 == 0); the rest is SIMT-only
    tc_ok = ((Kd % 8 == 0) if a_k else (M % 8 == 0)) and ((Kd % 8 == 0) if b_k else (N % 8 == 0))
    if force_simt:
        call()
        assert _native.last_backend() == "gemm_simt"
    elif tc_ok:
        call()
        assert _native.last_backend() == "gemm_tc"
    else:
        # strict tensor-core mode (the default) refuses the SIMT fallback
        with pytest.raises(RuntimeError, match="strict tensor-core"):
            call()
        with _native.strict_tc(False):
            call()
        assert _native.last_backend() == "gemm_simt"
    want = Af[0] @ Bf[0].T
    assert rel(C.float(), want) < (1e-5 if out == torch.float32 else 4e-3)


@pytest.mark.parametrize("force_simt", [False, True])
def test_gemm_batched_broadcast_split_k(K, force_simt):
    M, N, Kd, nb = 96, 160, 4096, 3
    A, Af, ars, acs, _ = make_operand(M, Kd, False, 1)      # broadcast over batch
    B, Bf, brs, bcs, bbs = make_operand(N, Kd, True, nb)
    C = torch.zeros(nb, M, N, device="cuda")
    K.gemm(K.Mat(A, ars, acs, bs1=0), K.Mat(B, brs, bcs, bs1=bbs), K.Mat(C, N, 1, bs1=M * N),
           M, N, Kd, B1=nb, split_k=8, force_simt=force_simt)
    want = torch.stack([Af[0] @ Bf[i].T for i in range(nb)])
    assert rel(C, want) < 1e-5


@pytest.mark.parametrize("force_simt", [False, True])
def test_gemm_epilogues_bf16_out(K, force_simt):
    M, N, Kd = 256, 384, 128
    A, Af, ars, acs, _ = make_operand(M, Kd, True)
    B, Bf, brs, bcs, _ = make_operand(N, Kd, False)
    bias = torch.randn(N, device="cuda")
    raw = Af[0] @ Bf[0].T * 0.5 + bias
    from paper_2211_00235_b200._native import EPI_RELU, EPI_SIGMOID_FROM
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, N, 1), M, N, Kd, alpha=0.5,
           bias=bias, epi=EPI_RELU, force_simt=force_simt)
    assert rel(C.float(), torch.relu(raw)) < 5e-3
    col0 = 200
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, N, 1), M, N, Kd, alpha=0.5,
           bias=bias, epi=EPI_SIGMOID_FROM, col0=col0, force_simt=force_simt)
    want = raw.clone()
    want[:, col0:] = torch.sigmoid(raw[:, col0:])
    assert rel(C.float(), want) < 5e-3
    # the gate columns alone (bf16 out: packed bf16x2 tanh on whole chunks)
    assert rel(C.float()[:, col0:], want[:, col0:]) < 5e-3
    assert float((C.float()[:, col0:] - want[:, col0:]).abs().max()) < 1e-2


@pytest.mark.parametrize("force_simt", [False, True])
def test_gemm_residual_accumulate_and_offsets(K, force_simt):
    M, N, Kd = 130, 256, 192
    A, Af, ars, acs, _ = make_operand(M, Kd, True)
    B, Bf, brs, bcs, _ = make_operand(N, Kd, True)
    R = torch.randn(M, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, N, 1), M, N, Kd, residual=R,
           force_simt=force_simt)
    want = Af[0] @ Bf[0].T + R
    assert rel(C, want) < 1e-5
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, N, 1), M, N, Kd, accumulate=True,
           force_simt=force_simt)
    assert rel(C, want + Af[0] @ Bf[0].T) < 1e-5
    # column-offset output into a wider buffer (packed projection layout)
    W = torch.zeros(M, 3 * N, device="cuda")
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(W, 3 * N, 1, off=N), M, N, Kd,
           force_simt=force_simt)
    assert rel(W[:, N:2 * N], Af[0] @ Bf[0].T) < 1e-5
    assert float(W[:, :N].abs().max()) == 0.0 and float(W[:, 2 * N:].abs().max()) == 0.0


@pytest.mark.parametrize("force_simt", [False, True])
def test_gemm_two_level_output_map(K, force_simt):
    """The outer-product-mean store: m=(i,p), n=(j,q) -> o[i,j,p,q]."""
    r, c, s = 24, 16, 40
    a = torch.randn(s, r * c, device="cuda").to(torch.bfloat16)
    b = torch.randn(s, r * c, device="cuda").to(torch.bfloat16)
    o = torch.empty(r, r, c, c, device="cuda")
    rc = r * c
    K.gemm(K.Mat(a, 1, rc), K.Mat(b, 1, rc),
           K.Mat(o, r * c * c, c * c, rdiv=c, rs0=c, cdiv=c, cs0=1), rc, rc, s, alpha=1.0 / s,
           force_simt=force_simt)
    want = torch.einsum("sip,sjq->ijpq", a.float().view(s, r, c), b.float().view(s, r, c)) / s
    assert rel(o, want) < 1e-5


def test_gemm_tc_path_is_taken(K):
    from paper_2211_00235_b200 import _native
    assert _native.lib().evo_tc_available() == 1
    A = torch.randn(512, 256, device="cuda").to(torch.bfloat16)
    B = torch.randn(256, 256, device="cuda").to(torch.bfloat16)
    C = torch.empty(512, 256, device="cuda")
    before = _native.backend_counts()
    K.gemm(K.Mat(A, 256, 1), K.Mat(B, 256, 1), K.Mat(C, 256, 1), 512, 256, 256)
    after = _native.backend_counts()
    torch.cuda.synchronize()
    assert after["gemm_tc"] == before["gemm_tc"] + 1
    assert after["gemm_simt"] == before["gemm_simt"]
    assert rel(C, A.float() @ B.float().T) < 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M,N,Kd,a_k", [(5000, 8, 128, True), (4100, 12, 100, False), (4099, 4, 128, True),
                                        (65536, 8, 128, True)])
def test_gemm_skinny_rowdot(K, dtype, M, N, Kd, a_k):
    """N <= 16 (the pair-bias projection): output in the [N, M] layout."""
    A, Af, ars, acs, _ = make_operand(M, Kd, a_k, dtype=dtype)
    B, Bf, brs, bcs, _ = make_operand(N, Kd, False, dtype=dtype)
    C = torch.empty(N, M, device="cuda")
    bias = torch.randn(N, device="cuda")
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, 1, M), M, N, Kd, bias=bias)
    want = (Af[0] @ Bf[0].T + bias).T
    assert rel(C, want) < 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M,N,Kd", [(4096, 128, 8), (5003, 136, 12), (4096, 32, 4), (4100, 44, 5)])
def test_gemm_skinny_expand_residual_accumulate(K, dtype, M, N, Kd):
    """K <= 16 (the pair-bias input gradient), A column-major like dbias."""
    A, Af, ars, acs, _ = make_operand(M, Kd, False, dtype=dtype)
    B, Bf, brs, bcs, _ = make_operand(N, Kd, True, dtype=dtype)
    R = torch.randn(M, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, N, 1), M, N, Kd, residual=R)
    want = Af[0] @ Bf[0].T + R
    assert rel(C, want) < 1e-5
    K.gemm(K.Mat(A, ars, acs), K.Mat(B, brs, bcs), K.Mat(C, N, 1), M, N, Kd, accumulate=True,
           alpha=0.5)
    assert rel(C, want + 0.5 * (Af[0] @ Bf[0].T)) < 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("M,N,Kd,nb,a_k,b_k", [(128, 8, 20000, 1, False, True),
                                               (32, 128, 16384, 1, False, False),
                                               (48, 24, 9000, 2, False, True),
                                               (200, 12, 8192, 1, True, False)])
def test_gemm_skinny_tall_k(K, dtype, M, N, Kd, nb, a_k, b_k):
    """Weight gradients of the narrow layers: tiny M*N, K = r*r rows."""
    A, Af, ars, acs, abs_ = make_operand(M, Kd, a_k, nb, dtype=dtype)
    B, Bf, brs, bcs, bbs = make_operand(N, Kd, b_k, nb, dtype=dtype)
    from paper_2211_00235_b200 import _native
    C = torch.empty(nb, M, N, device="cuda")

    def call():
        K.gemm(K.Mat(A, ars, acs, bs1=abs_), K.Mat(B, brs, bcs, bs1=bbs),
               K.Mat(C, N, 1, bs1=M * N), M, N, Kd, B1=nb)

    if dtype == torch.bfloat16 and a_k and not b_k:
        # K-major wide operand with a 12-wide MN-major narrow one: neither the
        # streaming tall-K kernel nor the tensor-core maps take this layout
        # (the product never forms it); strict mode refuses the SIMT fallback
        with pytest.raises(RuntimeError, match="strict tensor-core"):
            call()
        with _native.strict_tc(False):
            call()
        assert _native.last_backend() == "gemm_simt"
    else:
        call()
        if dtype == torch.bfloat16:
            assert _native.last_backend() in ("gemm_skinny", "gemm_tc")
    want = torch.stack([Af[i].double() @ Bf[i].double().T for i in range(nb)])
    # fp32 accumulation over K >= 8192 terms (tensor-core or SIMT partials)
    assert rel(C, want) < 5e-5


def test_gemm_tc_accumulate_two_level_map(K):
    """TMA reduce-add epilogue through the 3-D / 4-D output maps."""
    r, c, s = 32, 32, 64
    rc = r * c
    a = torch.randn(s, rc, device="cuda").to(torch.bfloat16)
    b = torch.randn(s, rc, device="cuda").to(torch.bfloat16)
    o = torch.randn(r, r, c, c, device="cuda")
    o0 = o.clone()
    K.gemm(K.Mat(a, 1, rc), K.Mat(b, 1, rc),
           K.Mat(o, r * c * c, c * c, rdiv=c, rs0=c, cdiv=c, cs0=1), rc, rc, s, alpha=1.0 / s,
           accumulate=True)
    want = o0 + torch.einsum("sip,sjq->ijpq", a.float().view(s, r, c), b.float().view(s, r, c)) / s
    assert rel(o, want) < 1e-6
    # 3-D map (column blocks only): C(m, (j,q)) at j*(r*c) ... + m*c + q
    C = torch.randn(r, rc, device="cuda")
    C0 = C.clone()
    K.gemm(K.Mat(a, 1, rc), K.Mat(b, 1, rc), K.Mat(C, c, r * c, cdiv=c, cs0=1), r, rc, s,
           accumulate=True)
    got = C.view(r, r, c).permute(1, 0, 2).reshape(r, rc)  # [m, (j,q)]
    want2 = C0.view(r, r, c).permute(1, 0, 2).reshape(r, rc) + a.float()[:, :r].T @ b.float()
    assert rel(got, want2) < 1e-6


def test_gemm_opm_layouts_bf16_out(K):
    """The outer-product-mean GEMMs exactly as the engine issues them, bf16
    output with c = 32 (the 4-D TMA-store box of the production path,
    engine.opm_fwd / opm_bwd): o[i,j,p,q] and the input-gradient layout
    do'[(i,p),(j,q)].  Every element is checked (a wrong store layout once
    passed a NaN-blind aggregate)."""
    from paper_2211_00235_b200 import _native
    c, s = 32, 128
    for r in (64, 96):
        rc = r * c
        ab = (torch.randn(2, s * r, c, device="cuda") * 0.5).to(torch.bfloat16)
        o = torch.full((r, r, c, c), float("nan"), device="cuda", dtype=torch.bfloat16)
        before = _native.backend_counts()["gemm_tc"]
        K.gemm(K.Mat(ab[0], 1, rc), K.Mat(ab[1], 1, rc),
               K.Mat(o, r * c * c, c * c, rdiv=c, rs0=c, cdiv=c, cs0=1), rc, rc, s,
               alpha=1.0 / s)
        torch.cuda.synchronize()
        assert _native.backend_counts()["gemm_tc"] == before + 1
        want = torch.einsum("sip,sjq->ijpq", ab[0].float().view(s, r, c),
                            ab[1].float().view(s, r, c)) / s
        err = (o.float() - want).abs()
        assert bool(torch.isfinite(o.float()).all())
        assert float(err.max()) <= 1e-2 * float(want.abs().max()), float(err.max())
        # do'[(i,p),(j,q)] = (1/s) dz[(i,j)] . Wo[(p,q)]
        cz = 128
        dz = (torch.randn(r * r, cz, device="cuda") * 0.5).to(torch.bfloat16)
        Wo = (torch.randn(c * c, cz, device="cuda") * 0.05).to(torch.bfloat16)
        dor = torch.full((rc, rc), float("nan"), device="cuda", dtype=torch.bfloat16)
        K.gemm(K.Mat(dz, cz, 1), K.Mat(Wo, cz, 1),
               K.Mat(dor, c * r * c, r * c, rdiv=r, rs0=c, cdiv=c, cs0=1), r * r, c * c, cz,
               alpha=1.0 / s)
        torch.cuda.synchronize()
        full = (dz.float() @ Wo.float().t()) / s
        want2 = full.reshape(r, r, c, c).permute(0, 2, 1, 3).reshape(rc, rc)
        assert bool(torch.isfinite(dor.float()).all())
        assert float((dor.float() - want2).abs().max()) <= 1e-2 * float(want2.abs().max())
