"""The fused gated attention entry points (evo_attention_fwd/bwd) against a
plain PyTorch fp32 reference of the same op, on the tcgen05 path (bf16)
and the SIMT path (fp32), over the four geometries of the block (row /
column / triangle-start / triangle-end: batch-major or sequence-major rows,
plain or transposed pair bias), ragged L and every supported head dim."""

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


def run_case(K, nb, L, H, D, seq_major, bias_mode, dtype, seed=0, gate_bias=False,
             keep_p=False):
    torch.manual_seed(seed)
    hc = H * D
    rows = nb * L
    # row index of (b, l): batch-major (row/tri-start) or sequence-major (col/tri-end)
    if seq_major:
        sb, sl = 1, nb
    else:
        sb, sl = L, 1
    proj = torch.randn(rows, 4 * hc, device="cuda")
    proj[:, 3 * hc:] = torch.sigmoid(proj[:, 3 * hc:])
    proj = proj.to(dtype)
    bias = None
    bh = bq = bk = 0
    if bias_mode != "none":
        bias = torch.randn(H, L * L, device="cuda")
        bh = L * L
        bq, bk = (L, 1) if bias_mode == "plain" else (1, L)
    o = torch.empty(rows, hc, device="cuda", dtype=dtype)
    gm = torch.empty_like(o)
    lse = torch.empty(nb, H, L, device="cuda")
    scale = D ** -0.5
    geo = dict(proj=proj, hc=hc, nb=nb, H=H, L=L, D=D, scale=scale, sb=sb * 4 * hc,
               sl=sl * 4 * hc, o=o, gm=gm, o_sb=sb * hc, o_sl=sl * hc, lse=lse, bias=bias,
               bh=bh, bq=bq, bk=bk)
    if keep_p:
        geo["p_store"] = torch.empty(K.long_p_elems(nb, H, L), device="cuda", dtype=dtype)
    from paper_2211_00235_b200 import _native
    before = _native.backend_counts()
    K.attention(**geo)
    dgm = torch.randn(rows, hc, device="cuda").to(dtype)
    dproj = torch.zeros(rows, 4 * hc, device="cuda", dtype=dtype)
    dbias = torch.empty(H, L * L, device="cuda") if bias is not None else None
    dgb = torch.empty(hc, device="cuda") if gate_bias else None
    K.attention(**geo, dgm=dgm, dproj=dproj, dbias=dbias, dgate_bias=dgb)
    torch.cuda.synchronize()
    after = _native.backend_counts()
    # which engine ran: the fused tcgen05 kernels, the GEMM-composed long-key
    # path (tcgen05 GEMMs) or the SIMT kernels (fp32 parity path)
    d_tc = after["attn_tc"] - before["attn_tc"]
    d_simt = after["attn_simt"] - before["attn_simt"]
    d_gemm = after["gemm_tc"] - before["gemm_tc"]
    d_fl = after["attn_flash"] - before["attn_flash"]
    if dtype == torch.float32:
        assert (d_tc, d_simt) == (0, 2), (d_tc, d_simt)
    elif K.use_flash(dtype, L, D):
        assert (d_tc, d_simt, d_fl) == (0, 0, 2), (d_tc, d_simt, d_fl)
    elif K.use_long(dtype, L, D):
        assert (d_tc, d_simt) == (0, 0) and d_gemm >= 6, (d_tc, d_simt, d_gemm)
    else:
        assert (d_tc, d_simt) == (2, 0), (d_tc, d_simt)

    # ---- torch fp32 reference on the same (rounded) inputs
    pf = proj.float()
    idx = (torch.arange(nb, device="cuda")[:, None] * sb +
           torch.arange(L, device="cuda")[None, :] * sl)          # [nb, L] row ids

    def heads(col0):
        x = pf[idx][:, :, col0:col0 + hc]                         # [nb, L, hc]
        return x.view(nb, L, H, D).permute(0, 2, 1, 3).contiguous()

    q = heads(0).requires_grad_(True)
    k = heads(hc).requires_grad_(True)
    v = heads(2 * hc).requires_grad_(True)
    g = heads(3 * hc)
    bt = None
    if bias is not None:
        hh, qq, kk = torch.meshgrid(torch.arange(H), torch.arange(L), torch.arange(L),
                                    indexing="ij")
        bt = bias.view(-1)[(hh * bh + qq * bq + kk * bk).cuda()].clone().requires_grad_(True)
    s = (q * scale) @ k.transpose(-1, -2)
    if bt is not None:
        s = s + bt
    p = torch.softmax(s, -1)
    O = p @ v
    G = g * O
    dG = dgm.float()[idx].view(nb, L, H, D).permute(0, 2, 1, 3)
    (G * dG).sum().backward()
    dgpre = dG * O.detach() * g * (1 - g)

    def gather(t):  # [nb, H, L, D] -> [nb, L, hc] by rows
        return t.permute(0, 2, 1, 3).reshape(nb, L, hc)

    errs = {
        "o": rel(o.float()[idx], gather(O.detach())),
        "gm": rel(gm.float()[idx], gather(G.detach())),
        "lse": rel(lse, torch.logsumexp(s.detach(), -1)),
        "dq": rel(dproj.float()[idx][:, :, :hc], gather(q.grad)),
        "dk": rel(dproj.float()[idx][:, :, hc:2 * hc], gather(k.grad)),
        "dv": rel(dproj.float()[idx][:, :, 2 * hc:3 * hc], gather(v.grad)),
        "dgpre": rel(dproj.float()[idx][:, :, 3 * hc:], gather(dgpre)),
    }
    if bt is not None:
        hh, qq, kk = torch.meshgrid(torch.arange(H), torch.arange(L), torch.arange(L),
                                    indexing="ij")
        got = dbias.view(-1)[(hh * bh + qq * bq + kk * bk).cuda()]
        errs["dbias"] = rel(got, bt.grad)
    if gate_bias:
        errs["dgate_bias"] = rel(dgb, gather(dgpre).sum((0, 1)))
    return errs


CASES = [
    # nb, L, H, D, seq_major, bias
    (6, 256, 2, 32, False, "plain"),     # row attention / triangle start
    (5, 256, 2, 32, True, "transposed"), # triangle end
    (7, 128, 2, 32, True, "none"),       # column attention
    (3, 100, 2, 32, False, "plain"),     # ragged L (masked keys, partial tile)
    (4, 64, 4, 16, False, "plain"),      # mid config head dim
    (4, 160, 2, 64, True, "transposed"),
    (9, 48, 3, 16, True, "none"),
    (3, 200, 2, 32, False, "plain"),     # ragged L in the pipelined (Lp = 256) path
    (5, 230, 3, 16, True, "transposed"),
    (150, 256, 4, 32, False, "plain"),   # 9-row chunks per CTA: row pipeline wrap-around
    (64, 256, 2, 32, True, "none"),
    (130, 128, 4, 32, True, "none"),     # column attention, many rows per CTA (Lp = 128 pipe)
    (40, 120, 2, 16, False, "transposed"),
]


@pytest.mark.parametrize("case", CASES)
def test_attention_tc_bf16(K, case):
    errs = run_case(K, *case, dtype=torch.bfloat16)
    bad = {k: v for k, v in errs.items() if v > 1.5e-2}
    assert not bad, errs


@pytest.mark.parametrize("case", CASES[:4])
def test_attention_simt_fp32(K, case):
    errs = run_case(K, *case, dtype=torch.float32)
    bad = {k: v for k, v in errs.items() if v > 2e-6}
    assert not bad, errs


# keys beyond the tensor-core kernel's 256: the SIMT kernels with 512 / 1024
# resident keys (crop r = 384 row / triangle attention, the extra-MSA column
# attention over s_e = 1024 at c_head = 8), gate-bias sums included
LONG = [
    (3, 384, 2, 32, False, "plain"),
    (2, 384, 2, 32, True, "transposed"),
    (4, 1024, 2, 8, True, "none"),
    (2, 700, 2, 16, False, "plain"),
]


@pytest.mark.parametrize("case", LONG)
@pytest.mark.parametrize("dtype,tol", [(torch.float32, 2e-6), (torch.bfloat16, 1.5e-2)])
def test_attention_long_keys(K, case, dtype, tol):
    errs = run_case(K, *case, dtype=dtype, gate_bias=True)
    bad = {k: v for k, v in errs.items() if v > tol}
    assert not bad, errs


@pytest.mark.parametrize("case", LONG)
def test_attention_long_keys_forward_p_kept(K, case):
    """The engine's long-key path: the forward keeps P for the backward."""
    errs = run_case(K, *case, dtype=torch.bfloat16, gate_bias=True, keep_p=True)
    bad = {k: v for k, v in errs.items() if v > 1.5e-2}
    assert not bad, errs


@pytest.mark.parametrize("case", [(7, 384, 2, 32, False, "plain"),
                                  (5, 384, 2, 32, True, "transposed"),
                                  (10, 320, 2, 16, True, "none")])
@pytest.mark.parametrize("keep_p", [False, True])
def test_attention_long_keys_multi_chunk(K, case, keep_p, monkeypatch):
    """The long-key path's batch-row chunk loop: chunks of 3 rows (uneven
    last chunk), so dbias accumulates across chunks and the P / lse / Dq
    offsets advance."""
    nb, L, H = case[0], case[1], case[2]
    monkeypatch.setattr(K, "LONG_CHUNK_ELEMS", 3 * H * L * L)
    errs = run_case(K, *case, dtype=torch.bfloat16, gate_bias=True, keep_p=keep_p)
    bad = {k: v for k, v in errs.items() if v > 1.5e-2}
    assert not bad, errs


# keys beyond 256 on the streamed-key fused kernels (csrc/attention_flash.cu):
# partial key / query tiles, both bias layouts, no bias, head dims 16 / 32,
# batch-row chunks for the dbias partials
FLASH = [
    (3, 384, 2, 32, False, "plain"),      # crop r = 384 row / triangle-start attention
    (2, 384, 3, 32, True, "transposed"),  # triangle end
    (4, 512, 2, 32, True, "none"),        # MSA column attention at s = 512
    (2, 300, 2, 16, False, "plain"),      # partial last key tile
    (3, 333, 2, 32, True, "transposed"),  # ragged L: padded plain bias copy
    (2, 1024, 2, 16, True, "none"),
    (40, 320, 4, 32, False, "plain"),     # several batch rows per dq CTA
    # head dim 8 (the extra-MSA stack, c_head = c_e / h = 8): zero-padded to
    # the 16-wide MMA K step
    (6, 64, 4, 8, False, "plain"),        # extra-MSA row attention (small r)
    (4, 256, 8, 8, True, "none"),         # column attention
    (3, 1024, 8, 8, True, "none"),        # C3 extra column attention over s_e = 1024
    (5, 200, 4, 8, True, "transposed"),   # triangle end
    (9, 130, 8, 8, False, "plain"),
]


@pytest.mark.parametrize("case", FLASH)
def test_attention_flash_bf16(K, case):
    assert K.use_flash(torch.bfloat16, case[1], case[3])
    errs = run_case(K, *case, dtype=torch.bfloat16, gate_bias=True)
    bad = {k: v for k, v in errs.items() if v > 1.5e-2}
    assert not bad, errs


def test_attention_flash_deterministic(K):
    a = run_case(K, 5, 384, 2, 32, False, "plain", dtype=torch.bfloat16, seed=4)
    b = run_case(K, 5, 384, 2, 32, False, "plain", dtype=torch.bfloat16, seed=4)
    assert a == b
