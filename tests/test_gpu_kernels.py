"""Bandwidth kernels (LayerNorm forward / backward incl. the fused hand-off
variant, column sums, ReLU backward, sum of squares) against plain PyTorch
fp32 references of the same ops (src/tensor.py:343, 366-392)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2211_00235_b200 import kernels
    return kernels


def rel(a, b):
    a, b = a.detach().double(), b.detach().double()
    v = float((a - b).norm() / b.norm().clamp_min(1e-30))
    return v if v == v and v != float("inf") else float("inf")


def ln_ref(x, g, b, eps=1e-5):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * g + b


# ragged row counts: partial last chunk of the TMA ring kernels (1004) and
# the register kernels' fallback for rows % 4 != 0 (1001)
@pytest.mark.parametrize("rows,cols", [(4096, 256), (8192, 128), (1000, 96), (1004, 256),
                                       (1001, 128), (1004, 128)])
def test_layernorm_fwd_bwd(K, rows, cols):
    torch.manual_seed(0)
    x = torch.randn(rows, cols, device="cuda")
    g = torch.randn(cols, device="cuda")
    b = torch.randn(cols, device="cuda")
    y = torch.empty(rows, cols, device="cuda")
    mu = torch.empty(rows, device="cuda")
    rs = torch.empty(rows, device="cuda")
    K.layernorm(x, rows, cols, g, b, y, mu, rs, 1e-5)
    xr = x.clone().requires_grad_(True)
    gr = g.clone().requires_grad_(True)
    br = b.clone().requires_grad_(True)
    yr = ln_ref(xr, gr, br)
    assert rel(y, yr) < 1e-5
    dy = torch.randn(rows, cols, device="cuda")
    res = torch.randn(rows, cols, device="cuda")
    yr.backward(dy)
    dx = torch.empty(rows, cols, device="cuda")
    dg = torch.empty(cols, device="cuda")
    db = torch.empty(cols, device="cuda")
    K.layernorm_bwd(dy, x, rows, cols, mu, rs, g, dx, dg, db, dres=res)
    assert rel(dx, xr.grad + res) < 1e-5
    assert rel(dg, gr.grad) < 1e-5
    assert rel(db, br.grad) < 1e-5


@pytest.mark.parametrize("rows,cols", [(4096, 256), (8192, 128)])
def test_layernorm_bwd_handoff(K, rows, cols):
    """The fused variant: dx plus its bf16 copy and column sums."""
    torch.manual_seed(1)
    x = torch.randn(rows, cols, device="cuda")
    g = torch.randn(cols, device="cuda")
    b = torch.randn(cols, device="cuda")
    y = torch.empty(rows, cols, device="cuda")
    mu = torch.empty(rows, device="cuda")
    rs = torch.empty(rows, device="cuda")
    K.layernorm(x, rows, cols, g, b, y, mu, rs, 1e-5)
    dy = torch.randn(rows, cols, device="cuda")
    res = torch.randn(rows, cols, device="cuda")
    dx0 = torch.empty(rows, cols, device="cuda")
    dg0, db0 = torch.empty(cols, device="cuda"), torch.empty(cols, device="cuda")
    K.layernorm_bwd(dy, x, rows, cols, mu, rs, g, dx0, dg0, db0, dres=res)
    dx = torch.empty(rows, cols, device="cuda")
    dxa = torch.empty(rows, cols, device="cuda", dtype=torch.bfloat16)
    dg, db, cs = (torch.empty(cols, device="cuda") for _ in range(3))
    K.layernorm_bwd_ex(dy, x, rows, cols, mu, rs, g, dx, dg, db, dres=res, dx_act=dxa,
                       dx_colsum=cs)
    assert torch.equal(dx, dx0)
    assert torch.equal(dxa, dx0.to(torch.bfloat16))
    assert torch.equal(dg, dg0) and torch.equal(db, db0)
    assert rel(cs, dx0.double().sum(0)) < 1e-6


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,cols", [(65536, 128), (5000, 72)])
def test_colsum(K, dtype, rows, cols):
    x = torch.randn(rows, cols, device="cuda").to(dtype)
    out = torch.empty(cols, device="cuda")
    K.colsum(x, rows, cols, out)
    assert rel(out, x.double().sum(0)) < 1e-6


def test_relu_bwd_and_sq_mean(K):
    h = torch.randn(1 << 20, device="cuda").to(torch.bfloat16)
    dh = torch.randn(1 << 20, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(dh)
    K.relu_bwd(dh, h, out, h.numel())
    assert torch.equal(out, torch.where(h > 0, dh, torch.zeros_like(dh)))
    x = torch.randn(3, 1000, device="cuda")
    loss = torch.zeros(1, device="cuda")
    dx = torch.empty_like(x)
    K.sq_mean(x, loss, dx)
    assert rel(loss, (x.double() ** 2).mean().reshape(1)) < 1e-6
    assert rel(dx, 2 * x / x.numel()) < 1e-6


@pytest.mark.parametrize("rows,h", [(4096, 8), (1004, 4)])
def test_layernorm_pair_bias_projection_fused(K, rows, h):
    """Backward of LN(z) followed by bias = LN(z) Wb, fused vs unfused kernels."""
    torch.manual_seed(2)
    cols = 128
    bf = torch.bfloat16
    x = torch.randn(rows, cols, device="cuda")
    g = torch.randn(cols, device="cuda")
    b = torch.randn(cols, device="cuda")
    Wb = (torch.randn(cols, h, device="cuda") * 0.1).to(bf)
    # forward LayerNorm (its statistics feed the fused backward)
    y0 = torch.empty(rows, cols, device="cuda", dtype=bf)
    mu0, rs0 = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    K.layernorm(x, rows, cols, g, b, y0, mu0, rs0, 1e-5)
    mu, rs = mu0, rs0
    # backward: dz = LN_bwd(dy + dbias Wb^T), dWb = y^T dbias
    dy = torch.randn(rows, cols, device="cuda")
    dbias = torch.randn(h, rows, device="cuda")
    dytot = dy + dbias.T @ Wb.float().T
    dx0 = torch.empty(rows, cols, device="cuda")
    dg0, db0 = torch.empty(cols, device="cuda"), torch.empty(cols, device="cuda")
    K.layernorm_bwd(dytot, x, rows, cols, mu0, rs0, g, dx0, dg0, db0)
    dW0 = y0.double().T @ dbias.double().T                # [cols, h]
    dx = torch.empty(rows, cols, device="cuda")
    dg, db = torch.empty(cols, device="cuda"), torch.empty(cols, device="cuda")
    dW = torch.empty(cols, h, device="cuda")
    K.layernorm_bwd_proj(dy, x, rows, mu, rs, g, b, dbias, rows, Wb, h, dx, dg, db, dW)
    assert rel(dx, dx0) < 1e-5
    assert rel(dg, dg0) < 1e-5 and rel(db, db0) < 1e-5
    assert rel(dW, dW0) < 1e-5
    # dy absent (row attention: the projection is the only consumer)
    K.layernorm_bwd_proj(None, x, rows, mu, rs, g, b, dbias, rows, Wb, h, dx, dg, db, dW)
    dytot = dbias.T @ Wb.float().T
    K.layernorm_bwd(dytot, x, rows, cols, mu0, rs0, g, dx0, dg0, db0)
    assert rel(dx, dx0) < 1e-5


def test_relu_bwd_colsum_fused(K):
    rows, cols = 5000, 1024
    h = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    dh = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(dh)
    cs = torch.empty(cols, device="cuda")
    K.relu_bwd_colsum(dh, h, out, rows, cols, cs)
    want = torch.where(h > 0, dh, torch.zeros_like(dh))
    assert torch.equal(out, want)
    assert rel(cs, want.double().sum(0)) < 1e-6


@pytest.mark.parametrize("rows,cols", [(4096, 128), (1003, 256)])
def test_layernorm_split_operand(K, rows, cols):
    """LN(x) straight into the [hi | lo | hi] bf16 operand of the 3-product
    transition projection == LN into fp32, then split."""
    torch.manual_seed(3)
    x = torch.randn(rows, cols, device="cuda")
    g, b = torch.randn(cols, device="cuda"), torch.randn(cols, device="cuda")
    y32 = torch.empty(rows, cols, device="cuda")
    mu0, rs0 = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    K.layernorm(x, rows, cols, g, b, y32, mu0, rs0, 1e-5)
    y3 = torch.empty(rows, 3 * cols, device="cuda", dtype=torch.bfloat16)
    mu, rs = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    assert K.layernorm_split(x, rows, cols, g, b, y3, mu, rs, 1e-5)
    hi = y32.to(torch.bfloat16)
    lo = (y32 - hi.float()).to(torch.bfloat16)
    assert torch.equal(y3[:, :cols], hi) and torch.equal(y3[:, 2 * cols:], hi)
    assert torch.equal(y3[:, cols:2 * cols], lo)
    assert torch.equal(mu, mu0) and torch.equal(rs, rs0)
    # the split kernel composes to the same operand
    y3b = torch.empty_like(y3)
    K.split_bf16(y32, rows, cols, y3b, y3b, h_rs=3 * cols, l_rs=3 * cols, hi2=y3b,
                 h2_rs=3 * cols, l_off=cols, h2_off=2 * cols)
    assert torch.equal(y3, y3b)
