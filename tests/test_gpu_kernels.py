"""GPU numerics of the dense and sparse kernels through the C ABI against a
plain PyTorch fp32 reference of the same op (bf16-rounded operands, fp32
accumulation): the tcgen05 GEMMs (contract, pmm.hpp:97-130, and its
transposed-operand forms) and the row-split SpMM (spmm, pmm.hpp:134-167)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(gg):
    import torch
    ctx = gg.Context()
    return ctx, torch


def _ld8(c):
    return ((max(c, 1) + 7) // 8) * 8


def _bf16_matrix(torch, rows, cols, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    ld = _ld8(cols)
    full = torch.zeros(rows, ld, dtype=torch.bfloat16, device="cuda")
    full[:, :cols] = (torch.randn(rows, cols, generator=g, device="cuda") * scale).to(torch.bfloat16)
    return full, ld


GEMM_SHAPES = [(128, 256, 256), (1000, 256, 256), (517, 48, 256), (300, 47, 256), (4096, 256, 100),
               (129, 16, 8), (77, 5, 24), (2000, 320, 64), (256, 256, 602), (1, 16, 16), (612, 128, 301)]


@pytest.mark.parametrize("m,n,k", GEMM_SHAPES)
def test_gemm_bf16(env, gg, m, n, k):
    ctx, torch = env
    a, lda = _bf16_matrix(torch, m, k, 1)
    bt, ldb = _bf16_matrix(torch, n, k, 2)
    c = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    ldcb = _ld8(n)
    cb = torch.zeros(m, ldcb, dtype=torch.bfloat16, device="cuda")
    gg.check(gg.lib().ggb_gemm_bf16(ctx.h, m, n, k, a.data_ptr(), lda, bt.data_ptr(), ldb, c.data_ptr(), n,
                                    cb.data_ptr(), ldcb))
    ctx.synchronize()
    want = a[:, :k].float() @ bt[:, :k].float().T
    err = (c - want).abs().max().item()
    assert err <= 1e-3 * max(1.0, want.abs().max().item()), err
    assert torch.equal(cb[:, :n], c.to(torch.bfloat16))


@pytest.mark.parametrize("m,n,k", [(1000, 256, 256), (300, 47, 256), (4096, 256, 100), (77, 5, 24),
                                   (2000, 320, 64), (612, 128, 301)])
def test_gemm_split_bf16_is_fp32_accurate(env, gg, m, n, k):
    """Split-bf16 (hi + lo pairs, 3 MMAs) reproduces the fp32 product to
    ~1e-5 relative — the forward contract of the accurate mode."""
    ctx, torch = env
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = torch.randn(m, k, generator=g, device="cuda")
    B = torch.randn(n, k, generator=g, device="cuda") * 0.1
    lda, ldb = _ld8(k), _ld8(k)

    def split(X, ld):
        hi = torch.zeros(X.shape[0], ld, dtype=torch.bfloat16, device="cuda")
        lo = torch.zeros_like(hi)
        hi[:, :X.shape[1]] = X.to(torch.bfloat16)
        lo[:, :X.shape[1]] = (X - hi[:, :X.shape[1]].float()).to(torch.bfloat16)
        return hi, lo

    ah, al = split(A, lda)
    bh, bl = split(B, ldb)
    c = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    gg.check(gg.lib().ggb_gemm_split_bf16(ctx.h, m, n, k, ah.data_ptr(), al.data_ptr(), lda, bh.data_ptr(),
                                          bl.data_ptr(), ldb, c.data_ptr(), n))
    ctx.synchronize()
    want = (A.double() @ B.double().T)
    scale = want.abs().max().item()
    assert (c.double() - want).abs().max().item() <= 2e-5 * scale


@pytest.mark.parametrize("m,kw,nw", [(128, 128, 256), (10000, 256, 256), (612, 100, 256), (5000, 256, 47),
                                     (20000, 200, 256), (153000, 256, 256), (3000, 129, 64),
                                     (333, 16, 16), (64, 8, 5), (20000, 301, 128), (1, 64, 64)])
def test_gemm_wgrad(env, gg, m, kw, nw):
    ctx, torch = env
    x, ldx = _bf16_matrix(torch, m, kw, 3)
    dy, lddy = _bf16_matrix(torch, m, nw, 4)
    dw = torch.full((kw, nw), float("nan"), dtype=torch.float32, device="cuda")
    gg.check(gg.lib().ggb_gemm_wgrad_bf16(ctx.h, m, kw, nw, x.data_ptr(), ldx, dy.data_ptr(), lddy, dw.data_ptr(),
                                          nw))
    ctx.synchronize()
    want = x[:, :kw].float().T @ dy[:, :nw].float()
    err = (dw - want).abs().max().item()
    assert err <= 1e-3 * max(1.0, want.abs().max().item()), err


def _random_csr(rows, cols, nnz_per_row, seed):
    rng = np.random.default_rng(seed)
    deg = rng.poisson(nnz_per_row, rows)
    deg[rng.integers(0, rows, max(1, rows // 10))] = 0  # empty rows
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(cols, d, replace=False)) if d else np.zeros(0, np.int64)
                          for d in np.minimum(deg, cols)]).astype(np.int32)
    rp = np.concatenate([[0], np.cumsum(np.minimum(deg, cols))]).astype(np.int64)
    val = rng.random(len(col)).astype(np.float32)
    return rp, col, val


@pytest.mark.parametrize("rows,fcols,deg", [(1000, 256, 13), (777, 128, 30), (500, 64, 5), (300, 40, 9),
                                            (257, 16, 3), (1200, 300, 7), (64, 256, 200)])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_spmm(env, gg, rows, fcols, deg, accumulate):
    ctx, torch = env
    frows = 900
    rp, col, val = _random_csr(rows, frows, deg, rows + fcols)
    f, ldf = _bf16_matrix(torch, frows, fcols, 5)
    trp, tcol, tval = (torch.from_numpy(x).cuda() for x in (rp, col, val))
    base = torch.randn(rows, fcols, device="cuda")
    out = base.clone() if accumulate else torch.full((rows, fcols), float("nan"), device="cuda")
    ldob = _ld8(fcols)
    outb = torch.zeros(rows, ldob, dtype=torch.bfloat16, device="cuda")
    gg.check(gg.lib().ggb_spmm_csr(ctx.h, rows, trp.data_ptr(), tcol.data_ptr(), tval.data_ptr(), f.data_ptr(), ldf,
                                   fcols, out.data_ptr(), fcols, outb.data_ptr(), ldob, accumulate))
    ctx.synchronize()
    A = torch.sparse_csr_tensor(trp, tcol.long(), tval, size=(rows, frows)).to_dense()
    want = A @ f[:, :fcols].float() + (base if accumulate else 0)
    assert (out - want).abs().max().item() < 1e-4 * max(1.0, want.abs().max().item())
    assert torch.equal(outb[:, :fcols], out.to(torch.bfloat16))


# The accurate forward's SpMM: fp32 feature rows (k_spmm_pipe<float, RB>;
# H = 256 gives 1 KB rows, the production instance of the C2/C3 step), fp32
# accumulation in CSR order as pmm.hpp:157-164, optional split-bf16 output.
@pytest.mark.parametrize("rows,frows,fcols,deg", [(20000, 30000, 256, 14), (1000, 900, 256, 40),
                                                  (3000, 5000, 128, 9), (777, 900, 100, 30),
                                                  (500, 600, 64, 5), (64, 300, 256, 200), (5, 7, 256, 3)])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_spmm_f32_rows(env, gg, rows, frows, fcols, deg, accumulate):
    ctx, torch = env
    rp, col, val = _random_csr(rows, frows, deg, rows + fcols + 1)
    g = torch.Generator(device="cuda").manual_seed(fcols)
    ldf = _ld8(fcols)
    f = torch.zeros(frows, ldf, device="cuda")
    f[:, :fcols] = torch.randn(frows, fcols, generator=g, device="cuda")
    trp, tcol, tval = (torch.from_numpy(x).cuda() for x in (rp, col, val))
    base = torch.randn(rows, fcols, device="cuda")
    out = base.clone() if accumulate else torch.full((rows, fcols), float("nan"), device="cuda")
    ldob = _ld8(fcols)
    hi = torch.zeros(rows, ldob, dtype=torch.bfloat16, device="cuda")
    lo = torch.zeros_like(hi)
    gg.check(gg.lib().ggb_spmm_csr_f32(ctx.h, rows, trp.data_ptr(), tcol.data_ptr(), tval.data_ptr(), f.data_ptr(),
                                       ldf, fcols, out.data_ptr(), fcols, hi.data_ptr(), lo.data_ptr(), ldob,
                                       accumulate))
    ctx.synchronize()
    A = torch.sparse_csr_tensor(trp, tcol.long(), tval.double(), size=(rows, frows))
    want = A @ f[:, :fcols].double() + (base.double() if accumulate else 0)
    scale = max(1.0, want.abs().max().item())
    assert (out.double() - want).abs().max().item() <= 1e-5 * scale
    assert torch.equal(hi[:, :fcols], out.to(torch.bfloat16))
    assert torch.equal(lo[:, :fcols], (out - hi[:, :fcols].float()).to(torch.bfloat16))


def _skewed_csr(rows, cols, seed):
    """Power-law rows (R-MAT-like): a few hub rows with thousands of nonzeros
    among short ones and empty ones."""
    rng = np.random.default_rng(seed)
    deg = np.minimum(rng.zipf(1.6, rows), cols)
    deg[rng.integers(0, rows, 3)] = cols  # full hub rows
    deg[rng.integers(0, rows, rows // 20)] = 0
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(cols, d, replace=False)) for d in deg]).astype(np.int32)
    return rp, col, rng.random(len(col)).astype(np.float32)


# rows shared by several warps (merge-path split of the pipelined SpMM) must
# give the same sums as the dense product; the fp32 and bf16 gathers, with
# and without accumulation into the output
@pytest.mark.parametrize("fcols", [256, 128, 100])
@pytest.mark.parametrize("accumulate", [0, 1])
def test_spmm_skewed_rows(env, gg, fcols, accumulate):
    ctx, torch = env
    rows, frows = 6000, 20000
    rp, col, val = _skewed_csr(rows, frows, fcols)
    assert np.diff(rp).max() > 100 * np.diff(rp).mean()
    g = torch.Generator(device="cuda").manual_seed(fcols)
    ldf = _ld8(fcols)
    f = torch.zeros(frows, ldf, device="cuda")
    f[:, :fcols] = torch.randn(frows, fcols, generator=g, device="cuda")
    fb = f.to(torch.bfloat16)
    trp, tcol, tval = (torch.from_numpy(x).cuda() for x in (rp, col, val))
    A = torch.sparse_csr_tensor(trp, tcol.long(), tval.double(), size=(rows, frows))
    base = torch.randn(rows, fcols, device="cuda")
    for name, src in (("f32", f), ("bf16", fb)):
        out = base.clone() if accumulate else torch.full((rows, fcols), float("nan"), device="cuda")
        hi = torch.zeros(rows, ldf, dtype=torch.bfloat16, device="cuda")
        lo = torch.zeros_like(hi)
        if name == "f32":
            gg.check(gg.lib().ggb_spmm_csr_f32(ctx.h, rows, trp.data_ptr(), tcol.data_ptr(), tval.data_ptr(),
                                               src.data_ptr(), ldf, fcols, out.data_ptr(), fcols, hi.data_ptr(),
                                               lo.data_ptr(), ldf, accumulate))
        else:
            gg.check(gg.lib().ggb_spmm_csr(ctx.h, rows, trp.data_ptr(), tcol.data_ptr(), tval.data_ptr(),
                                           src.data_ptr(), ldf, fcols, out.data_ptr(), fcols, hi.data_ptr(), ldf,
                                           accumulate))
        ctx.synchronize()
        want = A @ src[:, :fcols].double() + (base.double() if accumulate else 0)
        scale = max(1.0, want.abs().max().item())
        assert (out.double() - want).abs().max().item() <= 1e-5 * scale, name
        assert torch.equal(hi[:, :fcols], out.to(torch.bfloat16)), name
