"""The layer-level boundary (include/ggb.h ggb_contract / ggb_spmm /
ggb_transposed / ggb_gather_full / ggb_reshard / ggb_rmsnorm_fwd/bwd /
ggb_fused_elementwise_fwd/bwd / ggb_cross_entropy / ggb_loss / ggb_backward)
against the reference's own operators (pmm.hpp:76-401, called through
oracle/_ref on the one-rank grid).

Tolerances: contract (split-bf16 tcgen05, ~2^-16 per operand) and spmm
(fp32 FMA vs the reference's separate multiply-add) 1e-5 of the output scale;
RMSNorm / cross-entropy 1e-5 relative; dropout masks and the element-wise
backward bit-exact (same counter hash), the fused forward within one rounding
(FMA).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

X, Y, Z = 1, 2, 3


@pytest.fixture(scope="module")
def env(gg):
    import torch
    return gg.Context(), torch


def _blk(gg, t, layout):
    r, c = t.shape
    return gg.DeviceBlock(layout, r, c, np.array([0, r]), np.array([0, c]), t.data_ptr(), t.stride(0))


def _cuda(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("m,k,n", [(1000, 256, 256), (517, 100, 47), (64, 602, 256), (3, 5, 7), (2000, 256, 41)])
def test_contract(env, gg, ref, m, k, n):
    ctx, torch = env
    rng = np.random.default_rng(m + k + n)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = (rng.standard_normal((k, n)) * 0.1).astype(np.float32)
    ta, tb = _cuda(torch, a), _cuda(torch, b)
    tc = torch.full((m, n), float("nan"), device="cuda")
    gg.contract(ctx, _blk(gg, ta, (X, Y)), _blk(gg, tb, (Y, Z)), _blk(gg, tc, (X, Z)))
    ctx.synchronize()
    want = ref.contract(a, b)
    assert np.abs(tc.cpu().numpy() - want).max() <= 1e-5 * max(1.0, np.abs(want).max())


def test_contract_errors(env, gg):
    ctx, torch = env
    a = torch.zeros(4, 6, device="cuda")
    b = torch.zeros(6, 3, device="cuda")
    c = torch.zeros(4, 3, device="cuda")
    with pytest.raises(gg.CommContract):  # inner axes differ (pmm.hpp:101)
        gg.contract(ctx, _blk(gg, a, (X, Y)), _blk(gg, b, (Z, X)), _blk(gg, c, (X, Z)))
    with pytest.raises(gg.CommContract):  # output axes collide (pmm.hpp:104)
        gg.contract(ctx, _blk(gg, a, (X, Y)), _blk(gg, b, (Y, X)), _blk(gg, c, (X, Z)))
    with pytest.raises(gg.InvalidArgument):  # bad layout
        gg.contract(ctx, _blk(gg, a, (X, X)), _blk(gg, b, (X, Z)), _blk(gg, c, (X, Z)))


def test_spmm_on_a_batch_plane(env, gg, orc, ref):
    """spmm with the batch's own device CSR block (ggb_batch_csr_block) against
    the reference operator on the exported fp64 CSR."""
    ctx, torch = env
    n, b = 3000, 800
    ds = orc.generate_synthetic(n, 9.0, 8, 3, 5)
    g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, 3, 3)
    batch = gg.build_step_batch(ctx, g, b, 7, 2)
    for t in (False, True):
        a = gg.batch_csr_block(batch, 0, t)
        csr = batch.a_t(0) if t else batch.a(0)
        f = np.random.default_rng(1).standard_normal((b, 256)).astype(np.float32)
        tf = _cuda(torch, f)
        th = torch.full((b, 256), float("nan"), device="cuda")
        gg.spmm(ctx, a, gg.DeviceBlock((a.col_axis, Y), b, 256, np.array([0, b]), np.array([0, 256]), tf.data_ptr(),
                                       256),
                gg.DeviceBlock((a.row_axis, Y), b, 256, np.array([0, b]), np.array([0, 256]), th.data_ptr(), 256))
        ctx.synchronize()
        want = ref.spmm(csr, f)
        assert np.abs(th.cpu().numpy() - want).max() <= 1e-5 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("m,n", [(700, 256), (300, 100), (5, 512), (1, 3)])
def test_rmsnorm_fwd_bwd(env, gg, ref, m, n):
    ctx, torch = env
    rng = np.random.default_rng(m * n)
    x = rng.standard_normal((m, n)).astype(np.float32)
    gamma = (1 + 0.1 * rng.standard_normal(n)).astype(np.float32)
    dy = rng.standard_normal((m, n)).astype(np.float32)
    tx, tg, tdy = _cuda(torch, x), _cuda(torch, gamma), _cuda(torch, dy)
    ty, tdx = torch.empty(m, n, device="cuda"), torch.empty(m, n, device="cuda")
    trms, tdg = torch.empty(m, device="cuda"), torch.empty(n, device="cuda")
    gg.rmsnorm_fwd(ctx, _blk(gg, tx, (X, Y)), tg.data_ptr(), 1e-6, _blk(gg, ty, (X, Y)), trms.data_ptr())
    gg.rmsnorm_bwd(ctx, _blk(gg, tx, (X, Y)), tg.data_ptr(), trms.data_ptr(), _blk(gg, tdy, (X, Y)),
                   _blk(gg, tdx, (X, Y)), tdg.data_ptr())
    ctx.synchronize()
    y, rms, dx, dg = ref.rmsnorm(x, gamma, 1e-6, dy)
    for mine, want in ((ty, y), (trms, rms), (tdx, dx), (tdg, dg)):
        got = mine.cpu().numpy()
        assert np.abs(got - want).max() <= 1e-5 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("rate,training,res", [(0.1, True, True), (0.5, True, False), (0.3, False, True),
                                               (0.0, True, True)])
def test_fused_elementwise(env, gg, ref, rate, training, res):
    """out, the dropout mask (scale != 0) and dx bit-exact against the
    reference's fused_elementwise_fwd/bwd (pmm.hpp:299-341)."""
    ctx, torch = env
    m, n, key = 900, 256, 0x1234abcd
    rng = np.random.default_rng(7)
    x = rng.standard_normal((m, n)).astype(np.float32)
    h = rng.standard_normal((m, n)).astype(np.float32) if res else None
    dy = rng.standard_normal((m, n)).astype(np.float32)
    tx, tdy = _cuda(torch, x), _cuda(torch, dy)
    th = _cuda(torch, h) if res else None
    tout, tdx = torch.empty(m, n, device="cuda"), torch.empty(m, n, device="cuda")
    ldm = gg.mask_words(n)
    tbits = torch.zeros(m, ldm, dtype=torch.int32, device="cuda")
    gg.fused_elementwise_fwd(ctx, _blk(gg, tx, (X, Y)), _blk(gg, th, (X, Y)) if res else None, rate, key, training,
                             _blk(gg, tout, (X, Y)), tbits.data_ptr())
    gg.fused_elementwise_bwd(ctx, _blk(gg, tdy, (X, Y)), tbits.data_ptr(), gg.keep_scale(rate, training),
                             _blk(gg, tdx, (X, Y)))
    ctx.synchronize()
    out, scale, dx = ref.fused(x, h, rate, key, training, dy)
    # out = x * scale + h: one fused multiply-add here, a multiply then an add
    # in the reference -> within one rounding (the masks themselves are exact)
    got = tout.cpu().numpy()
    assert np.all(np.abs(got - out) <= 2 ** -23 * np.maximum(np.abs(out), np.abs(x * scale)) + 1e-30)
    assert np.array_equal(tdx.cpu().numpy(), dx)
    # the keep bits are scale != 0 (word 4j+i, bit l <-> column 128j + 4l + i)
    bits = tbits.cpu().numpy().view(np.uint32)
    cols = np.arange(n)
    word = 4 * (cols // 128) + cols % 4
    lane = (cols % 128) // 4
    mine = (bits[:, word] >> lane) & 1
    assert np.array_equal(mine.astype(bool), scale != 0)


def test_fused_elementwise_errors(env, gg):
    ctx, torch = env
    t = torch.zeros(4, 8, device="cuda")
    with pytest.raises(gg.InvalidArgument):  # pmm.hpp:304-305
        gg.fused_elementwise_fwd(ctx, _blk(gg, t, (X, Y)), None, 1.0, 1, True, _blk(gg, t, (X, Y)), None)
    r = torch.zeros(3, 8, device="cuda")
    with pytest.raises(gg.CommContract):  # residual layout mismatch (pmm.hpp:306-309)
        gg.fused_elementwise_fwd(ctx, _blk(gg, t, (X, Y)), _blk(gg, r, (X, Y)), 0.1, 1, True, _blk(gg, t, (X, Y)), None)


@pytest.mark.parametrize("m,n", [(600, 47), (100, 172), (2, 2), (33, 600)])
def test_cross_entropy(env, gg, ref, m, n):
    ctx, torch = env
    rng = np.random.default_rng(m + n)
    logits = (3 * rng.standard_normal((m, n))).astype(np.float32)
    labels = rng.integers(0, n, m).astype(np.int32)
    if m == 2:  # the reference's KAT: logits [0, 0] -> ln 2, grad -/+ 0.5 / B (test_pmm.cpp:462-520)
        logits[:] = 0
        labels[:] = [0, 1]
    tl, tlab = _cuda(torch, logits), _cuda(torch, labels)
    tg, tloss = torch.empty(m, n, device="cuda"), torch.empty(1, device="cuda")
    gg.cross_entropy(ctx, _blk(gg, tl, (X, Z)), tlab.data_ptr(), tloss.data_ptr(), _blk(gg, tg, (X, Z)))
    ctx.synchronize()
    loss, grad = ref.cross_entropy(logits, labels)
    assert abs(tloss.item() - loss) <= 1e-5 * abs(loss)
    assert np.abs(tg.cpu().numpy() - grad).max() <= 1e-6 * max(1.0, np.abs(grad).max()) + 1e-9


def test_transposed_gather_reshard_one_rank(env, gg):
    """On one rank: transposed is the exact transpose, gather_full the block,
    and reshard to another layout a copy (pure data movement)."""
    ctx, torch = env
    a = torch.randn(300, 77, device="cuda")
    t = torch.full((77, 300), float("nan"), device="cuda")
    gg.transposed(ctx, _blk(gg, a, (X, Y)), _blk(gg, t, (Y, X)))
    full = torch.full((300, 77), float("nan"), device="cuda")
    gg.gather_full(ctx, _blk(gg, a, (X, Y)), full.data_ptr(), 77)
    r = torch.full((300, 77), float("nan"), device="cuda")
    gg.reshard(ctx, _blk(gg, a, (X, Y)), _blk(gg, r, (Z, X)))
    ctx.synchronize()
    assert torch.equal(t, a.T) and torch.equal(full, a) and torch.equal(r, a)


def test_train_step_equals_forward_loss_backward(gg, orc):
    """train_step (model.hpp:459-478) split at the reference's seams: forward,
    parallel_cross_entropy (ggb_loss), backward — the same loss and gradients
    bit for bit."""
    n, d_in, ncls, b, seed = 2000, 12, 4, 600, 3
    ds = orc.generate_synthetic(n, 8.0, d_in, ncls, 6)
    ctx = gg.Context()
    g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls, 3)
    cfg = gg.ModelConfig(layers=3, d_in=d_in, d_h=64, d_out=ncls, dropout_rate=0.2)
    st_a, st_b = gg.init_state(ctx, cfg, seed), gg.init_state(ctx, cfg, seed)
    batch = gg.build_step_batch(ctx, g, b, gg.hash_combine(seed, 0), 1)
    la = gg.train_step(ctx, st_a, batch, gg.FP32, seed, 1)
    gg.forward(ctx, st_b, batch, gg.FP32, True, seed, 1)
    lb = gg.loss(ctx, st_b, batch)
    gg.backward(ctx, st_b, batch, gg.FP32)
    assert la == lb
    for x, y in zip(st_a.grads(), st_b.grads()):
        assert np.array_equal(x, y)
