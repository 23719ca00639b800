"""R-MAT input (BASELINE configs[0]: RMAT 2^16 vertices / ~1M edges, 64
features, 3-layer GCN hidden 128): the device R-MAT generator against its C
restatement (oracle.c orc_rmat_edges), the dataset it yields against the
reference's own loader (load_dataset, dataset.cpp:178-239, fed the files our
writers produce), and the GCN step on this skewed graph (max degree ~10K,
29% isolated vertices) against the reference: the batch bit-exact, three
Adam steps of train_run's loop within the north-star tolerances."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCALE, EDGES, D_IN, NCLS, SEED = 16, 1 << 20, 64, 16, 7


@pytest.fixture(scope="module")
def ctx(gg):
    return gg.Context()


@pytest.mark.parametrize("scale,m,seed,abc", [(16, 1 << 20, 7, (0.57, 0.19, 0.19)), (5, 300, 1, (0.57, 0.19, 0.19)),
                                              (10, 5000, 3, (0.25, 0.25, 0.25)), (12, 20000, 9, (0.45, 0.15, 0.3))])
def test_rmat_edges_match_oracle(gg, orc, ctx, scale, m, seed, abc):
    mine = gg.rmat_edges(ctx, scale, m, seed, *abc)
    want = orc.rmat_edges(scale, m, seed, *abc)
    assert np.array_equal(mine, want)
    assert mine.min() >= 0 and mine.max() < (1 << scale)


def test_rmat_is_skewed(gg, ctx):
    uv = gg.rmat_edges(ctx, SCALE, EDGES, SEED)
    deg = np.bincount(uv.ravel(), minlength=1 << SCALE)
    assert deg.max() > 100 * deg.mean()  # power-law hubs
    assert (deg == 0).sum() > (1 << SCALE) // 10  # and many isolated vertices


def test_rmat_files_load_identically_in_the_reference(gg, orc, ref, ctx, tmp_path):
    """Our dataset, written with our SGN*/edge-list writers, is read back by
    the reference's load_dataset into the same normalized CSR, features,
    labels and split; and our own builder equals the oracle's."""
    ds = gg.Dataset.generate_rmat(ctx, 12, 1 << 16, 16, 8, SEED)
    files = [tmp_path / f"r.{x}" for x in ("edges", "sgnf", "sgnl", "sgns")]
    ds.save(*files)
    (rp, ci, va), fe, la, sp, uv = ds.arrays()
    (rrp, rci, rva), rfe, rla, rsp, rncls = ref.load_files(*files)
    assert rncls == 8
    assert np.array_equal(rp, rrp) and np.array_equal(ci, rci)
    assert np.array_equal(va.view(np.uint64), rva.view(np.uint64))
    assert np.array_equal(fe.view(np.uint32), rfe.view(np.uint32))
    assert np.array_equal(la, rla) and np.array_equal(sp, rsp)
    o = orc.dataset_from_edges(1 << 12, uv, 16, 8, SEED)
    assert np.array_equal(o.adj.row_ptr, rp) and np.array_equal(o.adj.col_idx, ci)
    assert np.array_equal(o.labels, la)


@pytest.fixture(scope="module")
def c1r(gg, orc, ref, ctx):
    ds = gg.Dataset.generate_rmat(ctx, SCALE, EDGES, D_IN, NCLS, SEED)
    (rp, ci, va), fe, la, sp, uv = ds.arrays()
    n = 1 << SCALE
    h = ref.dataset_from(orc.Dataset(n, D_IN, NCLS, orc.Csr(n, n, rp, ci, va), fe, la, sp), uv)
    g = ds.to_graph(ctx, 3)
    yield ds, h, g
    ref.free_dataset(h)


@pytest.mark.parametrize("dims", [(1, 1, 1, 1), (1, 2, 2, 2)])
def test_rmat_batch_bit_exact(gg, ref, ctx, c1r, dims):
    """build_step_batch on the R-MAT graph: the 1x1x1x1 batch against ours,
    and every plane block of rank 0 of a 2x2x2 reference grid against the
    same rows / columns cut from our batch's sample."""
    ds, h, g = c1r
    b, gs, step = (1 << SCALE) // 4, gg.hash_combine(1, 0), 3
    want = ref.step_batch(h, dims, 0, 3, b, gs, step)
    batch = gg.build_step_batch(ctx, g, b, gs, step)
    assert np.array_equal(batch.sample, want["sample"])
    if dims != (1, 1, 1, 1):
        return
    assert (batch.nnz_extracted, batch.nnz_kept) == tuple(int(x) for x in want["counters"])
    for p in range(3):
        for t, mine in ((0, batch.a(p)), (1, batch.a_t(p))):
            w = want["planes"][p][t]["csr"]
            assert np.array_equal(mine.row_ptr, w.row_ptr) and np.array_equal(mine.col_idx, w.col_idx)
            assert np.array_equal(mine.values.view(np.uint64), w.values.view(np.uint64))
    assert np.array_equal(batch.x_in[1], want["x_in"][1])
    rows = np.diff(batch.a(0).row_ptr)
    assert rows.max() > 50 * max(rows.mean(), 1)  # the batch keeps the skew


def test_rmat_c1_adam_run_matches_reference(gg, orc, ref, ctx, c1r):
    """BASELINE configs[0] on R-MAT: three steps of train_run's loop (batch ->
    train_step -> dp_sync -> Adam), hidden 128, batch N/4: per-step losses
    rel <= 1e-3, final weights within 5e-2 of the reference's update."""
    ds, h, g = c1r
    b, seed = (1 << SCALE) // 4, 1
    cfg_kw = dict(layers=3, d_h=128, dropout_rate=0.1)
    st = gg.init_state(ctx, gg.ModelConfig(d_in=D_IN, d_out=NCLS, **cfg_kw), seed)
    got, batch = [], None
    for t in range(3):
        batch = gg.build_step_batch(ctx, g, b, gg.hash_combine(seed, 0), t, reuse=batch)
        got.append(gg.train_step(ctx, st, batch, gg.FP32, seed, t))
        if t == 0:
            grads0 = st.grads()
        gg.dp_sync(ctx, st)
        gg.optimizer_step(ctx, st, gg.ADAM, 1e-3)
    ocfg = orc.ModelConfig(d_in=D_IN, d_out=NCLS, **cfg_kw)
    _, _, rgrads0, _ = ref.train(h, (1, 1, 1, 1), ocfg, b, seed, 0, 1, want_logits=False)
    for mine, want in zip(grads0, rgrads0):
        assert np.linalg.norm(mine - want) <= 1e-2 * np.linalg.norm(want)
    losses, _, _, W = ref.train(h, (1, 1, 1, 1), ocfg, b, seed, 0, 3, optimizer=1, want_logits=False,
                                want_weights=True)
    assert np.all(np.abs(np.array(got) - losses) <= 1e-3 * np.abs(losses)), (got, losses)
    for mine, want, w0 in zip(st.weights(), W, ref.init_weights(ocfg, seed)):
        assert np.linalg.norm(mine.astype(np.float64) - want) <= 5e-2 * np.linalg.norm(want.astype(np.float64) - w0)
