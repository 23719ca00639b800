"""GPU parity of the sampler kernels through the C ABI: bit-exact against the
oracle restatement and against the reference compiled in place
(sampling.cpp:11-33, shardsample.cpp:47-156, model.hpp:250-309)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KATS = [
    ((100, 5, 7, 3), [7, 35, 43, 44, 54]),
    ((10, 3, 555, 0), [0, 1, 5]),
    ((1000, 8, 1, 0), [158, 205, 277, 528, 657, 698, 776, 817]),
    ((65536, 6, 1, 0), [6604, 10460, 16125, 24862, 36307, 55068]),
    ((2450000, 6, 9, 4), [809699, 840244, 883996, 2075223, 2216277, 2247394]),
    ((5, 5, 123, 0), [0, 1, 2, 3, 4]),
]


@pytest.mark.parametrize("args,want", KATS)
def test_sample_vertices_kat(gg, args, want):
    assert list(gg.sample_vertices(*args).vertices) == want


def test_sample_vertices_random_cases(gg, orc):
    rng = np.random.default_rng(0)
    cases = [(1, 1), (2, 1), (2, 2), (33, 33), (64, 63), (1000, 999), (4096, 1), (100000, 50000),
             (65536, 16384)]
    cases += [(int(n), int(rng.integers(1, n + 1))) for n in rng.integers(1, 5000, size=40)]
    for n, b in cases:
        seed, step = int(rng.integers(0, 2**63)), int(rng.integers(0, 1000))
        got = gg.sample_vertices(n, b, seed, step).vertices
        assert np.array_equal(got, orc.sample_vertices(n, b, seed, step)), (n, b, seed, step)


def test_sample_vertices_large(gg, orc):
    # products-shaped batch (C2): 612,500 of 2.45M
    got = gg.sample_vertices(2_450_000, 612_500, 9, 4).vertices
    assert np.array_equal(got, orc.sample_vertices(2_450_000, 612_500, 9, 4))


def test_sample_vertices_errors(gg):
    with pytest.raises(gg.InvalidArgument):
        gg.sample_vertices(10, 0, 0, 0)
    with pytest.raises(gg.InvalidArgument):
        gg.sample_vertices(10, 11, 0, 0)


def test_inclusion_frequency_uniform(gg):
    # test_sampling.cpp:41-53 (Monte Carlo), 20k draws on the GPU
    n, b, trials = 10, 3, 20000
    hits = np.zeros(n)
    for t in range(trials):
        hits[gg.sample_vertices(n, b, 555, t).vertices] += 1
    assert np.all(np.abs(hits / trials - 0.3) < 0.02)


def _graph(gg, ctx, ds, layers):
    return gg.Graph.from_csr(ctx, ds.n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels,
                             ds.n_classes, layers)


def _coord(dims, rank):
    r = rank
    z = r % dims[3]; r //= dims[3]
    y = r % dims[2]; r //= dims[2]
    x = r % dims[1]
    return (r // dims[1], x, y, z)


@pytest.mark.parametrize("dims", [(1, 1, 1, 1), (1, 2, 1, 1), (1, 2, 2, 1), (1, 2, 2, 2), (1, 3, 2, 2),
                                  (2, 2, 1, 1), (1, 1, 1, 3)])
def test_step_batch_bit_exact(gg, orc, ref, dims):
    """acceptance.cpp:93-160 on the GPU: every rank's StepBatch (sample,
    offsets, per-plane a_loc/a_t_loc with fp64 values, x_in, labels,
    counters) equals the reference's, with no communication."""
    n, b, layers = 3000, 700, 3
    ds = orc.generate_synthetic(n, 12.0, 10, 6, 3)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, 12.0, 3))
    try:
        grid = gg.DeviceGrid(*dims)
        for rank in range(grid.total()):
            ctx = gg.Context(grid, rank)
            g = _graph(gg, ctx, ds, layers)
            batch = None
            for seed, step in [(7, 4), (1, 0), (3, 9)]:
                gs = orc.hash_combine(seed, grid.dp_group(rank))
                want = ref.step_batch(h, dims, rank, layers, b, gs, step)
                batch = gg.build_step_batch(ctx, g, b, gs, step, reuse=batch)
                assert np.array_equal(batch.sample, want["sample"])
                for ax in (1, 2, 3):
                    assert np.array_equal(batch.batch_off(ax), want["batch_off"][ax])
                for p in range(3):
                    for t, mine in ((0, batch.a(p)), (1, batch.a_t(p))):
                        theirs = want["planes"][p][t]
                        assert list(theirs["dims"]) == [mine.n_rows, mine.n_cols, mine.nnz, mine.r0, mine.r1,
                                                        mine.c0, mine.c1]
                        c = theirs["csr"]
                        assert np.array_equal(mine.row_ptr, c.row_ptr)
                        assert np.array_equal(mine.col_idx, c.col_idx)
                        assert np.array_equal(mine.values.view(np.uint64), c.values.view(np.uint64))
                xd, x = batch.x_in
                assert list(xd) == list(want["x_in"][0])
                assert np.array_equal(x.view(np.uint32), want["x_in"][1].view(np.uint32))
                assert np.array_equal(batch.labels, want["labels"])
                assert [batch.nnz_extracted, batch.nnz_kept] == list(want["counters"])
            del batch, g, ctx
    finally:
        ref.free_dataset(h)


def test_step_batch_layers_and_edges(gg, orc, ref):
    """Fewer than three planes, b = n (identity sample), b = 2, empty rows."""
    n = 500
    ds = orc.generate_synthetic(n, 3.0, 4, 3, 21)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, 3.0, 21))
    try:
        for dims, layers, b in [((1, 1, 1, 1), 1, n), ((1, 2, 2, 2), 2, 2), ((1, 2, 1, 2), 1, 37)]:
            grid = gg.DeviceGrid(*dims)
            for rank in range(grid.total()):
                ctx = gg.Context(grid, rank)
                g = _graph(gg, ctx, ds, layers)
                want = ref.step_batch(h, dims, rank, layers, b, 5, 2)
                batch = gg.build_step_batch(ctx, g, b, 5, 2)
                assert batch.planes == len(want["planes"]) == min(layers, 3)
                for p in range(batch.planes):
                    for t, mine in ((0, batch.a(p)), (1, batch.a_t(p))):
                        c = want["planes"][p][t]["csr"]
                        assert np.array_equal(mine.row_ptr, c.row_ptr)
                        assert np.array_equal(mine.col_idx, c.col_idx)
                        assert np.array_equal(mine.values.view(np.uint64), c.values.view(np.uint64))
        with pytest.raises(gg.InvalidArgument):
            gg.build_step_batch(ctx, g, 1, 0, 0)  # build_local_minibatch: need 2 <= b <= N
    finally:
        ref.free_dataset(h)


def test_nonsymmetric_csr_uses_true_transpose(gg, orc):
    """A non-symmetric adjacency: a_t must be the stable transpose of a."""
    n, b = 400, 150
    rng = np.random.default_rng(3)
    rows, cols = rng.integers(0, n, 3000), rng.integers(0, n, 3000)
    key = np.unique(rows * n + cols)
    r, c = key // n, key % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    val = rng.random(len(key)) + 0.5
    adj = orc.Csr(n, n, rp, c.astype(np.int64), val)
    ctx = gg.Context(gg.DeviceGrid(1, 2, 2, 1), 3)
    feats = rng.standard_normal((n, 4)).astype(np.float32)
    g = gg.Graph.from_csr(ctx, n, rp, c, val, feats, np.zeros(n, np.int32), 2, 3, symmetric=False)
    batch = gg.build_step_batch(ctx, g, b, 9, 1)
    for p in range(3):
        a, at = batch.a(p), batch.a_t(p)
        # reference transpose: csr.cpp:74-94
        d = np.zeros((a.n_rows, a.n_cols))
        for i in range(a.n_rows):
            d[i, a.col_idx[a.row_ptr[i]:a.row_ptr[i + 1]]] = a.values[a.row_ptr[i]:a.row_ptr[i + 1]]
        dt = np.zeros((at.n_rows, at.n_cols))
        for i in range(at.n_rows):
            dt[i, at.col_idx[at.row_ptr[i]:at.row_ptr[i + 1]]] = at.values[at.row_ptr[i]:at.row_ptr[i + 1]]
        assert np.array_equal(d.T, dt)
        # and against the restatement for this rank's block
        lay = {0: (3, 1), 1: (2, 3), 2: (1, 2)}[p]
        co = _coord((1, 2, 2, 1), 3)
        ro_, co_ = orc.block_partition(n, (1, 2, 2, 1)[lay[0]]), orc.block_partition(n, (1, 2, 2, 1)[lay[1]])
        lb = orc.local_minibatch(adj, ro_[co[lay[0]]], ro_[co[lay[0]] + 1], co_[co[lay[1]]], co_[co[lay[1]] + 1],
                                 b, 9, 1)
        assert np.array_equal(lb.a.col_idx, a.col_idx) and np.array_equal(lb.a_t.col_idx, at.col_idx)
        assert np.array_equal(lb.a_t.values.view(np.uint64), at.values.view(np.uint64))


def test_native_generator_matches_reference(gg, ref):
    """ggb_graph_generate_synthetic == reference generate_synthetic (dataset.cpp:85-131)."""
    n, deg, d_in, ncls, seed = 5000, 14.0, 7, 5, 13
    h = ref.dataset_synthetic(n, deg, d_in, ncls, seed)
    try:
        want = ref.dataset_export(h)
        ctx = gg.Context()
        g = gg.Graph.generate_synthetic(ctx, n, deg, d_in, ncls, seed, 3)
        assert g.nnz == want.adj.nnz
        # compare through a batch with b = n: the identity sample exports the
        # full adjacency (values untouched on the diagonal, x1/p = x (n-1)/(n-1))
        batch = gg.build_step_batch(ctx, g, n, 0, 0)
        a = batch.a(0)
        assert np.array_equal(a.row_ptr, want.adj.row_ptr)
        assert np.array_equal(a.col_idx, want.adj.col_idx)
        assert np.array_equal(a.values.view(np.uint64), want.adj.values.view(np.uint64))
        _, x = batch.x_in
        assert np.array_equal(x.view(np.uint32), want.features.view(np.uint32))
        assert np.array_equal(batch.labels, want.labels)
    finally:
        ref.free_dataset(h)


# ---- the dataset generated on the device -----------------------------
@pytest.mark.parametrize("n,deg,d_in,ncls,seed", [(2, 1.0, 3, 2, 7), (50, 0.0, 4, 3, 1), (3000, 9.5, 17, 5, 7),
                                                  (65536, 30.52, 64, 16, 7)])
def test_device_generated_dataset_matches_generator(gg, orc, n, deg, d_in, ncls, seed):
    """generate_synthetic (dataset.cpp:85-150) on the GPU: normalized CSR
    (row_ptr, col_idx, fp64 values), labels and split tags bit-identical to
    the generator pinned to the reference; features the same polar sequence
    (fp64 log from CUDA: at most one fp32 ulp, in rare elements)."""
    ds = orc.generate_synthetic(n, deg, d_in, ncls, seed)
    ctx = gg.Context()
    g = gg.Graph.generate_synthetic_device(ctx, n, deg, d_in, ncls, seed, 3)
    (rp, ci, va), fe, la, sp = g.export()
    assert np.array_equal(rp, ds.adj.row_ptr) and np.array_equal(ci, ds.adj.col_idx)
    assert np.array_equal(va.view(np.uint64), ds.adj.values.view(np.uint64))
    assert np.array_equal(la, ds.labels) and np.array_equal(sp, ds.split)
    a, b = fe.view(np.int32).astype(np.int64), ds.features.view(np.int32).astype(np.int64)
    assert np.max(np.abs(a - b)) <= 1
    assert np.count_nonzero(a != b) <= max(1, a.size // 10000)


def test_device_generated_graph_trains_like_host_graph(gg, orc):
    """A device-built graph gives the same batches and losses as the host-built one."""
    n, deg, d_in, ncls, b, seed = 6000, 12.0, 24, 6, 1500, 3
    ctx = gg.Context()
    gh = gg.Graph.generate_synthetic(ctx, n, deg, d_in, ncls, seed, 3)
    gd = gg.Graph.generate_synthetic_device(ctx, n, deg, d_in, ncls, seed, 3)
    assert gd.nnz == gh.nnz
    cfg = gg.ModelConfig(layers=3, d_in=d_in, d_h=32, d_out=ncls, dropout_rate=0.1)
    sa, sb = gg.init_state(ctx, cfg, 1), gg.init_state(ctx, cfg, 1)
    for t in range(2):
        ba = gg.build_step_batch(ctx, gh, b, 5, t)
        bb = gg.build_step_batch(ctx, gd, b, 5, t)
        for p in range(3):
            x, y = ba.a(p), bb.a(p)
            assert np.array_equal(x.row_ptr, y.row_ptr) and np.array_equal(x.col_idx, y.col_idx)
            assert np.array_equal(x.values.view(np.uint64), y.values.view(np.uint64))
        assert np.array_equal(ba.labels, bb.labels)
        la = gg.train_step(ctx, sa, ba, gg.FP32, 1, t)
        lb = gg.train_step(ctx, sb, bb, gg.FP32, 1, t)
        assert abs(la - lb) <= 1e-5 * abs(la)


def test_graph_from_dataset_files(gg, orc, tmp_path):
    """a graph built from the reference's files (load_dataset)
    samples the same batches as one built from the in-memory dataset."""
    n, deg, d_in, ncls, seed = 4000, 8.0, 12, 5, 9
    p = [tmp_path / f"d.{e}" for e in ("edges", "sgnf", "sgnl", "sgns")]
    gg.Dataset.generate_synthetic(n, deg, d_in, ncls, seed).save(*p)
    ctx = gg.Context()
    g_file = gg.Dataset.load(*p).to_graph(ctx, 3)
    ds = orc.generate_synthetic(n, deg, d_in, ncls, seed)
    g_mem = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls, 3)
    a, b = gg.build_step_batch(ctx, g_file, 1000, 3, 2), gg.build_step_batch(ctx, g_mem, 1000, 3, 2)
    assert np.array_equal(a.a(0).col_idx, b.a(0).col_idx)
    assert np.array_equal(a.a(0).values.view(np.uint64), b.a(0).values.view(np.uint64))
    assert np.array_equal(a.x_in[1], b.x_in[1]) and np.array_equal(a.labels, b.labels)


def test_c2_batch_properties_at_full_size(gg):
    """BASELINE configs[1] at full size (2.45M vertices, 126M nonzeros, batch
    612,500): properties of the induced, rescaled batch adjacency that hold at
    any size — sorted distinct sample, canonical CSR, every self-loop kept,
    A == A^T bit for bit, nnz at its expectation, off-diagonal values
    = static value / p (fp64, exact) against the static CSR."""
    n, deg, b = 2_450_000, 50.53, 612_500
    ctx = gg.Context()
    g = gg.Graph.generate_synthetic_device(ctx, n, deg, 100, 47, 7, 3)
    (rp, ci, va), _, _, _ = g.export(features=False)
    bt = gg.build_step_batch(ctx, g, b, gg.hash_combine(1, 0), 3)
    s = bt.sample
    assert len(s) == b and s[0] >= 0 and s[-1] < n and np.all(np.diff(s) > 0)
    a = bt.a(0)
    assert a.row_ptr[0] == 0 and np.all(np.diff(a.row_ptr) >= 1)  # every row keeps its self-loop
    rows = np.repeat(np.arange(b), np.diff(a.row_ptr))
    cols = a.col_idx
    starts = a.row_ptr[:-1]
    first = np.zeros(len(cols), bool)
    first[starts] = True
    assert np.all((np.diff(cols) > 0) | first[1:])  # strictly increasing within rows
    nnz = len(cols)
    expect = b + (g.nnz - n) * (b / n) * ((b - 1) / (n - 1))
    assert abs(nnz - expect) <= 0.01 * expect
    # symmetric, values bit-identical: sort the transposed triples
    key = rows.astype(np.int64) * b + cols
    tkey = cols.astype(np.int64) * b + rows
    order = np.argsort(tkey, kind="stable")
    assert np.array_equal(key, tkey[order])
    assert np.array_equal(a.values.view(np.uint64), a.values[order].view(np.uint64))
    # rescale: off-diagonal entries = static value / p, diagonal unchanged
    p = (b - 1) / (n - 1)
    rng = np.random.default_rng(0)
    for k in rng.integers(0, nnz, 2000):
        u, v = int(s[rows[k]]), int(s[cols[k]])
        lo, hi = rp[u], rp[u + 1]
        pos = lo + np.searchsorted(ci[lo:hi], v)
        assert ci[pos] == v
        want = va[pos] if u == v else va[pos] / p
        assert np.float64(want).view(np.uint64) == np.float64(a.values[k]).view(np.uint64)


@pytest.mark.parametrize("n,b,reject_mod,seed", [(5000, 1000, 0, 1), (5000, 1000, 1 << 62, 3),
                                                 (100000, 20000, 25000, 7), (100000, 20000, 12000, 8),
                                                 (100000, 20000, 7000, 9), (20000, 20000, 900, 2),
                                                 (3000, 700, 3, 5)])
def test_rejected_draws_redrawn_exactly(gg, orc, n, b, reject_mod, seed):
    """next_below rejections (rng.hpp:38-45) shift every later draw's counter:
    the parallel re-draw passes (and the sequential replay beyond them) give
    the exact partial Fisher-Yates sample. A test-only rule (x % reject_mod
    == 0) makes rejections frequent: ~b / reject_mod per batch (0: none, up
    to hundreds, which takes the replay)."""
    ctx = gg.Context()
    out = np.empty(b, np.int64)
    gg.check(gg.lib().ggb_sample_vertices_test_reject(ctx.h, n, b, seed, 4, reject_mod, gg._ptr(out)))
    assert np.array_equal(out, orc.sample_vertices_reject(n, b, seed, 4, reject_mod))
    if reject_mod == 0:
        assert np.array_equal(out, orc.sample_vertices(n, b, seed, 4))
