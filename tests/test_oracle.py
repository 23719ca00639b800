"""CPU: pin the oracle restatement (oracle/oracle.c, oracle/oracle.py) to the
reference's own known answers and to the reference compiled in place."""
import numpy as np
import pytest

# Known answers from the reference's tests and from running it.
SAMPLE_KATS = [
    ((100, 5, 7, 3), [7, 35, 43, 44, 54]),
    ((10, 3, 555, 0), [0, 1, 5]),
    ((1000, 8, 1, 0), [158, 205, 277, 528, 657, 698, 776, 817]),
    ((65536, 6, 1, 0), [6604, 10460, 16125, 24862, 36307, 55068]),
    ((2450000, 6, 9, 4), [809699, 840244, 883996, 2075223, 2216277, 2247394]),
    ((5, 5, 123, 0), [0, 1, 2, 3, 4]),  # test_sampling.cpp:13-16
]


@pytest.mark.parametrize("args,want", SAMPLE_KATS)
def test_sample_vertices_kat(orc, args, want):
    assert list(orc.sample_vertices(*args)) == want


def test_sample_vertices_seed_plus_step(orc):
    # test_sampling.cpp:17-26: the per-step seed is seed + step
    assert np.array_equal(orc.sample_vertices(100, 10, 7, 4), orc.sample_vertices(100, 10, 11, 0))
    assert not np.array_equal(orc.sample_vertices(100, 10, 7, 3), orc.sample_vertices(100, 10, 7, 4))


def test_sample_vertices_errors(orc):
    with pytest.raises(ValueError):
        orc.sample_vertices(10, 0, 0, 0)
    with pytest.raises(ValueError):
        orc.sample_vertices(10, 11, 0, 0)


def test_rng_kats(orc):
    assert orc.splitmix64(0) == 0xE220A8397B1DCDAF
    assert orc.hash_combine(1, 0) == 0xE99FF867DBF682C9
    assert orc.element_unit(5, 0, 0) == 0.34388074042588201
    # bf16 RNE (test_comm.cpp:62-71)
    assert orc.bf16_round(0.1) == 0.10009765625
    assert orc.bf16_round(1.00390625) == 1.0
    assert orc.bf16_round(1.01171875) == 1.015625


def test_block_and_sample_partition(orc):
    # test_shardsample.cpp:34-39, 233-240
    assert list(orc.block_partition(10, 3)) == [0, 4, 7, 10]
    assert list(orc.block_partition(2, 3)) == [0, 1, 2, 2]
    s = np.array([1, 3, 6, 8])
    assert list(orc.sample_partition(s, np.array([0, 2, 4, 10]))) == [0, 1, 2, 4]


def test_rescale_kat(orc):
    # test_sampling.cpp:96-121 / test_shardsample.cpp:149-159: b=2, n=11 scales
    # off-diagonal values by 10 and leaves the diagonal bit-identical.
    rp = np.array([0, 2, 4] + [4] * 9, np.int64)
    col = np.array([0, 1, 0, 1], np.int64)
    val = np.array([0.5, 0.25, 0.25, 0.5])
    adj = orc.Csr(11, 11, rp, col, val)
    # find a (seed, step) whose sample is {0, 1}
    for step in range(2000):
        if list(orc.sample_vertices(11, 2, 3, step)) == [0, 1]:
            break
    else:
        pytest.skip("no step samples {0,1}")
    lb = orc.local_minibatch(adj, 0, 11, 0, 11, 2, 3, step)
    assert list(lb.a.values) == [0.5, 0.25 / 0.1, 0.25 / 0.1, 0.5]
    assert lb.a.values[0] == 0.5 and lb.a.values[3] == 0.5


def test_dataset_matches_reference(orc, ref):
    h = ref.dataset_synthetic(3000, 9.0, 12, 5, 11)
    try:
        want = ref.dataset_export(h)
    finally:
        ref.free_dataset(h)
    got = orc.generate_synthetic(3000, 9.0, 12, 5, 11)
    assert np.array_equal(got.adj.row_ptr, want.adj.row_ptr)
    assert np.array_equal(got.adj.col_idx, want.adj.col_idx)
    assert np.array_equal(got.adj.values.view(np.uint64), want.adj.values.view(np.uint64))
    assert np.array_equal(got.features.view(np.uint32), want.features.view(np.uint32))
    assert np.array_equal(got.labels, want.labels)
    assert np.array_equal(got.split, want.split)


LAY = {0: (3, 1), 1: (2, 3), 2: (1, 2)}  # adjacency_layout(p+1) = (row axis, col axis)


@pytest.mark.parametrize("dims", [(1, 1, 1, 1), (1, 2, 1, 1), (1, 2, 2, 1), (1, 2, 2, 2), (1, 3, 2, 2),
                                  (2, 2, 1, 1)])
def test_shard_extraction_matches_reference(orc, ref, dims):
    """acceptance.cpp:93-160 analogue for the restatement: every rank's plane
    blocks (a_loc and a_t_loc incl. fp64 values) equal build_step_batch's."""
    n, b = 1500, 400
    ds = orc.generate_synthetic(n, 10.0, 8, 4, 3)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, 10.0, 3))
    try:
        for rank in range(int(np.prod(dims))):
            gz, gy, gx = dims[3], dims[2], dims[1]
            r = rank
            z = r % gz; r //= gz
            y = r % gy; r //= gy
            x = r % gx; d = r // gx
            coord = (d, x, y, z)
            for seed, step in [(7, 4), (1, 0)]:
                gs = orc.hash_combine(seed, d)
                rb = ref.step_batch(h, dims, rank, 3, b, gs, step)
                ext = kept = 0
                for p in range(3):
                    ra, ca = LAY[p]
                    ro, co = orc.block_partition(n, dims[ra]), orc.block_partition(n, dims[ca])
                    lb = orc.local_minibatch(ds.adj, ro[coord[ra]], ro[coord[ra] + 1], co[coord[ca]],
                                             co[coord[ca] + 1], b, gs, step)
                    ext += lb.nnz_extracted
                    kept += lb.nnz_kept
                    for mine, theirs in ((lb.a, rb["planes"][p][0]["csr"]), (lb.a_t, rb["planes"][p][1]["csr"])):
                        assert np.array_equal(mine.row_ptr, theirs.row_ptr)
                        assert np.array_equal(mine.col_idx, theirs.col_idx)
                        assert np.array_equal(mine.values.view(np.uint64), theirs.values.view(np.uint64))
                assert list(rb["counters"]) == [ext, kept]
    finally:
        ref.free_dataset(h)


@pytest.mark.parametrize("cfg_kw", [
    dict(layers=3, d_h=32, dropout_rate=0.2),
    dict(layers=2, d_h=16, dropout_rate=0.0, use_rmsnorm=False, use_residual=False),
    dict(layers=4, d_h=24, dropout_rate=0.1, use_dropout=False),
])
def test_numpy_step_matches_reference(orc, ref, cfg_kw):
    n, d_in, ncls, b = 1200, 20, 5, 300
    ds = orc.generate_synthetic(n, 8.0, d_in, ncls, 3)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, 8.0, 3))
    try:
        cfg = orc.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw)
        ps = orc.init_params(cfg, 7)
        for a, w in zip(ps, ref.init_weights(cfg, 7)):
            assert np.array_equal(a, w)  # bit-exact init (model.hpp:139-149)
        res = orc.serial_train_step(cfg, ps, ds, b, 7, 4)
        losses, logits, grads, _ = ref.train(h, (1, 1, 1, 1), cfg, b, 7, step0=4)
        assert abs(res.loss - losses[0]) <= 1e-5 * max(1.0, abs(losses[0]))
        assert np.max(np.abs(res.logits - logits)) < 1e-4
        for g, w in zip(res.grads, grads):
            assert np.linalg.norm(g - w) <= 1e-5 * max(np.linalg.norm(w), 1e-12)
    finally:
        ref.free_dataset(h)


def test_numpy_adam_matches_reference(orc, ref):
    n, d_in, ncls, b = 1000, 16, 4, 250
    ds = orc.generate_synthetic(n, 8.0, d_in, ncls, 5)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, 8.0, 5))
    try:
        cfg = orc.ModelConfig(layers=3, d_in=d_in, d_h=16, d_out=ncls, dropout_rate=0.1)
        ps = orc.init_params(cfg, 1)
        ms = [np.zeros_like(p) for p in ps]
        vs = [np.zeros_like(p) for p in ps]
        L = []
        for t in range(4):
            r = orc.serial_train_step(cfg, ps, ds, b, 1, t)
            L.append(r.loss)
            orc.adam_step(ps, r.grads, ms, vs, t + 1)
        losses, _, _, W = ref.train(h, (1, 1, 1, 1), cfg, b, 1, 0, 4, optimizer=1, want_weights=True)
        assert np.allclose(L, losses, rtol=1e-5)
        for a, w in zip(ps, W):
            assert np.max(np.abs(a - w)) < 1e-6
    finally:
        ref.free_dataset(h)


def test_reference_comm_stats_accounting(orc, ref):
    """The accounting the GPU path is checked against (tests/test_gpu_commstats.py,
    tests/mgpu_worker.py): the reference's CommStats snapshot. Acceptance
    criterion 6 (Fig. 9): with a fixed PMM grid, per-group X bytes
    per step are exactly constant as G_d grows, D bytes follow the
    ring-equivalent rule, sampling is communication-free, and singleton groups
    charge nothing but still count their calls."""
    n, d_in, ncls, b, seed = 1200, 10, 5, 300, 4
    ds = orc.generate_synthetic(n, 8.0, d_in, ncls, 1)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, 8.0, 1))
    try:
        cfg = orc.ModelConfig(d_in=d_in, d_out=ncls, layers=2, d_h=32)
        one = ref.comm_stats(h, (1, 1, 1, 1), cfg, b, seed, 1)
        assert all(v == 0 for ax in one["bytes"].values() for v in ax.values())
        assert one["allreduce_calls"]["D"] == len(cfg.param_shapes())  # dp_sync: one per parameter view
        per_group = []
        for gd in (1, 2, 4):
            s = ref.comm_stats(h, (gd, 2, 1, 1), cfg, b // gd * gd, seed, 1)
            assert s["bytes"]["Y"] == s["bytes"]["Z"] == {p: 0 for p in s["bytes"]["Y"]}
            assert all(ax["sampling"] == 0 for ax in s["bytes"].values())
            per_group.append((s["bytes"]["X"]["forward"] // gd, s["bytes"]["X"]["backward"] // gd))
            dp = s["bytes"]["D"]["dp_sync"]
            # every rank all-reduces its parameter block over D: count * 4 * (gd-1)/gd each
            assert (dp == 0) if gd == 1 else (dp > 0)
        assert per_group[0] == per_group[1] == per_group[2]
    finally:
        ref.free_dataset(h)


def test_rmat_restatement_matches_python(orc):
    """orc_rmat_edges (restating gendata.cu k_rmat) against a pure-Python
    evaluation of the same quadrant descent on a small case."""
    scale, m, seed, a, b, c = 6, 200, 11, 0.57, 0.19, 0.19
    key = orc.hash_combine(seed, 0x7a3a7)
    want = []
    for e in range(m):
        ke = orc.hash_combine(key, e)
        u = v = 0
        for k in range(scale):
            x = (orc.splitmix64(orc.hash_combine(ke, k)) >> 11) * 2.0 ** -53
            bit = 1 << (scale - 1 - k)
            if x >= a + b + c:
                u |= bit
                v |= bit
            elif x >= a + b:
                u |= bit
            elif x >= a:
                v |= bit
        want.append((u, v))
    assert np.array_equal(orc.rmat_edges(scale, m, seed, a, b, c), np.array(want, np.int64))
