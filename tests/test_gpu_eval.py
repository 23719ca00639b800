"""GPU parity of evaluate_full_graph (model.hpp:493-537), the per-epoch
full-graph evaluation of train_run (model.hpp:621-626,686-688), against the
reference compiled in place.

The eval batch is build_step_batch(b = n, seed, step 0): every vertex, p = 1.
Bars:
  eval logits   max |diff| <= 2e-2 * max(1, max |logit|) (forward tolerance)
  counts        equal to the reference's, except rows whose top-2 logit
                margin is inside that tolerance (an argmax there may go
                either way): |correct - ref| <= #near-tie rows; totals exact
  ties          all-equal logits predict class 0 (lowest id, model.hpp:503-508)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(gg, orc, ref, n, deg, d_in, ncls, data_seed, layers):
    ds = orc.generate_synthetic(n, deg, d_in, ncls, data_seed)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, deg, data_seed))
    ctx = gg.Context(gg.DeviceGrid(1, 1, 1, 1), 0)
    g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls,
                          layers, split=ds.split)
    return ds, h, ctx, g


def _train(gg, ctx, g, st, b, seed, steps, lr=1e-2):
    gs = gg.hash_combine(seed, 0)
    batch = None
    for t in range(steps):
        batch = gg.build_step_batch(ctx, g, b, gs, t, reuse=batch)
        gg.train_step(ctx, st, batch, gg.FP32, seed, t)
        gg.dp_sync(ctx, st)
        gg.optimizer_step(ctx, st, gg.ADAM, lr)


def _near_ties(logits, tol):
    top2 = np.sort(logits, axis=1)[:, -2:]
    return int(np.sum(top2[:, 1] - top2[:, 0] <= tol))


@pytest.mark.parametrize("cfg_kw,steps", [(dict(layers=3, d_h=64, dropout_rate=0.1), 4),
                                          (dict(layers=2, d_h=32, dropout_rate=0.0, use_rmsnorm=False), 2),
                                          (dict(layers=4, d_h=48, dropout_rate=0.2, use_residual=False), 3)])
def test_evaluate_full_graph_matches_reference(gg, orc, ref, cfg_kw, steps):
    n, d_in, ncls, b, seed = 3000, 16, 5, 800, 11
    ds, h, ctx, g = _setup(gg, orc, ref, n, 9.0, d_in, ncls, 4, cfg_kw["layers"])
    try:
        st = gg.init_state(ctx, gg.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw), seed)
        _train(gg, ctx, g, st, b, seed, steps, lr=1e-3)
        ev = gg.build_eval_batch(ctx, g, seed)
        got = gg.evaluate_full_graph(ctx, st, ev, g)
        _, lg = st.logits()
        want, want_lg = ref.train_eval(h, n, (1, 1, 1, 1), orc.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw), b, seed,
                                       n_steps=steps, optimizer=1, lr=1e-3)
        tol = 2e-2 * max(1.0, float(np.max(np.abs(want_lg))))
        assert np.max(np.abs(lg - want_lg)) <= tol
        assert got.total == tuple(int(x) for x in want[3:])
        assert sum(got.total) == int(np.sum(ds.split < 3))
        slack = _near_ties(want_lg, 2 * tol)
        for s in range(3):
            assert abs(got.correct[s] - int(want[s])) <= slack, (got, want, slack)
        # the argmax itself, on rows with a clear winner
        clear = np.sort(want_lg, axis=1)[:, -1] - np.sort(want_lg, axis=1)[:, -2] > 2 * tol
        assert np.array_equal(np.argmax(lg[clear], axis=1), np.argmax(want_lg[clear], axis=1))
        assert 0.0 <= got.accuracy(0) <= 1.0
    finally:
        ref.free_dataset(h)


def test_evaluate_ties_go_to_lowest_class(gg, orc, ref):
    n, d_in, ncls = 1200, 8, 6
    ds, h, ctx, g = _setup(gg, orc, ref, n, 6.0, d_in, ncls, 2, 2)
    try:
        cfg = gg.ModelConfig(d_in=d_in, d_out=ncls, layers=2, d_h=16, dropout_rate=0.1)
        st = gg.init_state(ctx, cfg, 3)
        wout = len(st.blocks) - 1
        st.set_weight(wout, np.zeros_like(st.weights()[wout]))  # every logit 0
        counts = gg.evaluate_full_graph(ctx, st, gg.build_eval_batch(ctx, g, 3), g)
        for s in range(3):
            sel = ds.split == s
            assert counts.total[s] == int(sel.sum())
            assert counts.correct[s] == int(np.sum(ds.labels[sel] == 0))
    finally:
        ref.free_dataset(h)


def test_generated_graph_carries_split(gg, orc):
    n = 5000
    ctx = gg.Context(gg.DeviceGrid(1, 1, 1, 1), 0)
    g = gg.Graph.generate_synthetic(ctx, n, 8.0, 8, 4, 7, 2)
    ds = orc.generate_synthetic(n, 8.0, 8, 4, 7)
    st = gg.init_state(ctx, gg.ModelConfig(d_in=8, d_out=4, layers=2, d_h=16), 1)
    counts = gg.evaluate_full_graph(ctx, st, gg.build_eval_batch(ctx, g, 1), g)
    assert counts.total == tuple(int(np.sum(ds.split == s)) for s in range(3))


def test_evaluate_contract_errors(gg, orc, ref):
    n, d_in, ncls = 800, 8, 4
    ds, h, ctx, g = _setup(gg, orc, ref, n, 6.0, d_in, ncls, 2, 2)
    try:
        st = gg.init_state(ctx, gg.ModelConfig(d_in=d_in, d_out=ncls, layers=2, d_h=16), 1)
        small = gg.build_step_batch(ctx, g, 100, 1, 0)
        with pytest.raises(gg.InvalidArgument):
            gg.evaluate_full_graph(ctx, st, small, g)  # not the b = n eval batch
        g2 = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls, 2)
        with pytest.raises(gg.InvalidArgument):
            gg.evaluate_full_graph(ctx, st, gg.build_eval_batch(ctx, g2, 1), g2)  # no split tags
        with pytest.raises(gg.InvalidArgument):
            g2.set_split(np.full(n, 4, np.uint8))  # invalid tag (dataset.cpp:225)
    finally:
        ref.free_dataset(h)
