"""CommStats accounting (comm.hpp:75-117, 385-403) against the reference's own
counters: every logical collective of the train_run step loop (train_step's
forward / backward phases, dp_sync, evaluate_full_graph) is charged with the
reference's model at the reference's call sites, whatever this
implementation fuses, skips or replaces. On one GPU every group is a
singleton, so the bytes are 0 and the call counters carry the check (they
advance for singleton groups too); the sharded byte columns are checked
against the reference on 2 and 4 GPUs in tests/mgpu_worker.py.
"""
import pytest

pytestmark = pytest.mark.gpu


def _run(gg, ctx, g, cfg, b, seed, steps, prec, evaluate):
    st = gg.init_state(ctx, cfg, seed)
    ctx.comm_stats(reset=True)
    gs = gg.hash_combine(seed, 0)
    batch = None
    for t in range(steps):
        batch = gg.build_step_batch(ctx, g, b, gs, t, reuse=batch)
        gg.train_step(ctx, st, batch, prec, seed, t)
        gg.dp_sync(ctx, st)
        gg.optimizer_step(ctx, st, gg.ADAM, 1e-3)
    if evaluate:
        gg.evaluate_full_graph(ctx, st, gg.build_eval_batch(ctx, g, seed), g, prec)
    return ctx.comm_stats(grid_total=True)


@pytest.mark.parametrize("cfg_kw", [dict(layers=3, d_h=64, dropout_rate=0.1),
                                    dict(layers=2, d_h=32, dropout_rate=0.0, use_rmsnorm=False),
                                    dict(layers=4, d_h=48, dropout_rate=0.2, use_residual=False)])
@pytest.mark.parametrize("preagg", ["1", "0"])
def test_comm_stats_match_reference(gg, orc, ref, monkeypatch, cfg_kw, preagg):
    monkeypatch.setenv("GGB_PREAGG", preagg)
    n, d_in, ncls, b, seed = 2000, 12, 5, 600, 7
    ds = orc.generate_synthetic(n, 8.0, d_in, ncls, 2)
    h = ref.dataset_from(ds, orc.synthetic_edges(n, 8.0, 2))
    ctx = gg.Context(gg.DeviceGrid(1, 1, 1, 1), 0)
    try:
        g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls,
                              cfg_kw["layers"], split=ds.split)
        cfg = gg.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw)
        for steps, evaluate in ((2, False), (1, True)):
            got = _run(gg, ctx, g, cfg, b, seed, steps, gg.FP32, evaluate)
            want = ref.comm_stats(h, (1, 1, 1, 1), orc.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw), b, seed, steps,
                                  evaluate=evaluate)
            assert got == want
            assert all(v == 0 for ax in got["bytes"].values() for v in ax.values())
    finally:
        ref.free_dataset(h)
        ctx.close()


def test_comm_stats_reset_and_phases(gg, orc):
    n, d_in, ncls = 1500, 8, 4
    ds = orc.generate_synthetic(n, 6.0, d_in, ncls, 1)
    ctx = gg.Context(gg.DeviceGrid(1, 1, 1, 1), 0)
    try:
        g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls, 2,
                              split=ds.split)
        st = gg.init_state(ctx, gg.ModelConfig(d_in=d_in, d_out=ncls, layers=2, d_h=16), 3)
        ctx.comm_stats(reset=True)
        assert sum(ctx.comm_stats()["allreduce_calls"].values()) == 0
        gg.dp_sync(ctx, st)  # one D-axis all-reduce per parameter view (model.hpp:428-429)
        s = ctx.comm_stats(reset=True)
        assert s["allreduce_calls"] == {"D": len(st.blocks), "X": 0, "Y": 0, "Z": 0}
        assert ctx.comm_stats()["allreduce_calls"]["D"] == 0
    finally:
        ctx.close()
