"""The device backward against the device forward by central differences —
the GPU analogue of the reference's gradient oracle finite_difference_check
(model.hpp:749-786; acceptance criterion 4, acceptance.cpp:311-320).

The reference checks every element in fp64 (h = 1e-5, max rel < 1e-6). The
device path computes in fp32 / split-bf16 forwards and a bf16-operand
backward, so the check is stated as directional derivatives: for random unit
directions D over all parameters (the gradient direction plus a random
one), (L(W + hD) - L(W - hD)) / 2h must match
<g, D> within the north-star gradient tolerance (rel 1e-2), for a spread of
h (the difference quotient's truncation error shrinks with h, its rounding
error grows). Dropout is off so L is a deterministic function of W, as the
reference requires. Also checks the same thing per parameter tensor (D
supported on one tensor), so a wrong gradient of any single block fails.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _loss_at(gg, ctx, st, batch, seed, weights):
    for i, w in enumerate(weights):
        st.set_weight(i, w)
    gg.forward(ctx, st, batch, gg.FP32, True, seed, 0)
    return float(gg.loss(ctx, st, batch))


@pytest.mark.parametrize("cfg_kw", [dict(layers=3, d_h=64, use_dropout=False, dropout_rate=0.0),
                                    dict(layers=2, d_h=256, use_dropout=False, dropout_rate=0.0),
                                    dict(layers=3, d_h=32, use_dropout=False, dropout_rate=0.0,
                                         use_rmsnorm=False)])
def test_directional_derivatives_match_gradient(gg, orc, cfg_kw):
    n, d_in, ncls, b, seed = 3000, 24, 7, 900, 41
    ds = orc.generate_synthetic(n, 10.0, d_in, ncls, 3)
    ctx = gg.Context()
    g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls,
                          cfg_kw["layers"])
    cfg = gg.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw)
    st = gg.init_state(ctx, cfg, seed)
    batch = gg.build_step_batch(ctx, g, b, gg.hash_combine(seed, 0), 0)
    gg.train_step(ctx, st, batch, gg.FP32, seed, 0)
    grads = [x.astype(np.float64) for x in st.grads()]
    w0 = [x.copy() for x in st.weights()]
    rng = np.random.default_rng(5)

    def check(dirs, label):
        norm = np.sqrt(sum(float(np.sum(d * d)) for d in dirs))
        dirs = [d / norm for d in dirs]
        want = sum(float(np.sum(gr * d)) for gr, d in zip(grads, dirs))
        best = None
        for h in (3e-2, 1e-2, 3e-3):
            lp = _loss_at(gg, ctx, st, batch, seed, [w + (h * d).astype(np.float32) for w, d in zip(w0, dirs)])
            lm = _loss_at(gg, ctx, st, batch, seed, [w - (h * d).astype(np.float32) for w, d in zip(w0, dirs)])
            fd = (lp - lm) / (2 * h)
            rel = abs(fd - want) / max(abs(want), 1e-6)
            best = rel if best is None else min(best, rel)
        assert best <= 1e-2, (label, want, best)

    # all parameters at once: the gradient direction plus a random one of the
    # same norm (so <g, D> stays well away from zero while D probes every
    # element), three draws
    gnorm = np.sqrt(sum(float(np.sum(gr * gr)) for gr in grads))
    for k in range(3):
        r = [rng.standard_normal(w.shape) for w in w0]
        rnorm = np.sqrt(sum(float(np.sum(x * x)) for x in r))
        check([gr / gnorm + x / rnorm for gr, x in zip(grads, r)], f"all/{k}")
    # one tensor at a time, the direction along its own gradient (so <g, D>
    # is that tensor's gradient norm, well away from zero)
    for i, gr in enumerate(grads):
        if float(np.sum(gr * gr)) == 0.0:
            continue
        check([gr if j == i else np.zeros_like(w) for j, w in enumerate(w0)], f"tensor {i}")
    for i, w in enumerate(w0):  # leave the state as it was
        st.set_weight(i, w)
