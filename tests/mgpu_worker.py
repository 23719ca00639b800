"""Multi-GPU parity worker (launched by tests/test_multigpu.py under torchrun,
one process per GPU): every rank builds its shard of the same dataset, runs
train_step (PMM grids) or a few Adam steps (data-parallel grids) through
libggb with NCCL communicators, and rank 0 compares with the reference
compiled in place (oracle/_ref): sharded == serial, as acceptance.cpp:270-285
and test_model.cpp:136-191 check for the reference itself.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2604_02651_b200 import gridgnn as gg  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("GGB_WATCHDOG_S", "150")), exit=True)
    dims = tuple(int(x) for x in sys.argv[1].split("x"))
    prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    # the reference knows kFp32 and kBf16Roundtrip; the NCCL bf16 sum (2) is
    # checked against kBf16Roundtrip with the bf16-communication tolerance
    ref_prec = min(prec, 1)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    obj = [gg.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    grid = gg.DeviceGrid(*dims)
    assert grid.total() == world
    ctx = gg.Context(grid, rank, device=local, nccl_uid=obj[0])

    n, d_in, ncls, b, seed = 3000, 20, 7, 900, 5
    ds = O.generate_synthetic(n, 10.0, d_in, ncls, 3)
    g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls, 3,
                          split=ds.split)
    cfg_kw = dict(layers=3, d_h=64, dropout_rate=0.1)
    cfg = gg.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw)
    st = gg.init_state(ctx, cfg, seed)
    gs = gg.hash_combine(seed, grid.dp_group(rank))
    result = {}
    if dims[0] == 1:
        batch = gg.build_step_batch(ctx, g, b, gs, 2)
        loss = gg.train_step(ctx, st, batch, prec, seed, 2)
        blocks = [(bl.name, (bl.r0, bl.r1, bl.c0, bl.c1), gr.tolist()) for bl, gr in zip(st.blocks, st.grads())]
        ldims, lg = st.logits()
        result = {"loss": loss, "grads": blocks, "logits": (ldims, lg.tolist())}
    else:
        losses = []
        batch = None
        for t in range(3):
            batch = gg.build_step_batch(ctx, g, b, gs, t, reuse=batch)
            losses.append(gg.train_step(ctx, st, batch, prec, seed, t))
            gg.dp_sync(ctx, st)
            gg.optimizer_step(ctx, st, gg.ADAM, 1e-3)
        blocks = [(bl.name, (bl.r0, bl.r1, bl.c0, bl.c1), w.tolist()) for bl, w in zip(st.blocks, st.weights())]
        result = {"losses": losses, "weights": blocks}
    # evaluate_full_graph on the grid (model.hpp:493-537): counts identical on every rank
    ev = gg.build_eval_batch(ctx, g, seed)
    counts = gg.evaluate_full_graph(ctx, st, ev, g, prec)
    result["eval"] = (counts.correct, counts.total)
    # CommStats (comm.hpp:385-403): the byte accounting of 2 train_run steps +
    # one evaluation, summed over the grid, vs the reference's snapshot
    ctx.comm_stats(reset=True)
    sb = None
    for t in range(2):
        sb = gg.build_step_batch(ctx, g, b, gs, t, reuse=sb)
        gg.train_step(ctx, st, sb, prec, seed, t)
        gg.dp_sync(ctx, st)
        gg.optimizer_step(ctx, st, gg.ADAM, 1e-3)
    gg.evaluate_full_graph(ctx, st, ev, g, prec)
    stats = ctx.comm_stats(grid_total=True)
    gathered = [None] * world
    dist.all_gather_object(gathered, result)
    if rank == 0:
        R = O.Ref()
        h = R.dataset_from(ds, O.synthetic_edges(n, 10.0, 3))
        ocfg = O.ModelConfig(d_in=d_in, d_out=ncls, **cfg_kw)
        ok, report = True, {}
        # bf16 wire (Precision::kBf16Roundtrip): contributions rounded to bf16
        # at every PMM all-reduce; rounding of values within an ulp of a bf16
        # boundary can go either way vs the reference, flipping ReLU/dropout
        # decisions downstream -> the fast-mode tolerance applies
        grad_tol, logit_tol = (1e-2, 2e-2) if prec == 0 else (6e-2, 5e-2)
        if dims[0] == 1:
            losses, logits, grads, _ = R.train(h, (1, 1, 1, 1), ocfg, b, seed, step0=2, prec=ref_prec)
            lrel = max(abs(r["loss"] - losses[0]) / abs(losses[0]) for r in gathered)
            ok &= lrel <= 1e-3
            shapes = [s for _, s in ocfg.param_shapes()]
            worst = 0.0
            for pi, want in enumerate(grads):
                full = np.zeros(shapes[pi], np.float32)
                for r in gathered:
                    name, (r0, r1, c0, c1), gv = r["grads"][pi]
                    gv = np.asarray(gv, np.float32)
                    if len(shapes[pi]) == 1:
                        full[c0:c1] = gv
                    else:
                        full[r0:r1, c0:c1] = gv.reshape(r1 - r0, c1 - c0)
                rel = np.linalg.norm(full - want) / max(np.linalg.norm(want), 1e-30)
                worst = max(worst, rel)
            ok &= worst <= grad_tol
            full_lg = np.zeros_like(logits)
            for r in gathered:
                (r0, r1, c0, c1), lg = r["logits"]
                full_lg[r0:r1, c0:c1] = np.asarray(lg, np.float32).reshape(r1 - r0, c1 - c0)
            ldev = float(np.max(np.abs(full_lg - logits)))
            ok &= ldev <= logit_tol * max(1.0, float(np.max(np.abs(logits))))
            report = {"loss_rel": lrel, "grad_rel_worst": worst, "logits_maxdev": ldev}
        else:
            losses, _, _, W = R.train(h, dims, ocfg, b, seed, 0, 3, prec=ref_prec, optimizer=1, want_weights=True)
            # rank 0 of DP group 0 reports group-0 losses; compare the group-0 ranks
            lrel = max(abs(a - w) / abs(w) for a, w in zip(gathered[0]["losses"], losses))
            ok &= lrel <= 1e-3
            worst = 0.0
            for pi, want in enumerate(W):
                for r in gathered:
                    name, (r0, r1, c0, c1), wv = r["weights"][pi]
                    wv = np.asarray(wv, np.float32)
                    ref_blk = want[c0:c1] if want.ndim == 1 else want[r0:r1, c0:c1]
                    wv = wv.reshape(ref_blk.shape)
                    worst = max(worst, np.linalg.norm(wv - ref_blk) / max(np.linalg.norm(ref_blk), 1e-30))
            ok &= worst <= 1e-3
            report = {"loss_rel": lrel, "weight_rel_worst": worst}
        # eval: PMM grids evaluate the initial weights, DP grids the 3 Adam steps
        want, want_lg = R.train_eval(h, n, dims, ocfg, b, seed, n_steps=0 if dims[0] == 1 else 3, prec=ref_prec,
                                     optimizer=1, lr=1e-3)
        evs = [r["eval"] for r in gathered]
        ok &= all(e == evs[0] for e in evs)
        top2 = np.sort(want_lg, axis=1)[:, -2:]
        slack = int(np.sum(top2[:, 1] - top2[:, 0] <= 2 * (1e-3 if prec == 0 else logit_tol) * max(1.0, float(np.max(np.abs(want_lg))))))
        ok &= tuple(evs[0][1]) == tuple(int(x) for x in want[3:])
        ev_dev = max(abs(evs[0][0][s] - int(want[s])) for s in range(3))
        ok &= ev_dev <= slack
        report.update(eval_correct_dev=ev_dev, eval_slack=slack)
        want_stats = R.comm_stats(h, dims, ocfg, b, seed, 2, prec=ref_prec, evaluate=True)
        stats_ok = stats == want_stats
        if not stats_ok:
            print(json.dumps({"comm_stats": stats, "want": want_stats}), flush=True)
        ok &= stats_ok
        report.update(comm_stats_equal=stats_ok,
                      comm_bytes_total=sum(v for ax in stats["bytes"].values() for v in ax.values()))
        R.free_dataset(h)
        report = {k: float(v) for k, v in report.items()}
        print(json.dumps({"grid": dims, "prec": prec, "ok": bool(ok), **report}), flush=True)
        code = 0 if ok else 1
    else:
        code = 0
    dist.barrier()
    ctx.close()
    sys.exit(code)


if __name__ == "__main__":
    main()
