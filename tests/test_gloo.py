"""CPU, world size 2 over gloo: the host-side logic of the N>1 path.

* the NCCL unique-id hand-off bench.py / mgpu_worker.py use (bytes broadcast);
* communication-free sampling: every rank derives its plane blocks on its own
  (Alg. 2, here through the oracle restatement) and the blocks gathered from
  the ranks reassemble the serial mini-batch exactly (acceptance.cpp:93-160);
* the product's layout algebra (gridgnn.py, mirroring pmm.hpp:31-63) tiles
  every activation exactly once per replica set on the 2-rank grids;
* max-over-ranks step timing as bench.py reduces it.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    from oracle import oracle as O
    from paper_2604_02651_b200 import gridgnn as gg

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1. unique-id hand-off (128 opaque bytes)
        blob = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        assert blob[0] == bytes(range(128))

        grid = gg.DeviceGrid(*dims)
        coord = grid.coord_of(rank)
        n, b, seed, step = 800, 300, 7, 3
        ds = O.generate_synthetic(n, 9.0, 4, 3, 5)
        gs = O.hash_combine(seed, grid.dp_group(rank))
        # 2. this rank's blocks of every plane, computed with no communication
        blocks = []
        for p in range(3):
            ra, ca = gg.adjacency_layout(p + 1)
            ro, co = gg.block_partition(n, dims[ra]), gg.block_partition(n, dims[ca])
            lb = O.local_minibatch(ds.adj, int(ro[coord[ra]]), int(ro[coord[ra] + 1]), int(co[coord[ca]]),
                                   int(co[coord[ca] + 1]), b, gs, step)
            blocks.append((lb.row_lo, lb.col_lo, lb.a.dense()))
        # 3. layout algebra: feature blocks of every layer
        H = 10
        fblocks = []
        for l in range(1, 5):
            fl = gg.feature_layout(l)
            s = O.sample_vertices(n, b, gs, step)
            boff = {ax: gg.sample_partition(s, gg.block_partition(n, dims[ax])) for ax in (1, 2, 3)}
            ro, co = boff[fl[0]], gg.block_partition(H, dims[fl[1]])
            fblocks.append((int(ro[coord[fl[0]]]), int(ro[coord[fl[0]] + 1]), int(co[coord[fl[1]]]),
                            int(co[coord[fl[1]] + 1])))
        step_ms = 10.0 + rank  # 4. max over ranks
        t = torch.tensor([step_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        gathered = [None] * world
        dist.all_gather_object(gathered, (blocks, fblocks, grid.dp_group(rank)))
        if rank == 0:
            serial = O.local_minibatch(ds.adj, 0, n, 0, n, b, gs, step).a.dense()
            for p in range(3):
                full = np.zeros_like(serial)
                for bl, _, dpg in gathered:
                    if dpg != 0:
                        continue  # other DP groups sample their own batches
                    r0, c0, d = bl[p]
                    full[r0:r0 + d.shape[0], c0:c0 + d.shape[1]] = d
                assert np.array_equal(full, serial), f"plane {p} does not reassemble"
            for l in range(4):
                cover = np.zeros((b, H), np.int32)
                for _, fb, dpg in gathered:
                    if dpg != 0:
                        continue
                    r0, r1, c0, c1 = fb[l]
                    cover[r0:r1, c0:c1] += 1
                assert cover.min() >= 1 and np.all(cover == cover.flat[0]), f"layer {l + 1} feature tiling"
            assert t.item() == 10.0 + world - 1
        q.put((rank, "ok"))
    except Exception as e:  # reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(1, 1, 1, 2), (1, 2, 1, 1), (1, 1, 2, 1), (2, 1, 1, 1)])
def test_two_rank_host_logic(dims):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
