"""Worker of test_peer_matches_nccl (run under torchrun, one process per GPU):
three Adam steps of the GCN on a PMM grid at the C2 model width, then prints
rank 0's losses and every rank's weight and gradient blocks as raw bytes (hex)
so the test can compare a GGB_PEER=1 run with a GGB_PEER=0 run bit for bit."""
import hashlib
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (test input generator only)
from paper_2604_02651_b200 import gridgnn as gg  # noqa: E402


def main():
    dims = tuple(int(x) for x in sys.argv[1].split("x"))
    prec = int(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    obj = [gg.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    grid = gg.DeviceGrid(*dims)
    ctx = gg.Context(grid, rank, device=local, nccl_uid=obj[0])
    n, d_in, ncls, b, seed = 6000, 40, 9, 2400, 11
    ds = O.generate_synthetic(n, 12.0, d_in, ncls, 5)
    g = gg.Graph.from_csr(ctx, n, ds.adj.row_ptr, ds.adj.col_idx, ds.adj.values, ds.features, ds.labels, ncls, 3)
    cfg = gg.ModelConfig(layers=3, d_in=d_in, d_h=256, d_out=ncls, dropout_rate=0.1)
    st = gg.init_state(ctx, cfg, seed)
    gs = gg.hash_combine(seed, grid.dp_group(rank))
    losses, batch = [], None
    for t in range(3):
        batch = gg.build_step_batch(ctx, g, b, gs, t, reuse=batch)
        losses.append(gg.train_step(ctx, st, batch, prec, seed, t))
        grads = [np.ascontiguousarray(x).tobytes() for x in st.grads()]
        gg.dp_sync(ctx, st)
        gg.optimizer_step(ctx, st, gg.ADAM, 1e-3)
    weights = [np.ascontiguousarray(w).tobytes() for w in st.weights()]
    digest = hashlib.sha256(b"".join(grads + weights)).hexdigest()
    out = [None] * world
    dist.all_gather_object(out, {"rank": rank, "digest": digest,
                                 "losses": [np.float32(x).tobytes().hex() for x in losses]})
    if rank == 0:
        print(json.dumps({"grid": dims, "prec": prec, "ranks": out}), flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
