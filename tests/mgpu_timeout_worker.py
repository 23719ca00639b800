"""Collective watchdog worker (tests/test_multigpu.py, torchrun, 2 GPUs): rank
1 never joins rank 0's gradient all-reduce. Rank 0 must get CommTimeout
(comm.hpp:157-158, "collective timed out: not all group members arrived")
within its timeout, with the communicators aborted so the stream drains and
later collectives fail fast, instead of hanging forever."""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_02651_b200 import gridgnn as gg  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    obj = [gg.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = gg.Context(gg.DeviceGrid(2, 1, 1, 1), rank, device=rank, nccl_uid=obj[0])
    cfg = gg.ModelConfig(layers=2, d_in=8, d_h=16, d_out=3)
    st = gg.init_state(ctx, cfg, 1)
    res = {}
    log = lambda m: print(f"[rank {rank}] {m}", file=sys.stderr, flush=True)
    log("contexts up")
    if rank == 0:
        ctx.set_comm_timeout(3000)
        t0 = time.time()
        gg.dp_sync(ctx, st)  # rank 1 never arrives
        log("dp_sync enqueued")
        try:
            ctx.synchronize()
            res["raised"] = None
        except gg.CommTimeout as e:
            res["raised"] = "CommTimeout"
            res["msg"] = str(e)
        res["seconds"] = time.time() - t0
        log(f"synchronize returned: {res}")
        try:  # the aborted communicators fail fast afterwards
            gg.dp_sync(ctx, st)
            res["after"] = None
        except gg.CommTimeout:
            res["after"] = "CommTimeout"
        res["ok"] = (res["raised"] == "CommTimeout" and 2.5 < res["seconds"] < 30 and res["after"] == "CommTimeout"
                     and "not all group members arrived" in res["msg"])
        print(json.dumps(res), flush=True)
    else:
        time.sleep(12)  # stay alive past rank 0's deadline (a dead peer is an NCCL error, not a timeout)
    dist.barrier()
    os._exit(0)


if __name__ == "__main__":
    main()
