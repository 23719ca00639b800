"""NCCL bandwidth probe (torch.distributed, one process per GPU): all-reduce,
all-gather and send/recv of a few sizes, device-timed, max over ranks."""
import os, json, torch, torch.distributed as dist
dist.init_process_group("nccl")
r, w = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", r)))
out = {}
for mb in (8, 64, 313):
    n = mb * 2**20 // 4
    x = torch.ones(n, device="cuda")
    for name, fn in (("all_reduce", lambda: dist.all_reduce(x)),
                     ("all_gather", lambda: dist.all_gather_into_tensor(torch.empty(n * w, device="cuda"), x))):
        for _ in range(3): fn()
        torch.cuda.synchronize(); dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5): fn()
        b.record(); torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b) / 5], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        bus = (2 * (w - 1) / w if name == "all_reduce" else (w - 1) / w) * n * 4 / (ms.item() / 1e3) / 1e9
        out[f"{name}_{mb}MB"] = {"ms": round(ms.item(), 3), "busbw_GBps": round(bus, 1)}
if r == 0:
    print(json.dumps(out))
dist.destroy_process_group()
