"""All-to-all bandwidth on this box: torch.distributed (NCCL) all_to_all_single of S
bytes per rank (equal splits), device-timed, max over ranks; per-rank send GB/s counts
only the (P-1)/P remote part.  Run under torchrun; env vars select NCCL settings."""
import os
import torch
import torch.distributed as dist

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
P = dist.get_world_size()
res = []
for mb in (64, 256, 1024):
    n = mb * (1 << 20) // 4 // P * P
    a = torch.ones(n, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        dist.all_to_all_single(b, a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dist.all_to_all_single(b, a)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 5], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    res.append(f"{mb}MB {t.item():.3f}ms {4 * n * (P - 1) / P / (t.item() / 1e3) / 1e9:.0f}GB/s")
if dist.get_rank() == 0:
    print(os.environ.get("SWEEP_TAG", ""), "|", "  ".join(res), flush=True)
dist.destroy_process_group()
