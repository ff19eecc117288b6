import os
import torch
import torch.distributed as dist
dist.init_process_group("nccl")
r = dist.get_rank()
torch.cuda.set_device(r)
x = torch.ones(64 << 20, device="cuda")
for _ in range(3):
    dist.all_reduce(x)
torch.cuda.synchronize()
if r == 0:
    print("allreduce ok", x[0].item())
dist.destroy_process_group()
