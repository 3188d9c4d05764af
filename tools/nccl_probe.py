"""One-process NCCL group on cuda:0: the collective calls the N > 1 step issues (the
coalesced per-dtype allreduce of the aggregates) run through NCCL itself."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
dev = torch.device("cuda", 0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
from paper_2310_07240_b200.step import _allreduce_list_  # noqa: E402

a = torch.arange(10, dtype=torch.int64, device=dev)
b = torch.ones(3, dtype=torch.float64, device=dev)
c = torch.arange(4, dtype=torch.int64, device=dev)
_allreduce_list_([a, b, c])
torch.cuda.synchronize()
assert a.sum().item() == 45 and b.sum().item() == 3.0 and c.sum().item() == 6
print("NCCL per-dtype coalesced allreduce OK")
dist.destroy_process_group()
