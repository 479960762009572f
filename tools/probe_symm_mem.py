"""Probe: torch symmetric memory on a one-rank NCCL group (multicast pointer, barrier)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29633")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
print("multicast supported (torch):", symm_mem.is_nvshmem_available() if hasattr(symm_mem, "is_nvshmem_available") else "n/a")
try:
    buf = symm_mem.empty(1024, device="cuda:0", dtype=torch.float32)
    h = symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
    print("rendezvous ok; multicast_ptr =", h.multicast_ptr, "buffer_ptrs =", h.buffer_ptrs, "world", h.world_size)
    h.barrier(channel=0)
    torch.cuda.synchronize()
    print("barrier ok")
except Exception as e:
    print("symm_mem failed:", type(e).__name__, e)
print("device attr multicast:", torch.cuda.get_device_properties(0))
dist.destroy_process_group()
