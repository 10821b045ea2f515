"""Probe: does torch symmetric memory expose an NVLS multicast address on this box
(world size 1)?  Prints the handle's multicast_ptr and whether a store through it
lands in the local buffer."""
import os
import socket
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
for k in ("TORCH_SYMM_MEM_ALLOW_OVERLAPPING_DEVICES",):
    print(k, os.environ.get(k))
try:
    print("backend", symm.get_backend(torch.device("cuda", 0)))
except Exception as e:  # noqa: BLE001
    print("get_backend:", e)
t = symm.empty((1024,), dtype=torch.float64, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD)
print("buffer_ptrs", h.buffer_ptrs, "data_ptr", t.data_ptr())
print("multicast_ptr", getattr(h, "multicast_ptr", None), "has_multicast_support",
      symm.has_multicast_support(torch.device("cuda", 0).type, 0) if hasattr(symm, "has_multicast_support") else None)
print("attrs", [a for a in dir(h) if not a.startswith("_")])
dist.destroy_process_group()
