"""Probe: torch symmetric memory at NCCL world size 1 on one B200 -- peer
pointers, signal pads and whether a multicast (NVLS) address is available."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
torch.cuda.set_device(0)
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    err, v = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, 0)
    print("multicast supported attr:", err, v)
except Exception as e:
    print("cuda-python probe failed:", e)
print("backend:", symm.get_backend(torch.device("cuda")) if hasattr(symm, "get_backend") else None)
t = symm.empty(1 << 20, dtype=torch.uint8, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD.group_name)
for a in ("buffer_ptrs", "signal_pad_ptrs", "multicast_ptr", "world_size", "rank", "buffer_size", "signal_pad_size"):
    try:
        print(a, getattr(h, a))
    except Exception as e:
        print(a, "ERR", e)
print("t ptr", hex(t.data_ptr()))
dist.destroy_process_group()
