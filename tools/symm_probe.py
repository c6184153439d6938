"""Probe: torch symmetric memory (CUDA IPC) peer buffers + copy-engine pulls."""
import os
import time
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
group = dist.group.WORLD
symm_mem.enable_symm_mem_for_group(group.group_name)
n = 64 * 2**20
buf = symm_mem.empty((n,), dtype=torch.bfloat16, device=dev)
hdl = symm_mem.rendezvous(buf, group.group_name)
buf.fill_(rank + 1)
out = torch.empty(world * n, dtype=torch.bfloat16, device=dev)
s = torch.cuda.Stream()
torch.cuda.synchronize()
for it in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        hdl.barrier()
        e0.record()
        for step in range(world):
            r = (rank - step) % world
            out[r * n:(r + 1) * n].copy_(hdl.get_buffer(r, (n,), torch.bfloat16))
        e1.record()
        hdl.barrier()
    torch.cuda.synchronize()
    ok = all(bool((out[r * n:(r + 1) * n] == r + 1).all()) for r in range(world))
    gb = (world - 1) * n * 2 / 1e9
    if rank == 0:
        print(f"iter {it} ok={ok} pull {gb:.3f} GB in {e0.elapsed_time(e1):.3f} ms "
              f"-> {gb / e0.elapsed_time(e1) * 1e3:.1f} GB/s", flush=True)
dist.destroy_process_group()
