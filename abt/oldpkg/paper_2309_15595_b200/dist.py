"""Process-group plumbing for the 2D grid (one process per GPU): grid shape, rank -> (myrow,
mycol), and distribution of the NCCL unique id through torch.distributed ("a 2D NCCL
communicator has been built on top of the 2D MPI grid").  Host logic only."""
from __future__ import annotations

GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}


def grid_shape(world: int) -> tuple[int, int]:
    """p x q "as square as possible" with p >= q; 8 GPUs -> 2 x 4 per BASELINE."""
    if world in GRIDS:
        return GRIDS[world]
    p = int(world ** 0.5)
    while world % p:
        p -= 1
    return max(p, world // p), min(p, world // p)


def grid_coords(rank: int, p: int, q: int) -> tuple[int, int]:
    """World rank = myrow * q + mycol (include/chase.h chase_create)."""
    return rank // q, rank % q


def share_unique_id(get_id, group=None) -> bytes:
    """Rank 0 calls get_id() (chase_get_unique_id); every rank returns the same 128 bytes."""
    import torch.distributed as dist

    obj = [get_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def enable_fused_comm(chase, group=None):
    """Give a Chase handle a symmetric peer-mapped region (torch symmetric memory over the world
    group: device memory + IPC mappings only) so its filter steps run as fused HEMM + NVLink
    reduction kernels (include/chase.h chase_set_fused_workspace).  Collective over the group."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm

    import paper_2309_15595_b200 as cb

    group = group or dist.group.WORLD
    nbytes = cb.chase_fused_workspace_size(chase.h)
    buf = symm.empty(nbytes, dtype=torch.uint8, device=chase.device)
    hdl = symm.rendezvous(buf, group)
    ptrs = [int(x) for x in hdl.buffer_ptrs]
    cb.chase_set_fused_workspace(chase.h, buf.data_ptr(), ptrs)
    torch.cuda.synchronize(chase.device)
    dist.barrier(group)
    chase._fused_keepalive = (buf, hdl)
    return hdl


def disable_fused_comm(chase):
    import paper_2309_15595_b200 as cb

    cb.chase_set_fused_workspace(chase.h, None)
