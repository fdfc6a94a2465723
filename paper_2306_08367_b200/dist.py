"""Multi-GPU plumbing for the row-sharded fact table.

Fact rows are independent: rank r owns the contiguous row range
shard_range(n, r, world); dimensions are replicated.  Query accumulators
(int64 [G][count, sum]) are summed across ranks with one all-reduce; fused
predictions stay row-sharded and their global order is the rank order.
The product's own transport is the C-ABI communicator (laq_ctx_attach_nccl:
NCCL loaded inside liblaq_b200.so, all-reduce enqueued on the context stream);
attach() sets it up from an initialised torch.distributed group.  With a gloo
group (CPU tests, several ranks sharing one GPU) the context gets a host
all-reduce hook over that group instead.
"""
from __future__ import annotations

import torch


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of rank's contiguous share of n rows (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


def attach(ctx, group=None):
    """Give a device.Context the ranks of an initialised torch.distributed group:
    NCCL inside the C-ABI when the group's backend is nccl, else a host
    all-reduce hook over the group (gloo)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        return ctx
    if dist.get_backend(group) == "nccl":
        from .device import nccl_unique_id
        try:
            obj = [nccl_unique_id() if rank == 0 else None]
        except Exception as e:  # libnccl.so.2 not loadable from the library
            obj = [e]
        dist.broadcast_object_list(obj, src=0, group=group)
        ok = not isinstance(obj[0], Exception)
        if ok:
            try:
                ctx.attach_nccl(world, rank, obj[0])
            except Exception:
                ok = False
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if flag.item() == 1:
            ctx.transport = "nccl (C-ABI communicator)"
            return ctx
        # Fallback: the same int64 all-reduce through torch's NCCL group.
        def hook(buf):
            t = torch.from_numpy(buf).cuda()
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            buf[:] = t.cpu().numpy()
        ctx.set_allreduce_host(world, rank, hook)
        ctx.transport = "nccl (torch.distributed via the C-ABI host hook)"
    else:
        def hook(buf):
            t = torch.from_numpy(buf)  # shares memory with the C buffer
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        ctx.set_allreduce_host(world, rank, hook)
        ctx.transport = "gloo (C-ABI host hook)"
    return ctx


def allreduce_acc(acc: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the per-rank query accumulators in place (exact: int64)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


def gather_offsets(local_count: int, group=None, device=None) -> tuple[int, int]:
    """Exclusive prefix of per-rank survivor counts -> (global offset, global total):
    where rank r's fused predictions go in the global, rank-ordered output."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 0, local_count
    world = dist.get_world_size(group)
    t = torch.tensor([local_count], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    counts = [int(x.item()) for x in out]
    r = dist.get_rank(group)
    return sum(counts[:r]), sum(counts)
