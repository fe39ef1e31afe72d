"""Multi-process plumbing for field-parallel estimation (one process per GPU).

Fields are independent (Alg. 1 loops per field; the paper runs one
process per file), so ranks shard a stack of fields with no data-path
collective; the only collectives are control ones: the max over ranks of a timing
and the gathering of per-field results.  Backend-agnostic (NCCL on GPUs, gloo in the
CPU tests).
"""
from __future__ import annotations


def setup(backend: str = "nccl"):
    """(world, rank, local_rank) from the torchrun environment; initialises the process
    group when world > 1 (NCCL on GPUs, one process per GPU; gloo in the CPU tests)."""
    import os
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def shard(n_fields: int, rank: int, world: int) -> range:
    """Contiguous, balanced share of fields [0, n_fields) for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    q, r = divmod(n_fields, world)
    lo = rank * q + min(rank, r)
    return range(lo, lo + q + (1 if rank < r else 0))


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(local: dict) -> dict:
    """Merge {field_index: result} dicts from all ranks (control plane, pickled)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(local)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, local)
    out = {}
    for p in parts:
        out.update(p)
    return out
