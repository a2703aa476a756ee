"""Multi-GPU partitioning of the hot path.

* Conv workloads (configs 3/4) shard by batch: rank r owns images [r*B, (r+1)*B) (weak scaling,
  B images per GPU) and regenerates them from the counter-based generator; no collective in the
  step.
* The square GEMM (config 5) splits output channels: rank r owns rows [r*M/P, (r+1)*M/P) of W and
  C and the full second operand; one all-gather of the int32 row blocks gives every rank C.
* Timing reduces to the max over ranks.
These functions only move data / indices; the arithmetic runs in libdg."""
from __future__ import annotations

import torch


def batch_shard(rank: int, world: int, per_rank: int) -> range:
    return range(rank * per_rank, (rank + 1) * per_rank)


def row_shard(rank: int, world: int, n: int) -> tuple[int, int]:
    if n % world:
        raise ValueError(f"{n} rows are not divisible by {world} ranks")
    m = n // world
    return rank * m, (rank + 1) * m


def gather_rows(local: torch.Tensor, world: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather equal row blocks into the full [world*m][...] tensor (rank order = row order)."""
    import torch.distributed as dist
    if world == 1:
        return local
    if out is None:
        out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous())
    else:  # gloo (CPU tests): list form
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local.contiguous())
    return out


class PeerRows:
    """Fused all-gather destinations for config 5: every rank holds the full C in
    symmetric memory (CUDA P2P-mapped across the node's GPUs); rank r's GEMM epilogue stores its
    rows [r0, r1) into every peer's C directly (dg_lut_gemm_prepared_allgather), and a device-side
    barrier on the same stream orders those stores before anyone reads C."""

    def __init__(self, shape, dtype, device, rank: int, world: int, row0: int):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.full = symm_mem.empty(*shape, dtype=dtype, device=device)
        self.hdl = symm_mem.rendezvous(self.full, dist.group.WORLD)
        pitch = self.full.stride(0) * self.full.element_size()
        self.peers = [int(self.hdl.buffer_ptrs[j]) + row0 * pitch for j in range(world) if j != rank]

    def barrier(self):
        self.hdl.barrier(channel=0)


def max_over_ranks(v: float, world: int, device="cpu") -> float:
    import torch.distributed as dist
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
