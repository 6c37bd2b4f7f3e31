"""KV-head sharding of the hot path across G GPUs (one process per GPU).

SURVEY.md Sec. 8(e): every KV head is an independent unit (its 8 GQA query heads attend
only to it), so rank g of G owns KV heads [g*h, (g+1)*h) with h = 8 / G -- their K/V pages
for every request and the matching 8h query heads of every slot.  Page tables and batch
state are replicated.  Two exchanges remain, both through torch.distributed (NCCL on the
GPU box, gloo in the CPU tests):

  * the admission decision: rank 0's ``slot_admitted`` is broadcast once per step and
    every rank rebuilds its attention work list from it (taper_build_work), so ranks can
    never diverge;
  * the per-layer outputs: all-gather of out[S, 8h, 128] -> [G, S, 8h, 128], which is a
    permuted view of [S, 64, 128] (``to_slot_major``).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

N_KV_HEADS = 8
GQA = 8


def heads_per_rank(world: int) -> int:
    if world < 1 or N_KV_HEADS % world:
        raise ValueError(f"world size {world} must divide {N_KV_HEADS} KV heads")
    return N_KV_HEADS // world


def kv_head_range(rank: int, world: int) -> tuple[int, int]:
    h = heads_per_rank(world)
    return rank * h, (rank + 1) * h


def q_head_range(rank: int, world: int) -> tuple[int, int]:
    g0, g1 = kv_head_range(rank, world)
    return GQA * g0, GQA * g1


def _host_staged(group) -> bool:
    """gloo (CPU tests, the one-GPU multi-rank checks) exchanges host tensors."""
    return dist.get_backend(group) == "gloo"


def broadcast_admission(slot_admitted: torch.Tensor, group=None) -> torch.Tensor:
    """Replace every rank's admitted-slot mask by rank 0's (in place)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        if slot_admitted.is_cuda and _host_staged(group):
            h = slot_admitted.cpu()
            dist.broadcast(h, src=0, group=group)
            slot_admitted.copy_(h)
        else:
            dist.broadcast(slot_admitted, src=0, group=group)
    return slot_admitted


def gather_outputs(out_local: torch.Tensor, gathered: torch.Tensor | None = None,
                   group=None) -> torch.Tensor:
    """All-gather of this rank's out[S, 8h, 128] into [G, S, 8h, 128]."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return out_local.unsqueeze(0)
    if gathered is None:
        gathered = out_local.new_empty((world,) + tuple(out_local.shape))
    if out_local.is_cuda and _host_staged(group):
        # bit patterns as bytes (gloo's all-gather takes neither bf16 nor int16 here; a
        # gather only moves bits)
        hg = torch.empty(gathered.shape, dtype=gathered.dtype).view(torch.uint8)
        dist.all_gather_into_tensor(hg.view(-1, *hg.shape[2:]),
                                    out_local.cpu().contiguous().view(torch.uint8), group=group)
        gathered.copy_(hg.view(gathered.dtype))
        return gathered
    # concatenated [G*S, ...] view: the form both NCCL and gloo accept
    dist.all_gather_into_tensor(gathered.view(-1, *out_local.shape[1:]), out_local.contiguous(),
                                group=group)
    return gathered


def to_slot_major(gathered: torch.Tensor) -> torch.Tensor:
    """[G, S, 8h, 128] -> [S, 64, 128] (global Q head = 8h * rank + local head)."""
    G, S, qh, d = gathered.shape
    return gathered.permute(1, 0, 2, 3).reshape(S, G * qh, d)
