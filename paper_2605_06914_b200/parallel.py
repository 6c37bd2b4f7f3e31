"""KV-head sharding of the hot path across G GPUs (one process per GPU).

SURVEY.md Sec. 8(e): every KV head is an independent unit (its 8 GQA query heads attend
only to it), so rank g of G owns KV heads [g*h, (g+1)*h) with h = 8 / G -- their K/V pages
for every request and the matching 8h query heads of every slot.  Page tables and batch
state are replicated.  Two exchanges remain, both through torch.distributed (NCCL on the
GPU box, gloo in the CPU tests):

  * the admission decision: rank 0's ``slot_admitted`` is broadcast once per step and
    every rank rebuilds its attention work list from it (taper_build_work), so ranks can
    never diverge;
  * the per-layer outputs: either FUSED into the attention call (``PeerGather`` +
    taper_decode_attention_gather: the merge epilogue stores every row into all ranks'
    [S, 64, 128] buffers over NVLink, mapped with CUDA IPC, and raises a per-rank flag that
    taper_gather_wait consumes -- SURVEY 8(f) NEXT-4), or an all-gather of out[S, 8h, 128]
    -> [G, S, 8h, 128], a permuted view of [S, 64, 128] (``to_slot_major``).
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


class PeerGather:
    """Buffers of one rank for the fused output gather (SURVEY 8(f) NEXT-4,
    taper_decode_attention_gather): ``n_buf`` gathered outputs [S, 64, 128] bf16 and
    ``n_flag`` flag arrays int32[8], in ONE device allocation so that one CUDA IPC handle
    maps all of it into the other ranks' processes.  ``gather(buf, flag)`` is this rank's
    taper_gather for one call: every rank's output buffer ``buf`` and flag array ``flag``
    (reuse a flag array only after its taper_gather_wait, e.g. one per layer)."""

    FLAG_BYTES = 64  # int32[8], padded

    def __init__(self, n_slot: int, world: int, rank: int, n_buf: int = 2, n_flag: int = 1,
                 device=None, group=None, _peer_bases=None):
        from . import taper as T
        self.S, self.world, self.rank = n_slot, world, rank
        self.n_buf, self.n_flag = n_buf, n_flag
        self.out_bytes = n_slot * N_KV_HEADS * GQA * 128 * 2
        total = n_buf * self.out_bytes + n_flag * self.FLAG_BYTES
        self.buf = torch.zeros(total, dtype=torch.uint8, device=device)
        self._opened = []
        if _peer_bases is not None:          # in-process ranks (one-GPU tests)
            self.bases = _peer_bases
        elif world == 1:
            self.bases = [self.buf.data_ptr()]
        else:                                # CUDA IPC over the process group
            handle, off = T.taper_ipc_handle(self.buf)
            objs = [None] * world
            dist.all_gather_object(objs, (handle, off), group=group)
            self.bases = []
            for j, (h, o) in enumerate(objs):
                if j == rank:
                    self.bases.append(self.buf.data_ptr())
                else:
                    p = T.taper_ipc_open(h, o)
                    self._opened.append((p, o))
                    self.bases.append(p)

    @classmethod
    def in_process(cls, n_slot: int, world: int, n_buf: int = 2, n_flag: int = 1, device=None):
        """``world`` ranks' buffers in one process (every "peer" pointer is local): the
        fused-gather path on one GPU, for tests."""
        ranks = [cls(n_slot, world, r, n_buf, n_flag, device, _peer_bases=[]) for r in range(world)]
        bases = [r.buf.data_ptr() for r in ranks]
        for r in ranks:
            r.bases = bases
        return ranks

    def out(self, i: int) -> torch.Tensor:
        """This rank's gathered output buffer i as [S, 64, 128] bf16."""
        return self.buf[i * self.out_bytes:(i + 1) * self.out_bytes].view(torch.bfloat16).view(
            self.S, N_KV_HEADS * GQA, 128)

    def flags(self, k: int) -> torch.Tensor:
        o = self.n_buf * self.out_bytes + k * self.FLAG_BYTES
        return self.buf[o:o + self.FLAG_BYTES].view(torch.int32)

    def gather(self, i: int, k: int):
        from . import taper as T
        assert 0 <= i < self.n_buf and 0 <= k < self.n_flag
        fo = self.n_buf * self.out_bytes + k * self.FLAG_BYTES
        return T.Gather(self.world, self.rank, [b + i * self.out_bytes for b in self.bases],
                        [b + fo for b in self.bases])

    def close(self):
        from . import taper as T
        for p, o in self._opened:
            T.taper_ipc_close(p, o)
        self._opened = []
