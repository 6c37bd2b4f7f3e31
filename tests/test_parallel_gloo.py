"""World-size-2 CPU (gloo) tests of the KV-head-sharded path's host logic
(paper_2605_06914_b200/parallel.py): head ranges, the admission broadcast and the
output all-gather + slot-major view.  The per-rank compute is stood in by the oracle
restricted to the rank's heads, so the test checks exactly the partition/gather
indexing that the NCCL path uses on the GPU box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2605_06914_b200 import parallel as par

        b = synth.config_batch("c1", seed=0)
        lay = synth.make_layout(b, 64, np.random.default_rng(1), spare_pages=1)
        k, v = synth.make_kv(lay.num_pages, 8, 64, 128, seed=0)
        qq = synth.make_q(b.n_slot, 64, 128, seed=0)
        # admission broadcast: rank 1 starts with a different mask
        mask = torch.tensor([1, 1, 0, 1, 0], dtype=torch.uint8) if rank == 0 else \
            torch.ones(5, dtype=torch.uint8)
        par.broadcast_admission(mask)
        assert mask.tolist() == [1, 1, 0, 1, 0]
        # this rank's shard: KV heads [g0, g1), Q heads [8 g0, 8 g1)
        g0, g1 = par.kv_head_range(rank, world)
        h0, h1 = par.q_head_range(rank, world)
        assert (g1 - g0) == par.heads_per_rank(world) and h1 - h0 == 8 * (g1 - g0)
        S = b.n_slot
        es, eh = np.meshgrid(np.arange(S), np.arange(h1 - h0), indexing="ij")
        # local view of the shard: local heads 0..8h-1 over the rank's KV slice
        out, _ = oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len,
                                  lay.req_page_off, lay.req_pages, lay.slot_page_off,
                                  lay.slot_pages, k[:, g0:g1].contiguous(),
                                  v[:, g0:g1].contiguous(), qq[:, h0:h1].contiguous(),
                                  es.ravel(), eh.ravel())
        local = torch.from_numpy(out).reshape(S, h1 - h0, 128)
        gathered = par.gather_outputs(local)
        full = par.to_slot_major(gathered)
        es, eh = np.meshgrid(np.arange(S), np.arange(64), indexing="ij")
        ref, _ = oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len,
                                  lay.req_page_off, lay.req_pages, lay.slot_page_off,
                                  lay.slot_pages, k, v, qq, es.ravel(), eh.ravel())
        assert torch.equal(full, torch.from_numpy(ref).reshape(S, 64, 128))
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2])
def test_kv_head_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res


def test_head_ranges():
    from paper_2605_06914_b200 import parallel as par
    for G in (1, 2, 4, 8):
        rs = [par.kv_head_range(r, G) for r in range(G)]
        assert rs[0][0] == 0 and rs[-1][1] == 8
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    with pytest.raises(ValueError):
        par.heads_per_rank(3)
    g = torch.arange(2 * 3 * 4 * 2).reshape(2, 3, 4, 2)
    sm = par.to_slot_major(g)
    assert sm.shape == (3, 8, 2) and torch.equal(sm[1, 5], g[1, 1, 1])
