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


def _cuda_worker(rank, world, port, q):
    """One rank of the KV-head-sharded CUDA path on the shared GPU: rank 0
    alone admits, the admitted set is broadcast, rank 1 rebuilds its work list from it
    (taper_build_work), every rank runs the attention for its heads and the outputs are
    all-gathered -- the bench.py step, over gloo instead of NCCL (one GPU)."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2605_06914_b200 import parallel as par
        from paper_2605_06914_b200 import taper as T
        from tests.helpers import assert_close

        torch.cuda.set_device(0)
        b = synth.config_batch("c2", seed=6, slack_min_ms=30.0)
        lay = synth.make_layout(b, 64, np.random.default_rng(1), spare_pages=1)
        k, v = synth.make_kv(lay.num_pages, 8, 64, 128, seed=6)
        qq = synth.make_q(b.n_slot, 64, 128, seed=6)
        g0, g1 = par.kv_head_range(rank, world)
        h = g1 - g0
        db = T.DeviceBatch.from_host(b)
        adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
        ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, h, T.max_chunk_slots(
            b.req_shared_len, b.req_slot_off, b.slot_local_len)), dtype=torch.uint8, device="cuda")
        rpo, rp, spo, sp = T.page_tables_to_device(lay)
        kv = T.DeviceKV(k[:, g0:g1].contiguous().cuda(), v[:, g0:g1].contiguous().cuda(),
                        rpo, rp, spo, sp)
        ql = qq[:, 8 * g0:8 * g1].contiguous().cuda()
        if rank == 0:
            T.taper_admit(db, (12.0, 0.03, 2e-5), "taper", 0.8, adm, h, ws)
        par.broadcast_admission(adm.slot_admitted)
        if rank != 0:
            T.taper_build_work(db, adm, h, ws)
        out = torch.full_like(ql, float("nan"))
        T.taper_decode_attention(db, adm, kv, ql, out, None, 128 ** -0.5, ws)
        full = par.to_slot_major(par.gather_outputs(out)).cpu()
        mask = adm.slot_admitted.cpu().numpy()[:b.n_slot]
        assert int(adm.status.item()) == 0
        assert 0 < mask.sum() < b.n_slot  # partial admission
        if rank == 0:
            # the same shards run one after the other in this process: bitwise equal
            parts = []
            for g in range(world):
                a0, a1 = par.kv_head_range(g, world)
                adm2 = T.DeviceAdmission.empty(b.n_req, b.n_slot)
                adm2.slot_admitted.copy_(adm.slot_admitted)
                ws2 = torch.empty_like(ws)
                T.taper_build_work(db, adm2, a1 - a0, ws2)
                kv2 = T.DeviceKV(k[:, a0:a1].contiguous().cuda(), v[:, a0:a1].contiguous().cuda(),
                                 rpo, rp, spo, sp)
                q2 = qq[:, 8 * a0:8 * a1].contiguous().cuda()
                o2 = torch.full_like(q2, float("nan"))
                T.taper_decode_attention(db, adm2, kv2, q2, o2, None, 128 ** -0.5, ws2)
                parts.append(o2.cpu())
            seq = torch.cat(parts, dim=1)
            m = torch.from_numpy(mask.astype(bool))
            assert torch.equal(full[m], seq[m])
            o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                             (12.0, 0.03, 2e-5), "taper", 2, 0.8)
            assert (o.slot_admitted == mask).all()
            slots = np.flatnonzero(mask)[::7]
            es, eh = np.repeat(slots, 3), np.tile([1, 33, 62], len(slots))
            ref, _ = oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len,
                                      lay.req_page_off, lay.req_pages, lay.slot_page_off,
                                      lay.slot_pages, k, v, qq, es, eh)
            assert_close(full[es, eh].float().numpy(), ref, "gloo ranks")
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # surface worker failures in the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()[-1500:]))


@pytest.mark.gpu
def test_cuda_path_two_ranks_one_gpu_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cuda_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
