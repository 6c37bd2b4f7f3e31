"""Fused output gather (App. D, tensor parallelism over
NVLink): taper_decode_attention_gather stores every output row of a rank into ALL ranks'
gathered buffers [S, 64, 128] from the merge epilogue and raises a flag per rank;
taper_gather_wait waits for all ranks' flags.  On one GPU the "peers" are buffers of the same
device: (a) G ranks in one process (every rank's call, then every rank's wait), (b) two
processes that map each other's buffers with CUDA IPC under a gloo group.  Both must equal,
bitwise, the per-rank outputs of taper_decode_attention placed slot-major (what the NCCL
all-gather path produces), and the oracle on sampled rows."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from tests.helpers import assert_close

pytestmark = pytest.mark.gpu


def _rank_inputs(b, lay, k, v, qq, G, g, adm_mask, dev="cuda"):
    """Rank g's shard: KV heads [g h, (g+1) h), its Q heads, work list rebuilt from the mask."""
    from paper_2605_06914_b200 import parallel as par
    from paper_2605_06914_b200 import taper as T
    g0, g1 = par.kv_head_range(g, G)
    h = g1 - g0
    db = T.DeviceBatch.from_host(b, dev)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot, dev)
    adm.slot_admitted.copy_(adm_mask)
    ws = torch.empty(T.taper_workspace_size(b.n_req, b.n_slot, h, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len, h_local=1)), dtype=torch.uint8, device=dev)
    T.taper_build_work(db, adm, h, ws)
    rpo, rp, spo, sp = T.page_tables_to_device(lay, dev)
    kv = T.DeviceKV(k[:, g0:g1].contiguous().to(dev), v[:, g0:g1].contiguous().to(dev), rpo, rp, spo, sp)
    q = qq[:, 8 * g0:8 * g1].contiguous().to(dev)
    return db, adm, kv, q, ws


def _case(seed=5, kind="c2"):
    if kind == "wide":  # requests with >= 9 ready slots: row-mode items
        rng = np.random.default_rng(seed)
        fan = [12, 1, 16, 9, 3, 1]
        b = synth.make_batch([6000, 2500, 9000, 700, 4096, 1], fan,
                             rng.integers(1, 300, size=sum(fan)).tolist(), 15.0, 20.0, rng=rng)  # partial: widths 9,1,1,9,3,1
    else:
        b = synth.config_batch("c2", seed=seed, slack_min_ms=30.0)
    lay = synth.make_layout(b, 64, np.random.default_rng(seed + 1), spare_pages=1)
    k, v = synth.make_kv(lay.num_pages, 8, 64, 128, seed=seed)
    qq = synth.make_q(b.n_slot, 64, 128, seed=seed)
    o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                     (12.0, 0.03, 2e-5), "taper", 2, 0.8)
    return b, lay, k, v, qq, o.slot_admitted.astype(np.uint8)


def _per_rank_reference(b, lay, k, v, qq, G, mask):
    """taper_decode_attention per rank, slot-major: what the NCCL all-gather path yields."""
    from paper_2605_06914_b200 import taper as T
    parts = []
    m = torch.from_numpy(mask).cuda()
    for g in range(G):
        db, adm, kv, q, ws = _rank_inputs(b, lay, k, v, qq, G, g, m)
        out = torch.full_like(q, float("nan"))
        T.taper_decode_attention(db, adm, kv, q, out, None, 128 ** -0.5, ws)
        parts.append(out)
    torch.cuda.synchronize()
    return torch.cat(parts, dim=1).cpu()


@pytest.mark.parametrize("G,kind", [(2, "c2"), (4, "c2"), (8, "c2"), (2, "wide"), (8, "wide")])
def test_fused_gather_in_process(G, kind):
    from paper_2605_06914_b200 import parallel as par
    from paper_2605_06914_b200 import taper as T
    b, lay, k, v, qq, mask = _case(kind=kind)
    assert 0 < mask.sum() < b.n_slot
    ref = _per_rank_reference(b, lay, k, v, qq, G, mask)
    ranks = par.PeerGather.in_process(b.n_slot, G, n_buf=2, n_flag=2, device="cuda")
    m = torch.from_numpy(mask).cuda()
    for i in range(2):  # two layers: buffer / flag array i, same inputs
        for g in range(G):
            db, adm, kv, q, ws = _rank_inputs(b, lay, k, v, qq, G, g, m)
            T.taper_decode_attention_gather(db, adm, kv, q, ranks[g].gather(i, i), None,
                                            128 ** -0.5, ws)
            assert T.taper_last_launch_count() == 2
        for g in range(G):
            T.taper_gather_wait(ranks[g].gather(i, i))
        torch.cuda.synchronize()
        sel = torch.from_numpy(mask.astype(bool))
        for g in range(G):
            full = ranks[g].out(i).cpu()
            assert torch.equal(full[sel], ref[sel]), (G, g, i)
            assert int(ranks[g].flags(i).abs().sum()) == 0  # cleared by the wait
    slots = np.flatnonzero(mask)[::9]
    es, eh = np.repeat(slots, 4), np.tile([0, 21, 42, 63], len(slots))
    want, _ = oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len, lay.req_page_off,
                               lay.req_pages, lay.slot_page_off, lay.slot_pages, k, v, qq, es, eh)
    assert_close(ranks[G - 1].out(1).cpu()[es, eh].float().numpy(), want, f"gather G={G}")


def test_gather_argument_errors():
    from paper_2605_06914_b200 import parallel as par
    from paper_2605_06914_b200 import taper as T
    b, lay, k, v, qq, mask = _case()
    ranks = par.PeerGather.in_process(b.n_slot, 2, device="cuda")
    db, adm, kv, q, ws = _rank_inputs(b, lay, k, v, qq, 4, 0, torch.from_numpy(mask).cuda())
    with pytest.raises(T.TaperError, match="h_local"):  # h = 2 shard with a world of 2
        T.taper_decode_attention_gather(db, adm, kv, q, ranks[0].gather(0, 0), None, 0.1, ws)
    with pytest.raises(T.TaperError):
        T.taper_gather_wait(T.Gather(2, 3, [0, 0], [0, 0]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2605_06914_b200 import parallel as par
        from paper_2605_06914_b200 import taper as T
        torch.cuda.set_device(0)
        b, lay, k, v, qq, mask = _case(seed=8)
        pg = par.PeerGather(b.n_slot, world, rank, n_buf=1, n_flag=1, device="cuda")
        m = torch.from_numpy(mask).cuda()
        db, adm, kv, qd, ws = _rank_inputs(b, lay, k, v, qq, world, rank, m)
        torch.cuda.synchronize()
        dist.barrier()
        g = pg.gather(0, 0)
        T.taper_decode_attention_gather(db, adm, kv, qd, g, None, 128 ** -0.5, ws)
        T.taper_gather_wait(g)
        torch.cuda.synchronize()
        full = pg.out(0).cpu()
        ref = _per_rank_reference(b, lay, k, v, qq, world, mask)
        sel = torch.from_numpy(mask.astype(bool))
        assert torch.equal(full[sel], ref[sel])
        dist.barrier()  # peers are done reading / writing before the mappings go away
        pg.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()[-1500:]))


def test_fused_gather_two_processes_cuda_ipc():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
