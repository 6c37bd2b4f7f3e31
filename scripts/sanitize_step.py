"""One decode step (taper_admit -> taper_append_kv -> taper_decode_attention, twice, so the
second attention follows the first one's merge under PDL) on a config's batch, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).  Checks the outputs
against the oracle on a few (slot, head) pairs so a sanitizer run is also a parity run.

    compute-sanitizer --tool memcheck python scripts/sanitize_step.py c1|c2 [h_local]"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2605_06914_b200 import taper as T  # noqa: E402
from tests.helpers import assert_close  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    h = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    b = synth.config_batch(cfg, seed=0, slack_min_ms=30.0)
    lay = synth.make_layout(b, 64, np.random.default_rng(1), spare_pages=1)
    k, v = synth.make_kv(lay.num_pages, h, 64, 128, seed=0)
    q = synth.make_q(b.n_slot, 8 * h, 128, seed=0)
    db = T.DeviceBatch.from_host(b)
    adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
    ws = torch.zeros(T.taper_workspace_size(b.n_req, b.n_slot, h, T.max_chunk_slots(
        b.req_shared_len, b.req_slot_off, b.slot_local_len, h_local=h)), dtype=torch.uint8,
        device="cuda")
    rpo, rp, spo, sp = T.page_tables_to_device(lay)
    kv = T.DeviceKV(k.cuda(), v.cuda(), rpo, rp, spo, sp)
    g = torch.Generator().manual_seed(3)
    kn = torch.randn((b.n_slot, h, 128), generator=g).bfloat16()
    vn = torch.randn((b.n_slot, h, 128), generator=g).bfloat16()
    qd = q.cuda()
    outs = [torch.zeros_like(qd), torch.zeros_like(qd)]
    model = (12.0, 0.03, 2e-5)
    T.taper_admit(db, model, "taper", 0.8, adm, h, ws)
    T.taper_append_kv(db, adm, kv, kn.cuda(), vn.cuda())
    for o in outs:
        T.taper_decode_attention(db, adm, kv, qd, o, None, 1 / math.sqrt(128), ws)
    torch.cuda.synchronize()
    st = int(adm.status.item())
    assert st == 0, T.taper_status_string(st)
    assert torch.equal(outs[0], outs[1])
    mask = adm.slot_admitted.cpu().numpy()[:b.n_slot]
    o = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len, model,
                     "taper", 2, 0.8)
    assert (mask == o.slot_admitted).all()
    kc, vc = kv.k_pages.cpu(), kv.v_pages.cpu()
    slots = np.flatnonzero(mask)[:6]
    es, eh = np.repeat(slots, 2), np.tile([0, 8 * h - 1], len(slots))
    ref, _ = oracle.attention(b.req_slot_off, b.req_shared_len, b.slot_local_len, lay.req_page_off,
                              lay.req_pages, lay.slot_page_off, lay.slot_pages, kc, vc, q, es, eh)
    assert_close(outs[0].cpu()[es, eh].float().numpy(), ref, cfg)
    print(f"sanitize_step {cfg} h={h}: ok ({int(mask.sum())}/{b.n_slot} admitted)")


if __name__ == "__main__":
    main()
