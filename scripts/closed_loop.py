"""NEXT-2: closed-loop synthetic replay on B200 step times.

A synthetic analog of the paper's Fig. 2 / Table 1 loop (App. D), never a parity
claim against its numbers: requests arrive, decode, fan out into parallel phases and
reduce; every step the policy decides the admitted set from the requests' slack
(d_r = last progress + SLO, any admitted branch token counting as progress -- reading
C-adm-7), the step runs, and its realised duration advances the clock and feeds the next
step's slack.

  * admission: the product's device `taper_admit` (GPU run) or the oracle (CPU test);
  * step time: `taper_decode_attention` over the step's real composition, CUDA-event timed on
    `--timed-layers` layers and scaled to 64 (GPU run), plus a synthetic non-attention part
    `T_rest = a_r + b_r * n` standing in for the QKV/O projections and MLP this library does
    not have (no weights); the CPU test uses a linear model instead;
  * predictor given to TAPER: the B200 fit of profiles/latency_model_b200.json (cascade-aware
    per-request context, R^2 0.98) plus T_rest -- an accurate predictor by construction.

Metrics (App. D "Metrics", L387-391): throughput = tokens / time; goodput = tokens of the
requests whose maximum inter-token gap <= SLO / time; attainment = share of finished requests
meeting the SLO; admission rate = granted / ready opportunistic branches.

    python scripts/closed_loop.py [--steps 1500] [--policies off,cap2,cap5,eager,taper]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

SLO_MS = 50.0          # App. D: "All requests share a 50 ms TPOT target" (L199)
R_MAX = 96             # active-request cap of the engine
REST = (12.0, 0.12)    # synthetic non-attention step part: a_r ms + b_r ms per sequence


@dataclass
class Req:
    rid: int
    arrival: float
    lsh: int                       # shared context (prefix, + finished phases)
    stages: list                   # remaining stages: ("serial", n) | ("parallel", [targets])
    branches: list = field(default_factory=list)   # current phase: [local_len, target]
    serial_left: int = 0
    last_progress: float = 0.0
    max_gap: float = 0.0
    tokens: int = 0
    done: bool = False
    segs: list = None      # reduce stage: finished branches' lengths (canonical order)
    z: int = 0             # reduce tokens so far (the last local segment)
    phase: int = 0         # parallel phases started (the no-replanning ablation commits per phase)

    def start_stage(self):
        while self.stages:
            kind, arg = self.stages.pop(0)
            if kind == "serial" and arg > 0:
                self.serial_left = arg
                return
            if kind == "parallel":
                self.branches = [[1, t] for t in arg]  # the first branch token is in the cache
                self.phase += 1
                return
        self.done = True


def make_request(rng, rid, t):
    """PDR 50 % (L199): a decomposable request decodes a serial prelude, a parallel phase
    (Table-4 fanout, branch lengths U{32..256}) and a reduce stretch; the other half decode
    serially.  Prompt (prefix) U[1k, 8k]."""
    lsh = int(rng.integers(1024, 8193))
    if rng.random() < 0.5:
        n = int(synth.sample_fanout(rng, 1)[0])
        stages = [("serial", int(rng.integers(8, 33))),
                  ("parallel", [int(x) for x in rng.integers(32, 257, size=n)]),
                  ("serial", int(rng.integers(16, 65)))]
    else:
        stages = [("serial", int(rng.integers(64, 257)))]
    r = Req(rid, t, lsh, stages, last_progress=t)
    r.start_stage()
    return r


def arrival_rate(step, n_steps):
    """Requests per second: low / high / moderate regimes in the 240 / 150 / 210 proportions
    of the Azure-derived trace (L385, L199); scaled to this engine's R_MAX."""
    f = step / max(1, n_steps)
    return 5.0 if f < 0.4 else (40.0 if f < 0.65 else 15.0)


def batch_of(active, now):
    """A reduce-stage request is one slot whose local context is its finished branches in
    canonical order plus z, each segment in its own pages (Sec. 3.1):
    nothing is copied when a phase ends."""
    shared, fan, segs, slack = [], [], [], []
    for r in active:
        shared.append(r.lsh)
        if r.branches:
            live = [b for b in r.branches if b[0] < b[1]]
            fan.append(len(live))
            segs += [[b[0]] for b in live]
        elif r.segs is not None:
            fan.append(1)
            segs.append(r.segs + [r.z])
        else:
            fan.append(1)
            segs.append([])
        slack.append(r.last_progress + SLO_MS - now)
    b = synth.make_batch(shared, fan, [sum(x) for x in segs], 0.0, 0.0)
    b = synth.with_segments(b, segs)
    b.req_slack_ms = np.asarray(slack, np.float64)
    return b


def advance(active, b, slot_admitted, now):
    """Admitted slots emit one token at `now` (the end of the step)."""
    off = b.req_slot_off
    toks = 0
    for i, r in enumerate(active):
        adm = slot_admitted[off[i]:off[i + 1]]
        if not adm.any():
            continue
        r.max_gap = max(r.max_gap, now - r.last_progress)
        r.last_progress = now
        if r.branches:
            live = [x for x in r.branches if x[0] < x[1]]
            for x, a in zip(live, adm):
                if a:
                    x[0] += 1
                    toks += 1
            if all(x[0] >= x[1] for x in r.branches):  # phase complete -> reduce context
                r.segs = [x[0] for x in r.branches]       # read in place, not copied
                r.z = 0
                r.branches = []
                r.start_stage()
        else:
            if r.segs is not None:
                r.z += 1      # reduce token: appended to the last local segment
            else:
                r.lsh += 1
            r.serial_left -= 1
            toks += 1
            if r.serial_left <= 0:
                r.start_stage()
        r.tokens += int(adm.sum())
    return toks


class RollingFit:
    """App. C.2 (L337): the predictor is refreshed by OLS on a rolling window of the most
    recent 200 observed step latencies (here every `every` steps instead of 10 minutes)."""

    def __init__(self, model, window=200, every=50):
        self.model, self.window, self.every = tuple(model), window, every
        self.obs = []
        self.count = 0

    def observe(self, n, L, t):
        self.obs.append((n, L, t))
        self.obs = self.obs[-self.window:]
        self.count += 1
        if len(self.obs) >= 50 and self.count % self.every == 0:
            X = np.array([[1.0, o[0], o[1]] for o in self.obs])
            y = np.array([o[2] for o in self.obs])
            coef, *_ = np.linalg.lstsq(X, y, rcond=None)
            if coef[1] > 0 and coef[2] > 0 and coef[0] >= 0:  # keep T monotone (L341)
                self.model = tuple(float(c) for c in coef)


def context_per_request(b, adm):
    """Cascade-aware L_context of the admitted set (reading R-ctx): prefix once per request."""
    off = b.req_slot_off
    L = 0
    for r in range(b.n_req):
        a = adm[off[r]:off[r + 1]]
        if a.any():
            L += int(b.req_shared_len[r]) + int(b.slot_local_len[off[r]:off[r + 1]][a].sum())
    return L


def canonical_first(b, i, w):
    """Request i's first w ready slots in canonical order (ascending local length, then
    slot index -- reading C-adm-1): Cap(w) for one request."""
    off = b.req_slot_off
    slots = np.arange(off[i], off[i + 1])
    order = slots[np.lexsort((slots, b.slot_local_len[slots]))]
    m = np.zeros(b.n_slot, bool)
    m[order[:max(1, w)]] = True
    return m


def predict(model, b, adm):
    """App. C.1 T(S) = a + b n + c L with the cascade-aware per-request context."""
    return model[0] + model[1] * int(adm.sum()) + model[2] * context_per_request(b, adm)


# Table 1 ablations on top of the product's admission:
#   noslack : "without the slack budget" -- every request's slack is unbounded, so the
#             planner admits every branch that fits (near Eager);
#   noreplan: "without per-step replanning" -- a request's width is committed at the first
#             step of each parallel phase (TAPER's decision then) and held until the reduce;
#   const   : "with a constant latency predictor" -- every sequence costs the same, whatever
#             its context: T = a + (b + c L_ref) n with L_ref a fixed typical context;
#   rho     : the slack fraction sweep (taper at rho 0.5 / 1.0).
ABLATIONS = ("noslack", "noreplan", "const")
L_REF = 4096


def run(policy, admit_fn, step_fn, n_steps, seed=0, rho=0.8, model=None, refit=False,
        ablation=None, set_mask=None):
    """admit_fn(batch, policy, rho, model) -> (slot mask, predicted T(S) ms);
    step_fn(batch, mask) -> realised step ms; set_mask(batch, mask): hand a mask composed
    outside the admission (the no-replanning ablation) to the step's work list."""
    assert ablation in (None,) + ABLATIONS
    if ablation == "const" and model is not None:
        model = (model[0], model[1] + model[2] * L_REF, model[2] * 1e-9)
    committed = {}  # no-replanning: (rid, phase) -> width
    rng = np.random.default_rng(seed)
    fit = RollingFit(model) if model is not None else None
    pred_err = []
    now, rid = 0.0, 0
    queue, active, finished = [], [], []
    tokens = 0
    opp_ready = opp_granted = 0
    step_ms = []
    for step in range(n_steps):
        lam = arrival_rate(step, n_steps)
        dt = step_ms[-1] if step_ms else 20.0
        for _ in range(rng.poisson(lam * dt / 1e3)):
            queue.append(make_request(rng, rid, now))
            rid += 1
        while queue and len(active) < R_MAX:
            r = queue.pop(0)
            r.last_progress = now  # TPOT counts from the first decode step
            active.append(r)
        if not active:
            step_ms.append(1.0)
            now += 1.0
            continue
        b = batch_of(active, now)
        if ablation == "noslack":
            b.req_slack_ms = np.full(b.n_req, 1e12)
        adm, t_pred = admit_fn(b, policy, rho, fit.model if fit else None)
        if ablation == "noreplan":
            m = np.zeros(b.n_slot, bool)
            off = b.req_slot_off
            for i, r in enumerate(active):
                if r.branches:
                    key = (r.rid, r.phase)
                    if key not in committed:
                        committed[key] = int(adm[off[i]:off[i + 1]].sum())
                    m |= canonical_first(b, i, committed[key])
                else:
                    m[off[i]:off[i + 1]] = True
            if not np.array_equal(m, adm):
                adm = m
                t_pred = predict(fit.model, b, adm) if fit else t_pred
                if set_mask is not None:
                    set_mask(b, adm)
        t = step_fn(b, adm)
        pred_err.append((t - t_pred) / t)
        if fit is not None and refit:
            fit.observe(int(adm.sum()), context_per_request(b, adm), t)
        now += t
        step_ms.append(t)
        opp_ready += b.n_slot - b.n_req
        opp_granted += int(adm.sum()) - b.n_req
        tokens += advance(active, b, adm, now)
        still = []
        for r in active:
            if r.done:
                r.max_gap = max(r.max_gap, 0.0)
                finished.append(r)
            else:
                still.append(r)
        active = still
    met = [r for r in finished if r.max_gap <= SLO_MS]
    secs = now / 1e3
    return {
        "policy": policy, "rho": rho, "steps": n_steps, "sim_seconds": secs,
        "throughput_tok_s": tokens / secs,
        "goodput_tok_s": sum(r.tokens for r in met) / secs,
        "attainment": len(met) / max(1, len(finished)),
        "finished": len(finished),
        "mean_step_ms": float(np.mean(step_ms)), "p99_step_ms": float(np.percentile(step_ms, 99)),
        "admission_rate": opp_granted / max(1, opp_ready),
        "predictor_rel_err_median": float(np.median(pred_err)),
        "predictor_rel_err_p95_abs": float(np.percentile(np.abs(pred_err), 95)),
        "final_model": fit.model if fit else None,
        "ablation": ablation,
    }


# --------------------------------------------------------------------------- GPU drivers
POLICY_ARGS = {"off": ("off", 1), "cap2": ("cap", 2), "cap5": ("cap", 5), "eager": ("eager", 1),
               "taper": ("taper", 1)}


def gpu_drivers(timed_layers):
    import torch
    from paper_2605_06914_b200 import taper as T
    fit = json.load(open(os.path.join(ROOT, "profiles", "latency_model_b200.json")))["per_request"]
    model = (fit["a_ms"] + REST[0], fit["b_ms_per_seq"] + REST[1], fit["c_ms_per_token"])
    ws = torch.empty(T.taper_workspace_size(T.TAPER_MAX_SLOTS, T.TAPER_MAX_SLOTS, 8, 1 << 15),
                     dtype=torch.uint8, device="cuda")
    pool_pages = 24000
    g = torch.Generator(device="cuda").manual_seed(0)
    shape = (pool_pages, 8, 64, 128)
    k = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(shape, generator=g, device="cuda", dtype=torch.bfloat16)
    q = torch.randn((T.TAPER_MAX_SLOTS, 64, 128), generator=g, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(q)
    state = {}

    def admit_fn(b, policy, rho, mdl):
        kind, cap = POLICY_ARGS[policy]
        db = T.DeviceBatch.from_host(b)
        adm = T.DeviceAdmission.empty(b.n_req, b.n_slot)
        T.taper_admit(db, mdl, kind, rho, adm, 8, ws, cap, ctx="per_request")
        state["db"], state["adm"] = db, adm
        return (adm.slot_admitted.cpu().numpy()[:b.n_slot].astype(bool),
                float(adm.diag[2].item()))

    def set_mask(b, adm_mask):
        state["adm"].slot_admitted[:b.n_slot].copy_(torch.from_numpy(adm_mask.astype(np.uint8)))
        T.taper_build_work(state["db"], state["adm"], 8, ws)

    def step_fn(b, adm_mask):
        lay = synth.make_layout(b, 64, np.random.default_rng(len(b.slot_local_len)))
        assert lay.num_pages <= pool_pages, lay.num_pages
        rpo, rp, spo, sp = T.page_tables_to_device(lay)
        spg = torch.as_tensor(np.concatenate([lay.seg_page_off, [0]]).astype(np.int32)).cuda()
        kv = T.DeviceKV(k, v, rpo, rp, spo, sp, spg)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        sc = 1 / math.sqrt(128)
        T.taper_decode_attention(state["db"], state["adm"], kv, q, out, None, sc, ws)  # warm
        per = max(1, timed_layers // 3)
        ev[0].record()
        for i in range(3):  # three blocks of layers; the median block resists timing outliers
            for _ in range(per):
                T.taper_decode_attention(state["db"], state["adm"], kv, q, out, None, sc, ws)
            ev[i + 1].record()
        torch.cuda.synchronize()
        blocks = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        attn = float(np.median(blocks)) * 64 / per
        return attn + REST[0] + REST[1] * int(adm_mask.sum())

    return admit_fn, step_fn, model, set_mask


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1500)
    ap.add_argument("--policies", default="off,cap2,cap5,eager,taper")
    ap.add_argument("--rhos", default="0.5,1.0", help="extra TAPER rho sweep (Table 1)")
    ap.add_argument("--timed-layers", type=int, default=24)
    ap.add_argument("--ablations", default="noslack,noreplan,const",
                    help="Table 1 ablations of TAPER (PAPER.md L217-238)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "closed_loop.json"))
    args = ap.parse_args()
    admit_fn, step_fn, model, set_mask = gpu_drivers(args.timed_layers)
    runs = [(p, 0.8, None) for p in args.policies.split(",")]
    runs += [("taper", float(x), None) for x in args.rhos.split(",") if x]
    runs += [("taper", 0.8, a) for a in args.ablations.split(",") if a]
    res = []
    runs += [("taper-refit", 0.8, None)]  # App. C.2 rolling refresh (unstable here: see DESIGN)
    for p, rho, abl in runs:
        r = run(p.split("-")[0], admit_fn, step_fn, args.steps, rho=rho, model=model,
                refit=p.endswith("-refit"), ablation=abl, set_mask=set_mask)
        r["variant"] = p + (f"-{abl}" if abl else "")
        res.append(r)
        print(json.dumps(r), flush=True)
    off = next(r for r in res if r["variant"] == "off")
    table1 = {r["variant"] + (f"@rho{r['rho']}" if r["rho"] != 0.8 else ""):
              {"goodput_over_off": r["goodput_tok_s"] / off["goodput_tok_s"],
               "attainment": r["attainment"]} for r in res}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"predictor_ms": model, "rest_ms": REST, "slo_ms": SLO_MS, "table1_analog": table1,
               "runs": res}, open(args.out, "w"), indent=1)
    print(json.dumps({"table1_analog": table1}), flush=True)


if __name__ == "__main__":
    main()
