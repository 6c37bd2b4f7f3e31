"""Seeded synthetic inputs for the TAPER hot path.

This module is shared by the tests, bench.py and smoke(); it serves both the
oracle and the CUDA path and therefore holds NONE of the method's arithmetic:
no latency model, no budget, no admission, no attention.  It only draws batch
states (lengths, fanouts, slack), paged KV layouts and bf16 tensors from seeded
generators, following the recipe in DESIGN.md "Input recipe" (which restates
SURVEY.md Sec. 8(d)):

* Qwen3-32B attention shape: 64 Q heads, 8 KV heads, head_dim 128
  (App. D "Model"); page size 64; HND page pool
  [num_pages, h_kv, page, 128] bf16.
* Fanout pmf matched to Table 4 (P10..P90 = 2,3,4,5,7).
* Serial requests: one ready slot with branch-local length 0 (the whole
  context is the "shared" segment).  Parallel requests: n_r ready branches
  sharing the request's prefix P (+) H, each with its own local tokens.
* Slack: the most urgent request gets exactly ``slack_min_ms``; the others
  ``slack_min_ms + U[0, slack_spread_ms]``.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

Q_HEADS = 64
KV_HEADS = 8
HEAD_DIM = 128
GROUP = Q_HEADS // KV_HEADS
PAGE = 64
N_LAYERS = 64

# Table 4 matched pmf; SURVEY.md Sec. 8(d).
FANOUT_PMF = {2: .20, 3: .25, 4: .25, 5: .15, 6: .04, 7: .04, 8: .03, 9: .02, 10: .02}


@dataclass
class Batch:
    """Batch state in the C-ABI's SoA form (all host numpy arrays)."""
    req_shared_len: np.ndarray   # int32 [R]   Lsh_r
    req_slot_off: np.ndarray     # int32 [R+1] CSR of ready slots
    req_slack_ms: np.ndarray     # float64 [R] d_r(t) - t
    slot_local_len: np.ndarray   # int32 [S]   Lloc_s
    req_serial: np.ndarray = field(default=None)  # bool [R] (info only)
    slot_seg_off: np.ndarray = field(default=None)  # int32 [S+1] local segments, or None
    seg_len: np.ndarray = field(default=None)       # int32 [n_seg]

    @property
    def n_req(self) -> int:
        return int(self.req_shared_len.shape[0])

    @property
    def n_slot(self) -> int:
        return int(self.slot_local_len.shape[0])


@dataclass
class Layout:
    """Paged KV layout: page lists of every shared and local segment."""
    page_size: int
    num_pages: int
    req_page_off: np.ndarray   # int32 [R+1]
    req_pages: np.ndarray      # int32
    slot_page_off: np.ndarray  # int32 [S+1]
    slot_pages: np.ndarray     # int32
    seg_page_off: np.ndarray = None  # int32 [n_seg]: first page of each local segment


def _csr(counts) -> np.ndarray:
    off = np.zeros(len(counts) + 1, np.int64)
    off[1:] = np.cumsum(counts)
    return off.astype(np.int32)


def make_batch(shared_lens, fanouts, local_lens, slack_min_ms=30.0, slack_spread_ms=20.0,
               serial=None, rng=None) -> Batch:
    """Assemble a Batch.  ``fanouts[r]`` ready slots for request r; ``local_lens`` is the
    flat list of Lloc over all slots.  The slack of a random request is exactly
    ``slack_min_ms``; the others get ``+ U[0, slack_spread_ms]``."""
    rng = rng or np.random.default_rng(0)
    R = len(shared_lens)
    slack = slack_min_ms + rng.uniform(0.0, slack_spread_ms, size=R)
    if R:
        slack[rng.integers(R)] = slack_min_ms
    return Batch(np.asarray(shared_lens, np.int32), _csr(fanouts), slack.astype(np.float64),
                 np.asarray(local_lens, np.int32),
                 np.asarray(serial if serial is not None else [f == 1 for f in fanouts], bool))


def sample_fanout(rng, n) -> np.ndarray:
    ks = np.array(list(FANOUT_PMF.keys()))
    ps = np.array(list(FANOUT_PMF.values()))
    return rng.choice(ks, size=n, p=ps / ps.sum())


def config_batch(name: str, seed: int = 0, slack_min_ms: float = 1e3,
                 slack_spread_ms: float = 20.0) -> Batch:
    """The BASELINE.json configs as batch states.

    c1: tiny -- r0 serial (Lsh 512), r1 parallel with 4 branches of Lloc 32.
    c2: 64 requests, 32 serial + 32 parallel (n_r ~ U{2..8}), Lsh 4096, Lloc ~ U{1..256}.
    c3: 32 requests, 16 serial + 16 parallel (n_r ~ U{8..16}), Lsh ~ U[16384, 32768],
        Lloc ~ U{1..512}.
    c5: 256 requests, 128 serial + 128 parallel (Table-4 fanout pmf),
        Lsh log-uniform [1024, 32768], Lloc ~ U{1..256}.
    Serial/parallel requests are interleaved in a seeded random order.
    """
    rng = np.random.default_rng(seed)
    if name == "c1":
        return make_batch([512, 512], [1, 4], [0, 32, 32, 32, 32], slack_min_ms,
                          slack_spread_ms, rng=rng)
    if name == "c2":
        n_ser, n_par = 32, 32
        lsh = lambda n: np.full(n, 4096)
        fan = lambda n: rng.integers(2, 9, size=n)
        lloc_hi = 256
    elif name == "c3":
        n_ser, n_par = 16, 16
        lsh = lambda n: rng.integers(16384, 32769, size=n)
        fan = lambda n: rng.integers(8, 17, size=n)
        lloc_hi = 512
    elif name == "c5":
        n_ser, n_par = 128, 128
        lsh = lambda n: np.exp(rng.uniform(np.log(1024), np.log(32768), size=n)).astype(np.int64)
        fan = lambda n: sample_fanout(rng, n)
        lloc_hi = 256
    else:
        raise ValueError(f"unknown config {name!r}")
    kinds = np.array([True] * n_ser + [False] * n_par)
    rng.shuffle(kinds)
    R = len(kinds)
    shared = lsh(R)
    fanouts = np.where(kinds, 1, fan(R))
    local = []
    for r in range(R):
        if kinds[r]:
            local.append(0)
        else:
            local.extend(rng.integers(1, lloc_hi + 1, size=int(fanouts[r])).tolist())
    return make_batch(shared, fanouts, local, slack_min_ms, slack_spread_ms, serial=kinds,
                      rng=rng)


def random_small_batch(rng, max_req=6, max_fanout=5, max_shared=4096, max_local=64,
                       slack_range=(5.0, 60.0)) -> Batch:
    """Small random batch for admission fuzzing (ties in Lloc are likely)."""
    R = int(rng.integers(1, max_req + 1))
    fanouts = rng.integers(1, max_fanout + 1, size=R)
    shared = rng.integers(0, max_shared + 1, size=R)
    local = rng.integers(0, max_local + 1, size=int(fanouts.sum()))
    b = make_batch(shared, fanouts, local, 0.0, 0.0, rng=rng)
    b.req_slack_ms = rng.uniform(*slack_range, size=R)
    return b


def make_layout(batch: Batch, page_size: int = PAGE, rng=None, spare_pages: int = 0,
                local_capacity: int | None = None, contiguous: bool = False) -> Layout:
    """Give every shared segment ceil(Lsh/page) pages and every slot's local segment
    ceil(max(Lloc, local_capacity)/page) pages, drawn as a random permutation of
    the pool (so segments are not contiguous).  A batch with local segments gets
    ceil(seg_len/page) pages per segment instead (each segment starts on a page)."""
    rng = rng or np.random.default_rng(1)
    if batch.slot_seg_off is not None:
        need_sh = (batch.req_shared_len.astype(np.int64) + page_size - 1) // page_size
        need_seg = (batch.seg_len.astype(np.int64) + page_size - 1) // page_size
        total = int(need_sh.sum() + need_seg.sum()) + spare_pages
        perm = rng.permutation(max(total, 1)).astype(np.int32)
        seg_page_off = _csr(need_seg)
        so = batch.slot_seg_off
        per_slot = [int(need_seg[so[i]:so[i + 1]].sum()) for i in range(batch.n_slot)]
        return Layout(page_size, max(total, 1), _csr(need_sh),
                      np.ascontiguousarray(perm[: need_sh.sum()]), _csr(per_slot),
                      np.ascontiguousarray(perm[need_sh.sum(): need_sh.sum() + need_seg.sum()]),
                      np.ascontiguousarray(seg_page_off[:-1]))
    need_sh = (batch.req_shared_len.astype(np.int64) + page_size - 1) // page_size
    loc = batch.slot_local_len.astype(np.int64)
    if local_capacity is not None:
        loc = np.maximum(loc, local_capacity)
    need_loc = (loc + page_size - 1) // page_size
    total = int(need_sh.sum() + need_loc.sum()) + spare_pages
    perm = (np.arange(max(total, 1)) if contiguous else rng.permutation(max(total, 1))).astype(np.int32)
    req_pages = perm[: need_sh.sum()]
    slot_pages = perm[need_sh.sum(): need_sh.sum() + need_loc.sum()]
    return Layout(page_size, max(total, 1), _csr(need_sh), np.ascontiguousarray(req_pages),
                  _csr(need_loc), np.ascontiguousarray(slot_pages))


def make_kv(num_pages, h_kv=KV_HEADS, page_size=PAGE, d=HEAD_DIM, seed=0, device="cpu"):
    """K, V pools [num_pages, h_kv, page, d] bf16 ~ N(0, 1)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    shape = (num_pages, h_kv, page_size, d)
    k = torch.randn(shape, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    v = torch.randn(shape, generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    return k, v


def make_q(n_slot, q_heads=Q_HEADS, d=HEAD_DIM, seed=0, gain=1.0, device="cpu"):
    """Queries [S, q_heads, d] bf16 ~ N(0, gain^2) ("peaked" variant: gain 4)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed + 7919)
    q = torch.randn((n_slot, q_heads, d), generator=g, device=device, dtype=torch.float32)
    return (q * gain).to(torch.bfloat16)


def plant_sink(k_pages, q, batch: Batch, layout: Layout, gain: float = 32.0):
    """"sink" variant: overwrite prefix token 0 of each request and KV head with a key
    aligned to the mean of that request's queries of the GQA group, so one key
    dominates the softmax.  In place on CPU tensors."""
    import torch
    h_kv = k_pages.shape[1]
    group = q.shape[1] // h_kv
    off = batch.req_slot_off
    for r in range(batch.n_req):
        if batch.req_shared_len[r] < 1 or off[r + 1] == off[r]:
            continue
        page = int(layout.req_pages[layout.req_page_off[r]])
        for g in range(h_kv):
            qq = q[off[r]:off[r + 1], g * group:(g + 1) * group].float().reshape(-1, q.shape[2])
            mean = qq.mean(0)
            k_pages[page, g, 0] = (gain * mean / mean.norm().clamp_min(1e-6)).to(torch.bfloat16)


class TraceReplay:
    """Config 4: 1000 decode steps of the C2 shape with branch progression.

    Workload dynamics only (no admission, no latency model): the caller supplies the
    admitted-slot mask of each step (from whichever admission it is testing) and this
    class advances the state:
      * every admitted slot generates one token (serial: shared context +1; branch: +1);
      * a branch reaching its target length (~U{32..512}) completes and leaves the ready
        set; when every branch of a phase completed, the request enters a reduce stretch
        (serial) whose context is P (+) H (+) all branches in canonical order (P104-107),
        lasting U{16..128} tokens, then with probability 0.5 opens a new parallel phase
        (Table-4 fanout, each branch starting with 1 local token) or stays serial.
    ``slack_x(step)`` gives the regime schedule of SURVEY Sec. 8(d): x ~ U[1.2, 2] for
    steps 0-399 (low load), U[-0.5, 0.25] for 400-649 (high), U[0.25, 0.75] after.
    """

    def __init__(self, seed=0):
        self.rng = np.random.default_rng(seed)
        b = config_batch("c2", seed=seed)
        self.lsh = b.req_shared_len.astype(np.int64).tolist()
        off = b.req_slot_off
        self.branches = []   # per request: list of [local_len, target] (empty = serial)
        self.serial_left = []
        for r in range(b.n_req):
            if b.req_serial[r]:
                self.branches.append([])
                self.serial_left.append(None)  # serial forever
            else:
                self.branches.append([[int(b.slot_local_len[s]),
                                       int(self.rng.integers(max(32, b.slot_local_len[s] + 1), 513))]
                                      for s in range(off[r], off[r + 1])])
                self.serial_left.append(0)
        self.step_idx = 0

    def slack_x(self, step=None):
        step = self.step_idx if step is None else step
        if step < 400:
            return float(self.rng.uniform(1.2, 2.0))
        if step < 650:
            return float(self.rng.uniform(-0.5, 0.25))
        return float(self.rng.uniform(0.25, 0.75))

    def batch(self, slack_min_ms=0.0) -> Batch:
        fan, loc = [], []
        for r, br in enumerate(self.branches):
            if br:
                fan.append(len(br))
                loc += [l for l, _ in br]
            else:
                fan.append(1)
                loc.append(0)
        return make_batch(self.lsh, fan, loc, slack_min_ms, 20.0, rng=self.rng)

    def advance(self, slot_admitted):
        s = 0
        for r, br in enumerate(self.branches):
            if not br:
                if slot_admitted[s]:
                    self.lsh[r] += 1
                    if self.serial_left[r] is not None and self.serial_left[r] > 0:
                        self.serial_left[r] -= 1
                        if self.serial_left[r] == 0 and self.rng.random() < 0.5:
                            n = int(sample_fanout(self.rng, 1)[0])
                            self.branches[r] = [[1, int(self.rng.integers(32, 513))]
                                                for _ in range(n)]
                s += 1
                continue
            done = []
            for i in range(len(br)):
                if slot_admitted[s + i]:
                    br[i][0] += 1
                    if br[i][0] >= br[i][1]:
                        done.append(i)
            s += len(br)
            if done:
                self._finished = getattr(self, "_finished", {})
                fin = self._finished.setdefault(r, [])
                fin += [br[i][0] for i in done]
                self.branches[r] = [x for i, x in enumerate(br) if i not in done]
                if not self.branches[r]:
                    # reduce phase: context = prefix (+) all completed branches
                    self.lsh[r] += sum(self._finished.pop(r))
                    self.serial_left[r] = int(self.rng.integers(16, 129))
        self.step_idx += 1


def utility_table(rng, R: int, K: int, kind: str = "concave") -> np.ndarray:
    """Operator-supplied utility curves u_r(k), k = 0..K-1 (Sec. 3.4), as a float64
    [R, K] table with u_r(0) = 0 and non-decreasing columns.  Kinds (input shapes only):
      linear   u_r(k) = k (the paper's default)
      weighted u_r(k) = w_r k, w_r in {1, 2, 5, 10} ("priority operators weight by tenant")
      concave  increments non-increasing in k ("the first opportunistic branch matters more")
      plateau  concave, with zero increments after a random k (a request that wants no more)
    """
    k = np.arange(K, dtype=np.float64)
    if kind == "linear":
        return np.tile(k, (R, 1))
    if kind == "weighted":
        w = rng.choice([1.0, 2.0, 5.0, 10.0], size=R)
        return w[:, None] * k[None, :]
    inc = np.sort(rng.uniform(0.05, 4.0, size=(R, K - 1)), axis=1)[:, ::-1]
    if kind == "plateau":
        stop = rng.integers(0, K, size=R)
        inc = np.where(np.arange(K - 1)[None, :] >= stop[:, None], 0.0, inc)
    elif kind != "concave":
        raise ValueError(kind)
    return np.concatenate([np.zeros((R, 1)), np.cumsum(inc, axis=1)], axis=1)


def with_segments(batch: Batch, seg_lens_per_slot) -> Batch:
    """Attach multi-segment local contexts: ``seg_lens_per_slot[s]`` lists the lengths of
    slot s's local segments in order (their sum becomes Lloc_s)."""
    counts = [len(x) for x in seg_lens_per_slot]
    flat = [int(v) for x in seg_lens_per_slot for v in x]
    batch.slot_seg_off = _csr(counts)
    batch.seg_len = np.asarray(flat, np.int32)
    batch.slot_local_len = np.asarray([sum(x) for x in seg_lens_per_slot], np.int32)
    return batch


def reduce_batch(seed: int = 0, n_serial=16, n_parallel=16, n_reduce=16, prefix=4096,
                 slack_min_ms=1e3) -> Batch:
    """Reduce-step mix (Sec. 3.1): serial requests,
    parallel-phase requests (Table-4 fanout, one local segment of U{1..256} per branch) and
    reduce-phase requests whose single slot sees P (+) H (shared, ``prefix`` tokens) then
    every finished branch's h_i (+) y_i in canonical order (n ~ Table-4 fanout, lengths
    U{32..512}) then the reduce tokens z so far (U{1..128}) -- each a segment in its own
    pages, so the step reads the branches' KV where it lies."""
    rng = np.random.default_rng(seed)
    R = n_serial + n_parallel + n_reduce
    kinds = rng.permutation(np.array([0] * n_serial + [1] * n_parallel + [2] * n_reduce))
    fan, segs = [], []
    for k in kinds:
        if k == 0:
            fan.append(1)
            segs.append([])
        elif k == 1:
            n = int(sample_fanout(rng, 1)[0])
            fan.append(n)
            segs += [[int(rng.integers(1, 257))] for _ in range(n)]
        else:
            n = int(sample_fanout(rng, 1)[0])
            fan.append(1)
            segs.append([int(x) for x in rng.integers(32, 513, size=n)] + [int(rng.integers(1, 129))])
    b = make_batch(np.full(R, prefix), fan, [sum(x) for x in segs], slack_min_ms, 20.0,
                   serial=kinds != 1, rng=rng)
    return with_segments(b, segs)
