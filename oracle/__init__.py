"""fp64 CPU oracle for the TAPER hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2605_06914_b200``) never imports it and shares no code with it.

The arithmetic lives in ``taper_oracle.c`` (plain C, ``-ffp-contract=off``);
this module only builds that file with gcc and marshals numpy arrays.  Each
wrapper names the PAPER.md passage its C function follows.

Parity status of each function:
  * ``T``, ``admit``, ``bruteforce``, ``attention``: pinned by
    tests/test_oracle_*.py (worked examples, closed forms, brute force,
    torch SDPA cross-check, invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "taper_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

POLICY_OFF, POLICY_CAP, POLICY_EAGER, POLICY_GREEDY = 0, 1, 2, 3
POLICY_IDS = {"off": POLICY_OFF, "cap": POLICY_CAP, "eager": POLICY_EAGER,
              "taper": POLICY_GREEDY, "greedy": POLICY_GREEDY}
CTX_IDS = {"per_sequence": 0, "per_request": 1}


def build(force: bool = False) -> str:
    """Compile taper_oracle.c -> liboracle.so (gcc, fp64, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-fopenmp", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        lib.oracle_T.restype = f64
        lib.oracle_T.argtypes = [f64, f64, f64, i64, i64]
        lib.oracle_budget.restype = f64
        lib.oracle_budget.argtypes = [f64, f64, f64]
        lib.oracle_admit.restype = ctypes.c_int
        lib.oracle_admit.argtypes = [i32, i32, P, P, P, P, f64, f64, f64, i32, i32, f64,
                                     P, i32, P, P, P, P]
        lib.oracle_admit_ctx.restype = ctypes.c_int
        lib.oracle_admit_ctx.argtypes = [i32, i32, P, P, P, P, f64, f64, f64, i32, i32, f64,
                                         P, i32, i32, P, P, P, P]
        lib.oracle_bruteforce_ctx.restype = ctypes.c_int
        lib.oracle_bruteforce_ctx.argtypes = [i32, i32, P, P, P, P, f64, f64, f64, f64, P, i32,
                                              i32, P, P, P, P]
        lib.oracle_bruteforce.restype = ctypes.c_int
        lib.oracle_bruteforce.argtypes = [i32, i32, P, P, P, P, f64, f64, f64, f64, P, i32,
                                          P, P, P, P]
        lib.oracle_attention.restype = ctypes.c_int
        lib.oracle_attention.argtypes = [i32, P, i32, i32, i32, i32, P, P, P, P, P, P, P, P,
                                         P, i32, P, P, f64, P, P]
        lib.oracle_attention_seg.restype = ctypes.c_int
        lib.oracle_attention_seg.argtypes = [i32, P, i32, i32, i32, i32, P, P, P, P, P, P, P, P,
                                             P, P, P, P, i32, P, P, f64, P, P]
        lib.oracle_set_threads.restype = ctypes.c_int
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_set_threads(1)  # serial unless a caller asks for the host cores
        _lib = lib
    return _lib


def set_threads(n: int) -> int:
    """Host threads for ``attention`` (independent (slot, head) pairs in parallel; each
    pair's arithmetic is unchanged).  Returns the count in effect."""
    return _load().oracle_set_threads(int(n))


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.float64)


def T(a: float, b: float, c: float, n: int, L: int) -> float:
    """App. C.1: T(S) = a + b*n_tokens + c*L_context."""
    return _load().oracle_T(a, b, c, int(n), int(L))


def budget(T0: float, min_slack: float, rho: float) -> float:
    """Sec. 3.3 (L131-137): T0 + rho * max(0, min_slack - T0)."""
    return _load().oracle_budget(T0, min_slack, rho)


@dataclass
class Admission:
    status: int
    req_width: np.ndarray      # [R] int32
    slot_admitted: np.ndarray  # [S] uint8
    T0: float
    budget: float
    T_S: float
    E: float
    min_slack: float
    n_evals: int


def admit(req_shared_len, req_slot_off, req_slack_ms, slot_local_len, model, policy="taper",
          cap=2, rho=0.8, utility=None, ctx="per_sequence") -> Admission:
    """Alg. 1 literally, or a fixed policy (App. D).

    ``model`` = (a, b, c); ``utility`` = None (linear) or [R, K] table u_r(k).
    ``ctx`` = "per_sequence" (the paper's L_context, [C-adm-6]) or "per_request" (the
    prefix counted once per request, NEXT-1).
    """
    Lsh, off, Lloc = _i32(req_shared_len), _i32(req_slot_off), _i32(slot_local_len)
    slack = _f64(req_slack_ms)
    R, S = len(Lsh), len(Lloc)
    width = np.zeros(R, np.int32)
    adm = np.zeros(S, np.uint8)
    diag = np.zeros(5, np.float64)
    nev = np.zeros(1, np.int64)
    util = None if utility is None else _f64(utility)
    ustride = 0 if util is None else util.shape[1]
    a, b, c = (float(x) for x in model)
    st = _load().oracle_admit_ctx(R, S, _p(Lsh), _p(off), _p(slack), _p(Lloc), a, b, c,
                                  POLICY_IDS[policy], int(cap), float(rho), _p(util), ustride,
                                  CTX_IDS[ctx], _p(width), _p(adm), _p(diag), _p(nev))
    if st < 0:
        raise ValueError(f"oracle_admit error {st}")
    return Admission(st, width, adm, *diag.tolist(), int(nev[0]))


def bruteforce(req_shared_len, req_slot_off, req_slack_ms, slot_local_len, model, rho=0.8,
               utility=None, ctx="per_sequence"):
    """App. B (L290-296): best sum_r u_r(k_r) over all feasible subsets.

    Returns (best_utility, best_mask, n_opp, budget)."""
    Lsh, off, Lloc = _i32(req_shared_len), _i32(req_slot_off), _i32(slot_local_len)
    slack = _f64(req_slack_ms)
    util = None if utility is None else _f64(utility)
    ustride = 0 if util is None else util.shape[1]
    bu = np.zeros(1, np.float64)
    bm = np.zeros(1, np.int64)
    no = np.zeros(1, np.int32)
    bg = np.zeros(1, np.float64)
    a, b, c = (float(x) for x in model)
    st = _load().oracle_bruteforce_ctx(len(Lsh), len(Lloc), _p(Lsh), _p(off), _p(slack),
                                       _p(Lloc), a, b, c, float(rho), _p(util), ustride,
                                       CTX_IDS[ctx], _p(bu), _p(bm), _p(no), _p(bg))
    if st < 0:
        raise ValueError(f"oracle_bruteforce error {st}")
    return float(bu[0]), int(bm[0]), int(no[0]), float(bg[0])


def attention(req_slot_off, req_shared_len, slot_local_len, req_page_off, req_pages,
              slot_page_off, slot_pages, k_pages, v_pages, q, eval_slot, eval_qhead,
              scale=None, slot_seg_off=None, seg_len=None, seg_page_off=None):
    """Sec. 3.1 visibility rule (L100-103): fp64 softmax attention of (slot, q-head)
    pairs over the materialised [shared prefix ; branch-local] context.  With
    ``slot_seg_off`` the local context is the concatenation of the slot's segments
    (reduce step, L104-107), segment q holding ``seg_len[q]`` tokens in the page list
    starting at ``slot_pages[seg_page_off[q]]``.

    k_pages/v_pages: [num_pages, h_kv, page, d] bf16 (uint16 bit patterns or torch bf16).
    q: [S, q_heads, d] bf16 bits.  Returns (out [n, d] fp64, lse [n] fp64, natural log).
    """
    k_bits = _bits(k_pages)
    v_bits = _bits(v_pages)
    q_bits = _bits(q)
    _, h_kv, page_size, d = k_bits.shape
    q_heads = q_bits.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)  # [C-att-1]
    es, eh = _i32(eval_slot), _i32(eval_qhead)
    n = len(es)
    out = np.zeros((n, d), np.float64)
    lse = np.zeros(n, np.float64)
    off = _i32(req_slot_off)
    seg = [None, None, None] if slot_seg_off is None else \
        [_i32(slot_seg_off), _i32(seg_len), _i32(seg_page_off)]
    st = _load().oracle_attention_seg(len(off) - 1, _p(off), h_kv, q_heads, d, page_size,
                                      _p(k_bits), _p(v_bits), _p(_i32(req_shared_len)),
                                      _p(_i32(req_page_off)), _p(_i32(req_pages)),
                                      _p(_i32(slot_local_len)), _p(_i32(slot_page_off)),
                                      _p(_i32(slot_pages)), *[_p(a) for a in seg], _p(q_bits),
                                      n, _p(es), _p(eh), float(scale), _p(out), _p(lse))
    if st < 0:
        raise ValueError(f"oracle_attention error {st}")
    return out, lse


def _bits(t) -> np.ndarray:
    """bf16 tensor (torch) or uint16 array -> contiguous uint16 numpy bit patterns."""
    if hasattr(t, "view") and hasattr(t, "dtype") and str(t.dtype) == "torch.bfloat16":
        import torch
        return np.ascontiguousarray(t.detach().cpu().contiguous().view(torch.int16).numpy()
                                    .view(np.uint16))
    a = np.asarray(t)
    if a.dtype != np.uint16:
        raise TypeError("expected bf16 bit patterns (uint16) or a torch.bfloat16 tensor")
    return np.ascontiguousarray(a)
