"""Greedy / optimum utility ratio of Alg. 1 under operator utilities (SURVEY 8(f) NEXT-3,
reading C-adm-12).  Oracle only (literal Alg. 1 vs App. B brute force) on tiny random
batches; prints min / mean / share of instances below 1 and below 1/2 per utility kind.
usage: python tests/utility_ratio.py [instances]  (test infrastructure: it runs the oracle)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
for kind in ("linear", "concave", "plateau", "weighted"):
    rng = np.random.default_rng(99)
    ratios = []
    while len(ratios) < n:
        b = synth.random_small_batch(rng, max_req=5, max_fanout=4, max_local=40)
        if b.n_slot - b.n_req > 14:
            continue
        util = synth.utility_table(rng, b.n_req, 4, kind)
        model = (rng.uniform(0, 5), rng.uniform(1e-2, 0.5), rng.uniform(1e-4, 1e-2))
        rho = float(rng.uniform(0.1, 1.0))
        g = oracle.admit(b.req_shared_len, b.req_slot_off, b.req_slack_ms, b.slot_local_len,
                         model, "taper", 2, rho, util)
        best = oracle.bruteforce(b.req_shared_len, b.req_slot_off, b.req_slack_ms,
                                 b.slot_local_len, model, rho, util)[0]
        if best <= 0:
            continue
        got = sum(util[r, min(int(g.req_width[r]) - 1, 3)] for r in range(b.n_req))
        ratios.append(got / best)
    r = np.array(ratios)
    print(f"{kind:9s} n={n} min={r.min():.3f} mean={r.mean():.4f} "
          f"below1={np.mean(r < 1 - 1e-12):.3f} below_half={np.mean(r < 0.5):.4f}")
