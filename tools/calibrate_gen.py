"""Generator calibration (test tooling; runs the oracle's plan + select only).

Prints, per sampled head: type, D_JS, pattern, K_v/K_s/K_qa and the block
density of the final mask, so the gains in synth/gen.py can be tuned against
SURVEY.md §8(d)'s calibration target (VS density ~0.25-0.30 at gamma 0.9 and
~0.35-0.45 at 0.95 at 128k; both patterns trigger with margin around tau).
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import gen  # noqa: E402
from synth.configs import Workload  # noqa: E402
import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[2048, 8192, 32768])
    ap.add_argument("--H", type=int, default=32)
    ap.add_argument("--G", type=int, default=8)
    ap.add_argument("--heads", type=int, nargs="+", default=[0, 1, 3, 4, 7])
    ap.add_argument("--gamma", type=float, nargs="+", default=[0.9, 0.95])
    ap.add_argument("--seed", type=int, default=103)
    a = ap.parse_args()
    for n in a.n:
        w = Workload("cal", a.H, a.G, n, 0.9, 0.1, 0, a.seed)
        for h in a.heads:
            t0 = time.time()
            g = h * a.G // a.H
            Q = gen.bits_to_f64(gen.bf16_bits(gen.make_q(w.seed, a.H, a.G, n, h)))
            K = gen.bits_to_f64(gen.bf16_bits(gen.make_k(w.seed, a.H, a.G, n, g)))
            plan = oracle.plan_head(Q, K, 128, 0.1)
            nb = n // 128
            tot = nb * (nb + 1) // 2
            dens = []
            for gm in a.gamma:
                s = oracle.select_head(plan, Q, K, 128, gm, 0)
                ks = (s["tv"]["K"], s["ts"]["K"]) if plan["pattern"] == oracle.VS else (s["tq"]["K"],)
                dens.append((gm, ks, s["mask"].sum() / tot))
            typ = "QA" if gen.is_qa_type(h, a.H, a.G) else "VS"
            meta = gen.kv_meta(w.seed, a.H, a.G, n, g)
            av, as_ = plan["a_v"], plan["a_s"]
            sink = av[:4].sum()
            vert = av[meta["verts"]].sum()
            loc = as_[:256].sum()
            print(f"   mass on representative rows: sink={sink:.3f} heavy-hitters={vert:.3f} "
                  f"local(o<256)={loc:.3f}")
            print(f"n={n:6d} h={h:2d} {typ} D={plan['D']:.4f} pat={'QA' if plan['pattern'] else 'VS'} "
                  f"sink={sink:.3f} " + " ".join(f"g{gm}:K={ks} dens={d:.3f}" for gm, ks, d in dens)
                  + f" ({time.time()-t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
