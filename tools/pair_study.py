"""K/V-sharing study for the paired attention kernel: for candidate pairings of
(head, q-block) rows inside a KV group, the union of the two rows' key-block
lists (one K/V load per union entry) vs the blocks each row needs.

  loads   = sum over pairs of |A u B|       (K/V tiles fetched, one per entry)
  useful  = sum over rows of |row|          (tiles a v5-style kernel computes)
  issued  = 2 * loads                       (paired M=256 MMAs compute both rows)

    python tools/pair_study.py [workload ...]   (GPU: runs plan + select)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rows_of(row_ptr, col_idx, h, nb):
    rp = row_ptr[h]
    return [set(col_idx[h, rp[q]:rp[q + 1]].tolist()) for q in range(nb)]


def study(rows, pats, H, G, nb):
    g = H // G
    out = {}
    useful = sum(len(r) for hr in rows for r in hr)

    def tally(pairs):
        loads = 0
        for (h1, q1), (h2, q2) in pairs:
            a = rows[h1][q1]
            b = rows[h2][q2] if h2 >= 0 else set()
            loads += len(a | b)
        return loads

    # P1: (h, h^1) at the same q-block
    pairs = []
    for grp in range(G):
        hs = list(range(grp * g, (grp + 1) * g))
        for q in range(nb):
            for i in range(0, len(hs), 2):
                pairs.append(((hs[i], q), (hs[i + 1], q) if i + 1 < len(hs) else (-1, 0)))
    out["P1_same_qb_adjacent_heads"] = tally(pairs)
    # P2: heads of a group sorted by pattern (VS first), then paired at the same q-block
    pairs = []
    for grp in range(G):
        hs = sorted(range(grp * g, (grp + 1) * g), key=lambda h: (pats[h], h))
        for q in range(nb):
            for i in range(0, len(hs), 2):
                pairs.append(((hs[i], q), (hs[i + 1], q) if i + 1 < len(hs) else (-1, 0)))
    out["P2_same_qb_pattern_sorted"] = tally(pairs)
    # P3: same head, adjacent q-blocks (2j+1, 2j)
    pairs = []
    for h in range(H):
        for q in range(nb - 1, -1, -2):
            pairs.append(((h, q), (h, q - 1) if q >= 1 else (-1, 0)))
    out["P3_same_head_adjacent_qb"] = tally(pairs)
    res = {"useful_tiles": useful}
    for k, loads in out.items():
        res[k] = {"loads": loads, "loads_per_useful": round(loads / useful, 4),
                  "issued_over_useful": round(2 * loads / useful, 4)}
    return res


def main():
    import torch
    import paper_2502_20766_b200 as fp
    from synth import configs, gen
    fp.load_library()
    names = sys.argv[1:] or ["C3-llama8b-128k", "C3-llama8b-128k-g0.9", "C4-glm4-9b-128k",
                             "C5-qwen2-7b", "C5-yi-9b"]
    for name in names:
        w = configs.get(name)
        q, k, _ = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
        fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
        fpl.plan(q, k, w.tau)
        fpl.select(w.gamma, w.min_budget)
        st = fpl.stats()
        nb = -(-w.seq_len // 128)
        rp = fpl.row_ptr.cpu().numpy().reshape(w.heads, nb + 1)
        ci = fpl.col_idx.cpu().numpy().reshape(w.heads, -1)
        rows = [rows_of(rp, ci, h, nb) for h in range(w.heads)]
        pats = [s["pattern"] for s in st]
        rec = dict(workload=w.name, seq_len=w.seq_len, gamma=w.gamma, patterns=pats)
        rec.update(study(rows, pats, w.heads, w.kv_heads, nb))
        print(json.dumps(rec), flush=True)
        del q, k, fpl
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
