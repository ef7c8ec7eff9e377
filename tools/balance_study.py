"""Per-head cost (useful attention FLOPs from the selected CSR) and the rank
imbalance max_r F_r / mean_r F_r of the static contiguous head partition vs
LPT, for P = 2, 4, 8 (SURVEY.md §8(e) "scaling limiter"; next row f4).

    python tools/balance_study.py [workload ...]   (GPU: runs plan + select)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2502_20766_b200 import dist as D  # noqa: E402


def main():
    import torch
    import paper_2502_20766_b200 as fp
    from synth import configs, gen
    fp.load_library()
    names = sys.argv[1:] or ["C3-llama8b-128k", "C3-llama8b-128k-g0.9", "C4-glm4-9b-128k",
                             "C5-qwen2-7b", "C5-yi-9b"]
    for name in names:
        w = configs.get(name)
        if w.seq_len < 131072 and name.startswith("C5"):
            w = w.with_(seq_len=131072)
        q, k, _ = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
        fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
        fpl.plan(q, k, w.tau)
        fpl.select(w.gamma, w.min_budget)
        st = fpl.stats()
        nb = -(-w.seq_len // 128)
        costs = [D.head_cost(s["nnz_blocks"], nb) for s in st]
        rec = dict(workload=w.name, heads=w.heads, kv_heads=w.kv_heads, seq_len=w.seq_len,
                   gamma=w.gamma, patterns=[s["pattern"] for s in st],
                   nnz=[s["nnz_blocks"] for s in st])
        for P in (2, 4, 8):
            rec[f"static_P{P}"] = round(D.imbalance(costs, D.static_assignment(w.heads, P)), 4)
            rec[f"lpt_P{P}"] = round(D.imbalance(costs, D.lpt_assign(costs, P)), 4)
        print(json.dumps(rec), flush=True)
        del q, k, fpl
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
