"""A/B timing of fp_sparse_attn across library builds (same inputs, CUDA events).

    python tools/attn_ab.py path/to/lib.so [workload] [gamma]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402

fp.load_library(sys.argv[1])
import torch  # noqa: E402
from synth import gen, configs  # noqa: E402

w = configs.get(sys.argv[2] if len(sys.argv) > 2 else "C3-llama8b-128k")
if len(sys.argv) > 3:
    w = w.with_(gamma=float(sys.argv[3]))
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
out = torch.empty_like(q)
fpl.plan(q, k, w.tau)
fpl.select(w.gamma, w.min_budget)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {}
for name, fn in (("attn", lambda: fpl.attn(q, k, v, out)), ("dense", lambda: fpl.dense(q, k, v, out))):
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(4):
        a, b = ev(), ev()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    res[name] = min(ms)
print(f"{os.path.basename(sys.argv[1])} {w.name} g={w.gamma}: attn {res['attn']:.3f} ms  dense {res['dense']:.3f} ms")
