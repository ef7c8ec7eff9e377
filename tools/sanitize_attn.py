"""One plan/select/sparse-attention layer at a chosen workload, for compute-sanitizer runs
beyond the smoke layer (tools/sanitize.sh covers C1):

    compute-sanitizer --tool synccheck python tools/sanitize_attn.py C2-llama8b-32k [--heads 8]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2502_20766_b200 as fp  # noqa: E402
from synth import configs, gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2-llama8b-32k"
heads = int(sys.argv[sys.argv.index("--heads") + 1]) if "--heads" in sys.argv else None
seq = int(sys.argv[sys.argv.index("--seq-len") + 1]) if "--seq-len" in sys.argv else None
w = configs.get(name)
if seq:
    w = w.with_(seq_len=seq)
if heads:
    w = w.with_(heads=heads, kv_heads=max(1, heads * w.kv_heads // w.heads))
fp.load_library()
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
f = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
out = torch.empty_like(q)
f.layer(q, k, v, out, w.gamma, w.tau, w.min_budget)
f.dense(q, k, v, out)
torch.cuda.synchronize()
print(f"sanitize layer ok: {w.name} heads={w.heads}/{w.kv_heads} n={w.seq_len} nnz={int(f.row_ptr[:, -1].sum())}")
