"""Run fp_plan + fp_select a few times on a workload (for ncu launch lists and
captures of the stage-(i)/(ii) kernels).

    python tools/plan_run.py [--workload W] [--seq-len N] [--iters K]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3-llama8b-128k")
ap.add_argument("--seq-len", type=int, default=None)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--attn", action="store_true")
a = ap.parse_args()
fp.load_library()
import torch  # noqa: E402
from synth import configs, gen  # noqa: E402

w = configs.get(a.workload)
if a.seq_len:
    w = w.with_(seq_len=a.seq_len)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
out = torch.empty_like(q)
for _ in range(a.iters):
    fpl.plan(q, k, w.tau)
    fpl.select(w.gamma, w.min_budget, with_stats=False)
    if a.attn:
        fpl.attn(q, k, v, out)
torch.cuda.synchronize()
print("ok", w.name, w.seq_len)
