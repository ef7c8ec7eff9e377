"""Whole layer as one stream (plan -> select -> attention for all heads) vs the
KV groups as independent chains on up to 4 streams (plan/select of one group
overlapping the attention of another), both replayed from CUDA graphs.

    python tools/layer_streams.py [--workload W] [--seq-len N] [--streams 4]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C5-qwen2-7b")
ap.add_argument("--seq-len", type=int, default=None)
ap.add_argument("--streams", type=int, default=4)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
fp.load_library()
import torch  # noqa: E402
from synth import configs, gen  # noqa: E402

w = configs.get(a.workload)
if a.seq_len:
    w = w.with_(seq_len=a.seq_len)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
H, G, n = w.heads, w.kv_heads, w.seq_len
g = H // G
out1 = torch.empty_like(q)
out2 = torch.empty_like(q)
whole = fp.FlexPrefill(H, G, n)
groups = [fp.FlexPrefill(g, 1, n) for _ in range(G)]
S = min(a.streams, G)
main = torch.cuda.Stream()
side = [torch.cuda.Stream() for _ in range(S)]


def one_stream():
    whole.plan(q, k, w.tau, main)
    whole.select(w.gamma, w.min_budget, main, with_stats=False)
    whole.attn(q, k, v, out1, main)


def multi_stream():
    ev0 = torch.cuda.Event()
    ev0.record(main)
    done = []
    for c in range(G):
        s = side[c % S]
        s.wait_event(ev0)
        f = groups[c]
        qs, ks, vs, os_ = q[c * g:(c + 1) * g], k[c:c + 1], v[c:c + 1], out2[c * g:(c + 1) * g]
        f.plan(qs, ks, w.tau, s)
        f.select(w.gamma, w.min_budget, s, with_stats=False)
        f.attn(qs, ks, vs, os_, s)
    for s in side:
        e = torch.cuda.Event()
        e.record(s)
        main.wait_event(e)


def capture(fn):
    torch.cuda.synchronize()
    with torch.cuda.stream(main):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=main):
        fn()
    torch.cuda.synchronize()
    return gr


g1, g2 = capture(one_stream), capture(multi_stream)
res = {"one stream": [], f"{S} streams": []}
for _ in range(a.reps):
    for name, gr in (("one stream", g1), (f"{S} streams", g2)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(main):
            e0.record(main)
            gr.replay()
            e1.record(main)
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1))
torch.cuda.synchronize()
print(f"{w.name} n={n}: max |out1 - out2| = {(out1.float() - out2.float()).abs().max().item():.3e}")
for name, t in res.items():
    print(f"  {name:12s} median {np.median(t):.4f} ms  min {np.min(t):.4f}")
