"""A/B timing of fp_plan and fp_select from several library builds in one
process (ctypes, RTLD_LOCAL), same inputs, alternating blocks of launches.

    python tools/plan_ab.py lib_a.so lib_b.so [...] [--workload W] [--seq-len N]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--workload", default="C3-llama8b-128k")
ap.add_argument("--seq-len", type=int, default=None)
ap.add_argument("--blocks", type=int, default=3)
ap.add_argument("--block-len", type=int, default=10)
a = ap.parse_args()

fp.load_library()
import torch  # noqa: E402
from synth import configs, gen  # noqa: E402

w = configs.get(a.workload)
if a.seq_len:
    w = w.with_(seq_len=a.seq_len)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
P, I, Z, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_float
libs = []
for p in a.libs:
    L = ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL)
    L.fp_plan.argtypes = [P, P, I, I, I, I, I, F, P, Z, P, P, P]
    L.fp_select.argtypes = [I, I, I, I, I, F, I, P, Z, P, P, P, P]
    L.fp_workspace_bytes.restype = Z
    L.fp_workspace_bytes.argtypes = [I, I, I, I, I]
    libs.append(L)
# one workspace large enough for every build's layout
wsb = max(L.fp_workspace_bytes(w.heads, w.kv_heads, w.seq_len, 128, 128) for L in libs)
if wsb > fpl.ws_bytes:
    fpl.ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    fpl.ws_bytes = wsb
st = torch.cuda.current_stream().cuda_stream


def plan(L):
    assert L.fp_plan(q.data_ptr(), k.data_ptr(), w.heads, w.kv_heads, w.seq_len, 128, 128, w.tau,
                     fpl.ws.data_ptr(), fpl.ws_bytes, fpl.pattern.data_ptr(), fpl.jsd.data_ptr(),
                     st) == 0


def select(L):
    assert L.fp_select(w.heads, w.kv_heads, w.seq_len, 128, 128, w.gamma, w.min_budget,
                       fpl.ws.data_ptr(), fpl.ws_bytes, fpl.row_ptr.data_ptr(),
                       fpl.col_idx.data_ptr(), None, st) == 0


outs = []
for L in libs:
    plan(L)
    select(L)
    torch.cuda.synchronize()
    outs.append((fpl.jsd.clone(), fpl.row_ptr.clone(), fpl.col_idx.clone()))
for i in range(1, len(libs)):
    print(f"lib {i}: max |d jsd| {(outs[i][0] - outs[0][0]).abs().max().item():.2e}, "
          f"row_ptr equal {torch.equal(outs[i][1], outs[0][1])}, "
          f"col_idx equal {torch.equal(outs[i][2], outs[0][2])}")
res = {p: {"plan": [], "select": []} for p in a.libs}
for _ in range(a.blocks):
    for p, L in zip(a.libs, libs):
        for name, fn in (("plan", plan), ("select", select)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.block_len):
                fn(L)
            e1.record()
            torch.cuda.synchronize()
            res[p][name].append(e0.elapsed_time(e1) / a.block_len)
for p in a.libs:
    print(f"{os.path.basename(p):16s} {w.name} n={w.seq_len}: plan {np.median(res[p]['plan']):.4f} ms  "
          f"select {np.median(res[p]['select']):.4f} ms")
