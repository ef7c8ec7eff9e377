"""Per-phase clock64 breakdown of the v8 attention kernel (a library built with -DFP_TIMING).

    nvcc ... -DFP_TIMING -o ab_libs/v8_t.so ...   (see tools/attn_ab2.py for the flags)
    python tools/attn8_timing.py ab_libs/v8_t.so [--workload W] [--dense]

Softmax phases are thread 0 of each row's warpgroup (summed over rows and CTAs, per softmax
tile); issuer phases are the MMA thread (per union entry).
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lib")
ap.add_argument("--workload", default="C3-llama8b-128k")
ap.add_argument("--dense", action="store_true")
ap.add_argument("--v11", action="store_true")
ap.add_argument("--seq-len", type=int, default=None)
a = ap.parse_args()
fp.load_library(os.path.abspath(a.lib))
import torch  # noqa: E402
from synth import gen, configs  # noqa: E402

w = configs.get(a.workload)
if a.seq_len:
    w = w.with_(seq_len=a.seq_len)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
out = torch.empty_like(q)
fpl.plan(q, k, w.tau)
fpl.select(w.gamma, w.min_budget)
run = (lambda: fpl.dense(q, k, v, out)) if a.dense else (lambda: fpl.attn(q, k, v, out))
raw = ctypes.CDLL(os.path.abspath(a.lib))
buf = (ctypes.c_ulonglong * 20)()
dbg = raw.fp_debug_attn8_timing
run()
torch.cuda.synchronize()
dbg(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
dbg(buf, 1)
tiles, ents = max(buf[15], 1), max(buf[14], 1)
print(f"{w.name} {'dense' if a.dense else 'sparse'}: {e0.elapsed_time(e1):.3f} ms, softmax tiles "
      f"(thread 0 of each row) {tiles}, issuer entries {ents}")
names = {0: "wait S", 1: "softmax", 2: "P wait st", 3: "arrive"} if a.v11 else {0: "wait S", 1: "S ld", 2: "max/alpha", 3: "O rescale", 4: "P lo (exp+st)",
         5: "P hi (exp+st)", 6: "loop"}
tot = sum(buf[i] for i in names)
for i, nm in names.items():
    print(f"  softmax {nm:16s} {buf[i] / tiles:8.1f} cyc/tile  {100 * buf[i] / max(tot, 1):5.1f}%")
print(f"  softmax total            {tot / tiles:8.1f} cyc/tile")
inames = {8: "wait K", 9: "wait V", 10: "wait P lo" if not a.v11 else "wait P WG0", 11: "wait P hi" if not a.v11 else "wait P WG1", 12: "issue/other", 13: "S chain issue"}
itot = sum(buf[i] for i in inames)
for i, nm in inames.items():
    print(f"  issuer  {nm:16s} {buf[i] / ents:8.1f} cyc/entry  {100 * buf[i] / max(itot, 1):5.1f}%")
print(f"  issuer total             {itot / ents:8.1f} cyc/entry")

if not a.v11:
    print(f"  handoff p_full -> issuer wake   {buf[16] / ents:8.1f} cyc/entry (row A + B, thread 0's arrival)")
    print(f"  S commit -> softmax wake        {buf[17] / tiles:8.1f} cyc/tile (incl. the S MMAs still executing)")
