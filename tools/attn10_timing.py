"""Per-phase clock64 breakdown of the v10 attention kernel (a library built with
-DFP_TIMING -DFP_ATTN_V10, tools/build_variant.sh).

    python tools/attn10_timing.py ab_libs/a_v10t.so [--workload W] [--dense]
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
a = ap.parse_args()
fp.load_library(os.path.abspath(a.lib))
import torch  # noqa: E402
from synth import gen, configs  # noqa: E402

w = configs.get(a.workload)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
out = torch.empty_like(q)
fpl.plan(q, k, w.tau)
fpl.select(w.gamma, w.min_budget)
run = (lambda: fpl.dense(q, k, v, out)) if a.dense else (lambda: fpl.attn(q, k, v, out))
raw = ctypes.CDLL(os.path.abspath(a.lib))
buf = (ctypes.c_ulonglong * 16)()
run()
torch.cuda.synchronize()
raw.fp_debug_attn10_timing(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
raw.fp_debug_attn10_timing(buf, 1)
halves, ents = max(buf[15], 1), max(buf[14], 1)
print(f"{w.name} {'dense' if a.dense else 'sparse'}: {e0.elapsed_time(e1):.3f} ms, softmax halves "
      f"(thread 0 of each row) {halves}, issuer entries {ents}")
names = {0: "wait S", 1: "S ld + max", 2: "pv/rescale", 3: "exp + P st", 4: "loop"}
tot = sum(buf[i] for i in names)
for i, nm in names.items():
    print(f"  softmax {nm:16s} {buf[i] / halves:8.1f} cyc/half  {100 * buf[i] / max(tot, 1):5.1f}%")
print(f"  softmax total            {tot / halves:8.1f} cyc/half")
inames = {8: "wait K", 9: "wait V", 10: "wait P", 11: "S issue", 12: "PV issue", 13: "other"}
itot = sum(buf[i] for i in inames)
for i, nm in inames.items():
    print(f"  issuer  {nm:16s} {buf[i] / ents:8.1f} cyc/entry  {100 * buf[i] / max(itot, 1):5.1f}%")
print(f"  issuer total             {itot / ents:8.1f} cyc/entry")
