"""Per-phase clock64 breakdown of the attention softmax loop (build with -DFP_TIMING).

    python -m paper_2502_20766_b200.build  # normal
    FP_LIB=... python tools/attn_timing.py
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402
from paper_2502_20766_b200 import build as B  # noqa: E402

emu = os.environ.get("FP_EMU", "20")
rt = os.environ.get("FP_RT", "8.0f")
timing = os.environ.get("FP_TIMING", "1") == "1"
lib_t = os.path.join(ROOT, "gpurun_out", f"libflexprefill_t{int(timing)}_emu{emu}_rt{rt}.so")
if not os.path.exists(lib_t) or "--rebuild" in sys.argv:
    cmd = [B.NVCC, *B.FLAGS, *(["-DFP_TIMING"] if timing else []), f"-DFP_EMU={emu}",
           f"-DFP_RT={rt}", "-o", lib_t] + \
        [os.path.join(B.CSRC, x) for x in B.SOURCES]
    subprocess.check_call(cmd)
fp.load_library(lib_t)
import torch  # noqa: E402
from synth import gen, configs  # noqa: E402

w = configs.get(sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "C3-llama8b-128k")
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
out = torch.empty_like(q)
fpl.plan(q, k, w.tau)
fpl.select(w.gamma, w.min_budget)
fpl.attn(q, k, v, out)
torch.cuda.synchronize()
raw = ctypes.CDLL(lib_t)
buf = (ctypes.c_ulonglong * 16)()
if timing:
    raw.fp_debug_attn_timing(buf, 1)
fpl.attn(q, k, v, out)
torch.cuda.synchronize()
if timing:
    raw.fp_debug_attn_timing(buf, 1)
else:
    buf[8] = 1
tiles = buf[8]
names = ["wait S", "S ld", "softmax", "-", "O rescale", "P pack+st", "arrive", "loop"]
tot = sum(buf[i] for i in range(8))
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
fpl.attn(q, k, v, out)
t1.record()
torch.cuda.synchronize()
ms = []
for _ in range(3):
    t0.record()
    fpl.attn(q, k, v, out)
    t1.record()
    torch.cuda.synchronize()
    ms.append(t0.elapsed_time(t1))
print(f"emu={emu} rt={rt} best_of3_ms={min(ms):.3f} attn_ms={t0.elapsed_time(t1):.3f} tiles={tiles} cycles/tile={tot / tiles:.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:14s} {buf[i] / tiles:8.1f} cyc/tile  {100 * buf[i] / tot:5.1f}%")
