"""Configuration sweeps of BASELINE.json configs[3] and configs[4] (1 GPU).

    python tools/sweep.py c4            # GLM-4-9B-like 32/2 at 128k: gamma sweep, min budget 1024 and 0
    python tools/sweep.py c5            # Qwen2-7B 28/4 and Yi-9B 32/4: 4k..128k, tau sweep
    python tools/sweep.py c3            # Llama 32/8 128k at gamma 0.9 and 0.95

One JSON line per point: layer latency (plan+select+attn) and dense latency
(same library, same GPU) from CUDA events, speedup, tokens/s, density,
pattern counts, attention TFLOP/s on computed blocks. Inputs are generated
once per (layout, n) and reused across gamma / tau.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import configs as C  # noqa: E402
from synth import gen  # noqa: E402


def useful_flops(nnz, nb, b=128):
    return sum(4 * 128 * (b * b * (int(x) - nb) + nb * b * (b + 1) // 2) for x in nnz)


def measure(fp, torch, w, q, k, v, fpl, out, steps=5, warmup=2, dense=True, flush=None, opts=None):
    opts = opts or {}
    st = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def timed(fn, n_steps, n_warm):
        for _ in range(n_warm):
            fn()
        torch.cuda.synchronize()
        tot = []
        for _ in range(n_steps):
            if flush is not None:
                flush.zero_()
            a, b = ev(), ev()
            a.record(st)
            fn()
            b.record(st)
            tot.append((a, b))
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b) for a, b in tot]))

    def layer():
        fpl.plan(q, k, w.tau)
        fpl.select(w.gamma, w.min_budget, with_stats=False, **opts)
        fpl.attn(q, k, v, out)


    ms = timed(layer, steps, warmup)
    # the same layer replayed from one CUDA graph (no host launch gaps: short
    # sequences are launch-bound when timed eagerly)
    g = fpl.capture_layer(q, k, v, out, gamma=w.gamma, tau=w.tau, min_budget=w.min_budget) \
        if not opts else None
    ms_graph = timed(g.replay, steps, warmup) if g is not None else None
    gd = None
    if dense:
        import torch as _t
        side = _t.cuda.Stream()
        side.wait_stream(_t.cuda.current_stream())
        with _t.cuda.stream(side):
            fpl.dense(q, k, v, out)
            gd = _t.cuda.CUDAGraph()
            with _t.cuda.graph(gd, stream=side):
                fpl.dense(q, k, v, out)
        _t.cuda.current_stream().wait_stream(side)
    fpl.plan(q, k, w.tau)
    fpl.select(w.gamma, w.min_budget, **opts)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(st)
    fpl.attn(q, k, v, out)
    b.record(st)
    torch.cuda.synchronize()
    attn_ms = a.elapsed_time(b)
    stats = fpl.stats()
    nb = fpl.nb
    nnz = [s_["nnz_blocks"] for s_ in stats]
    pats = [s_["pattern"] for s_ in stats]
    dms = timed(lambda: fpl.dense(q, k, v, out), max(2, steps // 2), 1) if dense else None
    dms_graph = timed(gd.replay, max(2, steps // 2), 1) if gd is not None else None
    return {
        "workload": w.name, "heads": w.heads, "kv_heads": w.kv_heads, "seq_len": w.seq_len,
        "gamma": w.gamma, "tau": w.tau, "min_budget": w.min_budget, "select_options": opts,
        "layer_ms": ms, "tokens_per_s": w.seq_len / (ms / 1e3), "attn_ms": attn_ms,
        "dense_ms": dms, "speedup_vs_dense": (dms / ms) if dms else None,
        "layer_ms_graph": ms_graph, "dense_ms_graph": dms_graph,
        "speedup_vs_dense_graph": (dms_graph / ms_graph) if (dms_graph and ms_graph) else None,
        "density": float(np.sum(nnz)) / (len(nnz) * nb * (nb + 1) / 2),
        "qa_heads": int(np.sum(pats)), "vs_heads": int(len(pats) - np.sum(pats)),
        "budget_added": int(sum(s_["budget_added"] for s_ in stats)),
        "block_size": fpl.b,
        "attn_tflops_useful": useful_flops(nnz, nb, fpl.b) / (attn_ms / 1e3) / 1e12,
        "dense_tflops": (w.heads * 4 * 128 * w.seq_len * (w.seq_len + 1) / 2) / (dms / 1e3) / 1e12
        if dms else None,
    }


def points(which):
    if which == "c3":
        for g in (0.9, 0.95):
            yield C.C3.with_(gamma=g), None
    elif which == "variants":  # next rows f1 / f2 at C3
        for g in (0.9, 0.95):
            for o in ({"vs_mode": 1}, {"qa_mode": 1}, {"max_budget": 16384}, {"max_budget": 32768}):
                yield C.C3.with_(gamma=g), o
    elif which == "c4":
        for mb in (1024, 0):
            for g in C.C4_GAMMAS:
                yield C.C4.with_(gamma=g, min_budget=mb), None
    elif which == "b64":  # next row f3: block size 64 vs 128 on the same inputs
        for bs in (128, 64):
            for g in (0.9, 0.95):
                yield C.C3.with_(gamma=g), {"block_size": bs}
            for n in (8192, 32768):
                yield C.C5_QWEN.with_(seq_len=n, name=f"{C.C5_QWEN.name}-{n // 1024}k"), {"block_size": bs}
    elif which == "c5short":
        for base in (C.C5_QWEN, C.C5_YI):
            for n in (4096, 8192, 16384):
                yield base.with_(seq_len=n, name=f"{base.name}-{n // 1024}k"), None
    elif which == "c5":
        for base in (C.C5_QWEN, C.C5_YI):
            for n in C.C5_LENGTHS:
                for t in C.C5_TAUS:
                    yield base.with_(seq_len=n, tau=t, name=f"{base.name}-{n // 1024}k"), None


def main():
    import torch
    import paper_2502_20766_b200 as fp
    which = sys.argv[1]
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    fp.load_library()
    cache = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    f = open(out_path, "a") if out_path else None
    for w, opts in points(which):
        bs = (opts or {}).pop("block_size", 128) if opts else 128
        opts = opts or None
        key = (w.heads, w.kv_heads, w.seq_len, w.seed, bs)
        if key not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            t = time.time()
            qb, kb, vb = gen.make_layer_bits(w)
            q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in (qb, kb, vb))
            del qb, kb, vb
            fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len, block_size=bs)
            cache[key] = (q, k, v, fpl, torch.empty_like(q))
            print(f"# generated {key} in {time.time() - t:.1f}s", file=sys.stderr, flush=True)
        q, k, v, fpl, out = cache[key]
        steps = 5 if w.seq_len >= 65536 else 10
        r = measure(fp, torch, w, q, k, v, fpl, out, steps=steps, warmup=2, flush=flush, opts=opts)
        line = json.dumps(r)
        print(line, flush=True)
        if f:
            f.write(line + "\n")
            f.flush()


if __name__ == "__main__":
    main()
