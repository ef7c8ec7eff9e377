"""paper_2502_20766_b200 -- FlexPrefill sparse prefill attention on B200 (sm_100a).

Thin Python binding of libflexprefill.so (include/flexprefill.h). Argument
marshalling only: every step of the method runs in the library's CUDA
kernels. torch is used for device memory and streams. There is no CPU or
PyTorch fallback: if the library is missing or the device is not sm_100,
calls raise.

    import paper_2502_20766_b200 as fp
    fpl = fp.FlexPrefill(heads=32, kv_heads=8, seq_len=131072)
    fpl.plan(q, k, tau=0.1)           # Alg. 2 (+ line scores / pooled map)
    fpl.select(gamma=0.95)            # Alg. 3 / 4, forced blocks, min budget
    fpl.attn(q, k, v, out)            # y = A(Q, K, V, S)
"""
import ctypes
import os

__all__ = [
    "FlexPrefill", "FlexPrefillError", "load_library", "fp_workspace_bytes", "fp_col_idx_capacity",
    "fp_plan", "fp_select", "fp_select_ex", "fp_sparse_attn", "SelectOptions", "fp_dense_causal_attn", "fp_layer_host",
    "fp_debug_view", "fp_kernels_per_layer", "LIB_PATH", "SelectStats", "Layout", "fp_layout_bhsd",
    "fp_layout_bshd", "fp_plan_ex", "fp_sparse_attn_ex", "fp_dense_causal_attn_ex",
]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libflexprefill.so")

FP_STATUS = {0: "ok", 1: "null pointer", 2: "invalid shape", 3: "parameter out of range",
             4: "pointer not 16-byte aligned", 5: "workspace too small",
             6: "device is not sm_100 (B200)", 7: "CUDA launch error"}


class FlexPrefillError(RuntimeError):
    def __init__(self, fn, status, cuda_err=0):
        self.status = status
        msg = f"{fn} failed: {FP_STATUS.get(status, status)} (fp_status={status}"
        if status == 7:
            msg += f", cudaError={cuda_err}"
        super().__init__(msg + ")")


class SelectStats(ctypes.Structure):
    _fields_ = [("k_v", ctypes.c_int32), ("k_s", ctypes.c_int32), ("k_qa", ctypes.c_int32),
                ("nnz_blocks", ctypes.c_int32), ("budget_added", ctypes.c_int32),
                ("pattern", ctypes.c_int32), ("budget_removed", ctypes.c_int32),
                ("mass_v", ctypes.c_double), ("mass_s", ctypes.c_double),
                ("mass_qa", ctypes.c_double)]


class SelectOptions(ctypes.Structure):
    """fp_select_options: vs_mode (0 = element lines, 1 = block-pooled lines, f1),
    qa_mode (0 = flattened map, 1 = per query block, f2), max_budget (tokens, 0 = off)."""
    _fields_ = [("vs_mode", ctypes.c_int32), ("qa_mode", ctypes.c_int32),
                ("max_budget", ctypes.c_int32)]


class Layout(ctypes.Structure):
    """fp_layout: batch and per-tensor {batch, head, row} strides in elements."""
    _fields_ = [("batch", ctypes.c_int32), ("q_stride", ctypes.c_int64 * 3),
                ("k_stride", ctypes.c_int64 * 3), ("v_stride", ctypes.c_int64 * 3),
                ("o_stride", ctypes.c_int64 * 3)]


class DebugPtrs(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "a_v", "a_s", "a_hat", "a_bar", "k_bar", "q_bar", "A_bar", "As",
        "sel_v", "sel_s", "sel_qa", "sel_count", "row_nnz_pre", "attn_sched")]


_lib = None
_P, _I, _F, _Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t


def load_library(path=LIB_PATH):
    """Load libflexprefill.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2502_20766_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    sig = {
        "fp_workspace_bytes": (_Z, [_I, _I, _I, _I, _I]),
        "fp_col_idx_capacity": (_Z, [_I, _I]),
        "fp_plan": (_I, [_P, _P, _I, _I, _I, _I, _I, _F, _P, _Z, _P, _P, _P]),
        "fp_select": (_I, [_I, _I, _I, _I, _I, _F, _I, _P, _Z, _P, _P, _P, _P]),
        "fp_select_ex": (_I, [_I, _I, _I, _I, _I, _F, _I, ctypes.POINTER(SelectOptions), _P, _Z,
                              _P, _P, _P, _P]),
        "fp_sparse_attn": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _Z, _P]),
        "fp_dense_causal_attn": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _Z, _P]),
        "fp_layer_host": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _F, _F, _I,
                               _P, _Z, _P, _P, _P, _P, _P]),
        "fp_debug_view": (_I, [_P, _I, _I, _I, _I, _I, ctypes.POINTER(DebugPtrs)]),
        "fp_layout_bhsd": (_I, [_I, _I, _I, _I, ctypes.POINTER(Layout)]),
        "fp_layout_bshd": (_I, [_I, _I, _I, _I, ctypes.POINTER(Layout)]),
        "fp_plan_ex": (_I, [_P, _P, _I, _I, _I, _I, _I, ctypes.POINTER(Layout), _F, _P, _Z, _P, _P,
                            _P]),
        "fp_sparse_attn_ex": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, ctypes.POINTER(Layout), _P,
                                   _P, _P, _Z, _P]),
        "fp_dense_causal_attn_ex": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, ctypes.POINTER(Layout),
                                         _P, _Z, _P]),
        "fp_sparse_attn_peers": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I,
                                      ctypes.POINTER(Layout), _P, _P, _P, _Z, _P]),
        "fp_kernels_per_layer": (_I, []),
        "fp_status_string": (ctypes.c_char_p, [_I]),
        "fp_last_cuda_error": (_I, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _L():
    return _lib if _lib is not None else load_library()


def _check(fn, st):
    if st != 0:
        raise FlexPrefillError(fn, st, _L().fp_last_cuda_error())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------- C-ABI mirrors ---
def fp_workspace_bytes(heads, kv_heads, seq_len, head_dim=128, block_size=128):
    return _L().fp_workspace_bytes(heads, kv_heads, seq_len, head_dim, block_size)


def fp_col_idx_capacity(seq_len, block_size=128):
    return _L().fp_col_idx_capacity(seq_len, block_size)


def fp_kernels_per_layer():
    return _L().fp_kernels_per_layer()


def fp_plan(q, k, heads, kv_heads, seq_len, tau, ws, ws_bytes, pattern, jsd, stream=None,
            head_dim=128, block_size=128):
    _check("fp_plan", _L().fp_plan(_ptr(q), _ptr(k), heads, kv_heads, seq_len, head_dim, block_size,
                                   tau, _ptr(ws), ws_bytes, _ptr(pattern), _ptr(jsd), _stream(stream)))


def fp_select(heads, kv_heads, seq_len, gamma, min_budget, ws, ws_bytes, row_ptr, col_idx,
              stats=None, stream=None, head_dim=128, block_size=128):
    _check("fp_select", _L().fp_select(heads, kv_heads, seq_len, head_dim, block_size, gamma,
                                       min_budget, _ptr(ws), ws_bytes, _ptr(row_ptr),
                                       _ptr(col_idx), _ptr(stats), _stream(stream)))


def fp_select_ex(heads, kv_heads, seq_len, gamma, min_budget, ws, ws_bytes, row_ptr, col_idx,
                 stats=None, stream=None, vs_mode=0, qa_mode=0, max_budget=0, head_dim=128,
                 block_size=128):
    opt = SelectOptions(vs_mode, qa_mode, max_budget)
    _check("fp_select_ex", _L().fp_select_ex(heads, kv_heads, seq_len, head_dim, block_size, gamma,
                                             min_budget, ctypes.byref(opt), _ptr(ws), ws_bytes,
                                             _ptr(row_ptr), _ptr(col_idx), _ptr(stats),
                                             _stream(stream)))


def fp_sparse_attn(q, k, v, o, heads, kv_heads, seq_len, row_ptr, col_idx, ws=None, ws_bytes=0,
                   stream=None, head_dim=128, block_size=128):
    _check("fp_sparse_attn", _L().fp_sparse_attn(_ptr(q), _ptr(k), _ptr(v), _ptr(o), heads, kv_heads,
                                                 seq_len, head_dim, block_size, _ptr(row_ptr),
                                                 _ptr(col_idx), _ptr(ws), ws_bytes, _stream(stream)))


def fp_dense_causal_attn(q, k, v, o, heads, kv_heads, seq_len, ws=None, ws_bytes=0, stream=None,
                         head_dim=128, block_size=128):
    _check("fp_dense_causal_attn", _L().fp_dense_causal_attn(
        _ptr(q), _ptr(k), _ptr(v), _ptr(o), heads, kv_heads, seq_len, head_dim, block_size,
        _ptr(ws), ws_bytes, _stream(stream)))


def fp_layer_host(q_host, k_host, v_host, o_host, d_q, d_k, d_v, d_o, heads, kv_heads, seq_len,
                  gamma, tau, min_budget, ws, ws_bytes, pattern, jsd, row_ptr, col_idx,
                  stream=None, head_dim=128, block_size=128):
    _check("fp_layer_host", _L().fp_layer_host(
        _ptr(q_host), _ptr(k_host), _ptr(v_host), _ptr(o_host), _ptr(d_q), _ptr(d_k), _ptr(d_v),
        _ptr(d_o), heads, kv_heads, seq_len, head_dim, block_size, gamma, tau, min_budget,
        _ptr(ws), ws_bytes, _ptr(pattern), _ptr(jsd), _ptr(row_ptr), _ptr(col_idx),
        _stream(stream)))


def fp_layout_bhsd(batch, heads, kv_heads, seq_len):
    lay = Layout()
    _check("fp_layout_bhsd", _L().fp_layout_bhsd(batch, heads, kv_heads, seq_len, ctypes.byref(lay)))
    return lay


def fp_layout_bshd(batch, heads, kv_heads, seq_len):
    lay = Layout()
    _check("fp_layout_bshd", _L().fp_layout_bshd(batch, heads, kv_heads, seq_len, ctypes.byref(lay)))
    return lay


def _lay(layout):
    return None if layout is None else ctypes.byref(layout)


def fp_plan_ex(q, k, heads, kv_heads, seq_len, layout, tau, ws, ws_bytes, pattern, jsd, stream=None,
               head_dim=128, block_size=128):
    _check("fp_plan_ex", _L().fp_plan_ex(_ptr(q), _ptr(k), heads, kv_heads, seq_len, head_dim,
                                         block_size, _lay(layout), tau, _ptr(ws), ws_bytes,
                                         _ptr(pattern), _ptr(jsd), _stream(stream)))


def fp_sparse_attn_ex(q, k, v, o, heads, kv_heads, seq_len, layout, row_ptr, col_idx, ws=None,
                      ws_bytes=0, stream=None, head_dim=128, block_size=128):
    _check("fp_sparse_attn_ex", _L().fp_sparse_attn_ex(
        _ptr(q), _ptr(k), _ptr(v), _ptr(o), heads, kv_heads, seq_len, head_dim, block_size,
        _lay(layout), _ptr(row_ptr), _ptr(col_idx), _ptr(ws), ws_bytes, _stream(stream)))


def fp_sparse_attn_peers(q, k, v, o, peer_o, n_peer, heads, kv_heads, seq_len, row_ptr, col_idx,
                         layout=None, ws=None, ws_bytes=0, stream=None, head_dim=128,
                         block_size=128):
    """fp_sparse_attn whose epilogue also stores every output row into n_peer
    further buffers; peer_o: device int64 tensor (or address) of n_peer device
    pointers (next row f4: the fused output exchange)."""
    _check("fp_sparse_attn_peers", _L().fp_sparse_attn_peers(
        _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(peer_o), n_peer, heads, kv_heads, seq_len,
        head_dim, block_size, _lay(layout), _ptr(row_ptr), _ptr(col_idx), _ptr(ws), ws_bytes,
        _stream(stream)))


def fp_dense_causal_attn_ex(q, k, v, o, heads, kv_heads, seq_len, layout, ws=None, ws_bytes=0,
                            stream=None, head_dim=128, block_size=128):
    _check("fp_dense_causal_attn_ex", _L().fp_dense_causal_attn_ex(
        _ptr(q), _ptr(k), _ptr(v), _ptr(o), heads, kv_heads, seq_len, head_dim, block_size,
        _lay(layout), _ptr(ws), ws_bytes, _stream(stream)))


def fp_debug_view(ws, heads, kv_heads, seq_len, head_dim=128, block_size=128):
    d = DebugPtrs()
    _check("fp_debug_view", _L().fp_debug_view(_ptr(ws), heads, kv_heads, seq_len, head_dim,
                                               block_size, ctypes.byref(d)))
    return d


# ------------------------------------------------------------ convenience ---
# The paper's defaults: block 128, tau 0.1, every head computes at
# least 1024 tokens (minimum budget; per query-block row in kernel units, A12).
PAPER_MIN_BUDGET = 1024


class FlexPrefill:
    """Owns the workspace and CSR buffers for one (heads, kv_heads, seq_len) shape.

    batch > 1 or layout="bshd" (token-major [batch][seq][heads][128], the
    layout of a QKV projection) use the *_ex entry points; per-head buffers
    (pattern, jsd, CSR, stats) then cover batch * heads flattened heads."""

    def __init__(self, heads, kv_heads, seq_len, device="cuda", batch=1, layout="bhsd",
                 block_size=128):
        import torch
        if layout not in ("bhsd", "bshd"):
            raise ValueError(layout)
        self.heads, self.kv_heads, self.batch = heads, kv_heads, batch
        self.layout = None
        if batch != 1 or layout != "bhsd":
            mk = fp_layout_bhsd if layout == "bhsd" else fp_layout_bshd
            self.layout = mk(batch, heads, kv_heads, seq_len)
        heads, kv_heads = batch * heads, batch * kv_heads  # flattened
        self.H, self.G, self.n = heads, kv_heads, seq_len
        self.b = block_size
        self.nb = -(-seq_len // block_size)
        self.ws_bytes = fp_workspace_bytes(heads, kv_heads, seq_len, block_size=block_size)
        if self.ws_bytes == 0:
            raise FlexPrefillError("fp_workspace_bytes", 2)
        self.cap = fp_col_idx_capacity(seq_len, block_size)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        self.pattern = torch.empty(heads, dtype=torch.int32, device=device)
        self.jsd = torch.empty(heads, dtype=torch.float32, device=device)
        self.row_ptr = torch.empty(heads, self.nb + 1, dtype=torch.int32, device=device)
        self.col_idx = torch.empty(heads, self.cap, dtype=torch.int32, device=device)
        self.stats_buf = torch.empty(heads * ctypes.sizeof(SelectStats), dtype=torch.uint8,
                                     device=device)

    def plan(self, q, k, tau=0.1, stream=None):
        if self.layout is not None:
            fp_plan_ex(q, k, self.heads, self.kv_heads, self.n, self.layout, tau, self.ws,
                       self.ws_bytes, self.pattern, self.jsd, stream, block_size=self.b)
            return
        fp_plan(q, k, self.H, self.G, self.n, tau, self.ws, self.ws_bytes, self.pattern, self.jsd,
                stream, block_size=self.b)

    def select(self, gamma=0.95, min_budget=PAPER_MIN_BUDGET, stream=None, with_stats=True, vs_mode=0, qa_mode=0,
               max_budget=0):
        fp_select_ex(self.H, self.G, self.n, gamma, min_budget, self.ws, self.ws_bytes,
                     self.row_ptr, self.col_idx, self.stats_buf if with_stats else None, stream,
                     vs_mode, qa_mode, max_budget, block_size=self.b)

    def attn(self, q, k, v, out, stream=None):
        if self.layout is not None:
            fp_sparse_attn_ex(q, k, v, out, self.heads, self.kv_heads, self.n, self.layout,
                              self.row_ptr, self.col_idx, self.ws, self.ws_bytes, stream,
                              block_size=self.b)
            return
        fp_sparse_attn(q, k, v, out, self.H, self.G, self.n, self.row_ptr, self.col_idx, self.ws,
                       self.ws_bytes, stream, block_size=self.b)

    def dense(self, q, k, v, out, stream=None):
        if self.layout is not None:
            fp_dense_causal_attn_ex(q, k, v, out, self.heads, self.kv_heads, self.n, self.layout,
                                    self.ws, self.ws_bytes, stream, block_size=self.b)
            return
        fp_dense_causal_attn(q, k, v, out, self.H, self.G, self.n, self.ws, self.ws_bytes, stream,
                             block_size=self.b)

    def layer(self, q, k, v, out, gamma=0.95, tau=0.1, min_budget=PAPER_MIN_BUDGET, stream=None):
        self.plan(q, k, tau, stream)
        self.select(gamma, min_budget, stream, with_stats=False)
        self.attn(q, k, v, out, stream)

    def capture_layer(self, q, k, v, out, gamma=0.95, tau=0.1, min_budget=PAPER_MIN_BUDGET):
        """Record plan -> select -> attn into one CUDA graph (the C ABI only
        enqueues on the current stream, so the whole layer is capturable).
        Returns the torch.cuda.CUDAGraph; replay() reruns the layer on the
        same buffers."""
        import torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up outside capture (kernel attributes)
            self.layer(q, k, v, out, gamma, tau, min_budget)
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.layer(q, k, v, out, gamma, tau, min_budget)
        return graph

    def stats(self):
        raw = bytes(self.stats_buf.cpu().numpy().tobytes())
        arr = (SelectStats * self.H).from_buffer_copy(raw)
        return [{f: getattr(s, f) for f, _ in SelectStats._fields_} for s in arr]

    def debug(self):
        """Copies of the workspace intermediates (torch CPU tensors)."""
        import torch
        d = fp_debug_view(self.ws, self.H, self.G, self.n, block_size=self.b)
        base = self.ws.data_ptr()
        H, G, n, nb, tri = self.H, self.G, self.n, self.nb, self.cap

        def view(ptr, count, dtype, shape):
            off = ptr - base
            esz = torch.empty((), dtype=dtype).element_size()
            return self.ws[off: off + count * esz].view(dtype).reshape(shape).cpu()

        f32, i32 = torch.float32, torch.int32
        return dict(
            a_v=view(d.a_v, H * n, f32, (H, n)), a_s=view(d.a_s, H * n, f32, (H, n)),
            a_hat=view(d.a_hat, H * nb, f32, (H, nb)), a_bar=view(d.a_bar, H * nb, f32, (H, nb)),
            k_bar=view(d.k_bar, G * nb * 128, f32, (G, nb, 128)),
            q_bar=view(d.q_bar, H * nb * 128, f32, (H, nb, 128)),
            A_bar=view(d.A_bar, H * tri, f32, (H, tri)), As=view(d.As, H * nb, f32, (H, nb)),
            sel_v=view(d.sel_v, H * n, i32, (H, n)), sel_s=view(d.sel_s, H * n, i32, (H, n)),
            sel_qa=view(d.sel_qa, H * tri, i32, (H, tri)),
            sel_count=view(d.sel_count, H * 4, i32, (H, 4)),
            row_nnz_pre=view(d.row_nnz_pre, H * nb, i32, (H, nb)),
            attn_sched=view(d.attn_sched, 2, i32, (2,)),
        )
