// fp_api.cu -- the C ABI (include/flexprefill.h): validation, workspace
// layout, TMA descriptors, and the enqueue of the three stages.
#include <cudaTypedefs.h>
#include <math.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "fp_internal.h"

namespace fp {

static thread_local int g_last_cuda_error = 0;

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_tile_map(CUtensorMap* map, const void* base, const TLayout& t, int n, int batch,
                   int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)n, (cuuint64_t)t.per, (cuuint64_t)batch};
  // batch stride is unused when batch == 1 but must still be a valid value
  const long long bs = batch > 1 ? t.bs : t.hs * t.per;
  cuuint64_t strides[3] = {(cuuint64_t)t.rs * 2, (cuuint64_t)t.hs * 2, (cuuint64_t)bs * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t ensure_smem_attr(const void* fn, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  struct Done {
    const void* fn;
    int dev;
    size_t bytes;
  };
  static std::mutex mu;
  static std::vector<Done> done;
  std::lock_guard<std::mutex> lock(mu);
  for (const Done& d : done)
    if (d.fn == fn && d.dev == dev && d.bytes >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.push_back(Done{fn, dev, bytes});
  return e;
}

static fp_status check_shape(int heads, int kv_heads, int seq_len, int head_dim, int block_size) {
  if (heads <= 0 || kv_heads <= 0 || seq_len <= 0) return FP_ERR_SHAPE;
  if (heads % kv_heads != 0) return FP_ERR_SHAPE;
  if (head_dim != 128 || (block_size != 128 && block_size != 64)) return FP_ERR_SHAPE;
  // ragged n allowed (A26); n >= b (A13) and n >= 128 (the representative
  // passes read one 128-row tile; with b = 64 its last 64 rows are Q^)
  if (seq_len < 128) return FP_ERR_SHAPE;
  // bitmap / index capacity limit: nb <= 8192 blocks
  if (seq_len > (block_size == 64 ? (1 << 19) : (1 << 20))) return FP_ERR_SHAPE;
  return FP_OK;
}

// fp_layout -> internal Layout (validated); NULL = [heads][n][128] contiguous, batch 1
static fp_status to_layout(const fp_layout* in, int heads, int kv_heads, int seq_len, Layout* out) {
  if (!in) {
    *out = head_major_layout(1, heads, kv_heads, seq_len);
    return FP_OK;
  }
  if (in->batch < 1 || (long long)in->batch * heads > (1 << 24)) return FP_ERR_SHAPE;
  const int64_t* st[4] = {in->q_stride, in->k_stride, in->v_stride, in->o_stride};
  TLayout* t[4] = {&out->q, &out->k, &out->v, &out->o};
  for (int i = 0; i < 4; ++i) {
    for (int j = 0; j < 3; ++j) {
      if (j == 0 && in->batch == 1) continue;  // unused
      if (st[i][j] < 128 || st[i][j] >= (1ll << 38)) return FP_ERR_SHAPE;
      if (st[i][j] % 8) return FP_ERR_ALIGN;  // TMA: 16-byte global strides
    }
    const int per = (i == 1 || i == 2) ? kv_heads : heads;
    const long long bs = in->batch == 1 ? st[i][1] * per : st[i][0];
    *t[i] = TLayout{bs, st[i][1], st[i][2], per};
  }
  out->batch = in->batch;
  return FP_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

static fp_status check_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FP_ERR_DEVICE;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return FP_ERR_DEVICE;
  return FP_OK;
}

static fp_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FP_OK;
  g_last_cuda_error = (int)e;
  return FP_ERR_CUDA;
}

}  // namespace fp

using namespace fp;

extern "C" {

size_t fp_workspace_bytes(int heads, int kv_heads, int seq_len, int head_dim, int block_size) {
  if (check_shape(heads, kv_heads, seq_len, head_dim, block_size) != FP_OK) return 0;
  return ws_layout(make_shape(heads, kv_heads, seq_len, block_size)).total;
}

fp_status fp_layout_bhsd(int batch, int heads, int kv_heads, int seq_len, fp_layout* out) {
  if (!out) return FP_ERR_NULL;
  if (batch < 1 || heads <= 0 || kv_heads <= 0 || seq_len <= 0) return FP_ERR_SHAPE;
  const int64_t n = seq_len;
  const int64_t q[3] = {heads * n * 128, n * 128, 128}, k[3] = {kv_heads * n * 128, n * 128, 128};
  out->batch = batch;
  memcpy(out->q_stride, q, sizeof q);
  memcpy(out->o_stride, q, sizeof q);
  memcpy(out->k_stride, k, sizeof k);
  memcpy(out->v_stride, k, sizeof k);
  return FP_OK;
}

fp_status fp_layout_bshd(int batch, int heads, int kv_heads, int seq_len, fp_layout* out) {
  if (!out) return FP_ERR_NULL;
  if (batch < 1 || heads <= 0 || kv_heads <= 0 || seq_len <= 0) return FP_ERR_SHAPE;
  const int64_t n = seq_len;
  const int64_t q[3] = {n * heads * 128, 128, (int64_t)heads * 128};
  const int64_t k[3] = {n * kv_heads * 128, 128, (int64_t)kv_heads * 128};
  out->batch = batch;
  memcpy(out->q_stride, q, sizeof q);
  memcpy(out->o_stride, q, sizeof q);
  memcpy(out->k_stride, k, sizeof k);
  memcpy(out->v_stride, k, sizeof k);
  return FP_OK;
}

size_t fp_col_idx_capacity(int seq_len, int block_size) {
  if (block_size <= 0 || seq_len <= 0) return 0;
  const size_t nb = ((size_t)seq_len + block_size - 1) / block_size;
  return nb * (nb + 1) / 2;
}

// at most: fp_plan 8 (rep1, rep_stats -- folded into rep2 when n <= 32k --,
// rep2, line_sums, pattern, qbar, pooled_logits, pooled_softmax), fp_select 5
// (topmass, build_lines, assemble_rows, row_scan, write_cols), fp_sparse_attn 1
int fp_kernels_per_layer(void) { return 8 + 5 + 1; }

fp_status fp_plan(const void* q, const void* k, int heads, int kv_heads, int seq_len, int head_dim,
                  int block_size, float tau, void* ws, size_t ws_bytes, int32_t* pattern,
                  float* jsd, void* stream) {
  return fp_plan_ex(q, k, heads, kv_heads, seq_len, head_dim, block_size, nullptr, tau, ws, ws_bytes,
                    pattern, jsd, stream);
}

fp_status fp_plan_ex(const void* q, const void* k, int heads, int kv_heads, int seq_len,
                     int head_dim, int block_size, const fp_layout* layout, float tau, void* ws,
                     size_t ws_bytes, int32_t* pattern, float* jsd, void* stream) {
  if (!q || !k || !ws) return FP_ERR_NULL;
  fp_status st = check_shape(heads, kv_heads, seq_len, head_dim, block_size);
  if (st) return st;
  if (!(tau >= 0.f && tau <= 1.f)) return FP_ERR_RANGE;
  Layout lay;
  if ((st = to_layout(layout, heads, kv_heads, seq_len, &lay))) return st;
  if (!aligned16(q) || !aligned16(k) || !aligned16(ws)) return FP_ERR_ALIGN;
  const Shape s = make_shape(lay.batch * heads, lay.batch * kv_heads, seq_len, block_size);
  const WsLayout L = ws_layout(s);
  if (ws_bytes < L.total) return FP_ERR_WORKSPACE;
  if ((st = check_device())) return st;
  CUtensorMap qm, km;
  if (!make_tile_map(&qm, q, lay.q, seq_len, lay.batch) ||
      !make_tile_map(&km, k, lay.k, seq_len, lay.batch))
    return cuda_status(cudaErrorInvalidValue);
  return cuda_status(launch_plan(s, L, ws, q, k, lay, qm, km, tau, pattern, jsd,
                                 static_cast<cudaStream_t>(stream)));
}

fp_status fp_select(int heads, int kv_heads, int seq_len, int head_dim, int block_size, float gamma,
                    int min_budget, void* ws, size_t ws_bytes, int32_t* row_ptr, int32_t* col_idx,
                    fp_select_stats* stats, void* stream) {
  return fp_select_ex(heads, kv_heads, seq_len, head_dim, block_size, gamma, min_budget, nullptr, ws,
                      ws_bytes, row_ptr, col_idx, stats, stream);
}

fp_status fp_select_ex(int heads, int kv_heads, int seq_len, int head_dim, int block_size,
                       float gamma, int min_budget, const fp_select_options* opt_in, void* ws,
                       size_t ws_bytes, int32_t* row_ptr, int32_t* col_idx, fp_select_stats* stats,
                       void* stream) {
  if (!ws || !row_ptr || !col_idx) return FP_ERR_NULL;
  fp_status st = check_shape(heads, kv_heads, seq_len, head_dim, block_size);
  if (st) return st;
  if (!(gamma > 0.f) || isnan(gamma) || min_budget < 0) return FP_ERR_RANGE;
  fp_select_options opt = {0, 0, 0};
  if (opt_in) opt = *opt_in;
  if (opt.vs_mode < 0 || opt.vs_mode > 1 || opt.qa_mode < 0 || opt.qa_mode > 1 || opt.max_budget < 0)
    return FP_ERR_RANGE;
  // the maximum budget is applied after the minimum one (A23): a cap below the
  // floor would silently break the per-row minimum, so it is an error
  if (opt.max_budget > 0 && opt.max_budget < min_budget) return FP_ERR_RANGE;
  if (!aligned16(ws)) return FP_ERR_ALIGN;
  const Shape s = make_shape(heads, kv_heads, seq_len, block_size);
  const WsLayout L = ws_layout(s);
  if (ws_bytes < L.total) return FP_ERR_WORKSPACE;
  if ((st = check_device())) return st;
  return cuda_status(launch_select(s, L, ws, gamma, min_budget, opt, row_ptr, col_idx, stats,
                                   static_cast<cudaStream_t>(stream)));
}

static fp_status attn_common(const void* q, const void* k, const void* v, void* o, int heads,
                             int kv_heads, int seq_len, int head_dim, int block_size,
                             const fp_layout* layout, const int32_t* row_ptr,
                             const int32_t* col_idx, void* ws, size_t ws_bytes, void* stream,
                             bool dense, const void* const* peer_o = nullptr, int n_peer = 0) {
  if (!q || !k || !v || !o) return FP_ERR_NULL;
  if (n_peer < 0 || n_peer > FP_MAX_PEERS) return FP_ERR_RANGE;
  if (n_peer > 0 && !peer_o) return FP_ERR_NULL;
  if (n_peer > 0 && (reinterpret_cast<uintptr_t>(peer_o) & 7u)) return FP_ERR_ALIGN;
  if (!dense && (!row_ptr || !col_idx)) return FP_ERR_NULL;
  fp_status st = check_shape(heads, kv_heads, seq_len, head_dim, block_size);
  if (st) return st;
  Layout lay;
  if ((st = to_layout(layout, heads, kv_heads, seq_len, &lay))) return st;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o)) return FP_ERR_ALIGN;
  const Shape s = make_shape(lay.batch * heads, lay.batch * kv_heads, seq_len, block_size);
  const WsLayout L = ws_layout(s);
  // ws is optional (scheduler scratch): NULL = no scratch; otherwise it must be
  // a full workspace of this shape
  if (ws && !aligned16(ws)) return FP_ERR_ALIGN;
  if (ws && ws_bytes < L.total) return FP_ERR_WORKSPACE;
  if ((st = check_device())) return st;
  CUtensorMap qm, km, vm;
  if (!make_tile_map(&qm, q, lay.q, seq_len, lay.batch) ||
      !make_tile_map(&km, k, lay.k, seq_len, lay.batch, attn_kv_box_rows()) ||
      !make_tile_map(&vm, v, lay.v, seq_len, lay.batch, attn_kv_box_rows()))
    return cuda_status(cudaErrorInvalidValue);
  return cuda_status(launch_attn(s, L, ws, lay, qm, km, vm, o, row_ptr, col_idx, dense, peer_o,
                                 n_peer, static_cast<cudaStream_t>(stream)));
}

fp_status fp_sparse_attn(const void* q, const void* k, const void* v, void* o, int heads,
                         int kv_heads, int seq_len, int head_dim, int block_size,
                         const int32_t* row_ptr, const int32_t* col_idx, void* ws, size_t ws_bytes,
                         void* stream) {
  return attn_common(q, k, v, o, heads, kv_heads, seq_len, head_dim, block_size, nullptr, row_ptr,
                     col_idx, ws, ws_bytes, stream, false);
}

fp_status fp_sparse_attn_ex(const void* q, const void* k, const void* v, void* o, int heads,
                            int kv_heads, int seq_len, int head_dim, int block_size,
                            const fp_layout* layout, const int32_t* row_ptr,
                            const int32_t* col_idx, void* ws, size_t ws_bytes, void* stream) {
  return attn_common(q, k, v, o, heads, kv_heads, seq_len, head_dim, block_size, layout, row_ptr,
                     col_idx, ws, ws_bytes, stream, false);
}

fp_status fp_sparse_attn_peers(const void* q, const void* k, const void* v, void* o,
                               const void* const* peer_o, int n_peer, int heads, int kv_heads,
                               int seq_len, int head_dim, int block_size, const fp_layout* layout,
                               const int32_t* row_ptr, const int32_t* col_idx, void* ws,
                               size_t ws_bytes, void* stream) {
  return attn_common(q, k, v, o, heads, kv_heads, seq_len, head_dim, block_size, layout, row_ptr,
                     col_idx, ws, ws_bytes, stream, false, peer_o, n_peer);
}

fp_status fp_dense_causal_attn(const void* q, const void* k, const void* v, void* o, int heads,
                               int kv_heads, int seq_len, int head_dim, int block_size, void* ws,
                               size_t ws_bytes, void* stream) {
  return attn_common(q, k, v, o, heads, kv_heads, seq_len, head_dim, block_size, nullptr, nullptr,
                     nullptr, ws, ws_bytes, stream, true);
}

fp_status fp_dense_causal_attn_ex(const void* q, const void* k, const void* v, void* o, int heads,
                                  int kv_heads, int seq_len, int head_dim, int block_size,
                                  const fp_layout* layout, void* ws, size_t ws_bytes,
                                  void* stream) {
  return attn_common(q, k, v, o, heads, kv_heads, seq_len, head_dim, block_size, layout, nullptr,
                     nullptr, ws, ws_bytes, stream, true);
}

namespace fp {
// Streams and events of fp_layer_host, created on first use per (calling
// thread, device) and reused by every later call of that thread: no per-call
// create / destroy, and calls from different threads never share them.
// Events are re-recorded freely: cudaStreamWaitEvent captures the event's most
// recent record at the time of the wait call.
struct HostPipe {
  cudaStream_t sin = nullptr, scomp = nullptr, sout = nullptr;
  cudaEvent_t ev[6] = {};  // start, done, kq, v, head, comp
  bool ok = false;
  ~HostPipe() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
    if (sin) cudaStreamDestroy(sin);
    if (scomp) cudaStreamDestroy(scomp);
    if (sout) cudaStreamDestroy(sout);
  }
};
static HostPipe* host_pipe() {
  thread_local HostPipe pipes[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  HostPipe& p = pipes[dev];
  if (!p.ok) {
    bool good = cudaStreamCreateWithFlags(&p.sin, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&p.scomp, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&p.sout, cudaStreamNonBlocking) == cudaSuccess;
    for (cudaEvent_t& e : p.ev) good = good && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    if (!good) return nullptr;  // partially created handles are reused on the next try
    p.ok = true;
  }
  return &p;
}
static bool aligned4(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }
}  // namespace fp

fp_status fp_layer_host(const void* q_host, const void* k_host, const void* v_host, void* o_host,
                        void* d_q, void* d_k, void* d_v, void* d_o, int heads, int kv_heads,
                        int seq_len, int head_dim, int block_size, float gamma, float tau,
                        int min_budget, void* ws, size_t ws_bytes, int32_t* pattern, float* jsd,
                        int32_t* row_ptr, int32_t* col_idx, void* stream) {
  // ---- every check of the nested calls, up front: an invalid call enqueues nothing
  if (!q_host || !k_host || !v_host || !o_host || !d_q || !d_k || !d_v || !d_o || !ws || !pattern ||
      !jsd || !row_ptr || !col_idx)
    return FP_ERR_NULL;
  fp_status st = check_shape(heads, kv_heads, seq_len, head_dim, block_size);
  if (st) return st;
  if (!(gamma > 0.f) || isnan(gamma) || !(tau >= 0.f && tau <= 1.f) || min_budget < 0)
    return FP_ERR_RANGE;
  if (!aligned16(d_q) || !aligned16(d_k) || !aligned16(d_v) || !aligned16(d_o) || !aligned16(ws) ||
      !aligned4(pattern) || !aligned4(jsd) || !aligned4(row_ptr) || !aligned4(col_idx))
    return FP_ERR_ALIGN;
  if (ws_bytes < fp_workspace_bytes(heads, kv_heads, seq_len, head_dim, block_size))
    return FP_ERR_WORKSPACE;
  if ((st = check_device())) return st;
  HostPipe* hp = host_pipe();
  if (!hp) return cuda_status(cudaErrorUnknown);
  // Pipelined per chunk of Q heads (a KV group, g = heads / kv_heads Q heads +
  // their K/V; the first group split into single heads): host->device copies of
  // chunk c+1 and the device->host copies of chunk c-1 overlap the compute of
  // chunk c (three streams joined back to `stream`). Chunks alternate between
  // two workspace slots (the full-layer workspace holds at least two). Results
  // are bitwise those of the single whole-layer call: heads are independent and
  // no kernel's arithmetic depends on how many heads a call batches.
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaStream_t sin = hp->sin, scomp = hp->scomp, sout = hp->sout;
  cudaEvent_t e_start = hp->ev[0], e_done = hp->ev[1], e_kq = hp->ev[2], e_v = hp->ev[3],
              e_h = hp->ev[4], e_c = hp->ev[5];
  const int g = heads / kv_heads;
  const size_t n = (size_t)seq_len, nb = (n + block_size - 1) / block_size, cap = nb * (nb + 1) / 2;
  const size_t qb_bytes = (size_t)g * n * 128 * 2, kv_bytes = n * 128 * 2;
  const size_t slot = align256(fp_workspace_bytes(g, 1, seq_len, head_dim, block_size));
  const int nslots = (kv_heads > 1 && ws_bytes >= 2 * slot) ? 2 : 1;
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t r) {
    if (e == cudaSuccess && r != cudaSuccess) e = r;
    return e == cudaSuccess;
  };
  chk(cudaEventRecord(e_start, cs));
  chk(cudaStreamWaitEvent(sin, e_start, 0));
  chk(cudaStreamWaitEvent(scomp, e_start, 0));
  chk(cudaStreamWaitEvent(sout, e_start, 0));
  // Chunks of Q heads: the first KV group one head at a time (only its K + one
  // head of Q is uploaded before compute starts), every later group whole.
  struct Chunk {
    int grp, h0, nh;
  };
  const size_t hb = qb_bytes / g;  // one head of Q / O
  int nchunk = 0;
  for (int c = 0; c < kv_heads; ++c) nchunk += (c == 0) ? g : 1;
  for (int ci_ = 0; ci_ < nchunk && e == cudaSuccess && st == FP_OK; ++ci_) {
    const Chunk ch = ci_ < g ? Chunk{0, ci_, 1} : Chunk{ci_ - g + 1, 0, g};
    const int c = ch.grp;
    const bool first_of_group = (ch.h0 == 0);
    const char* qh = static_cast<const char*>(q_host) + c * qb_bytes + ch.h0 * hb;
    const char* kh = static_cast<const char*>(k_host) + c * kv_bytes;
    const char* vh = static_cast<const char*>(v_host) + c * kv_bytes;
    char* qd = static_cast<char*>(d_q) + c * qb_bytes + ch.h0 * hb;
    char* kd = static_cast<char*>(d_k) + c * kv_bytes;
    char* vd = static_cast<char*>(d_v) + c * kv_bytes;
    char* od = static_cast<char*>(d_o) + c * qb_bytes + ch.h0 * hb;
    // K and Q first (all fp_plan / fp_select read), V last (only the attention
    // reads it); K / V once per group (with the group's first chunk). The
    // attention runs one launch per head (bitwise the same result: work items
    // are per (head, query block)) and each head's output is copied back as
    // soon as it is done, so only the last head's D2H is exposed at the end.
    if (first_of_group) chk(cudaMemcpyAsync(kd, kh, kv_bytes, cudaMemcpyHostToDevice, sin));
    chk(cudaMemcpyAsync(qd, qh, ch.nh * hb, cudaMemcpyHostToDevice, sin));
    chk(cudaEventRecord(e_kq, sin));
    if (first_of_group) chk(cudaMemcpyAsync(vd, vh, kv_bytes, cudaMemcpyHostToDevice, sin));
    chk(cudaStreamWaitEvent(scomp, e_kq, 0));
    chk(cudaEventRecord(e_v, sin));
    void* wsc = static_cast<char*>(ws) + (ci_ % nslots) * slot;
    const int hg = c * g + ch.h0;  // first global head of the chunk
    int32_t* rp = row_ptr + (size_t)hg * (nb + 1);
    int32_t* ci = col_idx + (size_t)hg * cap;
    if (e == cudaSuccess &&
        !(st = fp_plan(qd, kd, ch.nh, 1, seq_len, head_dim, block_size, tau, wsc, slot, pattern + hg,
                       jsd + hg, scomp)))
      st = fp_select(ch.nh, 1, seq_len, head_dim, block_size, gamma, min_budget, wsc, slot, rp, ci,
                     nullptr, scomp);
    chk(cudaStreamWaitEvent(scomp, e_v, 0));
    // one attention launch per head (the chunk's workspace slot holds the
    // persistent scheduler's work counter), each head's output copied back as
    // soon as it is done: measured faster than one launch + one copy per chunk
    // (39.7 vs 40.6 ms at C3), the exposed tail is one head's download
    for (int i = 0; i < ch.nh && e == cudaSuccess && st == FP_OK; ++i) {
      st = fp_sparse_attn(qd + i * hb, kd, vd, od + i * hb, 1, 1, seq_len, head_dim, block_size,
                          rp + (size_t)i * (nb + 1), ci + (size_t)i * cap, wsc, slot, scomp);
      chk(cudaEventRecord(e_h, scomp));
      chk(cudaStreamWaitEvent(sout, e_h, 0));
      chk(cudaMemcpyAsync(static_cast<char*>(o_host) + c * qb_bytes + (ch.h0 + i) * hb, od + i * hb,
                          hb, cudaMemcpyDeviceToHost, sout));
    }
  }
  // join everything back into the caller's stream (also after an error, so the
  // internal streams never run ahead of the caller's later work)
  cudaEventRecord(e_c, scomp);
  cudaStreamWaitEvent(sout, e_c, 0);
  cudaEventRecord(e_done, sout);
  chk(cudaStreamWaitEvent(cs, e_done, 0));
  if (st) return st;
  return cuda_status(e);
}

fp_status fp_debug_view(const void* ws, int heads, int kv_heads, int seq_len, int head_dim,
                        int block_size, fp_debug_ptrs* out) {
  if (!ws || !out) return FP_ERR_NULL;
  fp_status st = check_shape(heads, kv_heads, seq_len, head_dim, block_size);
  if (st) return st;
  const WsLayout L = ws_layout(make_shape(heads, kv_heads, seq_len, block_size));
  void* w = const_cast<void*>(ws);
  out->a_v = wsp<float>(w, L.a_v);
  out->a_s = wsp<float>(w, L.a_s);
  out->a_hat = wsp<float>(w, L.a_hat);
  out->a_bar = wsp<float>(w, L.a_bar);
  out->k_bar = wsp<float>(w, L.k_bar);
  out->q_bar = wsp<float>(w, L.q_bar);
  out->A_bar = wsp<float>(w, L.A_bar);
  out->As = wsp<float>(w, L.As);
  out->sel_v = wsp<int32_t>(w, L.sel_v);
  out->sel_s = wsp<int32_t>(w, L.sel_s);
  out->sel_qa = wsp<int32_t>(w, L.sel_qa);
  out->sel_count = wsp<int32_t>(w, L.sel_count);
  out->row_nnz_pre = wsp<int32_t>(w, L.row_nnz_pre);
  out->attn_sched = wsp<int32_t>(w, L.sched);
  return FP_OK;
}

const char* fp_status_string(fp_status s) {
  switch (s) {
    case FP_OK: return "ok";
    case FP_ERR_NULL: return "null pointer";
    case FP_ERR_SHAPE: return "invalid shape";
    case FP_ERR_RANGE: return "parameter out of range";
    case FP_ERR_ALIGN: return "pointer not 16-byte aligned";
    case FP_ERR_WORKSPACE: return "workspace too small";
    case FP_ERR_DEVICE: return "device is not sm_100 (B200)";
    case FP_ERR_CUDA: return "CUDA launch error";
  }
  return "unknown status";
}

int fp_last_cuda_error(void) { return g_last_cuda_error; }

}  // extern "C"
