// fp_internal.h -- workspace layout and kernel launchers (host side).
#pragma once
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/flexprefill.h"

namespace fp {

#ifndef FP_CHUNK_TILES_MAX
#define FP_CHUNK_TILES_MAX 8
#endif
constexpr int kChunkTilesMax = FP_CHUNK_TILES_MAX;  // key tiles (128 keys) per representative-pass CTA (max)
#ifndef FP_MIN_CHUNKS
#define FP_MIN_CHUNKS 16
#endif
constexpr int kMinChunks = FP_MIN_CHUNKS;  // representative-pass chunks per head (min, see make_shape)

struct Shape {
  int H, G, n, nb, nchunks, g;  // flattened heads (batch * heads per sequence); g = H / G
  int b, lb;                    // block_size (64 or 128) and log2(b)
  int nt;                       // 128-key tiles of the representative passes: ceil(n / 128)
  int ct;                       // key tiles per representative-pass CTA
  long long tri;                // nb (nb + 1) / 2
};

inline Shape make_shape(int heads, int kv_heads, int seq_len, int block = 128) {
  Shape s;
  s.H = heads;
  s.G = kv_heads;
  s.n = seq_len;
  s.b = block;
  s.lb = block == 64 ? 6 : 7;
  s.nb = (seq_len + block - 1) / block;  // ragged n: the last block is partial (A26)
  s.nt = (seq_len + 127) / 128;
  // key tiles per representative-pass CTA: the largest power of two <= 8 that
  // leaves >= 8 chunks per head (short sequences: a few CTAs with several
  // tiles each instead of many one-tile CTAs whose setup dominates; measured
  // at 4k). A function of n ONLY: pass 1 sums each row's
  // exponentials within a chunk and rep_stats combines the chunks, so the fp32
  // summation order of the row statistics (and of everything derived from them:
  // a_v, a_s, a_hat, D_JS, the top-mass picks) must not depend on how many
  // heads one call batches (fp_layer_host per-group calls, multi-GPU head
  // slices and the whole-layer call give bitwise identical results).
  s.ct = kChunkTilesMax;
  while (s.ct > 1 && (s.nt + s.ct - 1) / s.ct < kMinChunks) s.ct >>= 1;
  s.nchunks = (s.nt + s.ct - 1) / s.ct;
  s.g = heads / kv_heads;
  s.tri = (long long)s.nb * (s.nb + 1) / 2;
  return s;
}

// Byte offsets of every workspace region (each 256-B aligned).
struct WsLayout {
  size_t m_part, l_part;     // fp32 [H][nchunks][128]  pass-1 partial row max / sum (log2 domain)
  size_t m_row, mp_row;      // fp32 [H][128]           combined row max, M' = max + log2(sum)
  size_t a_v, a_s;           // fp32 [H][n]
  size_t as_part;            // fp32 [H][nt][256]       per-key-tile slash partials
  size_t a_hat, a_bar, As;   // fp32 [H][nb]
  size_t k_bar;              // fp32 [G][nb][128]
  size_t q_bar;              // fp32 [H][nb][128]
  size_t A_bar;              // fp32 [H][tri]
  size_t pattern;            // int32 [H]
  size_t jsd;                // fp32 [H]
  size_t sel_v, sel_s;       // int32 [H][n]
  size_t sel_qa;             // int32 [H][tri]
  size_t sel_count;          // int32 [H][4]
  size_t sel_mass;           // uint64 [H][4] fixed-point mass (2^-60 units)
  size_t vbits, dbits;       // uint32 [H][nbw]   vertical-block / slash-diagonal bitmaps
  size_t rowbits;            // uint32 [H][nb][nbw] final row bitmaps
  size_t row_nnz, row_nnz_pre;  // int32 [H][nb]
  size_t budget_added;       // int32 [H][nb]
  size_t budget_removed;     // int32 [H][nb]
  size_t selbits;            // uint32 [H][nb][nbw] per-row QA selection (qa_mode 1)
  size_t sched;              // int32 [64] attention scheduler: [0] work counter, [1] redone items
  size_t total;
  int nbw;                   // words per bitmap row
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

inline WsLayout ws_layout(const Shape& s) {
  WsLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  const size_t H = s.H, G = s.G, n = s.n, nb = s.nb, tri = s.tri;
  L.nbw = (s.nb + 31) / 32;
  L.m_part = take(H * s.nchunks * 128 * 4);
  L.l_part = take(H * s.nchunks * 128 * 4);
  L.m_row = take(H * 128 * 4);
  L.mp_row = take(H * 128 * 4);
  L.a_v = take(H * n * 4);
  L.a_s = take(H * n * 4);
  L.as_part = take(H * (size_t)s.nt * 256 * 4);
  L.a_hat = take(H * nb * 4);
  L.a_bar = take(H * nb * 4);
  L.As = take(H * nb * 4);
  L.k_bar = take(G * nb * 128 * 4);
  L.q_bar = take(H * nb * 128 * 4);
  L.A_bar = take(H * tri * 4);
  L.pattern = take(H * 4);
  L.jsd = take(H * 4);
  L.sel_v = take(H * n * 4);
  L.sel_s = take(H * n * 4);
  L.sel_qa = take(H * tri * 4);
  L.sel_count = take(H * 4 * 4);
  L.sel_mass = take(H * 4 * 8);
  L.vbits = take(H * L.nbw * 4);
  L.dbits = take(H * L.nbw * 4);
  L.rowbits = take(H * nb * L.nbw * 4);
  L.row_nnz = take(H * nb * 4);
  L.row_nnz_pre = take(H * nb * 4);
  L.budget_added = take(H * nb * 4);
  L.budget_removed = take(H * nb * 4);
  L.selbits = take(H * nb * L.nbw * 4);
  L.sched = take(64 * 4);
  L.total = off;
  return L;
}

// Element (flattened head hh, position i, dim c) of a Q/K/V/O tensor lives at
// base + (hh / per) * bs + (hh % per) * hs + i * rs + c  (all in elements).
struct TLayout {
  long long bs, hs, rs;
  int per;  // heads per batch element
};
struct Layout {
  TLayout q, k, v, o;
  int batch;
};
#ifdef __CUDACC__
__host__ __device__
#endif
inline size_t toff(const TLayout& t, int hh, int i) {
  return (size_t)(hh / t.per) * (size_t)t.bs + (size_t)(hh % t.per) * (size_t)t.hs +
         (size_t)i * (size_t)t.rs;
}
// [batch][heads][n][128] contiguous (the default of the plain entry points)
inline Layout head_major_layout(int batch, int heads, int kv_heads, int n) {
  Layout L;
  L.batch = batch;
  L.q = TLayout{(long long)heads * n * 128, (long long)n * 128, 128, heads};
  L.k = TLayout{(long long)kv_heads * n * 128, (long long)n * 128, 128, kv_heads};
  L.v = L.k;
  L.o = L.q;
  return L;
}

template <typename T>
inline T* wsp(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// 4D bf16 tensor map {128 cols, n rows, per heads, batch} with the strides of
// `t`; box 64 cols x 128 rows, SWIZZLE_128B; rows >= n are zero-filled.
bool make_tile_map(CUtensorMap* map, const void* base, const TLayout& t, int n, int batch,
                   int box_rows = 128);
// rows per K/V TMA box of the attention kernel in use (v7: 64-key sub-tiles; v5: 128)
int attn_kv_box_rows();

// Raises `fn`'s dynamic shared-memory limit to `bytes` on the CURRENT device.
// Function attributes are per device context: this runs cudaFuncSetAttribute
// once per (kernel, device) under a mutex (thread-safe; several GPUs driven
// from one process each get their own setting) and returns its error.
cudaError_t ensure_smem_attr(const void* fn, size_t bytes);

// Kernel launch with programmatic stream serialization (PDL, see
// FP_PDL_ENTRY): build with -DFP_NO_PDL for plain stream-ordered launches.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
#ifdef FP_NO_PDL
  at[0].val.programmaticStreamSerializationAllowed = 0;
#else
  at[0].val.programmaticStreamSerializationAllowed = 1;
#endif
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
#define FP_LAUNCH(kern, grid, block, smem, st, ...) \
  ::fp::launch_pdl(kern, dim3(grid), dim3(block), (size_t)(smem), st, __VA_ARGS__)

// ---- launchers (return cudaGetLastError of their launches) ----
cudaError_t launch_plan(const Shape& s, const WsLayout& L, void* ws, const void* q, const void* k,
                        const Layout& lay, const CUtensorMap& qmap, const CUtensorMap& kmap, float tau,
                        int32_t* pattern_out, float* jsd_out, cudaStream_t st);
cudaError_t launch_select(const Shape& s, const WsLayout& L, void* ws, float gamma, int min_budget,
                          const fp_select_options& opt, int32_t* row_ptr, int32_t* col_idx,
                          fp_select_stats* stats, cudaStream_t st);
cudaError_t launch_attn(const Shape& s, const WsLayout& L, void* ws, const Layout& lay,
                        const CUtensorMap& qmap, const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                        const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                        const void* const* peer_o, int n_peer, cudaStream_t st);

}  // namespace fp
