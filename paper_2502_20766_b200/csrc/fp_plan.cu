// fp_plan.cu -- stage (i) of FlexPrefill: sparse pattern search (Alg. 2,
// P:299-327) plus the Vertical-Slash line scores of Alg. 3,
// computed once from the same representative attention, and the
// Query-Aware pooled map of Alg. 4 for QA heads.
//
// Kernels (one stream, no host sync):
//   rep1_kernel   N1a  (fp_rep.cu) S = Q^ K^T per (key chunk, KV group, <= 4
//                      heads) on tcgen05 -> partial row max / sum-exp
//   rep_stats         combine partials -> per-row max and M' = max + log2(sum)
//                     (n <= 32k: done by the rep2 CTAs themselves)
//   rep2_kernel   N1b  (fp_rep.cu) S^T = K Q^T per (key chunk, KV group, <= 2
//                      heads) -> p, a_v (column sums), per-tile slash
//                      partials; the first subset of a group writes K_bar
//   line_sums         a_s[o] from the overlapping tile partials (fixed order),
//                     a_hat[kb] = sum of a_v over kb (A2), As[D] (A12)
//   pattern_kernel N3 a_bar = softmax(avgpool(Q^) K_bar^T / sqrt d), D_JS, decision
//   qbar_kernel   N4a avg-pooled Q per block (QA heads only)
//   pooled_logits N4b block-causal pooled logits, 32x32 tiles (QA heads only)
//   pooled_softmax N4c A_bar row softmax over kb <= qb, / nb (QA heads only)
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

namespace fp {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// deterministic block reductions (fixed shuffle tree + fixed smem order)
template <int NT>
__device__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x == 0) {
    for (int w = 0; w < NT / 32; ++w) t += red[w];
    red[32] = t;
  }
  __syncthreads();
  t = red[32];
  __syncthreads();
  return t;
}
template <int NT>
__device__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < NT / 32; ++w) t += red[w];
    red[32] = t;
  }
  __syncthreads();
  t = red[32];
  __syncthreads();
  return t;
}
template <int NT>
__device__ float block_max(float v, float* red) {
  v = warp_max(v);
  if (lane_id() == 0) red[warp_id()] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = -INFINITY;
    for (int w = 0; w < NT / 32; ++w) t = fmaxf(t, red[w]);
    red[32] = t;
  }
  __syncthreads();
  float t = red[32];
  __syncthreads();
  return t;
}

// per-row softmax statistics from the chunk partials (fixed chunk order):
// m_row = max, mp_row = M'_r = m_r + log2(l_r) (pass 2 computes
// p = exp2(s * scale - M'_r) = exp(s / sqrt d - max) / sum); rows outside Q^
// (block size 64: r < 64) get M' = +inf, i.e. p = 0
__global__ void rep_stats(int nchunks, int r_lo, const float* __restrict__ m_part,
                          const float* __restrict__ l_part, float* __restrict__ m_row,
                          float* __restrict__ mp_row) {
  FP_PDL_ENTRY();
  const int h = blockIdx.x, r = threadIdx.x;
  const float* mp = m_part + (size_t)h * nchunks * 128 + r;
  const float* lp = l_part + (size_t)h * nchunks * 128 + r;
  float m = -INFINITY;
  for (int c = 0; c < nchunks; ++c) m = fmaxf(m, mp[c * 128]);
  float l = 0.f;
  for (int c = 0; c < nchunks; ++c) l += lp[c * 128] * exp2f(mp[c * 128] - m);
  m_row[h * 128 + r] = m;
  mp_row[h * 128 + r] = r < r_lo ? INFINITY : m + log2f(l);
}

// One CTA per (key block kb, head): the slash scores of the block's offsets
// a_s[o] = (sum of the overlapping per-tile diagonal partials) / b (A9), then
// a_hat[kb] = sum_{j in kb} a_v[j] (A2) and As[kb] = sum_{o in block kb} a_s[o]
// (A12) -- one launch for what were two kernels (slash combine, block sums).
__global__ void line_sums(int n, int nt, int nb, int b, float inv_b, const float* __restrict__ as_part,
                          const float* __restrict__ a_v, float* __restrict__ a_s, float* __restrict__ a_hat,
                          float* __restrict__ As) {
  FP_PDL_ENTRY();
  __shared__ float red[33];
  const int kb = blockIdx.x, h = blockIdx.y;
  const int o = kb * b + (int)threadIdx.x;
  const bool in = (int)threadIdx.x < b && o < n;  // ragged last block (A26)
  float as = 0.f;
  if (in) {
    const int q = n - 128 - o;  // base(kt) = n - 128 - 128 kt ; delta = o - base = 128 kt - q
    const int kt_hi = (q + 127) >= 0 ? (q + 127) / 128 : -1;
    float sum = 0.f;
    for (int kt = kt_hi - 1; kt <= kt_hi; ++kt) {  // ascending kt
      if (kt < 0 || kt >= nt) continue;
      const int delta = 128 * kt - q;
      if (delta < -127 || delta > 127) continue;
      sum += as_part[((size_t)h * nt + kt) * 256 + delta + 127];
    }
    as = sum * inv_b;
    a_s[(size_t)h * n + o] = as;
  }
  const float sv = block_sum<128>(in ? a_v[(size_t)h * n + o] : 0.f, red);
  const float ss = block_sum<128>(in ? as : 0.f, red);
  if (threadIdx.x == 0) {
    a_hat[(size_t)h * nb + kb] = sv;
    As[(size_t)h * nb + kb] = ss;
  }
}

// Alg. 2: a_bar, D_JS (base 2, A1), decision (strict <, A14). One CTA of 512
// threads per head: q_bar = avgpool(Q^) (4 row quarters x 128 dims), one
// pooled logit per thread and key block (a full 128-dim dot product with
// float4 loads of K_bar, fixed order), then the softmax and the JSD terms.
constexpr int kPatThreads = 512;
__global__ void __launch_bounds__(kPatThreads) pattern_kernel(
    const __nv_bfloat16* __restrict__ q, TLayout ql, const float* __restrict__ k_bar,
    const float* __restrict__ a_hat, int H, int G, int n, int nb, int b, float scale, float tau,
    float* __restrict__ a_bar, int32_t* __restrict__ pattern_ws, float* __restrict__ jsd_ws,
    int32_t* __restrict__ pattern_out, float* __restrict__ jsd_out) {
  FP_PDL_ENTRY();
  extern __shared__ __align__(16) float psm[];  // qbar[128] | qpart[4][128] | logits[nb] | red[33]
  float* qbar = psm;
  float* qpart = psm + 128;
  float* logit = qpart + 512;
  float* red = logit + nb;
  const int h = blockIdx.x, g = h / (H / G);
  const int tid = threadIdx.x;
  {
    // q_bar = avgpool(Q^), Q^ = the last b query rows
    const int d = tid & 127, rq = tid >> 7, rows = b / 4;
    const uint16_t* qh = reinterpret_cast<const uint16_t*>(q) + toff(ql, h, n - b + rq * rows) + d;
    float a0 = 0.f, a1 = 0.f;
#pragma unroll 4
    for (int r = 0; r < rows; r += 2) {
      a0 += bf16_to_f32(qh[(size_t)r * ql.rs]);
      a1 += bf16_to_f32(qh[(size_t)(r + 1) * ql.rs]);
    }
    qpart[rq * 128 + d] = a0 + a1;
  }
  __syncthreads();
  if (tid < 128) qbar[tid] = ((qpart[tid] + qpart[128 + tid]) + (qpart[256 + tid] + qpart[384 + tid])) / (float)b;
  __syncthreads();
  for (int kb = tid; kb < nb; kb += kPatThreads) {
    const float4* kv = reinterpret_cast<const float4*>(k_bar + ((size_t)g * nb + kb) * 128);
    float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      const float4 x = __ldg(kv + c);
      d0 = fmaf(qbar[4 * c], x.x, d0);
      d1 = fmaf(qbar[4 * c + 1], x.y, d1);
      d2 = fmaf(qbar[4 * c + 2], x.z, d2);
      d3 = fmaf(qbar[4 * c + 3], x.w, d3);
    }
    logit[kb] = ((d0 + d1) + (d2 + d3)) * scale;
  }
  __syncthreads();
  float mx = -INFINITY;
  for (int kb = tid; kb < nb; kb += kPatThreads) mx = fmaxf(mx, logit[kb]);
  mx = block_max<kPatThreads>(mx, red);
  float se = 0.f;
  for (int kb = tid; kb < nb; kb += kPatThreads) se += expf(logit[kb] - mx);
  se = block_sum<kPatThreads>(se, red);
  // JSD terms in fp64: D = sqrt(JSD) amplifies rounding near D = 0
  double js = 0.0;
  for (int kb = tid; kb < nb; kb += kPatThreads) {
    const float ab = expf(logit[kb] - mx) / se;
    a_bar[(size_t)h * nb + kb] = ab;
    const double pa = ab, ph = a_hat[(size_t)h * nb + kb];
    const double m = 0.5 * (pa + ph);
    if (pa > 0.0) js += pa * log2(pa / m);
    if (ph > 0.0) js += ph * log2(ph / m);
  }
  __shared__ double redd[33];
  js = block_sum_d<kPatThreads>(js, redd);
  if (tid == 0) {
    const float D = (float)sqrt(fmax(0.0, 0.5 * js));
    const int pat = (D < tau) ? 1 : 0;
    pattern_ws[h] = pat;
    jsd_ws[h] = D;
    if (pattern_out) pattern_out[h] = pat;
    if (jsd_out) jsd_out[h] = D;
  }
}

// avg-pooled queries of Query-Aware heads (Alg. 4 line 1)
// (a ragged last block averages over its actual rows, A26). 256 threads per
// (block, head): thread t sums 8 dims (one 16-B load per row) of b/16 rows,
// the 16 row groups are combined in a fixed order.
__global__ void __launch_bounds__(256) qbar_kernel(const __nv_bfloat16* __restrict__ q, TLayout ql,
                                                   const int32_t* __restrict__ pattern, int H, int n,
                                                   int nb, int b, float* __restrict__ q_bar) {
  FP_PDL_ENTRY();
  __shared__ float red[16][128];
  const int qb = blockIdx.x;
  // heads [h_lo, h_hi) of this CTA (one each when every head is pooled; the
  // Query-Aware heads of a range otherwise: no CTA per skipped head)
  const int h_lo = blockIdx.y * H / gridDim.y, h_hi = (blockIdx.y + 1) * H / gridDim.y;
  for (int h = h_lo; h < h_hi; ++h) {
  if (pattern && pattern[h] != 1) continue;  // pattern == nullptr: every head
  __syncthreads();  // red[] of the previous head consumed
  const int tid = threadIdx.x;
  const int c8 = tid & 15, rg = tid >> 4, rows = b >> 4;
  const int cnt = min(b, n - qb * b);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const __nv_bfloat16* base = q + toff(ql, h, qb * b) + c8 * 8;
#pragma unroll 8
  for (int rr = 0; rr < rows; ++rr) {
    const int row = rg * rows + rr;
    if (row < cnt) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(base + (size_t)row * ql.rs));
      const uint32_t wv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[2 * e] += __uint_as_float(wv[e] << 16);
        acc[2 * e + 1] += __uint_as_float(wv[e] & 0xffff0000u);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[rg][c8 * 8 + e] = acc[e];
  __syncthreads();
  if (tid < 128) {
    float sum = 0.f;
#pragma unroll
    for (int g2 = 0; g2 < 16; ++g2) sum += red[g2][tid];
    q_bar[((size_t)h * nb + qb) * 128 + tid] = sum / (float)cnt;
  }
  }
}

// A_bar[qb, kb <= qb] = softmax_row(scale * Qbar[qb] . Kbar[kb]) / nb  (A5)
// Two kernels: pooled_logits computes the block-causal logits tile by tile
// (PT x PT block pairs per CTA, fp32 FFMA dot products in fixed d order
// 0..127) straight into the packed A_bar rows; pooled_softmax normalises each
// row in place.
//
// pooled_logits: grid (ntri, head ranges); lower-triangle tile index -> (row
// tile rt, column tile ct <= rt). PT * PT / 16 threads, each a 4 x 4 block of
// logits. The work of a CTA is a list of units (QA head of its range, half of
// d); the Qbar / Kbar tiles of unit u + 1 are copied (cp.async, 16 B per
// thread and row chunk) into the other of two shared buffers while unit u is
// multiplied. Tiles are transposed [d / 4][row] with one float4 of padding per
// d row (the copies of a warp -- consecutive d / 4 of one row, coalesced in
// global memory -- land in distinct bank quads).
constexpr int kPLMaxHeads = 64;  // heads per range (launch: H / gridDim.y <= 64)
FP_DEV void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
FP_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
FP_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
template <int PT>
constexpr size_t pooled_logits_smem() {
  return sizeof(float4) * 2 * 2 * 16 * (PT + 1);
}
template <int PT>
__global__ void __launch_bounds__(PT * PT / 16) pooled_logits(
    const float* __restrict__ q_bar, const float* __restrict__ k_bar,
    const int32_t* __restrict__ pattern, int H, int G, int nb, float scale,
    float* __restrict__ A_bar) {
  constexpr int NT = PT * PT / 16;
  FP_PDL_ENTRY();
  extern __shared__ float4 pl_smem[];  // [buffer][q / k][16][PT + 1]
  __shared__ int qah[kPLMaxHeads];
  __shared__ int nqa_s;
  const int h_lo = blockIdx.y * H / gridDim.y, h_hi = (blockIdx.y + 1) * H / gridDim.y;
  // triangular decode of blockIdx.x = rt (rt + 1) / 2 + ct
  int rt = (int)((sqrtf(8.0f * (float)blockIdx.x + 1.0f) - 1.0f) * 0.5f);
  while ((rt + 1) * (rt + 2) / 2 <= (int)blockIdx.x) ++rt;
  while (rt * (rt + 1) / 2 > (int)blockIdx.x) --rt;
  const int ct = (int)blockIdx.x - rt * (rt + 1) / 2;
  const int tid = threadIdx.x;
  if (tid == 0) {
    int c = 0;
    for (int h = h_lo; h < h_hi; ++h)
      if (!pattern || pattern[h] == 1) qah[c++] = h;
    nqa_s = c;
  }
  __syncthreads();
  const int nu = 2 * nqa_s;
  if (nu == 0) return;
  auto buf = [&](int b, int qk, int d4, int row) -> float4* {
    return pl_smem + ((b * 2 + qk) * 16 + d4) * (PT + 1) + row;
  };
  auto fill = [&](int u) {
    const int h = qah[u >> 1], dh = u & 1, g = h / (H / G), b = u & 1;
    for (int e = tid; e < PT * 16; e += NT) {
      const int er = e >> 4, d4 = e & 15;
      const int qb = rt * PT + er, kb = ct * PT + er;
      cp_async16(buf(b, 0, d4, er), q_bar + ((size_t)h * nb + min(qb, nb - 1)) * 128 + (dh * 16 + d4) * 4, qb < nb);
      cp_async16(buf(b, 1, d4, er), k_bar + ((size_t)g * nb + min(kb, nb - 1)) * 128 + (dh * 16 + d4) * 4, kb < nb);
    }
    cp_async_commit();
  };
  // rows rr + TPR i, columns cc + TPR j: a warp's Kbar reads are consecutive
  // float4s (conflict-free), its A_bar stores consecutive kb
  constexpr int TPR = PT / 4;
  const int rr = tid / TPR, cc = tid % TPR;
  float acc[4][4];
  fill(0);
  for (int u = 0; u < nu; ++u) {
    if (u + 1 < nu) {
      fill(u + 1);  // buffer (u + 1) & 1: consumed by unit u - 1 (barrier at its end)
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if ((u & 1) == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    }
    const int b = u & 1;
#pragma unroll 4
    for (int d4 = 0; d4 < 16; ++d4) {
      float4 qv[4], kv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        qv[i] = *buf(b, 0, d4, rr + TPR * i);
        kv[i] = *buf(b, 1, d4, cc + TPR * i);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j] = fmaf(qv[i].x, kv[j].x, acc[i][j]);
          acc[i][j] = fmaf(qv[i].y, kv[j].y, acc[i][j]);
          acc[i][j] = fmaf(qv[i].z, kv[j].z, acc[i][j]);
          acc[i][j] = fmaf(qv[i].w, kv[j].w, acc[i][j]);
        }
    }
    __syncthreads();  // buffer b is free for unit u + 2
    if (u & 1) {
      const int h = qah[u >> 1];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int qb = rt * PT + rr + TPR * i;
        if (qb >= nb) continue;
        float* row = A_bar + (size_t)h * ((size_t)nb * (nb + 1) / 2) + (size_t)qb * (qb + 1) / 2;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int kb = ct * PT + cc + TPR * j;
          if (kb <= qb) row[kb] = acc[i][j] * scale;
        }
      }
    }
  }
}

constexpr int kMapThreads = 256;
__global__ void __launch_bounds__(kMapThreads) pooled_softmax(const int32_t* __restrict__ pattern,
                                                              int H, int nb, float* __restrict__ A_bar) {
  FP_PDL_ENTRY();
  __shared__ float red[33];
  const int qb = blockIdx.x;
  const int h_lo = blockIdx.y * H / gridDim.y, h_hi = (blockIdx.y + 1) * H / gridDim.y;
  for (int h = h_lo; h < h_hi; ++h) {
  if (pattern && pattern[h] != 1) continue;
  float* row = A_bar + (size_t)h * ((size_t)nb * (nb + 1) / 2) + (size_t)qb * (qb + 1) / 2;
  const int tid = threadIdx.x;
  float mx = -INFINITY;
  for (int kb = tid; kb <= qb; kb += kMapThreads) mx = fmaxf(mx, row[kb]);
  mx = block_max<kMapThreads>(mx, red);
  float se = 0.f;
  for (int kb = tid; kb <= qb; kb += kMapThreads) se += expf(row[kb] - mx);
  se = block_sum<kMapThreads>(se, red);
  const float inv_nb = 1.0f / (float)nb;
  for (int kb = tid; kb <= qb; kb += kMapThreads) row[kb] = (expf(row[kb] - mx) / se) * inv_nb;
  }
}

}  // namespace

// One non-blocking side stream per (calling thread, device) for the
// pooled-map branch of fp_plan, created on first use. Per thread, so calls
// from different threads never share it (no false dependencies between their
// streams, and a graph capture in one thread cannot pull another thread's
// work into its graph). nullptr if it cannot be created: the branch then runs
// in order on the caller's stream.
namespace {
struct SideStreams {
  cudaStream_t s[64] = {};
  ~SideStreams() {
    for (cudaStream_t x : s)
      if (x) cudaStreamDestroy(x);
  }
};
}  // namespace
cudaStream_t plan_side_stream() {
  thread_local SideStreams tl;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (!tl.s[dev] && cudaStreamCreateWithFlags(&tl.s[dev], cudaStreamNonBlocking) != cudaSuccess)
    tl.s[dev] = nullptr;
  return tl.s[dev];
}

cudaError_t launch_rep(const Shape& s, const CUtensorMap& qmap, const CUtensorMap& kmap, int Hp, int Gp,
                       float scale_log2, float* m_part, float* l_part, const float* mp_row, float* k_bar,
                       float* a_v, float* as_part, int pass, cudaStream_t st);

cudaError_t launch_plan(const Shape& s, const WsLayout& L, void* ws, const void* q, const void* k,
                        const Layout& lay, const CUtensorMap& qmap, const CUtensorMap& kmap, float tau,
                        int32_t* pattern_out, float* jsd_out, cudaStream_t st) {
  const float scale = 1.0f / sqrtf(128.0f);
  const float scale_log2 = scale * kLog2e;
  float* m_part = wsp<float>(ws, L.m_part);
  float* l_part = wsp<float>(ws, L.l_part);
  float* m_row = wsp<float>(ws, L.m_row);
  float* mp_row = wsp<float>(ws, L.mp_row);  // M'_r = m_r + log2 l_r
  (void)k;
  const int Hp = lay.q.per, Gp = lay.k.per;
  {
    cudaError_t ea = ensure_smem_attr((const void*)pooled_logits<64>, pooled_logits_smem<64>());
    if (ea == cudaSuccess) ea = ensure_smem_attr((const void*)pooled_logits<32>, pooled_logits_smem<32>());
    if (ea != cudaSuccess) return ea;
  }
  // The Query-Aware pooled map (a3: q_bar, pooled logits, row softmax) needs
  // only Q and K_bar, not the pattern: it can run for EVERY head on a side stream,
  // concurrently with the second representative pass .. pattern_kernel, and is
  // joined back before fp_plan returns (VS heads' maps are computed and
  // ignored). This takes the three kernels off the stage's critical path (they
  // are latency-bound at short n). Fork / join through events: stream-ordered
  // and graph-capturable. Only for short sequences (nb <= 256 blocks): there the
  // kernels are latency-bound and the extra maps of the VS heads are cheap; at
  // 128k the all-heads map costs more than it hides.
  cudaStream_t side = s.nb <= 256 ? plan_side_stream() : nullptr;
  cudaEvent_t e_fork = nullptr, e_kbar = nullptr, e_join = nullptr;
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t r) {
    if (e == cudaSuccess && r != cudaSuccess) e = r;
  };
  if (side) {
    chk(cudaEventCreateWithFlags(&e_fork, cudaEventDisableTiming));
    chk(cudaEventCreateWithFlags(&e_kbar, cudaEventDisableTiming));
    chk(cudaEventCreateWithFlags(&e_join, cudaEventDisableTiming));
    chk(cudaEventRecord(e_fork, st));
    chk(cudaStreamWaitEvent(side, e_fork, 0));
  }
  const int32_t* qa_only = side ? nullptr : wsp<int32_t>(ws, L.pattern);
  cudaStream_t sq = side ? side : st;
  // 64 x 64 logit tiles from nb >= 256 (fewer, larger CTAs: half the tile
  // traffic per logit); 32 x 32 at short n (more CTAs for few blocks)
  const bool big_tiles = s.nb >= 256;
  const int kPT = big_tiles ? 64 : 32;
  const int nt = (s.nb + kPT - 1) / kPT;
  // one CTA per head when every head is pooled (short n, side stream);
  // otherwise CTAs over head ranges (<= kPLMaxHeads heads) that skip the
  // Vertical-Slash heads
  const int hy = qa_only ? std::min(s.H, std::max(4, (s.H + kPLMaxHeads - 1) / kPLMaxHeads)) : s.H;
  if (side)  // q_bar does not need K_bar: start it at the fork
    FP_LAUNCH(qbar_kernel, dim3(s.nb, hy), 256, 0, sq, reinterpret_cast<const __nv_bfloat16*>(q), lay.q,
                                                 qa_only, s.H, s.n, s.nb, s.b, wsp<float>(ws, L.q_bar));
  auto pooled_map = [&]() {
    if (!side)
      FP_LAUNCH(qbar_kernel, dim3(s.nb, hy), 256, 0, sq, reinterpret_cast<const __nv_bfloat16*>(q), lay.q,
                                                   qa_only, s.H, s.n, s.nb, s.b, wsp<float>(ws, L.q_bar));
    if (side) chk(cudaStreamWaitEvent(side, e_kbar, 0));  // K_bar from the second pass
    if (big_tiles)
      FP_LAUNCH(pooled_logits<64>, dim3(nt * (nt + 1) / 2, hy), 256, pooled_logits_smem<64>(), sq,
                wsp<float>(ws, L.q_bar), wsp<float>(ws, L.k_bar), qa_only, s.H, s.G, s.nb, scale,
                wsp<float>(ws, L.A_bar));
    else
      FP_LAUNCH(pooled_logits<32>, dim3(nt * (nt + 1) / 2, hy), 64, pooled_logits_smem<32>(), sq,
                wsp<float>(ws, L.q_bar), wsp<float>(ws, L.k_bar), qa_only, s.H, s.G, s.nb, scale,
                wsp<float>(ws, L.A_bar));
    FP_LAUNCH(pooled_softmax, dim3(s.nb, hy), kMapThreads, 0, sq, qa_only, s.H, s.nb, wsp<float>(ws, L.A_bar));
  };
  chk(launch_rep(s, qmap, kmap, Hp, Gp, scale_log2, m_part, l_part, nullptr, nullptr, nullptr, nullptr, 1, st));
  // few chunks: pass 2 combines the row statistics itself (one launch less);
  // many: rep_stats once per head (every pass-2 CTA would re-read nchunks x 128 x 2)
  const bool fold = s.nchunks <= 32;
  if (!fold) FP_LAUNCH(rep_stats, s.H, 128, 0, st, s.nchunks, 128 - s.b, m_part, l_part, m_row, mp_row);
  chk(launch_rep(s, qmap, kmap, Hp, Gp, scale_log2, fold ? m_part : nullptr, fold ? l_part : nullptr, mp_row, wsp<float>(ws, L.k_bar),
                 wsp<float>(ws, L.a_v), wsp<float>(ws, L.as_part), 2, st));
  if (side) {
    chk(cudaEventRecord(e_kbar, st));
    pooled_map();
    chk(cudaEventRecord(e_join, side));
  }
  FP_LAUNCH(line_sums, dim3(s.nb, s.H), 128, 0, st, s.n, s.nt, s.nb, s.b, 1.0f / (float)s.b,
            wsp<float>(ws, L.as_part), wsp<float>(ws, L.a_v), wsp<float>(ws, L.a_s), wsp<float>(ws, L.a_hat),
            wsp<float>(ws, L.As));
  const size_t psm = (128 + 512 + (size_t)s.nb + 33) * 4;
  FP_LAUNCH(pattern_kernel, s.H, kPatThreads, psm, st, 
      reinterpret_cast<const __nv_bfloat16*>(q), lay.q, wsp<float>(ws, L.k_bar), wsp<float>(ws, L.a_hat),
      s.H, s.G, s.n, s.nb, s.b, scale, tau, wsp<float>(ws, L.a_bar), wsp<int32_t>(ws, L.pattern),
      wsp<float>(ws, L.jsd), pattern_out, jsd_out);
  if (side) {
    chk(cudaStreamWaitEvent(st, e_join, 0));
  } else {
    pooled_map();  // no side stream: QA heads only, after the pattern
  }
  if (e_fork) cudaEventDestroy(e_fork);
  if (e_kbar) cudaEventDestroy(e_kbar);
  if (e_join) cudaEventDestroy(e_join);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace fp
