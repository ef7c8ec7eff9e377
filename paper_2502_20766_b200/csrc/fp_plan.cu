// fp_plan.cu -- stage (i) of FlexPrefill: sparse pattern search (Alg. 2,
// P:299-327) plus the Vertical-Slash line scores of Alg. 3,
// computed once from the same representative attention, and the
// Query-Aware pooled map of Alg. 4 for QA heads.
//
// Kernels (one stream, no host sync):
//   rep_pass<1>   N1a  S = Q^ K^T per (key chunk, head) on tcgen05 -> partial
//                      row max / sum-exp; first head of each KV group also
//                      writes the avg-pooled keys K_bar
//   rep_stats         combine partials -> per-row max and 1/sum (fixed order)
//   rep_pass<2>   N1b  S^T = K Q^T per (key chunk, head) -> p = softmax entries,
//                      a_v (column sums) and per-tile slash (diagonal) partials
//   slash_combine     a_s[o] from the overlapping tile partials (fixed order)
//   block_sums        a_hat[kb] = sum of a_v over kb (A2); As[D] (A12)
//   pattern_kernel N3 a_bar = softmax(avgpool(Q^) K_bar^T / sqrt d), D_JS, decision
//   qbar_kernel   N4a avg-pooled Q per block (QA heads only)
//   pooled_logits N4b block-causal pooled logits, 32x32 tiles (QA heads only)
//   pooled_softmax N4c A_bar row softmax over kb <= qb, / nb (QA heads only)
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

namespace fp {

namespace {

constexpr int kRepThreads = 256;
constexpr int kStages = 2;

struct RepSmem {
  // tiles first (1024-B aligned by the dynamic smem base alignment)
  uint8_t qhat[kTileBytes];
  uint8_t kst[kStages][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kStages];
  uint64_t mma_done[2];
  uint32_t tmem_base;
  float m_row[128];
  float il_row[128];
  float red[512];
};
// pass-2 slash partials: per warp, 4 column segments of 16, 47 diagonals each
constexpr int kSeg = 4, kSegCols = 16, kSegDiag = kSegCols + 31, kSegStride = 48;

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

// --------------------------------------------------------------------------
// Representative pass. PASS 1: A = Q^ (128 rep rows), B = K tile -> TMEM
// lane = rep row r, column = key. PASS 2: A = K tile, B = Q^ -> lane = key,
// column = rep row r. Both are M=N=K=128 bf16 UMMAs on K-major SW128 tiles.
// 8 warps: warp w reads TMEM lane quarter (w % 4) and column half (w / 4).
template <int PASS>
__global__ void __launch_bounds__(kRepThreads, 2)
    rep_pass(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
             int H, int G, int Hp, int Gp, int n, int nb, int nt, int bsz, int nchunks, int ct,
             float scale_log2,
             float* __restrict__ m_part,
             float* __restrict__ l_part, const float* __restrict__ m_row,
             const float* __restrict__ il_row, float* __restrict__ k_bar, float* __restrict__ a_v,
             float* __restrict__ as_part) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SWIZZLE_128B tiles need 1024-B aligned shared addresses
  uint8_t* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  RepSmem& sm = *reinterpret_cast<RepSmem*>(sbase);
  float* P2 = reinterpret_cast<float*>(sbase + sizeof(RepSmem));  // PASS 2 slash partials

  const int tid = threadIdx.x;
  const int wq = warp_id() & 3, half = warp_id() >> 2;
  const int lane_row = wq * 32 + lane_id();  // TMEM lane of this thread
  const int chunk = blockIdx.x, h = blockIdx.y;
  const int g = h / (H / G);
  const int t0 = chunk * ct;
  const int ntile = min(ct, nt - t0);
  // block_size b = 64: Q^ is the last 64 rows, i.e. rows r >= 64 of the
  // 128-row representative tile (p_r = n - 128 + r either way)
  const int r_lo = 128 - bsz;
  const float inv_b = 1.0f / (float)bsz;
  const bool do_kbar = (PASS == 1) && (h % (H / G) == 0);

  if (warp_id() == 0) tmem_alloc(&sm.tmem_base, 256);
  if (tid == 0) {
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kStages; ++s) mbar_init(&sm.k_full[s], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&sm.mma_done[b], 1);
    mbar_fence_init();
  }
  if (PASS == 2 && tid < 128) {
    sm.m_row[tid] = m_row[h * 128 + tid];
    sm.il_row[tid] = il_row[h * 128 + tid];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  constexpr uint32_t idesc = make_idesc_bf16(128, 128, false);

  // issued by all of warp 0 (warp-uniform operands, elect.sync inside the
  // asm): a lane-0 issue loop cost ~50-130 cycles per MMA in R2UR / branch
  // overhead, and warp 0 also does softmax work the whole CTA waits for
  auto issue_mma = [&](int t) {
    const int s = t % kStages, b = t & 1;
    mbar_wait(&sm.k_full[s], (t / kStages) & 1);
    tc_fence_after();
    const uint64_t qd = sdesc_kmajor(smem_u32(sm.qhat), 0), kd = sdesc_kmajor(smem_u32(sm.kst[s]), 0);
    umma_ss_chain8_elect(tbase + b * 128, PASS == 1 ? qd : kd, PASS == 1 ? kd : qd, idesc);
    umma_commit_elect(&sm.mma_done[b]);
  };

  if (tid == 0) {
    mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
    tma_tile(sm.qhat, &qmap, &sm.q_full, n - 128, h, Hp);
    for (int s = 0; s < kStages && s < ntile; ++s) {
      mbar_arrive_expect_tx(&sm.k_full[s], kTileBytes);
      tma_tile(sm.kst[s], &kmap, &sm.k_full[s], (t0 + s) * 128, g, Gp);
    }
  }
  if (warp_id() == 0) {
    __syncwarp();
    mbar_wait(&sm.q_full, 0);
    issue_mma(0);
  }

  float m_loc = -INFINITY, l_loc = 0.f;  // PASS 1 running row stats of this column half (log2)

  for (int t = 0; t < ntile; ++t) {
    if (warp_id() == 0 && t + 1 < ntile) issue_mma(t + 1);
    const int b = t & 1;
    const int tile = t0 + t;
    // key tile*128 + c is visible from rep row r iff c <= lim + r (p_r = n-128+r);
    // only the last one or two tiles (ragged n) need the mask
    const int lim = n - 128 - tile * 128;
    const bool last = lim < 127;
    mbar_wait(&sm.mma_done[b], (t >> 1) & 1);
    tc_fence_after();

    uint32_t v[64];
    const uint32_t ta = tmem_addr(tbase + b * 128, wq * 32, half * 64);
    tmem_ld32(ta, v);
    tmem_ld32(ta + 32, v + 32);
    tmem_wait_ld();

    if (PASS == 1) {
      // lane = rep row r; key j = tile*128 + c visible iff j <= p_r = n-128+r
      const int r = lane_row;
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 64; ++c) {
        float x = __uint_as_float(v[c]) * scale_log2;
        if (last && half * 64 + c > lim + r) x = -INFINITY;
        v[c] = __float_as_uint(x);
        mx4[c & 3] = fmaxf(mx4[c & 3], x);
      }
      const float m_new = fmaxf(m_loc, fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])));
      // a column half can be fully masked (last tiles): keep it at -inf, sum 0
      const float m_safe = (m_new == -INFINITY) ? 0.f : m_new;
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 64; ++c) s4[c & 3] += fast_exp2(__uint_as_float(v[c]) - m_safe);
      l_loc = l_loc * fast_exp2(m_loc - m_safe) + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
      m_loc = m_new;
      if (do_kbar) {
        // avg-pooled key of this block: dimension d = tid % 128, rows of this half
        const uint8_t* kt = sm.kst[t % kStages];
        const int d = tid & 127, r0 = (tid >> 7) * 64;
        float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
        for (int row = 0; row < 64; row += 2) {
          a0 += bf16_to_f32(*reinterpret_cast<const uint16_t*>(kt + sw128_offset(r0 + row, d)));
          a1 += bf16_to_f32(*reinterpret_cast<const uint16_t*>(kt + sw128_offset(r0 + row + 1, d)));
        }
        sm.red[tid] = a0 + a1;
        __syncthreads();
        // ragged last block: zero-filled rows past n, mean over the actual rows (A26)
        if (bsz == 128) {
          if (tid < 128)
            k_bar[((size_t)g * nb + tile) * 128 + tid] =
                (sm.red[tid] + sm.red[tid + 128]) / (float)min(128, n - tile * 128);
        } else {  // two 64-key blocks per tile: thread halves are the blocks
          const int kb = 2 * tile + (tid >> 7);
          const int cnt = min(64, n - kb * 64);
          if (cnt > 0) k_bar[((size_t)g * nb + kb) * 128 + (tid & 127)] = sm.red[tid] / (float)cnt;
        }
      }
    } else {
      // lane = key j_local, columns = rep rows r = half*64 .. half*64+63
      const int jl = lane_row;
      float cs[4] = {0.f, 0.f, 0.f, 0.f};
      // Slash partials without a transpose: diagonal delta = r - jl. A running
      // sum that moves up one lane per column follows one diagonal of this
      // warp's 32 x 64 sub-tile (lane L adds its p at column c to the run of
      // delta_local = c - L). Four 16-column segments run as independent
      // chains; lane 31 emits each finished run, the other lanes emit theirs
      // after a segment's last column. Partials land in P2[warp][seg][idx],
      // idx = delta_local - (16 seg - 31).
      float* wp = P2 + warp_id() * (kSeg * kSegStride);
      float run[kSeg] = {0.f, 0.f, 0.f, 0.f};
      const bool active = half * 64 >= r_lo;  // rows outside Q^ (b = 64): no probability mass
#pragma unroll
      for (int i = 0; i < kSegCols; ++i) {
#pragma unroll
        for (int sg = 0; sg < kSeg; ++sg) {
          const int c = sg * kSegCols + i;
          const int r = half * 64 + c;
          float p = 0.f;
          if (active) {
            p = fast_exp2(fmaf(__uint_as_float(v[c]), scale_log2, -sm.m_row[r])) * sm.il_row[r];
            if (last && jl > lim + r) p = 0.f;
          }
          cs[c & 3] += p;
          run[sg] += p;
          if (lane_id() == 31) wp[sg * kSegStride + i] = run[sg];
          if (i + 1 < kSegCols) {
            run[sg] = __shfl_up_sync(0xffffffffu, run[sg], 1);
            if (lane_id() == 0) run[sg] = 0.f;
          }
        }
      }
#pragma unroll
      for (int sg = 0; sg < kSeg; ++sg)
        if (lane_id() < 31) wp[sg * kSegStride + kSegDiag - 1 - lane_id()] = run[sg];
      sm.red[half * 128 + jl] = (cs[0] + cs[1]) + (cs[2] + cs[3]);
      __syncthreads();
      if (tid < 128 && tile * 128 + tid < n)
        a_v[(size_t)h * n + tile * 128 + tid] = (sm.red[tid] + sm.red[128 + tid]) * inv_b;
      // slash partial of diagonal dl = r - jl in [-127, 127] of this tile, one
      // per thread, summed over the 8 warps and their segments in a fixed order;
      // offset o = p_r - j = (n - 128 - tile*128) + dl
      if (tid < 255) {
        const int dl = tid - 127;
        float acc = 0.f;
#pragma unroll
        for (int w8 = 0; w8 < 8; ++w8) {
          const int dloc = dl - (w8 >> 2) * 64 + (w8 & 3) * 32;  // delta_local in warp w8
#pragma unroll
          for (int sg = 0; sg < kSeg; ++sg) {
            const int idx = dloc - (sg * kSegCols - 31);
            if (idx >= 0 && idx < kSegDiag) acc += P2[(w8 * kSeg + sg) * kSegStride + idx];
          }
        }
        as_part[((size_t)h * nt + tile) * 256 + dl + 127] = acc;
      }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0 && t + kStages < ntile) {
      const int s = t % kStages;
      mbar_arrive_expect_tx(&sm.k_full[s], kTileBytes);
      tma_tile(sm.kst[s], &kmap, &sm.k_full[s], (t0 + t + kStages) * 128, g, Gp);
    }
  }

  if (PASS == 1) {
    // combine the two column halves of each row
    sm.red[tid] = m_loc;
    sm.red[256 + tid] = l_loc;
    __syncthreads();
    if (tid < 128) {
      const float m0 = sm.red[tid], m1 = sm.red[tid + 128];
      const float m = fmaxf(m0, m1);
      // ragged n: a whole chunk can be invisible to a row (m = -inf, l = 0)
      const float ms = (m == -INFINITY) ? 0.f : m;
      const float l = sm.red[256 + tid] * fast_exp2(m0 - ms) + sm.red[256 + tid + 128] * fast_exp2(m1 - ms);
      m_part[((size_t)h * nchunks + chunk) * 128 + tid] = m;
      l_part[((size_t)h * nchunks + chunk) * 128 + tid] = l;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc(tbase, 256);
}

// per-row softmax statistics from the chunk partials (fixed chunk order)
__global__ void rep_stats(int nchunks, const float* __restrict__ m_part,
                          const float* __restrict__ l_part, float* __restrict__ m_row,
                          float* __restrict__ il_row) {
  const int h = blockIdx.x, r = threadIdx.x;
  const float* mp = m_part + (size_t)h * nchunks * 128 + r;
  const float* lp = l_part + (size_t)h * nchunks * 128 + r;
  float m = -INFINITY;
  for (int c = 0; c < nchunks; ++c) m = fmaxf(m, mp[c * 128]);
  float l = 0.f;
  for (int c = 0; c < nchunks; ++c) l += lp[c * 128] * exp2f(mp[c * 128] - m);
  m_row[h * 128 + r] = m;
  il_row[h * 128 + r] = 1.0f / l;
}

// a_s[o] = (sum of the overlapping per-tile diagonal partials) / b  (A9)
__global__ void slash_combine(int n, int nt, float inv_b, const float* __restrict__ as_part,
                              float* __restrict__ a_s) {
  const int h = blockIdx.y;
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) return;
  const int q = n - 128 - o;  // base(kt) = n - 128 - 128 kt ; delta = o - base = 128 kt - q
  int kt_hi = (q + 127) >= 0 ? (q + 127) / 128 : -1;
  float s = 0.f;
  for (int kt = kt_hi - 1; kt <= kt_hi; ++kt) {  // ascending kt
    if (kt < 0 || kt >= nt) continue;
    const int delta = 128 * kt - q;
    if (delta < -127 || delta > 127) continue;
    s += as_part[((size_t)h * nt + kt) * 256 + delta + 127];
  }
  a_s[(size_t)h * n + o] = s * inv_b;
}

// a_hat[kb] = sum_{j in kb} a_v[j] (A2) and As[D] = sum_{o in block D} a_s[o] (A12)
__global__ void block_sums(int n, int nb, int b, const float* __restrict__ a_v,
                           const float* __restrict__ a_s, float* __restrict__ a_hat,
                           float* __restrict__ As) {
  __shared__ float red[33];
  const int kb = blockIdx.x, h = blockIdx.y;
  const size_t i = (size_t)h * n + (size_t)kb * b + threadIdx.x;
  const bool in = (int)threadIdx.x < b && kb * b + (int)threadIdx.x < n;  // ragged last block (A26)
  float sv = block_sum<128>(in ? a_v[i] : 0.f, red);
  float ss = block_sum<128>(in ? a_s[i] : 0.f, red);
  if (threadIdx.x == 0) {
    a_hat[(size_t)h * nb + kb] = sv;
    As[(size_t)h * nb + kb] = ss;
  }
}

// Alg. 2: a_bar, D_JS (base 2, A1), decision (strict <, A14)
constexpr int kPatThreads = 256;
__global__ void __launch_bounds__(kPatThreads) pattern_kernel(
    const __nv_bfloat16* __restrict__ q, TLayout ql, const float* __restrict__ k_bar,
    const float* __restrict__ a_hat, int H, int G, int n, int nb, int b, float scale, float tau,
    float* __restrict__ a_bar, int32_t* __restrict__ pattern_ws, float* __restrict__ jsd_ws,
    int32_t* __restrict__ pattern_out, float* __restrict__ jsd_out) {
  extern __shared__ float psm[];  // qbar[128] | logits[nb] | red[33]
  float* qbar = psm;
  float* logit = psm + 128;
  float* red = logit + nb;
  const int h = blockIdx.x, g = h / (H / G);
  const int tid = threadIdx.x;
  if (tid < 128) {
    // q_bar = avgpool(Q^), Q^ = the last b query rows
    const uint16_t* qh = reinterpret_cast<const uint16_t*>(q) + toff(ql, h, n - b) + tid;
    float acc = 0.f;
    for (int r = 0; r < b; ++r) acc += bf16_to_f32(qh[(size_t)r * ql.rs]);
    qbar[tid] = acc / (float)b;
  }
  __syncthreads();
  const int w = warp_id(), ln = lane_id();
  for (int kb = w; kb < nb; kb += kPatThreads / 32) {
    const float4 kv = *reinterpret_cast<const float4*>(k_bar + ((size_t)g * nb + kb) * 128 + ln * 4);
    float d = qbar[ln * 4] * kv.x + qbar[ln * 4 + 1] * kv.y + qbar[ln * 4 + 2] * kv.z +
              qbar[ln * 4 + 3] * kv.w;
    d = warp_sum(d);
    if (ln == 0) logit[kb] = d * scale;
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
// (a ragged last block averages over its actual rows, A26)
__global__ void qbar_kernel(const __nv_bfloat16* __restrict__ q, TLayout ql,
                            const int32_t* __restrict__ pattern, int n, int nb, int b,
                            float* __restrict__ q_bar) {
  const int qb = blockIdx.x, h = blockIdx.y;
  if (pattern && pattern[h] != 1) return;  // pattern == nullptr: every head
  const uint16_t* qh = reinterpret_cast<const uint16_t*>(q) + toff(ql, h, qb * b) + threadIdx.x;
  const int cnt = min(b, n - qb * b);
  float acc = 0.f;
#pragma unroll 8
  for (int r = 0; r < cnt; ++r) acc += bf16_to_f32(qh[(size_t)r * ql.rs]);
  q_bar[((size_t)h * nb + qb) * 128 + threadIdx.x] = acc / (float)cnt;
}

// A_bar[qb, kb <= qb] = softmax_row(scale * Qbar[qb] . Kbar[kb]) / nb  (A5)
// Two kernels: pooled_logits computes the block-causal logits tile by tile
// (32 x 32 block pairs per CTA, Qbar and Kbar tiles staged in shared memory,
// fp32 FFMA dot products in fixed d order) straight into the packed A_bar
// rows; pooled_softmax normalises each row in place.
constexpr int kPT = 32;  // row / column tile of the pooled logits
__global__ void __launch_bounds__(256) pooled_logits(
    const float* __restrict__ q_bar, const float* __restrict__ k_bar,
    const int32_t* __restrict__ pattern, int H, int G, int nb, float scale,
    float* __restrict__ A_bar) {
  const int rt = blockIdx.x, ct = blockIdx.y, h = blockIdx.z;
  if (ct > rt || (pattern && pattern[h] != 1)) return;
  __shared__ float qs[kPT][129];
  __shared__ float ks[kPT][129];
  const int g = h / (H / G);
  const int tid = threadIdx.x;
  for (int e = tid; e < kPT * 128; e += 256) {
    const int rr = e >> 7, d = e & 127;
    const int qb = rt * kPT + rr, kb = ct * kPT + rr;
    qs[rr][d] = (qb < nb) ? q_bar[((size_t)h * nb + qb) * 128 + d] : 0.f;
    ks[rr][d] = (kb < nb) ? k_bar[((size_t)g * nb + kb) * 128 + d] : 0.f;
  }
  __syncthreads();
  const int rr = tid >> 3, c0 = tid & 7;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int d = 0; d < 128; ++d) {
    const float qv = qs[rr][d];
#pragma unroll
    for (int m = 0; m < 4; ++m) acc[m] = fmaf(qv, ks[c0 + 8 * m][d], acc[m]);
  }
  const int qb = rt * kPT + rr;
  if (qb >= nb) return;
  float* row = A_bar + (size_t)h * ((size_t)nb * (nb + 1) / 2) + (size_t)qb * (qb + 1) / 2;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int kb = ct * kPT + c0 + 8 * m;
    if (kb <= qb) row[kb] = acc[m] * scale;
  }
}

constexpr int kMapThreads = 256;
__global__ void __launch_bounds__(kMapThreads) pooled_softmax(const int32_t* __restrict__ pattern,
                                                              int nb, float* __restrict__ A_bar) {
  __shared__ float red[33];
  const int qb = blockIdx.x, h = blockIdx.y;
  if (pattern && pattern[h] != 1) return;
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

size_t rep_smem_bytes(int pass) {
  size_t b = sizeof(RepSmem);
  if (pass == 2) b += (size_t)8 * kSeg * kSegStride * 4;
  return b + 1024;  // slack for manual alignment
}

cudaError_t launch_plan(const Shape& s, const WsLayout& L, void* ws, const void* q, const void* k,
                        const Layout& lay, const CUtensorMap& qmap, const CUtensorMap& kmap, float tau,
                        int32_t* pattern_out, float* jsd_out, cudaStream_t st) {
  const size_t sm1 = rep_smem_bytes(1), sm2 = rep_smem_bytes(2);
  cudaError_t ea = ensure_smem_attr((const void*)rep_pass<1>, sm1);
  if (ea == cudaSuccess) ea = ensure_smem_attr((const void*)rep_pass<2>, sm2);
  if (ea != cudaSuccess) return ea;
  const float scale = 1.0f / sqrtf(128.0f);
  const float scale_log2 = scale * kLog2e;
  float* m_part = wsp<float>(ws, L.m_part);
  float* l_part = wsp<float>(ws, L.l_part);
  float* m_row = wsp<float>(ws, L.m_row);
  float* il_row = wsp<float>(ws, L.il_row);
  dim3 grid(s.nchunks, s.H);
  (void)k;
  const int Hp = lay.q.per, Gp = lay.k.per;
  // The Query-Aware pooled map (a3: q_bar, pooled logits, row softmax) needs
  // only Q and K_bar, not the pattern: it can run for EVERY head on a side stream,
  // concurrently with rep_stats .. pattern_kernel, and is joined back before
  // fp_plan returns (VS heads' maps are computed and ignored). This takes the
  // three kernels off the stage's critical path (they are latency-bound at
  // short n). Fork / join through events: stream-ordered and graph-capturable.
  // Only for short sequences (nb <= 256 blocks): there the three kernels are
  // latency-bound and the extra maps of the VS heads are cheap; at 128k the
  // all-heads map costs more than it hides (measured with tools/plan_ab.py:
  // 4k plan 0.100 -> 0.083 ms, 8k 0.132 -> 0.117, 32k equal, 128k 1.42 -> 1.87).
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
  const int nt = (s.nb + kPT - 1) / kPT;
  auto pooled_map = [&]() {
    qbar_kernel<<<dim3(s.nb, s.H), 128, 0, sq>>>(reinterpret_cast<const __nv_bfloat16*>(q), lay.q,
                                                 qa_only, s.n, s.nb, s.b, wsp<float>(ws, L.q_bar));
    if (side) chk(cudaStreamWaitEvent(side, e_kbar, 0));  // K_bar from rep_pass<1>
    pooled_logits<<<dim3(nt, nt, s.H), 256, 0, sq>>>(wsp<float>(ws, L.q_bar), wsp<float>(ws, L.k_bar),
                                                     qa_only, s.H, s.G, s.nb, scale,
                                                     wsp<float>(ws, L.A_bar));
    pooled_softmax<<<dim3(s.nb, s.H), kMapThreads, 0, sq>>>(qa_only, s.nb, wsp<float>(ws, L.A_bar));
  };
  rep_pass<1><<<grid, kRepThreads, sm1, st>>>(qmap, kmap, s.H, s.G, Hp, Gp, s.n, s.nb, s.nt, s.b, s.nchunks, s.ct, scale_log2,
                                              m_part, l_part, m_row, il_row,
                                              wsp<float>(ws, L.k_bar), wsp<float>(ws, L.a_v),
                                              wsp<float>(ws, L.as_part));
  if (side) {
    chk(cudaEventRecord(e_kbar, st));
    pooled_map();
    chk(cudaEventRecord(e_join, side));
  }
  rep_stats<<<s.H, 128, 0, st>>>(s.nchunks, m_part, l_part, m_row, il_row);
  rep_pass<2><<<grid, kRepThreads, sm2, st>>>(qmap, kmap, s.H, s.G, Hp, Gp, s.n, s.nb, s.nt, s.b, s.nchunks, s.ct, scale_log2,
                                              m_part, l_part, m_row, il_row,
                                              wsp<float>(ws, L.k_bar), wsp<float>(ws, L.a_v),
                                              wsp<float>(ws, L.as_part));
  slash_combine<<<dim3((s.n + 255) / 256, s.H), 256, 0, st>>>(s.n, s.nt, 1.0f / (float)s.b,
                                                              wsp<float>(ws, L.as_part),
                                                              wsp<float>(ws, L.a_s));
  block_sums<<<dim3(s.nb, s.H), 128, 0, st>>>(s.n, s.nb, s.b, wsp<float>(ws, L.a_v),
                                              wsp<float>(ws, L.a_s), wsp<float>(ws, L.a_hat),
                                              wsp<float>(ws, L.As));
  const size_t psm = (128 + (size_t)s.nb + 33) * 4;
  pattern_kernel<<<s.H, kPatThreads, psm, st>>>(
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
