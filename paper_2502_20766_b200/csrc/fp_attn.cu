// fp_attn.cu -- stage (iii) of FlexPrefill: y = A(Q, K, V, S) (P:66-83,
// P:287-288): causal block-sparse attention over the selected (q-block,
// k-block) pairs with online softmax and GQA, on tcgen05 tensor cores.
//
// One CTA per (head, query block) work item, warp-specialised (384 threads;
// registers rebalanced with setmaxnreg: 224 per softmax thread, 56 otherwise):
//   warp 8   K producer    Q tile once, then the K tiles of the row's key blocks
//                          (indices from the CSR) into a 3-stage TMA ring
//   warp 10  V producer    the V tiles into their own 3-stage ring
//   warp 9   MMA issuer    S_i = Q K_i^T into TMEM buffer (i & 1), issued two
//                          tiles ahead; O_(i&1) += P_i V_i with P_i read from
//                          TMEM (tcgen05 "TS" form, A operand in tensor memory)
//   warps 0-3 / 4-7        two softmax warpgroups that ping-pong over the key
//                          tiles: warpgroup w owns tiles i = w, w+2, ..., its
//                          S/P buffer, its O accumulator and its own running
//                          (max, sum); one query row per thread. While one
//                          warpgroup exponentiates, the tensor core works for
//                          the other. The running max is lazy (O_w is rescaled
//                          only when the max grows by more than 2^8); the two
//                          partial softmaxes are merged once, in the epilogue.
// TMEM (512 columns): S/P buffers 0 and 1 (128 each), O_0, O_1 (128 each).
// Reusing an S/P buffer for S_(i+2) right after issuing PV_i relies on the
// in-order execution of one thread's tcgen05.mma stream (WAR on the P
// columns); a commit that follows S_i also guarantees PV_(i-2) is complete,
// which is what makes the O_w rescale safe without another barrier.
// A part of the exponentials runs on the FMA pipe (polynomial exp2) to keep
// the MUFU pipe below the tensor-core time. The diagonal block gets the
// intra-block causal mask (j <= i) in a separate code path. The dense causal
// kernel is the same template with the implicit list kb = 0..qb.
// Work order is KV-group-major (the K/V of one group, 64 MiB at 128k, stays
// in L2 while its heads run), query blocks descending within a group.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

#ifdef FP_TIMING
__device__ unsigned long long g_attn_timing[16];
#define FP_TMARK(k) do { if (timing_on) { long long _t = clock64(); tacc[k] += _t - tlast; tlast = _t; } } while (0)
#else
#define FP_TMARK(k) do { } while (0)
#endif

namespace fp {

namespace {

constexpr int kAttnThreads = 384;      // 8 softmax warps, K producer (8), MMA (9), V producer (10), spare (11)
#ifndef FP_EMU
#define FP_EMU 32
#endif
constexpr int kEmu = FP_EMU;           // exponentials per row (of 128) done on the FMA pipe
constexpr int kKV = 3;                 // K and V ring depths
constexpr float kRescaleThresh = 8.0f; // lazy rescale: tolerate P up to 2^8

struct AttnSmem {
  uint8_t q[kTileBytes];
  uint8_t k[kKV][kTileBytes];
  uint8_t v[kKV][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kKV], k_empty[kKV];
  uint64_t v_full[kKV], v_empty[kKV];
  uint64_t s_full[2], p_full[2], pv_done[2];
  uint32_t tmem_base;
  float ml[2][2][128];  // epilogue exchange: (max, sum) per warpgroup and row
};

FP_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
FP_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// (d0, d1) = (a0, a1) * (b0, b1) + (c0, c1) on the paired FMA pipe (FFMA2)
FP_DEV void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
FP_DEV void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// 2^x for a pair on the FMA/ALU pipes: x = j + f (j = rint(x), |f| <= 1/2),
// 2^f by a degree-3 minimax polynomial (max rel. error 7.5e-5; P is rounded to
// bf16 afterwards, 2^-9), 2^j added into the exponent field. x is clamped at
// -125 (the result is then < 2^-124, i.e. 0 for the bf16 P and the row sum).
FP_DEV void exp2_emu2(float x0, float x1, float& y0, float& y1) {
  const float kMagic = 12582912.0f;  // 1.5 * 2^23: rounds to an integer in the low mantissa bits
  x0 = fmaxf(x0, -125.0f);
  x1 = fmaxf(x1, -125.0f);
  float t0, t1, j0, j1, f0, f1, p0, p1;
  fadd2(t0, t1, x0, x1, kMagic, kMagic);
  fadd2(j0, j1, t0, t1, -kMagic, -kMagic);
  fadd2(f0, f1, x0, x1, -j0, -j1);
  ffma2(p0, p1, f0, f1, 0.0551716626f, 0.0551716626f, 0.242611155f, 0.242611155f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.69326099f, 0.69326099f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.999928072f, 0.999928072f);
  y0 = __uint_as_float(__float_as_uint(t0) * 8388608u + __float_as_uint(p0));
  y1 = __uint_as_float(__float_as_uint(t1) * 8388608u + __float_as_uint(p1));
}

// D[tmem] (+)= A[tmem] * B[smem]   (A = P, 128 rows x 16 keys, bf16 pairs per column)
FP_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// One key tile of one softmax warpgroup: S row (128 fp32) from TMEM -> lazy
// running max -> P = 2^(s - m) (bf16) written over the S columns. Returns the
// row sum of P; updates m_used and sets alpha (scale for the previous O / l).
#ifdef FP_TIMING
#define FP_TARGS , bool timing_on, long long* tacc, long long& tlast
#define FP_TPASS , timing_on, tacc, tlast
#else
#define FP_TARGS
#define FP_TPASS
#endif
template <bool DIAG>
FP_DEV float softmax_tile(uint32_t tS, uint32_t tO, int r, float scale_log2, float& m_used,
                          float& alpha, bool o_live FP_TARGS) {
  float v[128];
#pragma unroll
  for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, reinterpret_cast<uint32_t*>(v) + c * 32);
  tmem_wait_ld();
  FP_TMARK(1);
  if (DIAG) {
#pragma unroll
    for (int c = 0; c < 128; ++c)
      if (c > r) v[c] = -INFINITY;
  }
  // row max on the raw logits (scale > 0): 8 independent 3-input-max chains
  float acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = fmax3(v[u], v[u + 8], v[u + 16]);
#pragma unroll
  for (int c = 24; c < 120; c += 16)
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = fmax3(acc[u], v[c + u], v[c + 8 + u]);
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = fmaxf(acc[u], v[120 + u]);
  const float mx = fmax3(fmax3(acc[0], acc[1], acc[2]), fmax3(acc[3], acc[4], acc[5]),
                         fmaxf(acc[6], acc[7])) * scale_log2;
  // lazy running max: move it only when it grows by more than 2^kRescaleThresh
  alpha = 1.0f;
  const bool move = mx > m_used + kRescaleThresh;
  if (move) {
    alpha = exp2f(m_used - mx);  // 0 on the first tile
    m_used = mx;
  }
  FP_TMARK(2);
  if (o_live && __any_sync(0xffffffffu, move)) {
    // O_w = sum over this warpgroup's earlier tiles; the PV that wrote it last
    // completed before S of this tile (in-order tcgen05 stream + commit).
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld32(tO + c * 32, ov);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
      tmem_st32(tO + c * 32, ov);
    }
  }
  FP_TMARK(4);
  const float neg = -m_used;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  // 4 chunks of 32 columns: scale, exponentiate (MUFU / FMA pipe), sum, pack, store P
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    float* x = v + ch * 32;
#pragma unroll
    for (int c = 0; c < 32; c += 2) ffma2(x[c], x[c + 1], x[c], x[c + 1], scale_log2, scale_log2, neg, neg);
    constexpr int kEmuCh = kEmu / 4;  // emulated columns in each 32-column chunk
#pragma unroll
    for (int c = 0; c < 32 - kEmuCh; ++c) x[c] = fast_exp2(x[c]);
#pragma unroll
    for (int c = 32 - kEmuCh; c < 32; c += 2) exp2_emu2(x[c], x[c + 1], x[c], x[c + 1]);
    if (DIAG) {
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (ch * 32 + c > r) x[c] = 0.f;
    }
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
      fadd2(s0, s1, s0, s1, x[c], x[c + 1]);
      fadd2(s2, s3, s2, s3, x[c + 2], x[c + 3]);
      pk[c >> 1] = pack_bf16x2(x[c], x[c + 1]);
      pk[(c >> 1) + 1] = pack_bf16x2(x[c + 2], x[c + 3]);
    }
    tmem_st16(tS + ch * 16, pk);  // P columns overwrite S columns already in registers
  }
  return (s0 + s1) + (s2 + s3);
}

template <bool DENSE>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o, int H,
                int G, int n, int nb, long long cap, const int32_t* __restrict__ row_ptr,
                const int32_t* __restrict__ col_idx, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the 7 SW128 tiles fill 224 KiB: no room for alignment slack. The dynamic
  // shared memory window starts 1024-B aligned when the kernel has no static
  // shared memory; trap (fail loudly) if that ever stops holding.
  if (smem_u32(smem_raw) & 1023u) __trap();
  AttnSmem& sm = *reinterpret_cast<AttnSmem*>(smem_raw);

  const int tid = threadIdx.x;
  const int wid = warp_id();
  // work item (KV-group-major, q-blocks descending, heads of the group interleaved)
  const int gsz = H / G;
  const int per_group = gsz * nb;
  const int g = blockIdx.x / per_group;
  const int rem = blockIdx.x - g * per_group;
  const int qb = nb - 1 - rem / gsz;
  const int h = g * gsz + rem % gsz;
  int nk;
  const int32_t* list = nullptr;
  if (DENSE) {
    nk = qb + 1;
  } else {
    const int32_t* rp = row_ptr + (size_t)h * (nb + 1);
    const int beg = rp[qb];
    nk = rp[qb + 1] - beg;
    list = col_idx + (size_t)h * cap + beg;
  }

  if (wid == 9) tmem_alloc(&sm.tmem_base, 512);
  if (tid == 256) {  // warp 8 lane 0
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kKV; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.s_full[b], 1);
      mbar_init(&sm.p_full[b], 128);
      mbar_init(&sm.pv_done[b], 1);
    }
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  if (wid >= 8) {
  // producer / MMA warpgroup (warps 8-11) gives registers to the softmax warpgroups
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (wid == 8 || wid == 10) {
    // ------------------------------------------------ TMA producers (K: warp 8, V: warp 10)
    if (lane_id() == 0) {
      const bool isK = (wid == 8);
      const uint64_t pol_kv = policy_evict_last();
      if (isK) {
        mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
        tma_load_tile(sm.q, &qmap, &sm.q_full, h * n + qb * 128);
      }
      uint64_t* full = isK ? sm.k_full : sm.v_full;
      uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
      const CUtensorMap* map = isK ? &kmap : &vmap;
      for (int i = 0; i < nk; ++i) {
        const int s = i % kKV;
        const int kb = DENSE ? i : __ldg(list + i);
        if (i >= kKV) mbar_wait(&empty[s], ((i - kKV) / kKV) & 1);
        mbar_arrive_expect_tx(&full[s], kTileBytes);
        tma_load_tile_hint(isK ? sm.k[s] : sm.v[s], map, &full[s], g * n + kb * 128, pol_kv);
      }
    }
  } else if (wid == 9) {
    // ------------------------------------------------ MMA issuer
    if (lane_id() == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
      const uint32_t qa = smem_u32(sm.q);
      auto issue_s = [&](int i) {
        const int s = i % kKV, b = i & 1;
        mbar_wait(&sm.k_full[s], (i / kKV) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sm.k[s]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ss(tbase + b * 128, sdesc_kmajor(qa, kk), sdesc_kmajor(ka, kk), idesc_s, kk > 0);
        umma_commit(&sm.s_full[b]);
        umma_commit(&sm.k_empty[s]);
      };
      mbar_wait(&sm.q_full, 0);
      issue_s(0);
      if (nk > 1) issue_s(1);
      for (int i = 0; i < nk; ++i) {
        const int s = i % kKV, b = i & 1;
        mbar_wait(&sm.v_full[s], (i / kKV) & 1);
        mbar_wait(&sm.p_full[b], (i >> 1) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(sm.v[s]);
        const uint32_t tO = tbase + 256 + b * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts(tO, tbase + b * 128 + kk * 8, sdesc_mnmajor(va, kk), idesc_o, (i >= 2 || kk > 0));
        umma_commit(&sm.pv_done[b]);
        umma_commit(&sm.v_empty[s]);
        if (i + 2 < nk) issue_s(i + 2);  // same buffer b: in-order after PV_i
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ------------------------------------------------ softmax warpgroups
    const int w = wid >> 2;  // warpgroup: tiles i = w, w + 2, ...
    const int r = (wid & 3) * 32 + lane_id();  // query row within the block == TMEM lane
    const uint32_t lane_off = (uint32_t)((wid & 3) * 32) << 16;
    const uint32_t tS = tbase + w * 128 + lane_off;
    const uint32_t tO = tbase + 256 + w * 128 + lane_off;
    float m_used = -INFINITY, l = 0.f;
#ifdef FP_TIMING
    const bool timing_on = (tid == 0);
    long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
#endif
    for (int i = w; i < nk; i += 2) {
      const int kb = DENSE ? i : __ldg(list + i);
      FP_TMARK(7);
      mbar_wait(&sm.s_full[w], (i >> 1) & 1);
      tc_fence_after();
      FP_TMARK(0);
      float alpha;
      const float rs = (kb == qb)
                           ? softmax_tile<true>(tS, tO, r, scale_log2, m_used, alpha, i >= 2 FP_TPASS)
                           : softmax_tile<false>(tS, tO, r, scale_log2, m_used, alpha, i >= 2 FP_TPASS);
      l = l * alpha + rs;
      FP_TMARK(3);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm.p_full[w]);
      FP_TMARK(6);
    }
#ifdef FP_TIMING
    if (timing_on) {
      for (int k = 0; k < 8; ++k) atomicAdd(&g_attn_timing[k], (unsigned long long)tacc[k]);
      atomicAdd(&g_attn_timing[8], (unsigned long long)((nk + 1) / 2));
    }
#endif
    // epilogue: merge the two partial softmaxes, O = (a0 O_0 + a1 O_1) / (a0 l_0 + a1 l_1)
    const int n_mine = (nk - w + 1) / 2;  // tiles of this warpgroup
    if (n_mine > 0) {
      const int i_last = w + 2 * (n_mine - 1);
      mbar_wait(&sm.pv_done[w], (i_last >> 1) & 1);
    }
    sm.ml[w][0][r] = m_used;
    sm.ml[w][1][r] = l;
    named_bar_sync(1, 256);
    tc_fence_after();
    const float m0 = sm.ml[0][0][r], m1 = sm.ml[1][0][r];
    const float mm = fmaxf(m0, m1);
    const float a0 = exp2f(m0 - mm);
    const float a1 = (nk > 1) ? exp2f(m1 - mm) : 0.f;
    const float inv_l = 1.0f / (a0 * sm.ml[0][1][r] + a1 * sm.ml[1][1][r]);
    const float f0 = a0 * inv_l, f1 = a1 * inv_l;
    // this warpgroup writes output columns w*64 .. w*64+63
    const uint32_t tO0 = tbase + 256 + lane_off + w * 64, tO1 = tbase + 384 + lane_off + w * 64;
    uint4* dst = reinterpret_cast<uint4*>(o + ((size_t)h * n + (size_t)qb * 128 + r) * 128 + w * 64);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t o0[32], o1[32];
      tmem_ld32(tO0 + c * 32, o0);
      if (nk > 1) tmem_ld32(tO1 + c * 32, o1);
      tmem_wait_ld();
      float y[32];
#pragma unroll
      for (int e = 0; e < 32; ++e)
        y[e] = (nk > 1) ? fmaf(__uint_as_float(o0[e]), f0, __uint_as_float(o1[e]) * f1)
                        : __uint_as_float(o0[e]) * f0;
#pragma unroll
      for (int e = 0; e < 32; e += 8) {
        uint4 wv;
        wv.x = pack_bf16x2(y[e], y[e + 1]);
        wv.y = pack_bf16x2(y[e + 2], y[e + 3]);
        wv.z = pack_bf16x2(y[e + 4], y[e + 5]);
        wv.w = pack_bf16x2(y[e + 6], y[e + 7]);
        dst[(c * 32 + e) / 8] = wv;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 9) tmem_dealloc(tbase, 512);
}

}  // namespace

size_t attn_smem_bytes() { return sizeof(AttnSmem); }

cudaError_t launch_attn(const Shape& s, const WsLayout& L, void* ws, const CUtensorMap& qmap,
                        const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                        const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                        cudaStream_t st) {
  (void)L;
  (void)ws;
  static bool attr_done = false;
  const size_t smem = attn_smem_bytes();
  if (!attr_done) {
    cudaFuncSetAttribute(attn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(attn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  const dim3 grid(s.H * s.nb);
  if (dense)
    attn_kernel<true><<<grid, kAttnThreads, smem, st>>>(qmap, kmap, vmap,
                                                        reinterpret_cast<__nv_bfloat16*>(o), s.H,
                                                        s.G, s.n, s.nb, s.tri, row_ptr, col_idx,
                                                        scale_log2);
  else
    attn_kernel<false><<<grid, kAttnThreads, smem, st>>>(qmap, kmap, vmap,
                                                         reinterpret_cast<__nv_bfloat16*>(o), s.H,
                                                         s.G, s.n, s.nb, s.tri, row_ptr, col_idx,
                                                         scale_log2);
  return cudaGetLastError();
}

}  // namespace fp

#ifdef FP_TIMING
extern "C" int fp_debug_attn_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_attn_timing, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_attn_timing, z, sizeof(z));
  }
  return 0;
}
#endif
