// fp_attn.cu -- stage (iii) of FlexPrefill: y = A(Q, K, V, S) (P:66-83,
// P:287-288): causal block-sparse attention over the selected (q-block,
// k-block) pairs with online softmax and GQA, on tcgen05 tensor cores.
//
// One CTA per (head, query block) work item; warp-specialised:
//   warp 4  TMA producer   Q tile once, then K and V tiles of the row's key
//                          blocks (indices from the CSR) into separate 2-stage
//                          rings (K is released as soon as S is computed)
//   warp 5  MMA issuer     S_i = Q K_i^T into one of 3 TMEM S/P buffers, issued
//                          two tiles ahead; O += P_i V_i with P_i read from TMEM
//                          (tcgen05 "TS" form, A operand in tensor memory)
//   warps 0-3 softmax      one query row per thread: S row from TMEM, online
//                          softmax in the log2 domain with a lazy running max
//                          (O is rescaled in TMEM only when the max grows by
//                          more than 2^8), P (bf16) written back over S in TMEM,
//                          final O / l -> bf16 -> global
// The diagonal block gets the intra-block causal mask (j <= i). The dense
// causal kernel is the same template with the implicit list kb = 0..qb.
// Work order is KV-group-major (the K/V of one group, 64 MiB at 128k, stays
// in L2 while its heads run), query blocks descending within a group.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

namespace fp {

namespace {

constexpr int kAttnThreads = 224;       // 4 softmax warps, K producer, MMA, V producer
constexpr int kKV = 3;                   // K and V ring depths
constexpr int kSBuf = 3;                 // S/P buffers in TMEM (128 columns each)
constexpr float kRescaleThresh = 8.0f;   // lazy rescale: tolerate P up to 2^8

struct AttnSmem {
  uint8_t q[kTileBytes];
  uint8_t k[kKV][kTileBytes];
  uint8_t v[kKV][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kKV], k_empty[kKV];
  uint64_t v_full[kKV], v_empty[kKV];
  uint64_t s_full[kSBuf], p_full[kSBuf], pv_done[kSBuf];
  uint32_t tmem_base;
};

// D[tmem] (+)= A[tmem] * B[smem]   (A = P, 128 rows x 16 keys, bf16 pairs per column)
FP_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <bool DENSE>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o, int H,
                int G, int n, int nb, long long cap, const int32_t* __restrict__ row_ptr,
                const int32_t* __restrict__ col_idx, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  AttnSmem& sm = *reinterpret_cast<AttnSmem*>(sbase);

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

  if (wid == 5) tmem_alloc(&sm.tmem_base, 512);
  if (tid == 128) {  // warp 4 lane 0
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
    for (int b = 0; b < kSBuf; ++b) {
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
  const uint32_t tO = tbase + 384;

  if (wid == 4 || wid == 6) {
    // ------------------------------------------------ TMA producers (K: warp 4, V: warp 6)
    if (lane_id() == 0) {
      const bool isK = (wid == 4);
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
  } else if (wid == 5) {
    // ------------------------------------------------ MMA issuer
    if (lane_id() == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
      const uint32_t qa = smem_u32(sm.q);
      auto issue_s = [&](int i) {
        const int s = i % kKV, b = i % kSBuf;
        mbar_wait(&sm.k_full[s], (i / kKV) & 1);
        // buffer b was last used by tile i-3: its P must have been consumed
        if (i >= kSBuf) mbar_wait(&sm.pv_done[b], ((i - kSBuf) / kSBuf) & 1);
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
        const int s = i % kKV, b = i % kSBuf;
        mbar_wait(&sm.v_full[s], (i / kKV) & 1);
        mbar_wait(&sm.p_full[b], (i / kSBuf) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(sm.v[s]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts(tO, tbase + b * 128 + kk * 8, sdesc_mnmajor(va, kk), idesc_o, (i > 0 || kk > 0));
        umma_commit(&sm.pv_done[b]);
        umma_commit(&sm.v_empty[s]);
        if (i + 2 < nk) issue_s(i + 2);
      }
    }
  } else {
    // ------------------------------------------------ softmax warpgroup
    const int r = tid;  // query row within the block == TMEM lane
    const uint32_t lane_off = (uint32_t)(wid * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    for (int i = 0; i < nk; ++i) {
      const int b = i % kSBuf;
      const int kb = DENSE ? i : __ldg(list + i);
      const uint32_t tS = tbase + b * 128 + lane_off;
      mbar_wait(&sm.s_full[b], (i / kSBuf) & 1);
      tc_fence_after();
      uint32_t v[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, v + c * 32);
      tmem_wait_ld();
      if (kb == qb) {  // intra-block causal mask on the diagonal block
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > r) v[c] = __float_as_uint(-INFINITY);
      }
      // row max with 8 independent accumulators (raw logits; scale > 0)
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = __uint_as_float(v[u]);
#pragma unroll
      for (int c = 8; c < 128; c += 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = fmaxf(mx8[u], __uint_as_float(v[c + u]));
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * scale_log2;
      // lazy running max: move it only when it grows by more than 2^kRescaleThresh
      float alpha = 1.0f;
      const bool move = mx > m_used + kRescaleThresh;
      if (move) {
        alpha = exp2f(m_used - mx);  // 0 on the first tile
        m_used = mx;
      }
      const float neg = -m_used;
      float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      uint32_t pk[64];
#pragma unroll
      for (int c = 0; c < 128; c += 2) {
        const float p0 = fast_exp2(fmaf(__uint_as_float(v[c]), scale_log2, neg));
        const float p1 = fast_exp2(fmaf(__uint_as_float(v[c + 1]), scale_log2, neg));
        rs8[(c >> 1) & 7] += p0 + p1;
        pk[c >> 1] = pack_bf16x2(p0, p1);
      }
      const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
      l = l * alpha + rs;
      if (i > 0 && __any_sync(0xffffffffu, move)) {
        // O holds sum_{t<i} P_t V_t: wait for PV_{i-1} and rescale this warp's rows
        mbar_wait(&sm.pv_done[(i - 1) % kSBuf], ((i - 1) / kSBuf) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t ov[32];
          tmem_ld32(tO + lane_off + c * 32, ov);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
          tmem_st32(tO + lane_off + c * 32, ov);
        }
      }
      // P (bf16 pairs) over the first 64 columns of this S buffer
      tmem_st32(tS, pk);
      tmem_st32(tS + 32, pk + 32);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm.p_full[b]);
    }
    // epilogue: O / l -> bf16
    mbar_wait(&sm.pv_done[(nk - 1) % kSBuf], ((nk - 1) / kSBuf) & 1);
    tc_fence_after();
    const float inv_l = 1.0f / l;
    uint4* dst = reinterpret_cast<uint4*>(o + ((size_t)h * n + (size_t)qb * 128 + r) * 128);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t ov[32];
      tmem_ld32(tO + lane_off + c * 32, ov);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; e += 8) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(ov[e]) * inv_l, __uint_as_float(ov[e + 1]) * inv_l);
        w.y = pack_bf16x2(__uint_as_float(ov[e + 2]) * inv_l, __uint_as_float(ov[e + 3]) * inv_l);
        w.z = pack_bf16x2(__uint_as_float(ov[e + 4]) * inv_l, __uint_as_float(ov[e + 5]) * inv_l);
        w.w = pack_bf16x2(__uint_as_float(ov[e + 6]) * inv_l, __uint_as_float(ov[e + 7]) * inv_l);
        dst[(c * 32 + e) / 8] = w;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 5) tmem_dealloc(tbase, 512);
}

}  // namespace

size_t attn_smem_bytes() { return sizeof(AttnSmem) + 1024; }

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
