// fp_attn.cu -- stage (iii) of FlexPrefill: y = A(Q, K, V, S) (P:66-83,
// P:287-288): causal block-sparse attention over the selected (q-block,
// k-block) pairs with online softmax and GQA, on tcgen05 tensor cores.
//
// One CTA per (head, query block) work item; warp-specialised:
//   warp 4  TMA producer   Q tile once, then K/V tiles of the row's key
//                          blocks (indices from the CSR) into a 2-stage ring
//   warp 5  MMA issuer     S_i = Q K_i^T into TMEM (double buffered, issued one
//                          tile ahead), O += P_i V_i into TMEM
//   warps 0-3 softmax      one query row per thread: S row from TMEM, online
//                          softmax in the log2 domain, O rescale in TMEM when
//                          the running max moves, P (bf16) to shared memory,
//                          final O / l -> bf16 -> global
// The diagonal block gets the intra-block causal mask (j <= i). The dense
// causal kernel is the same template with the implicit list kb = 0..qb.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

namespace fp {

namespace {

constexpr int kAttnThreads = 192;

struct AttnSmem {
  uint8_t q[kTileBytes];
  uint8_t k[2][kTileBytes];
  uint8_t v[2][kTileBytes];
  uint8_t p[kTileBytes];
  uint64_t q_full;
  uint64_t kv_full[2];
  uint64_t kv_empty[2];
  uint64_t s_full[2];
  uint64_t s_empty[2];
  uint64_t p_full;
  uint64_t pv_done;
  uint32_t tmem_base;
};

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
  // work item: query blocks in descending order, heads interleaved so that the
  // heads of one KV group run side by side (K/V reuse through L2)
  const int h = blockIdx.x % H;
  const int qb = nb - 1 - blockIdx.x / H;
  const int g = h / (H / G);
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
  if (tid == 128) {
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&sm.kv_full[s], 1);
      mbar_init(&sm.kv_empty[s], 1);
      mbar_init(&sm.s_full[s], 1);
      mbar_init(&sm.s_empty[s], 128);
    }
    mbar_init(&sm.p_full, 128);
    mbar_init(&sm.pv_done, 1);
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  const uint32_t tS[2] = {tbase, tbase + 128};
  const uint32_t tO = tbase + 256;

  if (wid == 4) {
    // ------------------------------------------------ TMA producer
    if (lane_id() == 0) {
      const uint64_t pol_kv = policy_evict_last();
      mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
      tma_load_tile(sm.q, &qmap, &sm.q_full, h * n + qb * 128);
      for (int i = 0; i < nk; ++i) {
        const int s = i & 1;
        if (i >= 2) mbar_wait(&sm.kv_empty[s], ((i - 2) >> 1) & 1);
        const int kb = DENSE ? i : __ldg(list + i);
        mbar_arrive_expect_tx(&sm.kv_full[s], 2 * kTileBytes);
        tma_load_tile_hint(sm.k[s], &kmap, &sm.kv_full[s], g * n + kb * 128, pol_kv);
        tma_load_tile_hint(sm.v[s], &vmap, &sm.kv_full[s], g * n + kb * 128, pol_kv);
      }
    }
  } else if (wid == 5) {
    // ------------------------------------------------ MMA issuer
    if (lane_id() == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
      const uint32_t qa = smem_u32(sm.q), pa = smem_u32(sm.p);
      auto issue_s = [&](int i) {
        const int s = i & 1;
        mbar_wait(&sm.kv_full[s], (i >> 1) & 1);
        if (i >= 2) mbar_wait(&sm.s_empty[s], ((i - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sm.k[s]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ss(tS[s], sdesc_kmajor(qa, kk), sdesc_kmajor(ka, kk), idesc_s, kk > 0);
        umma_commit(&sm.s_full[s]);
      };
      mbar_wait(&sm.q_full, 0);
      issue_s(0);
      for (int i = 0; i < nk; ++i) {
        if (i + 1 < nk) issue_s(i + 1);
        mbar_wait(&sm.p_full, i & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(sm.v[i & 1]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ss(tO, sdesc_kmajor(pa, kk), sdesc_mnmajor(va, kk), idesc_o, (i > 0 || kk > 0));
        umma_commit(&sm.pv_done);
        umma_commit(&sm.kv_empty[i & 1]);
      }
    }
  } else {
    // ------------------------------------------------ softmax warpgroup
    const int r = tid;  // query row within the block == TMEM lane
    const uint32_t lane_off = (uint32_t)(wid * 32) << 16;
    float m = -INFINITY, l = 0.f;
    uint32_t v[128];
    for (int i = 0; i < nk; ++i) {
      const int s = i & 1;
      const int kb = DENSE ? i : __ldg(list + i);
      mbar_wait(&sm.s_full[s], (i >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS[s] + lane_off + c * 32, v + c * 32);
      tmem_wait_ld();
      const bool diag = (kb == qb);
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        float x = __uint_as_float(v[c]) * scale_log2;
        if (diag && c > r) x = -INFINITY;
        v[c] = __float_as_uint(x);
        mx = fmaxf(mx, x);
      }
      tc_fence_before();
      mbar_arrive(&sm.s_empty[s]);
      const float m_new = fmaxf(m, mx);
      const float alpha = exp2f(m - m_new);
      float rs = 0.f;
      uint32_t pk[64];
#pragma unroll
      for (int c = 0; c < 128; c += 2) {
        const float p0 = fast_exp2(__uint_as_float(v[c]) - m_new);
        const float p1 = fast_exp2(__uint_as_float(v[c + 1]) - m_new);
        rs += p0 + p1;
        pk[c >> 1] = pack_bf16x2(p0, p1);
      }
      l = l * alpha + rs;
      m = m_new;
      if (i > 0) {
        // PV_{i-1} done: P buffer is free and O is current
        mbar_wait(&sm.pv_done, (i - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t ov[32];
            tmem_ld32(tO + lane_off + c * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
            tmem_st32(tO + lane_off + c * 32, ov);
          }
          tmem_wait_st();
        }
      }
      // P row -> shared memory (K-major SW128 tile, the A operand of P.V)
#pragma unroll
      for (int ch = 0; ch < 16; ++ch) {
        const uint32_t off = sw128_offset(r, ch * 8);
        *reinterpret_cast<uint4*>(sm.p + off) =
            make_uint4(pk[ch * 4], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&sm.p_full);
    }
    // epilogue: O / l -> bf16
    mbar_wait(&sm.pv_done, (nk - 1) & 1);
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
