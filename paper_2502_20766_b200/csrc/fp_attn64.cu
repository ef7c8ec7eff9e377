// fp_attn64.cu -- stage (iii) of FlexPrefill, y = A(Q, K, V, S) (P:66-83,
// P:287-288), for block_size b = 64 (the paper's Triton block-size ablation,
// "different block sizes can be flexibly selected according to
// different hardware"; next row f3).
//
// On B200 the natural tile is 128 x 128 (M = 128 tcgen05.mma; N = 64 MMAs run
// at ~44 instead of 32 cycles, profiles/r01_ubench_tcgen05.txt). A 64-block
// CSR is therefore computed on COARSE 128 x 128 tiles: the CTA of coarse row J
// owns query blocks 2J (tile rows 0-63, "A") and 2J+1 (rows 64-127, "B") -- one
// contiguous 128-row Q tile -- and walks the union of the two rows' sorted
// 64-block lists by coarse key tile m = kb / 2. Each coarse entry carries a
// 4-bit mask, bit 2x + y = "query block 2J+x selected key block 2m+y"; the
// softmax sets every unselected quadrant to -inf, and the coarse diagonal
// tile (m == J) also takes the element causal mask key <= query (its (0,1)
// quadrant is above the diagonal and never selected). So exactly the selected
// 64 x 64 blocks contribute (the results are those of the b = 64 CSR; parity
// against the b = 64 oracle in tests/test_gpu_block64.py); quadrants computed
// but masked are the price of the 128-wide tensor-core tile.
//
// Pipeline: v5's (fp_attn.cu) -- K / V producers (warps 8, 10) over the coarse
// union entries, MMA issuer (warp 9) with Q copied once into TMEM, 2 S/P
// buffers with S issued two entries ahead, 8 softmax warps on the 16x256b TMEM
// shape (2 rows x 32 columns per thread, quad-shuffle row reductions), lazy
// running max, P over S, O / l in the epilogue.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

namespace fp {

namespace {

constexpr int kThreads64 = 384;
constexpr int kKV64 = 3;
constexpr uint32_t kColO64 = 256, kColQ64 = 384;
constexpr float kRescale64 = 8.0f;

struct Attn64Smem {
  uint8_t q[kTileBytes];
  uint8_t k[kKV64][kTileBytes];
  uint8_t v[kKV64][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kKV64], k_empty[kKV64];
  uint64_t v_full[kKV64], v_empty[kKV64];
  uint64_t s_full[2], p_full[2], pv_done[2];
  uint32_t tmem_base;
};

FP_DEV float fmax3_64(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
FP_DEV float quad_max64(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
FP_DEV float quad_sum64(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// 8 k-steps of an M=128 x N=128 MMA in one asm statement, A from TMEM columns
// a0 + 8 kk, B descriptors b0 + off(kk) (16-B units). Executed by the whole
// issuing warp (warp-uniform operands); one elected lane issues.
template <uint32_t O1, uint32_t O2, uint32_t O3, uint32_t O4, uint32_t O5, uint32_t O6, uint32_t O7>
FP_DEV void umma_ts_chain8_64(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q, ep;\n\tsetp.ne.b32 p, 1, 0;\n\tsetp.ne.b32 q, %18, 0;\n\t"
      "elect.sync _|ep, 0xffffffff;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %9, %17, q;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %10, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %11, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %12, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %13, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %14, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %15, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %16, %17, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "r"(a0 + 32), "r"(a0 + 40), "r"(a0 + 48),
      "r"(a0 + 56), "l"(b0), "l"(b0 + O1), "l"(b0 + O2), "l"(b0 + O3), "l"(b0 + O4), "l"(b0 + O5),
      "l"(b0 + O6), "l"(b0 + O7), "r"(idesc), "r"(acc0));
}
#define FP64_KMAJ_OFFS 2, 4, 6, 1024, 1026, 1028, 1030
#define FP64_MNMAJ_OFFS 128, 256, 384, 512, 640, 768, 896

// Union of the two 64-block rows (2J -> bits 0/1, 2J+1 -> bits 2/3) by coarse
// 128-key tile m = kb >> 1, ascending.
struct CoarseIter {
  const int32_t* la;
  const int32_t* lb;
  int na, nb_, ia, ib;
  FP_DEV bool done() const { return ia >= na && ib >= nb_; }
  FP_DEV int next(int& mask) {
    const int ka = ia < na ? (__ldg(la + ia) >> 1) : 0x7fffffff;
    const int kb = ib < nb_ ? (__ldg(lb + ib) >> 1) : 0x7fffffff;
    const int m = min(ka, kb);
    mask = 0;
    while (ia < na) {
      const int x = __ldg(la + ia);
      if ((x >> 1) != m) break;
      mask |= 1 << (x & 1);
      ++ia;
    }
    while (ib < nb_) {
      const int x = __ldg(lb + ib);
      if ((x >> 1) != m) break;
      mask |= 4 << (x & 1);
      ++ib;
    }
    return m;
  }
};

// One coarse tile for one softmax thread: rows R0, R0 + 8 of its 16-lane
// group, columns 8k + 2a, 8k + 2a + 1 (16x256b register order). Unselected
// quadrants -> -inf; on the coarse diagonal also key > query -> -inf.
FP_DEV void softmax_tile64(float* v, int R0, int a, int mask, bool diag, float scale_log2,
                           float* m_used, float* alpha, float* rs) {
  const int x0 = R0 >> 6, x1 = (R0 + 8) >> 6;  // row halves of the two rows
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c0 = 8 * k + 2 * a;
    const int y = c0 >> 6;  // both columns of the pair are in the same key half
    const bool q0 = (mask >> (2 * x0 + y)) & 1, q1 = (mask >> (2 * x1 + y)) & 1;
    if (!q0 || (diag && c0 > R0)) v[4 * k] = -INFINITY;
    if (!q0 || (diag && c0 + 1 > R0)) v[4 * k + 1] = -INFINITY;
    if (!q1 || (diag && c0 > R0 + 8)) v[4 * k + 2] = -INFINITY;
    if (!q1 || (diag && c0 + 1 > R0 + 8)) v[4 * k + 3] = -INFINITY;
  }
  float p0 = fmax3_64(v[0], v[1], v[4]), p1 = fmax3_64(v[5], v[8], v[9]);
  float q0 = fmax3_64(v[2], v[3], v[6]), q1 = fmax3_64(v[7], v[10], v[11]);
#pragma unroll
  for (int k = 3; k < 16; k += 2) {
    p0 = fmax3_64(p0, v[4 * k], v[4 * k + 1]);
    q0 = fmax3_64(q0, v[4 * k + 2], v[4 * k + 3]);
    if (k + 1 < 16) {
      p1 = fmax3_64(p1, v[4 * k + 4], v[4 * k + 5]);
      q1 = fmax3_64(q1, v[4 * k + 6], v[4 * k + 7]);
    }
  }
  const float mx0 = quad_max64(fmaxf(p0, p1)) * scale_log2;
  const float mx1 = quad_max64(fmaxf(q0, q1)) * scale_log2;
  alpha[0] = 1.f;
  alpha[1] = 1.f;
  if (mx0 > m_used[0] + kRescale64) {
    alpha[0] = exp2f(m_used[0] - mx0);
    m_used[0] = mx0;
  }
  if (mx1 > m_used[1] + kRescale64) {
    alpha[1] = exp2f(m_used[1] - mx1);
    m_used[1] = mx1;
  }
  // a row with no visible key so far (m_used = -inf) gets P = 2^-inf = 0
  const float n0 = (m_used[0] == -INFINITY) ? 0.f : -m_used[0];
  const float n1 = (m_used[1] == -INFINITY) ? 0.f : -m_used[1];
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    v[4 * k] = fast_exp2(fmaf(v[4 * k], scale_log2, n0));
    v[4 * k + 1] = fast_exp2(fmaf(v[4 * k + 1], scale_log2, n0));
    v[4 * k + 2] = fast_exp2(fmaf(v[4 * k + 2], scale_log2, n1));
    v[4 * k + 3] = fast_exp2(fmaf(v[4 * k + 3], scale_log2, n1));
    s0 += v[4 * k] + v[4 * k + 1];
    s1 += v[4 * k + 2] + v[4 * k + 3];
  }
  rs[0] = s0;
  rs[1] = s1;
}

__global__ void __launch_bounds__(kThreads64, 1)
    attn64_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                  const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o,
                  const TLayout ol, int Hp, int Gp, int H, int G, int n, int nb, int nt, long long cap,
                  const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                  float scale_log2) {
  FP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();
  Attn64Smem& sm = *reinterpret_cast<Attn64Smem*>(smem_raw);

  const int tid = threadIdx.x;
  const int wid = warp_id();
  // work item: KV-group-major, coarse rows descending, heads of the group interleaved
  const int gsz = H / G;
  const int per_group = gsz * nt;
  const int g = blockIdx.x / per_group;
  const int rem = blockIdx.x - g * per_group;
  const int J = nt - 1 - rem / gsz;
  const int h = g * gsz + rem % gsz;
  const int qa = 2 * J, qbb = 2 * J + 1;  // the tile's two 64-row query blocks
  const int32_t* rp = row_ptr + (size_t)h * (nb + 1);
  const int bA = rp[qa];
  const int nA = rp[qa + 1] - bA;
  const int nB = qbb < nb ? rp[qbb + 1] - rp[qbb] : 0;
  const int32_t* la = col_idx + (size_t)h * cap + bA;
  const int32_t* lb = la + nA;  // row 2J+1 follows row 2J in the head's CSR

  if (wid == 9) tmem_alloc(&sm.tmem_base, 512);
  if (tid == 256) {
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kKV64; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.s_full[b], 1);
      mbar_init(&sm.p_full[b], 256);
      mbar_init(&sm.pv_done[b], 1);
    }
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  if (wid >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (wid == 8 || wid == 10) {
      // ------------------------------------------------ TMA producers (K: warp 8, V: warp 10)
      if (lane_id() == 0) {
        const bool isK = (wid == 8);
        const uint64_t pol = policy_evict_last();
        if (isK) {
          mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
          tma_tile(sm.q, &qmap, &sm.q_full, J * 128, h, Hp);
        }
        uint64_t* full = isK ? sm.k_full : sm.v_full;
        uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
        const CUtensorMap* map = isK ? &kmap : &vmap;
        CoarseIter it{la, lb, nA, nB, 0, 0};
        int e = 0;
        for (; !it.done(); ++e) {
          int mask;
          const int m = it.next(mask);
          const int s = e % kKV64;
          if (e >= kKV64) mbar_wait(&empty[s], ((e - kKV64) / kKV64) & 1);
          mbar_arrive_expect_tx(&full[s], kTileBytes);
          tma_tile_hint(isK ? sm.k[s] : sm.v[s], map, &full[s], m * 128, g, Gp, pol);
        }
        for (int d = max(0, e - kKV64); d < e; ++d) mbar_wait(&empty[d % kKV64], (d / kKV64) & 1);
      }
    } else if (wid == 9) {
      // ------------------------------------------------ MMA issuer (whole warp,
      // elect.sync-predicated MMA / commit / copy, as fp_attn8.cu)
      {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
        const uint32_t qs = smem_u32(sm.q);
        CoarseIter it{la, lb, nA, nB, 0, 0};
        int ne = 0;  // entries whose S has been issued
        auto issue_s = [&]() {
          int mask;
          it.next(mask);
          const int i = ne++;
          const int s = i % kKV64, b = i & 1;
          mbar_wait(&sm.k_full[s], (i / kKV64) & 1);
          tc_fence_after();
          umma_ts_chain8_64<FP64_KMAJ_OFFS>(tbase + b * 128, tbase + kColQ64,
                                            sdesc_kmajor(smem_u32(sm.k[s]), 0), idesc_s, 0);
          umma_commit_elect(&sm.s_full[b]);
          umma_commit_elect(&sm.k_empty[s]);
        };
        mbar_wait(&sm.q_full, 0);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // Q -> TMEM columns kColQ64 + 8 kk
          asm volatile("{\n\t.reg .pred ep;\n\telect.sync _|ep, 0xffffffff;\n\t"
                       "@ep tcgen05.cp.cta_group::1.128x256b [%0], %1;\n\t}" ::"r"(tbase + kColQ64 + kk * 8),
                       "l"(sdesc_kmajor(qs, kk)));
        issue_s();
        if (!it.done()) issue_s();
        for (int i = 0; i < ne; ++i) {
          const int s = i % kKV64, b = i & 1;
          mbar_wait(&sm.v_full[s], (i / kKV64) & 1);
          mbar_wait(&sm.p_full[b], (i >> 1) & 1);
          tc_fence_after();
          umma_ts_chain8_64<FP64_MNMAJ_OFFS>(tbase + kColO64, tbase + b * 128,
                                             sdesc_mnmajor(smem_u32(sm.v[s]), 0), idesc_o, i > 0);
          umma_commit_elect(&sm.pv_done[b]);
          umma_commit_elect(&sm.v_empty[s]);
          if (!it.done()) issue_s();
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ------------------------------------------------ softmax warps 0-7 (v5 layout)
    const int lbase = (wid & 3) * 32 + (wid >> 2) * 16;
    const int a = lane_id() & 3;
    const int R0 = lbase + (lane_id() >> 2);
    const uint32_t lane_off = (uint32_t)lbase << 16;
    const uint32_t tO = tbase + kColO64 + lane_off;
    float m_used[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    CoarseIter it{la, lb, nA, nB, 0, 0};
    int i = 0;
    for (; !it.done(); ++i) {
      int mask;
      const int m = it.next(mask);
      const int b = i & 1;
      const uint32_t tS = tbase + b * 128 + lane_off;
      mbar_wait(&sm.s_full[b], (i >> 1) & 1);
      tc_fence_after();
      float v[64];
      tmem_ld_16x256b_x16(tS, reinterpret_cast<uint32_t*>(v));
      tmem_wait_ld();
      float alpha[2], rs[2];
      softmax_tile64(v, R0, a, mask, m == J, scale_log2, m_used, alpha, rs);
      l[0] = l[0] * alpha[0] + rs[0];
      l[1] = l[1] * alpha[1] + rs[1];
      if (i > 0) mbar_wait(&sm.pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
      if (i > 0 && __any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
        tc_fence_after();
        float ov[64];
        tmem_ld_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          ov[4 * k] *= alpha[0];
          ov[4 * k + 1] *= alpha[0];
          ov[4 * k + 2] *= alpha[1];
          ov[4 * k + 3] *= alpha[1];
        }
        tmem_st_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
      }
      uint32_t pk[32];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        pk[2 * k] = pack_bf16x2(v[4 * k], v[4 * k + 1]);
        pk[2 * k + 1] = pack_bf16x2(v[4 * k + 2], v[4 * k + 3]);
      }
      tmem_st_16x128b_x16(tS, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm.p_full[b]);
    }
    // epilogue: O / l -> bf16 -> global; rows past n (and the B half when
    // block 2J+1 does not exist) are not stored
    const float il0 = 1.0f / quad_sum64(l[0]), il1 = 1.0f / quad_sum64(l[1]);
    mbar_wait(&sm.pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
    tc_fence_after();
    float ov[64];
    tmem_ld_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
    tmem_wait_ld();
    const int row0 = J * 128 + R0;
    uint32_t* d0 = reinterpret_cast<uint32_t*>(o + toff(ol, h, row0)) + a;
    uint32_t* d1 = d0 + 4 * ol.rs;
    if (row0 < n) {
#pragma unroll
      for (int k = 0; k < 16; ++k) d0[4 * k] = pack_bf16x2(ov[4 * k] * il0, ov[4 * k + 1] * il0);
    }
    if (row0 + 8 < n) {
#pragma unroll
      for (int k = 0; k < 16; ++k) d1[4 * k] = pack_bf16x2(ov[4 * k + 2] * il1, ov[4 * k + 3] * il1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 9) tmem_dealloc(tbase, 512);
}

}  // namespace

cudaError_t launch_attn_b64(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                            const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                            const int32_t* row_ptr, const int32_t* col_idx, cudaStream_t st) {
  const size_t smem = sizeof(Attn64Smem);
  const cudaError_t ea = ensure_smem_attr((const void*)attn64_kernel, smem);
  if (ea != cudaSuccess) return ea;
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  const dim3 grid(s.H * s.nt);
  FP_LAUNCH(attn64_kernel, grid, kThreads64, smem, st, qmap, kmap, vmap, reinterpret_cast<__nv_bfloat16*>(o),
                                                lay.o, lay.q.per, lay.k.per, s.H, s.G, s.n, s.nb, s.nt,
                                                s.tri, row_ptr, col_idx, scale_log2);
  return cudaGetLastError();
}

}  // namespace fp
