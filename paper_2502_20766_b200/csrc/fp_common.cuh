// fp_common.cuh -- sm_100a building blocks shared by the FlexPrefill kernels:
// mbarriers, TMA tile loads, tcgen05 (UMMA) descriptors / MMA / TMEM access.
// Everything is inline PTX; no CUTLASS/CuTe types are used.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define FP_DEV __device__ __forceinline__

namespace fp {

// ----------------------------------------------------------- constants -----
constexpr int kBlock = 128;     // block_size
constexpr int kHeadDim = 128;   // d
constexpr int kTileBytes = kBlock * kHeadDim * 2;   // one 128x128 bf16 tile = 32 KiB
constexpr int kBoxBytes = kTileBytes / 2;            // one 128x64 TMA box (SW128) = 16 KiB
constexpr float kLog2e = 1.4426950408889634f;

// ------------------------------------------------------------- basics ------
// Programmatic dependent launch (every kernel of the library is launched with
// the PDL attribute, FP_LAUNCH in fp_internal.h): a kernel waits for the
// previous kernel of its stream to complete (and its memory to be visible)
// before touching anything, then lets the next one start launching, so the
// launch / ramp of kernel i+1 overlaps the tail of kernel i. Both are no-ops
// for a launch without the attribute.
#define FP_PDL_ENTRY()                                        \
  do {                                                        \
    asm volatile("griddepcontrol.wait;" ::: "memory");        \
    asm volatile("griddepcontrol.launch_dependents;" :::);    \
  } while (0)

FP_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

FP_DEV uint32_t warp_id() { return threadIdx.x >> 5; }
FP_DEV uint32_t lane_id() { return threadIdx.x & 31; }

FP_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------ mbarrier -----
FP_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
FP_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

FP_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
FP_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
FP_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking test of phase completion (for polling several barriers).
FP_DEV bool mbar_test(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for the phase with parity `parity` to complete. A wait that exceeds
// ~2^34 cycles (seconds) is a pipeline bug: trap instead of hanging the GPU.
FP_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try_wait(addr, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_wait(addr, parity)) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}

// ---------------------------------------------------------------- TMA ------
FP_DEV void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 2D tile load, coordinates (c0 = inner/column, c1 = row), completes on `bar`.
FP_DEV void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 2D tile load with an L2 cache-policy hint (createpolicy result).
FP_DEV void tma_load_2d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
FP_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
FP_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 4D tile loads: tensor {128 cols, rows, heads, batch} (fp_api.cu make_tile_map);
// rows past the end of a sequence are zero-filled by the TMA unit.
FP_DEV void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                        int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
FP_DEV void tma_load_4d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1,
                             int c2, int c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "l"(policy)
      : "memory");
}
// Flattened head index hh = batch * per + head  ->  (head, batch) coordinates.
struct HeadCoord {
  int h, b;
};
FP_DEV HeadCoord head_coord(int hh, int per) { return HeadCoord{hh % per, hh / per}; }
// 128 x 128 tile of rows [row, row + 128) of flattened head hh (two SW128 boxes).
FP_DEV void tma_tile(void* dst, const CUtensorMap* m, uint64_t* bar, int row, int hh, int per) {
  const HeadCoord c = head_coord(hh, per);
  tma_load_4d(dst, m, bar, 0, row, c.h, c.b);
  tma_load_4d(static_cast<char*>(dst) + kBoxBytes, m, bar, 64, row, c.h, c.b);
}
FP_DEV void tma_tile_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int row, int hh, int per,
                          uint64_t pol) {
  const HeadCoord c = head_coord(hh, per);
  tma_load_4d_hint(dst, m, bar, 0, row, c.h, c.b, pol);
  tma_load_4d_hint(static_cast<char*>(dst) + kBoxBytes, m, bar, 64, row, c.h, c.b, pol);
}

// Load a full 128-row x 128-col bf16 tile as two 128x64 SW128 boxes.
FP_DEV void tma_load_tile(void* dst, const CUtensorMap* m, uint64_t* bar, int row) {
  tma_load_2d(dst, m, bar, 0, row);
  tma_load_2d(static_cast<char*>(dst) + kBoxBytes, m, bar, 64, row);
}
FP_DEV void tma_load_tile_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int row, uint64_t pol) {
  tma_load_2d_hint(dst, m, bar, 0, row, pol);
  tma_load_2d_hint(static_cast<char*>(dst) + kBoxBytes, m, bar, 64, row, pol);
}

// generic-proxy smem writes -> visible to the async proxy (tensor core / TMA)
FP_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------ UMMA descriptors ---
// Shared-memory matrix descriptor (tcgen05 "matrix descriptor"):
//  [0,14) start>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 |
//  [49,52) base offset | [52] LBO mode | [61,64) layout (2 = SWIZZLE_128B)
FP_DEV uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// K-major SW128 operand made of two 128x64 boxes: k-step kk (16 elements)
// starts at box (kk/4), byte (kk%4)*32 inside the 128-B swizzle row.
// SBO = 1024 (8 rows x 128 B); LBO unused for swizzled K-major.
FP_DEV uint64_t sdesc_kmajor(uint32_t tile_saddr, int kk) {
  return make_sdesc(tile_saddr + (kk >> 2) * kBoxBytes + (kk & 3) * 32, 16, 1024);
}
// MN-major SW128 operand (V as the B operand of P.V): rows = keys (the K dim),
// 64 contiguous d per box. k-step kk covers keys [16kk, 16kk+16): +2048 B.
// LBO = stride between the two 64-wide MN atoms (one box, 16 KiB);
// SBO = stride between 8-key groups (1024 B).
FP_DEV uint64_t sdesc_mnmajor(uint32_t tile_saddr, int kk) {
  return make_sdesc(tile_saddr + kk * 2048, kBoxBytes, 1024);
}

// Instruction descriptor for kind::f16 (bf16 x bf16 -> fp32):
//  [4,6) D fmt (1 = F32) | [7,10) A fmt (1 = BF16) | [10,13) B fmt (1 = BF16)
//  [15] A major (0 = K) | [16] B major (0 = K, 1 = MN) | [17,23) N>>3 | [24,29) M>>4
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]
FP_DEV void umma_bf16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on `bar` when all previously issued tcgen05.mma of this thread complete
FP_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
FP_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FP_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// M=128 N=128 SS chain of 8 k-steps on K-major SW128 tiles of two 16 KiB boxes
// (k-step kk at box kk/4, +32 B per step), issued by ONE elected lane of a
// warp whose lanes all execute this with the same operands (keeps them in
// uniform registers: no per-MMA R2UR / branch loop).
FP_DEV void umma_ss_chain8_elect(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, ep;\n\tsetp.ne.b32 p, 1, 0;\n\telect.sync _|ep, 0xffffffff;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %9, %17, 0;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %10, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %11, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %12, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %13, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %14, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %15, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %16, %17, p;\n\t}" ::"r"(d),
      "l"(a0), "l"(a0 + 2), "l"(a0 + 4), "l"(a0 + 6), "l"(a0 + 1024), "l"(a0 + 1026),
      "l"(a0 + 1028), "l"(a0 + 1030), "l"(b0), "l"(b0 + 2), "l"(b0 + 4), "l"(b0 + 6),
      "l"(b0 + 1024), "l"(b0 + 1026), "l"(b0 + 1028), "l"(b0 + 1030), "r"(idesc));
}
FP_DEV void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred ep;\n\telect.sync _|ep, 0xffffffff;\n\t"
      "@ep tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------- TMEM --------
// Called by one full warp. Writes the allocated base column address to *dst.
FP_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
FP_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
// TMEM address: lane in [31:16], column in [15:0]
FP_DEV uint32_t tmem_addr(uint32_t base, uint32_t lane, uint32_t col) {
  return base + (lane << 16) + col;
}

// 32 lanes x 32b, 32 consecutive columns -> r[0..31] (one row per thread)
FP_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
FP_DEV void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
// 32 lanes x 32b, 16 consecutive columns
FP_DEV void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]));
}
// 16 lanes x 256b, 16 repetitions: thread t (a = t % 4, c = t / 4) gets, for
// k = 0..15, r[4k], r[4k+1] = (lane c, columns 8k+2a, 8k+2a+1) and
// r[4k+2], r[4k+3] = (lane c+8, same columns) -- 64 values, 2 rows x 32 columns
#define FP_R64(r)                                                                              \
  "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),          \
      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
      "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
      "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),            \
      "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]),            \
      "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]),            \
      "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),            \
      "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),            \
      "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]),            \
      "=r"(r[62]), "=r"(r[63])
#define FP_W64(r)                                                                              \
  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),      \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),        \
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),      \
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),      \
      "r"(r[29]), "r"(r[30]), "r"(r[31]), "r"(r[32]), "r"(r[33]), "r"(r[34]), "r"(r[35]),      \
      "r"(r[36]), "r"(r[37]), "r"(r[38]), "r"(r[39]), "r"(r[40]), "r"(r[41]), "r"(r[42]),      \
      "r"(r[43]), "r"(r[44]), "r"(r[45]), "r"(r[46]), "r"(r[47]), "r"(r[48]), "r"(r[49]),      \
      "r"(r[50]), "r"(r[51]), "r"(r[52]), "r"(r[53]), "r"(r[54]), "r"(r[55]), "r"(r[56]),      \
      "r"(r[57]), "r"(r[58]), "r"(r[59]), "r"(r[60]), "r"(r[61]), "r"(r[62]), "r"(r[63])
#define FP_REGLIST64                                                                          \
  "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,"    \
  "%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,"   \
  "%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}"
FP_DEV void tmem_ld_16x256b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x16.b32 " FP_REGLIST64 ", [%64];"
               : FP_R64(r)
               : "r"(taddr));
}
FP_DEV void tmem_st_16x256b_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x16.b32 [%64], " FP_REGLIST64 ";"
               :
               : FP_W64(r), "r"(taddr));
}
// 16 lanes x 128b, 16 repetitions: thread t (a = t % 4, c = t / 4) owns, for
// k = 0..15, r[2k] = (lane c, column 4k+a) and r[2k+1] = (lane c+8, column 4k+a)
FP_DEV void tmem_st_16x128b_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x128b.x16.b32 [%32], "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31};" ::"r"(r[0]),
      "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
      "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
      "r"(r[30]), "r"(r[31]), "r"(taddr));
}
FP_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
FP_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Byte offset of element (row, col) inside a 128x128 bf16 tile stored as two
// 128x64 SWIZZLE_128B boxes (the layout TMA writes and UMMA reads).
FP_DEV uint32_t sw128_offset(uint32_t row, uint32_t col) {
  uint32_t box = col >> 6;
  uint32_t cb = (col & 63) * 2;                // byte within the 128-B row
  uint32_t chunk = (cb >> 4) ^ (row & 7);      // 16-B chunk, XOR-swizzled
  return box * kBoxBytes + row * 128 + chunk * 16 + (cb & 15);
}

FP_DEV float bf16_to_f32(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }

FP_DEV uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi));
  return r;
}

FP_DEV float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace fp
