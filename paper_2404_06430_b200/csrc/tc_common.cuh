// sm_100a building blocks: mbarriers, TMA (cp.async.bulk.tensor), TMEM
// allocation / loads and tcgen05.mma with shared-memory descriptors.
// Written as inline PTX against the PTX ISA for sm_100a; descriptor bit
// layouts follow the UMMA descriptor definitions (instruction descriptor,
// K-major SWIZZLE_128B smem descriptor, version 1).
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace fb {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 4-D tiled load into shared memory, completion counted on `bar` (bytes)
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy global -> shared (bytes multiple of 16, 16-byte aligned)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// explicit shared-window loads / stores (32-bit smem addresses): pointers
// derived from the manually aligned dynamic-smem base are generic to the
// compiler, which then emits 64-bit generic ST/LD with address arithmetic
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_u16(uint32_t a, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
  return v;
}

// ----------------------------------------------------------------- TMEM
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// 32 lanes x 8 consecutive 32-bit columns -> 8 registers per thread
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ UMMA
// Instruction descriptor, kind::tf32, fp32 accumulate, both operands K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4)                      // D format F32
         | (2u << 7)                    // A format TF32
         | (2u << 10)                   // B format TF32
         | ((uint32_t)(N >> 3) << 17)   // N / 8
         | ((uint32_t)(M >> 4) << 24);  // M / 16
}
// K-major, SWIZZLE_128B smem descriptor: rows of 128 B, 8-row groups of
// 1024 B (SBO = 1024 B), tile base 1024-byte aligned; advancing K by 8 tf32
// (32 B) advances the start address by 32 B.
__device__ __forceinline__ uint64_t sdesc_k128(uint32_t smem_addr) {
  return (uint64_t)((smem_addr >> 4) & 0x3FFFu)  // start address
         | ((uint64_t)1 << 16)                    // LBO (ignored for swizzled K-major)
         | ((uint64_t)(1024 >> 4) << 32)          // SBO
         | ((uint64_t)1 << 46)                    // descriptor version (sm_100)
         | ((uint64_t)2 << 61);                   // SWIZZLE_128B
}
// MN-major, SWIZZLE_128B smem descriptor: 128-byte rows hold 32 consecutive
// M (or N) elements, 8-row K atoms at SBO = 1024 B, M/N blocks of 32 at `lbo`
// bytes.  `base_off` = the start address's row phase within the 1024 B
// swizzle atom when the start is not atom-aligned (0 when it is).
__device__ __forceinline__ uint64_t sdesc_mn128(uint32_t smem_addr, uint32_t lbo, uint32_t base_off) {
  return (uint64_t)((smem_addr >> 4) & 0x3FFFu)
         | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16)
         | ((uint64_t)(1024 >> 4) << 32)
         | ((uint64_t)1 << 46)
         | ((uint64_t)(base_off & 7u) << 49)
         | ((uint64_t)2 << 61);
}
// generic smem descriptor: layout 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
__device__ __forceinline__ uint64_t sdesc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((smem_addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
// kind::f16 (fp16 inputs, fp32 accumulate), both operands K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// kind::f16 (fp16 inputs, fp32 accumulate), both operands MN-major.  (The
// tensor core accepts MN-major operands for 16-bit kinds; kind::tf32 with an
// MN-major operand produced no output on sm_100a in our tests.)
__host__ __device__ constexpr uint32_t idesc_f16_mn(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24) | (1u << 15) | (1u << 16);
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// The 3-term split product of one K step, issued from ONE asm statement so the
// compiler elects / broadcasts the operands once per group instead of once per
// MMA (the single-thread issue path costs ~13 instructions per UTCHMMA):
//   dmain += Ahi*Bhi (accumulate if pm), dcross += Ahi*Blo (if px), dcross += Alo*Bhi.
__device__ __forceinline__ void mma3_f16(uint32_t dmain, uint32_t dcross, uint64_t ah, uint64_t al, uint64_t bh,
                                         uint64_t bl, uint32_t idesc, uint32_t pm, uint32_t px) {
  asm volatile(
      "{\n\t.reg .pred pm, px, pt;\n\t"
      "setp.ne.b32 pm, %7, 0;\n\t"
      "setp.ne.b32 px, %8, 0;\n\t"
      "setp.eq.b32 pt, %6, %6;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %6, pm;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %5, %6, px;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, pt;\n}" ::"r"(dmain),
      "r"(dcross), "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(pm), "r"(px)
      : "memory");
}
// mma2s for one K step with explicit descriptors: d (2N wide) += Ahi*[Bhi;Blo]
// (accumulate iff pacc), dcross (N wide) += Alo*Bhi.
__device__ __forceinline__ void mma2_f16(uint32_t d, uint32_t dcross, uint64_t ah, uint64_t al, uint64_t bh,
                                         uint32_t idesc2n, uint32_t idescn, uint32_t pacc) {
  asm volatile(
      "{\n\t.reg .pred pa, pt;\n\t"
      "setp.ne.b32 pa, %7, 0;\n\t"
      "setp.eq.b32 pt, %5, %5;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %5, pa;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, pt;\n}" ::"r"(d),
      "r"(dcross), "l"(ah), "l"(al), "l"(bh), "r"(idesc2n), "r"(idescn), "r"(pacc)
      : "memory");
}
// KS consecutive K steps of mma3_f16 in one asm statement: step k uses the
// descriptors advanced by k * AINC / BINC (descriptor units of 16 bytes); only
// step 0 takes the pm / px accumulate flags, later steps always accumulate.
template <int KS, int AINC, int BINC>
__device__ __forceinline__ void mma3_f16_ks(uint32_t dmain, uint32_t dcross, uint64_t ah, uint64_t al, uint64_t bh,
                                            uint64_t bl, uint32_t idesc, uint32_t pm, uint32_t px) {
  static_assert(KS == 2 || KS == 4, "mma3_f16_ks: 2 or 4 K steps");
  if constexpr (KS == 2) {
    asm volatile(
        "{\n\t.reg .pred pm, px, pt;\n\t.reg .b64 a1, c1, b1, e1;\n\t"
        "setp.ne.b32 pm, %7, 0;\n\t"
        "setp.ne.b32 px, %8, 0;\n\t"
        "setp.eq.b32 pt, %6, %6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %6, pm;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %5, %6, px;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, pt;\n\t"
        "add.s64 a1, %2, %9;\n\tadd.s64 c1, %3, %9;\n\tadd.s64 b1, %4, %10;\n\tadd.s64 e1, %5, %10;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], a1, e1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n}" ::"r"(dmain),
        "r"(dcross), "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(pm), "r"(px), "n"(AINC), "n"(BINC)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred pm, px, pt;\n\t.reg .b64 a1, c1, b1, e1;\n\t"
        "setp.ne.b32 pm, %7, 0;\n\t"
        "setp.ne.b32 px, %8, 0;\n\t"
        "setp.eq.b32 pt, %6, %6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %6, pm;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %5, %6, px;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, pt;\n\t"
        "add.s64 a1, %2, %9;\n\tadd.s64 c1, %3, %9;\n\tadd.s64 b1, %4, %10;\n\tadd.s64 e1, %5, %10;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], a1, e1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n\t"
        "add.s64 a1, %2, %11;\n\tadd.s64 c1, %3, %11;\n\tadd.s64 b1, %4, %12;\n\tadd.s64 e1, %5, %12;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], a1, e1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n\t"
        "add.s64 a1, %2, %13;\n\tadd.s64 c1, %3, %13;\n\tadd.s64 b1, %4, %14;\n\tadd.s64 e1, %5, %14;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], a1, e1, %6, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n}" ::"r"(dmain),
        "r"(dcross), "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(pm), "r"(px), "n"(AINC), "n"(BINC),
        "n"(2 * AINC), "n"(2 * BINC), "n"(3 * AINC), "n"(3 * BINC)
        : "memory");
  }
}
// The 3-term split product with the weight operand's hi and lo parts stacked
// along N: B = [Bhi; Blo] (2N rows) so ONE MMA of width 2N forms Ahi*Bhi into
// d[0, N) and Ahi*Blo into d[N, 2N); a second MMA of width N adds Alo*Bhi
// into d[N, 2N).  Two MMAs per K step instead of three, and the epilogue
// sums two accumulators (main | cross).  KS K steps at AINC / BINC
// descriptor units apart; step 0 accumulates iff pacc.
template <int KS, int AINC, int BINC>
__device__ __forceinline__ void mma2s_f16_ks(uint32_t d, uint32_t dcross, uint64_t ah, uint64_t al, uint64_t bh,
                                             uint32_t idesc2n, uint32_t idescn, uint32_t pacc) {
  static_assert(KS == 2 || KS == 4, "mma2s_f16_ks: 2 or 4 K steps");
  if constexpr (KS == 2) {
    asm volatile(
        "{\n\t.reg .pred pa, pt;\n\t.reg .b64 a1, c1, b1;\n\t"
        "setp.ne.b32 pa, %7, 0;\n\t"
        "setp.eq.b32 pt, %5, %5;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %5, pa;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, pt;\n\t"
        "add.s64 a1, %2, %8;\n\tadd.s64 c1, %3, %8;\n\tadd.s64 b1, %4, %9;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n}" ::"r"(d),
        "r"(dcross), "l"(ah), "l"(al), "l"(bh), "r"(idesc2n), "r"(idescn), "r"(pacc), "n"(AINC), "n"(BINC)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred pa, pt;\n\t.reg .b64 a1, c1, b1;\n\t"
        "setp.ne.b32 pa, %7, 0;\n\t"
        "setp.eq.b32 pt, %5, %5;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %5, pa;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %6, pt;\n\t"
        "add.s64 a1, %2, %8;\n\tadd.s64 c1, %3, %8;\n\tadd.s64 b1, %4, %9;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n\t"
        "add.s64 a1, %2, %10;\n\tadd.s64 c1, %3, %10;\n\tadd.s64 b1, %4, %11;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n\t"
        "add.s64 a1, %2, %12;\n\tadd.s64 c1, %3, %12;\n\tadd.s64 b1, %4, %13;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, pt;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], c1, b1, %6, pt;\n}" ::"r"(d),
        "r"(dcross), "l"(ah), "l"(al), "l"(bh), "r"(idesc2n), "r"(idescn), "r"(pacc), "n"(AINC), "n"(BINC),
        "n"(2 * AINC), "n"(2 * BINC), "n"(3 * AINC), "n"(3 * BINC)
        : "memory");
  }
}
// kind::tf32 instruction descriptor with both operands MN-major
__host__ __device__ constexpr uint32_t idesc_tf32_mn(int M, int N) {
  return idesc_tf32(M, N) | (1u << 15) | (1u << 16);
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` when all previously issued tcgen05.mma of this thread complete
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// ------------------------------------------------------ CTA pairs (cta_group::2)
// The two CTAs of a 2-CTA cluster run one M = 256 MMA: A rows 0-127 come from
// CTA 0's shared memory, rows 128-255 from CTA 1's (same offsets), B is split
// along N (CTA 0 holds the first N/2 rows), each CTA's TMEM holds its 128 rows.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_cluster(uint32_t cluster_addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_addr),
               "r"(bytes)
               : "memory");
}
// 4-D tiled load into this CTA's smem, completion bytes counted on an mbarrier of
// either CTA of the pair (the leader's, for the pair's MMA issuer)
__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                uint32_t bar_cluster_addr) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
      "[%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar_cluster_addr)
      : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem) {  // one warp of EACH CTA (same warp id)
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
// arrive on `bar` (same offset) in every CTA of `mask` once the pair's MMAs complete
__device__ __forceinline__ void mma_commit2_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::
                   "r"(smem_u32(bar)),
               "h"(mask)
               : "memory");
}
// M = 256 pair MMAs of the 3-term split for KS = 2 K steps: d[0, 2N) += ah * b1 (b1 = the
// CTA halves of [W hi; W lo]), d[N, 2N) += al * b2 (b2 = halves of W hi)
__device__ __forceinline__ void mma2p_f16_ks2(uint32_t d, uint32_t dcross, uint64_t ah, uint64_t al, uint64_t b1,
                                              uint64_t b2, uint32_t idesc2n, uint32_t idescn, uint32_t pacc) {
  asm volatile(
      "{\n\t.reg .pred pa, pt;\n\t.reg .b64 a1, c1, e1, f1;\n\t"
      "setp.ne.b32 pa, %8, 0;\n\t"
      "setp.eq.b32 pt, %6, %6;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %4, %6, pa;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], %3, %5, %7, pt;\n\t"
      "add.s64 a1, %2, 2;\n\tadd.s64 c1, %3, 2;\n\tadd.s64 e1, %4, 2;\n\tadd.s64 f1, %5, 2;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, e1, %6, pt;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%1], c1, f1, %7, pt;\n}" ::"r"(d),
      "r"(dcross), "l"(ah), "l"(al), "l"(b1), "l"(b2), "r"(idesc2n), "r"(idescn), "r"(pacc)
      : "memory");
}

// generic-proxy smem writes -> visible to the async proxy (TMA / tensor core)
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// fp32 -> (hi, lo) split for 3xTF32: hi = rna(x) (a tf32 value), lo = x - hi
// (exact in fp32; the tensor core reads its top tf32 bits)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  // rna to 10 mantissa bits as integer add + mask (2 instructions; cvt.rna.tf32 adds an
  // inf test): equal to cvt.rna.tf32.f32 for every finite x; a non-finite x leaves a
  // non-finite hi or lo, so the product stays non-finite
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
#ifdef FB_SPLIT_RNA_LO
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - hi));
  lo = __uint_as_float(l);
#else
  lo = x - hi;
#endif
}

// byte offset of element (row, k) in a K-major SWIZZLE_128B tile of 32 fp32 per row
__host__ __device__ __forceinline__ uint32_t sw128_offset(uint32_t row, uint32_t k) {
  const uint32_t chunk = k >> 2;  // 16-byte chunk within the 128-byte row
  return row * 128u + (((chunk ^ (row & 7u)) << 4) | ((k & 3u) << 2));
}

// 256-bit global load / store (sm_100): one full 32-byte sector per lane; p 32-byte aligned
__device__ __forceinline__ void ldg256(const float* p, float (&v)[8]) {
  asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void stg256f(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]) : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n}"
      : "=r"(pred));
  return pred != 0;
}

}  // namespace tc
}  // namespace fb
