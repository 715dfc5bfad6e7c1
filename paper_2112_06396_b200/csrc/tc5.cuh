// tcgen05 (5th-generation tensor core) helpers shared by the NTT column kernel
// (ntt_tc.cu) and the base conversion (bconv.cu): kind::i8 MMAs with operands in
// shared memory (canonical K-major, no swizzle) and s32 accumulators in TMEM.
#pragma once
#include "modarith.cuh"

namespace ck {
namespace tc5 {

// Canonical K-major SWIZZLE_NONE layout of `kbytes`-byte operand rows: 8 x 16-byte
// core matrices of 128 B; the kbytes/16 cores of an 8-row group are contiguous
// (LBO = 128 B between K-adjacent cores), groups follow each other
// (SBO = kbytes * 8 B between 8-row groups).
__host__ __device__ __forceinline__ unsigned kmaj_off(int row, int byte, int kbytes) {
  return ((((unsigned)row >> 3) * ((unsigned)kbytes >> 4) + ((unsigned)byte >> 4)) << 7) +
         (((unsigned)row & 7u) << 4) + ((unsigned)byte & 15u);
}

// shared-memory matrix descriptor (sm_100 format, bit 46) for that layout
__device__ __forceinline__ uint64_t smem_desc(unsigned saddr, int kbytes) {
  const uint64_t lbo = 128 >> 4, sbo = (uint64_t)(kbytes * 8) >> 4;
  return (uint64_t)((saddr >> 4) & 0x3FFF) | (lbo << 16) | (sbo << 32) | (1ull << 46);
}

// kind::i8 instruction descriptor: A/B unsigned 8-bit, D s32, K-major A and B, M = 128
__host__ __device__ __forceinline__ uint32_t idesc_i8(int n) {
  return (2u << 4) | (((uint32_t)n >> 3) << 17) | ((128u >> 4) << 24);
}

// D[tmem] (+)= A . B^T for one K step of 32 bytes
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(unsigned mbar_saddr) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   mbar_saddr)
               : "memory");
}

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned mbar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar),
      "r"(phase)
      : "memory");
}

// TMEM -> registers: this warp's 32 lanes x NCOL consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
        "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
        "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// s << n for a value whose top n bits are zero, as a rotate: a funnel shift can
// never be turned into an IMAD (ptxas otherwise moves shift-adds and register
// moves onto the fma-heavy pipe, the limiter of every epilogue here)
__device__ __forceinline__ u32 rotl32(u32 x, int n) {
  u32 r;
  asm("shf.l.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
  return r;
}

// V = sum_b s[b] 2^(8b), byte planes s[b] < 2^24 (V < 2^80), as lo + hi 2^32 + top 2^64;
// everything on the ALU pipe.
__device__ __forceinline__ void assemble_planes(const uint32_t* s, u32& lo, u32& hi, u32& top) {
  const u32 P0 = s[0] + rotl32(s[1], 8), P1 = s[2] + rotl32(s[3], 8);
  const u32 P2 = s[4] + rotl32(s[5], 8), P3 = s[6] + rotl32(s[7], 8);  // < 2^32
  // V = P0 + P1 2^16 + P2 2^32 + P3 2^48
  const u32 r1 = rotl32(P1, 16), r3 = rotl32(P3, 16);
  const u32 a_lo = r1 & 0xffff0000u, a_hi = r1 & 0xffffu;
  const u32 b_lo = r3 & 0xffff0000u, b_hi = r3 & 0xffffu;
  asm("add.cc.u32 %0, %1, %2;" : "=r"(lo) : "r"(P0), "r"(a_lo));
  asm("addc.cc.u32 %0, %1, %2;" : "=r"(hi) : "r"(P2), "r"(a_hi));
  asm("addc.u32 %0, %1, 0;" : "=r"(top) : "r"(b_hi));
  asm("add.cc.u32 %0, %0, %1;" : "+r"(hi) : "r"(b_lo));
  asm("addc.u32 %0, %0, 0;" : "+r"(top));
}

}  // namespace tc5
}  // namespace ck
