// NTT column phase (forward and inverse) on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).
//
// Forward: the column phase (stages m = 1 .. 128 of the reference's
// Cooley-Tukey ladder, rnspoly.py:48-62, on the 256 x 2^P2 storage matrix)
// maps every column c through the SAME 256 x 256 matrix.  Split by row bits
// r = 16 r_hi + r_lo:
//   stages m = 1..8   mix r_hi only, with twiddles that depend on r_hi alone:
//                     one 16 x 16 matrix M1, shared by every (r_lo, c);
//   stages m = 16..128 mix r_lo inside block beta = r_hi; that block evaluates
//                     mod (X^16 - gamma_beta), i.e. M2[beta] = F diag(d_beta)
//                     with F = M2[0] and a per-(beta, r_lo) twist d_beta.
// Inverse (Gentleman-Sande, rnspoly.py:64-79): blocks first, M1[beta] =
// diag(e_beta) G on r_lo (an output twist), then one shared matrix on r_hi;
// the INTT's n^-1 (times ihat) is a Shoup multiply in the last epilogue.
// The plan derives every matrix and twist from its twiddle tables and checks
// the factorisations entry by entry (ntt_tc_tables).
//
// Each 16-point product is an exact integer GEMM on bytes: with x = sum_a
// x_a 2^8a and B[(j,a)][(k,b)] = byte b of (Mat[k][j] 2^8a mod p),
//   S_kb = sum_(j,a) x_ja B[(j,a)][(k,b)]     (K = 128 bytes, < 2^23)
//   y_k == sum_b S_kb 2^8b  (mod p)
// so no modular reduction is needed inside the GEMM, any 64-bit input is
// allowed, and the epilogue reduces V = sum_b S_kb 2^8b < 2^80 once (FP64
// quotient, as in the tensor-core base conversion).
//
// Work unit = a tile of 8 columns x 256 rows of one limb; one CTA (512
// threads, one per SM: 164 KB SMEM, all 512 TMEM columns) runs 4 independent
// 4-warp pipelines over 32 tiles, sharing B1/B2 and the twists:
//   cp.async tile -> A1[(g1,c)][e1]         (128 x 128 B, canonical K-major)
//   MMA  D1 = A1 . B1^T                     (M128 N128 K128, 128 TMEM columns)
//   epilogue: y = (V mod p) * twist         -> A2[(o,c)][g1]   (same buffer)
//   MMA  D2 = A2 . B2^T
//   epilogue: V mod p                       -> global (forward: lazy (0, 4p);
//                                              inverse: times the scale, canonical)
// with the next tile's operand already streaming into the group's second
// buffer.  Forward outputs are lazy (the butterfly kernels leave [0, 16q));
// every consumer folds either.
#include "ck_internal.h"
#include "ntt.cuh"
#include "tc5.cuh"

#include <cstdlib>
#include <vector>

namespace ck {

namespace {

constexpr int kTcCols = 8;                   // columns per tile (M = 16 x 8 = 128 rows)
constexpr int kTcGroups = 4;                 // independent pipelines per CTA (share B)
#ifndef CKB200_TC_GW
#define CKB200_TC_GW 4
#endif
#ifndef CKB200_TC_DB
#define CKB200_TC_DB 1
#endif
constexpr int kTcGW = CKB200_TC_GW;          // warps per group: 4 = one per TMEM lane quarter at up to 128 registers, with
                                             // double-buffered TMEM loads (CKB200_TC_DB): 10.06 ms per C3 step against 10.13 for
                                             // 8 warps (two per quarter, 64 registers, one load in flight); 4 warps without the
                                             // double buffer 10.17
constexpr int kTcHalves = kTcGW / 4;
constexpr int kTcThreads = 32 * kTcGW * kTcGroups;
#ifndef CKB200_TC_TILES
#define CKB200_TC_TILES 32
#endif
constexpr int kTcTiles = CKB200_TC_TILES;    // tiles per CTA (B loaded once per CTA)
constexpr int kOpBytes = 128 * 128;          // one 128-row operand (A), bytes
constexpr int kBBytes = 128 * 128;           // one B matrix (N = 128 rows of K = 128 bytes)

// operands are rows of 128 bytes in the canonical K-major layout of tc5.cuh
__host__ __device__ __forceinline__ unsigned kmaj_off(int row, int byte) {
  return tc5::kmaj_off(row, byte, 128);
}
__device__ __forceinline__ uint64_t smem_desc(unsigned saddr) { return tc5::smem_desc(saddr, 128); }
// kind::i8, A/B unsigned 8-bit, D s32, K-major A and B, M = 128, N = 128
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  tc5::mma_i8(d_tmem, a, b, tc5::idesc_i8(128), acc);
}
__device__ __forceinline__ unsigned mbar_addr(const uint64_t* b) { return tc5::saddr(b); }
using tc5::mbar_wait;
using tc5::tmem_ld32;
using tc5::tmem_wait_ld;
__device__ __forceinline__ void tc_fence_before() { tc5::fence_before(); }
__device__ __forceinline__ void tc_fence_after() { tc5::fence_after(); }
using tc5::fence_async_smem;

// V = sum_b S_b 2^8b (S_b < 2^23, V < 2^80) reduced into (0, 4p), p > 2^49.5,
// integer-only: with vhi = floor(V / 2^32) < 2^49, W = floor(vhi / 2^17) < 2^32
// and m = round(2^81 / p) < 2^32, the quotient qh = floor(W m / 2^32) satisfies
//   V/p - qh in (-0.51, 2.22)
// (dropped low bits of vhi: < 2^49/p < 0.71; m's rounding: W |m - 2^81/p| / 2^32
// < 0.51; the floor: < 1), so V - qh p + p lands in (0, 4p), computed mod 2^64.
// One mul.hi replaces the FP64 estimate (whose DADD/DFMA bursts throttled the
// FP64 pipe in every epilogue); the byte-plane assembly stays on the ALU pipe.
// The byte-plane assembly (tc5::assemble_planes) is written so that ptxas keeps it on
// the ALU pipe: the fma-heavy pipe is this kernel's limiter and ptxas otherwise turns
// shift-adds and register moves into IMADs.
__device__ __forceinline__ u64 reduce_lazy(const uint32_t* s, u64 p, u32 m81) {
  u32 lo, hi, top;
  tc5::assemble_planes(s, lo, hi, top);  // V = lo + hi 2^32 + top 2^64
  // vhi = floor(V / 2^32) = hi + top 2^32 < 2^49, W = floor(vhi / 2^17)
  const u32 qh = __umulhi(__funnelshift_r(hi, top, 17), m81);
  const u64 v = ((u64)hi << 32) | lo;
  return v + p - (u64)qh * p;  // (mod 2^64)
}

// round(2^81 / p) for reduce_lazy (p > 2^49.5: < 2^31.5)
__device__ __forceinline__ u32 tc_m81(u64 p) {
  return (u32)__double2uint_rn(__ddiv_rn(2417851639229258349412352.0, (double)p));
}

// x * w mod p into [0, 4p) for any 64-bit x: the approximate-quotient Shoup product
// of the small-prime butterflies (modarith.cuh shoup_tw4: three 32-bit products for
// the quotient, the remainder as one multiply-accumulate chain with 2^64 - p).
// The next tensor-core pass accepts any 64-bit operand; canonical outputs
// fold it with two conditional subtractions.
__device__ __forceinline__ u64 shoup_tc(u64 x, u64 w, u64 wp, u64 np) { return shoup_tw4(x, w, wp, np); }

__device__ __forceinline__ void st_u64(unsigned char* base, int row, int elem, u64 v) {
  *(u64*)(base + kmaj_off(row, elem * 8)) = v;
}

// Tile t's 256 x 8 block goes straight from global memory into operand
// layout with 8-byte cp.async (no registers).  Pass-1 operand row
// (g1, c) = 8 g1 + c holds the 16 values of the contracted row bits e1:
// forward g1 = r_lo, e1 = r_hi; inverse g1 = r_hi, e1 = r_lo.  Lane ->
// (c = lane & 7, e1 = 4 (warp & 3) + lane / 8), iteration -> g1: a warp's 32
// copies land in two 128-byte core-matrix rows (no bank conflicts).
template <int P2, bool INV>
__device__ __forceinline__ void stage_tile(unsigned a_dst, const u64* base, int c0, int gw, int lane) {
  const int c = lane & 7, e1 = 4 * (gw & 3) + (lane >> 3);   // gw: warp within the group
#pragma unroll
  for (int g1 = (16 / kTcHalves) * (gw >> 2); g1 < (16 / kTcHalves) * ((gw >> 2) + 1); ++g1) {
    const int r = INV ? g1 * 16 + e1 : e1 * 16 + g1;
    const u64* src = base + ((long long)r << P2) + c0 + c;
    const unsigned dst = a_dst + kmaj_off(8 * g1 + c, 8 * e1);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Four warp groups per CTA (one CTA per SM: 512 TMEM columns)
// run independent tile pipelines (own double-buffered A operand, TMEM
// accumulator, mbarrier and named barrier) over tiles g, g+4, ...,
// sharing the CTA's B matrices and twists.  Tile t+4's data streams in
// (cp.async) while tile t is on the tensor cores and in the epilogues; a warp
// owns one TMEM lane quarter and keeps the next 32 accumulator columns in
// flight (tcgen05.ld) while it reduces the current ones.
template <int P2, bool INV, int TILES = kTcTiles>
__global__ void __launch_bounds__(kTcThreads, 1) ntt_col_tc_kernel(NttArgs a) {
  extern __shared__ __align__(1024) unsigned char tsm[];
  unsigned char* Bm = tsm + 2 * kTcGroups * kOpBytes;      // A[group][2] (16 KB each), then B1 | B2
  ulonglong2* tw = (ulonglong2*)(Bm + 2 * kBBytes);        // twists [beta][r_lo] (4 KB)
  uint64_t* mbar = (uint64_t*)(tw + 256);                  // [group], then the table barrier
  uint64_t* tbar = mbar + kTcGroups;
  uint32_t* tslot = (uint32_t*)(tbar + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp / kTcGW, gw = warp % kTcGW, gtid = tid % (32 * kTcGW);
  const int quarter = gw & 3, half = gw >> 2;
  const int job = blockIdx.y;
  const int prime = a.prime_idx[job];
  const u64 p = a.pc[prime].q;
  const u32 m81 = tc_m81(p);
  const u64 np = neg_opaque(p);
  u64* base = a.data + (a.row_off ? a.row_off[job] : ((long long)job << a.logn)) +
              (long long)blockIdx.z * a.batch_stride;
  const unsigned mb_s = (unsigned)__cvta_generic_to_shared(mbar + grp);
  const unsigned abuf_s = (unsigned)__cvta_generic_to_shared(tsm) + grp * 2 * kOpBytes;
  unsigned char* abuf = tsm + grp * 2 * kOpBytes;
  const unsigned b_s = (unsigned)__cvta_generic_to_shared(Bm);
  const int cbase = blockIdx.x * TILES * kTcCols;
  const int bar_id = 1 + grp;
  auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(32 * kTcGW) : "memory"); };

  pdl_trigger();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        (unsigned)__cvta_generic_to_shared(tslot)), "n"(128 * kTcGroups));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (gtid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb_s));
  if (tid == 0) {
    // the prime's B1 | B2 matrices (32 KB) and twists (4 KB): two TMA bulk copies,
    // in flight while the predecessor drains (plan tables, not its output)
    mbar_init(tbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(tbar, 2 * kBBytes + 256 * sizeof(ulonglong2));
    bulk_g2s(Bm, a.tcB + ((size_t)prime * 4 + (INV ? 2 : 0)) * kBBytes, 2 * kBBytes, tbar);
    bulk_g2s(tw, a.tcD + ((size_t)prime * 2 + (INV ? 1 : 0)) * 256, 256 * sizeof(ulonglong2), tbar);
  }
  pdl_wait();  // the predecessor's output is read from here on
  stage_tile<P2, INV>(abuf_s, base, cbase + grp * kTcCols, gw, lane);  // this group's first tile
  // inverse: the INTT's final scale n^-1 (times the optional extra constant)
  const ulonglong2 scl = !INV ? make_ulonglong2(0, 0)
                              : (a.scale ? a.scale[job] : make_ulonglong2(a.pc[prime].ninv, a.pc[prime].ninvp));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  mbar_wait(mbar_addr(tbar), 0);  // B matrices and twists have landed
  const uint32_t tacc = *tslot + grp * 128;                     // this group's accumulator columns
  const uint32_t tl = tacc + ((uint32_t)(quarter * 32) << 16);  // this warp's lane quarter
  const int m = quarter * 32 + lane;                            // this thread's D row
  unsigned phase = 0;

  for (int it = 0; grp + kTcGroups * it < TILES; ++it) {
    const int tile = grp + kTcGroups * it;
    const int c0 = cbase + tile * kTcCols;
    unsigned char* A = abuf + (it & 1) * kOpBytes;
    const unsigned a_s = abuf_s + (it & 1) * kOpBytes;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    fence_async_smem();
    tc_fence_before();
    gsync();
    tc_fence_after();
    if (tile + kTcGroups < TILES)
      stage_tile<P2, INV>(abuf_s + ((it + 1) & 1) * kOpBytes, base, c0 + kTcGroups * kTcCols, gw, lane);
    // ---- pass 1: D1[(r_lo,c)][(beta,b)] = A1 . B1^T
    if (gtid == 0) {
#pragma unroll
      for (int s = 0; s < 4; ++s) mma_i8(tacc, smem_desc(a_s + s * 256), smem_desc(b_s + s * 256), s > 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb_s)
                   : "memory");
    }
    mbar_wait(mb_s, phase);
    phase ^= 1;
    tc_fence_after();
    {
      const int g1 = m >> 3, c = m & 7;
      constexpr int NH = 4 / kTcHalves;               // TMEM loads of 4 outputs (32 columns) each
      const int h0 = NH * half;
      if constexpr (CKB200_TC_DB) {
        // double-buffered TMEM loads: the next 32 columns are in flight while these are reduced
        uint32_t sv[2][32];
        tmem_ld32(tl + h0 * 32, sv[0]);
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          tmem_wait_ld();
          if (hh + 1 < NH) tmem_ld32(tl + (h0 + hh + 1) * 32, sv[(hh + 1) & 1]);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int o = (h0 + hh) * 4 + u;
            const u64 y = reduce_lazy(sv[hh & 1] + 8 * u, p, m81);
            const ulonglong2 d = tw[o * 16 + g1];
            st_u64(A, o * 8 + c, g1, shoup_tc(y, d.x, d.y, np));  // [0, 4p)
          }
        }
      } else {
#pragma unroll 1
      for (int h = h0; h < h0 + NH; ++h) {   // 4 outputs (32 TMEM columns) per wait
        uint32_t sv[32];
        tmem_ld32(tl + h * 32, sv);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int o = h * 4 + u;                      // pass-1 output index
          const u64 y = reduce_lazy(sv + 8 * u, p, m81);
          const ulonglong2 d = tw[o * 16 + g1];
          st_u64(A, o * 8 + c, g1, shoup_tc(y, d.x, d.y, np));  // [0, 4p)
        }
      }
      }
    }
    fence_async_smem();
    tc_fence_before();
    gsync();
    tc_fence_after();
    // ---- pass 2: D2[(beta,c)][(k,b)] = A2 . B2^T
    if (gtid == 0) {
#pragma unroll
      for (int s = 0; s < 4; ++s)
        mma_i8(tacc, smem_desc(a_s + s * 256), smem_desc(b_s + kBBytes + s * 256), s > 0);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb_s)
                   : "memory");
    }
    mbar_wait(mb_s, phase);
    phase ^= 1;
    tc_fence_after();
    {
      const int o1 = m >> 3, c = m & 7;
      u64* col = base + c0 + c;
      constexpr int NH = 4 / kTcHalves;
      const int h0 = NH * half;
      auto out2 = [&](const uint32_t* sv, int h) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int o2 = h * 4 + u;
          const u64 v = reduce_lazy(sv + 8 * u, p, m81);
          if (INV)  // rows 16 o2 + o1; canonical (the base conversion needs exact residues)
            col[(long long)(o2 * 16 + o1) << P2] = csub(csub(shoup_tc(v, scl.x, scl.y, np), 2 * p), p);
          else      // rows 16 o1 + o2; lazy (0, 4p)
            col[(long long)(o1 * 16 + o2) << P2] = v;
        }
      };
      if constexpr (CKB200_TC_DB) {
        uint32_t sv[2][32];
        tmem_ld32(tl + h0 * 32, sv[0]);
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          tmem_wait_ld();
          if (hh + 1 < NH) tmem_ld32(tl + (h0 + hh + 1) * 32, sv[(hh + 1) & 1]);
          out2(sv[hh & 1], h0 + hh);
        }
      } else {
#pragma unroll 1
        for (int h = h0; h < h0 + NH; ++h) {
          uint32_t sv[32];
          tmem_ld32(tl + h * 32, sv);
          tmem_wait_ld();
          out2(sv, h);
        }
      }
    }
    tc_fence_before();   // the next tile's MMA rewrites D: TMEM reads are complete
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tslot), "n"(128 * kTcGroups));
  }
}

constexpr size_t kTcSmem = 2 * kTcGroups * kOpBytes + 2 * kBBytes + 256 * sizeof(ulonglong2) + 72;

template <int P2, bool INV, int TILES>
int launch_tt(const NttArgs& a, int jobs, int batch, cudaStream_t st) {
  // the shared-memory opt-in is per device: track it per device ordinal
  static unsigned done = 0;  // bit d: set on device d (ordinals < 32)
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 32 || !((done >> dev) & 1u)) {
    cudaFuncSetAttribute(ntt_col_tc_kernel<P2, INV, TILES>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
    if (dev < 32) __atomic_fetch_or(&done, 1u << dev, __ATOMIC_RELAXED);
  }
  const dim3 grid((1 << P2) / (kTcCols * TILES), jobs, batch);
  launch_pdl(ntt_col_tc_kernel<P2, INV, TILES>, grid, dim3(kTcThreads), kTcSmem, st, a);
  return 0;
}

// Tiles per CTA.  The kernel runs ONE CTA per SM (TMEM, shared memory), so a launch takes
// whole waves: kTcTiles = 32 (one table load and TMEM allocation per 32 column tiles) for
// large batches; for small launches (one ciphertext: 16-72 limb jobs; hoisted batches of a
// few) the count among 8 / 16 / 32 that minimises waves x (prologue + iterations), a CTA's
// prologue costing about two iterations of its four pipelines.
// CKB200_TC_SPLIT = 8 / 16 / 32 forces the count (0 / 1: 32 / 8) (measurements, tests).
template <int P2, bool INV>
int launch_t(const NttArgs& a, int jobs, int batch, cudaStream_t st) {
  static const int force = [] {
    const char* e = getenv("CKB200_TC_SPLIT");
    const int v = e ? atoi(e) : -1;
    return v == 0 ? 32 : v == 1 ? 8 : v;
  }();
  static const int sms = [] {
    int d = 0, n = 148;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    return n > 0 ? n : 148;
  }();
  int tiles = kTcTiles;
  const long long per = (long long)jobs * batch;
  if (force == 8 || force == 16 || force == 32) {
    tiles = force;
  } else if (per * ((1 << P2) / (kTcCols * kTcTiles)) < 8LL * sms) {
    long long best = -1;
    for (int c = 8; c <= kTcTiles; c *= 2) {
      const long long ctas = per * ((1 << P2) / (kTcCols * c));
      const long long cost = ((ctas + sms - 1) / sms) * (2 + c / kTcGroups);
      if (best < 0 || cost < best) {
        best = cost;
        tiles = c;
      }
    }
  }
  switch (tiles) {
    case 8: return launch_tt<P2, INV, 8>(a, jobs, batch, st);
    case 16: return launch_tt<P2, INV, 16>(a, jobs, batch, st);
    default: return launch_tt<P2, INV, kTcTiles>(a, jobs, batch, st);
  }
}

// ---------------------------------------------------------------- host side
using u128 = unsigned __int128;
u64 mm(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
u64 pw(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  for (; e; e >>= 1, a = mm(a, a, q))
    if (e & 1) r = mm(r, a, q);
  return r;
}

// Run CT stages s in [s0, s1) of the 256-row column phase on a 256-vector.
void col_stages(std::vector<u64>& x, const ulonglong2* tw, u64 q, int s0, int s1) {
  for (int s = s0; s < s1; ++s) {
    const int m = 1 << s, t = 128 >> s;
    for (int i = 0; i < m; ++i) {
      const u64 w = tw[m + i].x;
      for (int j = i * 2 * t; j < i * 2 * t + t; ++j) {
        const u64 u = x[j], v = mm(x[j + t], w, q);
        x[j] = (u + v) % q;
        x[j + t] = (u + q - v) % q;
      }
    }
  }
}

}  // namespace

namespace {

// Run GS stages s in [s0, s1) of the inverse 256-row column phase (rows at
// distance t = 2^s, twiddle itw[128/2^s + block], rnspoly.py:64-79).
void col_stages_inv(std::vector<u64>& x, const ulonglong2* itw, u64 q, int s0, int s1) {
  for (int s = s0; s < s1; ++s) {
    const int t = 1 << s, h = 128 >> s;
    for (int blk = 0; blk < h; ++blk) {
      const u64 w = itw[h + blk].x;
      for (int j = blk * 2 * t; j < blk * 2 * t + t; ++j) {
        const u64 u = x[j], v = x[j + t];
        x[j] = (u + v) % q;
        x[j + t] = mm((u + q - v) % q, w, q);
      }
    }
  }
}

void put_b(unsigned char* dst, const u64 (&mat)[16][16], u64 q) {
  // B[n = 8k + b][byte 8j + a] = byte b of (Mat[k][j] 2^8a mod q)
  for (int k = 0; k < 16; ++k)
    for (int j = 0; j < 16; ++j) {
      u64 v = mat[k][j];
      for (int aa = 0; aa < 8; ++aa) {
        for (int b = 0; b < 8; ++b) dst[kmaj_off(8 * k + b, 8 * j + aa)] = (unsigned char)(v >> (8 * b));
        v = mm(v, 256 % q, q);
      }
    }
}

ulonglong2 shp(u64 d, u64 q) { return make_ulonglong2(d, (u64)(((u128)d << 64) / q)); }

// Forward: M1 on r_hi (shared), then block beta = r_hi: M2[beta] = F diag(d_beta).
bool fwd_tables(u64 q, const ulonglong2* tw, unsigned char* B, ulonglong2* D) {
  u64 M1[16][16], M2[16][16][16];  // M2[beta][k][j]
  for (int j = 0; j < 16; ++j) {
    std::vector<u64> x(256, 0);
    x[16 * j] = 1;
    col_stages(x, tw, q, 0, 4);
    for (int k = 0; k < 16; ++k) M1[k][j] = x[16 * k];
    for (int beta = 0; beta < 16; ++beta) {
      std::vector<u64> y(256, 0);
      y[16 * beta + j] = 1;
      col_stages(y, tw, q, 4, 8);
      for (int k = 0; k < 16; ++k) M2[beta][k][j] = y[16 * beta + k];
      for (int r = 0; r < 256; ++r)
        if ((r >> 4) != beta && y[r]) return false;  // M2 must not leak across blocks
    }
  }
  for (int beta = 0; beta < 16; ++beta)
    for (int j = 0; j < 16; ++j) {
      if (M2[0][0][j] == 0) return false;
      const u64 d = mm(M2[beta][0][j], pw(M2[0][0][j], q - 2, q), q);
      for (int k = 0; k < 16; ++k)
        if (mm(M2[0][k][j], d, q) != M2[beta][k][j]) return false;
      D[beta * 16 + j] = shp(d, q);  // indexed [pass-1 output beta][pass-1 row bits r_lo]
    }
  put_b(B, M1, q);
  put_b(B + kBBytes, M2[0], q);
  return true;
}

// Inverse: block beta = r_hi first, M1[beta] = diag(e_beta) G on r_lo (output
// twist), then M2 on r_hi (shared).
bool inv_tables(u64 q, const ulonglong2* itw, unsigned char* B, ulonglong2* D) {
  u64 M1[16][16][16], M2[16][16];  // M1[beta][k][j]
  for (int j = 0; j < 16; ++j) {
    for (int beta = 0; beta < 16; ++beta) {
      std::vector<u64> y(256, 0);
      y[16 * beta + j] = 1;
      col_stages_inv(y, itw, q, 0, 4);
      for (int k = 0; k < 16; ++k) M1[beta][k][j] = y[16 * beta + k];
      for (int r = 0; r < 256; ++r)
        if ((r >> 4) != beta && y[r]) return false;
    }
    for (int r_lo : {0, 5}) {  // M2 must be the same for every r_lo
      std::vector<u64> x(256, 0);
      x[16 * j + r_lo] = 1;
      col_stages_inv(x, itw, q, 4, 8);
      for (int k = 0; k < 16; ++k) {
        if (r_lo == 0) M2[k][j] = x[16 * k];
        else if (x[16 * k + r_lo] != M2[k][j]) return false;
      }
    }
  }
  for (int beta = 0; beta < 16; ++beta)
    for (int k = 0; k < 16; ++k) {
      if (M1[0][k][0] == 0) return false;
      const u64 e = mm(M1[beta][k][0], pw(M1[0][k][0], q - 2, q), q);
      for (int j = 0; j < 16; ++j)
        if (mm(M1[0][k][j], e, q) != M1[beta][k][j]) return false;
      D[k * 16 + beta] = shp(e, q);  // indexed [pass-1 output k][pass-1 row bits beta]
    }
  put_b(B, M1[0], q);
  put_b(B + kBBytes, M2, q);
  return true;
}

}  // namespace

// Per plan prime: B = [fwd B1 | fwd B2 | inv B1 | inv B2] (4 x 16 KB, SMEM layout),
// D = [fwd twists | inv twists] (2 x 256 {d, d_shoup}).  False if any prime
// is too small for reduce_lazy or a factorisation check fails.
bool ntt_tc_tables(const u64* mod, int np, const ulonglong2* tw_host, const ulonglong2* itw_host,
                   long long n, std::vector<unsigned char>& B, std::vector<ulonglong2>& D) {
  B.assign((size_t)np * 4 * kBBytes, 0);
  D.assign((size_t)np * 512, make_ulonglong2(0, 0));
  for (int pi = 0; pi < np; ++pi) {
    const u64 q = mod[pi];
    if ((double)q < 796131459065721.0) return false;  // reduce_lazy needs p > 2^49.5
    if (!fwd_tables(q, tw_host + (size_t)pi * n, B.data() + (size_t)pi * 4 * kBBytes,
                    D.data() + (size_t)pi * 512))
      return false;
    if (!inv_tables(q, itw_host + (size_t)pi * n, B.data() + ((size_t)pi * 4 + 2) * kBBytes,
                    D.data() + (size_t)pi * 512 + 256))
      return false;
  }
  return true;
}

// Column phase on the tensor cores (P1 = 8 only); -1 if not applicable.
int launch_ntt_col_tc(const NttArgs& a, int jobs, int batch, bool inverse, cudaStream_t st) {
  if (!a.tcB || !a.tcD) return -1;
  switch (a.logn * 2 + (int)inverse) {
    case 32: return launch_t<8, false>(a, jobs, batch, st);
    case 33: return launch_t<8, true>(a, jobs, batch, st);
    case 34: return launch_t<9, false>(a, jobs, batch, st);
    case 35: return launch_t<9, true>(a, jobs, batch, st);
    default: return -1;
  }
}

}  // namespace ck
