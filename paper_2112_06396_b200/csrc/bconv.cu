// RNS fast basis conversion (ModUp) and centered conversion (ModDown).
//
// Reference: rnspoly.bc_convert (rnspoly.py:264-284) and
// bc_convert_centered (rnspoly.py:303-331).
//
//   v_i   = x_i * ihat_i mod q_i                (optionally pre-folded into the INTT)
//   y_j   = sum_i v_i * T_ij  mod p_j           (T_ij = Q/q_i mod p_j)
//   k     = rint( ((0 + fl(v_0) w_0) + fl(v_1) w_1) + ... )   w_i = 1.0/q_i
//   y_j  -= k * Q mod p_j                        (centered only)
//
// The sum is an exact integer reduced mod p_j, so any exact accumulation
// matches the reference.  It is a small modular contraction on CUDA cores
// (IMAD.WIDE is half-rate on sm_100, 32-bit IMAD full rate; measured in
// profiles/r01_microbench_int.txt), arranged to need only TWO 64-bit
// accumulators and one 2-step reduction per (coefficient, target):
//   v = v0 + v1 2^30 (30-bit pieces), T = t0 + t1 2^30, U = T 2^30 mod p = u0 + u1 2^30
//   v T == (v0 t0 + v1 u0) + (v0 t1 + v1 u1) 2^30   (mod p)
// Each 30x30-bit partial product is < 2^60, so up to 8 sources (16 partials
// per accumulator) accumulate without overflow; more sources are chunked.
// The float estimate replicates numpy's op order with explicit _rn
// intrinsics (no FMA contraction), round-half-even via rint().
#include <cstdlib>
#include "ck_internal.h"
#include "tc5.cuh"

#include <algorithm>

namespace ck {

constexpr int kBcThreads = 128;
constexpr int kBcCpt = 2;  // coefficients per thread

struct BcDst {
  u64 p, bar, c30, c30p;
};


template <int NS>
__global__ void __launch_bounds__(kBcThreads, 8) bconv_kernel(const __grid_constant__ BconvGroups G) {
  const BconvArgs& a = G.g[blockIdx.y];
  extern __shared__ __align__(16) unsigned char bc_smem[];
  const int nd = a.nd;
  uint4* Ts = (uint4*)bc_smem;                         // [NS][nd]
  BcDst* Ds = (BcDst*)(Ts + NS * nd);                  // [nd]
  u64* kQs = (u64*)(Ds + nd);                          // [nd][ns+1] (centered)
  const int ns = a.ns;                                 // <= NS; rows >= ns are zero
  for (int i = threadIdx.x; i < NS * nd; i += blockDim.x)
    Ts[i] = i < ns * nd ? a.T[i] : make_uint4(0, 0, 0, 0);
  for (int j = threadIdx.x; j < nd; j += blockDim.x) {
    const PrimeConst& P = a.pc[a.dst_prime[j]];
    Ds[j] = BcDst{P.q, P.bar, P.c30, P.c30p};
  }
  if (a.centered)
    for (int i = threadIdx.x; i < nd * (ns + 1); i += blockDim.x) kQs[i] = a.kQ[i];
  __syncthreads();

  const int n = 1 << a.logn;
  const int k0 = blockIdx.x * (kBcThreads * kBcCpt) + threadIdx.x;
  const u64* in = a.in + (long long)blockIdx.z * a.in_batch;
  u64* out = a.out + (long long)blockIdx.z * a.out_batch;

  u32 v0[kBcCpt][NS], v1[kBcCpt][NS];
  u32 kk[kBcCpt];
#pragma unroll
  for (int c = 0; c < kBcCpt; ++c) {
    const int k = k0 + c * kBcThreads;
    double est = 0.0;
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      u64 v = 0;
      if (i < ns) {
        const long long off = a.in_off ? a.in_off[i] : ((long long)i << a.logn);
        v = k < n ? in[off + k] : 0;
        if (a.src_scale) {
          const ulonglong2 s = a.src_scale[i];
          v = shoup(v, s.x, s.y, a.pc[a.src_prime[i]].q);
        }
        if (a.centered) est = __dadd_rn(est, __dmul_rn(__ull2double_rn(v), a.w[i]));
      }
      v0[c][i] = lo30(v);
      v1[c][i] = hi30(v);
    }
    kk[c] = a.centered ? (u32)rint(est) : 0u;
  }

  for (int j = 0; j < nd; ++j) {
    const BcDst D = Ds[j];
    u64 y[kBcCpt], lo[kBcCpt], hi[kBcCpt];
#pragma unroll
    for (int c = 0; c < kBcCpt; ++c) y[c] = lo[c] = hi[c] = 0;
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      const uint4 t = Ts[i * nd + j];
#pragma unroll
      for (int c = 0; c < kBcCpt; ++c) {
        lo[c] = madw(v0[c][i], t.x, lo[c]);
        lo[c] = madw(v1[c][i], t.z, lo[c]);
        hi[c] = madw(v0[c][i], t.y, hi[c]);
        hi[c] = madw(v1[c][i], t.w, hi[c]);
      }
      if ((i & 7) == 7 || i == NS - 1) {  // chunk of <= 8 sources: reduce
#pragma unroll
        for (int c = 0; c < kBcCpt; ++c) {
          // lo + hi 2^30 mod p, each piece lazily in [0, 2p)
          u64 r = (lo[c] - mulhi64(lo[c], D.bar) * D.p) + shoup_lazy(hi[c], D.c30, D.c30p, D.p);
          r = csub(r, 2 * D.p);
          r = csub(r, D.p);
          y[c] = i < 8 ? r : addmod(y[c], r, D.p);
          lo[c] = hi[c] = 0;
        }
      }
    }
    const long long off = a.out_off ? a.out_off[j] : ((long long)j << a.logn);
#pragma unroll
    for (int c = 0; c < kBcCpt; ++c) {
      const int k = k0 + c * kBcThreads;
      u64 r = y[c];
      if (a.centered) r = submod(r, kQs[j * (ns + 1) + kk[c]], D.p);
      if (k < n) out[off + k] = r;
    }
  }
}

template <int NS>
static void launch_ns(const BconvGroups& G, int ng, int batch, cudaStream_t st) {
  const int n = 1 << G.g[0].logn;
  const int per = kBcThreads * kBcCpt;
  const dim3 grid((n + per - 1) / per, ng, batch);
  size_t smem = 0;
  for (int i = 0; i < ng; ++i) {
    const BconvArgs& a = G.g[i];
    const size_t s = (size_t)NS * a.nd * sizeof(uint4) + a.nd * sizeof(BcDst) +
                     (a.centered ? (size_t)a.nd * (a.ns + 1) * sizeof(u64) : 0);
    smem = s > smem ? s : smem;
  }
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(bconv_kernel<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bconv_kernel<NS><<<grid, kBcThreads, smem, st>>>(G);
}


// ---------------------------------------------------------------------------
// Tensor-core form (default for rings of at least 128 coefficients).  The contraction
// is exact integer arithmetic, so it runs byte-sliced on the 5th-generation tensor
// cores (tcgen05.mma kind::i8, accumulators in TMEM) instead of the IMAD pipe that
// bounds the rest of the key-switch:
//   x_i        = sum_a x_ia 2^{8a}                 (little-endian bytes, a < 8)
//   T'_{iaj}   = T_ij 2^{8a} mod p_j = sum_b T'_{iajb} 2^{8b}
//   S_jb       = sum_{i,a} x_ia T'_{iajb}          (< 128 * 255^2 < 2^23)
//   y_j       == sum_b S_jb 2^{8b}   (mod p_j)
// Epilogue per (coefficient, target): V = sum_b S_jb 2^{8b} < 2^80; an integer quotient
// W = floor(V / 2^sh) < 2^32 (V/p < 2^31 is checked at plan time), qh = floor(W m / 2^32)
// with m = floor(2^(sh+32) / p) undershoots V/p by less than 3 (dropped low bits of V:
// < 2^sh/p <= 1; m's floor; qh's floor), so V - qh p is in [0, 3p).
//   A = [128 coefficients][Kp bytes]: byte a of source i at k = 8 i + a -- the u64
//       residues themselves, copied by 8-byte cp.async into the canonical K-major
//       operand layout (no repacking); Kp = 8 ns rounded up to the 32-byte K step.
//   B = [N = 8 NC rows (target jj, plane b)][Kp]: byte b of T_ij 2^(8a) mod p_j for
//       a chunk of NC <= 16 targets (tcgen05.mma M128, N = 8 NC, K32 steps).
//   D = 128 TMEM lanes (coefficients) x N columns of s32 planes.
// Epilogue: thread = coefficient (TMEM lane); per target the 8 planes are
// assembled on the ALU pipe (tc5::assemble_planes), reduced with that integer
// quotient, corrected by k Q (centered), and stored -- a warp writes 256
// contiguous bytes of one target row.
// One CTA per SM = 4 independent 4-warp pipelines (own double-buffered A operand,
// own 128 TMEM columns and mbarrier), sharing B and the per-target constants; a
// pipeline walks its tiles, the next tile's sources streaming in during the
// epilogues; warp w of a pipeline owns TMEM lanes 32 w .. 32 w + 31.
#ifndef CKB200_T5_GW
#define CKB200_T5_GW 4
#endif
// warps per pipeline: 4 (one per TMEM lane quarter, up to 128 registers; measured 10.50 vs 10.68 ms per C3 step against 8 = two per quarter at 64 registers)
#ifndef CKB200_T5_GROUPS
#define CKB200_T5_GROUPS 4
#endif
constexpr int kT5Groups = CKB200_T5_GROUPS, kT5GW = CKB200_T5_GW, kT5Threads = 32 * kT5GW * kT5Groups;
constexpr int kT5ColStride = (512 / kT5Groups) & ~31;  // TMEM columns per pipeline
constexpr int kT5Halves = kT5GW / 4;
constexpr int kT5Rows = 128;
#ifndef CKB200_T5_TILES
#define CKB200_T5_TILES 64
#endif
// tiles per CTA (B and the constants are loaded once per CTA): 64 for large batches (10.18 vs
// 10.23 ms per C3 step against 32), fewer
// when the launch would otherwise not fill the GPU (a single N = 2^12 key-switch)
constexpr int kT5Tiles = CKB200_T5_TILES;

struct T5Shape {
  int kp, nc, nchunk;
};
__host__ __device__ inline T5Shape t5_shape(int ns, int nd) {
  T5Shape s;
  s.kp = ((8 * ns + 31) / 32) * 32;
  s.nchunk = (nd + 15) / 16;
  s.nc = (nd + s.nchunk - 1) / s.nchunk;
  s.nc = (s.nc + 3) & ~3;                 // N = 8 nc a multiple of 32: each half of a chunk is whole pairs
  return s;
}
size_t bconv_t5_table_bytes(int ns, int nd) {
  const T5Shape s = t5_shape(ns, nd);
  return (size_t)s.nchunk * 8 * s.nc * s.kp;
}
// Host: B5[chunk][n = 8 jj + b][k = 8 i + a] in operand layout; Tp[(i*8 + a)*nd + j] =
// T_ij 2^(8a) mod p_j.
void bconv_t5_table(const u64* Tp, int ns, int nd, unsigned char* B5) {
  const T5Shape s = t5_shape(ns, nd);
  for (int c = 0; c < s.nchunk; ++c)
    for (int jj = 0; jj < s.nc; ++jj)
      for (int b = 0; b < 8; ++b)
        for (int k = 0; k < s.kp; ++k) {
          const int j = c * s.nc + jj, i = k >> 3, a = k & 7;
          unsigned char v = 0;
          if (j < nd && i < ns) v = (unsigned char)(Tp[((size_t)i * 8 + a) * nd + j] >> (8 * b));
          B5[(size_t)c * 8 * s.nc * s.kp + tc5::kmaj_off(8 * jj + b, k, s.kp)] = v;
        }
}

template <int NT>
struct T5Ld;
template <>
struct T5Ld<4> {
  uint32_t v[32];
  __device__ __forceinline__ void ld(uint32_t t) { tc5::tmem_ld32(t, v); }
};
template <>
struct T5Ld<2> {
  uint32_t v[16];
  __device__ __forceinline__ void ld(uint32_t t) { tc5::tmem_ld16(t, v); }
};

struct T5Target {
  u64 p, np;     // p_j and 2^64 - p_j
  u32 m;         // floor(2^(sh+32) / p)
  int sh;        // floor(log2 p) - 32: funnel-shift amount of the quotient window
  long long off; // element offset of the target row
};
// NT targets starting at j0 for this thread's coefficient: orow = out + coefficient,
// pmk = (p_j - k Q mod p_j) for this coefficient's k (centered; else nullptr).
// V - qh p lies in [0, 3p) (integer quotient, see above), plus p - kQ: [0, 4p);
// lazy outputs stop there (the forward NTT takes them), else two conditional subtractions.
template <int NT>
__device__ __forceinline__ void t5_targets(const uint32_t* v, int j0, int nd, const T5Target* tg,
                                           const u64* pmk, u64* orow, bool lazy) {
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const int j = min(j0 + u, nd - 1);   // padding targets recompute the last one (not stored)
    const T5Target T = tg[j];
    u32 lo, hi, top;
    tc5::assemble_planes(v + 8 * u, lo, hi, top);
    const u32 qh = __umulhi(__funnelshift_r(hi, top, T.sh), T.m);
    u64 r = (((u64)hi << 32) | lo) + (u64)qh * T.np;
    if (pmk) r += pmk[j];
    if (!lazy) r = csub(csub(r, 2 * T.p), T.p);
    if (j0 + u < nd) orow[T.off] = r;
  }
}
template <int NT>
__device__ __forceinline__ void t5_epilogue(uint32_t taddr, int j0, int nd, const T5Target* tg,
                                            const u64* pmk, u64* orow, bool lazy) {
  T5Ld<NT> L;
  L.ld(taddr);
  tc5::tmem_wait_ld();
  t5_targets<NT>(L.v, j0, nd, tg, pmk, orow, lazy);
}

__global__ void __launch_bounds__(kT5Threads, 1) bconv_t5_kernel(const __grid_constant__ BconvGroups G) {
  pdl_trigger();
  const BconvArgs& a = G.g[blockIdx.y];
  extern __shared__ __align__(1024) unsigned char t5sm[];
  const int nd = a.nd, ns = a.ns;
  const T5Shape sh = t5_shape(ns, nd);
  const int kp = sh.kp, nc = sh.nc, ncols = 8 * nc;
  const int abytes = kT5Rows * kp;                          // one A operand
  unsigned char* Bm = t5sm + 2 * kT5Groups * abytes;        // B5 chunks
  T5Target* tg = (T5Target*)(Bm + (size_t)sh.nchunk * ncols * kp);
  u64* kQs = (u64*)(tg + nd);                               // [ns + 1][nd]: p_j - k Q mod p_j
  unsigned char* kk = (unsigned char*)(kQs + (a.centered ? nd * (ns + 1) : 0));  // [groups][128]
  uint64_t* mbar = (uint64_t*)(((uintptr_t)(kk + kT5Groups * kT5Rows) + 7) & ~(uintptr_t)7);
  uint32_t* tslot = (uint32_t*)(mbar + kT5Groups);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = warp / kT5GW, gw = warp % kT5GW, gtid = tid % (32 * kT5GW);
  const int quarter = gw & 3, half = gw >> 2;  // half < kT5Halves
  const int n = 1 << a.logn;
  const int ntiles = n / kT5Rows;
  const int t0 = blockIdx.x * G.tiles_per_cta;
  const int t1 = min(t0 + G.tiles_per_cta, ntiles);
  const u64* in = a.in + (long long)blockIdx.z * a.in_batch;
  u64* out = a.out + (long long)blockIdx.z * a.out_batch;
  const unsigned mb_s = tc5::saddr(mbar + grp);
  unsigned char* abuf = t5sm + grp * 2 * abytes;
  const unsigned abuf_s = tc5::saddr(abuf);
  const unsigned b_s = tc5::saddr(Bm);
  const int bar_id = 1 + grp;
  auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "n"(32 * kT5GW) : "memory"); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        tc5::saddr(tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (gtid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb_s));
  // plan tables (not the predecessor's output): before the PDL wait
  {
    const uint4* src = (const uint4*)a.B5;
    uint4* dst = (uint4*)Bm;
    for (int i = tid; i < sh.nchunk * ncols * kp / 16; i += blockDim.x) dst[i] = src[i];
    for (int j = tid; j < nd; j += blockDim.x) {
      const u64 p = a.pc[a.dst_prime[j]].q;
      const int s = 63 - __clzll((long long)p);
      const u32 m = (u32)(((unsigned __int128)1 << (s + 32)) / p);
      tg[j] = T5Target{p, 0 - p, m, s - 32, a.out_off ? a.out_off[j] : ((long long)j << a.logn)};
    }
    if (a.centered)
      for (int i = tid; i < nd * (ns + 1); i += blockDim.x) {
        const int j = i / (ns + 1), k = i % (ns + 1);
        kQs[k * nd + j] = a.pc[a.dst_prime[j]].q - a.kQ[i];
      }
    // zero the padding source columns of this group's two A buffers once
    if (kp > 8 * ns) {
      const int padw = (kp - 8 * ns) / 8;
      for (int e = gtid; e < 2 * kT5Rows * padw; e += 32 * kT5GW) {
        const int bsel = e / (kT5Rows * padw), rem = e % (kT5Rows * padw);
        const int r = rem % kT5Rows, i = ns + rem / kT5Rows;
        *(u64*)(abuf + bsel * abytes + tc5::kmaj_off(r, 8 * i, kp)) = 0;
      }
    }
  }
  // tile staging: 128 coefficients x ns sources, 8-byte cp.async straight into operand
  // layout.  Thread -> coefficient r = gtid % 128 and sources i = gtid / 128 + 2 k: the
  // destination advances by one 128-byte core matrix per k, the source by 2 N elements.
  constexpr int kIs = kT5Halves;  // sources a thread steps over (threads per pipeline / 128)
  const int st_r = gtid & (kT5Rows - 1), st_i0 = gtid >> 7;
  const unsigned st_dst0 = tc5::kmaj_off(st_r, 0, kp);
  const u64* st_src0 = in + ((long long)st_i0 << a.logn) + st_r;
  const long long st_step = (long long)kIs << a.logn;
  auto stage = [&](int tile, int bsel) {
    const unsigned dst = abuf_s + bsel * abytes + st_dst0;
    const u64* src = st_src0 + (long long)tile * kT5Rows;
#pragma unroll 1
    for (int i = st_i0; i < ns; i += kIs, src += st_step)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + ((i >> 1) << 7) + ((i & 1) << 3)),
                   "l"(src) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  pdl_wait();  // the sources are the predecessor's output
  if (t0 + grp < t1) stage(t0 + grp, 0);
  // every thread wrote part of B (and the operand padding) with ordinary stores; the MMAs
  // read them through the async proxy: fence in the WRITING threads, before the barrier
  tc5::fence_async_smem();
  tc5::fence_before();
  __syncthreads();
  tc5::fence_after();
  const uint32_t tacc = *tslot + grp * kT5ColStride;
  const uint32_t tl = tacc + ((uint32_t)(quarter * 32) << 16);
  const int m = quarter * 32 + lane;          // this thread's coefficient within the tile
  const uint32_t idesc = tc5::idesc_i8(ncols);
  unsigned phase = 0;
  const bool lazy = a.lazy_out != 0;

  for (int it = 0; t0 + grp + kT5Groups * it < t1; ++it) {
    const int tile = t0 + grp + kT5Groups * it;
    unsigned char* A = abuf + (it & 1) * abytes;
    const unsigned a_s = abuf_s + (it & 1) * abytes;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    gsync();  // the tile is complete (every thread's copies), the other buffer is free
    if (tile + kT5Groups < t1) stage(tile + kT5Groups, (it + 1) & 1);
    if (a.src_scale) {
      for (int e = gtid; e < kT5Rows * ns; e += 32 * kT5GW) {
        const int i = e / kT5Rows, r = e % kT5Rows;
        const ulonglong2 sc = a.src_scale[i];
        u64* px = (u64*)(A + tc5::kmaj_off(r, 8 * i, kp));
        *px = shoup(*px, sc.x, sc.y, a.pc[a.src_prime[i]].q);
      }
      gsync();
    }
    if (a.centered) {
      // k = rint(sum_i fl(v_i) w_i) in the reference's op order (rnspoly.py:320-325)
      if (gtid < kT5Rows) {
        double est = 0.0;
        for (int i = 0; i < ns; ++i)
          est = __dadd_rn(est, __dmul_rn(__ull2double_rn(*(const u64*)(A + tc5::kmaj_off(gtid, 8 * i, kp))), a.w[i]));
        kk[grp * kT5Rows + gtid] = (unsigned char)rint(est);
      }
    }
    tc5::fence_async_smem();
    tc5::fence_before();
    gsync();
    tc5::fence_after();
    u64* orow = out + (long long)tile * kT5Rows + m;
    const u64* pmk = a.centered ? kQs + (int)kk[grp * kT5Rows + m] * nd : nullptr;
    for (int c = 0; c < sh.nchunk; ++c) {
      if (gtid == 0) {
        for (int s = 0; s < kp / 32; ++s)
          tc5::mma_i8(tacc, tc5::smem_desc(a_s + s * 256, kp),
                      tc5::smem_desc(b_s + c * ncols * kp + s * 256, kp), idesc, s > 0);
        tc5::mma_commit(mb_s);
      }
      tc5::mbar_wait(mb_s, phase);
      phase ^= 1;
      tc5::fence_after();
      // this warp's targets of the chunk: [half * nc/2 ...) in steps of 4 / 2
      const int jh = nc / kT5Halves;               // targets per warp (a multiple of 2)
      const int jb = c * nc + half * jh;           // first global target
      const uint32_t tcol = tl + half * jh * 8;
      int u = 0;
      // (double-buffered TMEM loads, as in the NTT column kernel, were measured here too:
      // 127 registers, 10.06 vs 9.99 ms per C3 step -- not kept)
#pragma unroll 1
      for (; u + 4 <= jh; u += 4) t5_epilogue<4>(tcol + 8 * u, jb + u, nd, tg, pmk, orow, lazy);
      if (u < jh) t5_epilogue<2>(tcol + 8 * u, jb + u, nd, tg, pmk, orow, lazy);  // nc % 4 == 0: jh is even
      tc5::fence_before();
      gsync();  // every warp has read D before the next MMA rewrites it
      tc5::fence_after();
    }
  }
  __syncthreads();
  if (warp == 0) {
    tc5::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tslot), "n"(512));
  }
}

static size_t t5_smem(const BconvArgs& a) {
  const T5Shape s = t5_shape(a.ns, a.nd);
  return (size_t)2 * kT5Groups * kT5Rows * s.kp + (size_t)s.nchunk * 8 * s.nc * s.kp +
         (size_t)a.nd * sizeof(T5Target) + (a.centered ? (size_t)a.nd * (a.ns + 1) * 8 : 0) +
         kT5Groups * kT5Rows + 8 + kT5Groups * 8 + 16;
}
static bool t5_ok(const BconvArgs& a) {
  return a.B5 != nullptr && a.in_off == nullptr && a.logn >= 7 && a.ns <= 16 && a.nd <= 64 &&
         8 * t5_shape(a.ns, a.nd).nc <= kT5ColStride && t5_smem(a) <= 200 * 1024;
}
static void launch_t5(BconvGroups& G, int ng, int batch, cudaStream_t st) {
  const int n = 1 << G.g[0].logn;
  const int tiles = n / kT5Rows;
  // at least ~2 CTAs per SM when the work allows, never below one tile per pipeline
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long total = (long long)tiles * ng * batch;
  int tpc = (int)std::min<long long>(kT5Tiles, std::max<long long>(kT5Groups, total / (2 * sms)));
  tpc = std::max(kT5Groups, (tpc / kT5Groups) * kT5Groups);
  // Small launches (one ciphertext, hoisted batches of a few): the kernel runs ONE CTA per SM
  // (TMEM and shared memory), so the grid is sized in whole waves -- pick the tiles per CTA
  // that minimise waves x (prologue + iterations), a CTA's prologue (TMEM allocation, B table)
  // costing about two tile iterations.  CKB200_T5_WAVES=0 keeps the plain rule (measurements).
  static const int wave_rule = [] {
    const char* e = getenv("CKB200_T5_WAVES");
    return e ? atoi(e) : 1;
  }();
  if (wave_rule && total < 4LL * kT5Tiles * sms) {
    long long best = -1;
    for (int c = kT5Groups; c <= kT5Tiles; c += kT5Groups) {
      const long long ctas = (long long)((tiles + c - 1) / c) * ng * batch;
      const long long cost = ((ctas + sms - 1) / sms) * (2 + c / kT5Groups);
      if (best < 0 || cost < best) {
        best = cost;
        tpc = c;
      }
    }
  }
  G.tiles_per_cta = tpc;
  size_t smem = 0;
  for (int i = 0; i < ng; ++i) smem = std::max(smem, t5_smem(G.g[i]));
  static unsigned done = 0;  // per-device shared-memory opt-in
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 32 || !((done >> dev) & 1u)) {
    cudaFuncSetAttribute(bconv_t5_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (dev < 32) __atomic_fetch_or(&done, 1u << dev, __ATOMIC_RELAXED);
  }
  const dim3 grid((tiles + tpc - 1) / tpc, ng, batch);
  launch_pdl(bconv_t5_kernel, grid, dim3(kT5Threads), smem, st, G);
}

int launch_bconv_groups(const BconvArgs* gs, int ng, int batch, cudaStream_t st) {
  if (ng <= 0 || batch <= 0) return 0;
  if (ng > kMaxBcGroups) return CK_ERR_ARG;
  BconvGroups G;
  G.tiles_per_cta = 0;
  int ns = 0;
  for (int i = 0; i < ng; ++i) {
    if (gs[i].nd <= 0 || gs[i].ns < 1) return CK_ERR_ARG;
    G.g[i] = gs[i];
    ns = gs[i].ns > ns ? gs[i].ns : ns;
  }
  count_launches(1);
  bool t5 = true;
  for (int i = 0; i < ng; ++i) t5 = t5 && t5_ok(gs[i]);
  if (t5) {
    launch_t5(G, ng, batch, st);
    return (int)cudaGetLastError();
  }
  // smallest compiled source count >= ns (extra source rows are zero)
  if (ns <= 1) launch_ns<1>(G, ng, batch, st);
  else if (ns <= 2) launch_ns<2>(G, ng, batch, st);
  else if (ns <= 4) launch_ns<4>(G, ng, batch, st);
  else if (ns <= 8) launch_ns<8>(G, ng, batch, st);
  else if (ns <= 9) launch_ns<9>(G, ng, batch, st);
  else if (ns <= 10) launch_ns<10>(G, ng, batch, st);
  else if (ns <= 12) launch_ns<12>(G, ng, batch, st);
  else if (ns <= 16) launch_ns<16>(G, ng, batch, st);
  else if (ns <= 24) launch_ns<24>(G, ng, batch, st);
  else if (ns <= 32) launch_ns<32>(G, ng, batch, st);
  else if (ns <= 48) launch_ns<48>(G, ng, batch, st);
  else return CK_ERR_ARG;
  return (int)cudaGetLastError();
}

int launch_bconv(const BconvArgs& a, int batch, cudaStream_t st) {
  if (a.nd <= 0 || batch <= 0) return 0;
  return launch_bconv_groups(&a, 1, batch, st);
}

}  // namespace ck
