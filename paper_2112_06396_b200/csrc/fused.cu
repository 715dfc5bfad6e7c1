// Fused key-switch row kernels (the NTT's row phase + what follows it).
//
// ks_row_kernel: for raised limb i and a tile of storage rows r
//   digit_d[i][r, :] = automorph( NTT_row( ModUp target row ) )   (or the
//                      input a_eval row for the digit's own limbs,
//                      ckks.py:433-440)
//   u[i][r, :] = sum_d digit_d * key_a[d][row_i],  v likewise      (_kskip,
//                      ckks.py:450-465, on automorph'ed digits, ckks.py:663)
//   special limbs (i >= l): optionally run the INTT row phase on u, v right
//   away -- the first half of ModDown's INTT (ckks.py:409).
// The digits never touch HBM in evaluation form.  The automorphism maps a
// storage row r to a single source row sigma(r) (see kskip.cu), so each CTA
// loads whole source rows and gathers within shared memory.
//
// md_row_kernel: ModDown epilogue fused with the forward NTT row phase of the
//   converted polynomial (ckks.py:410-416, 664-666):
//   out[j][r, :] = (x[j][r, :] - NTT_row(conv[j])[r, :]) * P^-1 [+ automorph(b)]
#include "ck_internal.h"
#include "ntt.cuh"

#include <algorithm>
#include <atomic>

namespace ck {

template <int P2, int EPC = 2048>
struct FusedCfg {
  static constexpr int S = 1 << P2;
  static constexpr int G = S / kE;         // threads per row
  static constexpr int TR = EPC / S;       // rows per CTA (EPC elements)
  static constexpr int NT = TR * G;        // EPC / 16 threads
  static constexpr int RS = row_stride<P2>();
};
#ifndef CKB200_MD_EPC
#define CKB200_MD_EPC 2048
#endif
#ifndef CKB200_KS_EPC
#define CKB200_KS_EPC 1024
#endif
#ifndef CKB200_KS_MINB
#define CKB200_KS_MINB 6
#endif
// CKB200_KS_RING = S > 0: the key tiles reach shared memory through a ring of S
// stages of TMA bulk copies (one stage = one MAC iteration's 2*BETA key segments),
// the first S issued at kernel start so they land during the digit NTTs
#ifndef CKB200_KS_RING
#define CKB200_KS_RING 1
#endif
#ifndef CKB200_KS_EARLY
#define CKB200_KS_EARLY 1
#endif
// ks_row elements per CTA (1024: 64 threads; with a 1-stage key ring that is refilled as soon
// as the key words are in registers 32 KB of SMEM, 6 CTAs/SM: 10.35 ms per C3 step against
// 10.48 for the 2-stage ring at 5 CTAs/SM and 10.65 for 3 stages at 4; DESIGN sections 10-11)
constexpr int kKsEpc = CKB200_KS_EPC;

// Forward row phase of one digit tile in shared memory (natural order in and
// out).  Not inlined (CKB200_KS_NOINLINE, default 1): ONE copy of this code per kernel instead
// of one per digit: ks_row_kernel<8,8,3> is ~140 KB of SASS, above the SM's
// instruction cache (no_instruction stalls; measured +1.3% with the call).
#ifndef CKB200_KS_NOINLINE
#define CKB200_KS_NOINLINE 1
#endif
#if CKB200_KS_NOINLINE
#define CK_KS_DIGIT_INLINE __noinline__
#else
#define CK_KS_DIGIT_INLINE __forceinline__
#endif
template <int P2, int LOGN>
__device__ CK_KS_DIGIT_INLINE void ks_digit_ntt(u64* srow, int g, int sr, const ulonglong2* tw,
                                                u64 q, u64 two_q, bool canon) {
  u64 x[kE];
  row_from_smem<P2, 0, false>(x, g, srow);
  row_transform<P2, false, LOGN>(x, g, sr << P2, srow, tw, q, two_q);
  // the 30-bit-split MAC only needs digits < 2^61 (three products of a value below 2^61 and a
  // residue accumulate without overflow, their sum stays below 2^64 2^sh for the Barrett step):
  // for q < 2^56 the lazy range [0, 16q) already is; larger (special) primes are folded to
  // [0, 2q), and to [0, q) for callers that need canonical values (md_row's exact epilogue)
  if (q >= (1ull << 56)) {
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      u64 v = csub(x[k], q << 3);
      v = csub(v, q << 2);
      v = csub(v, q << 1);
      x[k] = canon ? csub(v, q) : v;
    }
  }
  __syncthreads();
  row_to_smem<P2, RowLast<P2>::value, false>(x, g, srow);
}
// Primes below 2^54 (small_prime): approximate-quotient butterflies, no folding;
// inputs below 16q, outputs below (16 + 4 P2) q < 2^60.
template <int P2, int LOGN>
__device__ CK_KS_DIGIT_INLINE void ks_digit_ntt_small(u64* srow, int g, int sr,
                                                      const ulonglong2* tw, u64 q) {
  u64 x[kE];
  row_from_smem<P2, 0, false>(x, g, srow);
  row_transform<P2, false, LOGN, SyncCta, true>(x, g, sr << P2, srow, tw, neg_opaque(q), q << 2);
  __syncthreads();
  row_to_smem<P2, RowLast<P2>::value, false>(x, g, srow);
}
#ifndef CKB200_SMALLQ
#define CKB200_SMALLQ 1
#endif
template <int P2, int LOGN>
CK_D void ks_digit_ntt_any(u64* srow, int g, int sr, const ulonglong2* tw, u64 q, u64 two_q,
                           bool canon) {
  if (CKB200_SMALLQ && small_prime(q)) ks_digit_ntt_small<P2, LOGN>(srow, g, sr, tw, q);
  else ks_digit_ntt<P2, LOGN>(srow, g, sr, tw, q, two_q, canon);
}

// KSKIP output: canonical, or [0, 3q) where the consumer takes lazy values
CK_D u64 ks_out(const Acc3& s, const PrimeConst& P, bool lazy) {
  const u64 r = acc3_reduce_lazy(s, P);
  return lazy ? r : csub(csub(r, P.two_q), P.q);
}

// ---------------------------------------------------------------- KSKIP row
// BETA > 0: compile-time digit count (fully unrolled inner product, so the
// 2*BETA key loads of an element are independent and stay in flight);
// BETA == 0: runtime a.beta (generic fallback).
//
// Shared memory: one padded row-tile slot per digit.  Slot d is digit d's
// NTT exchange buffer and then holds its natural-order row, so the
// automorphism gather happens at MAC time (one permutation index per element,
// shared by all digits) -- no separate staging buffer.
template <int P1, int P2, int BETA>
__global__ void __launch_bounds__(FusedCfg<P2, kKsEpc>::NT, CKB200_KS_MINB) ks_row_kernel(KsRowArgs a) {
  using F = FusedCfg<P2, kKsEpc>;
  constexpr int LOGN = P1 + P2;
  constexpr int SLOT = F::TR * F::RS;
  extern __shared__ __align__(16) u64 fsm[];
  pdl_trigger();
  const int i = blockIdx.z + a.row0;   // grid (row tile, batch, limb): twiddle reuse across the batch
  const long long b = blockIdx.y;
  const int prime = a.prime[i];
  const PrimeConst& Pg = a.pc[prime];
  const u64 q = Pg.q, two_q = Pg.two_q;
  const int rl = threadIdx.x / F::G, g = threadIdx.x % F::G;
  const int r = blockIdx.x * F::TR + rl;
  const u64 t = a.galois ? a.galois[b] : a.galois_t;
  const int sr = t == 1 ? r : (int)(automorph_src((u32)r << P2, (u32)t, LOGN) >> P2);
  const ulonglong2* tw = a.tw + ((long long)prime << LOGN);
  constexpr int NB = BETA > 0 ? BETA : 8;
  const int beta = BETA > 0 ? BETA : a.beta;
  constexpr int NSK = BETA > 0 ? CKB200_KS_RING : 0;
  constexpr int SEG = 2 * F::NT;                          // words per key segment (one iteration)
  u64* ring = fsm + (BETA > 0 ? BETA : 0) * SLOT;         // [NSK][2 BETA][SEG]
  uint64_t* kbar = (uint64_t*)(ring + NSK * 2 * (BETA > 0 ? BETA : 1) * SEG);
  const long long ktile0 = (long long)blockIdx.x * F::TR << P2;
  const u64* kta = key_block(a.key_a, a.key_a_ptrs, a.key_batch, b) + ((long long)prime << LOGN) + ktile0;
  const u64* ktb = key_block(a.key_b, a.key_b_ptrs, a.key_batch, b) + ((long long)prime << LOGN) + ktile0;
  auto ring_issue = [&](int m) {  // thread 0: iteration m's 2 BETA segments into slot m % NSK
    if constexpr (NSK > 0) {
      const int sl = m % NSK;
      mbar_expect_tx(&kbar[sl], (unsigned)(2 * BETA * SEG * 8));
#pragma unroll
      for (int d = 0; d < BETA; ++d) {
        bulk_g2s(ring + (sl * 2 * BETA + 2 * d) * SEG, kta + d * a.key_digit_stride + SEG * m,
                 SEG * 8, &kbar[sl]);
        bulk_g2s(ring + (sl * 2 * BETA + 2 * d + 1) * SEG, ktb + d * a.key_digit_stride + SEG * m,
                 SEG * 8, &kbar[sl]);
      }
    }
  };
  if constexpr (NSK > 0) {
    constexpr int ITER0 = (F::TR * F::S) / (2 * F::NT);
    if (threadIdx.x == 0) {
      for (int sl = 0; sl < NSK; ++sl) mbar_init(&kbar[sl], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int m = 0; m < NSK && m < ITER0; ++m) ring_issue(m);  // keys are inputs: before the PDL wait
    }
  }

  // Key tiles are only needed after the digit NTTs: start streaming them to L2
  // now (one bulk prefetch per key row-tile, contiguous TR*S words), so the
  // inner product below hits L2 instead of waiting on HBM.
  // key_prefetch = k: prefetch the first k/8 of each key row-tile (k = 8: all)
  if (NSK == 0 && a.key_prefetch && threadIdx.x < 2 * beta) {
    const int d = threadIdx.x >> 1;
    const u64* kbase = (threadIdx.x & 1) ? key_block(a.key_a, a.key_a_ptrs, a.key_batch, b)
                                         : key_block(a.key_b, a.key_b_ptrs, a.key_batch, b);
    prefetch_l2(kbase + d * a.key_digit_stride + ((long long)prime << LOGN) +
                    ((long long)blockIdx.x * F::TR << P2),
                (F::TR * F::S * 8 / 8) * min(a.key_prefetch, 8));
  }
  pdl_wait();  // digits and the ciphertext rows are the predecessors' output
  if constexpr (BETA > 0) {
    // All digits' source rows are requested up front with async copies into
    // their own slots (natural order), so the loads of digits 1.. overlap the
    // NTT of digit 0.  Each thread copies exactly the elements it will read
    // back first, so only cp.async.wait_group is needed before use.
#pragma unroll
    for (int d = 0; d < BETA; ++d) {
      const bool own = i < a.l && i >= a.lo[d] && i < a.hi[d];
      const u64* src = (own ? a.a_eval + b * a.a_batch + ((long long)i << LOGN)
                            : a.dig + b * a.dig_batch + ((long long)(d * a.R + i) << LOGN)) +
                       ((long long)sr << P2);
      u64* srow = fsm + d * SLOT + rl * F::RS;
#pragma unroll
      for (int k = 0; k < kE; ++k) {
        const int s0 = sub_index<P2, 0, false>(g, k);
        cp_async8(srow + sidx(s0), src + s0);
      }
      cp_async_commit();
    }
#pragma unroll
    for (int d = 0; d < BETA; ++d) {
      const bool own = i < a.l && i >= a.lo[d] && i < a.hi[d];
      u64* srow = fsm + d * SLOT + rl * F::RS;
      if (d == 0) cp_async_wait<BETA - 1>();
      else if (d == 1) cp_async_wait<(BETA >= 2 ? BETA - 2 : 0)>();
      else if (d == 2) cp_async_wait<(BETA >= 3 ? BETA - 3 : 0)>();
      else cp_async_wait<0>();
      if (!own) ks_digit_ntt_any<P2, LOGN>(srow, g, sr, tw, q, two_q, false);  // own rows are in place
    }
  } else {
#pragma unroll 1
  for (int d = 0; d < beta; ++d) {
    const bool own = i < a.l && i >= a.lo[d] && i < a.hi[d];
    u64* srow = fsm + d * SLOT + rl * F::RS;
    u64 x[kE];
    if (own) {
      const u64* src = a.a_eval + b * a.a_batch + ((long long)i << LOGN) + ((long long)sr << P2);
#pragma unroll
      for (int k = 0; k < kE; ++k) x[k] = src[sub_index<P2, 0, false>(g, k)];
      row_to_smem<P2, 0, false>(x, g, srow);
    } else {
      const u64* src = a.dig + b * a.dig_batch + ((long long)(d * a.R + i) << LOGN) +
                       ((long long)sr << P2);
#pragma unroll
      for (int k = 0; k < kE; ++k) x[k] = src[sub_index<P2, 0, false>(g, k)];
      row_transform<P2, false, LOGN>(x, g, sr << P2, srow, tw, q, two_q);
#pragma unroll
      for (int k = 0; k < kE; ++k) x[k] = fwd_final(x[k], q);
      __syncthreads();
      row_to_smem<P2, RowLast<P2>::value, false>(x, g, srow);
    }
  }
  }
  __syncthreads();

  // Inner product with the key rows.  MAC mapping (independent of the NTT
  // layout): thread t owns element pairs e = 2t + 2*NT*m + {0,1} of the
  // CTA's contiguous TR*S tile, so key loads / u,v stores are 16-byte
  // vectors and every warp instruction covers 512 contiguous bytes.
  // Output column c of row r reads column pi_r(c) of row sigma(r).
  // reduction constants in registers for the MAC loop only (loaded after the
  // NTTs: a reference into global memory would reload them after every store)
  const PrimeConst P = Pg;
  const bool lazy_out = i < a.lazy_keep && q < ((u64)1 << 59);  // [0, 3q) for md_row
  const long long tile0 = (long long)blockIdx.x * F::TR << P2;
  const u64* ka = key_block(a.key_a, a.key_a_ptrs, a.key_batch, b) + ((long long)prime << LOGN) + tile0;
  const u64* kb = key_block(a.key_b, a.key_b_ptrs, a.key_batch, b) + ((long long)prime << LOGN) + tile0;
  u64* ubase = a.uv + b * a.uv_batch + ((long long)i << LOGN);
  constexpr int ITER = (F::TR * F::S) / (2 * F::NT);
  if constexpr (BETA > 0 && NSK > 0) {
    // keys from the TMA ring: iteration m waits for its stage, frees it after a barrier
#pragma unroll 1
    for (int m = 0; m < ITER; ++m) {
      const int e = 2 * (int)threadIdx.x + 2 * F::NT * m;
      const int sl = m % NSK;
      mbar_wait_parity(&kbar[sl], (unsigned)((m / NSK) & 1));
      ulonglong2 ya[BETA], yb[BETA];
#pragma unroll
      for (int d = 0; d < BETA; ++d) {
        ya[d] = *(const ulonglong2*)(ring + (sl * 2 * BETA + 2 * d) * SEG + 2 * threadIdx.x);
        yb[d] = *(const ulonglong2*)(ring + (sl * 2 * BETA + 2 * d + 1) * SEG + 2 * threadIdx.x);
      }
#if CKB200_KS_EARLY
      // the stage is free as soon as every thread holds its key words in registers: refill it
      // now, so the copy has this whole iteration (MACs, reductions, stores) to land.  The
      // barrier alone does not wait for shared-memory loads still in flight, and the bulk
      // copy writes through the async proxy: the proxy fence orders this thread's reads of
      // the stage before the refill (without it the copy overtook loads: sporadic mismatches).
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0 && m + NSK < ITER) ring_issue(m + NSK);
#endif
      const int er = e >> P2, ec = e & (F::S - 1);
      const int rr = blockIdx.x * F::TR + er;
      int sc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        sc[h] = t == 1 ? ec + h
                       : (int)(automorph_src(((u32)rr << P2) + ec + h, (u32)t, LOGN) & (F::S - 1));
      Acc3 su[2], sv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        acc3_zero(su[h]);
        acc3_zero(sv[h]);
      }
#pragma unroll
      for (int d = 0; d < BETA; ++d) {
        const u64* drow = fsm + d * SLOT + er * F::RS;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const u64 x = drow[sidx(sc[h])];
          const u64 ax = h ? ya[d].y : ya[d].x, bx = h ? yb[d].y : yb[d].x;
          const u32 x0 = lo30(x), x1 = hi30(x);
          acc3_mac(su[h], x0, x1, lo30(ax), hi30(ax));
          acc3_mac(sv[h], x0, x1, lo30(bx), hi30(bx));
        }
      }
      u64* uw = ubase + tile0 + e;
      *(ulonglong2*)uw = make_ulonglong2(ks_out(su[0], P, lazy_out), ks_out(su[1], P, lazy_out));
      *(ulonglong2*)(uw + a.v_off) = make_ulonglong2(ks_out(sv[0], P, lazy_out), ks_out(sv[1], P, lazy_out));
#if !CKB200_KS_EARLY
      __syncthreads();  // every thread is done with slot sl
      if (threadIdx.x == 0 && m + NSK < ITER) ring_issue(m + NSK);
#endif
    }
  } else if constexpr (BETA > 0) {
    // software-pipelined: the key vectors of iteration m+1 are in flight while
    // iteration m multiplies (the MAC phase is otherwise load-latency bound)
    ulonglong2 ya[BETA], yb[BETA];
#pragma unroll
    for (int d = 0; d < BETA; ++d) {
      ya[d] = __ldg((const ulonglong2*)(ka + d * a.key_digit_stride + 2 * (int)threadIdx.x));
      yb[d] = __ldg((const ulonglong2*)(kb + d * a.key_digit_stride + 2 * (int)threadIdx.x));
    }
#pragma unroll 1
    for (int m = 0; m < ITER; ++m) {
      const int e = 2 * (int)threadIdx.x + 2 * F::NT * m;
      ulonglong2 na[BETA], nb[BETA];
      if (m + 1 < ITER) {
#pragma unroll
        for (int d = 0; d < BETA; ++d) {
          na[d] = __ldg((const ulonglong2*)(ka + d * a.key_digit_stride + e + 2 * F::NT));
          nb[d] = __ldg((const ulonglong2*)(kb + d * a.key_digit_stride + e + 2 * F::NT));
        }
      }
      const int er = e >> P2, ec = e & (F::S - 1);
      const int rr = blockIdx.x * F::TR + er;
      int sc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        sc[h] = t == 1 ? ec + h
                       : (int)(automorph_src(((u32)rr << P2) + ec + h, (u32)t, LOGN) & (F::S - 1));
      Acc3 su[2], sv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        acc3_zero(su[h]);
        acc3_zero(sv[h]);
      }
#pragma unroll
      for (int d = 0; d < BETA; ++d) {
        const u64* drow = fsm + d * SLOT + er * F::RS;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const u64 x = drow[sidx(sc[h])];
          const u64 ax = h ? ya[d].y : ya[d].x, bx = h ? yb[d].y : yb[d].x;
          const u32 x0 = lo30(x), x1 = hi30(x);
          acc3_mac(su[h], x0, x1, lo30(ax), hi30(ax));
          acc3_mac(sv[h], x0, x1, lo30(bx), hi30(bx));
        }
      }
      u64* uw = ubase + tile0 + e;
      *(ulonglong2*)uw = make_ulonglong2(ks_out(su[0], P, lazy_out), ks_out(su[1], P, lazy_out));
      *(ulonglong2*)(uw + a.v_off) = make_ulonglong2(ks_out(sv[0], P, lazy_out), ks_out(sv[1], P, lazy_out));
      if (m + 1 < ITER) {
#pragma unroll
        for (int d = 0; d < BETA; ++d) {
          ya[d] = na[d];
          yb[d] = nb[d];
        }
      }
    }
  } else {
#pragma unroll 2
  for (int m = 0; m < ITER; ++m) {
    const int e = 2 * (int)threadIdx.x + 2 * F::NT * m;
    const int er = e >> P2, ec = e & (F::S - 1);
    const int rr = blockIdx.x * F::TR + er;
    int sc[2];
#pragma unroll
    for (int h = 0; h < 2; ++h)
      sc[h] = t == 1 ? ec + h
                     : (int)(automorph_src(((u32)rr << P2) + ec + h, (u32)t, LOGN) & (F::S - 1));
    Acc3 su[2], sv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      acc3_zero(su[h]);
      acc3_zero(sv[h]);
    }
#pragma unroll
    for (int d = 0; d < NB; ++d) {
      if (d >= beta) break;
      const ulonglong2 ya = __ldg((const ulonglong2*)(ka + d * a.key_digit_stride + e));
      const ulonglong2 yb = __ldg((const ulonglong2*)(kb + d * a.key_digit_stride + e));
      const u64* drow = fsm + d * SLOT + er * F::RS;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const u64 x = drow[sidx(sc[h])];
        const u64 ax = h ? ya.y : ya.x, bx = h ? yb.y : yb.x;
        const u32 x0 = lo30(x), x1 = hi30(x);
        acc3_mac(su[h], x0, x1, lo30(ax), hi30(ax));
        acc3_mac(sv[h], x0, x1, lo30(bx), hi30(bx));
      }
    }
    u64* uw = ubase + tile0 + e;
    *(ulonglong2*)uw = make_ulonglong2(ks_out(su[0], P, lazy_out), ks_out(su[1], P, lazy_out));
    *(ulonglong2*)(uw + a.v_off) = make_ulonglong2(ks_out(sv[0], P, lazy_out), ks_out(sv[1], P, lazy_out));
  }
  }
}

// ------------------------------------------------------------ ModDown row
template <int P1, int P2, bool LAZY>
#ifndef CKB200_MD_MINB
#define CKB200_MD_MINB 6
#endif
#ifndef CKB200_MD_CALL
#define CKB200_MD_CALL 1
#endif
#ifndef CKB200_MD_INLINE_SMALL
#define CKB200_MD_INLINE_SMALL 1
#endif
// (also re-measured and rejected: prefetching the x / addend lines before the row NTT,
// 10.44 vs 10.41 ms)
// (the x operand staged by per-thread cp.async during the row NTT was measured again with
// the cheaper butterflies: 10.9 vs 10.43 ms per C3 step -- removed)
__global__ void __launch_bounds__(FusedCfg<P2, CKB200_MD_EPC>::NT, CKB200_MD_MINB) md_row_kernel(MdRowArgs a) {
  using F = FusedCfg<P2, CKB200_MD_EPC>;
  constexpr int LOGN = P1 + P2;
  __shared__ u64 stage[F::TR * F::RS];
  const int j = blockIdx.z;  // grid (row tile, item group, limb)
  const int prime = a.prime[j];
  const PrimeConst& P = a.pc[prime];  // (a register copy spills at 64 registers)
  const u64 q = P.q, two_q = P.two_q;
  const ulonglong2 pinv = a.pinv[j];
  const int rl = threadIdx.x / F::G, g = threadIdx.x % F::G;
  const int r = blockIdx.x * F::TR + rl;
  u64* srow = stage + rl * F::RS;
  const ulonglong2* tw = a.tw + ((long long)prime << LOGN);
  const long long ro = ((long long)j << LOGN) + ((long long)r << P2);
  pdl_trigger();
  pdl_wait();
  // a CTA runs `group` consecutive items (batch x {u, v}) of the SAME limb and
  // rows: the row twiddles come from L1 after the first item
  const int items = a.pair ? 2 * a.batch : a.batch;
  const int i_end = min(items, ((int)blockIdx.y + 1) * a.group);
#pragma unroll 1
  for (int item = blockIdx.y * a.group; item < i_end; ++item) {
  const int w = a.pair ? (item & 1) : 1;   // w = 1: the polynomial that gets the addend
  const long long b = a.pair ? (item >> 1) : item;
  const u64* conv = a.conv + b * a.conv_batch + ro + (a.pair && w ? a.conv_w : 0);
  const u64* x = a.x + b * a.x_batch + ro + (a.pair && w ? a.x_w : 0);
#if CKB200_MD_CALL
  // Small primes (every chain prime of C3/C5): the row NTT inline, straight from the
  // registers the converted row was loaded into.  Larger primes: the shared non-inlined
  // ks_digit_ntt (both forms inlined are ~54 KB of SASS, above the instruction cache; a
  // launch only ever executes one of them per row).
  const bool small = CKB200_SMALLQ && small_prime(q);
  {
    u64 y[kE];
#pragma unroll
    for (int k = 0; k < kE; ++k) y[k] = conv[sub_index<P2, 0, false>(g, k)];
    if (CKB200_MD_INLINE_SMALL && small) {
      row_transform<P2, false, LOGN, SyncCta, true>(y, g, r << P2, srow, tw, neg_opaque(q), q << 2);
      __syncthreads();
      row_to_smem<P2, RowLast<P2>::value, false>(y, g, srow);
    } else {
      row_to_smem<P2, 0, false>(y, g, srow);
      ks_digit_ntt_any<P2, LOGN>(srow, g, r, tw, q, two_q, true);  // lazy [0,16q); q >= 2^56 canonical
    }
  }
  // LAZY instantiation: every kept prime is below 2^59; otherwise decide per row
  const bool lazy = LAZY || q < ((u64)1 << 59);
  const u64 qoff = small ? q << 6 : q << 4;   // small primes leave [0, 64q)
  __syncthreads();
#else
  u64 y[kE];
#pragma unroll
  for (int k = 0; k < kE; ++k) y[k] = conv[sub_index<P2, 0, false>(g, k)];
  row_transform<P2, false, LOGN>(y, g, r << P2, srow, tw, q, two_q);
  // conv stays lazy in [0, 16q) when x + 16q - conv fits 64 bits (q < 2^59,
  // LAZY instantiation); the Shoup multiply below accepts any 64-bit input
  constexpr bool lazy = LAZY;
  if (!lazy) {
#pragma unroll
    for (int k = 0; k < kE; ++k) y[k] = fwd_final(y[k], q);
  }
  __syncthreads();
  row_to_smem<P2, RowLast<P2>::value, false>(y, g, srow);
  __syncthreads();
#endif
  u64 o[kE];
#pragma unroll
  for (int k = 0; k < kE; ++k) {
    const int c = sub_index<P2, 0, false>(g, k);
    const u64 xv = x[c];
    o[k] = lazy ? shoup(xv + qoff - srow[sidx(c)], pinv.x, pinv.y, q)
                : shoup(submod(xv, srow[sidx(c)], q), pinv.x, pinv.y, q);
  }
  const u64* addp = w ? a.addend : a.addend_u;
  if (addp) {
    const u64 t = a.galois ? a.galois[b] : a.galois_t;
    const int sr = t == 1 ? r : (int)(automorph_src((u32)r << P2, (u32)t, LOGN) >> P2);
    const u64* add = addp + b * a.addend_batch + ((long long)j << LOGN) + ((long long)sr << P2);
    // relinearisation: pmodup(b3) through the merged ModDown is b3 * q_last^-1
    const ulonglong2 asc = a.add_scale ? a.add_scale[j] : make_ulonglong2(0, 0);
    u64 z[kE];
#pragma unroll
    for (int k = 0; k < kE; ++k) z[k] = add[sub_index<P2, 0, false>(g, k)];
    __syncthreads();
    row_to_smem<P2, 0, false>(z, g, srow);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      const int c = sub_index<P2, 0, false>(g, k);
      const int sc = t == 1 ? c
                            : (int)(automorph_src(((u32)r << P2) + c, (u32)t, LOGN) & (F::S - 1));
      const u64 z = srow[sidx(sc)];
      o[k] = addmod(o[k], a.add_scale ? shoup(z, asc.x, asc.y, q) : z, q);
    }
  }
  u64* out = (a.pair && w ? a.out2 : a.out) + b * a.out_batch + ((long long)j << LOGN) +
             ((long long)r << P2);
#pragma unroll
  for (int k = 0; k < kE; ++k) out[sub_index<P2, 0, false>(g, k)] = o[k];
  __syncthreads();  // srow is the next item's exchange buffer
  }
}

// ------------------------------------------------------------------ launch
template <int P1, int P2>
static int launch_ks_row_t(const KsRowArgs& a, int rows, int batch, cudaStream_t st) {
  using F = FusedCfg<P2, kKsEpc>;
  const int bsel = a.beta <= 4 ? a.beta : 0;
  // digit slots (+ the key ring and its mbarriers for compile-time BETA)
  const size_t ring = bsel && CKB200_KS_RING
                          ? (size_t)CKB200_KS_RING * (2 * bsel * 2 * F::NT * 8 + 8)
                          : 0;
  const size_t smem = (size_t)a.beta * F::TR * F::RS * 8 + ring;
  auto kern = bsel == 1   ? ks_row_kernel<P1, P2, 1>
              : bsel == 2 ? ks_row_kernel<P1, P2, 2>
              : bsel == 3 ? ks_row_kernel<P1, P2, 3>
              : bsel == 4 ? ks_row_kernel<P1, P2, 4>
                          : ks_row_kernel<P1, P2, 0>;
  if (smem > 48 * 1024) {
    // the opt-in is per (device, kernel): set it once (host cost on the launch-bound C1 path)
    static std::atomic<unsigned> done[5];
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned bit = dev < 32 ? 1u << dev : 0u;
    if (!bit || !(done[bsel].load(std::memory_order_relaxed) & bit)) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)((size_t)(bsel ? bsel : 8) * F::TR * F::RS * 8 + ring));
      done[bsel].fetch_or(bit, std::memory_order_relaxed);
    }
  }
  launch_pdl(kern, dim3((1 << P1) / F::TR, batch, rows), dim3(F::NT), smem, st, a);
  return 0;
}

template <int P1, int P2>
static int launch_md_row_t(const MdRowArgs& a, int rows, int batch, cudaStream_t st) {
  using F = FusedCfg<P2, CKB200_MD_EPC>;
  MdRowArgs g = a;
  g.batch = batch;
  const int items = batch * (a.pair ? 2 : 1);
  if (g.group < 1) g.group = 1;
  const dim3 grid((1 << P1) / F::TR, (items + g.group - 1) / g.group, rows);
  if (a.lazy) launch_pdl(md_row_kernel<P1, P2, true>, grid, dim3(F::NT), 0, st, g);
  else launch_pdl(md_row_kernel<P1, P2, false>, grid, dim3(F::NT), 0, st, g);
  return 0;
}

bool fused_supported(int logn) { return logn >= 12 && logn <= 20; }

int launch_ks_row(const KsRowArgs& a, int rows, int batch, cudaStream_t st) {
  if (rows <= 0 || batch <= 0) return 0;
  if (a.beta < 1 || a.beta > 8) return CK_ERR_ARG;
  count_launches(1);
  switch (a.logn) {
    case 12: launch_ks_row_t<6, 6>(a, rows, batch, st); break;
    case 13: launch_ks_row_t<6, 7>(a, rows, batch, st); break;
    case 14: launch_ks_row_t<7, 7>(a, rows, batch, st); break;
    case 15: launch_ks_row_t<7, 8>(a, rows, batch, st); break;
    case 16: launch_ks_row_t<8, 8>(a, rows, batch, st); break;
    case 17: launch_ks_row_t<8, 9>(a, rows, batch, st); break;
    case 18: launch_ks_row_t<9, 9>(a, rows, batch, st); break;
    case 19: launch_ks_row_t<9, 10>(a, rows, batch, st); break;
    case 20: launch_ks_row_t<10, 10>(a, rows, batch, st); break;
    default: return CK_ERR_ARG;
  }
  return (int)cudaGetLastError();
}

int launch_md_row(const MdRowArgs& a, int rows, int batch, cudaStream_t st) {
  if (rows <= 0 || batch <= 0) return 0;
  count_launches(1);
  switch (a.logn) {
    case 12: launch_md_row_t<6, 6>(a, rows, batch, st); break;
    case 13: launch_md_row_t<6, 7>(a, rows, batch, st); break;
    case 14: launch_md_row_t<7, 7>(a, rows, batch, st); break;
    case 15: launch_md_row_t<7, 8>(a, rows, batch, st); break;
    case 16: launch_md_row_t<8, 8>(a, rows, batch, st); break;
    case 17: launch_md_row_t<8, 9>(a, rows, batch, st); break;
    case 18: launch_md_row_t<9, 9>(a, rows, batch, st); break;
    case 19: launch_md_row_t<9, 10>(a, rows, batch, st); break;
    case 20: launch_md_row_t<10, 10>(a, rows, batch, st); break;
    default: return CK_ERR_ARG;
  }
  return (int)cudaGetLastError();
}

}  // namespace ck
