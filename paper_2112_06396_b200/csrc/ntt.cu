// NTT / INTT kernels (see ntt.cuh for the decomposition).
#include "ntt.cuh"
#include "ck_internal.h"


namespace ck {

CK_D long long job_offset(const NttArgs& a, int job, int bz) {
  return (a.row_off ? a.row_off[job] : ((long long)job << a.logn)) + (long long)bz * a.batch_stride;
}

// ------------------------------------------------------------ column phase
// grid = (2^P2 / kTC, jobs, batch); block = kTC * 2^P1 / kE
#ifndef CKB200_NTT_MINB
#define CKB200_NTT_MINB 3
#endif
// row kernel: 4 CTAs/SM (64 registers) for rows up to 256 points -- measured +0.5% on
// C3 with the small-prime butterflies; longer rows spill there and stay at 3
#ifndef CKB200_NTT_ROW_MINB
#define CKB200_NTT_ROW_MINB 4
#endif
template <int P1, int P2, bool INV>
__global__ void __launch_bounds__(col_tc<P1>() * (1 << P1) / kE, CKB200_NTT_MINB)
ntt_col_kernel(NttArgs a) {
  constexpr int S = 1 << P1;
  constexpr int TC = col_tc<P1>();
  constexpr int NP = Sched<P1>::np;
  __shared__ u64 sm[S * TC];
  __shared__ ulonglong2 tws[S];
  const int job = blockIdx.y;
  const int prime = a.prime_idx[job];
  const u64 q = a.pc[prime].q, two_q = a.pc[prime].two_q;
  {
    const ulonglong2* tw = (INV ? a.itw : a.tw) + ((long long)prime << a.logn);
    for (int i = threadIdx.x; i < S; i += blockDim.x) tws[i] = tw[i];
  }
  u64* base = a.data + job_offset(a, job, blockIdx.z);
  const int col = threadIdx.x % TC, g = threadIdx.x / TC;
  const int c = blockIdx.x * TC + col;
  u64 x[kE];
#pragma unroll
  for (int r = 0; r < kE; ++r) x[r] = base[((long long)sub_index<P1, 0, INV>(g, r) << P2) + c];
  __syncthreads();
#define CK_COL_PASS(PP) run_pass<P1, PP, INV, true, P1 + P2, P2>(x, g, c, tws, q, two_q);
  CK_COL_PASS(0)
  if constexpr (NP > 1) {
#pragma unroll
    for (int r = 0; r < kE; ++r) sm[sub_index<P1, 0, INV>(g, r) * TC + col] = x[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kE; ++r) x[r] = sm[sub_index<P1, 1, INV>(g, r) * TC + col];
    if (!INV) fwd_fold(x, q << 3);
    CK_COL_PASS(1)
  }
  if constexpr (NP > 2) {
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kE; ++r) sm[sub_index<P1, 1, INV>(g, r) * TC + col] = x[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kE; ++r) x[r] = sm[sub_index<P1, 2, INV>(g, r) * TC + col];
    if (!INV) fwd_fold(x, q << 3);
    CK_COL_PASS(2)
  }
#undef CK_COL_PASS
  static_assert(NP <= 3, "sub-transform too large");
  if (INV) {
    // end of the inverse: scale by n^-1 (times the optional extra constant)
    const ulonglong2 s = a.scale ? a.scale[job]
                                 : make_ulonglong2(a.pc[prime].ninv, a.pc[prime].ninvp);
#pragma unroll
    for (int r = 0; r < kE; ++r) x[r] = shoup(x[r], s.x, s.y, q);
  }
  // forward: values stay lazy in [0,16q) for the row phase
#pragma unroll
  for (int r = 0; r < kE; ++r)
    base[((long long)sub_index<P1, NP - 1, INV>(g, r) << P2) + c] = x[r];
}

// --------------------------------------------------------------- row phase
// grid = (2^P1 / TR, jobs, batch); block = TR * 2^P2 / kE
// 128 threads per CTA (8 CTAs/SM for rows up to 256 points): 10.13 vs 10.22 ms per C3 step
// against 256-thread CTAs.  (A per-row shared-memory cache of the four finest levels'
// twiddles, filled by cp.async, was measured too: 30 KB per 8 rows halves the occupancy,
// 10.50 ms -- not kept.)
#ifndef CKB200_NTT_ROW_THREADS
#define CKB200_NTT_ROW_THREADS 128
#endif
template <int P2>
struct RowCfg {
  static constexpr int S = 1 << P2;
  static constexpr int G = S / kE;
  static constexpr int TR = CKB200_NTT_ROW_THREADS / G > 0 ? CKB200_NTT_ROW_THREADS / G : 1;
  static constexpr int RS = S + S / 16;  // padded smem row stride
};

#ifndef CKB200_SMALLQ
#define CKB200_SMALLQ 1
#endif
template <int P1, int P2, bool INV>
__global__ void __launch_bounds__(RowCfg<P2>::TR * RowCfg<P2>::G,
                                  (P2 <= 8 ? CKB200_NTT_ROW_MINB : CKB200_NTT_MINB) * (256 / CKB200_NTT_ROW_THREADS))
ntt_row_kernel(NttArgs a) {
  using R = RowCfg<P2>;
  constexpr int NP = Sched<P2>::np;
  __shared__ u64 sm[R::TR * R::RS];
  pdl_trigger();
  const int job = blockIdx.z;  // grid (row tile, batch, job): twiddle reuse across the batch
  const int prime = a.prime_idx[job];
  const u64 q = a.pc[prime].q, two_q = a.pc[prime].two_q;
  const ulonglong2* tw = (INV ? a.itw : a.tw) + ((long long)prime << a.logn);
  pdl_wait();
  u64* base = a.data + job_offset(a, job, blockIdx.y);
  const u64* ibase = a.src ? a.src + ((long long)job << a.logn) + (long long)blockIdx.y * a.src_batch_stride
                           : base;  // out-of-place input (e.g. ModUp reads the ciphertext directly)
  const int rl = threadIdx.x / R::G, g = threadIdx.x % R::G;
  const int row = blockIdx.x * R::TR + rl;
  u64* rowp = base + ((long long)row << P2);
  const u64* irowp = ibase + ((long long)row << P2);
  u64* srow = sm + rl * R::RS;
  const int jbase = row << P2;
  u64 x[kE];
  auto sidx = [](int s) { return s + (s >> 4); };
  if (!INV) {
#pragma unroll
    for (int r = 0; r < kE; ++r) x[r] = irowp[sub_index<P2, 0, INV>(g, r)];
  } else {
    // pass 0 of the inverse reads contiguous runs: stage through smem
    const u64* tile = ibase + ((long long)blockIdx.x * R::TR << P2);
    for (int i = threadIdx.x; i < R::TR * R::S; i += blockDim.x)
      sm[(i >> P2) * R::RS + sidx(i & (R::S - 1))] = tile[i];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kE; ++r) x[r] = srow[sidx(sub_index<P2, 0, INV>(g, r))];
  }
  // primes below 2^54: approximate-quotient butterflies without range folding
  // (ntt.cuh SMALL); inverse outputs are then below 2^(P2+1) q: the tensor-core
  // column phase takes any 64-bit operand, the butterfly column kernel needs [0, 2q)
  const bool small = CKB200_SMALLQ && (INV ? small_prime_inv(q, P2) : small_prime(q));
  if (small) {
    row_transform<P2, INV, P1 + P2, SyncCta, true>(x, g, jbase, srow, tw, neg_opaque(q), INV ? q : q << 2);
    if (INV && !(P1 == 8 && a.tcB && a.tcD)) {
      const PrimeConst& Pc = a.pc[prime];
#pragma unroll
      for (int r = 0; r < kE; ++r) x[r] = red64_lazy(x[r], Pc);
    }
  } else {
    row_transform<P2, INV, P1 + P2>(x, g, jbase, srow, tw, q, two_q);
  }
  static_assert(NP <= 3, "sub-transform too large");
  if (!INV) {
    // end of the forward transform: canonical residues; stores staged
    // through smem so the global writes are coalesced
    if (small) {  // below (16 + 4 P2) q: one Barrett step
      const PrimeConst& Pc = a.pc[prime];
#pragma unroll
      for (int r = 0; r < kE; ++r) x[r] = red64(x[r], Pc);
    } else {
#pragma unroll
      for (int r = 0; r < kE; ++r) x[r] = fwd_final(x[r], q);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kE; ++r) srow[sidx(sub_index<P2, RowLast<P2>::value, INV>(g, r))] = x[r];
    __syncthreads();
    u64* tile = base + ((long long)blockIdx.x * R::TR << P2);
    for (int i = threadIdx.x; i < R::TR * R::S; i += blockDim.x)
      tile[i] = sm[(i >> P2) * R::RS + sidx(i & (R::S - 1))];
  } else {
#pragma unroll
    for (int r = 0; r < kE; ++r) rowp[sub_index<P2, RowLast<P2>::value, INV>(g, r)] = x[r];
  }
}

// ------------------------------------------------------- small N (<= 2^11)
// One CTA per limb; plain radix-2 stages in shared memory.
template <bool INV>
__global__ void __launch_bounds__(512) ntt_small_kernel(NttArgs a) {
  extern __shared__ u64 sx[];
  const int n = 1 << a.logn;
  const int job = blockIdx.y;
  const int prime = a.prime_idx[job];
  const u64 q = a.pc[prime].q, two_q = a.pc[prime].two_q;
  const ulonglong2* tw = (INV ? a.itw : a.tw) + ((long long)prime << a.logn);
  u64* base = a.data + job_offset(a, job, blockIdx.z);
  for (int i = threadIdx.x; i < n; i += blockDim.x) sx[i] = base[i];
  __syncthreads();
  if (!INV) {
    for (int logt = a.logn - 1; logt >= 0; --logt) {
      const int t = 1 << logt, m = n >> (logt + 1);
      for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
        const int blk = b >> logt, off = b & (t - 1);
        const int j = (blk << (logt + 1)) + off;
        const ulonglong2 w = tw[m + blk];
        bfly_ct(sx[j], sx[j + t], w.x, w.y, q, two_q);
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) base[i] = csub(csub(sx[i], two_q), q);
  } else {
    for (int logt = 0; logt < a.logn; ++logt) {
      const int t = 1 << logt, h = n >> (logt + 1);
      for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
        const int blk = b >> logt, off = b & (t - 1);
        const int j = (blk << (logt + 1)) + off;
        const ulonglong2 w = tw[h + blk];
        bfly_gs(sx[j], sx[j + t], w.x, w.y, q, two_q);
      }
      __syncthreads();
    }
    const ulonglong2 s = a.scale ? a.scale[job]
                                 : make_ulonglong2(a.pc[prime].ninv, a.pc[prime].ninvp);
    for (int i = threadIdx.x; i < n; i += blockDim.x) base[i] = shoup(sx[i], s.x, s.y, q);
  }
}

// ------------------------------------------------------------------ launch
template <int P1, int P2>
static void launch_split(const NttArgs& a, int jobs, int batch, bool inv, int phase,
                         cudaStream_t st) {
  const dim3 gcol((1 << P2) / col_tc<P1>(), jobs, batch), bcol(col_tc<P1>() * (1 << P1) / kE);
  using R = RowCfg<P2>;
  const dim3 grow((1 << P1) / R::TR, batch, jobs), brow(R::TR * R::G);
  const bool col = phase != 2, row = phase != 1;
  count_launches((int)col + (int)row);
  if (!inv) {
    if (col && P1 == 8 && a.tcB && launch_ntt_col_tc(a, jobs, batch, false, st) == 0) {
      // forward column phase ran on the tensor cores (ntt_tc.cu)
    } else if (col) {
      ntt_col_kernel<P1, P2, false><<<gcol, bcol, 0, st>>>(a);
    }
    if (row) launch_pdl(ntt_row_kernel<P1, P2, false>, grow, brow, 0, st, a);
  } else {
    if (row) launch_pdl(ntt_row_kernel<P1, P2, true>, grow, brow, 0, st, a);
    if (col && P1 == 8 && a.tcB && launch_ntt_col_tc(a, jobs, batch, true, st) == 0) {
      // inverse column phase ran on the tensor cores (ntt_tc.cu)
    } else if (col) {
      ntt_col_kernel<P1, P2, true><<<gcol, bcol, 0, st>>>(a);
    }
  }
}

// phase: 0 = full transform, 1 = column phase only, 2 = row phase only
// (split transforms are used by the fused key-switch; logn >= 12 only).
int launch_ntt_phase(const NttArgs& a, int jobs, int batch, bool inverse, int phase,
                     cudaStream_t st) {
  if (jobs <= 0 || batch <= 0) return 0;
  switch (a.logn) {
    case 12: launch_split<6, 6>(a, jobs, batch, inverse, phase, st); break;
    case 13: launch_split<6, 7>(a, jobs, batch, inverse, phase, st); break;
    case 14: launch_split<7, 7>(a, jobs, batch, inverse, phase, st); break;
    case 15: launch_split<7, 8>(a, jobs, batch, inverse, phase, st); break;
    case 16: launch_split<8, 8>(a, jobs, batch, inverse, phase, st); break;
    case 17: launch_split<8, 9>(a, jobs, batch, inverse, phase, st); break;
    case 18: launch_split<9, 9>(a, jobs, batch, inverse, phase, st); break;
    case 19: launch_split<9, 10>(a, jobs, batch, inverse, phase, st); break;
    case 20: launch_split<10, 10>(a, jobs, batch, inverse, phase, st); break;
    default: {
      if (phase != 0 || a.logn < 1 || a.logn > 11) return CK_ERR_ARG;
      count_launches(1);
      const int n = 1 << a.logn;
      const dim3 grid(1, jobs, batch), blk(n / 2 < 512 ? (n / 2 > 0 ? n / 2 : 1) : 512);
      if (inverse) ntt_small_kernel<true><<<grid, blk, n * sizeof(u64), st>>>(a);
      else ntt_small_kernel<false><<<grid, blk, n * sizeof(u64), st>>>(a);
    }
  }
  return (int)cudaGetLastError();
}

int launch_ntt(const NttArgs& a, int jobs, int batch, bool inverse, cudaStream_t st) {
  return launch_ntt_phase(a, jobs, batch, inverse, 0, st);
}

}  // namespace ck
