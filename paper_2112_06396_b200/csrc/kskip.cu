// Key-switching inner product (KSKIP) with the Galois automorphism folded in.
//
// Reference: ckks._kskip (ckks.py:450-465) on digits that hrotate first
// permutes with RnsPoly.automorph (rnspoly.py:228-233):
//   u[i][k] = sum_j d_j[i][perm(k)] * a_j[row_i][k]  mod q_i
//   v[i][k] = sum_j d_j[i][perm(k)] * b_j[row_i][k]  mod q_i
//
// Storage-row structure of the eval-domain automorphism: with the storage
// index split as i = r * 2^P2 + c (the NTT's row phase), perm maps a whole
// output row r to a single input row r' (the affine map j -> t j + (t-1)/2
// on natural indices keeps the low P1 bits of j, i.e. the storage row,
// independent of c).  So each CTA stages the needed input rows in shared
// memory with coalesced loads and gathers from there.
#include "ck_internal.h"

namespace ck {

// any storage split works (see above); rows of <= 512 elements fit the tile
CK_HD int ks_row_bits(int logn) { return logn < 9 ? logn : 9; }

constexpr int kKsThreads = 256;
constexpr int kKsMaxBeta = 8;

// grid = (batch, N / TILE, rows); TILE = 512 elements (or N if smaller).
// BETA > 0: compile-time digit count, every key element of a thread's
// coefficients is requested before the first multiply (the kernel streams
// keys, so memory-level parallelism is what matters); BETA = 0: runtime.
template <int TILE, int BETA = 0>
__global__ void __launch_bounds__(kKsThreads) kskip_kernel(KskipArgs a) {
  __shared__ u64 sd[kKsMaxBeta][TILE];
  const int logn = a.logn;
  const int p2 = ks_row_bits(logn);
  const int rowlen = 1 << p2;
  // grid (batch, tile, row): the batch items that share a digit tile (hoisted
  // rotations: same digits, different keys / Galois elements) run back to back,
  // so the tile is still in L2 for all of them
  const int i = blockIdx.z;
  const long long bz = blockIdx.x;
  const int prime = a.prime[i];
  const PrimeConst P = a.pc[prime];
  const u64 t = a.galois ? a.galois[bz] : a.galois_t;
  const long long tile0 = (long long)blockIdx.y * TILE;
  const int krow = a.key_row[i];
  // key_digit0: first digit of this chunk (pointer-array keys point at digit 0)
  const long long kd0 = a.key_b_ptrs ? (long long)a.key_digit0 * a.key_digit_stride : 0;
  const u64* kb = key_block(a.key_b, a.key_b_ptrs, a.key_batch, bz) + kd0 + ((long long)krow << logn);
  const u64* ka = key_block(a.key_a, a.key_a_ptrs, a.key_batch, bz) + kd0 + ((long long)krow << logn);
  const u64* dig = a.digits + bz * a.digits_batch + ((long long)i << logn);
  // stage the gathered digit rows: for each storage row in the tile load the
  // source row perm maps it to
  for (int d = 0; d < a.beta; ++d) {
    const u64* dd = dig + d * a.digit_stride;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
      const long long o = tile0 + e;
      const long long rowstart = o & ~(long long)(rowlen - 1);
      const long long src_row = t == 1 ? rowstart
                                       : (long long)(automorph_src((u32)rowstart, (u32)t, logn) &
                                                     ~(u32)(rowlen - 1));
      sd[d][e] = dd[src_row + (o & (rowlen - 1))];
    }
  }
  __syncthreads();
  u64* uo = a.u + bz * a.out_batch + ((long long)i << logn);
  u64* vo = a.v + bz * a.out_batch + ((long long)i << logn);
  if constexpr (BETA > 0) {
    constexpr int PER = TILE / kKsThreads;  // coefficients per thread
    u64 ya[PER][BETA], yb[PER][BETA];
#pragma unroll
    for (int h = 0; h < PER; ++h)
#pragma unroll
      for (int d = 0; d < BETA; ++d) {
        const long long o = tile0 + threadIdx.x + h * kKsThreads;
        ya[h][d] = __ldg(ka + d * a.key_digit_stride + o);
        yb[h][d] = __ldg(kb + d * a.key_digit_stride + o);
      }
#pragma unroll
    for (int h = 0; h < PER; ++h) {
      const int e = threadIdx.x + h * kKsThreads;
      const long long o = tile0 + e;
      int se = e;
      if (t != 1) {
        const u32 src = automorph_src((u32)o, (u32)t, logn);
        se = (int)((o & ~(long long)(rowlen - 1)) - tile0) + (int)(src & (rowlen - 1));
      }
      Acc3 su, sv;
      acc3_zero(su);
      acc3_zero(sv);
#pragma unroll
      for (int d = 0; d < BETA; ++d) {
        const u64 x = sd[d][se];
        const u32 x0 = lo30(x), x1 = hi30(x);
        acc3_mac(su, x0, x1, lo30(ya[h][d]), hi30(ya[h][d]));
        acc3_mac(sv, x0, x1, lo30(yb[h][d]), hi30(yb[h][d]));
      }
      uo[o] = a.accumulate ? addmod(uo[o], acc3_reduce(su, P), P.q) : acc3_reduce(su, P);
      vo[o] = a.accumulate ? addmod(vo[o], acc3_reduce(sv, P), P.q) : acc3_reduce(sv, P);
    }
    return;
  }
  for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
    const long long o = tile0 + e;
    int se = e;
    if (t != 1) {
      const u32 src = automorph_src((u32)o, (u32)t, logn);
      se = (int)((o & ~(long long)(rowlen - 1)) - tile0) + (int)(src & (rowlen - 1));
    }
    Acc3 su, sv;
    acc3_zero(su);
    acc3_zero(sv);
    for (int d = 0; d < a.beta; ++d) {
      const u64 x = sd[d][se];
      const u64 ya = __ldg(ka + d * a.key_digit_stride + o);
      const u64 yb = __ldg(kb + d * a.key_digit_stride + o);
      const u32 x0 = lo30(x), x1 = hi30(x);
      acc3_mac(su, x0, x1, lo30(ya), hi30(ya));
      acc3_mac(sv, x0, x1, lo30(yb), hi30(yb));
    }
    uo[o] = a.accumulate ? addmod(uo[o], acc3_reduce(su, P), P.q) : acc3_reduce(su, P);
    vo[o] = a.accumulate ? addmod(vo[o], acc3_reduce(sv, P), P.q) : acc3_reduce(sv, P);
  }
}

int launch_kskip(const KskipArgs& a0, int rows, int batch, cudaStream_t st) {
  if (rows <= 0 || batch <= 0) return 0;
  if (a0.beta < 1) return CK_ERR_ARG;
  if (a0.beta > kKsMaxBeta) {
    // any dnum: chunks of kKsMaxBeta digits, later chunks accumulate into u, v
    for (int d0 = 0; d0 < a0.beta; d0 += kKsMaxBeta) {
      KskipArgs c = a0;
      c.beta = a0.beta - d0 < kKsMaxBeta ? a0.beta - d0 : kKsMaxBeta;
      c.digits = a0.digits + d0 * a0.digit_stride;
      if (c.key_b) c.key_b += d0 * a0.key_digit_stride;
      if (c.key_a) c.key_a += d0 * a0.key_digit_stride;
      c.key_digit0 = a0.key_digit0 + d0;
      c.accumulate = a0.accumulate || d0 > 0;
      const int e = launch_kskip(c, rows, batch, st);
      if (e) return e;
    }
    return 0;
  }
  const KskipArgs& a = a0;
  const int n = 1 << a.logn;
  count_launches(1);
  if (n >= 512) {
    const dim3 g(batch, n / 512, rows);
    if (a.beta == 3) kskip_kernel<512, 3><<<g, kKsThreads, 0, st>>>(a);
    else if (a.beta == 4) kskip_kernel<512, 4><<<g, kKsThreads, 0, st>>>(a);
    else kskip_kernel<512><<<g, kKsThreads, 0, st>>>(a);
  } else {
    // small rings: one tile holds the whole limb (row_bits == logn)
    switch (a.logn) {
#define CK_KS_SMALL(L) \
  case L: kskip_kernel<(1 << L)><<<dim3(batch, 1, rows), kKsThreads, 0, st>>>(a); break;
      CK_KS_SMALL(1) CK_KS_SMALL(2) CK_KS_SMALL(3) CK_KS_SMALL(4) CK_KS_SMALL(5)
      CK_KS_SMALL(6) CK_KS_SMALL(7) CK_KS_SMALL(8)
#undef CK_KS_SMALL
      default: return CK_ERR_ARG;
    }
  }
  return (int)cudaGetLastError();
}

}  // namespace ck
