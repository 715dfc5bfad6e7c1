// Hoisted BSGS linear transform: the diagonal multiply-accumulate.
//
// SURVEY 8(a) a19 / composites.py:249-293; per giant group j the raised-basis
// accumulators of ckks.pt_matvec (ckks.py:699-711):
//   acc_u[j] = sum_k diag[j][k] * u_k
//   acc_v[j] = sum_k diag[j][k] * (v_k + [P]_q * automorph(b, t_k))   (pmodup: chain rows only)
// where (u_k, v_k) is the baby-step KSKIP output for rotation k (one shared
// ModUp).  One thread owns one coefficient of one raised row for BOTH the
// baby inputs (kept in registers) and every giant output, so each diagonal
// element is read exactly once and each (u_k, v_k) element once per call.
// More than kMaxBaby babies / diagonals: the caller runs chunks of <= 32 with
// `accumulate` set after the first, into the same raised accumulators.
#include "ck_internal.h"

namespace ck {

// threads per CTA: the baby inputs (2 x MB u64 per thread) fit 32 KB of static SMEM
template <int MB>
constexpr int diag_threads() { return MB <= 16 ? 128 : 64; }
constexpr int kMaxBaby = 32;

// MB: compile-time upper bound on the baby count (fully unrolled, baby
// inputs stay in registers; entries k >= baby are never touched).  A thread
// owns one coefficient of one raised row for BOTH u and v, so every diagonal
// element is loaded once and feeds two accumulators.
template <int MB>
__global__ void __launch_bounds__(diag_threads<MB>(), 4) diag_mac_kernel(DiagArgs a) {
  constexpr int NT = diag_threads<MB>();
  // baby inputs of this thread's coefficient, u then v (thread-private columns:
  // shared memory only keeps them out of the register file)
  __shared__ u64 xs[2 * MB][NT];
  const int n = 1 << a.logn;
  const int c = blockIdx.x * NT + threadIdx.x;
  const int i = blockIdx.y;
  if (c >= n) return;
  const int t = threadIdx.x;
  const PrimeConst& P = a.pc[a.prime[i]];
  const long long rowN = (long long)a.R << a.logn;
  const long long off = ((long long)i << a.logn) + c;
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    if (k < a.baby) {
      xs[2 * k][t] = a.uv[(2LL * k) * rowN + off];
      u64 v = a.uv[(2LL * k + 1) * rowN + off];
      if (i < a.l) {
        const u64 g = a.galois[k];
        const u64 bv = a.b[((long long)i << a.logn) + automorph_src((u32)c, (u32)g, a.logn)];
        const ulonglong2 pm = a.pmod[i];
        v = addmod(v, shoup(bv, pm.x, pm.y, P.q), P.q);
      }
      xs[2 * k + 1][t] = v;
    }
  }
  for (int j = 0; j < a.giant; ++j) {
    const long long dj = (long long)j * a.diag_stride;
    u64* au = a.acc + (2LL * j) * rowN + off;
    u64* av = a.acc + (2LL * j + 1) * rowN + off;
    u64 yu = a.accumulate ? *au : 0, yv = a.accumulate ? *av : 0;
    // every diagonal of this giant group is requested before the first MAC
    constexpr int KL = MB < 16 ? MB : 16;
#pragma unroll
    for (int k1 = 0; k1 < MB; k1 += KL) {
    if (k1 >= a.baby) continue;
    u64 m[KL];
#pragma unroll
    for (int kk = 0; kk < KL; ++kk) {
      const int k = k1 + kk;
      m[kk] = k < a.baby ? __ldg(a.diag_ptrs ? a.diag_ptrs[dj + k] + off : a.diags + (dj + k) * rowN + off)
                         : 0;
    }
#pragma unroll
    for (int k0 = k1; k0 < k1 + KL; k0 += 8) {
      if (k0 >= a.baby) continue;
      Acc3 su, sv;
      acc3_zero(su);
      acc3_zero(sv);
#pragma unroll
      for (int kk = 0; kk < 8 && k0 + kk < MB; ++kk) {
        const int k = k0 + kk;
        if (k < a.baby) {
          const u32 m0 = lo30(m[k - k1]), m1 = hi30(m[k - k1]);
          const u64 xu = xs[2 * k][t], xv = xs[2 * k + 1][t];
          acc3_mac(su, m0, m1, lo30(xu), hi30(xu));
          acc3_mac(sv, m0, m1, lo30(xv), hi30(xv));
        }
      }
      yu = addmod(yu, acc3_reduce(su, P), P.q);
      yv = addmod(yv, acc3_reduce(sv, P), P.q);
    }
    }
    *au = yu;
    *av = yv;
  }
}

int launch_diag_mac(const DiagArgs& a, cudaStream_t st) {
  if (a.baby < 1 || a.baby > kMaxBaby || a.giant < 1 || a.diag_stride < a.baby) return CK_ERR_ARG;
  count_launches(1);
  const int n = 1 << a.logn;
#define CK_DIAG(MB)                                                                    \
  diag_mac_kernel<MB><<<dim3((n + diag_threads<MB>() - 1) / diag_threads<MB>(), a.R),       \
                        diag_threads<MB>(), 0, st>>>(a)
  if (a.baby <= 4) CK_DIAG(4);
  else if (a.baby <= 8) CK_DIAG(8);
  else if (a.baby <= 16) CK_DIAG(16);
  else CK_DIAG(32);
#undef CK_DIAG
  return (int)cudaGetLastError();
}

}  // namespace ck
