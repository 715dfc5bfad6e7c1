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
#include "ck_internal.h"

namespace ck {

constexpr int kDiagThreads = 256;
constexpr int kMaxBaby = 32;

// MB: compile-time upper bound on the baby count (fully unrolled, baby
// inputs stay in registers; entries k >= baby are never touched).
template <int MB>
__global__ void __launch_bounds__(kDiagThreads) diag_mac_kernel(DiagArgs a) {
  const int n = 1 << a.logn;
  const int c = blockIdx.x * kDiagThreads + threadIdx.x;
  const int i = blockIdx.y;
  const int w = blockIdx.z;  // 0: u, 1: v
  if (c >= n) return;
  const PrimeConst& P = a.pc[a.prime[i]];
  const long long rowN = (long long)a.R << a.logn;
  u64 x[MB];
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    x[k] = 0;
    if (k < a.baby) {
      u64 v = a.uv[(2LL * k + w) * rowN + ((long long)i << a.logn) + c];
      if (w == 1 && i < a.l) {
        const u64 t = a.galois[k];
        const u64 bv = a.b[((long long)i << a.logn) + automorph_src((u32)c, (u32)t, a.logn)];
        const ulonglong2 pm = a.pmod[i];
        v = addmod(v, shoup(bv, pm.x, pm.y, P.q), P.q);
      }
      x[k] = v;
    }
  }
  for (int j = 0; j < a.giant; ++j) {
    const u64* d = a.diags + (long long)j * a.baby * rowN + ((long long)i << a.logn) + c;
    u64 y = 0;
#pragma unroll
    for (int k0 = 0; k0 < MB; k0 += 8) {
      if (k0 >= a.baby) continue;
      Acc3 s;
      acc3_zero(s);
#pragma unroll
      for (int kk = 0; kk < 8 && k0 + kk < MB; ++kk) {
        const int k = k0 + kk;
        if (k < a.baby) {
          const u64 m = __ldg(d + k * rowN);
          acc3_mac(s, lo30(m), hi30(m), lo30(x[k]), hi30(x[k]));
        }
      }
      y = addmod(y, acc3_reduce(s, P), P.q);
    }
    a.acc[(2LL * j + w) * rowN + ((long long)i << a.logn) + c] = y;
  }
}

int launch_diag_mac(const DiagArgs& a, cudaStream_t st) {
  if (a.baby < 1 || a.baby > kMaxBaby || a.giant < 1) return CK_ERR_ARG;
  count_launches(1);
  const int n = 1 << a.logn;
  const dim3 grid((n + kDiagThreads - 1) / kDiagThreads, a.R, 2);
  if (a.baby <= 4) diag_mac_kernel<4><<<grid, kDiagThreads, 0, st>>>(a);
  else if (a.baby <= 8) diag_mac_kernel<8><<<grid, kDiagThreads, 0, st>>>(a);
  else if (a.baby <= 16) diag_mac_kernel<16><<<grid, kDiagThreads, 0, st>>>(a);
  else diag_mac_kernel<32><<<grid, kDiagThreads, 0, st>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace ck
