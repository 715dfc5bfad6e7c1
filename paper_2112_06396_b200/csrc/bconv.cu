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
// matches the reference.  Here it is a small modular contraction on CUDA
// cores with 30-bit split operands: four 32x32->64 IMAD.WIDE per term into
// three 64-bit accumulators, one reduction per (coefficient, target).
// The float estimate replicates numpy's op order with explicit _rn
// intrinsics (no FMA contraction), round-half-even via rint().
#include "ck_internal.h"

namespace ck {

constexpr int kBcThreads = 128;

template <int MAXS>
__global__ void __launch_bounds__(kBcThreads) bconv_kernel(BconvArgs a) {
  __shared__ uint2 Ts[MAXS * 48];
  const int ns = a.ns, nd = a.nd;
  const bool tab_smem = ns * nd <= MAXS * 48;
  if (tab_smem) {
    for (int i = threadIdx.x; i < ns * nd; i += blockDim.x) {
      const u64 t = a.T[i];
      Ts[i] = make_uint2(lo30(t), hi30(t));
    }
  }
  __syncthreads();
  const int n = 1 << a.logn;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const u64* in = a.in + (long long)blockIdx.z * a.in_batch;
  u64* out = a.out + (long long)blockIdx.z * a.out_batch;

  u32 v0[MAXS], v1[MAXS];
  double est = 0.0;
#pragma unroll
  for (int i = 0; i < MAXS; ++i) {
    if (i < ns) {
      const long long off = a.in_off ? a.in_off[i] : ((long long)i << a.logn);
      u64 v = in[off + k];
      if (a.src_scale) {
        const ulonglong2 s = a.src_scale[i];
        v = shoup(v, s.x, s.y, a.pc[a.src_prime[i]].q);
      }
      if (a.centered) est = __dadd_rn(est, __dmul_rn(__ull2double_rn(v), a.w[i]));
      v0[i] = lo30(v);
      v1[i] = hi30(v);
    }
  }
  const u64 kk = a.centered ? (u64)rint(est) : 0;

  for (int j = 0; j < nd; ++j) {
    const PrimeConst P = a.pc[a.dst_prime[j]];
    u64 y = 0;
    for (int i0 = 0; i0 < ns; i0 += 8) {
      Acc3 s;
      acc3_zero(s);
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) {
        const int i = i0 + ii;
        if (i < ns && i < MAXS) {
          uint2 t;
          if (tab_smem) t = Ts[i * nd + j];
          else {
            const u64 tt = a.T[i * nd + j];
            t = make_uint2(lo30(tt), hi30(tt));
          }
          acc3_mac(s, v0[i], v1[i], t.x, t.y);
        }
      }
      y = addmod(y, acc3_reduce(s, P), P.q);
    }
    if (a.centered) y = submod(y, a.kQ[j * (ns + 1) + kk], P.q);
    const long long off = a.out_off ? a.out_off[j] : ((long long)j << a.logn);
    out[off + k] = y;
  }
}

int launch_bconv(const BconvArgs& a, int batch, cudaStream_t st) {
  if (a.nd <= 0 || batch <= 0) return 0;
  if (a.ns <= 0) return CK_ERR_ARG;
  const int n = 1 << a.logn;
  const dim3 grid((n + kBcThreads - 1) / kBcThreads, 1, batch);
  count_launches(1);
  if (a.ns <= 8) bconv_kernel<8><<<grid, kBcThreads, 0, st>>>(a);
  else if (a.ns <= 16) bconv_kernel<16><<<grid, kBcThreads, 0, st>>>(a);
  else if (a.ns <= 64) bconv_kernel<64><<<grid, kBcThreads, 0, st>>>(a);
  else return CK_ERR_ARG;
  return (int)cudaGetLastError();
}

}  // namespace ck
