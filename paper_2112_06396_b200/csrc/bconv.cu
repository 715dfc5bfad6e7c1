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
#include "ck_internal.h"

namespace ck {

constexpr int kBcThreads = 128;
constexpr int kBcCpt = 2;  // coefficients per thread

struct BcDst {
  u64 p, bar, c30, c30p;
};

// Several independent conversions (e.g. the beta ModUp digits) share one
// launch: grid.y selects the group.
struct BconvGroups {
  BconvArgs g[kMaxBcGroups];
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

int launch_bconv_groups(const BconvArgs* gs, int ng, int batch, cudaStream_t st) {
  if (ng <= 0 || batch <= 0) return 0;
  if (ng > kMaxBcGroups) return CK_ERR_ARG;
  BconvGroups G;
  int ns = 0;
  for (int i = 0; i < ng; ++i) {
    if (gs[i].nd <= 0 || gs[i].ns < 1) return CK_ERR_ARG;
    G.g[i] = gs[i];
    ns = gs[i].ns > ns ? gs[i].ns : ns;
  }
  count_launches(1);
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
