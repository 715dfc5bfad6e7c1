// Base conversion fused with the forward NTT column phase of its targets.
//
// ModUp (ckks.py:427-438) and ModDown (ckks.py:409-410) both convert a set of
// coefficient-domain source rows to target rows and immediately run the
// forward NTT on every target.  Done separately, every target row is written
// to HBM by the conversion and read back by the column phase (2.4 GB per C3
// step for ModUp alone).  Here one CTA owns a 2^P1 x 4 column tile of the
// storage matrix (1024 coefficients at N = 2^16) and one group of 4 targets:
//   1. the INT8 tensor-core contraction of bconv.cu (byte-sliced sources as the
//      A operand straight from global/L2, per-plan B fragments in registers),
//      FP64-quotient epilogue (+ centered correction for ModDown), written to a
//      shared-memory tile [row][4 targets x 4 columns];
//   2. the forward column phase of ntt_col_kernel on the 16 virtual columns of
//      that tile (each target with its own prime and twiddles), stored to the
//      target rows, lazily reduced exactly like ntt_col_kernel's output.
// The CTAs of one column tile differ only in the target group and are
// launched next to each other, so the sources are read from HBM once and
// re-read from L2.
#include "ck_internal.h"
#include "ntt.cuh"

namespace ck {

namespace {

constexpr int kFcCols = 4;                    // storage columns per CTA
constexpr int kFcV = 4 * kFcCols;             // virtual columns: 4 targets x 4 columns

__device__ __forceinline__ void mma_u8x(int (&c)[4], const u32 (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

__device__ __forceinline__ double u32_f64(u32 v) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)v), 4503599627370496.0);
}

template <int KS, int P1, int P2>
__global__ void __launch_bounds__(1 << P1, (P1 >= 8 ? 4 : 8))
bc_col_kernel(const __grid_constant__ BconvGroups G, int ngroups, const ulonglong2* __restrict__ twt) {
  constexpr int S = 1 << P1;                  // rows of the storage matrix = threads
  constexpr int NP = Sched<P1>::np;
  constexpr int LOGN = P1 + P2;
  constexpr int NW = S / 32;                  // warps
  constexpr int MB = S * kFcCols / 16;        // m16 blocks of coefficients
  constexpr int MBW = MB / NW;                // per warp (= 8)
  extern __shared__ __align__(16) unsigned char fc_smem[];
  u64* sm = (u64*)fc_smem;                                   // [S][kFcV]
  ulonglong2* tws = (ulonglong2*)(sm + S * kFcV);            // [4][S]
  unsigned char* kk = (unsigned char*)(tws + 4 * S);         // [S * kFcCols]

  const int grp = blockIdx.x;                 // target group (fastest: L2 reuse of sources)
  const int c0 = blockIdx.y * kFcCols;
  const int gi = blockIdx.z % ngroups;
  const long long bz = blockIdx.z / ngroups;
  const BconvArgs& a = G.g[gi];
  const int nd = a.nd, ns = a.ns;
  const int ngrp = (nd + 3) >> 2;
  if (grp >= ngrp) return;                    // uniform per CTA
  const int ntile = ngrp * 4;
  const int tid = threadIdx.x;
  const u64* in = a.in + bz * a.in_batch;
  u64* out = a.out + bz * a.out_batch;

  // twiddles of the (up to) 4 targets of this group
  for (int e = tid; e < 4 * S; e += S) {
    const int t = e / S, i = e - t * S;
    const int j = 4 * grp + t;
    tws[e] = j < nd ? twt[((long long)a.dst_prime[j] << LOGN) + i] : make_ulonglong2(0, 0);
  }
  if (a.centered) {
    // k = rint(sum_i fl(v_i) w_i) in the reference's op order (rnspoly.py:320-325)
    for (int e = tid; e < S * kFcCols; e += S) {
      const int row = e / kFcCols, cc = e - row * kFcCols;
      double est = 0.0;
      for (int i = 0; i < ns; ++i) {
        const long long off = (long long)i << LOGN;
        const u64 v = in[off + ((long long)row << P2) + c0 + cc];
        est = __dadd_rn(est, __dmul_rn(__ull2double_rn(v), a.w[i]));
      }
      kk[e] = (unsigned char)rint(est);
    }
  }

  // ---- 1. contraction on the tensor cores, epilogue into the tile
  const int warp = tid >> 5, lane = tid & 31, gid = lane >> 2, tig = lane & 3;
  uint2 bfr[KS][4];
#pragma unroll
  for (int s = 0; s < KS; ++s)
#pragma unroll
    for (int u = 0; u < 4; ++u)
      bfr[s][u] = s < a.tc_ks ? a.Bf[(s * ntile + grp * 4 + u) * 32 + lane] : make_uint2(0, 0);
  const int j = 4 * grp + tig;                // this lane's target
  const bool jv = j < nd;
  const int jp = jv ? a.dst_prime[j] : 0;
  const u64 p = a.pc[jp].q;
  const double pinv = 1.0 / (double)p;
  const u64* kq = a.centered ? a.kQ + (long long)(jv ? j : 0) * (ns + 1) : nullptr;
  __syncthreads();  // kk ready
#pragma unroll 1
  for (int mi = 0; mi < MBW; ++mi) {
    const int mb = warp * MBW + mi;
    const int r0 = 4 * mb;                    // m16 block = rows r0..r0+3 x 4 columns
    const int ra = r0 + (gid >> 2), rb = ra + 2, cc = gid & 3;
    const long long ea = ((long long)ra << P2) + c0 + cc, eb = ((long long)rb << P2) + c0 + cc;
    u32 af[KS][4];
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      const int i0 = 4 * s + (tig >> 1), i1 = i0 + 2, w = tig & 1;
      const u32* s0 = (const u32*)(in + ((long long)i0 << LOGN));
      const u32* s1 = (const u32*)(in + ((long long)i1 << LOGN));
      af[s][0] = i0 < ns ? s0[2 * ea + w] : 0u;
      af[s][1] = i0 < ns ? s0[2 * eb + w] : 0u;
      af[s][2] = i1 < ns ? s1[2 * ea + w] : 0u;
      af[s][3] = i1 < ns ? s1[2 * eb + w] : 0u;
    }
    int acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[u][c] = 0;
#pragma unroll
    for (int s = 0; s < KS; ++s)
#pragma unroll
      for (int u = 0; u < 4; ++u) mma_u8x(acc[u], af[s], bfr[s][u]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const u32 P0 = (u32)acc[0][2 * h] + ((u32)acc[0][2 * h + 1] << 8);
      const u32 P1v = (u32)acc[1][2 * h] + ((u32)acc[1][2 * h + 1] << 8);
      const u32 P2v = (u32)acc[2][2 * h] + ((u32)acc[2][2 * h + 1] << 8);
      const u32 P3 = (u32)acc[3][2 * h] + ((u32)acc[3][2 * h + 1] << 8);
      const u64 vlo = (u64)P0 + ((u64)P1v << 16) + ((u64)P2v << 32) + ((u64)P3 << 48);
      const double vd = __fma_rn(u32_f64(P3), 281474976710656.0,
                                 __fma_rn(u32_f64(P2v), 4294967296.0,
                                          __dmul_rn(u32_f64(P1v), 65536.0)));
      const u32 qh = (u32)__double2loint(__fma_rn(vd, pinv, 6755399441055744.0));
      u64 r = vlo - (u64)qh * p;
      r += ((long long)r < 0) ? p : 0ull;
      const int row = h ? rb : ra;
      if (a.centered) r = submod(r, kq[kk[row * kFcCols + cc]], p);
      sm[row * kFcV + tig * kFcCols + cc] = r;
    }
  }
  __syncthreads();

  // ---- 2. forward column phase on the 16 virtual columns (ntt_col_kernel, INV = false)
  const int v = tid % kFcV, g = tid / kFcV;   // S/16 threads per virtual column
  const int t = v / kFcCols;
  const int c = c0 + (v % kFcCols);           // limb-global column
  const int jt = 4 * grp + t;
  const bool tv = jt < nd;
  const PrimeConst& P = a.pc[tv ? a.dst_prime[jt] : 0];
  const u64 q = P.q, two_q = P.two_q;
  const ulonglong2* tw = tws + t * S;
  u64 x[kE];
#pragma unroll
  for (int r = 0; r < kE; ++r) x[r] = sm[sub_index<P1, 0, false>(g, r) * kFcV + v];
  run_pass<P1, 0, false, true, LOGN, P2>(x, g, c, tw, q, two_q);
  if constexpr (NP > 1) {
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kE; ++r) sm[sub_index<P1, 0, false>(g, r) * kFcV + v] = x[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kE; ++r) x[r] = sm[sub_index<P1, 1, false>(g, r) * kFcV + v];
    fwd_fold(x, q << 3);
    run_pass<P1, 1, false, true, LOGN, P2>(x, g, c, tw, q, two_q);
  }
  static_assert(NP <= 2, "column sub-transform too large");
  if (tv) {
    u64* base = out + (a.out_off ? a.out_off[jt] : ((long long)jt << LOGN));
#pragma unroll
    for (int r = 0; r < kE; ++r) base[((long long)sub_index<P1, NP - 1, false>(g, r) << P2) + c] = x[r];
  }
}

template <int KS, int P1, int P2>
int launch_t(const BconvGroups& G, int ng, int batch, const ulonglong2* tw, cudaStream_t st) {
  constexpr int S = 1 << P1;
  int ngrp = 0;
  for (int i = 0; i < ng; ++i) ngrp = max(ngrp, (G.g[i].nd + 3) / 4);
  const size_t smem = (size_t)S * kFcV * 8 + 4 * S * sizeof(ulonglong2) + S * kFcCols;
  auto kern = bc_col_kernel<KS, P1, P2>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<dim3(ngrp, (1 << P2) / kFcCols, ng * batch), S, smem, st>>>(G, ng, tw);
  return (int)cudaGetLastError();
}

template <int KS>
int launch_ks(const BconvGroups& G, int ng, int batch, const ulonglong2* tw, int logn, cudaStream_t st) {
  switch (logn) {
    case 12: return launch_t<KS, 6, 6>(G, ng, batch, tw, st);
    case 13: return launch_t<KS, 6, 7>(G, ng, batch, tw, st);
    case 14: return launch_t<KS, 7, 7>(G, ng, batch, tw, st);
    case 15: return launch_t<KS, 7, 8>(G, ng, batch, tw, st);
    case 16: return launch_t<KS, 8, 8>(G, ng, batch, tw, st);
    case 17: return launch_t<KS, 8, 9>(G, ng, batch, tw, st);
    default: return CK_ERR_ARG;
  }
}

}  // namespace

bool bc_col_supported(const BconvArgs* gs, int ng, int logn) {
  if (logn < 12 || logn > 17 || ng < 1 || ng > kMaxBcGroups) return false;
  for (int i = 0; i < ng; ++i) {
    const BconvArgs& a = gs[i];
    if (!a.Bf || !a.c3248 || a.tc_ks < 1 || a.tc_ks > 4 || a.ns > 4 * a.tc_ks || a.src_scale ||
        a.in_off || a.nd < 1 || a.logn != logn)
      return false;
  }
  return true;
}

int launch_bc_col(const BconvArgs* gs, int ng, int batch, const ulonglong2* tw, cudaStream_t st) {
  if (ng <= 0 || batch <= 0) return 0;
  if (!bc_col_supported(gs, ng, gs[0].logn)) return CK_ERR_ARG;
  BconvGroups G;
  int ks = 0;
  for (int i = 0; i < ng; ++i) {
    G.g[i] = gs[i];
    ks = max(ks, gs[i].tc_ks);
  }
  count_launches(1);
  const int logn = gs[0].logn;
  if (ks <= 1) return launch_ks<1>(G, ng, batch, tw, logn, st);
  if (ks <= 2) return launch_ks<2>(G, ng, batch, tw, logn, st);
  if (ks <= 3) return launch_ks<3>(G, ng, batch, tw, logn, st);
  return launch_ks<4>(G, ng, batch, tw, logn, st);
}

}  // namespace ck
