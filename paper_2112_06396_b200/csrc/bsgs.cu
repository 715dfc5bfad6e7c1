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
constexpr int kDiagKL = 8;      // diagonals per staged chunk
constexpr int kDiagStages = 3;  // chunks in flight per thread
constexpr int kDiagPtrs = 512;  // diagonal pointers staged in shared memory (giant x baby)
template <int MB>
constexpr size_t diag_smem() {
  return (size_t)(2 * MB + kDiagStages * kDiagKL) * diag_threads<MB>() * 8 + kDiagPtrs * 8;
}

// Memory-level parallelism without barriers: every thread only ever reads the
// shared-memory words its own cp.async wrote (its coefficient's column), so
// the baby inputs (u_k, v_k) and the diagonal stream are plain 8-byte async
// copies -- all baby inputs at once, the diagonals kDiagStages chunks ahead
// of the multiply-accumulate -- and no __syncthreads is needed anywhere.
template <int MB>
__global__ void __launch_bounds__(diag_threads<MB>(), 4) diag_mac_kernel(DiagArgs a) {
  constexpr int NT = diag_threads<MB>();
  constexpr int KL = kDiagKL, NS = kDiagStages;
  extern __shared__ __align__(16) u64 dsm[];
  u64 (*xs)[NT] = (u64 (*)[NT])dsm;                          // [2 MB][NT] baby inputs
  u64 (*ds)[KL][NT] = (u64 (*)[KL][NT])(dsm + 2 * MB * NT);  // [NS][KL][NT] diagonals
  const u64** dps = (const u64**)(dsm + (2 * MB + NS * KL) * NT);  // [giant][baby] diagonal rows
  const int n = 1 << a.logn;
  const int c = blockIdx.x * NT + threadIdx.x;
  const int i = blockIdx.y;
  const int t = threadIdx.x;
  // the diagonal pointers, once per CTA (a cp.async whose address waits on a
  // global pointer load stalls the whole stream)
  const bool staged = a.diag_ptrs && a.giant * a.baby <= kDiagPtrs;
  if (staged) {
    for (int e = t; e < a.giant * a.baby; e += NT)
      dps[e] = a.diag_ptrs[(long long)(e / a.baby) * a.diag_stride + e % a.baby];
    __syncthreads();
  }
  if (c >= n) return;
  const PrimeConst P = a.pc[a.prime[i]];  // a register copy: global reads of P would reload after every store
  const long long rowN = (long long)a.R << a.logn;
  const long long off = ((long long)i << a.logn) + c;
  const int nk = (a.baby + KL - 1) / KL;   // chunks per giant group
  const int nq = a.giant * nk;             // chunks in all
  auto stage = [&](int q) {                // one commit group per chunk (possibly empty)
    if (q < nq) {
      const int s = q % NS, j = q / nk, k1 = (q % nk) * KL;
      const long long dj = (long long)j * a.diag_stride;
#pragma unroll
      for (int kk = 0; kk < KL; ++kk) {
        const int k = k1 + kk;
        if (k < a.baby)
          cp_async8(&ds[s][kk][t], staged ? dps[j * a.baby + k] + off
                                   : a.diag_ptrs ? a.diag_ptrs[dj + k] + off
                                                 : a.diags + (dj + k) * rowN + off);
      }
    }
    cp_async_commit();
  };
  // baby inputs: all in flight at once (group 0), then the first diagonal chunks
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    if (k < a.baby) {
      cp_async8(&xs[2 * k][t], a.uv + (2LL * k) * rowN + off);
      cp_async8(&xs[2 * k + 1][t], a.uv + (2LL * k + 1) * rowN + off);
    }
  }
  cp_async_commit();
#pragma unroll
  for (int q = 0; q < NS - 1; ++q) stage(q);
  // pmodup(automorph(b, t_k)) for the v inputs (chain rows): gathers in registers
  u64 bv[MB];
  const bool chain = i < a.l;
  if (chain) {
#pragma unroll
    for (int k = 0; k < MB; ++k)
      if (k < a.baby)
        bv[k] = a.b[((long long)i << a.logn) + automorph_src((u32)c, (u32)a.galois[k], a.logn)];
  }
  cp_async_wait<NS - 1>();  // group 0 (baby inputs) has landed
  if (chain) {
    const ulonglong2 pm = a.pmod[i];
#pragma unroll
    for (int k = 0; k < MB; ++k)
      if (k < a.baby) xs[2 * k + 1][t] = addmod(xs[2 * k + 1][t], shoup(bv[k], pm.x, pm.y, P.q), P.q);
  }
  u64 yu = 0, yv = 0;
#pragma unroll 1
  for (int q = 0; q < nq; ++q) {
    const int s = q % NS, j = q / nk, k1 = (q % nk) * KL;
    stage(q + NS - 1);          // refills the stage chunk q-1 used
    cp_async_wait<NS - 1>();    // chunk q has landed
    if (k1 == 0) {
      yu = a.accumulate ? a.acc[(2LL * j) * rowN + off] : 0;
      yv = a.accumulate ? a.acc[(2LL * j + 1) * rowN + off] : 0;
    }
    Acc3 su, sv;
    acc3_zero(su);
    acc3_zero(sv);
#pragma unroll
    for (int kk = 0; kk < KL; ++kk) {
      const int k = k1 + kk;
      if (k < a.baby) {
        const u64 mv = ds[s][kk][t];
        const u32 m0 = lo30(mv), m1 = hi30(mv);
        const u64 xu = xs[2 * k][t], xv = xs[2 * k + 1][t];
        acc3_mac(su, m0, m1, lo30(xu), hi30(xu));
        acc3_mac(sv, m0, m1, lo30(xv), hi30(xv));
      }
    }
    yu = addmod(yu, acc3_reduce(su, P), P.q);
    yv = addmod(yv, acc3_reduce(sv, P), P.q);
    if (k1 + KL >= a.baby) {   // last chunk of giant group j
      a.acc[(2LL * j) * rowN + off] = yu;
      a.acc[(2LL * j + 1) * rowN + off] = yv;
    }
  }
}

int launch_diag_mac(const DiagArgs& a, cudaStream_t st) {
  if (a.baby < 1 || a.baby > kMaxBaby || a.giant < 1 || a.diag_stride < a.baby) return CK_ERR_ARG;
  count_launches(1);
  const int n = 1 << a.logn;
#define CK_DIAG(MB)                                                                          \
  do {                                                                                        \
    static unsigned done = 0;                                                                 \
    int dev = 0;                                                                              \
    cudaGetDevice(&dev);                                                                      \
    if (dev >= 32 || !((done >> dev) & 1u)) {                                                 \
      cudaFuncSetAttribute(diag_mac_kernel<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                           (int)diag_smem<MB>());                                             \
      if (dev < 32) __atomic_fetch_or(&done, 1u << dev, __ATOMIC_RELAXED);                    \
    }                                                                                         \
    diag_mac_kernel<MB><<<dim3((n + diag_threads<MB>() - 1) / diag_threads<MB>(), a.R),      \
                          diag_threads<MB>(), diag_smem<MB>(), st>>>(a);                      \
  } while (0)
  if (a.baby <= 4) CK_DIAG(4);
  else if (a.baby <= 8) CK_DIAG(8);
  else if (a.baby <= 16) CK_DIAG(16);
  else CK_DIAG(32);
#undef CK_DIAG
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Fused baby-step KSKIP + diagonal MAC.  One thread = one coefficient c of one
// raised row i.  Per baby k (compile-time unrolled, MB <= 16): its BETA digit
// values at the automorphism's source index and its 2 BETA key words arrive by
// per-thread 8-byte cp.async (a ring NSB babies deep, thread-private columns:
// no barriers); u_k = sum_d digit_d[perm_k(c)] key_a[k][d][i][c],
// v_k = sum_d digit_d[perm_k(c)] key_b[k][d][i][c] + [P] b[i][perm_k(c)] stay in
// registers (_kskip + pmodup, ckks.py:450-465, 478-489, 699-711).  Then per
// giant group j the MB diagonals of row i stream in (ring NSG giants deep) and
//   acc_u[j] = sum_k diag[j][k] u_k,  acc_v[j] = sum_k diag[j][k] v_k.
#ifndef CKB200_BM_NSB
#define CKB200_BM_NSB 2
#endif
#ifndef CKB200_BM_NSG
#define CKB200_BM_NSG 2
#endif
#ifndef CKB200_BM_NT
#define CKB200_BM_NT 128
#endif
constexpr int kBmNT = CKB200_BM_NT, kBmNSB = CKB200_BM_NSB, kBmNSG = CKB200_BM_NSG, kBmMB = 16;
template <int BETA>
constexpr size_t bsgs_mac_smem() {
  return (size_t)(kBmNSB * 3 * BETA + kBmNSG * kBmMB) * kBmNT * 8 + (2 * kBmMB + 512) * 8;
}

template <int BETA>
#ifndef CKB200_BM_MINB
#define CKB200_BM_MINB 2
#endif
__global__ void __launch_bounds__(kBmNT, CKB200_BM_MINB) bsgs_mac_kernel(BsgsMacArgs a) {
  constexpr int NT = kBmNT, MB = kBmMB, NSB = kBmNSB, NSG = kBmNSG;
  extern __shared__ __align__(16) u64 bsm[];
  u64 (*bs)[3 * BETA][NT] = (u64 (*)[3 * BETA][NT])bsm;                       // [NSB][3 BETA][NT]
  u64 (*gs)[MB][NT] = (u64 (*)[MB][NT])(bsm + NSB * 3 * BETA * NT);          // [NSG][MB][NT]
  const u64** kbp = (const u64**)(bsm + (NSB * 3 * BETA + NSG * MB) * NT);   // [MB]
  const u64** kap = kbp + MB;                                                 // [MB]
  const u64** dps = kap + MB;                                                 // [giant][baby]
  const DiagArgs& d = a.d;
  const int n = 1 << d.logn;
  const int c = blockIdx.x * NT + threadIdx.x;
  const int i = blockIdx.y;
  const int t = threadIdx.x;
  const int baby = d.baby, giant = d.giant;
  for (int e = t; e < baby; e += NT) {
    kbp[e] = a.key_b_ptrs[e];
    kap[e] = a.key_a_ptrs[e];
  }
  for (int e = t; e < giant * baby; e += NT)
    dps[e] = d.diag_ptrs[(long long)(e / baby) * d.diag_stride + e % baby];
  __syncthreads();
  if (c >= n) return;
  const int prime = d.prime[i];
  const PrimeConst P = d.pc[prime];
  const long long rowN = (long long)d.R << d.logn;
  const long long off = ((long long)i << d.logn) + c;
  const long long koff = ((long long)prime << d.logn) + c;  // key row i == prime index
  const bool chain = i < d.l;
  // baby k's operands -> ring slot k % NSB (one commit group per baby, possibly empty)
  auto stage_baby = [&](int k) {
    if (k < baby) {
      const int s = k % NSB;
      const u32 src = automorph_src((u32)c, (u32)d.galois[k], d.logn);
      const u64* dg = a.digits + ((long long)i << d.logn) + src;
#pragma unroll
      for (int dd = 0; dd < BETA; ++dd) {
        cp_async8(&bs[s][dd][t], dg + dd * a.digit_stride);
        cp_async8(&bs[s][BETA + dd][t], kap[k] + dd * a.key_digit_stride + koff);
        cp_async8(&bs[s][2 * BETA + dd][t], kbp[k] + dd * a.key_digit_stride + koff);
      }
    }
    cp_async_commit();
  };
  auto stage_giant = [&](int j) {
    if (j < giant) {
      const int s = j % NSG;
#pragma unroll
      for (int k = 0; k < MB; ++k)
        if (k < baby) cp_async8(&gs[s][k][t], dps[j * baby + k] + off);
    }
    cp_async_commit();
  };
  const ulonglong2 pm = chain ? d.pmod[i] : make_ulonglong2(0, 0);
  u64 x[2 * MB];
#pragma unroll
  for (int k = 0; k < NSB - 1; ++k) stage_baby(k);
#pragma unroll
  for (int k = 0; k < MB; ++k) {
    stage_baby(k + NSB - 1);
    cp_async_wait<NSB - 1>();
    if (k < baby) {
      const int s = k % NSB;
      Acc3 su, sv;
      acc3_zero(su);
      acc3_zero(sv);
#pragma unroll
      for (int dd = 0; dd < BETA; ++dd) {
        const u64 dv = bs[s][dd][t], ka = bs[s][BETA + dd][t], kb = bs[s][2 * BETA + dd][t];
        const u32 d0 = lo30(dv), d1 = hi30(dv);
        acc3_mac(su, d0, d1, lo30(ka), hi30(ka));
        acc3_mac(sv, d0, d1, lo30(kb), hi30(kb));
      }
      x[2 * k] = acc3_reduce(su, P);
      u64 v = acc3_reduce(sv, P);
      if (chain) {
        const u64 bv = d.b[((long long)i << d.logn) +
                           automorph_src((u32)c, (u32)d.galois[k], d.logn)];
        v = addmod(v, shoup(bv, pm.x, pm.y, P.q), P.q);
      }
      x[2 * k + 1] = v;
    }
  }
  // drain the (empty) baby groups, then stream the giant groups' diagonals
  cp_async_wait<0>();
#pragma unroll
  for (int j = 0; j < NSG - 1; ++j) stage_giant(j);
#pragma unroll 1
  for (int j = 0; j < giant; ++j) {
    stage_giant(j + NSG - 1);
    cp_async_wait<NSG - 1>();
    const int s = j % NSG;
    u64 yu = d.accumulate ? d.acc[(2LL * j) * rowN + off] : 0;
    u64 yv = d.accumulate ? d.acc[(2LL * j + 1) * rowN + off] : 0;
#pragma unroll
    for (int k0 = 0; k0 < MB; k0 += 8) {
      if (k0 >= baby) continue;
      Acc3 su, sv;
      acc3_zero(su);
      acc3_zero(sv);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int k = k0 + kk;
        if (k < baby) {
          const u64 mv = gs[s][k][t];
          const u32 m0 = lo30(mv), m1 = hi30(mv);
          acc3_mac(su, m0, m1, lo30(x[2 * k]), hi30(x[2 * k]));
          acc3_mac(sv, m0, m1, lo30(x[2 * k + 1]), hi30(x[2 * k + 1]));
        }
      }
      yu = addmod(yu, acc3_reduce(su, P), P.q);
      yv = addmod(yv, acc3_reduce(sv, P), P.q);
    }
    d.acc[(2LL * j) * rowN + off] = yu;
    d.acc[(2LL * j + 1) * rowN + off] = yv;
  }
}

int launch_bsgs_mac(const BsgsMacArgs& a, cudaStream_t st) {
  const DiagArgs& d = a.d;
  if (d.baby < 1 || d.baby > kBmMB || d.giant < 1 || d.giant * d.baby > 512 || a.beta < 1 ||
      a.beta > 4 || !d.diag_ptrs || !a.key_b_ptrs || !a.key_a_ptrs || d.logn < 7)
    return -1;
  count_launches(1);
  const int n = 1 << d.logn;
  const dim3 grid((n + kBmNT - 1) / kBmNT, d.R);
#define CK_BM(B)                                                                            \
  do {                                                                                      \
    static unsigned done = 0;                                                               \
    int dev = 0;                                                                            \
    cudaGetDevice(&dev);                                                                    \
    if (dev >= 32 || !((done >> dev) & 1u)) {                                               \
      cudaFuncSetAttribute(bsgs_mac_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)bsgs_mac_smem<B>());                                        \
      if (dev < 32) __atomic_fetch_or(&done, 1u << dev, __ATOMIC_RELAXED);                  \
    }                                                                                       \
    bsgs_mac_kernel<B><<<grid, kBmNT, bsgs_mac_smem<B>(), st>>>(a);                        \
  } while (0)
  switch (a.beta) {
    case 1: CK_BM(1); break;
    case 2: CK_BM(2); break;
    case 3: CK_BM(3); break;
    default: CK_BM(4); break;
  }
#undef CK_BM
  return (int)cudaGetLastError();
}

}  // namespace ck
