// Negacyclic NTT / INTT for one RNS limb row of N = 2^logn uint64 residues.
//
// Semantics are those of the reference NttContext (rnspoly.py:48-79):
// forward = Cooley-Tukey DIT with bit-reversed twiddles tw[m + block]
// (natural in, bit-reversed out); inverse = Gentleman-Sande ladder with
// itw[h + block], then * n^-1 (here: * a per-row scale, n^-1 times an
// optional extra constant such as the ModUp/ModDown ihat, folded exactly).
//
// B200 layout: a limb (512 KB at N=2^16) does not fit one SM, so the
// transform is split as N = 2^P1 x 2^P2 over the storage matrix
// x[r * 2^P2 + c]:
//   * column phase: stages with m < 2^P1 only mix rows of one column
//     (twiddles tw[1 .. 2^P1) shared by all columns, staged in SMEM);
//   * row phase: stages with m >= 2^P1 only mix a contiguous row of 2^P2
//     elements (twiddles for that row read through L1/L2).
// Inside a phase each thread keeps E = 16 elements in registers and runs up
// to 4 radix-2 stages on them (a radix-16 pass); passes exchange through
// shared memory.  Arithmetic: 64-bit Shoup/Harvey lazy butterflies
// (modarith.cuh), values in [0,4q) between stages, canonical on output.
#pragma once
#include "modarith.cuh"

namespace ck {

constexpr int kElog = 4;
constexpr int kE = 1 << kElog;  // elements per thread
constexpr int kTC = 16;         // columns per column-phase CTA (128 B rows)
// columns per column-phase CTA for a 2^P1-row column: 16 up to 256 rows, fewer
// above so the CTA's shared tile (2^P1 x TC words) stays within 32 KB
template <int P1>
CK_HD constexpr int col_tc() { return P1 <= 8 ? kTC : (P1 == 9 ? 8 : 4); }

struct NttArgs {
  u64* data;
  const int* prime_idx;        // per job: index into the plan's prime table
  const long long* row_off;    // per job: element offset of the limb (nullable: job*N)
  const PrimeConst* pc;
  const ulonglong2* tw;        // [prime][N] {w, w_shoup}, forward
  const ulonglong2* itw;       // [prime][N] inverse
  const ulonglong2* scale;     // per job {s, s_shoup} applied after INTT (nullable: n^-1)
  long long batch_stride;      // elements between batch items (grid.z)
  const u64* src;              // row kernels: read input from here (nullable: in place)
  long long src_batch_stride;  //   with this batch stride (rows at job*N)
  int logn;
  // tensor-core forward column phase (ntt_tc.cu; nullable: butterfly kernels)
  const unsigned char* tcB = nullptr;  // [prime][2][128 x 128 B] B1 | B2 in SMEM layout
  const ulonglong2* tcD = nullptr;     // [prime][2][16][16] twists {d, d_shoup}
};

// ---- compile-time pass schedule for a 2^P-point sub-transform ----
template <int P>
struct Sched {
  static constexpr int np = (P + kElog - 1) / kElog;
  static constexpr int C(int p) { return p < np - 1 ? kElog : P - kElog * (np - 1); }
  static constexpr int sumC(int p) { return p < 0 ? 0 : C(p) + sumC(p - 1); }
  // log2 of the smallest in-pass distance
  static constexpr int logD(int p, bool inv) { return inv ? sumC(p - 1) : P - sumC(p); }
};

// Sub-index (within the 2^P-point sub-transform) of register r of thread g.
template <int P, int p, bool INV>
CK_D int sub_index(int g, int r) {
  constexpr int C = Sched<P>::C(p);
  constexpr int LD = Sched<P>::logD(p, INV);
  constexpr int NG = kE >> C;
  const int h = r >> C, k = r & ((1 << C) - 1);
  const int gamma = g * NG + h;
  const int blk = gamma >> LD, lo = gamma & ((1 << LD) - 1);
  return (blk << (LD + C)) + lo + (k << LD);
}

// One register pass.  j(s) = jbase + (s << JSHIFT) is the limb-global index.
// Forward passes skip the per-butterfly correction: inputs in [0, 8q) grow
// by 2q per stage to < 16q < 2^64 (q < 2^60); the caller folds them back
// with one csub(8q) per element per pass (fwd_fold) -- half the ALU work of
// Harvey's per-butterfly correction.
// SMALL (row phases, q < 2^54): approximate-quotient butterflies without any
// range folding (modarith.cuh bfly_ct4 / bfly_gs4); q / two_q then carry
// 2^64 - q and 4q (forward) or q (inverse; inputs below 2q).
template <int P, int p, bool INV, bool TW_SMEM, int LOGN, int JSHIFT, bool SMALL = false>
CK_D void run_pass(u64 (&x)[kE], int g, int jbase, const ulonglong2* __restrict__ tw, u64 q,
                   u64 two_q) {
  static_assert(!SMALL || JSHIFT == 0, "small-prime variant: row phases only");
  constexpr int C = Sched<P>::C(p);
  constexpr int LD = Sched<P>::logD(p, INV);
  constexpr int NG = kE >> C;
#pragma unroll
  for (int h = 0; h < NG; ++h) {
    const int s0 = sub_index<P, p, INV>(g, h << C);
#pragma unroll
    for (int st = 0; st < C; ++st) {
      // forward: distances shrink (half = 2^(C-1-st)); inverse: grow (2^st)
      const int lhalf = INV ? st : (C - 1 - st);
      const int half = 1 << lhalf;
      const int logt = LD + lhalf + JSHIFT;  // log2 of limb-global distance
      const int logm = LOGN - 1 - logt;      // stage m (fwd) or h (inv)
#pragma unroll
      for (int b = 0; b < (1 << C) / (2 * half); ++b) {
        const int k0 = b * 2 * half;
        const int j = jbase + ((s0 + (k0 << LD)) << JSHIFT);
        const int idx = (1 << logm) + (j >> (logt + 1));
        ulonglong2 w;
        if (TW_SMEM) w = tw[idx];
        else w = __ldg(tw + idx);
#pragma unroll
        for (int k = k0; k < k0 + half; ++k) {
          u64& X = x[(h << C) + k];
          u64& Y = x[(h << C) + k + half];
          if (INV && SMALL) {
            bfly_gs4(X, Y, w.x, w.y, q, two_q << (LD + lhalf + 1));
          } else if (INV) {
            bfly_gs(X, Y, w.x, w.y, q, two_q);
          } else if (SMALL) {
            bfly_ct4(X, Y, w.x, w.y, q, two_q);
          } else {
            const u64 t = shoup_tw(Y, w.x, w.y, q, two_q);
            const u64 xx = X;
            X = xx + t;
            Y = xx - t + two_q;
          }
        }
      }
    }
  }
}

// Forward lazy range maintenance: [0, 16q) -> [0, 8q).
CK_D void fwd_fold(u64 (&x)[kE], u64 q8) {
#pragma unroll
  for (int r = 0; r < kE; ++r) x[r] = csub(x[r], q8);
}
// [0, 16q) -> [0, q)
CK_D u64 fwd_final(u64 v, u64 q) {
  v = csub(v, q << 3);
  v = csub(v, q << 2);
  v = csub(v, q << 1);
  return csub(v, q);
}

// ---------------------------------------------------------------- row helpers
// A "row" is 2^P2 contiguous elements held by G = 2^P2/16 threads (thread g);
// srow is that row's padded shared-memory slice (row_stride<P2>() entries).
template <int P2>
CK_HD constexpr int row_stride() { return (1 << P2) + (1 << P2) / 16; }
CK_D int sidx(int s) { return s + (s >> 4); }

template <int P2, int p, bool INV>
CK_D void row_to_smem(const u64 (&x)[kE], int g, u64* srow) {
#pragma unroll
  for (int r = 0; r < kE; ++r) srow[sidx(sub_index<P2, p, INV>(g, r))] = x[r];
}
template <int P2, int p, bool INV>
CK_D void row_from_smem(u64 (&x)[kE], int g, const u64* srow) {
#pragma unroll
  for (int r = 0; r < kE; ++r) x[r] = srow[sidx(sub_index<P2, p, INV>(g, r))];
}

// Full row phase of a forward (INV=false) or inverse transform.  On entry x
// holds the pass-0 layout, on exit the last-pass layout.  Contains
// __syncthreads(): every thread of the CTA must call it.  Forward inputs may
// be lazy in [0, 16q); forward outputs are lazy in [0, 16q) (fwd_final to
// finish); inverse inputs/outputs are in [0, 2q).
// Barrier policies for row_transform: the whole CTA, or one warp group
// (named barrier ID over NT threads) in warp-specialised kernels.
struct SyncCta {
  CK_D static void sync() { __syncthreads(); }
};
template <int ID, int NT>
struct SyncGroup {
  CK_D static void sync() { asm volatile("bar.sync %0, %1;" ::"r"(ID), "r"(NT) : "memory"); }
};
CK_D void bar_sync_n(int id, int nt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nt) : "memory"); }
CK_D void bar_arrive_n(int id, int nt) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nt) : "memory");
}

// The lone 9th level of a 512-point row (P = 9: passes of 4 + 4 + 1 levels) without
// a third shared-memory round trip: in the pass-1 layout a row is one warp and the
// level's partner elements sit in lane g^1 (forward, distance 1) or g^16 (inverse,
// distance 256) at the SAME register index.  The lower lane computes the pairs of
// registers k < 8, the upper lane those of k >= 8 (8 butterflies each, no
// divergence): one shuffle brings each lane the other operand, one more returns
// the partner's result.  Values stay in the pass-1 layout (RowLast<9> = 1).
CK_D u64 shfl_xor64(u64 v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

template <int P, bool INV, int LOGN, bool SMALL = false>
CK_D void last_level_shfl(u64 (&x)[kE], int g, int jbase, const ulonglong2* __restrict__ tw,
                          u64 q, u64 two_q) {
  static_assert(P == 9 && kE == 16, "512-point rows: 32 threads = one warp per row");
  constexpr int X = INV ? 16 : 1;  // lane distance of the partner
  const bool lower = (g & X) == 0;  // holds the pairs' first (lower-index) elements
  if (!INV && !SMALL) fwd_fold(x, q << 3);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const u64 recv = shfl_xor64(lower ? x[kk + 8] : x[kk], X);
    const int k = lower ? kk : kk + 8;
    u64 xv = lower ? x[kk] : recv;        // first element of pair k
    u64 yv = lower ? recv : x[kk + 8];    // second element of pair k
    const int j = jbase + sub_index<P, 1, INV>(g & ~X, k);
    if (!INV) {
      const ulonglong2 w = __ldg(tw + (1 << (LOGN - 1)) + (j >> 1));
      if (SMALL) {
        bfly_ct4(xv, yv, w.x, w.y, q, two_q);
      } else {
        const u64 t = shoup_tw(yv, w.x, w.y, q, two_q);
        const u64 xx = xv;
        xv = xx + t;
        yv = xx - t + two_q;
      }
    } else {
      const ulonglong2 w = __ldg(tw + (1 << (LOGN - 9)) + (j >> 9));
      if (SMALL) bfly_gs4(xv, yv, w.x, w.y, q, two_q << 9);
      else bfly_gs(xv, yv, w.x, w.y, q, two_q);
    }
    const u64 back = shfl_xor64(lower ? yv : xv, X);
    if (lower) {
      x[kk] = xv;
      x[kk + 8] = back;
    } else {
      x[kk + 8] = yv;
      x[kk] = back;
    }
  }
}

// Pass whose layout holds a row's final values (row_to_smem after row_transform).
template <int P>
struct RowLast {
  static constexpr int value = P == 9 ? 1 : Sched<P>::np - 1;
};

// SMALL (forward, q < 2^54): inputs below 16q, outputs below (16 + 4 P2) q, no
// folding; pass 2^64 - q and 4q in place of q and 2q.
template <int P2, bool INV, int LOGN, class Sync = SyncCta, bool SMALL = false>
CK_D void row_transform(u64 (&x)[kE], int g, int jbase, u64* srow,
                        const ulonglong2* __restrict__ tw, u64 q, u64 two_q) {
  constexpr int NP = Sched<P2>::np;
  static_assert(NP <= 3, "row too long");
  constexpr bool FOLD = !INV && !SMALL;
  if (FOLD) fwd_fold(x, q << 3);
  run_pass<P2, 0, INV, false, LOGN, 0, SMALL>(x, g, jbase, tw, q, two_q);
  if constexpr (NP > 1) {
    Sync::sync();
    row_to_smem<P2, 0, INV>(x, g, srow);
    Sync::sync();
    row_from_smem<P2, 1, INV>(x, g, srow);
    if (FOLD) fwd_fold(x, q << 3);
    run_pass<P2, 1, INV, false, LOGN, 0, SMALL>(x, g, jbase, tw, q, two_q);
  }
  if constexpr (P2 == 9) {
    last_level_shfl<P2, INV, LOGN, SMALL>(x, g, jbase, tw, q, two_q);
  } else if constexpr (NP > 2) {
    Sync::sync();
    row_to_smem<P2, 1, INV>(x, g, srow);
    Sync::sync();
    row_from_smem<P2, 2, INV>(x, g, srow);
    if (FOLD) fwd_fold(x, q << 3);
    run_pass<P2, 2, INV, false, LOGN, 0, SMALL>(x, g, jbase, tw, q, two_q);
  }
}

}  // namespace ck
