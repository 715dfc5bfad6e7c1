// 64-bit modular arithmetic on CUDA cores for word-sized NTT primes (q < 2^60).
//
// Replaces the reference's numpy vector ops (zq.py:145-194).  Every routine
// returns the exact residue (canonical once fully reduced), so results are
// bit-identical to the reference's float80-estimate mulmod (zq.py:161-177)
// regardless of the reduction method used here.
//
// Lazy ("Harvey") ranges are used inside NTT butterflies: values live in
// [0, 2q) or [0, 4q) between stages; 4q < 2^62 for q < 2^60.
#pragma once
#include <cstdint>

typedef unsigned long long u64;
typedef unsigned int u32;

#define CK_HD __host__ __device__ __forceinline__
#define CK_D __device__ __forceinline__

// Per-prime constants, built on the host (plan.cpp) and read from global memory.
struct PrimeConst {
  u64 q;
  u64 two_q;
  u64 bar;        // floor(2^64 / q)           (Shoup companion of 1)
  u64 c30, c30p;  // 2^30 mod q, Shoup companion
  u64 c60, c60p;  // 2^60 mod q, Shoup companion
  u64 r64, r64p;  // 2^64 mod q, Shoup companion
  u64 ninv, ninvp;
  u64 nq;         // 2^64 - q
  u64 mu;         // floor(2^(sh + 64) / q), sh = bitlen(q) - 1   (128-bit Barrett, acc3_reduce)
  u64 sh;
};

CK_D u64 mulhi64(u64 a, u64 b) { return __umul64hi(a, b); }

// x * w mod q in [0, 2q) for ANY 64-bit x; w < q, wp = floor(w * 2^64 / q).
CK_D u64 shoup_lazy(u64 x, u64 w, u64 wp, u64 q) {
  u64 qh = mulhi64(x, wp);
  return x * w - qh * q;
}

CK_D u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }

// 2^64 - q as a value the compiler cannot see through (it would otherwise rewrite
// Q * (0 - q) as -(Q * q) and undo the single multiply-accumulate chain)
CK_D u64 neg_opaque(u64 q) {
  u64 r = 0 - q;
  asm("mov.b64 %0, %0;" : "+l"(r));
  return r;
}

// NTT twiddle product in [0, 2q) for any 64-bit x (same contract as
// shoup_lazy).  A variant with an approximate quotient (dropping the low
// partial products) was measured 39% slower on C3 (register spills in the
// 64-register NTT kernels) and removed; see DESIGN.md.
CK_D u64 madw(u32 a, u32 b, u64 acc);
CK_D u64 shoup_tw(u64 x, u64 w, u64 wp, u64 q, u64 two_q) {
  // x w - Q q as ONE multiply-accumulate chain with 2^64 - q (no negation / recombination:
  // 7% fewer instructions per radix-16 pass than x * w - Q * q)
  return x * w + __umul64hi(x, wp) * neg_opaque(q);
}

CK_D u64 shoup(u64 x, u64 w, u64 wp, u64 q) { return csub(shoup_lazy(x, w, wp, q), q); }

CK_D u64 addmod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
CK_D u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// Any 64-bit x reduced into [0, 2q).
CK_D u64 red64_lazy(u64 x, const PrimeConst& P) { return x - mulhi64(x, P.bar) * P.q; }
CK_D u64 red64(u64 x, const PrimeConst& P) { return csub(red64_lazy(x, P), P.q); }

// Full 128-bit value (hi:lo) mod q.
CK_D u64 red128(u64 hi, u64 lo, const PrimeConst& P) {
  u64 r = shoup_lazy(hi, P.r64, P.r64p, P.q) + red64_lazy(lo, P);  // < 4q
  r = csub(r, P.two_q);
  return csub(r, P.q);
}

CK_D u64 mulmod(u64 a, u64 b, const PrimeConst& P) {
  return red128(mulhi64(a, b), a * b, P);
}

// 30-bit split accumulators: for a, b < 2^60 the product is
//   a0 b0 + (a0 b1 + a1 b0) 2^30 + a1 b1 2^60,  pieces < 2^30.
// Up to 8 products accumulate without overflow (mid term: 16 partials < 2^64).
// acc + (u64)a * b with a, b < 2^32: exactly one IMAD.WIDE.U32 (plain C++
// `acc += (u64)a * b` makes nvcc emit extra zero-high-word adds).
CK_D u64 madw(u32 a, u32 b, u64 acc) {
  u64 d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(acc));
  return d;
}

struct Acc3 {
  u64 lo, mid, hi;
};
CK_D void acc3_zero(Acc3& s) { s.lo = s.mid = s.hi = 0; }
CK_D void acc3_mac(Acc3& s, u32 a0, u32 a1, u32 b0, u32 b1) {
  s.lo = madw(a0, b0, s.lo);
  s.mid = madw(a0, b1, s.mid);
  s.mid = madw(a1, b0, s.mid);
  s.hi = madw(a1, b1, s.hi);
}
CK_D u32 lo30(u64 x) { return (u32)x & 0x3fffffffu; }
CK_D u32 hi30(u64 x) { return (u32)(x >> 30); }

// Reduce V = lo + mid*2^30 + hi*2^60 (V < 2^64 * 2^sh, i.e. at most 8 products of a
// value below 2^60 with a residue): assemble the exact 128-bit value with funnel
// shifts and carries (ALU pipe), then ONE Barrett step on its top 64 bits:
//   Vt = floor(V / 2^sh), Q = floor(Vt mu / 2^64) in (V/q - 3, V/q]
// (dropped bits of V: < 2^sh/q <= 1; mu's floor: Vt/2^64 < 1; the last floor: < 1),
// so V - Q q (mod 2^64) lies in [0, 3q).  One 64-bit high product and one low
// product instead of the two Shoup-style steps of red128.
CK_D u64 acc3_reduce_lazy(const Acc3& s, const PrimeConst& P) {
  u64 lo = s.lo, hi = 0;
  const u64 m_lo = s.mid << 30, m_hi = s.mid >> 34;
  const u64 h_lo = s.hi << 60, h_hi = s.hi >> 4;
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(m_lo), "l"(m_hi));
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(h_lo), "l"(h_hi));
  const int sh = (int)P.sh;  // 49 .. 59
  const u64 vt = (hi << (64 - sh)) | (lo >> sh);
  return lo - mulhi64(vt, P.mu) * P.q;
}
CK_D u64 acc3_reduce(const Acc3& s, const PrimeConst& P) {
  return csub(csub(acc3_reduce_lazy(s, P), P.two_q), P.q);
}

// ---- NTT butterflies (Harvey lazy) ----
// Forward CT: X, Y in [0, 4q) -> [0, 4q).
CK_D void bfly_ct(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 two_q) {
  u64 x = csub(X, two_q);
  u64 t = shoup_tw(Y, w, wp, q, two_q);
  X = x + t;
  Y = x - t + two_q;
}
// Inverse GS: X, Y in [0, 2q) -> [0, 2q).
CK_D void bfly_gs(u64& X, u64& Y, u64 w, u64 wp, u64 q, u64 two_q) {
  u64 x = X, y = Y;
  X = csub(x + y, two_q);
  Y = shoup_tw(x - y + two_q, w, wp, q, two_q);
}

// ---- small-prime forward butterfly (q < 2^54) ----
// Approximate Shoup quotient from three 32-bit products (the low x low product
// and the carries of the cross terms are dropped): Q in [floor(y wp / 2^64) - 2,
// floor(y wp / 2^64)], so t = y w - Q q lies in [0, 4q) for ANY 64-bit y.
// With nq = 2^64 - q the remainder is one multiply-accumulate chain
// (y w + Q nq mod 2^64), no negation.  Values grow by 4q per level and are
// never folded: a row phase of up to 10 levels starting below 16q stays
// below 56q < 2^60 (the bound the 30-bit-split key MAC needs).
CK_D u64 shoup_tw4(u64 y, u64 w, u64 wp, u64 nq) {
  // explicit 32-bit products (plain C++ makes nvcc emit 64-bit multiplies of the
  // shifted halves and re-roll the unrolled butterfly loops around them)
  u32 y0, y1, p0, p1, h1, h2;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(y0), "=r"(y1) : "l"(y));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(p0), "=r"(p1) : "l"(wp));
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(h1) : "r"(y0), "r"(p1));
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(h2) : "r"(y1), "r"(p0));
  u64 Q;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(Q) : "r"(y1), "r"(p1));
  Q += (u64)h1 + h2;
  return y * w + Q * nq;
}
CK_D void bfly_ct4(u64& X, u64& Y, u64 w, u64 wp, u64 nq, u64 q4) {
  const u64 t = shoup_tw4(Y, w, wp, nq);
  const u64 xx = X;
  X = xx + t;
  Y = xx - t + q4;
}
// Inverse (Gentleman-Sande) counterpart: no conditional subtraction on the sum, so
// values double per level (inputs of level k below 2^(k+1) q, B = 2^(k+1) q keeps the
// difference non-negative); the product is back in [0, 4q).
CK_D void bfly_gs4(u64& X, u64& Y, u64 w, u64 wp, u64 nq, u64 B) {
  const u64 x = X, y = Y;
  X = x + y;
  Y = shoup_tw4(x - y + B, w, wp, nq);
}
// true when the no-fold forward row phase applies to this prime
CK_D bool small_prime(u64 q) { return (q >> 54) == 0; }
// ... and the no-fold inverse row phase of 2^P2-point rows (outputs below 2^(P2+1) q)
CK_D bool small_prime_inv(u64 q, int p2) { return small_prime(q) && (q >> (63 - p2)) == 0; }

// ---- index helpers ----
CK_D u32 brev_bits(u32 x, int bits) { return bits ? (__brev(x) >> (32 - bits)) : 0u; }

// Eval-domain Galois gather: out[i] = in[perm(i)],
// perm(i) = br(((t * (2 br(i) + 1)) mod 2N - 1) / 2)   (rnspoly.py:127-135).
CK_D u32 automorph_src(u32 i, u32 t, int logn) {
  u32 j = brev_bits(i, logn);
  // only the product mod 2N <= 2^31 is needed: 32-bit wrap-around IMAD
  u32 e = (t * (2u * j + 1u)) & ((2u << logn) - 1u);
  return brev_bits((e - 1u) >> 1, logn);
}

// Bulk L2 prefetch (sm_90+): pull `bytes` (multiple of 16, 16-B aligned)
// toward L2 without touching shared memory or registers.
CK_D void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// TMA bulk copies (cp.async.bulk, no tensor map): `bytes` (multiple of 16,
// 16-B aligned) global -> shared, completion counted on an mbarrier.
CK_D void mbar_init(void* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(count) : "memory");
}
CK_D void mbar_expect_tx(void* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)), "r"(bytes) : "memory");
}
CK_D void bulk_g2s(void* dst, const void* src, unsigned bytes, void* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
               "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}
CK_D void mbar_wait_parity(void* bar, unsigned phase) {
  asm volatile("{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@!P1 bra WAIT_%=;\n\t}\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(phase) : "memory");
}

// Ampere-style async copies (LDGSTS): 8-byte global -> shared, grouped.
CK_D void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
CK_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
CK_D void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
