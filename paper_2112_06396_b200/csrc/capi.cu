// C ABI: plan creation (host tables) and the key-switching pipeline.
//
// Host-side table construction restates, with exact 128-bit integer
// arithmetic, the reference's setup code:
//   psi / twiddles ........ zq.primitive_root_2n (zq.py:79-84),
//                           NttContext.__init__ (rnspoly.py:34-46)
//   BC tables ............. _bc_tables (rnspoly.py:248-261),
//                           _bc_center_tables (rnspoly.py:290-300)
//   digit spans / rows .... CkksParams.digit_spans (ckks.py:56-62),
//                           _key_rows (ckks.py:444-447)
//   P^-1, [P]_q ........... _moddown_poly (ckks.py:411-416), pmodup (ckks.py:478-489)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "ck_internal.h"
#include "ntt.cuh"

typedef unsigned __int128 u128;

#include <atomic>
static std::atomic<long long> g_launches{0};
namespace ck {
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("CKB200_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace ck

namespace {

// ------------------------------------------------------------ host number theory
u64 mulmod_h(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
u64 powmod_h(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod_h(r, a, q);
    a = mulmod_h(a, a, q);
    e >>= 1;
  }
  return r;
}
u64 invmod_h(u64 a, u64 q) { return powmod_h(a, q - 2, q); }
u64 shoup_h(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

bool isprime_h(u64 n) {
  if (n < 2) return false;
  static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (u64 p : bases)
    if (n % p == 0) return n == p;
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) { d >>= 1; ++r; }
  for (u64 a : bases) {
    u64 x = powmod_h(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < r; ++i) {
      x = mulmod_h(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}

// Pollard-rho (Brent) factor finding: q - 1 for any q < 2^60 factors in
// milliseconds (trial division to sqrt(q-1) is quadratic-time for unlucky primes)
u64 rho_factor(u64 n) {
  if (n % 2 == 0) return 2;
  for (u64 c = 1;; ++c) {
    auto f = [&](u64 x) { return (u64)(((u128)x * x + c) % n); };
    u64 x = 2, y = 2, d = 1, q = 1, ys = 2;
    const u64 m = 128;
    u64 r = 1;
    do {
      x = y;
      for (u64 i = 0; i < r; ++i) y = f(y);
      u64 k = 0;
      do {
        ys = y;
        for (u64 i = 0; i < m && i < r - k; ++i) {
          y = f(y);
          q = (u64)((u128)q * (x > y ? x - y : y - x) % n);
        }
        u64 a = q, b = n;
        while (b) { const u64 t = a % b; a = b; b = t; }
        d = a;
        k += m;
      } while (k < r && d == 1);
      r <<= 1;
    } while (d == 1);
    if (d == n) {  // backtrack one step at a time
      do {
        ys = f(ys);
        u64 a = x > ys ? x - ys : ys - x, b = n;
        while (b) { const u64 t = a % b; a = b; b = t; }
        d = a;
      } while (d == 1);
    }
    if (d != n) return d;
  }
}

void factor_into(u64 m, std::vector<u64>& f) {
  if (m == 1) return;
  if (isprime_h(m)) {
    if (std::find(f.begin(), f.end(), m) == f.end()) f.push_back(m);
    return;
  }
  for (u64 p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull}) {
    if (m % p == 0) {
      if (std::find(f.begin(), f.end(), p) == f.end()) f.push_back(p);
      while (m % p == 0) m /= p;
      factor_into(m, f);
      return;
    }
  }
  const u64 d = rho_factor(m);
  factor_into(d, f);
  factor_into(m / d, f);
}

std::vector<u64> prime_factors(u64 m) {
  std::vector<u64> f;
  factor_into(m, f);
  std::sort(f.begin(), f.end());
  return f;
}

// psi = g^((q-1)/2N), g the smallest primitive root (== sympy.primitive_root)
u64 psi_for(u64 q, int logn) {
  const std::vector<u64> f = prime_factors(q - 1);
  for (u64 g = 2;; ++g) {
    bool ok = true;
    for (u64 p : f)
      if (powmod_h(g, (q - 1) / p, q) == 1) { ok = false; break; }
    if (ok) return powmod_h(g, (q - 1) >> (logn + 1), q);
  }
}

u32 brev_h(u32 x, int bits) {
  u32 r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

}  // namespace

// ------------------------------------------------------------------- plan types
struct ck_bconv {
  int ns = 0, nd = 0, centered = 0;
  int* d_src = nullptr;
  int* d_dst = nullptr;
  ulonglong2* d_ihat = nullptr;   // plain ihat (generic apply)
  uint4* d_T = nullptr;
  unsigned char* d_B5 = nullptr;  // tcgen05 B chunks (bconv_t5_kernel); null: CUDA-core kernel only
  double* d_w = nullptr;
  u64* d_kQ = nullptr;
  long long* d_out_off = nullptr; // optional
  std::vector<void*> allocs;
  ~ck_bconv() {
    for (void* p : allocs) cudaFree(p);
  }
};

namespace {

struct ModDownTab {
  bool valid = false;
  int keep = 0, ndrop = 0, drop_row0 = 0;
  ck_bconv* bc = nullptr;             // centered, drop -> keep
  ulonglong2* d_drop_scale = nullptr; // ihat * n^-1 per drop row
  long long* d_drop_off = nullptr;    // row offsets of the drop rows
  int* d_drop_prime = nullptr;
  int* d_keep_prime = nullptr;
  ulonglong2* d_pinv = nullptr;       // [P_drop]^-1 mod q_j per keep row
  ulonglong2* d_dinv = nullptr;       // (product of the dropped CHAIN primes)^-1 mod q_j per keep
                                      // row: pmodup(x) through this ModDown is x * d_dinv
};

struct LevelTab {
  int l = 0, beta = 0, R = 0;
  std::vector<int> lo, hi;
  int* d_chain_prime = nullptr;       // [l]
  int* d_raised_prime = nullptr;      // [R] (== full-basis key row)
  ulonglong2* d_modup_scale = nullptr;// [l] ihat(digit) * n^-1
  std::vector<ck_bconv*> modup_bc;    // per digit, targets = raised \ own
  long long* d_modup_ntt_off = nullptr;
  int* d_modup_ntt_prime = nullptr;
  int modup_ntt_jobs = 0;
  ulonglong2* d_pmod = nullptr;       // [P]_q per chain row
  ModDownTab md[3];
};

}  // namespace

struct ck_plan {
  int logn = 0, n = 0, L = 0, K = 0, dnum = 0, alpha = 0, key_digits = 0;
  bool fused = true;  // CKB200_UNFUSED=1 at plan creation selects the unfused pipeline
  int md_group = 4;   // md_row items per CTA (CKB200_MD_G)
  int bsgs_fused = 1; // fused baby KSKIP + diagonal MAC (CKB200_BSGS_FUSED=0: two kernels)
  int key_prefetch = 2;    // L2 prefetch of the first 2/8 of each key tile in ks_row (8/8: +4 GB DRAM re-reads; 2 best)
  int bc_tc = 1;      // CKB200_BCTC=0: CUDA-core base conversion instead of the tcgen05 form
  unsigned char* d_tcB = nullptr;  // tensor-core column-phase tables (ntt_tc.cu; CKB200_NTTTC=0 disables)
  ulonglong2* d_tcD = nullptr;
  std::vector<u64> mod, psi;
  PrimeConst* d_pc = nullptr;
  u64* d_mod = nullptr;    // full basis chain || special (key-row moduli)
  ulonglong2* d_tw = nullptr;
  ulonglong2* d_itw = nullptr;
  std::vector<LevelTab> lv;  // index = level
  std::vector<void*> allocs;
  std::vector<ck_bconv*> bcs;
  ~ck_plan() {
    for (ck_bconv* b : bcs) delete b;
    for (void* p : allocs) cudaFree(p);
  }
};

namespace {

template <class T>
T* upload(std::vector<void*>& allocs, const std::vector<T>& v, int* err) {
  if (v.empty()) return nullptr;
  void* p = nullptr;
  if (cudaMalloc(&p, v.size() * sizeof(T)) != cudaSuccess) { *err = CK_ERR_ALLOC; return nullptr; }
  allocs.push_back(p);
  cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return (T*)p;
}

PrimeConst make_pc(u64 q, int logn) {
  PrimeConst P;
  std::memset(&P, 0, sizeof(P));
  P.q = q;
  P.two_q = 2 * q;
  P.bar = (u64)(((u128)1 << 64) / q);
  P.c30 = ((u64)1 << 30) % q;
  P.c30p = shoup_h(P.c30, q);
  P.c60 = ((u64)1 << 60) % q;
  P.c60p = shoup_h(P.c60, q);
  P.r64 = (u64)(((u128)1 << 64) % q);
  P.r64p = shoup_h(P.r64, q);
  P.ninv = invmod_h(((u64)1 << logn) % q, q);
  P.ninvp = shoup_h(P.ninv, q);
  P.nq = (u64)0 - q;
  int bl = 0;
  while (bl < 64 && (q >> bl)) ++bl;
  P.sh = (u64)(bl - 1);
  P.mu = (u64)(((u128)1 << (P.sh + 64)) / q);  // q is not a power of two: < 2^64
  return P;
}

ulonglong2 sh2(u64 w, u64 q) { return make_ulonglong2(w, shoup_h(w, q)); }

// BC tables between plan primes (rnspoly.py:248-261, 290-300)
ck_bconv* build_bconv(ck_plan* p, const std::vector<int>& src, const std::vector<int>& dst,
                      bool centered, int* err) {
  ck_bconv* b = new ck_bconv();
  b->ns = (int)src.size();
  b->nd = (int)dst.size();
  b->centered = centered;
  std::vector<ulonglong2> ihat(src.size());
  std::vector<uint4> T(src.size() * dst.size());
  std::vector<double> w(src.size());
  for (size_t i = 0; i < src.size(); ++i) {
    const u64 qi = p->mod[src[i]];
    u64 prod = 1 % qi;  // (Q/q_i) mod q_i
    for (size_t k = 0; k < src.size(); ++k)
      if (k != i) prod = mulmod_h(prod, p->mod[src[k]] % qi, qi);
    ihat[i] = sh2(invmod_h(prod, qi), qi);
    for (size_t j = 0; j < dst.size(); ++j) {
      const u64 pj = p->mod[dst[j]];
      u64 t = 1 % pj;
      for (size_t k = 0; k < src.size(); ++k)
        if (k != i) t = mulmod_h(t, p->mod[src[k]] % pj, pj);
      // 30-bit pieces of T and of U = T * 2^30 mod p (bconv.cu: two accumulators)
      const u64 u = mulmod_h(t, (u64)1 << 30, pj);
      const u32 m30 = (1u << 30) - 1;
      T[i * dst.size() + j] = make_uint4((u32)t & m30, (u32)(t >> 30), (u32)u & m30, (u32)(u >> 30));
    }
    w[i] = 1.0 / (double)qi;  // Python: 1.0 / q  (q rounded to double first)
  }
  std::vector<u64> kQ(dst.size() * (src.size() + 1));
  for (size_t j = 0; j < dst.size(); ++j) {
    const u64 pj = p->mod[dst[j]];
    u64 qm = 1 % pj;
    for (size_t k = 0; k < src.size(); ++k) qm = mulmod_h(qm, p->mod[src[k]] % pj, pj);
    for (size_t k = 0; k <= src.size(); ++k) kQ[j * (src.size() + 1) + k] = mulmod_h(k % pj, qm, pj);
  }
  // tensor-core B matrix: B[(j,b)][(i,a)] = byte b of T_ij 2^{8a} mod p_j, in tcgen05
  // operand layout (bconv.cu bconv_t5_table)
  {
    const int ns = (int)src.size(), nd = (int)dst.size();
    std::vector<u64> Tp((size_t)ns * 8 * nd);  // [i][a][j]
    for (int i = 0; i < ns; ++i)
      for (int j = 0; j < nd; ++j) {
        const u64 pj = p->mod[dst[j]];
        const uint4 q4 = T[(size_t)i * nd + j];
        const u64 t = (u64)q4.x | ((u64)q4.y << 30);
        u64 sh = 1 % pj;
        for (int aa = 0; aa < 8; ++aa) {
          Tp[((size_t)i * 8 + aa) * nd + j] = mulmod_h(t, sh, pj);
          sh = mulmod_h(sh, 256 % pj, pj);
        }
      }
    // The epilogue quotient V/p must fit 31 bits: bound V = sum_b S_b 2^8b with
    // S_b <= Kp 255^2 (every K byte, padding included) and check V / p_j + 2 < 2^31
    // for every target (C3: p > 2^53; C5's 50-bit chain: 2^28.6); the quotient
    // window also shifts by floor(log2 p) - 32 >= 8.
    const int kp = ((8 * ns + 31) / 32) * 32;
    const double s_max = (double)kp * 255.0 * 255.0;
    const double v_max = s_max * 257.0 * (1.0 + 65536.0 + 4294967296.0 + 281474976710656.0);
    bool big = ns >= 1 && ns <= 16 && nd >= 1 && nd <= 64;
    for (int j = 0; j < nd; ++j)
      big = big && v_max / (double)p->mod[dst[j]] + 2.0 < 2147483648.0 &&
            p->mod[dst[j]] > ((u64)1 << 40);
    if (big) {
      std::vector<unsigned char> B5(ck::bconv_t5_table_bytes(ns, nd));
      ck::bconv_t5_table(Tp.data(), ns, nd, B5.data());
      b->d_B5 = upload(b->allocs, B5, err);
    }
  }
  b->d_src = upload(b->allocs, src, err);
  b->d_dst = upload(b->allocs, dst, err);
  b->d_ihat = upload(b->allocs, ihat, err);
  b->d_T = upload(b->allocs, T, err);
  b->d_w = upload(b->allocs, w, err);
  b->d_kQ = upload(b->allocs, kQ, err);
  return b;
}

void build_moddown(ck_plan* p, ModDownTab& t, const std::vector<int>& keep,
                   const std::vector<int>& drop, int drop_row0, int* err) {
  t.valid = true;
  t.keep = (int)keep.size();
  t.ndrop = (int)drop.size();
  t.drop_row0 = drop_row0;
  t.bc = build_bconv(p, drop, keep, true, err);
  p->bcs.push_back(t.bc);
  std::vector<ulonglong2> dscale(drop.size());
  std::vector<long long> doff(drop.size());
  for (size_t i = 0; i < drop.size(); ++i) {
    const u64 qi = p->mod[drop[i]];
    u64 prod = 1 % qi;
    for (size_t k = 0; k < drop.size(); ++k)
      if (k != i) prod = mulmod_h(prod, p->mod[drop[k]] % qi, qi);
    const u64 ninv = invmod_h((u64)p->n % qi, qi);
    dscale[i] = sh2(mulmod_h(invmod_h(prod, qi), ninv, qi), qi);
    doff[i] = (long long)(drop_row0 + (int)i) << p->logn;
  }
  std::vector<ulonglong2> pinv(keep.size()), dinv(keep.size());
  for (size_t j = 0; j < keep.size(); ++j) {
    const u64 qj = p->mod[keep[j]];
    u64 bp = 1 % qj;
    for (int d : drop) bp = mulmod_h(bp, p->mod[d] % qj, qj);
    pinv[j] = sh2(invmod_h(bp, qj), qj);
    u64 bc = 1 % qj;
    for (int d : drop)
      if (d < p->L) bc = mulmod_h(bc, p->mod[d] % qj, qj);
    dinv[j] = sh2(invmod_h(bc, qj), qj);
  }
  t.d_drop_scale = upload(p->allocs, dscale, err);
  t.d_drop_off = upload(p->allocs, doff, err);
  t.d_drop_prime = upload(p->allocs, drop, err);
  t.d_keep_prime = upload(p->allocs, keep, err);
  t.d_pinv = upload(p->allocs, pinv, err);
  t.d_dinv = upload(p->allocs, dinv, err);
}

int build_level(ck_plan* p, int l) {
  int err = 0;
  LevelTab& t = p->lv[l];
  t.l = l;
  t.R = l + p->K;
  for (int j = 0; j < l; j += p->alpha) {
    t.lo.push_back(j);
    t.hi.push_back(std::min(j + p->alpha, l));
  }
  t.beta = (int)t.lo.size();
  std::vector<int> chain(l), raised;
  for (int i = 0; i < l; ++i) chain[i] = i;
  raised = chain;
  for (int k = 0; k < p->K; ++k) raised.push_back(p->L + k);
  t.d_chain_prime = upload(p->allocs, chain, &err);
  t.d_raised_prime = upload(p->allocs, raised, &err);
  // ModUp: per digit, own = chain[lo:hi], targets = raised minus own (raised order)
  std::vector<ulonglong2> mscale(l);
  std::vector<long long> ntt_off;
  std::vector<int> ntt_prime;
  for (int d = 0; d < t.beta; ++d) {
    std::vector<int> own, tgt;
    std::vector<long long> out_off;
    for (int i = t.lo[d]; i < t.hi[d]; ++i) own.push_back(i);
    for (int r = 0; r < t.R; ++r) {
      if (r >= t.lo[d] && r < t.hi[d]) continue;
      tgt.push_back(raised[r]);
      out_off.push_back((long long)r << p->logn);
      ntt_off.push_back(((long long)d * t.R + r) << p->logn);
      ntt_prime.push_back(raised[r]);
    }
    ck_bconv* bc = build_bconv(p, own, tgt, false, &err);
    bc->d_out_off = upload(bc->allocs, out_off, &err);
    p->bcs.push_back(bc);
    t.modup_bc.push_back(bc);
    for (size_t i = 0; i < own.size(); ++i) {
      const u64 qi = p->mod[own[i]];
      u64 prod = 1 % qi;
      for (size_t k = 0; k < own.size(); ++k)
        if (k != i) prod = mulmod_h(prod, p->mod[own[k]] % qi, qi);
      const u64 ninv = invmod_h((u64)p->n % qi, qi);
      mscale[own[i]] = sh2(mulmod_h(invmod_h(prod, qi), ninv, qi), qi);
    }
  }
  t.d_modup_scale = upload(p->allocs, mscale, &err);
  t.d_modup_ntt_off = upload(p->allocs, ntt_off, &err);
  t.d_modup_ntt_prime = upload(p->allocs, ntt_prime, &err);
  t.modup_ntt_jobs = (int)ntt_off.size();
  // [P]_q per chain row (pmodup)
  std::vector<ulonglong2> pm(l);
  for (int i = 0; i < l; ++i) {
    u64 bp = 1 % p->mod[i];
    for (int k = 0; k < p->K; ++k) bp = mulmod_h(bp, p->mod[p->L + k] % p->mod[i], p->mod[i]);
    pm[i] = sh2(bp, p->mod[i]);
  }
  t.d_pmod = upload(p->allocs, pm, &err);
  // ModDown variants
  std::vector<int> spec;
  for (int k = 0; k < p->K; ++k) spec.push_back(p->L + k);
  if (p->K > 0) build_moddown(p, t.md[0], chain, spec, l, &err);
  if (l >= 2) {
    std::vector<int> keep(chain.begin(), chain.end() - 1), drop{l - 1};
    drop.insert(drop.end(), spec.begin(), spec.end());
    build_moddown(p, t.md[1], keep, drop, l - 1, &err);
    build_moddown(p, t.md[2], keep, std::vector<int>{l - 1}, l - 1, &err);
  }
  return err;
}

// ------------------------------------------------------------------ launchers
int ntt_rows(const ck_plan* p, u64* base, const int* prime, const long long* off,
             const ulonglong2* scale, int jobs, int batch, long long bstride, bool inv,
             cudaStream_t st) {
  ck::NttArgs a;
  a.data = base;
  a.prime_idx = prime;
  a.row_off = off;
  a.pc = p->d_pc;
  a.tw = p->d_tw;
  a.itw = p->d_itw;
  a.scale = scale;
  a.batch_stride = bstride;
  a.src = nullptr;
  a.src_batch_stride = 0;
  a.logn = p->logn;
  a.tcB = p->d_tcB;
  a.tcD = p->d_tcD;
  return ck::launch_ntt(a, jobs, batch, inv, st);
}

int ntt_phase(const ck_plan* p, u64* base, const int* prime, const long long* off,
              const ulonglong2* scale, int jobs, int batch, long long bstride, bool inv,
              int phase, cudaStream_t st, const u64* src = nullptr, long long src_bstride = 0) {
  ck::NttArgs a;
  a.data = base;
  a.prime_idx = prime;
  a.row_off = off;
  a.pc = p->d_pc;
  a.tw = p->d_tw;
  a.itw = p->d_itw;
  a.scale = scale;
  a.batch_stride = bstride;
  a.src = src;
  a.src_batch_stride = src_bstride;
  a.logn = p->logn;
  a.tcB = p->d_tcB;
  a.tcD = p->d_tcD;
  return ck::launch_ntt_phase(a, jobs, batch, inv, phase, st);
}

// lazy: a forward NTT consumes the outputs (it takes values below 4p; only the tcgen05
// kernel uses the flag, every other path writes canonical residues)
ck::BconvArgs bconv_args(const ck_plan* p, const ck_bconv* bc, const u64* in, long long in_batch,
                         u64* out, long long out_batch, bool prescale, bool lazy = false) {
  ck::BconvArgs a;
  a.in = in;
  a.in_batch = in_batch;
  a.in_off = nullptr;
  a.out = out;
  a.out_batch = out_batch;
  a.out_off = bc->d_out_off;
  a.src_prime = bc->d_src;
  a.dst_prime = bc->d_dst;
  a.pc = p->d_pc;
  a.src_scale = prescale ? bc->d_ihat : nullptr;
  a.T = bc->d_T;
  a.w = bc->d_w;
  a.kQ = bc->d_kQ;
  a.B5 = p->bc_tc ? bc->d_B5 : nullptr;
  a.ns = bc->ns;
  a.nd = bc->nd;
  a.logn = p->logn;
  a.centered = bc->centered;
  a.lazy_out = lazy ? 1 : 0;
  return a;
}

int bconv_run(const ck_plan* p, const ck_bconv* bc, const u64* in, long long in_batch,
              u64* out, long long out_batch, bool prescale, int batch, cudaStream_t st,
              bool lazy = false) {
  const ck::BconvArgs a = bconv_args(p, bc, in, in_batch, out, out_batch, prescale, lazy);
  return ck::launch_bconv(a, batch, st);
}

int ew_run(const ck_plan* p, int op, u64* out, long long ob, const u64* x, long long xb,
           const u64* y, long long yb, const u64* z, long long zb, const int* prime,
           const ulonglong2* cst, u64 gt, const u64* galois, int rows, int batch,
           cudaStream_t st) {
  ck::EwArgs a;
  a.out = out;
  a.x = x;
  a.y = y;
  a.z = z;
  a.out_batch = ob;
  a.x_batch = xb;
  a.y_batch = yb;
  a.z_batch = zb;
  a.prime = prime;
  a.pc = p->d_pc;
  a.cst = cst;
  a.galois_t = gt;
  a.galois = galois;
  a.op = op;
  a.logn = p->logn;
  return ck::launch_ew(a, rows, batch, st);
}

#define CK_TRY(x)            \
  do {                       \
    int _e = (x);            \
    if (_e) return _e;       \
  } while (0)

bool level_ok(const ck_plan* p, int l) { return p && l >= 1 && l <= p->L; }

// workspace regions (elements), each [batch][rows][N]
struct Ws {
  u64 *tmp, *conv, *rot, *uv, *dig;
};
Ws ws_layout(const ck_plan* p, int l, int batch, u64* base) {
  const LevelTab& t = p->lv[l];
  const long long N = p->n, B = batch;
  Ws w;
  w.rot = base;  // conjugate's automorphed (a, b): whole batch
  w.tmp = w.rot + B * 2 * l * N;
  w.conv = w.tmp + B * l * N;
  w.uv = w.conv + B * 2 * l * N;
  w.dig = w.uv + B * 2 * t.R * N;
  return w;
}

// ModUp: digits [B][beta][R][N] from a [B][l][N] (eval).  tmp: [B][l][N].
int modup_impl(const ck_plan* p, int l, const u64* a, u64* digits, u64* tmp, int B,
               cudaStream_t st) {
  const LevelTab& t = p->lv[l];
  const long long N = p->n;
  const long long dig_b = (long long)t.beta * t.R * N;
  // INTT of every chain row, scaled by its digit's ihat (rnspoly.py:274-275)
  if (ck::fused_supported(p->logn)) {
    // row phase reads the input directly (no copy), then the column phase
    CK_TRY(ntt_phase(p, tmp, t.d_chain_prime, nullptr, nullptr, l, B, l * N, true, 2, st, a,
                     l * N));
    CK_TRY(ntt_phase(p, tmp, t.d_chain_prime, nullptr, t.d_modup_scale, l, B, l * N, true, 1,
                     st));
  } else {
    CK_TRY((int)cudaMemcpyAsync(tmp, a, sizeof(u64) * B * l * N, cudaMemcpyDeviceToDevice, st));
    CK_TRY(ntt_rows(p, tmp, t.d_chain_prime, nullptr, t.d_modup_scale, l, B, l * N, true, st));
  }
  if (t.beta <= ck::kMaxBcGroups) {  // all digits' conversions in one launch
    ck::BconvArgs gs[ck::kMaxBcGroups];
    for (int d = 0; d < t.beta; ++d)
      gs[d] = bconv_args(p, t.modup_bc[d], tmp + t.lo[d] * N, l * N, digits + d * t.R * N, dig_b,
                         false, true);
    CK_TRY(ck::launch_bconv_groups(gs, t.beta, B, st));
  } else {
    for (int d = 0; d < t.beta; ++d)
      CK_TRY(bconv_run(p, t.modup_bc[d], tmp + t.lo[d] * N, l * N, digits + d * t.R * N, dig_b,
                       false, B, st, true));
  }
  CK_TRY(ntt_rows(p, digits, t.d_modup_ntt_prime, t.d_modup_ntt_off, nullptr, t.modup_ntt_jobs, B,
                  dig_b, false, st));
  for (int d = 0; d < t.beta; ++d) {
    const int own = t.hi[d] - t.lo[d];
    CK_TRY((int)cudaMemcpy2DAsync(digits + d * t.R * N + t.lo[d] * N, dig_b * sizeof(u64),
                                  a + t.lo[d] * N, l * N * sizeof(u64), own * N * sizeof(u64), B,
                                  cudaMemcpyDeviceToDevice, st));
  }
  return 0;
}

// Switching keys of a batch: contiguous [B][dnum][L+K][N] blocks (base) or a
// DEVICE array of B per-item block pointers (ptrs; SURVEY 8(b) key_ptrs[]).
struct Keys {
  const u64* b = nullptr;
  const u64* a = nullptr;
  const u64* const* bp = nullptr;
  const u64* const* ap = nullptr;
  bool shared = false;  // one key for the whole batch (relinearisation)
  bool ok() const { return (b && a) || (bp && ap); }
};
Keys keys_block(const u64* b, const u64* a) {
  Keys k;
  k.b = b;
  k.a = a;
  return k;
}
Keys keys_ptrs(const u64* const* b, const u64* const* a, long long first = 0) {
  Keys k;
  k.bp = b ? b + first : nullptr;
  k.ap = a ? a + first : nullptr;
  return k;
}

int kskip_impl(const ck_plan* p, int l, const u64* digits, const Keys& keys,
               u64 gt, const u64* galois, u64* u, u64* v, long long uv_batch, int B,
               cudaStream_t st, bool shared_digits = false) {
  const LevelTab& t = p->lv[l];
  const long long N = p->n;
  ck::KskipArgs a;
  a.digits = digits;
  a.digit_stride = (long long)t.R * N;
  a.digits_batch = shared_digits ? 0 : (long long)t.beta * t.R * N;
  a.key_b = keys.b;
  a.key_a = keys.a;
  a.key_b_ptrs = keys.bp;
  a.key_a_ptrs = keys.ap;
  a.key_digit_stride = (long long)(p->L + p->K) * N;
  a.key_batch = keys.shared ? 0 : (long long)p->key_digits * (p->L + p->K) * N;
  a.key_row = t.d_raised_prime;
  a.prime = t.d_raised_prime;
  a.pc = p->d_pc;
  a.u = u;
  a.v = v;
  a.out_batch = uv_batch;
  a.galois = galois;
  a.galois_t = gt % (2ull * p->n);
  a.beta = t.beta;
  a.logn = p->logn;
  a.accumulate = 0;
  a.key_digit0 = 0;
  return ck::launch_kskip(a, t.R, B, st);
}

// ModDown steps 1-3 on a flattened batch: x [B][xrows][N] -> conv [B][keep][N]
int moddown_core(const ck_plan* p, const ModDownTab& m, u64* x, long long xb, u64* conv, int B,
                 cudaStream_t st) {
  const long long N = p->n;
  CK_TRY(ntt_rows(p, x, m.d_drop_prime, m.d_drop_off, m.d_drop_scale, m.ndrop, B, xb, true, st));
  CK_TRY(bconv_run(p, m.bc, x + (long long)m.drop_row0 * N, xb, conv, (long long)m.keep * N, false,
                   B, st, true));
  return ntt_rows(p, conv, m.d_keep_prime, nullptr, nullptr, m.keep, B, (long long)m.keep * N,
                  false, st);
}

// ModDown of B (u, v) pairs laid out [B][2][R][N] (v at +R N) into out_a, out_b
// [B][keep][N] with the fused kernels: INTT of the dropped rows (row + column
// phase), centered BC, forward column phase of the converted rows, then md_row
// (their forward row phase + (x - conv) P^-1 + addends, u and v in one launch).
// addend_v: added to v after the automorphism by gal[b] (or gt); addend_u /
// add_scale: relinearisation's pmodup terms (see keyswitch_fused).
int moddown_pairs(const ck_plan* p, const ModDownTab& m, u64* x, long long R, u64* conv, int B,
                  u64* out_a, u64* out_b, const u64* addend_v, const u64* addend_u,
                  const ulonglong2* add_scale, long long add_batch, u64 gt, const u64* gal,
                  cudaStream_t st) {
  const long long N = p->n, keep = m.keep;
  CK_TRY(ntt_phase(p, x, m.d_drop_prime, m.d_drop_off, m.d_drop_scale, m.ndrop, 2 * B, R * N,
                   true, 0, st));
  const ck::BconvArgs g1 = bconv_args(p, m.bc, x + (long long)m.drop_row0 * N, R * N, conv,
                                      keep * N, false, true);
  CK_TRY(ck::launch_bconv(g1, 2 * B, st));
  CK_TRY(ntt_phase(p, conv, m.d_keep_prime, nullptr, nullptr, m.keep, 2 * B, keep * N, false, 1,
                   st));
  ck::MdRowArgs ma{};
  ma.prime = m.d_keep_prime;
  ma.pinv = m.d_pinv;
  ma.pc = p->d_pc;
  ma.tw = p->d_tw;
  ma.logn = p->logn;
  ma.x = x;
  ma.x_batch = 2 * R * N;
  ma.conv = conv;
  ma.conv_batch = 2 * keep * N;
  ma.addend = addend_v;
  ma.addend_u = addend_u;
  ma.add_scale = add_scale;
  ma.addend_batch = add_batch;
  ma.out = out_a;
  ma.out_batch = keep * N;
  ma.galois = gal;
  ma.galois_t = gt;
  ma.pair = 1;
  ma.x_w = R * N;
  ma.conv_w = keep * N;
  ma.out2 = out_b;
  ma.lazy = 1;
  for (int k = 0; k < keep; ++k) ma.lazy &= p->mod[k] < ((u64)1 << 59) ? 1 : 0;
  ma.group = p->md_group;
  return ck::launch_md_row(ma, (int)keep, B, st);
}

// Fused key-switch of a batch (see fused.cu): ModUp (INTT row + column phase,
// BC, forward column phase), ks_row (digit row phases + automorphism + KSKIP),
// ModDown (INTT of the dropped rows, centered BC, forward column phase) and
// md_row (forward row phase of the converted rows + epilogue); 10 launches.
//   rotation (relin == nullptr): out = (u, v + automorph(b_add, egt/egal))
//     after ModDown by P (ckks.py:655-681).
//   relinearisation (relin = {b3, c3}, kgt = 1): u[l-1] += [P] b3[l-1],
//     v[l-1] += [P] c3[l-1] before the merged ModDown by P*q_last; the kept rows'
//     pmodup(b3), pmodup(c3) fold into the md_row epilogue as b3 * q_last^-1
//     (exact mod q_j) -- new_mult's relinearisation (ckks.py:639-651).
struct Relin {
  const u64* b3;
  const u64* c3;
  long long stride;  // elements between batch items of b3 (and of c3)
};
int keyswitch_fused(const ck_plan* p, int level, const u64* a_src, const u64* b_add,
                    const Keys& keys, u64 kgt, const u64* kgal, u64 egt, const u64* egal,
                    const Relin* relin, u64* out_a, u64* out_b, const Ws& w, int B,
                    cudaStream_t st) {
  const LevelTab& t = p->lv[level];
  const ModDownTab& m = t.md[relin ? 1 : 0];
  const long long N = p->n, l = level, R = t.R, keep = m.keep;
  const long long dig_b = (long long)t.beta * R * N;
  // ---- ModUp: INTT of a (row then column phase, ihat*n^-1 folded), BC, fwd column phase
  CK_TRY(ntt_phase(p, w.tmp, t.d_chain_prime, nullptr, nullptr, level, B, l * N, true, 2, st,
                   a_src, l * N));  // row phase reads the ciphertext directly
  CK_TRY(ntt_phase(p, w.tmp, t.d_chain_prime, nullptr, t.d_modup_scale, level, B, l * N, true, 1,
                   st));
  if (t.beta <= ck::kMaxBcGroups) {  // all digits' conversions in one launch
    ck::BconvArgs gs[ck::kMaxBcGroups];
    for (int d = 0; d < t.beta; ++d)
      gs[d] = bconv_args(p, t.modup_bc[d], w.tmp + t.lo[d] * N, l * N, w.dig + d * R * N, dig_b,
                         false, true);
    CK_TRY(ck::launch_bconv_groups(gs, t.beta, B, st));
  } else {
    for (int d = 0; d < t.beta; ++d)
      CK_TRY(bconv_run(p, t.modup_bc[d], w.tmp + t.lo[d] * N, l * N, w.dig + d * R * N, dig_b,
                       false, B, st, true));
  }
  CK_TRY(ntt_phase(p, w.dig, t.d_modup_ntt_prime, t.d_modup_ntt_off, nullptr, t.modup_ntt_jobs,
                     B, dig_b, false, 1, st));
  // ---- row phase + automorph + KSKIP
  ck::KsRowArgs ka_{};
  ka_.a_eval = a_src;
  ka_.a_batch = l * N;
  ka_.dig = w.dig;
  ka_.dig_batch = dig_b;
  ka_.key_b = keys.b;
  ka_.key_a = keys.a;
  ka_.key_b_ptrs = keys.bp;
  ka_.key_a_ptrs = keys.ap;
  ka_.key_digit_stride = (long long)(p->L + p->K) * N;
  ka_.key_batch = keys.shared ? 0 : (long long)p->key_digits * (p->L + p->K) * N;
  ka_.uv = w.uv;
  ka_.uv_batch = 2 * R * N;
  ka_.v_off = R * N;
  ka_.prime = t.d_raised_prime;
  ka_.pc = p->d_pc;
  ka_.tw = p->d_tw;
  ka_.itw = p->d_itw;
  ka_.galois = kgal;
  ka_.galois_t = kgt;
  for (int d = 0; d < 16; ++d) {
    ka_.lo[d] = d < t.beta ? t.lo[d] : 0;
    ka_.hi[d] = d < t.beta ? t.hi[d] : 0;
  }
  ka_.beta = t.beta;
  ka_.l = level;
  ka_.R = (int)R;
  ka_.logn = p->logn;
  ka_.key_prefetch = p->key_prefetch;
  ka_.row0 = 0;
  ka_.lazy_keep = (int)keep;  // the kept rows go to md_row only
  CK_TRY(ck::launch_ks_row(ka_, (int)R, B, st));
  if (relin) {
    // pmodup (ckks.py:478-489) on the dropped chain row q_last: it feeds the BC
    const int* lp = t.d_chain_prime + (l - 1);
    const ulonglong2* pm = t.d_pmod + (l - 1);
    CK_TRY(ew_run(p, ck::EW_ADDMULC, w.uv + (l - 1) * N, 2 * R * N, w.uv + (l - 1) * N, 2 * R * N,
                  relin->b3 + (l - 1) * N, relin->stride, nullptr, 0, lp, pm, 1, nullptr, 1, B, st));
    CK_TRY(ew_run(p, ck::EW_ADDMULC, w.uv + (R + l - 1) * N, 2 * R * N, w.uv + (R + l - 1) * N,
                  2 * R * N, relin->c3 + (l - 1) * N, relin->stride, nullptr, 0, lp, pm, 1, nullptr, 1, B,
                  st));
  }
  // ---- ModDown pair (fused): INTT, BC, column phase, md_row epilogue
  return moddown_pairs(p, m, w.uv, R, w.conv, B, out_a, out_b, relin ? relin->c3 : b_add,
                       relin ? relin->b3 : nullptr, relin ? m.d_dinv : nullptr,
                       relin ? relin->stride : l * N,
                       relin ? 1 : egt, relin ? nullptr : egal, st);
}

}  // namespace

// ==================================================================== C ABI
extern "C" {

int ck_version(void) { return 1; }

int64_t ck_launch_count(void) { return g_launches.load(); }

const char* ck_error_string(int code) {
  switch (code) {
    case CK_OK: return "ok";
    case CK_ERR_ARG: return "invalid argument";
    case CK_ERR_MODULUS: return "invalid modulus";
    case CK_ERR_ALLOC: return "device allocation failed";
    case CK_ERR_DEVICE: return "no CUDA device";
    default: return code > 0 ? cudaGetErrorString((cudaError_t)code) : "unknown error";
  }
}

int ck_plan_create(int log_n, const uint64_t* chain, int n_chain, const uint64_t* special,
                   int n_special, int dnum, ck_plan** out) {
  if (!out || log_n < 1 || log_n > 20 || n_chain < 1 || n_special < 0 || dnum < 1 || !chain ||
      (n_special > 0 && !special))
    return CK_ERR_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return CK_ERR_DEVICE;
  ck_plan* p = new ck_plan();
  p->logn = log_n;
  p->n = 1 << log_n;
  p->L = n_chain;
  p->K = n_special;
  p->dnum = dnum;
  p->alpha = (n_chain + dnum - 1) / dnum;
  p->key_digits = (n_chain + p->alpha - 1) / p->alpha;
  {
    const char* e = getenv("CKB200_UNFUSED");
    p->fused = !(e && e[0] == '1');
    if (const char* mg = getenv("CKB200_MD_G")) p->md_group = std::max(1, atoi(mg));
    if (const char* bf = getenv("CKB200_BSGS_FUSED")) p->bsgs_fused = atoi(bf);
    const char* tc = getenv("CKB200_BCTC");
    if (tc) p->bc_tc = atoi(tc);
  }
  for (int i = 0; i < n_chain; ++i) p->mod.push_back(chain[i]);
  for (int i = 0; i < n_special; ++i) p->mod.push_back(special[i]);
  const u64 two_n = 2ull << log_n;
  for (size_t i = 0; i < p->mod.size(); ++i) {
    const u64 q = p->mod[i];
    if (q >= (1ull << 60) || q % two_n != 1 || !isprime_h(q)) { delete p; return CK_ERR_MODULUS; }
    for (size_t j = 0; j < i; ++j)
      if (p->mod[j] == q) { delete p; return CK_ERR_MODULUS; }
  }
  const int np = (int)p->mod.size();
  const long long N = p->n;
  p->psi.resize(np);
  std::vector<PrimeConst> pcs(np);
  std::vector<ulonglong2> tw((size_t)np * N), itw((size_t)np * N);
  std::vector<u32> br(N);
  for (u32 i = 0; i < (u32)N; ++i) br[i] = brev_h(i, log_n);
  auto work = [&](int i) {
    const u64 q = p->mod[i];
    const u64 psi = psi_for(q, log_n);
    p->psi[i] = psi;
    pcs[i] = make_pc(q, log_n);
    std::vector<u64> pw(N), ipw(N);
    const u64 ipsi = invmod_h(psi, q);
    pw[0] = ipw[0] = 1;
    for (long long k = 1; k < N; ++k) {
      pw[k] = mulmod_h(pw[k - 1], psi, q);
      ipw[k] = mulmod_h(ipw[k - 1], ipsi, q);
    }
    for (long long k = 0; k < N; ++k) {
      tw[(size_t)i * N + k] = sh2(pw[br[k]], q);
      itw[(size_t)i * N + k] = sh2(ipw[br[k]], q);
    }
  };
  {
    const int nth = std::max(1, std::min(np, (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < nth; ++t)
      th.emplace_back([&, t] {
        for (int i = t; i < np; i += nth) work(i);
      });
    for (auto& x : th) x.join();
  }
  int err = 0;
  p->d_pc = upload(p->allocs, pcs, &err);
  p->d_mod = upload(p->allocs, p->mod, &err);
  p->d_tw = upload(p->allocs, tw, &err);
  p->d_itw = upload(p->allocs, itw, &err);
  if (log_n == 16 || log_n == 17) {
    const char* e = getenv("CKB200_NTTTC");
    if (!(e && e[0] == '0')) {
      std::vector<unsigned char> tb;
      std::vector<ulonglong2> td;
      if (ck::ntt_tc_tables(p->mod.data(), np, tw.data(), itw.data(), N, tb, td)) {
        p->d_tcB = upload(p->allocs, tb, &err);
        p->d_tcD = upload(p->allocs, td, &err);
      }
    }
  }
  p->lv.resize(n_chain + 1);
  for (int l = 1; l <= n_chain && !err; ++l) err = build_level(p, l);
  if (err) { delete p; return err; }
  *out = p;
  return 0;
}

int ck_plan_destroy(ck_plan* plan) {
  delete plan;
  return 0;
}

int ck_plan_info(const ck_plan* p, int64_t* out) {
  if (!p || !out) return CK_ERR_ARG;
  out[0] = p->n;
  out[1] = p->L;
  out[2] = p->K;
  out[3] = p->dnum;
  out[4] = p->alpha;
  return 0;
}

int ck_plan_psi(const ck_plan* p, uint64_t* psi_out) {
  if (!p || !psi_out) return CK_ERR_ARG;
  for (size_t i = 0; i < p->psi.size(); ++i) psi_out[i] = p->psi[i];
  return 0;
}

int ck_plan_twiddles(const ck_plan* p, int prime, int inverse, uint64_t* out) {
  if (!p || !out || prime < 0 || prime >= (int)p->mod.size()) return CK_ERR_ARG;
  std::vector<ulonglong2> h(p->n);
  const ulonglong2* src = (inverse ? p->d_itw : p->d_tw) + (size_t)prime * p->n;
  CK_TRY((int)cudaMemcpy(h.data(), src, sizeof(ulonglong2) * p->n, cudaMemcpyDeviceToHost));
  for (int i = 0; i < p->n; ++i) out[i] = h[i].x;
  return 0;
}

int ck_ntt(const ck_plan* p, uint64_t* data_, const int32_t* prime_idx, int rows, int batch,
           int64_t batch_stride, int inverse, ck_stream stream) {
  u64* data = (u64*)data_;
  if (!p || !data || !prime_idx || rows < 0 || batch < 0) return CK_ERR_ARG;
  return ntt_rows(p, data, prime_idx, nullptr, nullptr, rows, batch, batch_stride, inverse != 0,
                  (cudaStream_t)stream);
}

int ck_poly_op(const ck_plan* p, int op, uint64_t* out_, const uint64_t* x_, const uint64_t* y_,
               const int32_t* prime_idx, const uint64_t* cst, int rows, ck_stream stream) {
  u64* out = (u64*)out_;
  const u64* x = (const u64*)x_;
  const u64* y = (const u64*)y_;
  if (!p || !out || !x || !prime_idx || op < 0 || op > 6) return CK_ERR_ARG;
  if ((op <= 2) && !y) return CK_ERR_ARG;
  if ((op == 4 || op == 6) && !cst) return CK_ERR_ARG;
  return ew_run(p, op == 6 ? ck::EW_ADDC : op, out, 0, x, 0, y, 0, nullptr, 0, prime_idx,
                (const ulonglong2*)cst, 1,
                nullptr, rows, 1, (cudaStream_t)stream);
}

int ck_automorph(const ck_plan* p, uint64_t* out_, const uint64_t* x_, int rows, uint64_t galois_t,
                 ck_stream stream) {
  u64* out = (u64*)out_;
  const u64* x = (const u64*)x_;
  if (!p || !out || !x || rows < 0 || (galois_t & 1) == 0) return CK_ERR_ARG;
  if (rows == 0) return 0;
  return ew_run(p, ck::EW_AUTOMORPH, out, 0, x, 0, nullptr, 0, nullptr, 0, nullptr, nullptr,
                galois_t % (2ull * p->n), nullptr, rows, 1, (cudaStream_t)stream);
}

int ck_bconv_create(const ck_plan* p, const int32_t* src_idx, int ns, const int32_t* dst_idx,
                    int nd, int centered, ck_bconv** out) {
  if (!p || !src_idx || !dst_idx || ns < 1 || nd < 1 || !out) return CK_ERR_ARG;
  std::vector<int> s(src_idx, src_idx + ns), d(dst_idx, dst_idx + nd);
  for (int v : s)
    if (v < 0 || v >= (int)p->mod.size()) return CK_ERR_ARG;
  for (int v : d)
    if (v < 0 || v >= (int)p->mod.size()) return CK_ERR_ARG;
  int err = 0;
  ck_bconv* b = build_bconv(const_cast<ck_plan*>(p), s, d, centered != 0, &err);
  if (err) { delete b; return err; }
  *out = b;
  return 0;
}

int ck_bconv_destroy(ck_bconv* bc) {
  delete bc;
  return 0;
}

int ck_bconv_apply(const ck_plan* p, const ck_bconv* bc, const uint64_t* in_, uint64_t* out_,
                   ck_stream stream) {
  const u64* in = (const u64*)in_;
  u64* out = (u64*)out_;
  if (!p || !bc || !in || !out) return CK_ERR_ARG;
  return bconv_run(p, bc, in, 0, out, 0, true, 1, (cudaStream_t)stream);
}

size_t ck_workspace_bytes(const ck_plan* p, int level, int batch) {
  if (!level_ok(p, level) || batch < 1) return 0;
  const LevelTab& t = p->lv[level];
  const long long rows = level + 2LL * level + 2LL * level + 2LL * t.R + (long long)t.beta * t.R;
  return (size_t)rows * p->n * sizeof(u64) * batch;
}

int ck_modup(const ck_plan* p, const uint64_t* a_eval_, int level, uint64_t* digits_,
             uint64_t* workspace_, int batch, ck_stream stream) {
  const u64* a_eval = (const u64*)a_eval_;
  u64* digits = (u64*)digits_;
  u64* workspace = (u64*)workspace_;
  if (!level_ok(p, level) || !a_eval || !digits || !workspace || batch < 1) return CK_ERR_ARG;
  const Ws w = ws_layout(p, level, batch, workspace);
  return modup_impl(p, level, a_eval, digits, w.tmp, batch, (cudaStream_t)stream);
}

int ck_kskip(const ck_plan* p, const uint64_t* digits_, const uint64_t* key_b_,
             const uint64_t* key_a_, int level, uint64_t galois_t, const uint64_t* galois_,
             uint64_t* u_, uint64_t* v_, int batch, ck_stream stream) {
  const u64 *digits = (const u64*)digits_, *key_b = (const u64*)key_b_, *key_a = (const u64*)key_a_,
            *galois = (const u64*)galois_;
  u64 *u = (u64*)u_, *v = (u64*)v_;
  if (!level_ok(p, level) || !digits || !key_b || !key_a || !u || !v || batch < 1 ||
      (galois_t & 1) == 0)
    return CK_ERR_ARG;
  const long long ub = (long long)p->lv[level].R * p->n;
  return kskip_impl(p, level, digits, keys_block(key_b, key_a), galois_t, galois, u, v, ub, batch,
                    (cudaStream_t)stream);
}

int ck_moddown(const ck_plan* p, uint64_t* x_, int level, int merged, uint64_t* out_,
               const uint64_t* addend_, uint64_t galois_t, uint64_t* workspace_, int batch,
               ck_stream stream) {
  u64 *x = (u64*)x_, *out = (u64*)out_, *workspace = (u64*)workspace_;
  const u64* addend = (const u64*)addend_;
  if (!level_ok(p, level) || !x || !out || !workspace || merged < 0 || merged > 2 || batch < 1 ||
      (galois_t & 1) == 0)
    return CK_ERR_ARG;
  const LevelTab& t = p->lv[level];
  const ModDownTab& m = t.md[merged];
  if (!m.valid) return CK_ERR_ARG;
  const long long N = p->n;
  const long long xrows = merged == 2 ? level : t.R;
  const Ws w = ws_layout(p, level, batch, workspace);
  cudaStream_t st = (cudaStream_t)stream;
  CK_TRY(moddown_core(p, m, x, xrows * N, w.conv, batch, st));
  return ew_run(p, ck::EW_MODDOWN, out, m.keep * N, x, xrows * N, w.conv, m.keep * N, addend,
                m.keep * N, m.d_keep_prime, m.d_pinv, galois_t % (2ull * p->n), nullptr, m.keep,
                batch, st);
}

}  // extern "C"

namespace {
// rotation / conjugation key-switch of a batch (ck_rotate; giant steps of ck_bsgs)
int rotate_impl(const ck_plan* p, const u64* a, const u64* b, const Keys& keys, int level,
                uint64_t galois_t, const u64* galois, int mode, u64* out_a, u64* out_b,
                u64* workspace, int batch, cudaStream_t st) {
  if (!level_ok(p, level) || !a || !b || !keys.ok() || !out_a || !out_b || !workspace ||
      batch < 1 || (mode != 0 && mode != 1) || (galois_t & 1) == 0 || p->K < 1)
    return CK_ERR_ARG;
  if (mode == 1 && galois) return CK_ERR_ARG;
  const LevelTab& t = p->lv[level];
  const long long N = p->n, l = level, R = t.R;
  const Ws w = ws_layout(p, level, batch, workspace);
  const u64 gt = galois_t % (2ull * p->n);
  const u64* a_src = a;
  const u64* b_add = b;
  u64 kgt = gt, egt = gt;
  const u64* kgal = galois;
  if (mode == 1) {
    // conjugate: automorph first (ckks.py:677-678)
    CK_TRY(ew_run(p, ck::EW_AUTOMORPH, w.rot, l * N, a, l * N, nullptr, 0, nullptr, 0,
                  t.d_chain_prime, nullptr, gt, nullptr, level, batch, st));
    CK_TRY(ew_run(p, ck::EW_AUTOMORPH, w.rot + batch * l * N, l * N, b, l * N, nullptr, 0,
                  nullptr, 0, t.d_chain_prime, nullptr, gt, nullptr, level, batch, st));
    a_src = w.rot;
    b_add = w.rot + batch * l * N;
    kgt = 1;
    egt = 1;
    kgal = nullptr;
  }
  if (ck::fused_supported(p->logn) && p->fused && t.beta <= 8) {
    const u64* egal = mode == 1 ? nullptr : galois;
    return keyswitch_fused(p, level, a_src, b_add, keys, kgt, kgal, egt, egal, nullptr, out_a,
                           out_b, w, batch, st);
  }
  CK_TRY(modup_impl(p, level, a_src, w.dig, w.tmp, batch, st));
  // uv: [B][2][R][N]
  CK_TRY(kskip_impl(p, level, w.dig, keys, kgt, kgal, w.uv, w.uv + R * N, 2 * R * N, batch, st));
  const ModDownTab& m = t.md[0];
  CK_TRY(moddown_core(p, m, w.uv, R * N, w.conv, 2 * batch, st));
  // conv: [B][2][l][N]
  CK_TRY(ew_run(p, ck::EW_MODDOWN, out_a, l * N, w.uv, 2 * R * N, w.conv, 2 * l * N, nullptr, 0,
                m.d_keep_prime, m.d_pinv, 1, nullptr, level, batch, st));
  return ew_run(p, ck::EW_MODDOWN, out_b, l * N, w.uv + R * N, 2 * R * N, w.conv + l * N,
                2 * l * N, b_add, l * N, m.d_keep_prime, m.d_pinv, egt, mode == 1 ? nullptr : galois,
                level, batch, st);
}
}  // namespace

namespace {
int relin_impl(const ck_plan* p, const uint64_t* a3_, const uint64_t* b3_, const uint64_t* c3_,
               long long bc_stride, const uint64_t* key_b, const uint64_t* key_a, int level,
               uint64_t* out_a_, uint64_t* out_b_, uint64_t* workspace_, int batch,
               ck_stream stream);
}  // namespace

extern "C" {

int ck_rotate(const ck_plan* p, const uint64_t* a_, const uint64_t* b_, const uint64_t* key_b_,
              const uint64_t* key_a_, int level, uint64_t galois_t, const uint64_t* galois_,
              int mode, uint64_t* out_a_, uint64_t* out_b_, uint64_t* workspace_, int batch,
              ck_stream stream) {
  return rotate_impl(p, (const u64*)a_, (const u64*)b_,
                     keys_block((const u64*)key_b_, (const u64*)key_a_), level, galois_t,
                     (const u64*)galois_, mode, (u64*)out_a_, (u64*)out_b_, (u64*)workspace_,
                     batch, (cudaStream_t)stream);
}

size_t ck_keyswitch_workspace_bytes(const ck_plan* p, int level, int mode, int batch) {
  if (mode < 0 || mode > 2 || batch < 1) return 0;
  return mode == 2 ? ck_relin_workspace_bytes(p, level, batch) : ck_workspace_bytes(p, level, batch);
}

int ck_keyswitch(const ck_plan* p, const uint64_t* a, const uint64_t* b, const uint64_t* key_b,
                 const uint64_t* key_a, int level, uint64_t galois_t, const uint64_t* galois,
                 int mode, uint64_t* out_a, uint64_t* out_b, uint64_t* workspace, int batch,
                 ck_stream stream) {
  if (mode == 0 || mode == 1)
    return ck_rotate(p, a, b, key_b, key_a, level, galois_t, galois, mode, out_a, out_b,
                     workspace, batch, stream);
  if (mode != 2 || !p || !b) return CK_ERR_ARG;
  const long long ln = (long long)level * p->n;
  return relin_impl(p, a, b, b + ln, 2 * ln, key_b, key_a, level, out_a, out_b, workspace, batch,
                    stream);
}

size_t ck_relin_workspace_bytes(const ck_plan* p, int level, int batch) {
  if (!level_ok(p, level) || level < 2 || batch < 1) return 0;
  return ck_workspace_bytes(p, level, batch);
}

}  // extern "C"

namespace {
// bc_stride: elements between batch items of b3 and of c3 (level N for ck_relin,
// 2 level N for ck_keyswitch's interleaved (b3, c3) block)
int relin_impl(const ck_plan* p, const uint64_t* a3_, const uint64_t* b3_, const uint64_t* c3_,
               long long bc_stride, const uint64_t* key_b, const uint64_t* key_a, int level,
               uint64_t* out_a_, uint64_t* out_b_, uint64_t* workspace_, int batch,
               ck_stream stream) {
  const u64 *a3 = (const u64*)a3_, *b3 = (const u64*)b3_, *c3 = (const u64*)c3_;
  u64 *out_a = (u64*)out_a_, *out_b = (u64*)out_b_, *ws = (u64*)workspace_;
  if (!level_ok(p, level) || level < 2 || !a3 || !b3 || !c3 || !key_b || !key_a || !out_a ||
      !out_b || !ws || batch < 1 || p->K < 1)
    return CK_ERR_ARG;
  const LevelTab& t = p->lv[level];
  if (!t.md[1].valid) return CK_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const long long N = p->n, R = t.R, l = level;
  const Ws w = ws_layout(p, level, batch, ws);
  Keys keys = keys_block((const u64*)key_b, (const u64*)key_a);
  keys.shared = true;  // one relinearisation key for the whole batch
  if (ck::fused_supported(p->logn) && p->fused && t.beta <= 8) {
    const Relin rl{b3, c3, bc_stride};
    return keyswitch_fused(p, level, a3, nullptr, keys, 1, nullptr, 1, nullptr, &rl, out_a, out_b,
                           w, batch, st);
  }
  // unfused pipeline (small rings): ModUp, relin KSKIP, pmodup add, ModDown by P * q_last
  const ModDownTab& m = t.md[1];
  CK_TRY(modup_impl(p, level, a3, w.dig, w.tmp, batch, st));
  CK_TRY(kskip_impl(p, level, w.dig, keys, 1, nullptr, w.uv, w.uv + R * N, 2 * R * N, batch, st));
  // pmodup (ckks.py:478-489): chain rows += [P]_q * x, special rows += 0
  CK_TRY(ew_run(p, ck::EW_ADDMULC, w.uv, 2 * R * N, w.uv, 2 * R * N, b3, bc_stride, nullptr, 0,
                t.d_chain_prime, t.d_pmod, 1, nullptr, (int)l, batch, st));
  CK_TRY(ew_run(p, ck::EW_ADDMULC, w.uv + R * N, 2 * R * N, w.uv + R * N, 2 * R * N, c3, bc_stride,
                nullptr, 0, t.d_chain_prime, t.d_pmod, 1, nullptr, (int)l, batch, st));
  // ModDown pair by P * q_last (ckks.py:643-651), u and v as one batch of 2B
  CK_TRY(moddown_core(p, m, w.uv, R * N, w.conv, 2 * batch, st));
  const long long lo = m.keep;
  CK_TRY(ew_run(p, ck::EW_MODDOWN, out_a, lo * N, w.uv, 2 * R * N, w.conv, 2 * lo * N, nullptr, 0,
                m.d_keep_prime, m.d_pinv, 1, nullptr, (int)lo, batch, st));
  return ew_run(p, ck::EW_MODDOWN, out_b, lo * N, w.uv + R * N, 2 * R * N, w.conv + lo * N,
                2 * lo * N, nullptr, 0, m.d_keep_prime, m.d_pinv, 1, nullptr, (int)lo, batch, st);
}
}  // namespace

extern "C" {

int ck_relin(const ck_plan* p, const uint64_t* a3, const uint64_t* b3, const uint64_t* c3,
             const uint64_t* key_b, const uint64_t* key_a, int level, uint64_t* out_a,
             uint64_t* out_b, uint64_t* workspace, int batch, ck_stream stream) {
  const long long ln = p ? (long long)level * p->n : 0;
  return relin_impl(p, a3, b3, c3, ln, key_b, key_a, level, out_a, out_b, workspace, batch,
                    stream);
}

size_t ck_hrotate_workspace_bytes(const ck_plan* p, int level, int n_rot) {
  if (!level_ok(p, level) || n_rot < 1 || p->K < 1) return 0;
  const LevelTab& t = p->lv[level];
  const long long rows = (long long)t.beta * t.R + level + (long long)n_rot * 2 * t.R +
                         (long long)n_rot * 2 * level;
  return (size_t)rows * p->n * sizeof(u64);
}

int ck_hrotate(const ck_plan* p, const uint64_t* a_, const uint64_t* b_,
               const uint64_t* const* key_b_, const uint64_t* const* key_a_,
               const uint64_t* galois_, int level, int n_rot, uint64_t* out_a_, uint64_t* out_b_,
               uint64_t* workspace_, ck_stream stream) {
  const u64 *a = (const u64*)a_, *b = (const u64*)b_, *gal = (const u64*)galois_;
  const Keys keys = keys_ptrs((const u64* const*)key_b_, (const u64* const*)key_a_);
  u64 *out_a = (u64*)out_a_, *out_b = (u64*)out_b_, *ws = (u64*)workspace_;
  if (!level_ok(p, level) || !a || !b || !keys.ok() || !gal || !out_a || !out_b || !ws ||
      n_rot < 1 || p->K < 1)
    return CK_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const LevelTab& t = p->lv[level];
  const ModDownTab& m = t.md[0];
  const long long N = p->n, l = level, R = t.R;
  u64* dig = ws;
  u64* tmp = dig + (long long)t.beta * R * N;
  u64* uv = tmp + l * N;                          // [n][2][R][N]
  u64* conv = uv + (long long)n_rot * 2 * R * N;  // [n][2][l][N]
  // one shared ModUp (the hoisting, ckks.py:660), digits in evaluation form
  CK_TRY(modup_impl(p, level, a, dig, tmp, 1, st));
  // every rotation's KSKIP in one launch: digits shared, automorphism folded
  // into the gather, per-rotation key (pointer array) and Galois element
  CK_TRY(kskip_impl(p, level, dig, keys, 1, gal, uv, uv + R * N, 2 * R * N, n_rot, st, true));
  // ModDown pair of every rotation (ckks.py:664-666): b is shared, gathered
  // with each rotation's Galois element
  if (ck::fused_supported(p->logn) && p->fused)
    return moddown_pairs(p, m, uv, R, conv, n_rot, out_a, out_b, b, nullptr, nullptr, 0, 1, gal,
                         st);
  CK_TRY(moddown_core(p, m, uv, R * N, conv, 2 * n_rot, st));
  CK_TRY(ew_run(p, ck::EW_MODDOWN, out_a, l * N, uv, 2 * R * N, conv, 2 * l * N, nullptr, 0,
                m.d_keep_prime, m.d_pinv, 1, nullptr, level, n_rot, st));
  return ew_run(p, ck::EW_MODDOWN, out_b, l * N, uv + R * N, 2 * R * N, conv + l * N, 2 * l * N, b,
                0, m.d_keep_prime, m.d_pinv, 1, gal, level, n_rot, st);
}

// diagonals / baby steps per diag_mac launch (bsgs.cu kMaxBaby); more run in chunks
constexpr int kDiagChunk = 32;

size_t ck_pt_matvec_workspace_bytes(const ck_plan* p, int level, int n_diag) {
  if (!level_ok(p, level) || level < 2 || n_diag < 1 || p->K < 1) return 0;
  const LevelTab& t = p->lv[level];
  const long long chunk = std::min(n_diag, kDiagChunk);
  const long long rows = (long long)t.beta * t.R + level + chunk * 2 * t.R + 2LL * t.R +
                         2LL * level;
  return (size_t)rows * p->n * sizeof(u64);
}

int ck_pt_matvec(const ck_plan* p, const uint64_t* a_, const uint64_t* b_,
                 const uint64_t* const* key_b_, const uint64_t* const* key_a_,
                 const uint64_t* galois_, const uint64_t* const* diags_, int level, int n_rot,
                 int has_identity, uint64_t* out_a_, uint64_t* out_b_, uint64_t* workspace_,
                 ck_stream stream) {
  const u64 *a = (const u64*)a_, *b = (const u64*)b_, *gal = (const u64*)galois_;
  const u64* const* diags = (const u64* const*)diags_;
  const Keys keys = keys_ptrs((const u64* const*)key_b_, (const u64* const*)key_a_);
  u64 *out_a = (u64*)out_a_, *out_b = (u64*)out_b_, *ws = (u64*)workspace_;
  const int nd = n_rot + (has_identity ? 1 : 0);
  if (!level_ok(p, level) || level < 2 || !a || !b || !diags || !gal || !out_a || !out_b ||
      !ws || n_rot < 0 || nd < 1 || p->K < 1 || (n_rot > 0 && !keys.ok()))
    return CK_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const LevelTab& t = p->lv[level];
  const ModDownTab& m = t.md[1];
  const long long N = p->n, l = level, R = t.R, lo = l - 1;
  const int chunk = std::min(nd, kDiagChunk);
  u64* dig = ws;
  u64* tmp = dig + (long long)t.beta * R * N;
  u64* uvb = tmp + l * N;                         // [chunk][2][R][N]
  u64* acc = uvb + (long long)chunk * 2 * R * N;  // [2][R][N]
  u64* conv = acc + 2 * R * N;                    // [2][l][N]
  if (n_rot > 0) CK_TRY(modup_impl(p, level, a, dig, tmp, 1, st));
  // any number of diagonals (ckks.py:699-711): chunks of <= 32 accumulate into
  // the same raised accumulators before the single merged ModDown
  for (int c0 = 0; c0 < nd; c0 += chunk) {
    const int cnt = std::min(chunk, nd - c0);
    const int nrot_c = std::max(0, std::min(cnt, n_rot - c0));
    if (nrot_c > 0)
      CK_TRY(kskip_impl(p, level, dig, keys_ptrs(keys.bp, keys.ap, c0), 1, gal + c0, uvb,
                        uvb + R * N, 2 * R * N, nrot_c, st, true));
    if (nrot_c < cnt) {
      // identity diagonal (ckks.py:701-704): u = pmodup(a), v = 0 (+ P b added by
      // the MAC kernel with Galois element 1 -> pmodup(b))
      u64* ui = uvb + (long long)nrot_c * 2 * R * N;
      CK_TRY((int)cudaMemsetAsync(ui, 0, sizeof(u64) * 2 * R * N, st));
      CK_TRY(ew_run(p, ck::EW_MULC, ui, 0, a, 0, nullptr, 0, nullptr, 0, t.d_chain_prime,
                    t.d_pmod, 1, nullptr, level, 1, st));
    }
    ck::DiagArgs da{};
    da.uv = uvb;
    da.b = b;
    da.diag_ptrs = diags + c0;
    da.diag_stride = cnt;
    da.accumulate = c0 > 0;
    da.acc = acc;
    da.galois = gal + c0;  // identity's element is 1 (set by the caller)
    da.prime = t.d_raised_prime;
    da.pmod = t.d_pmod;
    da.pc = p->d_pc;
    da.baby = cnt;
    da.giant = 1;
    da.R = (int)R;
    da.l = level;
    da.logn = p->logn;
    CK_TRY(ck::launch_diag_mac(da, st));
  }
  // one merged ModDown pair by P * q_last (ckks.py:712-717)
  if (ck::fused_supported(p->logn) && p->fused)
    return moddown_pairs(p, m, acc, R, conv, 1, out_a, out_b, nullptr, nullptr, nullptr, 0, 1,
                         nullptr, st);
  CK_TRY(moddown_core(p, m, acc, R * N, conv, 2, st));
  CK_TRY(ew_run(p, ck::EW_MODDOWN, out_a, 0, acc, 0, conv, 0, nullptr, 0, m.d_keep_prime, m.d_pinv,
                1, nullptr, (int)lo, 1, st));
  return ew_run(p, ck::EW_MODDOWN, out_b, 0, acc + R * N, 0, conv + lo * N, 0, nullptr, 0,
                m.d_keep_prime, m.d_pinv, 1, nullptr, (int)lo, 1, st);
}

size_t ck_bsgs_workspace_bytes(const ck_plan* p, int level, int baby, int giant) {
  if (!level_ok(p, level) || level < 2 || baby < 1 || giant < 1) return 0;
  const LevelTab& t = p->lv[level];
  const long long N = p->n, l = level, R = t.R;
  const long long chunk = std::min(baby, kDiagChunk);
  const long long rows = (long long)t.beta * R + l + chunk * 2 * R +
                         (long long)giant * 2 * R + (long long)giant * 2 * l +
                         (long long)giant * 4 * (l - 1);
  return (size_t)rows * N * sizeof(u64) + ck_workspace_bytes(p, level - 1, giant);
}

int ck_bsgs(const ck_plan* p, const uint64_t* a_, const uint64_t* b_,
            const uint64_t* const* bkb_, const uint64_t* const* bka_,
            const uint64_t* const* gkb_, const uint64_t* const* gka_,
            const uint64_t* const* diags_, const uint64_t* baby_galois_,
            const uint64_t* giant_galois_, int level, int baby, int giant, uint64_t* out_a_,
            uint64_t* out_b_, uint64_t* workspace_, ck_stream stream) {
  const u64 *a = (const u64*)a_, *b = (const u64*)b_, *bgal = (const u64*)baby_galois_,
            *ggal = (const u64*)giant_galois_;
  const u64* const* diags = (const u64* const*)diags_;
  const Keys bkeys = keys_ptrs((const u64* const*)bkb_, (const u64* const*)bka_);
  const Keys gkeys = keys_ptrs((const u64* const*)gkb_, (const u64* const*)gka_);
  u64 *out_a = (u64*)out_a_, *out_b = (u64*)out_b_, *ws = (u64*)workspace_;
  if (!level_ok(p, level) || level < 2 || !a || !b || !bkeys.ok() || !gkeys.ok() || !diags ||
      !bgal || !ggal || !out_a || !out_b || !ws || baby < 1 || giant < 1 || p->K < 1)
    return CK_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const LevelTab& t = p->lv[level];
  const ModDownTab& m = t.md[1];
  const long long N = p->n, l = level, R = t.R, lo = l - 1;
  // chunks of 16 babies for the fused kernel (its register-resident baby outputs), 32 else
  const int chunk = std::min(baby, p->bsgs_fused ? 16 : kDiagChunk);
  u64* dig = ws;
  u64* tmp = dig + (long long)t.beta * R * N;
  u64* uvb = tmp + l * N;                        // [chunk][2][R][N]
  u64* acc = uvb + (long long)chunk * 2 * R * N; // [giant][2][R][N]
  u64* conv = acc + (long long)giant * 2 * R * N;
  u64* ga = conv + (long long)giant * 2 * l * N; // [giant][l-1][N]
  u64* gb = ga + (long long)giant * lo * N;
  u64* ra = gb + (long long)giant * lo * N;      // rotated giants
  u64* rb = ra + (long long)giant * lo * N;
  u64* rws = rb + (long long)giant * lo * N;
  // 1. one shared ModUp (hoisting)
  CK_TRY(modup_impl(p, level, a, dig, tmp, 1, st));
  for (int c0 = 0; c0 < baby; c0 += chunk) {
    const int cnt = std::min(chunk, baby - c0);
    // 2+3. baby KSKIPs and the diagonal MAC into the giant accumulators
    //      (pmodup(automorph(b)) folded in); chunks after the first accumulate
    ck::DiagArgs da{};
    da.uv = uvb;
    da.b = b;
    da.diag_ptrs = diags + c0;
    da.diag_stride = baby;
    da.accumulate = c0 > 0;
    da.acc = acc;
    da.galois = bgal + c0;
    da.prime = t.d_raised_prime;
    da.pmod = t.d_pmod;
    da.pc = p->d_pc;
    da.baby = cnt;
    da.giant = giant;
    da.R = (int)R;
    da.l = level;
    da.logn = p->logn;
    // fused: baby outputs stay in registers (no u_k / v_k round trip through HBM)
    ck::BsgsMacArgs ba;
    ba.d = da;
    ba.digits = dig;
    ba.digit_stride = R * N;
    ba.key_b_ptrs = bkeys.bp + c0;
    ba.key_a_ptrs = bkeys.ap + c0;
    ba.key_digit_stride = (long long)(p->L + p->K) * N;
    ba.beta = t.beta;
    const int e = p->bsgs_fused ? ck::launch_bsgs_mac(ba, st) : -1;
    if (e > 0) return e;
    if (e < 0) {
      CK_TRY(kskip_impl(p, level, dig, keys_ptrs(bkeys.bp, bkeys.ap, c0), 1, bgal + c0, uvb,
                        uvb + R * N, 2 * R * N, cnt, st, true));
      CK_TRY(ck::launch_diag_mac(da, st));
    }
  }
  // 4. merged ModDown (P * q_last) of every accumulator -> level l-1
  if (ck::fused_supported(p->logn) && p->fused) {
    CK_TRY(moddown_pairs(p, m, acc, R, conv, giant, ga, gb, nullptr, nullptr, nullptr, 0, 1,
                         nullptr, st));
  } else {
    CK_TRY(moddown_core(p, m, acc, R * N, conv, 2 * giant, st));
    CK_TRY(ew_run(p, ck::EW_MODDOWN, ga, lo * N, acc, 2 * R * N, conv, 2 * lo * N, nullptr, 0,
                  m.d_keep_prime, m.d_pinv, 1, nullptr, (int)lo, giant, st));
    CK_TRY(ew_run(p, ck::EW_MODDOWN, gb, lo * N, acc + R * N, 2 * R * N, conv + lo * N, 2 * lo * N,
                  nullptr, 0, m.d_keep_prime, m.d_pinv, 1, nullptr, (int)lo, giant, st));
  }
  // 5. giant rotations at l-1, batched
  CK_TRY(rotate_impl(p, ga, gb, gkeys, (int)lo, 1, ggal, 0, ra, rb, rws, giant, st));
  // 6. sum of the rotated giants
  const int* kp = p->lv[lo].d_chain_prime;
  if (giant == 1) {
    CK_TRY(ew_run(p, ck::EW_COPY, out_a, 0, ra, 0, nullptr, 0, nullptr, 0, kp, nullptr, 1, nullptr,
                  (int)lo, 1, st));
    return ew_run(p, ck::EW_COPY, out_b, 0, rb, 0, nullptr, 0, nullptr, 0, kp, nullptr, 1, nullptr,
                  (int)lo, 1, st);
  }
  // one pass over all giants per output (instead of giant - 1 pairwise adds)
  for (int half = 0; half < 2; ++half) {
    const u64* src = half ? rb : ra;
    u64* dst = half ? out_b : out_a;
    for (int j0 = 0; j0 < giant; j0 += 16) {
      const int cnt = std::min(16, giant - j0);
      ck::EwArgs e{};
      e.out = dst;
      e.x = j0 ? dst : src;
      e.y = nullptr;
      e.y_batch = lo * N;
      e.prime = kp;
      e.pc = p->d_pc;
      e.galois_t = 1;
      e.op = ck::EW_SUMN;
      e.logn = p->logn;
      e.count = cnt;
      if (j0) {  // running total + the next chunk: fold the chunk into dst pairwise
        for (int j = j0; j < j0 + cnt; ++j)
          CK_TRY(ew_run(p, ck::EW_ADD, dst, 0, dst, 0, src + j * lo * N, 0, nullptr, 0, kp, nullptr,
                        1, nullptr, (int)lo, 1, st));
        continue;
      }
      CK_TRY(ck::launch_ew(e, (int)lo, 1, st));
    }
  }
  return 0;
}

int ck_xof_uniform(const uint8_t* msgs, const int32_t* msg_lens, int64_t msg_stride,
                    const uint64_t* moduli, int rows, int n, uint64_t* out, ck_stream stream) {
  if (rows < 0 || n < 0 || (rows > 0 && (!msgs || !msg_lens || !moduli || !out)) ||
      msg_stride < 0)
    return CK_ERR_ARG;
  if (rows == 0 || n == 0) return 0;
  ck::XofArgs a;
  a.msg = msgs;
  a.msg_len = msg_lens;
  a.msg_stride = msg_stride;
  a.moduli = (const u64*)moduli;
  a.out = (u64*)out;
  a.rows = rows;
  a.rows_per_item = 1;
  a.limbs = 1;
  a.n = n;
  a.tag_mode = 0;
  return ck::launch_xof(a, (cudaStream_t)stream);
}

int ck_expand_key_a(const ck_plan* p, const uint8_t* seeds, const int32_t* seed_lens,
                    int64_t seed_stride, int n_keys, uint64_t* key_a, ck_stream stream) {
  if (!p || n_keys < 0 || seed_stride < 0 || (n_keys > 0 && (!seeds || !seed_lens || !key_a)))
    return CK_ERR_ARG;
  if (n_keys == 0) return 0;
  const int limbs = p->L + p->K;
  const int digits = p->lv[p->L].beta;
  ck::XofArgs a;
  a.msg = seeds;
  a.msg_len = seed_lens;
  a.msg_stride = seed_stride;
  a.moduli = p->d_mod;
  a.out = (u64*)key_a;
  a.rows_per_item = digits * limbs;
  a.rows = n_keys * a.rows_per_item;
  a.limbs = limbs;
  a.n = p->n;
  a.tag_mode = 1;
  return ck::launch_xof(a, (cudaStream_t)stream);
}

int ck_fill_uniform(uint64_t* out_, int64_t rows, int log_n, const uint64_t* keys_,
                    const uint64_t* qs_, ck_stream stream) {
  u64* out = (u64*)out_;
  const u64 *keys = (const u64*)keys_, *qs = (const u64*)qs_;
  if (!out || !keys || !qs || rows < 0 || log_n < 1 || log_n > 20) return CK_ERR_ARG;
  return ck::launch_fill_uniform(out, rows, log_n, keys, qs, (cudaStream_t)stream);
}

}  // extern "C"
