// SHAKE256 rejection-sampled uniform rows: the compressed evaluation-key
// expansion of the reference (ckks._xof_uniform ckks.py:169-185 called by
// SwitchingKey.a_row / expand ckks.py:201-215).
//
// One thread per output row.  The sponge squeeze is inherently sequential
// (each 136-byte block is a permutation of the previous state), so a row is
// one thread's serial stream; rows are independent, and a batch of keys
// gives thousands of them.  Per row: absorb message = seed || tag (tag =
// "ksk<digit>:<limb>" when generated here), pad 0x1F..0x80, then squeeze
// 17 little-endian words per permutation, keep words < floor(2^64/q)*q in
// stream order, reduce mod q, stop after n kept words.  This is exactly the
// reference's chunked digest() loop: its chunks are consecutive slices of the
// same XOF stream.
#include "ck_internal.h"
#include "keccak.cuh"

namespace ck {

namespace {

__device__ __forceinline__ int ndigits(unsigned v) {
  int d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

__device__ __forceinline__ unsigned pow10u(int e) {
  unsigned p = 1;
  while (e-- > 0) p *= 10;
  return p;
}

// k-th byte of "ksk<digit>:<limb>" (b"ksk%d:%d", ckks.py:205)
__device__ __forceinline__ unsigned char tag_byte(int k, unsigned digit, unsigned limb) {
  if (k < 3) return k == 1 ? 's' : 'k';
  k -= 3;
  const int nd = ndigits(digit);
  if (k < nd) return (unsigned char)('0' + (digit / pow10u(nd - 1 - k)) % 10);
  k -= nd;
  if (k == 0) return ':';
  k -= 1;
  const int nl = ndigits(limb);
  return (unsigned char)('0' + (limb / pow10u(nl - 1 - k)) % 10);
}

__device__ __forceinline__ int tag_len(unsigned digit, unsigned limb) {
  return 4 + ndigits(digit) + ndigits(limb);
}

// floor(2^64 / q) * q and the Barrett factor floor((2^64-1)/q) (equal floors
// for odd q > 1)
__device__ __forceinline__ u64 reduce_word(u64 w, u64 q, u64 m) {
  u64 r = w - __umul64hi(w, m) * q;  // < 3q
  if (r >= q) r -= q;
  if (r >= q) r -= q;
  return r;
}

constexpr int kRate = 136;
constexpr int kRateWords = 17;
constexpr int kThreads = 32;  // spread the latency-bound row streams over more SMs

__global__ void __launch_bounds__(kThreads) xof_kernel(XofArgs a) {
  __shared__ u64 stage[kThreads][kRateWords];
  const int row = blockIdx.x * kThreads + threadIdx.x;
  if (row >= a.rows) return;  // no block-level synchronisation below
  const int item = row / a.rows_per_item;
  const int r = row - item * a.rows_per_item;
  const unsigned digit = a.tag_mode ? (unsigned)(r / a.limbs) : 0u;
  const unsigned limb = a.tag_mode ? (unsigned)(r % a.limbs) : 0u;
  const u64 q = a.moduli[a.tag_mode ? (int)limb : row];
  const unsigned char* seed = a.msg + (long long)item * a.msg_stride;
  const int slen = a.msg_len[item];
  const int mlen = slen + (a.tag_mode ? tag_len(digit, limb) : 0);
  const int total = ((mlen + 1 + kRate - 1) / kRate) * kRate;

  u64 s[25];
#pragma unroll
  for (int k = 0; k < 25; ++k) s[k] = 0;
  unsigned char* blk = reinterpret_cast<unsigned char*>(stage[threadIdx.x]);
  for (int off = 0; off < total; off += kRate) {
    for (int p = 0; p < kRate; ++p) {
      const int g = off + p;
      unsigned char c = 0;
      if (g < slen)
        c = seed[g];
      else if (g < mlen)
        c = tag_byte(g - slen, digit, limb);
      if (g == mlen) c ^= 0x1F;         // SHAKE domain bits + first pad bit
      if (g == total - 1) c ^= 0x80;    // last pad bit
      blk[p] = c;
    }
#pragma unroll
    for (int k = 0; k < kRateWords; ++k) s[k] ^= stage[threadIdx.x][k];
    keccak_f1600(s);
  }

  const u64 m = ~0ull / q;
  const u64 bound = m * q;
  u64* out = a.out + (long long)row * a.n;
  const int n = a.n;
  int have = 0;
  while (true) {
    // keep mask of this block's 17 words; each kept word's output slot is
    // have + (number of kept words before it), so the stores are independent
    unsigned keep = 0;
#pragma unroll
    for (int k = 0; k < kRateWords; ++k) keep |= (unsigned)(s[k] < bound) << k;
#pragma unroll
    for (int k = 0; k < kRateWords; ++k) {
      const int pos = have + __popc(keep & ((1u << k) - 1u));
      if (((keep >> k) & 1u) && pos < n) out[pos] = reduce_word(s[k], q, m);
    }
    have += __popc(keep);
    if (have >= n) break;
    keccak_f1600(s);
  }
}

// ------------------------------------------------------ lane-parallel form
// One WARP per row: lane l < 25 holds state lane A[l % 5][l / 5], so a
// Keccak round is ~40 warp instructions (shuffles for theta's column
// parities, pi's lane permutation and chi's neighbours) instead of ~200 in
// one thread.  The row stream is still sequential; what shrinks is the
// latency of each permutation, which is what bounds the expansion (rows run
// in parallel, but each needs ~3,900 permutations at N = 2^16).  Squeeze:
// lanes 0..16 hold the 17 rate words in stream order; a ballot gives the kept
// words and their output slots, so the kept words are stored by consecutive
// lanes to consecutive addresses.
__device__ __forceinline__ u64 shfl64(u64 v, int src) {
  const unsigned lo = __shfl_sync(0xffffffffu, (unsigned)v, src);
  const unsigned hi = __shfl_sync(0xffffffffu, (unsigned)(v >> 32), src);
  return ((u64)hi << 32) | lo;
}
__device__ __forceinline__ u64 rotl_any(u64 x, int n) { return n ? (x << n) | (x >> (64 - n)) : x; }

__constant__ int kRho[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
                             25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};

__device__ __forceinline__ void keccak_lanes(u64& A, int lane) {
  const int l = lane < 25 ? lane : 0;
  const int x = l % 5, y = l / 5;
  const int rho = kRho[l];
  // pi: destination (X, Y) = (x, y) takes source (3 (Y - 3X) mod 5, X)
  const int psrc = ((3 * (y - 3 * x) % 5 + 5) % 5) + 5 * x;
  const int c1 = (x + 1) % 5 + 5 * y, c2 = (x + 2) % 5 + 5 * y;
  const int xm = (x + 4) % 5, xp = (x + 1) % 5;
#pragma unroll 1
  for (int r = 0; r < 24; ++r) {
    const u64 C = shfl64(A, x) ^ shfl64(A, x + 5) ^ shfl64(A, x + 10) ^ shfl64(A, x + 15) ^
                  shfl64(A, x + 20);
    const u64 D = shfl64(C, xm) ^ rotl_any(shfl64(C, xp), 1);
    const u64 B = shfl64(rotl_any(A ^ D, rho), psrc);
    A = B ^ (~shfl64(B, c1) & shfl64(B, c2));
    if (lane == 0) A ^= kKeccakRC[r];
  }
}

__global__ void __launch_bounds__(128) xof_lanes_kernel(XofArgs a) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (row >= a.rows) return;  // whole warps exit together
  const int item = row / a.rows_per_item;
  const int r = row - item * a.rows_per_item;
  const unsigned digit = a.tag_mode ? (unsigned)(r / a.limbs) : 0u;
  const unsigned limb = a.tag_mode ? (unsigned)(r % a.limbs) : 0u;
  const u64 q = a.moduli[a.tag_mode ? (int)limb : row];
  const unsigned char* seed = a.msg + (long long)item * a.msg_stride;
  const int slen = a.msg_len[item];
  const int mlen = slen + (a.tag_mode ? tag_len(digit, limb) : 0);
  const int total = ((mlen + 1 + kRate - 1) / kRate) * kRate;

  u64 A = 0;
  for (int off = 0; off < total; off += kRate) {
    if (lane < kRateWords) {  // this lane's 8 message bytes (little-endian word)
      u64 w = 0;
      for (int p = 0; p < 8; ++p) {
        const int g = off + 8 * lane + p;
        unsigned c = 0;
        if (g < slen)
          c = seed[g];
        else if (g < mlen)
          c = tag_byte(g - slen, digit, limb);
        if (g == mlen) c ^= 0x1F;
        if (g == total - 1) c ^= 0x80;
        w |= (u64)c << (8 * p);
      }
      A ^= w;
    }
    keccak_lanes(A, lane);
  }
  const u64 m = ~0ull / q;
  const u64 bound = m * q;
  u64* out = a.out + (long long)row * a.n;
  const int n = a.n;
  int have = 0;
  while (true) {
    const bool keep = lane < kRateWords && A < bound;
    const unsigned mask = __ballot_sync(0xffffffffu, keep);
    const int pos = have + __popc(mask & ((1u << lane) - 1u));
    if (keep && pos < n) out[pos] = reduce_word(A, q, m);
    have += __popc(mask);
    if (have >= n) break;
    keccak_lanes(A, lane);
  }
}

}  // namespace

int launch_xof(const XofArgs& a, cudaStream_t st) {
  if (a.rows <= 0) return 0;
  // Few rows: latency-bound, one warp per row (measured 11 ms vs 26 ms for one
  // C3 key, 96 rows).  Many rows: throughput-bound on the shuffles, one thread
  // per row (26 ms vs 49 ms for 64 keys, 6144 rows).  Crossover ~3,000 rows.
  if (a.rows <= 3072)
    xof_lanes_kernel<<<(a.rows + 3) / 4, 128, 0, st>>>(a);
  else
    xof_kernel<<<(a.rows + kThreads - 1) / kThreads, kThreads, 0, st>>>(a);
  count_launches(1);
  return (int)cudaGetLastError();
}

}  // namespace ck
