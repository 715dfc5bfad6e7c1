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
#pragma unroll
    for (int k = 0; k < kRateWords; ++k) {
      const u64 w = s[k];
      if (w < bound && have < n) out[have++] = reduce_word(w, q, m);
    }
    if (have >= n) break;
    keccak_f1600(s);
  }
}

}  // namespace

int launch_xof(const XofArgs& a, cudaStream_t st) {
  if (a.rows <= 0) return 0;
  xof_kernel<<<(a.rows + kThreads - 1) / kThreads, kThreads, 0, st>>>(a);
  count_launches(1);
  return (int)cudaGetLastError();
}

}  // namespace ck
