// Keccak-f[1600] (FIPS 202) for the SHAKE256 key-expansion XOF.
// Used by xof.cu (device) and tools/keccak_host_check.cu (host self-check).
// Lane i of the state is A[x = i % 5][y = i / 5]; lanes are little-endian u64.
#pragma once
#include <cstdint>

namespace ck {

typedef unsigned long long u64;

#ifdef __CUDA_ARCH__
__constant__ u64 kKeccakRC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808Aull, 0x8000000080008000ull,
    0x000000000000808Bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008Aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000Aull,
    0x000000008000808Bull, 0x800000000000008Bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800Aull, 0x800000008000000Aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};
#else
static const u64 kKeccakRC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808Aull, 0x8000000080008000ull,
    0x000000000000808Bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008Aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000Aull,
    0x000000008000808Bull, 0x800000000000008Bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800Aull, 0x800000008000000Aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};
#endif

__host__ __device__ __forceinline__ u64 rotl64(u64 x, int n) {
  return (x << n) | (x >> (64 - n));
}

// The permutation: 24 rounds of theta, rho+pi, chi, iota; the whole state
// stays in registers (all lane indices are compile-time constants).
#ifndef CKB200_KECCAK_UNROLL
#define CKB200_KECCAK_UNROLL 1
#endif
constexpr int kKeccakUnroll = CKB200_KECCAK_UNROLL;
__host__ __device__ __forceinline__ void keccak_f1600(u64 (&s)[25]) {
#pragma unroll kKeccakUnroll
  for (int r = 0; r < 24; ++r) {
    const u64 c0 = s[0] ^ s[5] ^ s[10] ^ s[15] ^ s[20];
    const u64 c1 = s[1] ^ s[6] ^ s[11] ^ s[16] ^ s[21];
    const u64 c2 = s[2] ^ s[7] ^ s[12] ^ s[17] ^ s[22];
    const u64 c3 = s[3] ^ s[8] ^ s[13] ^ s[18] ^ s[23];
    const u64 c4 = s[4] ^ s[9] ^ s[14] ^ s[19] ^ s[24];
    const u64 d0 = c4 ^ rotl64(c1, 1);
    const u64 d1 = c0 ^ rotl64(c2, 1);
    const u64 d2 = c1 ^ rotl64(c3, 1);
    const u64 d3 = c2 ^ rotl64(c4, 1);
    const u64 d4 = c3 ^ rotl64(c0, 1);
    // theta applied, then rho (rotate) and pi (B[y][2x+3y] = A[x][y])
    const u64 b0 = s[0] ^ d0;
    const u64 b1 = rotl64(s[6] ^ d1, 44);
    const u64 b2 = rotl64(s[12] ^ d2, 43);
    const u64 b3 = rotl64(s[18] ^ d3, 21);
    const u64 b4 = rotl64(s[24] ^ d4, 14);
    const u64 b5 = rotl64(s[3] ^ d3, 28);
    const u64 b6 = rotl64(s[9] ^ d4, 20);
    const u64 b7 = rotl64(s[10] ^ d0, 3);
    const u64 b8 = rotl64(s[16] ^ d1, 45);
    const u64 b9 = rotl64(s[22] ^ d2, 61);
    const u64 b10 = rotl64(s[1] ^ d1, 1);
    const u64 b11 = rotl64(s[7] ^ d2, 6);
    const u64 b12 = rotl64(s[13] ^ d3, 25);
    const u64 b13 = rotl64(s[19] ^ d4, 8);
    const u64 b14 = rotl64(s[20] ^ d0, 18);
    const u64 b15 = rotl64(s[4] ^ d4, 27);
    const u64 b16 = rotl64(s[5] ^ d0, 36);
    const u64 b17 = rotl64(s[11] ^ d1, 10);
    const u64 b18 = rotl64(s[17] ^ d2, 15);
    const u64 b19 = rotl64(s[23] ^ d3, 56);
    const u64 b20 = rotl64(s[2] ^ d2, 62);
    const u64 b21 = rotl64(s[8] ^ d3, 55);
    const u64 b22 = rotl64(s[14] ^ d4, 39);
    const u64 b23 = rotl64(s[15] ^ d0, 41);
    const u64 b24 = rotl64(s[21] ^ d1, 2);
    // chi
    s[0] = b0 ^ (~b1 & b2);
    s[1] = b1 ^ (~b2 & b3);
    s[2] = b2 ^ (~b3 & b4);
    s[3] = b3 ^ (~b4 & b0);
    s[4] = b4 ^ (~b0 & b1);
    s[5] = b5 ^ (~b6 & b7);
    s[6] = b6 ^ (~b7 & b8);
    s[7] = b7 ^ (~b8 & b9);
    s[8] = b8 ^ (~b9 & b5);
    s[9] = b9 ^ (~b5 & b6);
    s[10] = b10 ^ (~b11 & b12);
    s[11] = b11 ^ (~b12 & b13);
    s[12] = b12 ^ (~b13 & b14);
    s[13] = b13 ^ (~b14 & b10);
    s[14] = b14 ^ (~b10 & b11);
    s[15] = b15 ^ (~b16 & b17);
    s[16] = b16 ^ (~b17 & b18);
    s[17] = b17 ^ (~b18 & b19);
    s[18] = b18 ^ (~b19 & b15);
    s[19] = b19 ^ (~b15 & b16);
    s[20] = b20 ^ (~b21 & b22);
    s[21] = b21 ^ (~b22 & b23);
    s[22] = b22 ^ (~b23 & b24);
    s[23] = b23 ^ (~b24 & b20);
    s[24] = b24 ^ (~b20 & b21);
    // iota
    s[0] ^= kKeccakRC[r];
  }
}

}  // namespace ck
