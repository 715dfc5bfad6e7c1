// Host self-check of csrc/keccak.cuh: SHAKE256(msg) printed as hex, compared
// against Python's hashlib by tools/keccak_host_check.sh (dev tool, no GPU).
#include <cstdio>
#include <cstring>
#include "../paper_2112_06396_b200/csrc/keccak.cuh"

using ck::u64;

static void shake256(const unsigned char* m, size_t len, unsigned char* out, size_t outlen) {
  u64 s[25] = {0};
  const size_t rate = 136;
  size_t total = ((len + 1 + rate - 1) / rate) * rate;
  for (size_t off = 0; off < total; off += rate) {
    unsigned char blk[136] = {0};
    for (size_t p = 0; p < rate; ++p) {
      size_t g = off + p;
      unsigned char c = g < len ? m[g] : 0;
      if (g == len) c ^= 0x1F;
      if (g == total - 1) c ^= 0x80;
      blk[p] = c;
    }
    for (int k = 0; k < 17; ++k) {
      u64 w;
      memcpy(&w, blk + 8 * k, 8);
      s[k] ^= w;
    }
    ck::keccak_f1600(s);
  }
  size_t have = 0;
  while (true) {
    for (int k = 0; k < 17 && have < outlen; ++k)
      for (int b = 0; b < 8 && have < outlen; ++b) out[have++] = (unsigned char)(s[k] >> (8 * b));
    if (have >= outlen) break;
    ck::keccak_f1600(s);
  }
}

int main(int argc, char** argv) {
  for (int i = 1; i < argc; ++i) {
    unsigned char out[300];
    shake256((const unsigned char*)argv[i], strlen(argv[i]), out, sizeof out);
    for (unsigned char c : out) printf("%02x", c);
    printf("\n");
  }
  return 0;
}
