// Throughput of the FP64-assisted constant modmul vs the integer Shoup modmul,
// plus conversion / co-issue probes (B200, sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_fp64 tools/microbench_fp64.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
typedef unsigned int u32;
constexpr int CH = 8;
constexpr int IT = 2048;

struct Cst { u64 w, wp, q, W0, W1, nq; double f0, f1, G0, G1; };

__device__ __forceinline__ u64 shoup_int(u64 y, const Cst& c) {
  return y * c.w - __umul64hi(y, c.wp) * c.q;
}
// FP64-quotient modmul: y*w mod q in (0.99q, 3.01q) + offset 2q
__device__ __forceinline__ u64 shoup_fp(u64 y, const Cst& c) {
  const u32 y0 = (u32)y, y1 = (u32)(y >> 32);
  const double d0 = __hiloint2double(0x43300000, y0);
  const double d1 = __hiloint2double(0x43300000, y1);
  const double e0 = __fma_rn(d0, c.f0, c.G0);   // = 1.5*2^52 + round(y0*W0/q)
  const double e1 = __fma_rn(d1, c.f1, c.G1);
  const u32 q0 = (u32)__double2loint(e0), q1 = (u32)__double2loint(e1);
  u64 r = (u64)y0 * c.W0 + (u64)q0 * c.nq;       // mod 2^64
  r += (u64)y1 * c.W1 + (u64)q1 * c.nq;
  return r + 3 * c.q;
}

__global__ void k_int(u64* out, Cst c) {
  u64 x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 7919ull + i;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = shoup_int(x[i], c);
  u64 s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_fp(u64* out, Cst c) {
  u64 x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 7919ull + i;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = shoup_fp(x[i], c);
  u64 s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_i2f(u64* out, u32 seed) {
  double x[CH];
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = (double)((u32)__double2loint(x[i]) + seed);
  double s = 0;
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345) out[0] = s;
}
// correctness: compare against exact result
__global__ void k_check(u64* bad, Cst c, u64 seed) {
  u64 y = seed * 0x9E3779B97F4A7C15ull + threadIdx.x + blockIdx.x * 1000003ull;
  for (int it = 0; it < 64; ++it) {
    y = y * 6364136223846793005ull + 1442695040888963407ull;
    const u64 r = shoup_fp(y, c);
    const unsigned __int128 e = (unsigned __int128)y * c.w % c.q;
    const u64 rr = r % c.q;
    if (rr != (u64)e || r >= 6 * c.q) atomicAdd(bad, 1ull);
  }
}

int main() {
  const u64 q = 0xffffffffffc0001ull;  // 60-bit special prime (worst case)
  const u64 w = 0x0abcdef123456789ull % q;
  Cst c;
  c.w = w; c.q = q;
  c.wp = (u64)(((unsigned __int128)w << 64) / q);
  c.W0 = w;
  c.W1 = (u64)(((unsigned __int128)w << 32) % q);
  c.nq = (u64)(0 - q);
  c.f0 = (double)c.W0 / (double)q;   // host reference only: real tables use exact rounding
  c.f1 = (double)c.W1 / (double)q;
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  c.G0 = M - 4503599627370496.0 * c.f0;
  c.G1 = M - 4503599627370496.0 * c.f1;
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  u64* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  k_check<<<4096, 256>>>(d, c, 1);
  u64 bad = 0;
  cudaMemcpy(&bad, d, 8, cudaMemcpyDeviceToHost);
  printf("fp64-shoup mismatches: %llu of %d\n", bad, 4096 * 256 * 64);
  const int threads = 256, blocks = sms * 8;
  const double ops = (double)threads * blocks * CH * IT;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
#define T(K, ...)                                                            \
  K<<<blocks, threads>>>(d, __VA_ARGS__);                                    \
  cudaEventRecord(a);                                                        \
  K<<<blocks, threads>>>(d, __VA_ARGS__);                                    \
  cudaEventRecord(b);                                                        \
  cudaEventSynchronize(b);                                                   \
  cudaEventElapsedTime(&ms, a, b);                                           \
  printf("%-8s %8.3f ms %7.2f ops/clk/SM\n", #K, ms, ops / (ms * 1e-3) / sms / (clk * 1e3));
  T(k_int, c)
  T(k_fp, c)
  T(k_i2f, 3u)
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
