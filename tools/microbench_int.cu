// Instruction-throughput microbenchmark for the integer ops the key-switch
// path is built from (B200, sm_100a).  Prints thread-ops per SM per clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_int.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned int u32;
constexpr int CH = 8;      // independent chains per thread
constexpr int IT = 4096;   // iterations

#define KERNEL(NAME, T, INIT, BODY)                                        \
  __global__ void NAME(T* out, T seed) {                                   \
    T x[CH];                                                               \
    _Pragma("unroll") for (int c = 0; c < CH; ++c) x[c] = INIT;            \
    for (int it = 0; it < IT; ++it) {                                      \
      _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }             \
    }                                                                      \
    T s = 0;                                                               \
    _Pragma("unroll") for (int c = 0; c < CH; ++c) s += x[c];              \
    if (s == (T)0x12345) out[threadIdx.x] = s;                            \
  }

KERNEL(k_imad32, u32, seed + threadIdx.x + c, x[c] = x[c] * 0x9E3779B9u + seed)
KERNEL(k_imadhi, u32, seed + threadIdx.x + c, x[c] = __umulhi(x[c], 0x9E3779B9u) + seed)
KERNEL(k_imadwide, u64, seed + threadIdx.x + c,
       x[c] = (u64)(u32)x[c] * (u64)(u32)(seed) + x[c])
KERNEL(k_mullo64, u64, seed + threadIdx.x + c, x[c] = x[c] * 0x9E3779B97F4A7C15ull + seed)
KERNEL(k_mulhi64, u64, seed + threadIdx.x + c, x[c] = __umul64hi(x[c], 0x9E3779B97F4A7C15ull) + seed)
KERNEL(k_iadd3, u32, seed + threadIdx.x + c, x[c] = x[c] + (u32)seed + (x[c] >> 1))
KERNEL(k_lop3, u32, seed + threadIdx.x + c, x[c] = (x[c] ^ (u32)seed) & (x[c] | 0x55u))
KERNEL(k_add64, u64, seed + threadIdx.x + c, x[c] = x[c] + seed)
KERNEL(k_dfma, double, (double)(seed + threadIdx.x + c), x[c] = fma(x[c], 1.0000001, 0.5))
KERNEL(k_ffma, float, (float)(seed + threadIdx.x + c), x[c] = fmaf(x[c], 1.0000001f, 0.5f))
// Shoup modmul: x*w - mulhi(x, wp)*q
KERNEL(k_shoup, u64, seed + threadIdx.x + c,
       x[c] = x[c] * 0x123456789ull - __umul64hi(x[c], 0x9E3779B97F4A7C15ull) * 0x3fffffffd60001ull)

template <class F>
float time_kernel(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* out;
  cudaMalloc(&out, 1 << 20);
  const int threads = 256, blocks = sms * 8;
  const double ops = (double)threads * blocks * CH * IT;
#define RUN(K, T)                                                                   \
  {                                                                                 \
    float ms = time_kernel([&] { K<<<blocks, threads>>>((T*)out, (T)3); });         \
    double per_s = ops / (ms * 1e-3);                                               \
    printf("%-12s %8.3f ms  %8.1f Gop/s  %6.1f ops/clk/SM (at %d MHz)\n", #K, ms,  \
           per_s * 1e-9, per_s / sms / (clk * 1e3), clk / 1000);                    \
  }
  RUN(k_imad32, u32)
  RUN(k_imadhi, u32)
  RUN(k_imadwide, u64)
  RUN(k_mullo64, u64)
  RUN(k_mulhi64, u64)
  RUN(k_iadd3, u32)
  RUN(k_lop3, u32)
  RUN(k_add64, u64)
  RUN(k_dfma, double)
  RUN(k_ffma, float)
  RUN(k_shoup, u64)
  cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
