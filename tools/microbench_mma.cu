// Legacy warp-level tensor-core throughput on B200 (mma.sync): u8 (IMMA
// m16n8k32) and bf16 (HMMA m16n8k16).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__global__ void mma_loop(int iters, int* sink) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 9, b1 = a0 ^ 11;
  int acc[8][4] = {};
  float facc[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (KIND == 0) {
        asm volatile(
            "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};\n"
            : "+r"(acc[k][0]), "+r"(acc[k][1]), "+r"(acc[k][2]), "+r"(acc[k][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};\n"
            : "+f"(facc[k][0]), "+f"(facc[k][1]), "+f"(facc[k][2]), "+f"(facc[k][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
  }
  int s = 0;
  for (int k = 0; k < 8; ++k)
    for (int j = 0; j < 4; ++j) s += acc[k][j] + (int)facc[k][j];
  if (s == 0x12345) *sink = s;
}

int main() {
  int* sink;
  cudaMalloc(&sink, 4);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int kind = 0; kind < 2; ++kind)
    for (int warps : {4, 8, 16}) {
      const int iters = 4096;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&]() {
        if (kind == 0) mma_loop<0><<<sms * 2, warps * 16>>>(iters, sink);
        else mma_loop<1><<<sms * 2, warps * 16>>>(iters, sink);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double mnk = kind == 0 ? 16.0 * 8 * 32 : 16.0 * 8 * 16;
      const double macs = (double)sms * 2 * warps / 2 * iters * 8 * mnk;
      printf("%s warps/SM=%d: %.1f T MAC/s (%.2f ms)\n", kind == 0 ? "u8 m16n8k32" : "bf16 m16n8k16",
             warps, macs / ms / 1e9, ms);
    }
  return 0;
}
