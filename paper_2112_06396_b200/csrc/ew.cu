// Elementwise limb-row kernels: RnsPoly add/sub/neg/mul/mul_scalars
// (rnspoly.py:182-210, zq.py:145-181), the eval-domain automorphism gather
// (rnspoly.py:228-233) and the ModDown epilogue
// (x - conv) * P^-1 [+ automorph(addend)] (ckks.py:411-416, 664-666).
#include "ck_internal.h"

namespace ck {

constexpr int kEwThreads = 256;

__global__ void __launch_bounds__(kEwThreads) ew_kernel(EwArgs a) {
  const int n = 1 << a.logn;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int row = blockIdx.y;
  const long long bz = blockIdx.z;
  const long long ro = ((long long)row << a.logn);
  const bool needs_q = a.op != EW_COPY && a.op != EW_AUTOMORPH;
  const PrimeConst& P = a.pc[needs_q ? a.prime[row] : 0];
  const u64 q = needs_q ? P.q : 0;
  const u64* x = a.x ? a.x + bz * a.x_batch + ro : nullptr;
  const u64* y = a.y ? a.y + bz * a.y_batch + ro : nullptr;
  const u64 gt = a.galois ? a.galois[bz] : a.galois_t;
  u64 r;
  switch (a.op) {
    case EW_ADD: r = addmod(x[k], y[k], q); break;
    case EW_SUB: r = submod(x[k], y[k], q); break;
    case EW_MUL: r = mulmod(x[k], y[k], P); break;
    case EW_NEG: { const u64 v = x[k]; r = v ? q - v : 0; } break;
    case EW_MULC: { const ulonglong2 c = a.cst[row]; r = shoup(x[k], c.x, c.y, q); } break;
    case EW_ADDC: r = addmod(x[k], a.cst[row].x, q); break;
    case EW_ADDMULC: { const ulonglong2 c = a.cst[row]; r = addmod(x[k], shoup(y[k], c.x, c.y, q), q); } break;
    case EW_COPY: r = x[k]; break;
    case EW_AUTOMORPH:
      r = gt == 1 ? x[k] : x[automorph_src((u32)k, (u32)gt, a.logn)];
      break;
    case EW_MODDOWN: {
      const ulonglong2 c = a.cst[row];
      r = shoup(submod(x[k], y[k], q), c.x, c.y, q);
      if (a.z) {
        const u64* z = a.z + bz * a.z_batch + ro;
        const u32 src = gt == 1 ? (u32)k : automorph_src((u32)k, (u32)gt, a.logn);
        r = addmod(r, z[src], q);
      }
    } break;
    case EW_SUMN: {  // canonical inputs, count <= 16: the u64 sum cannot wrap (q < 2^60)
      u64 acc = 0;
      for (int j = 0; j < a.count; ++j) acc += x[(long long)j * a.y_batch + k];
      r = red64(acc, P);
    } break;
    default: r = 0;
  }
  a.out[bz * a.out_batch + ro + k] = r;
}

int launch_ew(const EwArgs& a, int rows, int batch, cudaStream_t st) {
  if (rows <= 0 || batch <= 0) return 0;
  const int n = 1 << a.logn;
  const dim3 grid((n + kEwThreads - 1) / kEwThreads, rows, batch);
  count_launches(1);
  ew_kernel<<<grid, kEwThreads, 0, st>>>(a);
  return (int)cudaGetLastError();
}

// ---------------------------------------------------------------- synth
// Counter-based uniform residues; bit-identical to paper_2112_06396_b200.synth.
__device__ __forceinline__ u64 splitmix64(u64 z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(u64* out, int logn, const u64* keys, const u64* qs) {
  const long long row = blockIdx.y + (long long)blockIdx.z * gridDim.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= (1 << logn)) return;
  const u64 x = splitmix64(keys[row] + (u64)k);
  out[(row << logn) + k] = __umul64hi(x, qs[row]);
}

int launch_fill_uniform(u64* out, long long rows, int logn, const u64* keys, const u64* qs,
                        cudaStream_t st) {
  if (rows <= 0) return 0;
  const int n = 1 << logn;
  const int threads = n < 256 ? n : 256;
  long long gy = rows, gz = 1;
  while (gy > 65535) { gy = (gy + 1) / 2; gz *= 2; }
  if (gy * gz != rows) {
    // split into exact launches
    long long done = 0;
    while (done < rows) {
      const long long chunk = rows - done < 65535 ? rows - done : 65535;
      count_launches(1);
      fill_uniform_kernel<<<dim3((n + threads - 1) / threads, (unsigned)chunk, 1), threads, 0, st>>>(
          out + (done << logn), logn, keys + done, qs + done);
      done += chunk;
    }
  } else {
    count_launches(1);
    fill_uniform_kernel<<<dim3((n + threads - 1) / threads, (unsigned)gy, (unsigned)gz), threads, 0, st>>>(
        out, logn, keys, qs);
  }
  return (int)cudaGetLastError();
}

}  // namespace ck
