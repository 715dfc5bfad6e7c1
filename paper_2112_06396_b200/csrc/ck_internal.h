// Internal declarations shared by the CUDA translation units and plan.cpp.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>
#include "../../include/ckks_b200.h"

#ifdef __CUDACC__
#include "modarith.cuh"
#else
typedef unsigned long long u64;
struct PrimeConst {
  u64 q, two_q, bar, c30, c30p, c60, c60p, r64, r64p, ninv, ninvp, nq, mu, sh;
};
#endif

namespace ck {

// process-wide count of kernel launches (ck_launch_count)
void count_launches(int n);

// Programmatic dependent launch (PDL) for the key-switch pipeline's kernels:
// a kernel waits for its predecessor's results (griddepcontrol.wait) only
// after its own prologue (constant tables, TMEM allocation), so that prologue
// and the launch overlap the predecessor's completion.  Measured: +0.2% with
// the implicit trigger at grid completion; an explicit early trigger
// (griddepcontrol.launch_dependents at CTA start, -DCKB200_PDL_TRIGGER=1) made
// the step 8% SLOWER (early dependent CTAs park on SM resources).
// CKB200_PDL=0 launches normally (the wait is then a no-op).
bool pdl_enabled();
#ifdef __CUDACC__
#ifndef CKB200_PDL_TRIGGER
#define CKB200_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_trigger() {
  if (CKB200_PDL_TRIGGER) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
#endif

struct NttArgs;
int launch_ntt(const NttArgs& a, int jobs, int batch, bool inverse, cudaStream_t st);
int launch_ntt_phase(const NttArgs& a, int jobs, int batch, bool inverse, int phase,
                     cudaStream_t st);
bool fused_supported(int logn);
// tensor-core forward column phase (ntt_tc.cu): tables per plan prime, launch
// (returns -1 when the shape is not covered; the caller uses the butterflies)
#ifdef __CUDACC__
bool ntt_tc_tables(const u64* mod, int np, const ulonglong2* tw_host, const ulonglong2* itw_host,
                   long long n, std::vector<unsigned char>& B, std::vector<ulonglong2>& D);
#endif
int launch_ntt_col_tc(const NttArgs& a, int jobs, int batch, bool inverse, cudaStream_t st);

// Fused row kernels (fused.cu)
struct KsRowArgs {
  const u64* a_eval;            // [B][l][N] eval input (own digit rows)
  long long a_batch;
  const u64* dig;               // [B][beta][R][N] ModUp targets after the column phase
  long long dig_batch;
  const u64* key_b;
  const u64* key_a;
  long long key_digit_stride, key_batch;
  const u64* const* key_b_ptrs; // nullable: per-item key blocks [B] (overrides key_b + b*key_batch)
  const u64* const* key_a_ptrs;
  u64* uv;                      // u at uv + i*N, v at uv + v_off + i*N (per batch item)
  long long uv_batch, v_off;
  const int* prime;             // [R] raised prime index (== full-basis key row)
  const PrimeConst* pc;
  const ulonglong2* tw;
  const ulonglong2* itw;
  const u64* galois;            // per batch item (nullable: galois_t)
  u64 galois_t;
  int lo[16], hi[16];           // digit spans (chain rows)
  int beta, l, R, logn;
  int key_prefetch;             // bulk L2 prefetch of the first k/8 of each key tile at kernel start
  int row0;                     // first raised row of the launch (grid.z = rows from row0)
  int lazy_keep;                // rows i < lazy_keep with q < 2^59 may stay in [0, 3q): md_row's lazy
                                // epilogue (x + c q - conv, then a Shoup product) takes them as they are
};
int launch_ks_row(const KsRowArgs& a, int rows, int batch, cudaStream_t st);


#ifdef __CUDACC__
// base of batch item b's key block: pointer array when given, else base + b * stride
__device__ __forceinline__ const u64* key_block(const u64* base, const u64* const* ptrs,
                                                long long stride, long long b) {
  return ptrs ? ptrs[b] : base + b * stride;
}
#endif

struct MdRowArgs {
  const u64* x;                 // [B][..][N] raised-basis rows (kept rows j = 0..keep)
  long long x_batch;
  const u64* conv;              // [B][keep][N] converted rows after the column phase
  long long conv_batch;
  const u64* addend;            // nullable [B][keep][N], gathered with galois (v / out2 only)
  const u64* addend_u;          // nullable [B][keep][N], pair mode's first polynomial (u / out)
  long long addend_batch;
  const ulonglong2* add_scale;  // nullable [keep] Shoup pairs: addends multiplied by them
  u64* out;
  long long out_batch;
  const int* prime;             // [keep]
  const ulonglong2* pinv;       // [keep]
  const PrimeConst* pc;
  const ulonglong2* tw;
  const u64* galois;
  u64 galois_t;
  int logn;
  // pair mode: grid.y = 2*batch; odd items are the second polynomial at
  // x + x_w, conv + conv_w, written to out2 with the addend (u/v of ModDown)
  int pair;
  long long x_w, conv_w;
  u64* out2;
  int lazy;                     // every kept prime < 2^59: conv stays lazy (md_row_kernel<.., true>)
  int group;                    // items (batch x {u,v}) per CTA, same limb and rows (L1 twiddle reuse)
  int batch;                    // set by launch_md_row
};
int launch_md_row(const MdRowArgs& a, int rows, int batch, cudaStream_t st);

// BSGS diagonal multiply-accumulate (bsgs.cu)
struct DiagArgs {
  const u64* uv;                // [baby][2][R][N]
  const u64* b;                 // [l][N]
  const u64* diags;             // [giant][baby][R][N]
  const u64* const* diag_ptrs;  // nullable: [giant][baby] per-diagonal [R][N] rows (overrides diags)
  int diag_stride;              // diag_ptrs row stride (entries between giant groups)
  int accumulate;               // 1: acc += (chunks of > 32 diagonals / babies)
  u64* acc;                     // [giant][2][R][N]
  const u64* galois;            // [baby] device
  const int* prime;             // [R]
  const ulonglong2* pmod;       // [l] [P]_q Shoup pairs
  const PrimeConst* pc;
  int baby, giant, R, l, logn;
};
int launch_diag_mac(const DiagArgs& a, cudaStream_t st);

// Fused hoisted baby-step KSKIP + diagonal MAC (bsgs.cu bsgs_mac_kernel): the
// baby outputs (u_k, v_k + P automorph(b, t_k)) stay in registers and feed the
// giant accumulators directly -- they never touch HBM.
struct BsgsMacArgs {
  DiagArgs d;                   // uv unused; galois = baby Galois elements
  const u64* digits;            // [beta][R][N] shared ModUp digits (evaluation form)
  long long digit_stride;       // R N
  const u64* const* key_b_ptrs; // [baby] per-baby key blocks [dnum][L+K][N]
  const u64* const* key_a_ptrs;
  long long key_digit_stride;   // (L+K) N
  int beta;
};
// returns -1 when the shape is not covered (the caller runs kskip + diag_mac)
int launch_bsgs_mac(const BsgsMacArgs& a, cudaStream_t st);

// Basis conversion: ns source rows (coefficient rep, same coefficient index)
// -> nd destination rows.  T[i*nd+j] = (Q/q_i) mod p_j.
struct BconvArgs {
  const u64* in;
  long long in_batch;           // elements between batch items
  const long long* in_off;      // [ns] element offsets (nullable: i*N)
  u64* out;
  long long out_batch;
  const long long* out_off;     // [nd] element offsets (nullable: j*N)
  const int* src_prime;         // [ns]
  const int* dst_prime;         // [nd]
  const PrimeConst* pc;
  const ulonglong2* src_scale;  // [ns] ihat Shoup pairs; nullable = already scaled
  const uint4* T;               // [ns*nd] {t0,t1,u0,u1}: T = t0+t1 2^30, T 2^30 mod p = u0+u1 2^30
  const double* w;              // [ns] 1.0/q_i   (centered only)
  const u64* kQ;                // [nd*(ns+1)] k*Q mod p_j  (centered only)
  const unsigned char* B5;      // tensor-core form (bconv_t5_kernel): B chunks in tcgen05 operand
                                // layout; nullable -> CUDA-core kernel
  int ns, nd, logn, centered;
  int lazy_out;                 // tcgen05 form: outputs may stay in [0, 4 p_j) (a forward NTT follows)
};
int launch_bconv(const BconvArgs& a, int batch, cudaStream_t st);
constexpr int kMaxBcGroups = 8;
// Several independent conversions (e.g. the beta ModUp digits) share one
// launch: a grid dimension selects the group.
struct BconvGroups {
  BconvArgs g[kMaxBcGroups];
  int tiles_per_cta;            // bconv_t5_kernel: 128-coefficient tiles one CTA walks
};
int launch_bconv_groups(const BconvArgs* gs, int ng, int batch, cudaStream_t st);
// tcgen05 B table (host): Tp[(i*8 + a)*nd + j] = T_ij 2^(8a) mod p_j -> operand-layout chunks
size_t bconv_t5_table_bytes(int ns, int nd);
void bconv_t5_table(const u64* Tp, int ns, int nd, unsigned char* B5);
// Key-switching inner product with a fused eval-domain automorphism.
struct KskipArgs {
  const u64* digits;            // [beta][R][N] raised-basis eval rows
  long long digit_stride;       // elements between digits
  long long digits_batch;
  const u64* key_b;             // [dnum][LK][N] full-basis rows
  const u64* key_a;
  long long key_digit_stride;   // elements between key digits (LK*N)
  long long key_batch;
  const u64* const* key_b_ptrs; // nullable: per-item key blocks [B] (overrides key_b + b*key_batch)
  const u64* const* key_a_ptrs;
  const int* key_row;           // [R] full-basis row of raised row i
  const int* prime;             // [R] prime index of raised row i
  const PrimeConst* pc;
  u64* u;                       // [R][N]
  u64* v;
  long long out_batch;
  const u64* galois;            // per batch item Galois element (nullable: galois_t)
  u64 galois_t;                 // 1 = no automorphism
  int beta, logn;
  int accumulate;               // 1: u += .., v += .. (digit chunks beyond kKsMaxBeta)
  int key_digit0;               // first key digit of this launch (pointer-array keys)
};
int launch_kskip(const KskipArgs& a, int rows, int batch, cudaStream_t st);

// Elementwise ops over limb rows.
enum EwOp { EW_ADD = 0, EW_SUB = 1, EW_MUL = 2, EW_NEG = 3, EW_MULC = 4, EW_COPY = 5,
            EW_MODDOWN = 6, EW_AUTOMORPH = 7, EW_SUMN = 8, EW_ADDC = 9,
            EW_ADDMULC = 10 };
struct EwArgs {
  u64* out;
  const u64* x;
  const u64* y;
  const u64* z;                 // optional addend (moddown: gathered with galois)
  long long out_batch, x_batch, y_batch, z_batch;
  const int* prime;             // [rows]
  const PrimeConst* pc;
  const ulonglong2* cst;        // [rows] Shoup constants (MULC, MODDOWN)
  u64 galois_t;                 // AUTOMORPH / MODDOWN addend gather (1 = none)
  const u64* galois;            // per batch item (nullable: galois_t)
  int op, logn;
  int count = 0;                // SUMN: out = sum_{j < count} x[j * y_batch] (count <= 16)
};
int launch_ew(const EwArgs& a, int rows, int batch, cudaStream_t st);

// SHAKE256 uniform rows (xof.cu)
struct XofArgs {
  const unsigned char* msg;     // [items][msg_stride] seed bytes (device)
  const int* msg_len;           // [items] (device)
  long long msg_stride;
  const u64* moduli;            // tag_mode: [limbs] per limb; else [rows]
  u64* out;                     // [rows][n]
  int rows, rows_per_item, limbs, n;
  int tag_mode;                 // 1: message = seed || "ksk<digit>:<limb>" (row = digit*limbs+limb)
};
int launch_xof(const XofArgs& a, cudaStream_t st);

int launch_fill_uniform(u64* out, long long rows, int logn, const u64* keys, const u64* qs,
                        cudaStream_t st);

}  // namespace ck
