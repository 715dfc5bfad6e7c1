/*
 * ckks_b200.h -- C ABI of the B200-native CKKS key-switching library.
 *
 * Drop-in boundary for the reference package `ckkslab` (pure Python, no FFI
 * of its own): each entry point below replaces the numpy routine cited next
 * to it (paths under /root/reference/pkg/src/ckkslab/).  The Python mirror
 * paper_2112_06396_b200/{rnspoly,ckks}.py binds these with ctypes, keeping
 * the reference's function names, argument meaning and error behaviour.
 *
 * Conventions
 *   - Polynomials are row-major [limb][N] uint64 arrays of canonical residues
 *     in DEVICE memory (caller-owned, e.g. torch uint64 tensors).  A "batch"
 *     is a leading dimension with the stated stride.
 *   - Prime indices refer to the plan's full basis: chain[0..L) then
 *     special[0..K)  (== the full-basis row of a switching key).
 *   - Everything is stream-ordered on `stream` (a cudaStream_t); no host
 *     synchronisation, no allocation on the hot path (workspace is passed in).
 *   - Return value: 0 on success, a negative CK_ERR_* argument/state code, or
 *     a positive cudaError_t.
 *   - A plan is immutable after creation and may be shared across threads.
 */
#ifndef CKKS_B200_H
#define CKKS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CK_OK 0
#define CK_ERR_ARG (-1)       /* bad argument (shape, level, null pointer) */
#define CK_ERR_MODULUS (-2)   /* modulus not prime / not 1 mod 2N / >= 2^60 */
#define CK_ERR_ALLOC (-3)     /* device allocation failed (plan creation only) */
#define CK_ERR_DEVICE (-4)    /* no CUDA device */

typedef struct ck_plan ck_plan;
typedef struct ck_bconv ck_bconv;
typedef void* ck_stream; /* cudaStream_t */

int ck_version(void);
const char* ck_error_string(int code);
/* number of CUDA kernels this library has launched so far (process-wide) */
int64_t ck_launch_count(void);

/* ---- plan: ring degree, basis, twiddles, per-level conversion tables ----
 * Replaces CkksParams (ckks.py:31-65) + NttContext/get_ctx (rnspoly.py:24-105)
 * + the _bc_tables/_bc_center_tables caches (rnspoly.py:245-300).
 * psi for each modulus is g^((q-1)/2N) with g the smallest primitive root
 * (zq.py:79-84), so eval-domain slot order equals the reference's.        */
int ck_plan_create(int log_n, const uint64_t* chain, int n_chain, const uint64_t* special,
                   int n_special, int dnum, ck_plan** out);
int ck_plan_destroy(ck_plan* plan);
/* out[0..4] = {N, n_chain, n_special, dnum, alpha} */
int ck_plan_info(const ck_plan* plan, int64_t* out);
/* psi per prime (host array of n_chain + n_special) */
int ck_plan_psi(const ck_plan* plan, uint64_t* psi_out);
/* copy the w-part of a twiddle table (host array of N): NttContext.tw / .itw */
int ck_plan_twiddles(const ck_plan* plan, int prime, int inverse, uint64_t* out);

/* ---- NTT / INTT over `rows` contiguous limbs (x batch) ----
 * NttContext.ntt / .intt (rnspoly.py:48-79), _ntt_rows (ckks.py:359-364).
 * prime_idx: DEVICE int32[rows].  In place.                               */
int ck_ntt(const ck_plan* plan, uint64_t* data, const int32_t* prime_idx, int rows, int batch,
           int64_t batch_stride, int inverse, ck_stream stream);

/* ---- elementwise (RnsPoly.add/sub/mul/neg/mul_scalars, rnspoly.py:182-210) ----
 * op: 0 add, 1 sub, 2 mul, 3 neg, 4 mul by per-row constant, 5 copy,
 *     6 add per-row constant (encode_const + pt_add, ckks.py:557-568: the
 *       evaluation form of a degree-0 polynomial is that residue in every slot).
 * cst: DEVICE {c, floor(c*2^64/q)} pairs per row (ops 4 and 6).            */
int ck_poly_op(const ck_plan* plan, int op, uint64_t* out, const uint64_t* x, const uint64_t* y,
               const int32_t* prime_idx, const uint64_t* cst, int rows, ck_stream stream);

/* ---- eval-domain Galois automorphism X -> X^t (RnsPoly.automorph eval,
 * rnspoly.py:127-135, 228-233); gather, prime-independent.                */
int ck_automorph(const ck_plan* plan, uint64_t* out, const uint64_t* x, int rows,
                 uint64_t galois_t, ck_stream stream);

/* ---- generic basis conversion between two sets of plan primes ----
 * bc_convert (rnspoly.py:264-284) / bc_convert_centered (rnspoly.py:303-331).
 * Input rows: ns coefficient-rep rows (contiguous); output: nd rows.       */
int ck_bconv_create(const ck_plan* plan, const int32_t* src_idx, int ns, const int32_t* dst_idx,
                    int nd, int centered, ck_bconv** out);
int ck_bconv_destroy(ck_bconv* bc);
int ck_bconv_apply(const ck_plan* plan, const ck_bconv* bc, const uint64_t* in, uint64_t* out,
                   ck_stream stream);

/* ---- key switching at `level` chain limbs (l <= n_chain) ----
 * Layouts (per batch item):  a, b: [l][N];  digits: [beta][l+K][N];
 * key_b, key_a: [dnum][L+K][N] full-basis rows (SwitchingKey, ckks.py:188-199);
 * u, v: [l+K][N].  beta = number of digit spans at level l (ckks.py:56-62). */
size_t ck_workspace_bytes(const ck_plan* plan, int level, int batch);

/* _decomp_modup (ckks.py:421-441) */
int ck_modup(const ck_plan* plan, const uint64_t* a_eval, int level, uint64_t* digits,
             uint64_t* workspace, int batch, ck_stream stream);

/* _kskip (ckks.py:450-465) on automorph(digits, t) (t = 1: none).
 * galois: optional DEVICE uint64[batch] per-item elements (overrides t).   */
int ck_kskip(const ck_plan* plan, const uint64_t* digits, const uint64_t* key_b,
             const uint64_t* key_a, int level, uint64_t galois_t, const uint64_t* galois,
             uint64_t* u, uint64_t* v, int batch, ck_stream stream);

/* _moddown_poly (ckks.py:397-416): x [l+K][N] eval -> out [keep][N].
 * merged = 0: drop the K specials, keep l   (_moddown_pair, ckks.py:468-475)
 * merged = 1: drop (q_{l-1},) + specials, keep l-1 (ckks.py:643-651, 712-717)
 * merged = 2: rescale: x has l rows, drop q_{l-1} (ckks.py:375-394)
 * addend (nullable, [keep][N]) is added after automorph by galois_t.
 * x's dropped rows are CLOBBERED (used as scratch).                        */
int ck_moddown(const ck_plan* plan, uint64_t* x, int level, int merged, uint64_t* out,
               const uint64_t* addend, uint64_t galois_t, uint64_t* workspace, int batch,
               ck_stream stream);

/* Full rotation key-switch (ckks.hrotate for one rotation, ckks.py:655-667;
 * mode 1 = conjugate order, automorph first, ckks.py:674-681):
 *   (out_a, out_b) = (u, v + automorph(b, t)) after ModUp/KSKIP/ModDown.
 * galois: optional DEVICE uint64[batch] (distinct element per item).        */
int ck_rotate(const ck_plan* plan, const uint64_t* a, const uint64_t* b, const uint64_t* key_b,
              const uint64_t* key_a, int level, uint64_t galois_t, const uint64_t* galois,
              int mode, uint64_t* out_a, uint64_t* out_b, uint64_t* workspace, int batch,
              ck_stream stream);

/* ---- one entry for every key-switch flavour (SURVEY 8(b) ck_keyswitch) ----
 * mode 0: rotation (ck_rotate mode 0), 1: conjugation (ck_rotate mode 1), one
 * key per batch item as ck_rotate takes them ([batch][dnum][L+K][N]);
 * 2: relinearisation (ck_relin): `a` = a3 [batch][level][N] and `b` = (b3, c3) as
 * [batch][2][level][N]; outputs [batch][level-1][N]; galois_t / galois ignored, the
 * key is one relin key shared by the batch.  Workspace: ck_keyswitch_workspace_bytes. */
size_t ck_keyswitch_workspace_bytes(const ck_plan* plan, int level, int mode, int batch);
int ck_keyswitch(const ck_plan* plan, const uint64_t* a, const uint64_t* b, const uint64_t* key_b,
                 const uint64_t* key_a, int level, uint64_t galois_t, const uint64_t* galois,
                 int mode, uint64_t* out_a, uint64_t* out_b, uint64_t* workspace, int batch,
                 ck_stream stream);
/* ---- relinearisation key-switch of new_mult (ckks.py:639-651) ----
 * (a3, b3, c3) at `level` chain limbs (value_mult / addend / const already
 * folded into b3, c3 by the caller, ckks.py:624-638) ->
 *   digits = ModUp(a3); (u, v) = KSKIP(digits, relin key, t = 1);
 *   u += pmodup(b3); v += pmodup(c3);  out = ModDown by P * q_last (l-1 limbs).
 * batch independent products: a3, b3, c3 [batch][level][N], outputs
 * [batch][level-1][N] each; ONE relinearisation key [dnum][L+K][N] shared by
 * the batch (KeySet.relin, ckks.py:230).  level >= 2.  Runs the fused
 * key-switch pipeline of ck_rotate (no automorphism; the pmodup terms fold
 * into the ModDown epilogue).  No host round trips.                          */
size_t ck_relin_workspace_bytes(const ck_plan* plan, int level, int batch);
int ck_relin(const ck_plan* plan, const uint64_t* a3, const uint64_t* b3, const uint64_t* c3,
             const uint64_t* key_b, const uint64_t* key_a, int level, uint64_t* out_a,
             uint64_t* out_b, uint64_t* workspace, int batch, ck_stream stream);
/* ---- hoisted rotations (ckks.hrotate, ckks.py:655-667) ----
 * One shared ModUp of a; n_rot KSKIPs in one launch (shared evaluation-form
 * digits, per-rotation key and Galois element); ModDown pairs batched.
 * key_b, key_a: DEVICE arrays of n_rot pointers, each to one switching key's
 * [dnum][L+K][N] rows (SwitchingKey.b / .a, ckks.py:188-199) -- the keys stay
 * where the caller keeps them (KeySet.rot, ckks.py:231), nothing is stacked.
 * galois: DEVICE uint64[n_rot].  Outputs [n_rot][level][N] x 2.              */
size_t ck_hrotate_workspace_bytes(const ck_plan* plan, int level, int n_rot);
int ck_hrotate(const ck_plan* plan, const uint64_t* a, const uint64_t* b,
               const uint64_t* const* key_b, const uint64_t* const* key_a,
               const uint64_t* galois, int level, int n_rot, uint64_t* out_a, uint64_t* out_b,
               uint64_t* workspace, ck_stream stream);
/* ---- double-hoisted plaintext matrix-vector product (ckks.pt_matvec, ckks.py:684-719) ----
 * Any number of diagonals (the reference takes any dict; a radix-r bootstrap
 * stage has 2r-1, bootstrap.py:128-133).  diags: DEVICE array of
 * n_rot + has_identity pointers to [level+K][N] raised-basis rows, rotated
 * offsets first (matching key_b/key_a, DEVICE pointer arrays [n_rot] as in
 * ck_hrotate), identity last; galois: DEVICE uint64[n_rot + has_identity]
 * (identity's element = 1).  One shared ModUp, KSKIP + diagonal MAC in chunks
 * of <= 32 diagonals accumulating on the raised basis, one merged ModDown.
 * Output [level-1][N].                                                       */
size_t ck_pt_matvec_workspace_bytes(const ck_plan* plan, int level, int n_diag);
int ck_pt_matvec(const ck_plan* plan, const uint64_t* a, const uint64_t* b,
                 const uint64_t* const* key_b, const uint64_t* const* key_a,
                 const uint64_t* galois, const uint64_t* const* diags, int level, int n_rot,
                 int has_identity, uint64_t* out_a, uint64_t* out_b, uint64_t* workspace,
                 ck_stream stream);
/* ---- hoisted BSGS linear transform (composites.py:249-293) ----
 * == sum_{j=1..giant} rotate(pt_matvec(ct, {k: diag[j][k]}), -baby*j)  (ckks.py:684-719)
 * One shared ModUp; `baby` KSKIPs (Galois 5^k, k = 1..baby; chunks of <= 32);
 * diagonal MACs into `giant` raised accumulators; merged ModDown (P*q_last);
 * `giant` batched rotations at level-1 (Galois 5^(baby*j)); sum.
 * a, b: [level][N]; baby / giant keys: DEVICE pointer arrays [baby] / [giant]
 * (one [dnum][L+K][N] block each); diags: DEVICE pointer array [giant][baby]
 * of [level+K][N] raised-basis eval rows; galois arrays DEVICE uint64.
 * Output: [level-1][N] x 2.                                                  */
size_t ck_bsgs_workspace_bytes(const ck_plan* plan, int level, int baby, int giant);
int ck_bsgs(const ck_plan* plan, const uint64_t* a, const uint64_t* b,
            const uint64_t* const* baby_key_b, const uint64_t* const* baby_key_a,
            const uint64_t* const* giant_key_b, const uint64_t* const* giant_key_a,
            const uint64_t* const* diags, const uint64_t* baby_galois,
            const uint64_t* giant_galois, int level, int baby, int giant, uint64_t* out_a,
            uint64_t* out_b, uint64_t* workspace, ck_stream stream);
/* ---- compressed evaluation keys: SHAKE256 uniform rows (ckks.py:169-215) ----
 * ck_xof_uniform: row r = first n words of SHAKE256(msgs[r][0:msg_lens[r]])
 * (little-endian u64) below floor(2^64/q_r)*q_r, each reduced mod q_r
 * (ckks._xof_uniform, ckks.py:169-185).  msgs, msg_lens, moduli: DEVICE arrays.
 * ck_expand_key_a: the a-rows of n_keys compressed switching keys
 * (SwitchingKey.expand, ckks.py:207-215): key_a[k][j][i] =
 * _xof_uniform(seed_k || "ksk<j>:<i>", q_i, N) over the plan's full basis
 * (chain || special) and its top-level digit count; seeds [n_keys][seed_stride]
 * and seed_lens [n_keys] are DEVICE arrays; output [n_keys][dnum][L+K][N].  */
int ck_xof_uniform(const uint8_t* msgs, const int32_t* msg_lens, int64_t msg_stride,
                   const uint64_t* moduli, int rows, int n, uint64_t* out, ck_stream stream);
int ck_expand_key_a(const ck_plan* plan, const uint8_t* seeds, const int32_t* seed_lens,
                    int64_t seed_stride, int n_keys, uint64_t* key_a, ck_stream stream);

/* ---- synthetic inputs: counter-based uniform residues (paper_2112_06396_b200.synth) ----
 * row r: out[r][k] = mulhi(splitmix64(keys[r] + k), qs[r]).  keys, qs: DEVICE. */
int ck_fill_uniform(uint64_t* out, int64_t rows, int log_n, const uint64_t* keys,
                    const uint64_t* qs, ck_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* CKKS_B200_H */
