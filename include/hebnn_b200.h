/*
 * hebnn_b200 — C ABI of the B200-native TFHE/CGGI gate-bootstrapping engine.
 *
 * This is the drop-in boundary underneath the reference's Python plugin
 * interface `GateBackend` (/root/reference/pkg/src/hebnn/backend.py:116-150).
 * The reference has no FFI for this path (it is pure Python and simulates
 * ciphertexts in plaintext, backend.py:161-257); the entry points below are the
 * ones its `GateBackend` methods bind to through ctypes in
 * paper_1806_03461_b200/backend.py (see INTEGRATION.md for the binding):
 *
 *   hb_keygen            <- SimContext.__init__            backend.py:171-174
 *                           (where a real backend creates keys; cli.py:72)
 *   hb_encrypt           <- SimContext.encrypt             backend.py:178-181
 *   hb_decrypt/hb_phase  <- SimContext.decrypt             backend.py:188-190
 *   hb_run_gates         <- SimContext._binary_gate/g_and/g_or/g_xor/g_xnor
 *                           backend.py:205-221 and g_mux 230-237, batched one
 *                           ASAP level (backend.py:207,235) at a time
 *   (trivial_const 183-186 and g_not 223-228 are free and never cross the ABI)
 *
 * Conventions: plain C types, caller-allocated buffers, `int` status (0 = ok,
 * <0 = error, message via hb_last_error(), thread-local). Torus elements are
 * uint32_t (arithmetic mod 2^32). Bit encoding: 1 -> +1/8 (2^29), 0 -> -1/8.
 * No torch or CUDA types appear in any signature.
 */
#ifndef HEBNN_B200_H
#define HEBNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_ABI_VERSION 4

/* status codes */
#define HB_OK 0
#define HB_EINVAL -1   /* bad argument (user error) */
#define HB_ECUDA -2    /* CUDA/driver failure (device error, never a user error) */
#define HB_ENOMEM -3   /* allocation failure */

/* TFHE parameter set (BASELINE.json configs[0] defaults from hb_default_params). */
typedef struct hb_params {
    int32_t n;            /* LWE dimension, 630 */
    int32_t N;            /* ring degree, 1024 */
    int32_t k;            /* TRLWE k, 1 */
    int32_t bg_bits;      /* log2 gadget base Bg, 7 */
    int32_t l;            /* gadget length, 3 */
    int32_t ks_base_bits; /* log2 key-switch base, 2 */
    int32_t ks_t;         /* key-switch length, 8 */
    int32_t bk_unroll;    /* blind-rotation key layout: 1 (or 0) = one TGSW(s_i) per key bit
                           * (CGGI), 2 = key pairs: TGSW(s_i s_j), TGSW(s_i (1-s_j)),
                           * TGSW((1-s_i) s_j) per (i, j) = (2m, 2m+1), one external
                           * product per pair (n must be even) */
    double lwe_stdev;     /* 2^-15: fresh LWE and KSK noise */
    double bk_stdev;      /* 2^-25: bootstrapping-key noise */
} hb_params;

/* One gate record of a level (all gates of one call are independent).
 *   kind HB_GATE_LIN2: pool[dst] = KS(BS((0,c0) + alpha*pool[src_a] + beta*pool[src_b]))
 *                      alpha, beta in {-2,-1,0,1,2}; NOT flags fold into signs.
 *   kind HB_GATE_MUX : pool[dst] = src_a ? src_b : src_c (native CGGI MUX:
 *                      2 blind rotations + 1 key switch); alpha / beta are the
 *                      signs (+-1) applied to src_b / src_c (NOT flags).
 *   kind HB_GATE_LIN3: pool[dst] = KS(BS((0,c0) + alpha*pool[src_a] + beta*pool[src_b]
 *                      + gamma*pool[src_c])), alpha, beta, gamma in {-2,-1,0,1,2}:
 *                      one bootstrap for 3-input threshold gates, e.g. majority
 *                      (c0 0, 1 1 1: a full adder's carry) and 3-input XOR
 *                      (c0 0, -2 -2 -2: a full adder's sum).
 *   kind HB_GATE_HA  : half adder from ONE blind rotation of
 *                      psi = (0,c0) + alpha*pool[src_a] + beta*pool[src_b], c0 = -1/8
 *                      (the AND of the literals alpha*A, beta*B); the accumulator
 *                      is extracted at index 0 (S0) and N/2 (S1):
 *                        pool[dst]   = KS(S0)                                 (AND)
 *                        pool[src_c] = KS(gamma (S1 - S0) + (0, -gamma/8))     (XOR,
 *                      gamma = +1; gamma = -1 its negation).  2 key switches.
 * Slot numbers address the engine pool; with `lanes` > 1 every record is run
 * for lanes l = 0..lanes-1 on slots (slot * lanes + l). */
typedef struct hb_gate {
    uint32_t dst, src_a, src_b, src_c;
    uint32_t c0;
    int8_t alpha, beta, kind, gamma;
} hb_gate;

#define HB_GATE_LIN2 0
#define HB_GATE_MUX 1
#define HB_GATE_LIN3 2
#define HB_GATE_HA 3

typedef struct hb_engine hb_engine;

int hb_abi_version(void);
const char *hb_last_error(void);
void hb_default_params(hb_params *p);
/* 1 if the kernels support these parameters (N = 1024, k = 1, Bg = 2^7, l = 3,
 * KS 2^2 x 8, 0 < n <= 639, even n for key pairs), else 0. Every entry point
 * taking params also checks them (HB_EINVAL); this lets a loader validate a
 * deserialised key document before sizing buffers from it. (ABI v4) */
int hb_params_valid(const hb_params *p);
size_t hb_lwe_words(const hb_params *p);   /* n + 1 */
size_t hb_bk_words(const hb_params *p);    /* T * (k+1)l * (k+1) * N, T = n (bk_unroll 1) or 3n/2 (2) */
size_t hb_ksk_words(const hb_params *p);   /* kN * t * (base-1) * (n+1) */

/* ---- host key material / encryption (replaces SimContext plaintext store) ---- */

/* Deterministic keygen from `seed` (ChaCha20 streams).
 * lwe_key[n], trlwe_key[k*N] (bits as u32), bk[T][(k+1)l][k+1][N] (coefficient
 * domain; T = n TGSW(s_i) for bk_unroll 1, T = 3n/2 for key pairs: TGSW(s_i s_j),
 * TGSW(s_i (1-s_j)), TGSW((1-s_i) s_j) per pair), ksk[kN][t][base-1][n+1].
 * threads <= 0 selects all host cores. */
int hb_keygen(const hb_params *p, uint64_t seed, uint32_t *lwe_key, uint32_t *trlwe_key,
              uint32_t *bk, uint32_t *ksk, int threads);

/* Encrypt count bits (each 0/1, else HB_EINVAL) into out[count][out_stride]
 * (out_stride >= n+1). Ciphertext i uses ChaCha nonce
 * (0x05<<56) | ((stream & 0xFFFFF) << 32) | (first_index + i) with the key
 * expanded from seed (first_index + count <= 2^32). */
int hb_encrypt(const hb_params *p, const uint32_t *lwe_key, uint64_t seed, uint64_t stream,
               uint64_t first_index, const uint8_t *bits, size_t count, uint32_t *out,
               size_t out_stride);

/* phase = b - <a, s> (int32, i.e. signed torus * 2^32); bit = phase > 0. */
int hb_phase(const hb_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
             size_t stride, int32_t *phase_out);
int hb_decrypt(const hb_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
               size_t stride, uint8_t *bits_out);

/* ---- device engine (sm_100a) ---- */

/* Create an engine on CUDA device `device`: uploads the KSK, uploads the BK and
 * transforms it to the FP64 negacyclic Fourier domain on the device. */
int hb_engine_create(int device, const hb_params *p, const uint32_t *bk, const uint32_t *ksk,
                     hb_engine **out);
int hb_engine_destroy(hb_engine *e);

/* Ciphertext pool: `slots` LWE samples of hb_pool_stride() words each. Growing
 * preserves contents. */
int hb_pool_reserve(hb_engine *e, size_t slots);
size_t hb_pool_capacity(const hb_engine *e);
size_t hb_pool_stride(const hb_engine *e);
/* contiguous slot range <-> host (host rows of host_stride >= n+1 words) */
int hb_pool_upload(hb_engine *e, size_t first_slot, size_t count, const uint32_t *host,
                   size_t host_stride);
int hb_pool_download(hb_engine *e, size_t first_slot, size_t count, uint32_t *host,
                     size_t host_stride);
/* Asynchronous variants on the engine's copy streams (overlap transfers with
 * compute; host buffers must be pinned and stay valid until hb_sync).  An
 * async upload may overlap the most recently issued level but waits for every
 * earlier one (double-buffered slot regions); the next hb_run_gates waits for
 * the last async upload; an async download waits for every level issued
 * before it. */
int hb_pool_upload_async(hb_engine *e, size_t first_slot, size_t count, const uint32_t *host,
                         size_t host_stride);
int hb_pool_download_async(hb_engine *e, size_t first_slot, size_t count, uint32_t *host,
                           size_t host_stride);
/* scattered slots -> host (gathered on the device, one copy) */
/* Device-resident exchange (multi-GPU all-gather without host staging): copy
 * pool slots `slots[count]` into / consecutive slots from a device buffer of
 * this engine's GPU with row stride dev_stride (>= n+1 words); synchronous. */
int hb_pool_gather_device(hb_engine *e, const uint32_t *slots, size_t count, uint32_t *dev_out,
                          size_t dev_stride);
int hb_pool_put_device(hb_engine *e, size_t first_slot, size_t count, const uint32_t *dev_in,
                       size_t dev_stride);
int hb_pool_gather(hb_engine *e, const uint32_t *slots, size_t count, uint32_t *host,
                   size_t host_stride);

/* Run one level of independent gates (asynchronous on the engine stream).
 * Fused prologue (linear combination + mod switch) -> blind rotation ->
 * sample extract, then batched key switch into pool[dst].  Very wide levels
 * (> 2^20 blind rotations x lanes) are split into several launches. */
int hb_run_gates(hb_engine *e, const hb_gate *gates, size_t n, uint32_t lanes);
int hb_sync(hb_engine *e);  /* compute and copy streams */

/* Device time (ms, CUDA events on the engine stream) of the blind-rotation and
 * key-switch kernels of the most recent hb_run_gates launch (its last chunk);
 * accumulated counters of
 * executed blind rotations and key switches since creation. */
int hb_last_timing(hb_engine *e, float *br_ms, float *ks_ms);
int hb_counters(hb_engine *e, uint64_t *blind_rotations, uint64_t *key_switches,
                uint64_t *kernel_launches);

/* Write `bytes` (0: 256 MiB, i.e. > 2x the 126 MB L2) of scratch on the engine
 * stream so the next launch starts with a cold L2 (benchmark hygiene). */
int hb_flush_l2(hb_engine *e, size_t bytes);
/* FP64 roofline probe: DFMA throughput (TFLOP/s) of this device, measured with
 * CUDA events on the engine stream (8 independent FMA chains per thread). */
int hb_measure_fp64_peak(hb_engine *e, double *tflops);

/* ---- stage entry points for bit-level parity (synchronous, host buffers) ---- */

/* ACC after the first `iters` key bits of the blind rotation of lwe[n+1]
 * (key pairs: iters/2 pair steps) with test vector mu: acc_out[(k+1)N]. */
int hb_debug_blind_rotate(hb_engine *e, const uint32_t *lwe, uint32_t mu, int32_t iters,
                          uint32_t *acc_out);
/* count independent bootstraps without key switch: lin[count][n+1] -> out[count][kN+1] */
int hb_debug_bootstrap_wo_ks(hb_engine *e, const uint32_t *lin, size_t count, uint32_t *out);
/* count key switches: in[count][kN+1] -> out[count][n+1] */
int hb_debug_keyswitch(hb_engine *e, const uint32_t *in, size_t count, uint32_t *out);
/* max |x - round(x)| over all coefficients of all inverse FFTs of the last
 * hb_debug_bootstrap_wo_ks call (FFT rounding margin; exactness needs < 0.5). */
int hb_debug_fft_margin(hb_engine *e, double *max_err);
/* which = 0: forward negacyclic FFT (scaled by 1/512) of count u32 polynomials
 * polys[count][N] -> out[count][N/2][2]; which = 1: copy the first `count`
 * polynomials of the device BK Fourier table (polys ignored; key pairs store
 * it in ring-stage order). */
int hb_debug_fourier(hb_engine *e, const uint32_t *polys, size_t count, double *out, int which);

#ifdef __cplusplus
}
#endif
#endif
