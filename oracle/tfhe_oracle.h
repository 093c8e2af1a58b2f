/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement (plain C, exact integer arithmetic)
 * of the CGGI/TFHE gate-bootstrapping path that the reference's GateBackend
 * (`/root/reference/pkg/src/hebnn/backend.py:116-150`, SimContext gates at
 * 205-237) declares but only simulates in plaintext.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or the
 * timed CPU baseline; the product path (paper_1806_03461_b200) never links it.
 *
 * Parity status:
 *   - decrypted-bit semantics: PINNED against the reference's own tests
 *     (test_backend.py truth tables / random sequences, test_circuits.py,
 *     test_compiler.py, test_acceptance.py) replayed on an oracle-backed
 *     GateBackend in tests/test_oracle_semantics.py;
 *   - ciphertext coefficients: the reference ships no TFHE code, keys or
 *     known-answer ciphertexts, so the ciphertext level
 *     is "parity unpinned" against the reference; it is pinned internally by
 *     (a) NTT products cross-checked against schoolbook mod 2^32 products,
 *     (b) committed golden vectors in tests/golden/ produced by this oracle.
 *
 * Algorithm: the published CGGI gate bootstrap (Chillotti, Gama, Georgieva,
 * Izabachene, "Faster fully homomorphic encryption: bootstrapping in less than
 * 0.1 seconds", ASIACRYPT 2016; the paper cites it at PAPER.md:259), restated
 * at BASELINE.json configs[0]: n=630, N=1024, k=1, Bg=2^7, l=3, KS base 2^2,
 * t=8, 32-bit torus, sigma_lwe=sigma_ks=2^-15, sigma_bk=2^-25.
 * Negacyclic products are exact: NTT modulo p = 2^64 - 2^32 + 1.
 */
#ifndef TFHE_ORACLE_H
#define TFHE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_params {
    int32_t n;            /* LWE dimension (630) */
    int32_t N;            /* ring degree (1024) */
    int32_t k;            /* TRLWE k (1) */
    int32_t bg_bits;      /* log2 Bg (7) */
    int32_t l;            /* gadget length (3) */
    int32_t ks_base_bits; /* log2 KS base (2) */
    int32_t ks_t;         /* KS length (8) */
    int32_t bk_unroll;    /* 1 (or 0): BK_i = TGSW(s_i); 2: key pairs, 3 TGSW per pair */
    double lwe_stdev;     /* 2^-15 (input LWE and KSK) */
    double bk_stdev;      /* 2^-25 */
} or_params;

void or_default_params(or_params *p);

/* ChaCha20-based deterministic stream (documented in DESIGN.md §PRNG). */
void or_chacha_block(const uint32_t key[8], uint64_t nonce, uint64_t counter, uint32_t out[16]);

/* Key generation (all arrays caller-allocated):
 *   lwe_key  [n]                              bits as u32 (0/1)
 *   trlwe_key[k*N]                            bits as u32 (0/1)
 *   bk       [n][(k+1)*l][(k+1)][N]           torus u32, coefficient domain (bk_unroll 1)
 *            [n/2][3][(k+1)*l][(k+1)][N]      bk_unroll 2: per pair (2m, 2m+1) the TGSWs of
 *                                             s_i s_j, s_i (1-s_j), (1-s_i) s_j
 *   ksk      [k*N][t][base-1][n+1]            torus u32 (digit value 0 omitted) */
int or_keygen(const or_params *p, uint64_t seed, uint32_t *lwe_key, uint32_t *trlwe_key,
              uint32_t *bk, uint32_t *ksk);

/* Encrypt bits under lwe_key: out[count][n+1]; ciphertext i uses the
 * ChaCha nonce (0x05<<56) | ((stream & 0xFFFFF) << 32) | (first_index + i). */
int or_encrypt(const or_params *p, const uint32_t *lwe_key, uint64_t seed, uint64_t stream,
               uint64_t first_index, const uint8_t *bits, size_t count, uint32_t *out);
void or_phase(const or_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
              int32_t *phase_out);
void or_decrypt(const or_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
                uint8_t *bits_out);
/* Phase of an extracted N-dimensional LWE under the TRLWE key. */
void or_phase_big(const or_params *p, const uint32_t *trlwe_key, const uint32_t *cts,
                  size_t count, int32_t *phase_out);

/* Exact negacyclic products (for cross-checks): out = a * b mod (X^N+1, 2^32). */
void or_negacyclic_mul_schoolbook(int32_t N, const int32_t *a, const uint32_t *b, uint32_t *out);
void or_negacyclic_mul_ntt(int32_t N, const int32_t *a, const uint32_t *b, uint32_t *out);

typedef struct or_ctx or_ctx;
or_ctx *or_ctx_create(const or_params *p, const uint32_t *bk, const uint32_t *ksk);
void or_ctx_destroy(or_ctx *c);

/* Stage entry points (bit-level parity of each stage). */
/* mod-switch of an LWE_n sample to Z_2N: out[n+1] (a_0..a_{n-1}, b). */
void or_modswitch(const or_ctx *c, const uint32_t *lwe, uint32_t *out);
/* Blind rotation from a test vector mu, stopping after `iters` key bits
 * (bk_unroll 2: after iters/2 key pairs); acc_out[(k+1)*N]. */
void or_blind_rotate(const or_ctx *c, const uint32_t *lwe, uint32_t mu, int32_t iters,
                     uint32_t *acc_out);
/* Bootstrap without key switching: out[k*N+1] extracted LWE. */
void or_bootstrap_wo_ks(const or_ctx *c, const uint32_t *lwe, uint32_t mu, uint32_t *out);
/* Key switch: in[k*N+1] -> out[n+1]. */
void or_keyswitch(const or_ctx *c, const uint32_t *in, uint32_t *out);

/* Generic bootstrapped 2-input gate: out = KS(BS((0,c0) + alpha*A + beta*B)).
 * (alpha, beta) in {-2,-1,0,1,2}; B may be NULL when beta == 0. */
void or_gate(const or_ctx *c, uint32_t c0, int32_t alpha, const uint32_t *A, int32_t beta,
             const uint32_t *B, uint32_t *out);
/* Three-input bootstrapped threshold gate: out = KS(BS((0,c0) + alpha*A + beta*B + gamma*C)). */
void or_gate3(const or_ctx *c, uint32_t c0, int32_t alpha, const uint32_t *A, int32_t beta,
              const uint32_t *B, int32_t gamma, const uint32_t *C, uint32_t *out);
/* Half adder from one blind rotation (kind HA): out_and = KS(S0),
 * out_xor = KS(sigma (S1 - S0) + (0, -sigma/8)), S0 / S1 the extractions at index
 * 0 / N/2 of BR((0,c0) + alpha*A + beta*B) (c0 = -1/8: the AND of the literals). */
void or_half_adder(const or_ctx *c, uint32_t c0, int32_t alpha, const uint32_t *A, int32_t beta,
                   const uint32_t *B, int32_t sigma, uint32_t *out_and, uint32_t *out_xor);
/* Native CGGI MUX: S ? A : B = KS((0,1/8) + BS((0,-1/8)+S+A) + BS((0,-1/8)-S+B)). */
void or_mux(const or_ctx *c, const uint32_t *S, const uint32_t *A, const uint32_t *B,
            uint32_t *out);

/* Batch of gates over a ciphertext pool with `threads` pthreads (CPU baseline).
 * Record layout mirrors include/hebnn_b200.h hb_gate. */
typedef struct or_gate_rec {
    uint32_t dst, src_a, src_b, src_c;
    uint32_t c0;
    int8_t alpha, beta, kind, gamma;  /* kind 0 LIN2, 1 MUX, 2 LIN3 (gamma * src_c),
                                         3 HA (dst = AND, src_c = XOR, gamma = XOR orientation) */
} or_gate_rec;
int or_run_gates(const or_ctx *c, const or_gate_rec *gates, size_t n, uint32_t *pool,
                 size_t pool_stride, int threads);

#ifdef __cplusplus
}
#endif
#endif
