/*
 * TEST INFRASTRUCTURE ONLY — see tfhe_oracle.h for scope, parity status and
 * the rule that only tests/, smoke() and bench.py's CPU legs may load it.
 *
 * Plain-C exact-integer restatement of the CGGI gate bootstrap behind the
 * reference's GateBackend (backend.py:116-150).  Each function names the
 * reference behaviour it realises; the cryptographic steps follow the
 * published CGGI algorithm (PAPER.md:259 cites it) at BASELINE.json configs[0].
 */
#define _GNU_SOURCE
#include "tfhe_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* parameters                                                                */
/* ------------------------------------------------------------------------ */

void or_default_params(or_params *p) {
    p->n = 630;
    p->N = 1024;
    p->k = 1;
    p->bg_bits = 7;
    p->l = 3;
    p->ks_base_bits = 2;
    p->ks_t = 8;
    p->bk_unroll = 2;  /* key pairs */
    p->lwe_stdev = 1.0 / 32768.0;      /* 2^-15 */
    p->bk_stdev = 1.0 / 33554432.0;    /* 2^-25 */
}

/* ------------------------------------------------------------------------ */
/* ChaCha20 stream: key = 8 words from the 64-bit seed,    */
/* nonce = 64-bit domain/item id, 64-bit block counter.                      */
/* ------------------------------------------------------------------------ */

#define ROTL(a, b) (((a) << (b)) | ((a) >> (32 - (b))))
#define QR(a, b, c, d)                                                        \
    do {                                                                      \
        a += b; d ^= a; d = ROTL(d, 16);                                      \
        c += d; b ^= c; b = ROTL(b, 12);                                      \
        a += b; d ^= a; d = ROTL(d, 8);                                       \
        c += d; b ^= c; b = ROTL(b, 7);                                       \
    } while (0)

void or_chacha_block(const uint32_t key[8], uint64_t nonce, uint64_t counter, uint32_t out[16]) {
    uint32_t s[16];
    s[0] = 0x61707865u; s[1] = 0x3320646eu; s[2] = 0x79622d32u; s[3] = 0x6b206574u;
    for (int i = 0; i < 8; i++) s[4 + i] = key[i];
    s[12] = (uint32_t)counter; s[13] = (uint32_t)(counter >> 32);
    s[14] = (uint32_t)nonce;   s[15] = (uint32_t)(nonce >> 32);
    uint32_t x[16];
    memcpy(x, s, sizeof x);
    for (int r = 0; r < 10; r++) {
        QR(x[0], x[4], x[8], x[12]); QR(x[1], x[5], x[9], x[13]);
        QR(x[2], x[6], x[10], x[14]); QR(x[3], x[7], x[11], x[15]);
        QR(x[0], x[5], x[10], x[15]); QR(x[1], x[6], x[11], x[12]);
        QR(x[2], x[7], x[8], x[13]); QR(x[3], x[4], x[9], x[14]);
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

typedef struct {
    uint32_t key[8];
    uint64_t nonce, counter;
    uint32_t buf[16];
    int pos;
} rng_t;

static void seed_key(uint64_t seed, uint32_t key[8]) {
    /* splitmix64 expansion of the seed into 256 key bits */
    uint64_t z = seed;
    for (int i = 0; i < 4; i++) {
        z += 0x9E3779B97F4A7C15ull;
        uint64_t t = z;
        t = (t ^ (t >> 30)) * 0xBF58476D1CE4E5B9ull;
        t = (t ^ (t >> 27)) * 0x94D049BB133111EBull;
        t ^= t >> 31;
        key[2 * i] = (uint32_t)t;
        key[2 * i + 1] = (uint32_t)(t >> 32);
    }
}

static void rng_init(rng_t *r, uint64_t seed, uint64_t nonce) {
    seed_key(seed, r->key);
    r->nonce = nonce;
    r->counter = 0;
    r->pos = 16;
}

static uint32_t rng_u32(rng_t *r) {
    if (r->pos == 16) {
        or_chacha_block(r->key, r->nonce, r->counter++, r->buf);
        r->pos = 0;
    }
    return r->buf[r->pos++];
}

static uint64_t rng_u64(rng_t *r) {
    uint64_t lo = rng_u32(r);
    uint64_t hi = rng_u32(r);
    return lo | (hi << 32);
}

/* Box-Muller (cosine branch only), rounded to the 2^32 torus. */
static uint32_t rng_gauss_torus(rng_t *r, double stdev) {
    double u1 = (double)((rng_u64(r) >> 11) + 1) * (1.0 / 9007199254740992.0);
    double u2 = (double)(rng_u64(r) >> 11) * (1.0 / 9007199254740992.0);
    double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
    double scale = stdev * 4294967296.0;
    double v = z * scale;
    int64_t e = llround(v);
    return (uint32_t)e;
}

#define DOM_LWE_KEY 0x01ull
#define DOM_TRLWE_KEY 0x02ull
#define DOM_BK 0x03ull
#define DOM_KSK 0x04ull
#define DOM_ENC 0x05ull
#define DOM_BK2 0x06ull

/* bk_unroll 0 is read as 1 */
static inline int bk_unroll(const or_params *p) { return p->bk_unroll == 2 ? 2 : 1; }

/* ------------------------------------------------------------------------ */
/* negacyclic arithmetic                                                     */
/* ------------------------------------------------------------------------ */

/* out = X^a * in  (a in [0, 2N)) */
static void poly_mul_xai(int N, int a, const uint32_t *in, uint32_t *out) {
    if (a < N) {
        for (int i = 0; i < a; i++) out[i] = 0u - in[i - a + N];
        for (int i = a; i < N; i++) out[i] = in[i - a];
    } else {
        int aa = a - N;
        for (int i = 0; i < aa; i++) out[i] = in[i - aa + N];
        for (int i = aa; i < N; i++) out[i] = 0u - in[i - aa];
    }
}

void or_negacyclic_mul_schoolbook(int32_t N, const int32_t *a, const uint32_t *b, uint32_t *out) {
    for (int i = 0; i < N; i++) out[i] = 0;
    for (int i = 0; i < N; i++) {
        uint32_t ai = (uint32_t)a[i];
        for (int j = 0; j < N; j++) {
            uint32_t prod = ai * b[j];
            int d = i + j;
            if (d < N) out[d] += prod;
            else out[d - N] -= prod;
        }
    }
}

/* Goldilocks field p = 2^64 - 2^32 + 1 */
#define GL_P 0xFFFFFFFF00000001ull
#define GL_EPS 0xFFFFFFFFull

static inline uint64_t gl_reduce128(unsigned __int128 x) {
    /* branch-free Goldilocks reduction: 2^64 = 2^32 - 1, 2^96 = -1 (mod p) */
    const uint64_t lo = (uint64_t)x, hi = (uint64_t)(x >> 64);
    const uint64_t hh = hi >> 32, hl = hi & GL_EPS;
    uint64_t t0 = lo - hh;
    t0 -= (0 - (uint64_t)(lo < hh)) & GL_EPS;
    const uint64_t t1 = hl * GL_EPS;
    uint64_t r = t0 + t1;
    r += (0 - (uint64_t)(r < t1)) & GL_EPS;
    r -= (0 - (uint64_t)(r >= GL_P)) & GL_P;
    return r;
}
static inline uint64_t gl_mul(uint64_t a, uint64_t b) {
    return gl_reduce128((unsigned __int128)a * b);
}
static inline uint64_t gl_add(uint64_t a, uint64_t b) {
    const uint64_t r = a + b;
    const uint64_t over = (uint64_t)(r < a) | (uint64_t)(r >= GL_P);
    return r - ((0 - over) & GL_P);
}
static inline uint64_t gl_sub(uint64_t a, uint64_t b) {
    const uint64_t r = a - b;
    return r + ((0 - (uint64_t)(a < b)) & GL_P);
}
static uint64_t gl_pow(uint64_t b, uint64_t e) {
    uint64_t r = 1;
    while (e) {
        if (e & 1) r = gl_mul(r, b);
        b = gl_mul(b, b);
        e >>= 1;
    }
    return r;
}
static inline uint64_t gl_from_i64(int64_t v) {
    return v >= 0 ? (uint64_t)v : GL_P - (uint64_t)(-v);
}
static inline uint32_t gl_to_torus(uint64_t v) {
    /* centred lift to (-p/2, p/2], then reduce mod 2^32 */
    int64_t s = v > GL_P / 2 ? -(int64_t)(GL_P - v) : (int64_t)v;
    return (uint32_t)s;
}

typedef struct {
    int N, logN;
    uint64_t *psi_pows;      /* psi^j, j < N */
    uint64_t *psi_inv_pows;  /* psi^-j * N^-1 */
    uint64_t *w;             /* omega^j bit-reversed table for CT butterflies */
    uint64_t *winv;
    int *rev;                /* bit-reversal permutation */
    uint64_t *ws, *wsinv;    /* per-stage contiguous twiddles: stage len -> [len/2] at offset len/2 - 1 */
} ntt_plan;

static int bitrev(int x, int bits) {
    int r = 0;
    for (int i = 0; i < bits; i++) r |= ((x >> i) & 1) << (bits - 1 - i);
    return r;
}

static void ntt_plan_init(ntt_plan *pl, int N) {
    pl->N = N;
    pl->logN = 0;
    while ((1 << pl->logN) < N) pl->logN++;
    /* 7 generates F_p^*; psi = primitive 2N-th root of unity */
    uint64_t psi = gl_pow(7, (GL_P - 1) / (uint64_t)(2 * N));
    uint64_t psi_inv = gl_pow(psi, 2 * (uint64_t)N - 1);
    uint64_t n_inv = gl_pow((uint64_t)N, GL_P - 2);
    uint64_t omega = gl_mul(psi, psi), omega_inv = gl_mul(psi_inv, psi_inv);
    pl->psi_pows = malloc(sizeof(uint64_t) * N);
    pl->psi_inv_pows = malloc(sizeof(uint64_t) * N);
    pl->w = malloc(sizeof(uint64_t) * N);
    pl->winv = malloc(sizeof(uint64_t) * N);
    pl->rev = malloc(sizeof(int) * N);
    for (int j = 0; j < N; j++) pl->rev[j] = bitrev(j, pl->logN);
    uint64_t a = 1, b = n_inv;
    for (int j = 0; j < N; j++) {
        pl->psi_pows[j] = a;
        pl->psi_inv_pows[j] = b;
        a = gl_mul(a, psi);
        b = gl_mul(b, psi_inv);
    }
    /* w[j] = omega^j for j < N/2 (natural order) */
    uint64_t x = 1, y = 1;
    for (int j = 0; j < N / 2; j++) {
        pl->w[j] = x;
        pl->winv[j] = y;
        x = gl_mul(x, omega);
        y = gl_mul(y, omega_inv);
    }
    pl->ws = malloc(sizeof(uint64_t) * N);
    pl->wsinv = malloc(sizeof(uint64_t) * N);
    for (int len = 2; len <= N; len <<= 1) {
        const int half = len >> 1, step = N / len;
        for (int j = 0; j < half; j++) {
            pl->ws[half - 1 + j] = pl->w[j * step];
            pl->wsinv[half - 1 + j] = pl->winv[j * step];
        }
    }
}

static void ntt_plan_free(ntt_plan *pl) {
    free(pl->psi_pows); free(pl->psi_inv_pows); free(pl->w); free(pl->winv); free(pl->rev);
    free(pl->ws); free(pl->wsinv);
}

/* in-place cyclic NTT, natural-order input -> natural-order output
 * (bit reversal, then radix-2 Cooley-Tukey with contiguous per-stage twiddles) */
static void ntt_core(const ntt_plan *pl, uint64_t *a, const uint64_t *w) {
    const int N = pl->N;
    const uint64_t *stage_w = (w == pl->w) ? pl->ws : pl->wsinv;
    for (int i = 0; i < N; i++) {
        int j = pl->rev[i];
        if (j > i) { uint64_t t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (int len = 2; len <= N; len <<= 1) {
        const int half = len >> 1;
        const uint64_t *ww = stage_w + half - 1;
        for (int s = 0; s < N; s += len) {
            uint64_t *lo = a + s, *hi = a + s + half;
            for (int j = 0; j < half; j++) {
                const uint64_t u = lo[j];
                const uint64_t v = gl_mul(hi[j], ww[j]);
                lo[j] = gl_add(u, v);
                hi[j] = gl_sub(u, v);
            }
        }
    }
}

static void ntt_forward_i64(const ntt_plan *pl, const int64_t *in, uint64_t *out) {
    for (int j = 0; j < pl->N; j++) out[j] = gl_mul(gl_from_i64(in[j]), pl->psi_pows[j]);
    ntt_core(pl, out, pl->w);
}

static void ntt_inverse_torus(const ntt_plan *pl, uint64_t *a, uint32_t *out) {
    ntt_core(pl, a, pl->winv);
    for (int j = 0; j < pl->N; j++) out[j] = gl_to_torus(gl_mul(a[j], pl->psi_inv_pows[j]));
}

void or_negacyclic_mul_ntt(int32_t N, const int32_t *a, const uint32_t *b, uint32_t *out) {
    ntt_plan pl;
    ntt_plan_init(&pl, N);
    int64_t *ai = malloc(sizeof(int64_t) * N), *bi = malloc(sizeof(int64_t) * N);
    uint64_t *A = malloc(sizeof(uint64_t) * N), *B = malloc(sizeof(uint64_t) * N);
    for (int j = 0; j < N; j++) { ai[j] = a[j]; bi[j] = (int32_t)b[j]; }
    ntt_forward_i64(&pl, ai, A);
    ntt_forward_i64(&pl, bi, B);
    for (int j = 0; j < N; j++) A[j] = gl_mul(A[j], B[j]);
    ntt_inverse_torus(&pl, A, out);
    free(ai); free(bi); free(A); free(B);
    ntt_plan_free(&pl);
}

/* ------------------------------------------------------------------------ */
/* key generation / encryption (reference: SimContext.encrypt/decrypt,       */
/* backend.py:178-190; real CGGI encryption replaces the plaintext store)    */
/* ------------------------------------------------------------------------ */

static uint32_t lwe_dot(const uint32_t *a, const uint32_t *key, int n) {
    uint32_t acc = 0;
    for (int i = 0; i < n; i++) acc += a[i] & (0u - key[i]);
    return acc;
}

/* poly * binary key: out = a * s mod X^N+1, exact (s in {0,1}) */
static void poly_mul_binary(int N, const uint32_t *a, const uint32_t *s, uint32_t *out) {
    memset(out, 0, sizeof(uint32_t) * N);
    for (int i = 0; i < N; i++) {
        if (!s[i]) continue;
        /* out += X^i * a */
        for (int j = 0; j < N; j++) {
            int d = i + j;
            if (d < N) out[d] += a[j];
            else out[d - N] -= a[j];
        }
    }
}

int or_keygen(const or_params *p, uint64_t seed, uint32_t *lwe_key, uint32_t *trlwe_key,
              uint32_t *bk, uint32_t *ksk) {
    const int n = p->n, N = p->N, k = p->k, l = p->l;
    if (bk_unroll(p) == 2 && (n & 1)) return -1;
    const int base = 1 << p->ks_base_bits, t = p->ks_t;
    rng_t r;
    rng_init(&r, seed, DOM_LWE_KEY << 56);
    for (int i = 0; i < n; i++) lwe_key[i] = rng_u32(&r) & 1u;
    rng_init(&r, seed, DOM_TRLWE_KEY << 56);
    for (int i = 0; i < k * N; i++) trlwe_key[i] = rng_u32(&r) & 1u;

    /* BK_i = TGSW(s_i): rows (q, pp) are TRLWE encryptions of zero plus
     * s_i * h_pp added to polynomial q (q = 0..k-1 masks, q = k body).
     * bk_unroll 2: per key pair (i, j) = (2m, 2m+1) three TGSWs, of the
     * messages s_i s_j, s_i (1 - s_j) and (1 - s_i) s_j. */
    const int rows = (k + 1) * l;
    const int unroll = bk_unroll(p);
    const int ntgsw = unroll == 2 ? (n / 2) * 3 : n;
    uint32_t *tmp = malloc(sizeof(uint32_t) * N);
    for (int g = 0; g < ntgsw; g++) {
        uint32_t msg;
        if (unroll == 2) {
            const uint32_t si = lwe_key[2 * (g / 3)], sj = lwe_key[2 * (g / 3) + 1];
            const int comp = g % 3;
            msg = comp == 0 ? (si & sj) : comp == 1 ? (si & (1u - sj)) : ((1u - si) & sj);
        } else {
            msg = lwe_key[g];
        }
        for (int row = 0; row < rows; row++) {
            uint32_t *trlwe = bk + ((size_t)g * rows + row) * (size_t)(k + 1) * N;
            const uint64_t nonce = unroll == 2
                ? (DOM_BK2 << 56) | ((uint64_t)(g / 3) << 16) | ((uint64_t)(g % 3) << 8) | (uint64_t)row
                : (DOM_BK << 56) | ((uint64_t)g << 16) | (uint64_t)row;
            rng_init(&r, seed, nonce);
            uint32_t *body = trlwe + (size_t)k * N;
            for (int q = 0; q < k; q++)
                for (int j = 0; j < N; j++) trlwe[(size_t)q * N + j] = rng_u32(&r);
            for (int j = 0; j < N; j++) body[j] = rng_gauss_torus(&r, p->bk_stdev);
            for (int q = 0; q < k; q++) {
                poly_mul_binary(N, trlwe + (size_t)q * N, trlwe_key + (size_t)q * N, tmp);
                for (int j = 0; j < N; j++) body[j] += tmp[j];
            }
            int q = row / l, pp = row % l;
            uint32_t h = 1u << (32 - (pp + 1) * p->bg_bits);
            trlwe[(size_t)q * N] += msg * h;
        }
    }
    free(tmp);

    /* KSK[i][j][v-1] = LWE_s(v * s'_i / base^(j+1)), s' = extracted TRLWE key */
    const int nin = k * N;
    for (int i = 0; i < nin; i++) {
        for (int j = 0; j < t; j++) {
            for (int v = 1; v < base; v++) {
                uint32_t *ct = ksk + (((size_t)i * t + j) * (base - 1) + (v - 1)) * (size_t)(n + 1);
                uint64_t item = ((uint64_t)i * t + j) * base + v;
                rng_init(&r, seed, (DOM_KSK << 56) | item);
                for (int a = 0; a < n; a++) ct[a] = rng_u32(&r);
                uint32_t msg = (trlwe_key[i] * (uint32_t)v) << (32 - (j + 1) * p->ks_base_bits);
                ct[n] = lwe_dot(ct, lwe_key, n) + rng_gauss_torus(&r, p->lwe_stdev) + msg;
            }
        }
    }
    return 0;
}

int or_encrypt(const or_params *p, const uint32_t *lwe_key, uint64_t seed, uint64_t stream,
               uint64_t first_index, const uint8_t *bits, size_t count, uint32_t *out) {
    const int n = p->n;
    for (size_t idx = 0; idx < count; idx++) {
        if (bits[idx] > 1) return -1;
        rng_t r;
        rng_init(&r, seed, (DOM_ENC << 56) | ((stream & 0xFFFFFull) << 32) | (first_index + (uint64_t)idx));
        uint32_t *ct = out + idx * (size_t)(n + 1);
        for (int a = 0; a < n; a++) ct[a] = rng_u32(&r);
        uint32_t mu = bits[idx] ? (1u << 29) : (0u - (1u << 29));
        ct[n] = lwe_dot(ct, lwe_key, n) + rng_gauss_torus(&r, p->lwe_stdev) + mu;
    }
    return 0;
}

void or_phase(const or_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
              int32_t *phase_out) {
    for (size_t i = 0; i < count; i++) {
        const uint32_t *ct = cts + i * (size_t)(p->n + 1);
        phase_out[i] = (int32_t)(ct[p->n] - lwe_dot(ct, lwe_key, p->n));
    }
}

void or_phase_big(const or_params *p, const uint32_t *trlwe_key, const uint32_t *cts,
                  size_t count, int32_t *phase_out) {
    int nb = p->k * p->N;
    for (size_t i = 0; i < count; i++) {
        const uint32_t *ct = cts + i * (size_t)(nb + 1);
        phase_out[i] = (int32_t)(ct[nb] - lwe_dot(ct, trlwe_key, nb));
    }
}

void or_decrypt(const or_params *p, const uint32_t *lwe_key, const uint32_t *cts, size_t count,
                uint8_t *bits_out) {
    for (size_t i = 0; i < count; i++) {
        int32_t ph;
        or_phase(p, lwe_key, cts + i * (size_t)(p->n + 1), 1, &ph);
        bits_out[i] = ph > 0 ? 1 : 0;
    }
}

/* ------------------------------------------------------------------------ */
/* bootstrapping context                                                     */
/* ------------------------------------------------------------------------ */

struct or_ctx {
    or_params p;
    ntt_plan pl;
    uint64_t *bk_ntt;   /* [n][rows][k+1][N]  (bk_unroll 2: [n/2][3][rows][k+1][N]) */
    uint64_t *psi2;     /* psi^u, u < 2N: X^e evaluates to psi2[e (2j+1) mod 2N] at NTT bin j */
    uint32_t *ksk;      /* [kN][t][base-1][n+1] */
};

or_ctx *or_ctx_create(const or_params *p, const uint32_t *bk, const uint32_t *ksk) {
    or_ctx *c = calloc(1, sizeof(or_ctx));
    c->p = *p;
    const int N = p->N, rows = (p->k + 1) * p->l, kp1 = p->k + 1;
    ntt_plan_init(&c->pl, N);
    c->psi2 = malloc(sizeof(uint64_t) * 2 * N);
    for (int u = 0; u < N; u++) {
        c->psi2[u] = c->pl.psi_pows[u];
        c->psi2[u + N] = GL_P - c->pl.psi_pows[u];  /* psi^N = -1 */
    }
    const size_t ntgsw = bk_unroll(p) == 2 ? (size_t)(p->n / 2) * 3 : (size_t)p->n;
    size_t npoly = ntgsw * rows * kp1;
    c->bk_ntt = malloc(sizeof(uint64_t) * npoly * N);
    int64_t *tmp = malloc(sizeof(int64_t) * N);
    for (size_t q = 0; q < npoly; q++) {
        for (int j = 0; j < N; j++) tmp[j] = (int32_t)bk[q * N + j];
        ntt_forward_i64(&c->pl, tmp, c->bk_ntt + q * N);
    }
    free(tmp);
    size_t ksk_words = (size_t)p->k * N * p->ks_t * ((1 << p->ks_base_bits) - 1) * (p->n + 1);
    c->ksk = malloc(sizeof(uint32_t) * ksk_words);
    memcpy(c->ksk, ksk, sizeof(uint32_t) * ksk_words);
    return c;
}

void or_ctx_destroy(or_ctx *c) {
    if (!c) return;
    ntt_plan_free(&c->pl);
    free(c->bk_ntt);
    free(c->psi2);
    free(c->ksk);
    free(c);
}

/* modSwitchFromTorus32(x, 2N): round(x * 2N / 2^32) mod 2N */
static inline uint32_t mod_switch(uint32_t x, int N) {
    int shift = 32 - 1;
    int logN2 = 0;
    while ((1 << logN2) < 2 * N) logN2++;
    shift = 32 - logN2;
    return ((x + (1u << (shift - 1))) >> shift) & (uint32_t)(2 * N - 1);
}

void or_modswitch(const or_ctx *c, const uint32_t *lwe, uint32_t *out) {
    for (int i = 0; i <= c->p.n; i++) out[i] = mod_switch(lwe[i], c->p.N);
}

/* gadget decomposition offset sum_q Bg/2 * 2^(32-(q+1)bg_bits) (tfhe tGswTorus32PolynomialDecompH) */
static inline uint32_t decomp_offset(int bg_bits, int l) {
    const uint32_t half = 1u << (bg_bits - 1);
    uint32_t offset = 0;
    for (int q = 0; q < l; q++) offset += half << (32 - (q + 1) * bg_bits);
    return offset;
}
/* gadget decomposition digit pp of x (buf = x + offset), in [-Bg/2, Bg/2) */
static inline int32_t decomp_digit(uint32_t buf, int pp, int bg_bits) {
    return (int32_t)((buf >> (32 - (pp + 1) * bg_bits)) & ((1u << bg_bits) - 1)) - (int32_t)(1u << (bg_bits - 1));
}

/* ACC <- ACC + BK_i [x] ((X^a - 1) ACC), exact (CGGI CMux step) */
static void cmux_step(const or_ctx *c, int i, int a, uint32_t *acc, uint32_t *rot,
                      int64_t *dig, uint64_t *dig_ntt, uint64_t *sum) {
    const int N = c->p.N, kp1 = c->p.k + 1, l = c->p.l, rows = kp1 * l;
    for (int q = 0; q < kp1; q++) {
        poly_mul_xai(N, a, acc + (size_t)q * N, rot + (size_t)q * N);
        for (int j = 0; j < N; j++) rot[(size_t)q * N + j] -= acc[(size_t)q * N + j];
    }
    memset(sum, 0, sizeof(uint64_t) * (size_t)kp1 * N);
    const uint32_t offset = decomp_offset(c->p.bg_bits, l);
    for (int row = 0; row < rows; row++) {
        int q = row / l, pp = row % l;
        for (int j = 0; j < N; j++) dig[j] = decomp_digit(rot[(size_t)q * N + j] + offset, pp, c->p.bg_bits);
        ntt_forward_i64(&c->pl, dig, dig_ntt);
        const uint64_t *bkrow = c->bk_ntt + (((size_t)i * rows + row) * kp1) * N;
        for (int o = 0; o < kp1; o++)
            for (int j = 0; j < N; j++)
                sum[(size_t)o * N + j] = gl_add(sum[(size_t)o * N + j], gl_mul(dig_ntt[j], bkrow[(size_t)o * N + j]));
    }
    for (int o = 0; o < kp1; o++) {
        ntt_inverse_torus(&c->pl, sum + (size_t)o * N, rot + (size_t)o * N);
        for (int j = 0; j < N; j++) acc[(size_t)o * N + j] += rot[(size_t)o * N + j];
    }
}

/* Key-pair CMux (bk_unroll 2): ACC <- ACC + BK_m [x] ACC with the combined
 * TGSW BK_m = (X^{a_i+a_j} - 1) BK_m,0 + (X^{a_i} - 1) BK_m,1 + (X^{a_j} - 1) BK_m,2,
 * whose message is X^{a_i s_i + a_j s_j} - 1, so ACC <- X^{a_i s_i + a_j s_j} ACC.
 * Exact: digits of ACC are NTT-transformed once, multiplied by each component
 * and by the NTT image of X^e - 1, summed in the field and lifted (the true
 * integer result is below 2^53 << p/2), then reduced mod 2^32. */
static void cmux_pair(const or_ctx *c, int m, const int e[3], uint32_t *acc, uint32_t *rot,
                      int64_t *dig, uint64_t *dig_ntt, uint64_t *sum) {
    const int N = c->p.N, kp1 = c->p.k + 1, l = c->p.l, rows = kp1 * l;
    if (e[0] == 0 && e[1] == 0 && e[2] == 0) return;
    const uint32_t offset = decomp_offset(c->p.bg_bits, l);
    for (int row = 0; row < rows; row++) {
        const int q = row / l, pp = row % l;
        for (int j = 0; j < N; j++) dig[j] = decomp_digit(acc[(size_t)q * N + j] + offset, pp, c->p.bg_bits);
        ntt_forward_i64(&c->pl, dig, dig_ntt + (size_t)row * N);
    }
    memset(sum, 0, sizeof(uint64_t) * (size_t)kp1 * N);
    for (int comp = 0; comp < 3; comp++) {
        if (e[comp] == 0) continue;  /* X^0 - 1 = 0 */
        const uint64_t *bk = c->bk_ntt + ((size_t)m * 3 + comp) * rows * kp1 * N;
        for (int o = 0; o < kp1; o++) {
            for (int j = 0; j < N; j++) {
                uint64_t t = 0;
                for (int row = 0; row < rows; row++)
                    t = gl_add(t, gl_mul(dig_ntt[(size_t)row * N + j], bk[((size_t)row * kp1 + o) * N + j]));
                const uint64_t f = gl_sub(c->psi2[((uint64_t)e[comp] * (2 * j + 1)) & (2 * N - 1)], 1);
                sum[(size_t)o * N + j] = gl_add(sum[(size_t)o * N + j], gl_mul(f, t));
            }
        }
    }
    for (int o = 0; o < kp1; o++) {
        ntt_inverse_torus(&c->pl, sum + (size_t)o * N, rot + (size_t)o * N);
        for (int j = 0; j < N; j++) acc[(size_t)o * N + j] += rot[(size_t)o * N + j];
    }
}

void or_blind_rotate(const or_ctx *c, const uint32_t *lwe, uint32_t mu, int32_t iters,
                     uint32_t *acc) {
    const int n = c->p.n, N = c->p.N, kp1 = c->p.k + 1, rows = kp1 * c->p.l;
    uint32_t *bar = malloc(sizeof(uint32_t) * (n + 1));
    or_modswitch(c, lwe, bar);
    /* ACC = X^{-barb} * (0, ..., 0, testvect), testvect = mu everywhere */
    memset(acc, 0, sizeof(uint32_t) * (size_t)kp1 * N);
    uint32_t *tv = malloc(sizeof(uint32_t) * N);
    for (int j = 0; j < N; j++) tv[j] = mu;
    int rotb = (2 * N - (int)bar[n]) & (2 * N - 1);
    poly_mul_xai(N, rotb, tv, acc + (size_t)c->p.k * N);
    uint32_t *rot = malloc(sizeof(uint32_t) * (size_t)kp1 * N);
    int64_t *dig = malloc(sizeof(int64_t) * N);
    uint64_t *dig_ntt = malloc(sizeof(uint64_t) * (size_t)rows * N);
    uint64_t *sum = malloc(sizeof(uint64_t) * (size_t)kp1 * N);
    if (iters < 0 || iters > n) iters = n;
    if (bk_unroll(&c->p) == 2) {
        for (int m = 0; m < iters / 2; m++) {
            const int ai = (int)bar[2 * m], aj = (int)bar[2 * m + 1];
            const int e[3] = {(ai + aj) & (2 * N - 1), ai, aj};
            cmux_pair(c, m, e, acc, rot, dig, dig_ntt, sum);
        }
    } else {
        for (int i = 0; i < iters; i++) {
            if (bar[i] == 0) continue;
            cmux_step(c, i, (int)bar[i], acc, rot, dig, dig_ntt, sum);
        }
    }
    free(bar); free(tv); free(rot); free(dig); free(dig_ntt); free(sum);
}

/* SampleExtract at index 0: a'_0 = A_0, a'_j = -A_{N-j}; b' = B_0 */
static void sample_extract(int N, int k, const uint32_t *acc, uint32_t *out) {
    for (int q = 0; q < k; q++) {
        const uint32_t *A = acc + (size_t)q * N;
        out[(size_t)q * N] = A[0];
        for (int j = 1; j < N; j++) out[(size_t)q * N + j] = 0u - A[N - j];
    }
    out[(size_t)k * N] = acc[(size_t)k * N];
}

/* SampleExtract at index j: a'_i = A_{j-i} (i <= j), -A_{N+j-i} (i > j); b' = B_j */
static void sample_extract_at(int N, int k, const uint32_t *acc, int j, uint32_t *out) {
    for (int q = 0; q < k; q++) {
        const uint32_t *A = acc + (size_t)q * N;
        for (int i = 0; i < N; i++) out[(size_t)q * N + i] = i <= j ? A[j - i] : 0u - A[N + j - i];
    }
    out[(size_t)k * N] = acc[(size_t)k * N + j];
}

void or_bootstrap_wo_ks(const or_ctx *c, const uint32_t *lwe, uint32_t mu, uint32_t *out) {
    const int N = c->p.N, kp1 = c->p.k + 1;
    uint32_t *acc = malloc(sizeof(uint32_t) * (size_t)kp1 * N);
    or_blind_rotate(c, lwe, mu, c->p.n, acc);
    sample_extract(N, c->p.k, acc, out);
    free(acc);
}

void or_keyswitch(const or_ctx *c, const uint32_t *in, uint32_t *out) {
    const int n = c->p.n, nin = c->p.k * c->p.N, t = c->p.ks_t, bb = c->p.ks_base_bits;
    const int base = 1 << bb;
    const uint32_t prec_offset = 1u << (32 - (1 + bb * t));
    memset(out, 0, sizeof(uint32_t) * n);
    out[n] = in[nin];
    for (int i = 0; i < nin; i++) {
        uint32_t abar = in[i] + prec_offset;
        for (int j = 0; j < t; j++) {
            uint32_t d = (abar >> (32 - (j + 1) * bb)) & (uint32_t)(base - 1);
            if (!d) continue;
            const uint32_t *row = c->ksk + (((size_t)i * t + j) * (base - 1) + (d - 1)) * (size_t)(n + 1);
            for (int a = 0; a <= n; a++) out[a] -= row[a];
        }
    }
}

static void lin_comb(int n, uint32_t c0, int32_t alpha, const uint32_t *A, int32_t beta,
                     const uint32_t *B, uint32_t *out) {
    for (int i = 0; i <= n; i++) {
        uint32_t v = (uint32_t)alpha * A[i];
        if (beta) v += (uint32_t)beta * B[i];
        out[i] = v;
    }
    out[n] += c0;
}

void or_gate(const or_ctx *c, uint32_t c0, int32_t alpha, const uint32_t *A, int32_t beta,
             const uint32_t *B, uint32_t *out) {
    const int n = c->p.n, nb = c->p.k * c->p.N;
    uint32_t *lin = malloc(sizeof(uint32_t) * (n + 1));
    uint32_t *big = malloc(sizeof(uint32_t) * (nb + 1));
    lin_comb(n, c0, alpha, A, beta, B, lin);
    or_bootstrap_wo_ks(c, lin, 1u << 29, big);
    or_keyswitch(c, big, out);
    free(lin); free(big);
}

/* 3-input threshold gate (hb_gate kind LIN3): majority with (0; 1, 1, 1),
 * 3-input XOR with (0; -2, -2, -2) — the phases +-1/8 sum to +-1/8 or +-3/8,
 * doubled to +-1/4 mod 1 with the sign carrying the parity. */
void or_gate3(const or_ctx *c, uint32_t c0, int32_t alpha, const uint32_t *A, int32_t beta,
              const uint32_t *B, int32_t gamma, const uint32_t *C, uint32_t *out) {
    const int n = c->p.n, nb = c->p.k * c->p.N;
    uint32_t *lin = malloc(sizeof(uint32_t) * (n + 1));
    uint32_t *big = malloc(sizeof(uint32_t) * (nb + 1));
    for (int i = 0; i <= n; i++)
        lin[i] = (uint32_t)alpha * A[i] + (uint32_t)beta * B[i] + (uint32_t)gamma * C[i];
    lin[n] += c0;
    or_bootstrap_wo_ks(c, lin, 1u << 29, big);
    or_keyswitch(c, big, out);
    free(lin); free(big);
}

/* Half adder from one blind rotation (hb_gate kind HA): psi = (0,c0) + alpha*A + beta*B
 * with c0 = -1/8 is the AND of the literals (alpha A, beta B).  The accumulator
 * X^{-psi} * (mu...mu) is extracted twice: at index 0 (S0 = +-1/8 by psi in
 * [0, 1/2): the AND) and at index N/2 (S1 = +-1/8 by psi in [-1/4, 1/4)).  Over the
 * three phases psi in {-3/8, -1/8, 1/8} of the literal sum, S1 - S0 - 1/8 is the XOR
 * of the literals; sigma = +-1 orients it:
 *   out_and = KS(S0),  out_xor = KS(sigma (S1 - S0) + (0, -sigma/8)). */
void or_half_adder(const or_ctx *c, uint32_t c0, int32_t alpha, const uint32_t *A, int32_t beta,
                   const uint32_t *B, int32_t sigma, uint32_t *out_and, uint32_t *out_xor) {
    const int n = c->p.n, N = c->p.N, kp1 = c->p.k + 1, nb = c->p.k * c->p.N;
    const uint32_t eighth = 1u << 29;
    uint32_t *lin = malloc(sizeof(uint32_t) * (n + 1));
    uint32_t *acc = malloc(sizeof(uint32_t) * (size_t)kp1 * N);
    uint32_t *s0 = malloc(sizeof(uint32_t) * (nb + 1));
    uint32_t *s1 = malloc(sizeof(uint32_t) * (nb + 1));
    lin_comb(n, c0, alpha, A, beta, B, lin);
    or_blind_rotate(c, lin, eighth, n, acc);
    sample_extract_at(N, c->p.k, acc, 0, s0);
    sample_extract_at(N, c->p.k, acc, N / 2, s1);
    or_keyswitch(c, s0, out_and);
    for (int i = 0; i <= nb; i++) s1[i] = sigma > 0 ? s1[i] - s0[i] : s0[i] - s1[i];
    s1[nb] += sigma > 0 ? 0u - eighth : eighth;
    or_keyswitch(c, s1, out_xor);
    free(lin); free(acc); free(s0); free(s1);
}

void or_mux(const or_ctx *c, const uint32_t *S, const uint32_t *A, const uint32_t *B,
            uint32_t *out) {
    const int n = c->p.n, nb = c->p.k * c->p.N;
    const uint32_t eighth = 1u << 29;
    uint32_t *lin = malloc(sizeof(uint32_t) * (n + 1));
    uint32_t *u1 = malloc(sizeof(uint32_t) * (nb + 1));
    uint32_t *u2 = malloc(sizeof(uint32_t) * (nb + 1));
    lin_comb(n, 0u - eighth, 1, S, 1, A, lin);
    or_bootstrap_wo_ks(c, lin, eighth, u1);
    lin_comb(n, 0u - eighth, -1, S, 1, B, lin);
    or_bootstrap_wo_ks(c, lin, eighth, u2);
    for (int i = 0; i <= nb; i++) u1[i] += u2[i];
    u1[nb] += eighth;
    or_keyswitch(c, u1, out);
    free(lin); free(u1); free(u2);
}

/* ------------------------------------------------------------------------ */
/* threaded batch (CPU baseline)                                             */
/* ------------------------------------------------------------------------ */

typedef struct {
    const or_ctx *c;
    const or_gate_rec *gates;
    size_t n, stride;
    uint32_t *pool;
    size_t next;
    pthread_mutex_t mu;
} batch_job;

static void run_one(const or_ctx *c, const or_gate_rec *g, uint32_t *pool, size_t stride) {
    uint32_t *dst = pool + (size_t)g->dst * stride;
    const uint32_t *A = pool + (size_t)g->src_a * stride;
    const uint32_t *B = pool + (size_t)g->src_b * stride;
    if (g->kind == 1) {
        /* MUX: S=src_a, A=src_b (selected when S=1), B=src_c; alpha/beta = signs of A/B */
        const int n = c->p.n, nb = c->p.k * c->p.N;
        const uint32_t eighth = 1u << 29;
        const uint32_t *C = pool + (size_t)g->src_c * stride;
        uint32_t lin[1024 + 1], u1[4096 + 1], u2[4096 + 1];
        lin_comb(n, 0u - eighth, 1, A, g->alpha, B, lin);
        or_bootstrap_wo_ks(c, lin, eighth, u1);
        lin_comb(n, 0u - eighth, -1, A, g->beta, C, lin);
        or_bootstrap_wo_ks(c, lin, eighth, u2);
        for (int i = 0; i <= nb; i++) u1[i] += u2[i];
        u1[nb] += eighth;
        or_keyswitch(c, u1, dst);
    } else if (g->kind == 2) {
        or_gate3(c, g->c0, g->alpha, A, g->beta, B, g->gamma, pool + (size_t)g->src_c * stride, dst);
    } else if (g->kind == 3) {
        /* HA: dst = AND of the literals, src_c = their XOR (gamma = orientation) */
        or_half_adder(c, g->c0, g->alpha, A, g->beta, B, g->gamma, dst, pool + (size_t)g->src_c * stride);
    } else {
        or_gate(c, g->c0, g->alpha, A, g->beta, g->beta ? B : NULL, dst);
    }
}

static void *batch_worker(void *arg) {
    batch_job *job = arg;
    for (;;) {
        pthread_mutex_lock(&job->mu);
        size_t i = job->next++;
        pthread_mutex_unlock(&job->mu);
        if (i >= job->n) break;
        run_one(job->c, &job->gates[i], job->pool, job->stride);
    }
    return NULL;
}

int or_run_gates(const or_ctx *c, const or_gate_rec *gates, size_t n, uint32_t *pool,
                 size_t pool_stride, int threads) {
    if (threads < 1) threads = 1;
    batch_job job = {c, gates, n, pool_stride, pool, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t *th = malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; i++) pthread_create(&th[i], NULL, batch_worker, &job);
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    free(th);
    return 0;
}
