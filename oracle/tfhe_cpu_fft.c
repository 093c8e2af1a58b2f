/*
 * TEST / BENCH INFRASTRUCTURE ONLY — vectorised FP64-FFT CPU implementation of
 * the same CGGI gate bootstrap as tfhe_oracle.c (key-pair blind rotation,
 * bk_unroll 2), used as the *fast* CPU baseline of bench.py (cpu_baseline and
 * --impl reference) and checked bit-for-bit against the exact-integer oracle
 * in tests/test_cpu_fft.py.  Never linked by the product path.
 *
 * The reference (/root/reference/pkg/src/hebnn/backend.py:116-150, gates at
 * 205-237) has no crypto to time; a CPU TFHE library runs this algorithm with
 * a double-precision FFT, which is what this file does (the exact Goldilocks
 * NTT of tfhe_oracle.c is ~20x slower by construction).
 *
 * Layout: eight gates advance in lockstep, one per SIMD lane (v8d = 8 doubles:
 * one AVX-512 register, or two AVX2 registers through GCC's vector
 * extensions).  Every butterfly, digit extraction and Fourier product is a
 * plain element-wise vector operation and every bootstrapping-key value is
 * loaded once per eight gates.  Negacyclic transform: the folded polynomial
 * z_j = (a_j + i a_{j+N/2}) psi^j, psi = e^{i pi / N}, goes through an in-place
 * radix-2 DIF complex FFT of N/2 points (output in bit-reversed order: bin
 * k = bitrev(p) at position p holds A(psi^{4k+1})); the inverse is the
 * matching DIT.  Products are exact after rounding because the true integer
 * result is below 2^53 (same argument as the GPU kernels).
 */
#include "tfhe_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define CF_N 1024
#define CF_M 512
#define CF_ROWS 6
#define CF_L 8 /* lanes */

typedef double v8d __attribute__((vector_size(64), aligned(64)));
typedef uint32_t v8u __attribute__((vector_size(32), aligned(32)));
typedef int32_t v8i __attribute__((vector_size(32), aligned(32)));
typedef long long v8q __attribute__((vector_size(64), aligned(64)));

#if defined(__x86_64__)
#define CF_CLONES __attribute__((target_clones("avx512f", "avx2,fma", "default")))
#else
#define CF_CLONES
#endif

typedef struct cf_ctx {
    or_params p;
    int pairs;
    double *bk;        /* [pair][pos p][comp 3][row 6][out 2][re, im]  (Fourier domain, bit-reversed bins) */
    double tw_re[CF_M], tw_im[CF_M];     /* stage h: e^{2 pi i j / 2h} at [h + j] */
    double ps_re[CF_M], ps_im[CF_M];     /* psi^j */
    double x_re[2 * CF_N], x_im[2 * CF_N]; /* psi^u, u < 2N */
    uint16_t k4p1[CF_M];                 /* 4 bitrev(p) + 1 */
    uint32_t *ksk;                       /* [N][t][base-1][n+1] */
} cf_ctx;

static int bitrev9(int x) {
    int r = 0;
    for (int b = 0; b < 9; b++) r |= ((x >> b) & 1) << (8 - b);
    return r;
}

/* scalar forward transform (context creation only) */
static void fft_fwd_scalar(const cf_ctx *c, double *re, double *im) {
    for (int h = CF_M / 2; h >= 1; h >>= 1)
        for (int s = 0; s < CF_M; s += 2 * h)
            for (int j = 0; j < h; j++) {
                const double ur = re[s + j], ui = im[s + j], vr = re[s + j + h], vi = im[s + j + h];
                const double dr = ur - vr, di = ui - vi, wr = c->tw_re[h + j], wi = c->tw_im[h + j];
                re[s + j] = ur + vr;
                im[s + j] = ui + vi;
                re[s + j + h] = dr * wr - di * wi;
                im[s + j + h] = dr * wi + di * wr;
            }
}

cf_ctx *cf_ctx_create(const or_params *p, const uint32_t *bk, const uint32_t *ksk) {
    if (p->N != CF_N || p->k != 1 || p->l != 3 || p->bk_unroll != 2 || (p->n & 1) || p->bg_bits * p->l > 32)
        return NULL;
    cf_ctx *c = aligned_alloc(64, (sizeof(cf_ctx) + 63) / 64 * 64);
    memset(c, 0, sizeof(*c));
    c->p = *p;
    c->pairs = p->n / 2;
    for (int h = 1; h < CF_M; h <<= 1)
        for (int j = 0; j < h; j++) {
            c->tw_re[h + j] = cos(M_PI * j / h);
            c->tw_im[h + j] = sin(M_PI * j / h);
        }
    for (int u = 0; u < 2 * CF_N; u++) {
        c->x_re[u] = cos(M_PI * u / CF_N);
        c->x_im[u] = sin(M_PI * u / CF_N);
    }
    for (int j = 0; j < CF_M; j++) {
        c->ps_re[j] = c->x_re[j];
        c->ps_im[j] = c->x_im[j];
        c->k4p1[j] = (uint16_t)(4 * bitrev9(j) + 1);
    }
    const size_t npoly = (size_t)c->pairs * 3 * CF_ROWS * 2;
    c->bk = aligned_alloc(64, sizeof(double) * npoly * CF_N);
    double re[CF_M], im[CF_M];
    for (size_t q = 0; q < npoly; q++) {
        const uint32_t *src = bk + q * CF_N;
        for (int j = 0; j < CF_M; j++) {
            const double a = (double)(int32_t)src[j], b = (double)(int32_t)src[j + CF_M];
            re[j] = a * c->ps_re[j] - b * c->ps_im[j];
            im[j] = a * c->ps_im[j] + b * c->ps_re[j];
        }
        fft_fwd_scalar(c, re, im);
        /* q = ((pair * 3 + comp) * 6 + row) * 2 + out */
        const size_t out = q & 1, row = (q >> 1) % CF_ROWS, comp = (q / (2 * CF_ROWS)) % 3, pair = q / (2 * CF_ROWS * 3);
        for (int pz = 0; pz < CF_M; pz++) {
            double *dst = c->bk + ((((pair * CF_M + pz) * 3 + comp) * CF_ROWS + row) * 2 + out) * 2;
            dst[0] = re[pz];
            dst[1] = im[pz];
        }
    }
    const size_t ksk_words = (size_t)CF_N * p->ks_t * ((1 << p->ks_base_bits) - 1) * (p->n + 1);
    c->ksk = malloc(sizeof(uint32_t) * ksk_words);
    memcpy(c->ksk, ksk, sizeof(uint32_t) * ksk_words);
    return c;
}

void cf_ctx_destroy(cf_ctx *c) {
    if (!c) return;
    free(c->bk);
    free(c->ksk);
    free(c);
}

/* per-thread scratch of one 8-gate block */
typedef struct {
    v8d dre[CF_ROWS][CF_M], dim[CF_ROWS][CF_M];   /* digit spectra */
    v8d sre[2][CF_M], sim[2][CF_M];               /* output spectra */
    v8d fre[3][CF_M], fim[3][CF_M];               /* X^{e_c} - 1 at the bins */
    v8u acc[2][CF_N];                             /* TRLWE accumulators, lane = gate */
    uint32_t lin[CF_L][CF_N];                     /* gate inputs; later the extracted LWE a-part */
    uint16_t bar[CF_L][CF_N];                     /* mod-switched coefficients */
    uint32_t big_b[CF_L];
} cf_work;

static inline __attribute__((always_inline)) void fwd_stage(const cf_ctx *c, v8d *re, v8d *im, int base, int len, int h) {
    for (int s = base; s < base + len; s += 2 * h)
        for (int j = 0; j < h; j++) {
            const v8d ur = re[s + j], ui = im[s + j], vr = re[s + j + h], vi = im[s + j + h];
            const v8d dr = ur - vr, di = ui - vi;
            const double wr = c->tw_re[h + j], wi = c->tw_im[h + j];
            re[s + j] = ur + vr;
            im[s + j] = ui + vi;
            re[s + j + h] = dr * wr - di * wi;
            im[s + j + h] = dr * wi + di * wr;
        }
}
static inline __attribute__((always_inline)) void inv_stage(const cf_ctx *c, v8d *re, v8d *im, int base, int len, int h) {
    for (int s = base; s < base + len; s += 2 * h)
        for (int j = 0; j < h; j++) {
            const double wr = c->tw_re[h + j], wi = c->tw_im[h + j];
            const v8d ur = re[s + j], ui = im[s + j], xr = re[s + j + h], xi = im[s + j + h];
            const v8d vr = xr * wr + xi * wi, vi = xi * wr - xr * wi;  /* x * conj(w) */
            re[s + j] = ur + vr;
            im[s + j] = ui + vi;
            re[s + j + h] = ur - vr;
            im[s + j + h] = ui - vi;
        }
}
/* the two widest stages sweep the whole array, the rest runs in 64-point blocks that stay in L1 */
#define CF_BLK 64
static inline __attribute__((always_inline)) void fft_fwd(const cf_ctx *c, v8d *re, v8d *im) {
    for (int h = CF_M / 2; h >= CF_BLK; h >>= 1) fwd_stage(c, re, im, 0, CF_M, h);
    for (int b = 0; b < CF_M; b += CF_BLK)
        for (int h = CF_BLK / 2; h >= 1; h >>= 1) fwd_stage(c, re, im, b, CF_BLK, h);
}
static inline __attribute__((always_inline)) void fft_inv(const cf_ctx *c, v8d *re, v8d *im) {
    for (int b = 0; b < CF_M; b += CF_BLK)
        for (int h = 1; h < CF_BLK; h <<= 1) inv_stage(c, re, im, b, CF_BLK, h);
    for (int h = CF_BLK; h < CF_M; h <<= 1) inv_stage(c, re, im, 0, CF_M, h);
}

/* one key pair for the 8 gates of the block: ACC <- ACC + BK_m [x] ACC */
CF_CLONES
static void cf_pair(const cf_ctx *c, cf_work *w, int m) {
    const int bgb = c->p.bg_bits;
    uint32_t offset = 0;
    for (int q = 0; q < 3; q++) offset += (1u << (bgb - 1)) << (32 - (q + 1) * bgb);
    const uint32_t mask = (1u << bgb) - 1;
    const int32_t halfbg = 1 << (bgb - 1);
    /* digits -> folded, twisted, transformed */
    for (int row = 0; row < CF_ROWS; row++) {
        const int q = row / 3, sh = 32 - (row % 3 + 1) * bgb;
        v8d *re = w->dre[row], *im = w->dim[row];
        for (int j = 0; j < CF_M; j++) {
            const v8i lo = (v8i)(((w->acc[q][j] + offset) >> sh) & mask) - halfbg;
            const v8i hi = (v8i)(((w->acc[q][j + CF_M] + offset) >> sh) & mask) - halfbg;
            const v8d a = __builtin_convertvector(lo, v8d), b = __builtin_convertvector(hi, v8d);
            const double pr = c->ps_re[j], pi = c->ps_im[j];
            re[j] = a * pr - b * pi;
            im[j] = a * pi + b * pr;
        }
        fft_fwd(c, re, im);
    }
    /* F_c = psi^{e_c (4k+1)} - 1 per lane (table gathers, lanes innermost) */
    {
        uint32_t e[3][CF_L];
        for (int lane = 0; lane < CF_L; lane++) {
            const uint32_t ai = w->bar[lane][2 * m], aj = w->bar[lane][2 * m + 1];
            e[0][lane] = (ai + aj) & (2 * CF_N - 1);
            e[1][lane] = ai;
            e[2][lane] = aj;
        }
        for (int comp = 0; comp < 3; comp++) {
            double *fr = (double *)w->fre[comp], *fi = (double *)w->fim[comp];
            for (int pz = 0; pz < CF_M; pz++) {
                const uint32_t k = c->k4p1[pz];
                for (int lane = 0; lane < CF_L; lane++) {
                    const uint32_t u = (e[comp][lane] * k) & (2 * CF_N - 1);
                    fr[pz * CF_L + lane] = c->x_re[u] - 1.0;
                    fi[pz * CF_L + lane] = c->x_im[u];
                }
            }
        }
    }
    /* out_o = sum_c F_c * (sum_row dig_row * BK_{c,row,o}) */
    const double *bk = c->bk + (size_t)m * CF_M * 3 * CF_ROWS * 2 * 2;
    for (int pz = 0; pz < CF_M; pz++, bk += 3 * CF_ROWS * 2 * 2) {
        v8d xr[CF_ROWS], xi[CF_ROWS];
        for (int row = 0; row < CF_ROWS; row++) {
            xr[row] = w->dre[row][pz];
            xi[row] = w->dim[row][pz];
        }
        v8d s0r = {0}, s0i = {0}, s1r = {0}, s1i = {0};
        for (int comp = 0; comp < 3; comp++) {
            const double *b = bk + comp * CF_ROWS * 4;
            v8d t0r = {0}, t0i = {0}, t1r = {0}, t1i = {0};
            for (int row = 0; row < CF_ROWS; row++, b += 4) {
                t0r += xr[row] * b[0] - xi[row] * b[1];
                t0i += xr[row] * b[1] + xi[row] * b[0];
                t1r += xr[row] * b[2] - xi[row] * b[3];
                t1i += xr[row] * b[3] + xi[row] * b[2];
            }
            const v8d fr = w->fre[comp][pz], fi = w->fim[comp][pz];
            s0r += fr * t0r - fi * t0i;
            s0i += fr * t0i + fi * t0r;
            s1r += fr * t1r - fi * t1i;
            s1i += fr * t1i + fi * t1r;
        }
        w->sre[0][pz] = s0r;
        w->sim[0][pz] = s0i;
        w->sre[1][pz] = s1r;
        w->sim[1][pz] = s1i;
    }
    /* inverse, untwist, exact rounding, accumulate */
    const v8d magic = {6755399441055744.0, 6755399441055744.0, 6755399441055744.0, 6755399441055744.0,
                       6755399441055744.0, 6755399441055744.0, 6755399441055744.0, 6755399441055744.0};
    const double scale = 1.0 / CF_M;
    for (int o = 0; o < 2; o++) {
        v8d *re = w->sre[o], *im = w->sim[o];
        fft_inv(c, re, im);
        for (int j = 0; j < CF_M; j++) {
            const double pr = c->ps_re[j] * scale, pi = c->ps_im[j] * scale;
            const v8d lo = re[j] * pr + im[j] * pi;   /* Re(z conj(psi^j)) / M */
            const v8d hi = im[j] * pr - re[j] * pi;
            const v8q ql = (v8q)(lo + magic), qh = (v8q)(hi + magic);
            w->acc[o][j] += __builtin_convertvector(ql, v8u);
            w->acc[o][j + CF_M] += __builtin_convertvector(qh, v8u);
        }
    }
}

/* key switch of the block's extracted samples; lane-by-lane row subtractions */
CF_CLONES
static void cf_keyswitch(const cf_ctx *c, const uint32_t *big_a, uint32_t big_b, uint32_t *out) {
    const int n = c->p.n, t = c->p.ks_t, bb = c->p.ks_base_bits, base = 1 << bb;
    const uint32_t prec_offset = 1u << (32 - (1 + bb * t));
    memset(out, 0, sizeof(uint32_t) * n);
    out[n] = big_b;
    for (int i = 0; i < CF_N; i++) {
        const uint32_t abar = big_a[i] + prec_offset;
        for (int j = 0; j < t; j++) {
            const uint32_t d = (abar >> (32 - (j + 1) * bb)) & (uint32_t)(base - 1);
            if (!d) continue;
            const uint32_t *row = c->ksk + (((size_t)i * t + j) * (base - 1) + (d - 1)) * (size_t)(n + 1);
            for (int a = 0; a <= n; a++) out[a] -= row[a];
        }
    }
}

static void cf_block(const cf_ctx *c, cf_work *w, const or_gate_rec *gates, size_t count, uint32_t *pool, size_t stride) {
    const int n = c->p.n;
    const uint32_t mu = 1u << 29;
    uint32_t barb[CF_L];
    for (int lane = 0; lane < CF_L; lane++) {
        const or_gate_rec *g = &gates[(size_t)lane < count ? (size_t)lane : 0];
        const uint32_t *A = pool + (size_t)g->src_a * stride, *B = pool + (size_t)g->src_b * stride;
        const uint32_t *C = pool + (size_t)g->src_c * stride;
        for (int i = 0; i <= n; i++) {
            uint32_t v = (uint32_t)g->alpha * A[i];
            if (g->beta) v += (uint32_t)g->beta * B[i];
            if (g->kind == 2) v += (uint32_t)g->gamma * C[i];
            if (i == n) v += g->c0;
            /* modSwitchFromTorus32(x, 2N) */
            const uint32_t ms = ((v + (1u << 20)) >> 21) & (2 * CF_N - 1);
            if (i < n) w->bar[lane][i] = (uint16_t)ms; else barb[lane] = ms;
        }
    }
    /* ACC = X^{-barb} (0, mu ... mu) */
    for (int j = 0; j < CF_N; j++) {
        uint32_t v[CF_L];
        for (int lane = 0; lane < CF_L; lane++) v[lane] = ((j + (int)barb[lane]) & CF_N) ? 0u - mu : mu;
        memset(&w->acc[0][j], 0, sizeof(v8u));
        memcpy(&w->acc[1][j], v, sizeof(v8u));
    }
    for (int m = 0; m < c->pairs; m++) cf_pair(c, w, m);
    /* sample extraction at 0 and key switch, lane by lane */
    for (int lane = 0; lane < CF_L && (size_t)lane < count; lane++) {
        uint32_t *a = w->lin[lane];
        const uint32_t *A0 = (const uint32_t *)w->acc[0], *B0 = (const uint32_t *)w->acc[1];
        a[0] = A0[lane];
        for (int j = 1; j < CF_N; j++) a[j] = 0u - A0[(size_t)(CF_N - j) * CF_L + lane];
        cf_keyswitch(c, a, B0[lane], pool + (size_t)gates[lane].dst * stride);
    }
}

typedef struct {
    const cf_ctx *c;
    const or_gate_rec *gates;
    size_t n, stride;
    uint32_t *pool;
    size_t next;
    pthread_mutex_t mu;
} cf_job;

static void *cf_worker(void *arg) {
    cf_job *job = arg;
    cf_work *w = aligned_alloc(64, (sizeof(cf_work) + 63) / 64 * 64);
    for (;;) {
        pthread_mutex_lock(&job->mu);
        const size_t i = job->next;
        job->next += CF_L;
        pthread_mutex_unlock(&job->mu);
        if (i >= job->n) break;
        const size_t count = job->n - i < CF_L ? job->n - i : CF_L;
        cf_block(job->c, w, job->gates + i, count, job->pool, job->stride);
    }
    free(w);
    return NULL;
}

/* Independent gates of kinds LIN2 (0) and LIN3 (2), eight per SIMD block; -1 on other kinds. */
int cf_run_gates(const cf_ctx *c, const or_gate_rec *gates, size_t n, uint32_t *pool, size_t pool_stride,
                 int threads) {
    for (size_t i = 0; i < n; i++)
        if (gates[i].kind != 0 && gates[i].kind != 2) return -1;
    if (threads < 1) threads = 1;
    cf_job job = {c, gates, n, pool_stride, pool, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t *th = malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; i++) pthread_create(&th[i], NULL, cf_worker, &job);
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    free(th);
    return 0;
}
