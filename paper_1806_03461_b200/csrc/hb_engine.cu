// B200 (sm_100a) gate-bootstrapping engine: the device half of the
// GateBackend drop-in (reference: /root/reference/pkg/src/hebnn/backend.py
// 205-237, where SimContext only simulates each gate in plaintext).
//
// Kernels:
//   k_bk_to_fourier        K6  BK (u32 coefficients) -> FP64 negacyclic Fourier domain
//   k_blind_rotate_u2      K1+K2+K3 fused, key-pair bootstrapping key (default):
//                          gate linear combination (2 or 3 inputs) + mod switch,
//                          315 external products with the combined TGSW
//                          sum_c (X^e_c - 1) BK_c (gadget decomposition, FP64 FFT in
//                          registers/shared memory, BK stages streamed by
//                          cp.async.bulk into a shared-memory ring and reused by
//                          every gate of the CTA), sample extraction
//   k_blind_rotate_u2_lat  the same for narrow levels: one bootstrap per CTA
//   k_blind_rotate_u2_clu  the same for very narrow levels: one bootstrap per 2-CTA cluster
//   k_blind_rotate[_lat]   CGGI bootstrapping key (bk_unroll 1): 630 CMux steps
//   k_keyswitch            K4  batched LWE key switch (uint32), KSK table chunks
//                          shared by a tile of gates
//   k_gather               pool slots -> contiguous buffer for download
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hb_internal.h"

using namespace hb;

#define HB_CUDA_TRY(expr)                                                                   \
    do {                                                                                    \
        cudaError_t _err = (expr);                                                          \
        if (_err != cudaSuccess) {                                                          \
            set_error(std::string(#expr) + ": " + cudaGetErrorString(_err));               \
            return HB_ECUDA;                                                                \
        }                                                                                   \
    } while (0)

namespace {

// ---------------------------------------------------------------------------
// FP64 negacyclic FFT: 512-point complex transform of the folded polynomial
// z_j = (a_j + i a_{j+512}) psi^j, psi = e^{i pi / 1024}; Z_k = A(psi^{4k+1}).
// 64 threads per polynomial, 8 points per thread, three radix-8 passes with two
// shared-memory exchanges.  Thread t holds points t + 64 m (m = 0..7) on input
// and bins t + 64 m on output (natural order on both sides).
// ---------------------------------------------------------------------------

constexpr int kXchStride = 520;  // double2 per exchange buffer (65-padded layout)
#ifndef HB_EXP_SKIP
// timing experiments only (results wrong): 1 skip fwd FFT, 2 skip MAC, 4 skip inverse FFT,
// 8 skip rotation, 16 skip ACC update, 32/64 replace the 2nd/1st FFT barrier by __syncwarp
#define HB_EXP_SKIP 0
#endif

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// acc += a * b
__device__ __forceinline__ void cmac(double2 &acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}

// In-place DFT-8 with kernel e^{+2 pi i / 8}; output in bit-reversed order.
__device__ __forceinline__ void dft8(double2 (&x)[8]) {
    const double r = 0.70710678118654752440;
#pragma unroll
    for (int m = 0; m < 4; m++) {
        double2 a = x[m], b = x[m + 4];
        x[m] = cadd(a, b);
        double2 d = csub(a, b);
        if (m == 0) x[m + 4] = d;
        else if (m == 1) x[m + 4] = make_double2((d.x - d.y) * r, (d.x + d.y) * r);
        else if (m == 2) x[m + 4] = make_double2(-d.y, d.x);
        else x[m + 4] = make_double2((-d.x - d.y) * r, (d.x - d.y) * r);
    }
#pragma unroll
    for (int h = 0; h < 8; h += 4) {
#pragma unroll
        for (int m = 0; m < 2; m++) {
            double2 a = x[h + m], b = x[h + m + 2];
            x[h + m] = cadd(a, b);
            double2 d = csub(a, b);
            x[h + m + 2] = (m == 0) ? d : make_double2(-d.y, d.x);
        }
    }
#pragma unroll
    for (int h = 0; h < 8; h += 2) {
        double2 a = x[h], b = x[h + 1];
        x[h] = cadd(a, b);
        x[h + 1] = csub(a, b);
    }
}

__device__ __forceinline__ constexpr int rev3(int k) { return ((k & 1) << 2) | (k & 2) | ((k >> 2) & 1); }

__device__ __forceinline__ void group_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(64) : "memory");
}

// Forward 512-point FFT (kernel e^{+2 pi i jk/512}) of x held as described
// above.  W[e] = e^{2 pi i e / 512}.  S0/S1: two exchange buffers (double
// buffered so each exchange costs one barrier).
__device__ __forceinline__ void fft512(double2 (&x)[8], double2 *S0, double2 *S1, int t,
                                       const double2 *__restrict__ W, int bar_id) {
    // pass A: DFT over m (stride-64 points); thread t = j0 + 8 j1
    dft8(x);
    {
        const int j0 = t & 7, j1 = t >> 3;
#pragma unroll
        for (int k2 = 0; k2 < 8; k2++) {
            double2 y = x[rev3(k2)];
            if (k2) y = cmul(y, __ldg(&W[(t * k2) & 511]));
            S0[j0 * 65 + k2 * 8 + j1] = y;
        }
    }
    group_bar(bar_id);
    // pass B: thread u = j0 + 8 k2 gathers j1 = 0..7
    {
        const int j0 = t & 7, k2 = t >> 3;
#pragma unroll
        for (int j1 = 0; j1 < 8; j1++) x[j1] = S0[j0 * 65 + k2 * 8 + j1];
        dft8(x);
#pragma unroll
        for (int k1 = 0; k1 < 8; k1++) {
            double2 y = x[rev3(k1)];
            if (k1) y = cmul(y, __ldg(&W[(8 * j0 * k1) & 511]));
            S1[k2 * 65 + k1 * 8 + j0] = y;
        }
    }
    group_bar(bar_id);
    // pass C: thread v = k2 + 8 k1 gathers j0 = 0..7; output bin v + 64 k0
    {
        const int k2 = t & 7, k1 = t >> 3;
        double2 y[8];
#pragma unroll
        for (int j0 = 0; j0 < 8; j0++) y[j0] = S1[k2 * 65 + k1 * 8 + j0];
        dft8(y);
#pragma unroll
        for (int k0 = 0; k0 < 8; k0++) x[k0] = y[rev3(k0)];
    }
}

// c_m = psi^{64 m} = e^{i pi m / 16}, m = 0..7 (compile-time constants)
__device__ __forceinline__ double2 c16(int m) {
    constexpr double c1 = 0.98078528040323044913, s1 = 0.19509032201612826785;
    constexpr double c2 = 0.92387953251128675613, s2 = 0.38268343236508977173;
    constexpr double c3 = 0.83146961230254523708, s3 = 0.55557023301960222474;
    constexpr double r = 0.70710678118654752440;
    switch (m) {
        case 0: return make_double2(1.0, 0.0);
        case 1: return make_double2(c1, s1);
        case 2: return make_double2(c2, s2);
        case 3: return make_double2(c3, s3);
        case 4: return make_double2(r, r);
        case 5: return make_double2(s3, c3);
        case 6: return make_double2(s2, c2);
        default: return make_double2(s1, c1);
    }
}

// Per-thread twiddle seeds of the table-free transforms (thread t of a group):
//   f_a0 = psi^t, step_a = psi^{4t} = W^t, step_b = W64^{t&7} = psi^{32 (t&7)},
//   i_b0 = psi^{t>>3}, i_stepb = psi^{32 (t&7) + 8}
struct TwSeeds {
    double2 f_a0, step_a, step_b, i_b0, i_stepb;
};

// T[k] = T0 * step^k, k = 0..7, as a depth-4 product tree (shorter dependency
// chain and smaller rounding error than the serial recurrence).
__device__ __forceinline__ void tw_powers(double2 T0, double2 step, bool t0_is_one, double2 (&T)[8]) {
    const double2 s2 = cmul(step, step);
    const double2 s4 = cmul(s2, s2);
    if (t0_is_one) {
        T[0] = make_double2(1.0, 0.0);
        T[1] = step;
        T[2] = s2;
        T[3] = cmul(step, s2);
    } else {
        T[0] = T0;
        T[1] = cmul(T0, step);
        T[2] = cmul(T0, s2);
        T[3] = cmul(T[1], s2);
    }
    T[4] = t0_is_one ? s4 : cmul(T0, s4);
    T[5] = cmul(T[1], s4);
    T[6] = cmul(T[2], s4);
    T[7] = cmul(T[3], s4);
}

// NP-polynomial variants: the passes of NP independent transforms are
// interleaved (ILP for the FP64 pipe), share one twiddle recurrence and one
// barrier per exchange.  xch: [NP][2][kXchStride] (double-buffered exchanges).
// kSB (single buffer): xch is [NP][kXchStride]; both exchanges share one
// buffer, at the price of two more barriers (one before the first store, one
// between the second exchange's loads and stores).
template <int NP, bool kSB = false>
__device__ __forceinline__ void nega_fft_fwd_n(double2 (&x)[NP][8], double2 *xch, int t, const TwSeeds &tw,
                                               int bar_id) {
    constexpr int kB0 = kSB ? 1 : 2, kB1 = kSB ? 0 : 1;  // buffer q of exchange 1 / 2: q * kB0 + kB1 * (..)
#pragma unroll
    for (int q = 0; q < NP; q++) {
#pragma unroll
        for (int m = 1; m < 8; m++) x[q][m] = cmul(x[q][m], c16(m));
        dft8(x[q]);
    }
    if (kSB) group_bar(bar_id);  // previous transform's readers are done
    {
        const int j0 = t & 7, j1 = t >> 3;
        double2 T[8];
        tw_powers(tw.f_a0, tw.step_a, false, T);
#pragma unroll
        for (int k2 = 0; k2 < 8; k2++) {
#pragma unroll
            for (int q = 0; q < NP; q++) xch[(kB0 * q) * kXchStride + j0 * 65 + k2 * 8 + j1] = cmul(x[q][rev3(k2)], T[k2]);
        }
    }
    if (HB_EXP_SKIP & 64) __syncwarp(); else group_bar(bar_id);
    {
        const int j0 = t & 7, k2 = t >> 3;
#pragma unroll
        for (int q = 0; q < NP; q++) {
#pragma unroll
            for (int j1 = 0; j1 < 8; j1++) x[q][j1] = xch[(kB0 * q) * kXchStride + j0 * 65 + k2 * 8 + j1];
            dft8(x[q]);
            if (!kSB) xch[(kB0 * q + kB1) * kXchStride + k2 * 65 + j0] = x[q][0];
        }
        if (kSB) {
            group_bar(bar_id);
#pragma unroll
            for (int q = 0; q < NP; q++) xch[(kB0 * q + kB1) * kXchStride + k2 * 65 + j0] = x[q][0];
        }
        double2 T[8];
        tw_powers(tw.step_b, tw.step_b, true, T);
#pragma unroll
        for (int k1 = 1; k1 < 8; k1++) {
#pragma unroll
            for (int q = 0; q < NP; q++)
                xch[(kB0 * q + kB1) * kXchStride + k2 * 65 + k1 * 8 + j0] = cmul(x[q][rev3(k1)], T[k1]);
        }
    }
    if (HB_EXP_SKIP & 32) __syncwarp(); else group_bar(bar_id);
    {
        const int k2 = t & 7, k1 = t >> 3;
#pragma unroll
        for (int q = 0; q < NP; q++) {
            double2 y[8];
#pragma unroll
            for (int j0 = 0; j0 < 8; j0++) y[j0] = xch[(kB0 * q + kB1) * kXchStride + k2 * 65 + k1 * 8 + j0];
            dft8(y);
#pragma unroll
            for (int k0 = 0; k0 < 8; k0++) x[q][k0] = y[rev3(k0)];
        }
    }
}

template <int NP, bool kSB = false>
__device__ __forceinline__ void nega_fft_inv_n(double2 (&x)[NP][8], double2 *xch, int t, const TwSeeds &tw,
                                               int bar_id) {
    constexpr int kB0 = kSB ? 1 : 2, kB1 = kSB ? 0 : 1;
#pragma unroll
    for (int q = 0; q < NP; q++) {
#pragma unroll
        for (int m = 0; m < 8; m++) x[q][m].y = -x[q][m].y;
        dft8(x[q]);
    }
    if (kSB) group_bar(bar_id);
    {
        const int j0 = t & 7, j1 = t >> 3;
#pragma unroll
        for (int q = 0; q < NP; q++) xch[(kB0 * q) * kXchStride + j0 * 65 + j1] = x[q][0];
        double2 T[8];
        tw_powers(tw.step_a, tw.step_a, true, T);
#pragma unroll
        for (int k2 = 1; k2 < 8; k2++) {
#pragma unroll
            for (int q = 0; q < NP; q++) xch[(kB0 * q) * kXchStride + j0 * 65 + k2 * 8 + j1] = cmul(x[q][rev3(k2)], T[k2]);
        }
    }
    if (HB_EXP_SKIP & 64) __syncwarp(); else group_bar(bar_id);
    {
        const int j0 = t & 7, k2 = t >> 3;
#pragma unroll
        for (int q = 0; q < NP; q++) {
#pragma unroll
            for (int j1 = 0; j1 < 8; j1++) x[q][j1] = xch[(kB0 * q) * kXchStride + j0 * 65 + k2 * 8 + j1];
            dft8(x[q]);
        }
        if (kSB) group_bar(bar_id);
        double2 T[8];
        tw_powers(tw.i_b0, tw.i_stepb, false, T);
#pragma unroll
        for (int k1 = 0; k1 < 8; k1++) {
#pragma unroll
            for (int q = 0; q < NP; q++)
                xch[(kB0 * q + kB1) * kXchStride + k2 * 65 + k1 * 8 + j0] = cmul(x[q][rev3(k1)], T[k1]);
        }
    }
    if (HB_EXP_SKIP & 32) __syncwarp(); else group_bar(bar_id);
    {
        const int k2 = t & 7, k1 = t >> 3;
#pragma unroll
        for (int q = 0; q < NP; q++) {
            double2 y[8];
#pragma unroll
            for (int j0 = 0; j0 < 8; j0++) y[j0] = xch[(kB0 * q + kB1) * kXchStride + k2 * 65 + k1 * 8 + j0];
            dft8(y);
#pragma unroll
            for (int k0 = 0; k0 < 8; k0++) {
                double2 v = (k0 == 0) ? y[0] : cmul(y[rev3(k0)], c16(k0));
                x[q][k0] = make_double2(v.x, -v.y);
            }
        }
    }
}

#ifndef HB_I2F
#define HB_I2F 0
#endif
// double from a small signed integer: magic-number DADD (default) or I2F.F64
__device__ __forceinline__ double small_int_to_double(int32_t d) {
#if HB_I2F
    return (double)d;
#else
    // (2^52 + 2^51 + 2^31 + d) - (2^52 + 2^51 + 2^31)
    return __hiloint2double(0x43380000, (int)((uint32_t)d ^ 0x80000000u)) - 6755401588539392.0;
#endif
}
// round(v) mod 2^32 for |v| < 2^51 via the 1.5 * 2^52 magic constant
__device__ __forceinline__ uint32_t round_to_torus(double v) {
    return (uint32_t)__double2loint(v + 6755399441055744.0);
}

// gadget digit p (0..2) of the CGGI decomposition, in [-64, 64)
__device__ __forceinline__ int32_t gadget_digit(uint32_t x, int p) {
    constexpr uint32_t kOffset = (64u << 25) + (64u << 18) + (64u << 11);
    const uint32_t buf = x + kOffset;
    return (int32_t)((buf >> (25 - 7 * p)) & 127u) - 64;
}

// X^a rotation lookup: coefficient i of X^a * P (a in [0, 2N))
__device__ __forceinline__ uint32_t rot_coef(const uint32_t *P, int i, int a) {
    const int idx = (i - a) & (2 * kN - 1);
    const uint32_t v = P[idx & (kN - 1)];
    return (idx & kN) ? 0u - v : v;
}

// ---------------------------------------------------------------------------
// mbarrier / bulk-copy helpers (sm_90+ PTX; SASS: SYNCS.*, UBLKCP)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ---------------------------------------------------------------------------
// K6: BK to Fourier.  One 64-thread group per polynomial; output scaled by
// 1/512 (the inverse-FFT normalisation, exact power of two) in natural bin
// order: bkf[poly][k], poly = ((i * 6 + row) * 2 + q).
// ---------------------------------------------------------------------------
// bk_unroll 2 (key pairs): input poly ((g * 6 + row) * 2 + o) with g = 3 m + comp
// is stored at stage-major position ((((m * 3 + row / 2) * 3 + comp) * 2 + row % 2) * 2 + o),
// the order in which k_blind_rotate_u2 consumes (row pair, component, row) stages.
__global__ void __launch_bounds__(128) k_bk_to_fourier(const uint32_t *__restrict__ bk, double2 *__restrict__ bkf,
                                                      int npoly, const double2 *__restrict__ W,
                                                      const double2 *__restrict__ TW, int unroll) {
    __shared__ double2 xch[2][2][kXchStride];
    const int grp = threadIdx.x >> 6, t = threadIdx.x & 63;
    const int poly = blockIdx.x * 2 + grp;
    const bool active = poly < npoly;
    const uint32_t *src = bk + (size_t)(active ? poly : 0) * kN;
    double2 x[8];
#pragma unroll
    for (int m = 0; m < 8; m++) {
        const int j = t + 64 * m;
        const double lo = (double)(int32_t)src[j], hi = (double)(int32_t)src[j + kNH];
        x[m] = cmul(make_double2(lo, hi), TW[j]);
    }
    fft512(x, xch[grp][0], xch[grp][1], t, W, 1 + grp);
    if (active) {
        size_t dst = (size_t)poly;
        if (unroll == 2) {
            const int o = poly & 1, row = (poly >> 1) % kRows, g = (poly >> 1) / kRows;
            const int m = g / 3, comp = g % 3;
            dst = ((((size_t)m * 3 + row / 2) * 3 + comp) * 2 + (row & 1)) * 2 + o;
        }
#pragma unroll
        for (int m = 0; m < 8; m++)
            bkf[dst * kNH + t + 64 * m] = make_double2(x[m].x * (1.0 / 512), x[m].y * (1.0 / 512));
    }
}

// ---------------------------------------------------------------------------
// K1+K2+K3: fused gate prologue, blind rotation and sample extraction.
// ---------------------------------------------------------------------------
struct BrArgs {
    const uint32_t *pool;     // [slots * lanes][pool_stride]
    uint32_t pool_stride;
    uint32_t lanes;
    const BrItem *items;      // [n_items]
    uint32_t n_work;          // n_items * lanes
    int32_t n;                // LWE dimension
    uint32_t mu;              // test-vector value (1/8)
    const double2 *bkf;       // [n][6][2][512]
    uint32_t *big;            // [n_work][kBigStride] extracted LWE
    const double2 *W;         // [512] e^{2 pi i e/512}
    const double2 *TW;        // [512] e^{i pi j/1024}
    const double2 *PSI;       // [2048] e^{i pi u/1024} (key-pair monomials)
    // debug
    int32_t iters;            // CMux steps to run (n in production)
    uint32_t *acc_dump;       // if set: [n_work][2N] raw accumulator
    unsigned long long *margin;  // if set: max |v - round(v)| as double bits
};

// K1: linear combination (0, c0) + alpha A + beta B (+ gamma C) of work item e's
// gate inputs and modulus switch of its n+1 coefficients to Z_2N (bar[0..n]);
// threads tid = 0..nthreads-1 of the caller share the loop.
__device__ __forceinline__ void k1_modswitch(const BrArgs &args, uint32_t e, uint16_t *bar, int tid, int nthreads) {
    const int n = args.n;
    const uint32_t lanes = args.lanes;
    const BrItem it = args.items[e / lanes];
    const uint32_t lane_id = e % lanes;
    const int alpha = (int8_t)(it.coef & 0xFF), beta = (int8_t)((it.coef >> 8) & 0xFF);
    const int gamma = (int8_t)((it.coef >> 16) & 0xFF);
    const uint32_t *A = args.pool + ((size_t)it.src_a * lanes + lane_id) * args.pool_stride;
    const uint32_t *B = args.pool + ((size_t)it.src_b * lanes + lane_id) * args.pool_stride;
    const uint32_t *C = args.pool + ((size_t)it.src_c * lanes + lane_id) * args.pool_stride;
    for (int c = tid; c <= n; c += nthreads) {
        uint32_t v = (uint32_t)alpha * __ldg(&A[c]);
        if (beta) v += (uint32_t)beta * __ldg(&B[c]);
        if (gamma) v += (uint32_t)gamma * __ldg(&C[c]);
        if (c == n) v += it.c0;
        bar[c] = (uint16_t)(((v + (1u << 20)) >> 21) & (2 * kN - 1));
    }
}

// ACC = X^{-barb} (0, mu...mu): the A polynomial zero, B the rotated test vector
__device__ __forceinline__ void acc_init(uint32_t *accA, uint32_t *accB, int barb, uint32_t mu, int tid, int nthreads) {
    for (int i = tid; i < kN; i += nthreads) {
        if (accA) accA[i] = 0;
        if (accB) accB[i] = (((i + barb) & kN) ? 0u - mu : mu);
    }
}

// K3: sample extraction at index 0 of (A, B) into the big-LWE scratch row
__device__ __forceinline__ void sample_extract(const uint32_t *accA, const uint32_t *accB, uint32_t *out, int tid,
                                               int nthreads) {
    for (int c = tid; c <= kN; c += nthreads) {
        uint32_t v;
        if (c == 0) v = accA[0];
        else if (c < kN) v = 0u - accA[kN - c];
        else v = accB[0];
        out[c] = v;
    }
}

constexpr int kStages = 3;  // BK rows in the shared-memory ring
#ifndef HB_PAIR_UNROLL
#define HB_PAIR_UNROLL 3  // fully unrolled pair loop: rows (q, p) become compile-time
#endif
constexpr int kPairUnroll = HB_PAIR_UNROLL;

constexpr uint32_t kRowBytes = 2 * kNH * sizeof(double2);  // 16 KiB: one TGSW row, both output polys

#ifndef HB_BK_LDG
#define HB_BK_LDG 0  // 1: BK rows read through L1 (LDG + prefetch) instead of the smem ring
#endif
constexpr int kRingStages = HB_BK_LDG ? 1 : kStages;
template <int G>
struct BrSmem {
    double2 bk[kRingStages][2 * kNH];       // BK row ring
    uint64_t full[kStages], empty[kStages];
    uint32_t acc[G][2][kN];                  // TRLWE accumulators (A, B)
    double2 xch[G][2][2][kXchStride];        // FFT exchange buffers: [poly pair][double buffer]
    uint16_t bar[G][kMaxLweN + 1];           // mod-switched LWE (a_0..a_{n-1}, b)
    TwSeeds tws[64];                          // per-thread twiddle seeds
};

template <int G, bool kDebug>
__global__ void __launch_bounds__(64 * G, 1) k_blind_rotate(const BrArgs args) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrSmem<G> &sm = *reinterpret_cast<BrSmem<G> *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = args.n;
    const int iters = min(n, args.iters);
    const int rows_needed = iters * kRows;
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);

    // BK row ring: thread 0 is the producer.  Row `it` goes to stage it % kStages;
    // it is issued kLookahead rows ahead of its use, after every consumer warp
    // released the row that previously occupied the stage.
    if (threadIdx.x < 64) {
        const int tt = threadIdx.x;
        TwSeeds ts;
        ts.f_a0 = args.TW[tt];
        ts.step_a = args.W[tt];
        ts.step_b = args.W[8 * (tt & 7)];
        ts.i_b0 = args.TW[tt >> 3];
        ts.i_stepb = args.TW[32 * (tt & 7) + 8];
        sm.tws[tt] = ts;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 2 * G);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int it = 0; it < kStages && it < rows_needed && !HB_BK_LDG; it++) {
            mbar_arrive_expect_tx(&sm.full[it], kRowBytes);
            bulk_g2s(sm.bk[it], bk_src + (size_t)it * kRowBytes, kRowBytes, &sm.full[it]);
        }
    }
    __syncthreads();

    // ---- gate groups: 64 threads (2 warps) per bootstrap ----
    const int g = warp >> 1;
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + g;
    const uint32_t e_raw = blockIdx.x * G + g;
    const bool active = e_raw < args.n_work;
    const uint32_t e = active ? e_raw : args.n_work - 1;
    uint32_t *accA = sm.acc[g][0];
    uint32_t *accB = sm.acc[g][1];
    double2 *xch = &sm.xch[g][0][0][0];
    uint16_t *bar = sm.bar[g];

    k1_modswitch(args, e, bar, t, 64);  // K1
    group_bar(bar_id);
    acc_init(accA, accB, bar[n], args.mu, t, 64);  // ACC = X^{-barb} (0, mu...mu)
    group_bar(bar_id);

    double max_err = 0.0;
    int row_it = 0;  // global BK row counter (i * 6 + row)
    for (int i = 0; i < iters; i++) {
        const int a = bar[i];
        // rotation differences (X^a - 1) ACC for both polynomials
        uint32_t dlo[2][8], dhi[2][8];
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const uint32_t *P = q ? accB : accA;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int j = t + 64 * m;
#if HB_EXP_SKIP & 8
                dlo[q][m] = P[j] * 2654435761u;
                dhi[q][m] = P[j + kNH] * 2246822519u;
#else
                dlo[q][m] = rot_coef(P, j, a) - P[j];
                dhi[q][m] = rot_coef(P, j + kNH, a) - P[j + kNH];
#endif
            }
        }
        double2 f0[8], f1[8];  // Fourier accumulators of the two output polys
#pragma unroll kPairUnroll
        for (int pr = 0; pr < kRows / 2; pr++, row_it += 2) {
#if HB_BK_LDG
            {   // prefetch the next pair's two BK rows (32 KiB) into L1: 4 x 128-B lines per thread
                const char *nxt = bk_src + (size_t)(row_it + 2) * kRowBytes;
                if (row_it + 2 < rows_needed) {
#pragma unroll
                    for (int u = 0; u < 4; u++)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(nxt + (size_t)(t + 64 * u) * 128));
                }
            }
#endif
            // producer: rows row_it+1 and row_it+2 (stages freed by rows row_it-2, row_it-1)
            if (!HB_BK_LDG && threadIdx.x == 0) {
#pragma unroll 1
                for (int nx = row_it + 1; nx <= row_it + 2; nx++) {
                    if (nx < kStages || nx >= rows_needed) continue;
                    const int s2 = nx % kStages;
                    mbar_wait(&sm.empty[s2], ((nx / kStages) - 1) & 1);
                    mbar_arrive_expect_tx(&sm.full[s2], kRowBytes);
                    bulk_g2s(sm.bk[s2], bk_src + (size_t)nx * kRowBytes, kRowBytes, &sm.full[s2]);
                }
            }
            __syncwarp();
            double2 x[2][8];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int row = 2 * pr + h;
                const int q = row / kL, p = row % kL;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const uint32_t lo = q ? dlo[1][m] : dlo[0][m];
                    const uint32_t hi = q ? dhi[1][m] : dhi[0][m];
                    x[h][m] = make_double2(small_int_to_double(gadget_digit(lo, p)),
                                           small_int_to_double(gadget_digit(hi, p)));
                }
            }
            if (!(HB_EXP_SKIP & 1)) nega_fft_fwd_n<2>(x, xch, t, sm.tws[t], bar_id);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int rr = row_it + h;
                const int s = rr % kStages;
#if HB_BK_LDG
                const double2 *bk0 = args.bkf + (size_t)rr * 2 * kNH;
                const double2 *bk1 = bk0 + kNH;
#else
                mbar_wait(&sm.full[s], (rr / kStages) & 1);
                const double2 *bk0 = sm.bk[s];
                const double2 *bk1 = sm.bk[s] + kNH;
#endif
                if (kDebug && args.margin == nullptr && args.acc_dump != nullptr && args.n_work == 2) {
                    bk0 = args.bkf + (size_t)rr * 2 * kNH;  // bypass the ring (debug A/B)
                    bk1 = bk0 + kNH;
                }
                if (HB_EXP_SKIP & 2) {
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        if (pr == 0 && h == 0) { f0[m] = x[h][m]; f1[m] = x[h][m]; }
                        else { f0[m] = cadd(f0[m], x[h][m]); f1[m] = csub(f1[m], x[h][m]); }
                    }
                } else if (pr == 0 && h == 0) {
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        f0[m] = cmul(x[h][m], bk0[t + 64 * m]);
                        f1[m] = cmul(x[h][m], bk1[t + 64 * m]);
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        cmac(f0[m], x[h][m], bk0[t + 64 * m]);
                        cmac(f1[m], x[h][m], bk1[t + 64 * m]);
                    }
                }
                __syncwarp();
                if (!HB_BK_LDG && lane == 0) mbar_arrive(&sm.empty[s]);
            }
        }
        // inverse transforms of both output polynomials + round + ACC update
        {
            double2 x[2][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                x[0][m] = f0[m];
                x[1][m] = f1[m];
            }
            if (!(HB_EXP_SKIP & 4)) nega_fft_inv_n<2>(x, xch, t, sm.tws[t], bar_id);
#pragma unroll
            for (int q = 0; q < 2; q++) {
                uint32_t *P = q ? accB : accA;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const double lo = x[q][m].x, hi = x[q][m].y;
                    if (kDebug) {
                        max_err = fmax(max_err, fabs(lo - rint(lo)));
                        max_err = fmax(max_err, fabs(hi - rint(hi)));
                    }
                    const int j = t + 64 * m;
#if HB_EXP_SKIP & 16
                    if (lo == 12345.0) P[j] += 1;  // keep the computation alive
                    if (hi == 12345.0) P[j + kNH] += 1;
#else
                    P[j] += round_to_torus(lo);
                    P[j + kNH] += round_to_torus(hi);
#endif
                }
            }
        }
        group_bar(bar_id);
    }

    if (!active) return;
    if (kDebug && args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
    if (kDebug && args.acc_dump) {
        uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN;
        for (int c = t; c < 2 * kN; c += 64) dst[c] = (c < kN) ? accA[c] : accB[c - kN];
    }
    // K3: sample extract at index 0
    sample_extract(accA, accB, args.big + (size_t)e * kBigStride, t, 64);
}

// ---------------------------------------------------------------------------
// Latency mode (narrow levels): one bootstrap per CTA, three 64-thread groups.
// Group r takes TGSW rows 2r, 2r+1 of every CMux step (one dual forward FFT +
// MAC into a partial Fourier accumulator); groups 0/1 then sum the three
// partials of output polynomial 0/1, run its inverse FFT and update ACC.  The
// per-step critical path is one dual FFT instead of three.  Each group's two
// BK rows (32 KiB) arrive by cp.async.bulk into its own buffer, issued as soon
// as the previous step's partials have been consumed.  Bit-identical to the
// throughput kernel (different FP64 summation order; every rounding exact).
// ---------------------------------------------------------------------------
struct BrLatSmem {
    double2 bk[3][2][2 * kNH];               // per group: 2 rows x 2 output polys (32 KiB); reused for partials
    uint64_t full[3];
    uint32_t acc[2][kN];
    double2 xch[3][2][2][kXchStride];        // per group dual-FFT exchange buffers
    uint16_t bar[kMaxLweN + 1];
    TwSeeds tws[64];
};

template <bool kDebug>
__global__ void __launch_bounds__(192, 1) k_blind_rotate_lat(const BrArgs args) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrLatSmem &sm = *reinterpret_cast<BrLatSmem *>(smem_raw);
    const int warp = threadIdx.x >> 5;
    const int grp = warp >> 1;          // 0..2
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + grp;
    const int n = args.n;
    const int iters = min(n, args.iters);
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);
    const uint32_t e = blockIdx.x;      // one bootstrap per CTA (grid == n_work)
    uint32_t *accA = sm.acc[0];
    uint32_t *accB = sm.acc[1];
    double2 *xch = &sm.xch[grp][0][0][0];

    if (threadIdx.x < 64) {
        TwSeeds ts;
        ts.f_a0 = args.TW[t];
        ts.step_a = args.W[t];
        ts.step_b = args.W[8 * (t & 7)];
        ts.i_b0 = args.TW[t >> 3];
        ts.i_stepb = args.TW[32 * (t & 7) + 8];
        sm.tws[t] = ts;
    }
    // this group's rows of step 0
    if (t == 0) {
        mbar_init(&sm.full[grp], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (iters > 0) {
            mbar_arrive_expect_tx(&sm.full[grp], 2 * kRowBytes);
            bulk_g2s(sm.bk[grp], bk_src + (size_t)(2 * grp) * kRowBytes, 2 * kRowBytes, &sm.full[grp]);
        }
    }
    k1_modswitch(args, e, sm.bar, threadIdx.x, 192);  // K1
    __syncthreads();
    acc_init(accA, accB, sm.bar[n], args.mu, threadIdx.x, 192);  // ACC = X^{-barb} (0, mu...mu)
    __syncthreads();

    double max_err = 0.0;
    for (int i = 0; i < iters; i++) {
        const int a = sm.bar[i];
        // digits of this group's two rows: row = 2 grp + h, q = row / 3, p = row % 3
        double2 x[2][8];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int row = 2 * grp + h;
            const int q = row / kL, p = row % kL;
            const uint32_t *P = q ? accB : accA;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int j = t + 64 * m;
                const uint32_t lo = rot_coef(P, j, a) - P[j];
                const uint32_t hi = rot_coef(P, j + kNH, a) - P[j + kNH];
                x[h][m] = make_double2(small_int_to_double(gadget_digit(lo, p)),
                                       small_int_to_double(gadget_digit(hi, p)));
            }
        }
        nega_fft_fwd_n<2>(x, xch, t, sm.tws[t], bar_id);
        mbar_wait(&sm.full[grp], i & 1);
        double2 f0[8], f1[8];
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const double2 *b0 = sm.bk[grp][0], *b1 = sm.bk[grp][1];
            f0[m] = cmul(x[0][m], b0[t + 64 * m]);
            f1[m] = cmul(x[0][m], b0[kNH + t + 64 * m]);
            cmac(f0[m], x[1][m], b1[t + 64 * m]);
            cmac(f1[m], x[1][m], b1[kNH + t + 64 * m]);
        }
        group_bar(bar_id);  // all MAC reads of this group's BK buffer done
        // partials overwrite the (consumed) BK buffer: [0][.] = output poly 0, [1][.] = output poly 1
#pragma unroll
        for (int m = 0; m < 8; m++) {
            sm.bk[grp][0][t + 64 * m] = f0[m];
            sm.bk[grp][1][t + 64 * m] = f1[m];
        }
        __syncthreads();
        if (grp < 2) {
            // group o sums the three partials of output polynomial o, inverse FFT, ACC update
            double2 y[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int k = t + 64 * m;
                y[0][m] = cadd(cadd(sm.bk[0][grp][k], sm.bk[1][grp][k]), sm.bk[2][grp][k]);
            }
            nega_fft_inv_n<1>(y, xch, t, sm.tws[t], bar_id);
            uint32_t *P = grp ? accB : accA;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const double lo = y[0][m].x, hi = y[0][m].y;
                if (kDebug) {
                    max_err = fmax(max_err, fabs(lo - rint(lo)));
                    max_err = fmax(max_err, fabs(hi - rint(hi)));
                }
                const int j = t + 64 * m;
                P[j] += round_to_torus(lo);
                P[j + kNH] += round_to_torus(hi);
            }
        }
        __syncthreads();  // partials consumed, ACC updated
        if (t == 0 && i + 1 < iters) {  // next step's rows for this group
            // generic-proxy reads/writes of this buffer (MAC, partials) before the async-proxy refill
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_expect_tx(&sm.full[grp], 2 * kRowBytes);
            bulk_g2s(sm.bk[grp], bk_src + (size_t)((i + 1) * kRows + 2 * grp) * kRowBytes, 2 * kRowBytes,
                     &sm.full[grp]);
        }
    }

    if (kDebug && args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
    if (kDebug && args.acc_dump) {
        uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN;
        for (int c = threadIdx.x; c < 2 * kN; c += 192) dst[c] = (c < kN) ? accA[c] : accB[c - kN];
    }
    sample_extract(accA, accB, args.big + (size_t)e * kBigStride, threadIdx.x, 192);
}

// ---------------------------------------------------------------------------
// Tensor memory (TMEM) as per-thread private storage: each thread of a warp
// owns one TMEM lane (warp w -> lanes 32 (w % 4) ..); 32x32b loads / stores
// move 32 consecutive 32-bit columns of that lane to / from registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// one warp allocates `cols` columns (power of two >= 32) and publishes the base
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_addr(dst_smem)), "r"(cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t base, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(base), "r"(cols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// ---------------------------------------------------------------------------
// K1+K2+K3 with the key-pair bootstrapping key (bk_unroll 2).  One external
// product per key pair (i, j) = (2m, 2m+1):
//   ACC <- ACC + BK_m [x] ACC,  BK_m = sum_c (X^{e_c} - 1) BK_{m,c},
//   (e_0, e_1, e_2) = (a_i + a_j, a_i, a_j),
// whose TGSW message is X^{a_i s_i + a_j s_j} - 1.  Per pair: 6 forward
// transforms of the digits of ACC itself (no rotation), 2 inverse transforms,
// and for every digit row and component a Fourier MAC with the digit spectrum
// pre-multiplied by F_c = (X^{e_c} - 1)(psi^{4k+1}) — half the transforms of
// two CGGI steps for 1.5x the MAC.  The BK arrives as 16 KiB (row, component)
// stages through a 7-deep cp.async.bulk ring; the FFT exchange is
// single-buffered to make room for it.  Same rounding argument as the CGGI
// kernel: the exact integer result (< 2^53) is recovered by the final rounding.
// ---------------------------------------------------------------------------
constexpr int kStagesU2 = 7;
constexpr int kStagesPerPair = 3 * kRows;  // (row pair, component, row) stages per key pair
#ifndef HB_TRACE
#define HB_TRACE 0  // per-phase clock64 trace of the cluster latency kernel (printf, one pair)
#endif
#ifndef HB_EXP_BK_SAME
#define HB_EXP_BK_SAME 0  // timing experiment only (results wrong): every pair re-reads pair 0's stages
#endif
__device__ __forceinline__ size_t u2_stage(int s) { return HB_EXP_BK_SAME ? (size_t)(s % kStagesPerPair) : (size_t)s; }

__constant__ double2 c_w8[8] = {{1.0, 0.0},
                                {0.70710678118654752440, 0.70710678118654752440},
                                {0.0, 1.0},
                                {-0.70710678118654752440, 0.70710678118654752440},
                                {-1.0, 0.0},
                                {-0.70710678118654752440, -0.70710678118654752440},
                                {0.0, -1.0},
                                {0.70710678118654752440, -0.70710678118654752440}};

template <int G, int R = kStagesU2, bool TM = false>
struct BrSmemU2 {
    double2 bk[R][2 * kNH];                  // stage ring: [output poly][bin]
    uint64_t full[R], empty[R];
    uint32_t acc[TM ? 1 : G][2][TM ? 1 : kN];  // TRLWE accumulators (TM: in tensor memory instead)
    double2 xch[G][2][kXchStride];           // single-buffered dual-FFT exchange
    uint16_t bar[G][kMaxLweN + 1];
    TwSeeds tws[64];
    uint32_t tmem_base;
};

// R: ring stages; MB: resident CTAs per SM the launch bounds target.  A ring
// shallower than one row pair (R < 7) is refilled after every consumed stage.
// TM: the accumulators live in tensor memory.  In this kernel every thread
// reads and updates only its own ACC coefficients (bins t + 64 m of both
// polynomials, no rotation), so ACC is thread-private: 32 TMEM columns of the
// thread's lane, and the 32 KiB of shared memory go to the BK ring.
template <int G, bool kDebug, int R = kStagesU2, int MB = 1, bool TM = false>
__global__ void __launch_bounds__(64 * G, MB) k_blind_rotate_u2(const BrArgs args) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrSmemU2<G, R, TM> &sm = *reinterpret_cast<BrSmemU2<G, R, TM> *>(smem_raw);
    constexpr bool kMidIssue = R < kRows + 1;
    constexpr uint32_t kTmemCols = G > 2 ? 64 : 32;  // warps w and w + 4 share a lane quarter
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = args.n;
    const int pairs = min(n, args.iters) / 2;
    const int stages_needed = pairs * kStagesPerPair;
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);

    if (threadIdx.x < 64) {
        const int tt = threadIdx.x;
        TwSeeds ts;
        ts.f_a0 = args.TW[tt];
        ts.step_a = args.W[tt];
        ts.step_b = args.W[8 * (tt & 7)];
        ts.i_b0 = args.TW[tt >> 3];
        ts.i_stepb = args.TW[32 * (tt & 7) + 8];
        sm.tws[tt] = ts;
    }
    int issued = 0;  // producer (thread 0) state: stages issued so far
    if (threadIdx.x == 0) {
        for (int s = 0; s < R; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 2 * G);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (; issued < R && issued < stages_needed; issued++) {
            mbar_arrive_expect_tx(&sm.full[issued], kRowBytes);
            bulk_g2s(sm.bk[issued], bk_src + u2_stage(issued) * kRowBytes, kRowBytes, &sm.full[issued]);
        }
    }
    if (TM && warp == 0) tmem_alloc(&sm.tmem_base, kTmemCols);
    if (TM) tmem_fence_before();
    __syncthreads();
    if (TM) tmem_fence_after();
    // this thread's 32 ACC columns: A at +0..15, B at +16..31 (lo bins m, then hi bins m)
    const uint32_t tacc = TM ? sm.tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + 32u * (uint32_t)(warp >> 2) : 0u;

    const int g = warp >> 1;
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + g;
    const uint32_t e_raw = blockIdx.x * G + g;
    const bool active = e_raw < args.n_work;
    const uint32_t e = active ? e_raw : args.n_work - 1;
    uint32_t *accA = sm.acc[TM ? 0 : g][0];
    uint32_t *accB = sm.acc[TM ? 0 : g][1];
    double2 *xch = &sm.xch[g][0][0];
    uint16_t *bar = sm.bar[g];

    k1_modswitch(args, e, bar, t, 64);  // K1
    group_bar(bar_id);
    if (TM) {  // ACC = X^{-barb} (0, mu...mu) at this thread's bins
        const int barb = bar[n];
        uint32_t v[32];
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const int j = t + 64 * m;
            v[m] = 0;
            v[8 + m] = 0;
            v[16 + m] = ((j + barb) & kN) ? 0u - args.mu : args.mu;
            v[24 + m] = ((j + kNH + barb) & kN) ? 0u - args.mu : args.mu;
        }
        tmem_st32(tacc, v);
    } else {
        acc_init(accA, accB, bar[n], args.mu, t, 64);  // ACC = X^{-barb} (0, mu...mu)
        group_bar(bar_id);
    }

    double max_err = 0.0;
    int st = 0;  // next stage to consume
    for (int pm = 0; pm < pairs; pm++) {
        const int ai = bar[2 * pm], aj = bar[2 * pm + 1];
        // F_c at this thread's bins k = t + 64 m: psi^{e (4k+1)} - 1 =
        // psi^{e (4t+1)} * w8^{e m} - 1 (the exponent is warp-uniform)
        int ex[3];
        double2 base[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            ex[c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            base[c] = __ldg(&args.PSI[(ex[c] * (4 * t + 1)) & (2 * kN - 1)]);
        }
        double2 f0[8], f1[8];
#pragma unroll 1
        for (int rp = 0; rp < kRows / 2; rp++) {
            // producer: refill the ring up to R stages ahead of this row pair
            if (threadIdx.x == 0) {
#pragma unroll 1
                for (; issued < st + R && issued < stages_needed; issued++) {
                    const int s2 = issued % R;
                    mbar_wait(&sm.empty[s2], ((issued / R) - 1) & 1);
                    mbar_arrive_expect_tx(&sm.full[s2], kRowBytes);
                    bulk_g2s(sm.bk[s2], bk_src + u2_stage(issued) * kRowBytes, kRowBytes, &sm.full[s2]);
                }
            }
            __syncwarp();
            double2 x[2][8];
            if (TM) {
                uint32_t v[32];
                tmem_ld32(tacc, v);
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int row = 2 * rp + h;
                    const int q = row / kL, p = row % kL;
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        const uint32_t lo = q ? v[16 + m] : v[m], hi = q ? v[24 + m] : v[8 + m];
                        x[h][m] = make_double2(small_int_to_double(gadget_digit(lo, p)),
                                               small_int_to_double(gadget_digit(hi, p)));
                    }
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int row = 2 * rp + h;
                    const int q = row / kL, p = row % kL;
                    const uint32_t *P = q ? accB : accA;
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        const int j = t + 64 * m;
                        x[h][m] = make_double2(small_int_to_double(gadget_digit(P[j], p)),
                                               small_int_to_double(gadget_digit(P[j + kNH], p)));
                    }
                }
            }
            nega_fft_fwd_n<2, true>(x, xch, t, sm.tws[t], bar_id);
#pragma unroll
            for (int c = 0; c < 3; c++) {
                double2 F[8];  // (X^{e_c} - 1) at this thread's bins (recomputed per row pair: registers)
                {
                    // psi^{e(4t+1)} w8^{e m}: w8^{4e} = (-1)^e, so bins m + 4 are bins m
                    // with the sign flipped for odd e (integer sign-bit flips, no FP64 work)
                    const long long flip = (long long)(ex[c] & 1) << 63;
                    double2 p[4];
#pragma unroll
                    for (int m = 0; m < 4; m++) p[m] = m == 0 ? base[c] : cmul(base[c], c_w8[(ex[c] * m) & 7]);
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        F[m] = make_double2(p[m].x - 1.0, p[m].y);
                        F[m + 4] = make_double2(__longlong_as_double(__double_as_longlong(p[m].x) ^ flip) - 1.0,
                                                __longlong_as_double(__double_as_longlong(p[m].y) ^ flip));
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; h++, st++) {
                    const int s = st % R;
                    mbar_wait(&sm.full[s], (st / R) & 1);
                    const double2 *bk0 = sm.bk[s];
                    const double2 *bk1 = sm.bk[s] + kNH;
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        const double2 y = cmul(x[h][m], F[m]);
                        if (rp == 0 && c == 0 && h == 0) {
                            f0[m] = cmul(y, bk0[t + 64 * m]);
                            f1[m] = cmul(y, bk1[t + 64 * m]);
                        } else {
                            cmac(f0[m], y, bk0[t + 64 * m]);
                            cmac(f1[m], y, bk1[t + 64 * m]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.empty[s]);
                    if (kMidIssue && threadIdx.x == 0) {  // shallow ring: refill behind consumption
#pragma unroll 1
                        for (; issued < st + 1 + R && issued < stages_needed; issued++) {
                            const int s2 = issued % R;
                            mbar_wait(&sm.empty[s2], ((issued / R) - 1) & 1);
                            mbar_arrive_expect_tx(&sm.full[s2], kRowBytes);
                            bulk_g2s(sm.bk[s2], bk_src + u2_stage(issued) * kRowBytes, kRowBytes, &sm.full[s2]);
                        }
                    }
                    __syncwarp();
                }
            }
        }
        {
            double2 x[2][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                x[0][m] = f0[m];
                x[1][m] = f1[m];
            }
            nega_fft_inv_n<2, true>(x, xch, t, sm.tws[t], bar_id);
            if (kDebug) {
#pragma unroll
                for (int q = 0; q < 2; q++)
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        max_err = fmax(max_err, fabs(x[q][m].x - rint(x[q][m].x)));
                        max_err = fmax(max_err, fabs(x[q][m].y - rint(x[q][m].y)));
                    }
            }
            if (TM) {
                uint32_t v[32];
                tmem_ld32(tacc, v);
#pragma unroll
                for (int q = 0; q < 2; q++)
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        v[16 * q + m] += round_to_torus(x[q][m].x);
                        v[16 * q + 8 + m] += round_to_torus(x[q][m].y);
                    }
                tmem_st32(tacc, v);
            } else {
#pragma unroll
                for (int q = 0; q < 2; q++) {
                    uint32_t *P = q ? accB : accA;
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        const int j = t + 64 * m;
                        P[j] += round_to_torus(x[q][m].x);
                        P[j + kNH] += round_to_torus(x[q][m].y);
                    }
                }
            }
        }
        if (!TM) group_bar(bar_id);  // TM: ACC is thread-private; the next FFT starts with a barrier
    }

    if (TM) {
        uint32_t v[32];
        tmem_ld32(tacc, v);
        if (active) {
            if (kDebug && args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
            if (kDebug && args.acc_dump) {
                uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const int j = t + 64 * m;
                    dst[j] = v[m];
                    dst[j + kNH] = v[8 + m];
                    dst[kN + j] = v[16 + m];
                    dst[kN + j + kNH] = v[24 + m];
                }
            }
            // K3: sample extraction at index 0 from this thread's coefficients:
            // a'_0 = A_0, a'_c = -A_{N-c}, b' = B_0
            uint32_t *out = args.big + (size_t)e * kBigStride;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int j = t + 64 * m;
                if (j == 0) {
                    out[0] = v[0];
                    out[kN] = v[16];
                } else {
                    out[kN - j] = 0u - v[m];
                }
                out[kNH - j] = 0u - v[8 + m];  // coefficient j + 512
            }
        }
        tmem_fence_before();
        __syncthreads();
        tmem_fence_after();
        if (warp == 0) tmem_dealloc(sm.tmem_base, kTmemCols);
        return;
    }
    if (!active) return;
    if (kDebug && args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
    if (kDebug && args.acc_dump) {
        uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN;
        for (int c = t; c < 2 * kN; c += 64) dst[c] = (c < kN) ? accA[c] : accB[c - kN];
    }
    sample_extract(accA, accB, args.big + (size_t)e * kBigStride, t, 64);
}

// ---------------------------------------------------------------------------
// Latency mode with the key-pair key (narrow levels): one bootstrap per CTA,
// three 64-thread groups; group r takes digit rows 2r, 2r+1 of every key pair
// (one dual forward FFT + the 6 (component, row) MAC stages, streamed through a
// 3-deep per-group ring), writes its partial Fourier sums into its exchange
// buffer; groups 0/1 sum the partials of output polynomial 0/1, run its inverse
// FFT and update ACC.
// ---------------------------------------------------------------------------
constexpr int kLatStagesU2 = 3;

struct BrLatSmemU2 {
    double2 bk[3][kLatStagesU2][2 * kNH];    // per-group stage rings
    uint64_t full[3][kLatStagesU2], empty[3][kLatStagesU2];
    uint32_t acc[2][kN];
    double2 xch[3][2][kXchStride];           // per-group single-buffered exchange; partials [o][512]
    uint16_t bar[kMaxLweN + 1];
    TwSeeds tws[64];
};

template <bool kDebug>
__global__ void __launch_bounds__(192, 1) k_blind_rotate_u2_lat(const BrArgs args) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrLatSmemU2 &sm = *reinterpret_cast<BrLatSmemU2 *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = warp >> 1;
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + grp;
    const int n = args.n;
    const int pairs = min(n, args.iters) / 2;
    const int stages_needed = pairs * 6;  // this group's stages
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);
    const uint32_t e = blockIdx.x;
    uint32_t *accA = sm.acc[0];
    uint32_t *accB = sm.acc[1];
    double2 *xch = &sm.xch[grp][0][0];
    uint64_t *full = sm.full[grp], *empty = sm.empty[grp];
    // group-local stage s -> global stage (s / 6) * 18 + grp * 6 + s % 6
    auto stage_src = [&](int s) {
        return bk_src + (size_t)((s / 6) * kStagesPerPair + grp * 6 + s % 6) * kRowBytes;
    };

    if (threadIdx.x < 64) {
        TwSeeds ts;
        ts.f_a0 = args.TW[t];
        ts.step_a = args.W[t];
        ts.step_b = args.W[8 * (t & 7)];
        ts.i_b0 = args.TW[t >> 3];
        ts.i_stepb = args.TW[32 * (t & 7) + 8];
        sm.tws[t] = ts;
    }
    int issued = 0;  // group producer (t == 0) state
    if (t == 0) {
        for (int s = 0; s < kLatStagesU2; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 2);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (; issued < kLatStagesU2 && issued < stages_needed; issued++) {
            mbar_arrive_expect_tx(&full[issued], kRowBytes);
            bulk_g2s(sm.bk[grp][issued], stage_src(issued), kRowBytes, &full[issued]);
        }
    }
    k1_modswitch(args, e, sm.bar, threadIdx.x, 192);  // K1
    __syncthreads();
    acc_init(accA, accB, sm.bar[n], args.mu, threadIdx.x, 192);  // ACC = X^{-barb} (0, mu...mu)
    __syncthreads();

    double max_err = 0.0;
    int st = 0;  // this group's next stage
    for (int pm = 0; pm < pairs; pm++) {
        const int ai = sm.bar[2 * pm], aj = sm.bar[2 * pm + 1];
        int ex[3];
        double2 base[3];  // issued before the FFT: the table loads' L2 latency overlaps it
#pragma unroll
        for (int c = 0; c < 3; c++) {
            ex[c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            base[c] = __ldg(&args.PSI[(ex[c] * (4 * t + 1)) & (2 * kN - 1)]);
        }
        double2 x[2][8];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int row = 2 * grp + h;
            const int q = row / kL, p = row % kL;
            const uint32_t *P = q ? accB : accA;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int j = t + 64 * m;
                x[h][m] = make_double2(small_int_to_double(gadget_digit(P[j], p)),
                                       small_int_to_double(gadget_digit(P[j + kNH], p)));
            }
        }
        nega_fft_fwd_n<2, true>(x, xch, t, sm.tws[t], bar_id);
        double2 f0[8], f1[8];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const int ec = ex[c];
            double2 F[8];
            {
                const long long flip = (long long)(ec & 1) << 63;
                double2 p[4];
#pragma unroll
                for (int m = 0; m < 4; m++) p[m] = m == 0 ? base[c] : cmul(base[c], c_w8[(ec * m) & 7]);
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    F[m] = make_double2(p[m].x - 1.0, p[m].y);
                    F[m + 4] = make_double2(__longlong_as_double(__double_as_longlong(p[m].x) ^ flip) - 1.0,
                                            __longlong_as_double(__double_as_longlong(p[m].y) ^ flip));
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++, st++) {
                const int s = st % kLatStagesU2;
                mbar_wait(&full[s], (st / kLatStagesU2) & 1);
                const double2 *bk0 = sm.bk[grp][s];
                const double2 *bk1 = sm.bk[grp][s] + kNH;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const double2 y = cmul(x[h][m], F[m]);
                    if (c == 0 && h == 0) {
                        f0[m] = cmul(y, bk0[t + 64 * m]);
                        f1[m] = cmul(y, bk1[t + 64 * m]);
                    } else {
                        cmac(f0[m], y, bk0[t + 64 * m]);
                        cmac(f1[m], y, bk1[t + 64 * m]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (t == 0 && issued < stages_needed) {  // refill this slot kLatStagesU2 stages ahead
                    mbar_wait(&empty[s], ((issued / kLatStagesU2) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], kRowBytes);
                    bulk_g2s(sm.bk[grp][s], stage_src(issued), kRowBytes, &full[s]);
                    issued++;
                }
                __syncwarp();
            }
        }
        // partials into this group's exchange buffer: [0][.] output poly 0, [1][.] output poly 1
        group_bar(bar_id);  // the forward FFT's last readers of xch are done
#pragma unroll
        for (int m = 0; m < 8; m++) {
            xch[t + 64 * m] = f0[m];
            xch[kNH + t + 64 * m] = f1[m];
        }
        __syncthreads();
        if (grp < 2) {
            double2 y[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int k = grp * kNH + t + 64 * m;
                y[0][m] = cadd(cadd(sm.xch[0][0][k], sm.xch[1][0][k]), sm.xch[2][0][k]);
            }
            asm volatile("bar.sync 4, 128;" ::: "memory");  // groups 0/1: partial reads done before reuse
            nega_fft_inv_n<1, true>(y, xch, t, sm.tws[t], bar_id);
            uint32_t *P = grp ? accB : accA;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const double lo = y[0][m].x, hi = y[0][m].y;
                if (kDebug) {
                    max_err = fmax(max_err, fabs(lo - rint(lo)));
                    max_err = fmax(max_err, fabs(hi - rint(hi)));
                }
                const int j = t + 64 * m;
                P[j] += round_to_torus(lo);
                P[j + kNH] += round_to_torus(hi);
            }
        }
        __syncthreads();  // ACC updated, partials consumed
    }

    if (kDebug && args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
    if (kDebug && args.acc_dump) {
        uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN;
        for (int c = threadIdx.x; c < 2 * kN; c += 192) dst[c] = (c < kN) ? accA[c] : accB[c - kN];
    }
    sample_extract(accA, accB, args.big + (size_t)e * kBigStride, threadIdx.x, 192);
}

// ---------------------------------------------------------------------------
// Latency mode for very narrow levels (<= #SM/2 bootstraps), key pairs: one
// bootstrap per 2-CTA cluster.  CTA q owns TRLWE polynomial q (ACC_q and its
// three digit rows 3q..3q+2); group g of CTA q transforms digit row 3q+g
// (single FFT) and runs its 3 (component) MAC stages from a 3-slot ring
// (slot c = component c, refilled with the next pair's stage as soon as it is
// consumed).  Partials meet over distributed shared memory: group 0 of CTA q
// sums output polynomial q over the six groups (3 local, 3 in the peer CTA),
// inverse-transforms it and updates ACC_q.  Two cluster barriers per pair.
// ---------------------------------------------------------------------------
// cluster barriers: the full (release/acquire) form publishes shared-memory
// writes to the peer CTA; the relaxed arrive only orders execution (used once
// the peer's DSMEM loads have been consumed) and its wait is deferred.
__device__ __forceinline__ void cluster_sync_acq_rel() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

struct BrCluSmemU2 {
    double2 bk[3][3][2 * kNH];               // [group][component slot][output poly][bin]
    uint64_t full[3][3];
    uint32_t acc[kN];                        // ACC_q
    double2 xch[3][2][kXchStride];           // per group: [0] FFT exchange, then own partial; [1] peer's partial
    double2 inv[kXchStride];                 // group 0's inverse-FFT exchange
    uint16_t bar[kMaxLweN + 1];
    TwSeeds tws[64];
};

template <bool kDebug>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1) k_blind_rotate_u2_clu(const BrArgs args) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrCluSmemU2 &sm = *reinterpret_cast<BrCluSmemU2 *>(smem_raw);
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int q = (int)cluster.block_rank();   // TRLWE polynomial owned by this CTA
    BrCluSmemU2 &peer = *cluster.map_shared_rank(&sm, q ^ 1);
    const int warp = threadIdx.x >> 5;
    const int grp = warp >> 1;
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + grp;
    const int n = args.n;
    const int pairs = min(n, args.iters) / 2;
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);
    const uint32_t e = blockIdx.x >> 1;
    const int row = 3 * q + grp, p = grp;         // digit row of this group: poly q, digit p
    const int rp = row >> 1, h = row & 1;
    auto stage_src = [&](int pm, int c) {
        return bk_src + (size_t)(pm * kStagesPerPair + rp * 6 + c * 2 + h) * kRowBytes;
    };
    double2 *xch = &sm.xch[grp][0][0];

    if (threadIdx.x < 64) {
        TwSeeds ts;
        ts.f_a0 = args.TW[t];
        ts.step_a = args.W[t];
        ts.step_b = args.W[8 * (t & 7)];
        ts.i_b0 = args.TW[t >> 3];
        ts.i_stepb = args.TW[32 * (t & 7) + 8];
        sm.tws[t] = ts;
    }
    if (t == 0) {
        for (int c = 0; c < 3; c++) mbar_init(&sm.full[grp][c], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (pairs > 0) {
            for (int c = 0; c < 3; c++) {
                mbar_arrive_expect_tx(&sm.full[grp][c], kRowBytes);
                bulk_g2s(sm.bk[grp][c], stage_src(0, c), kRowBytes, &sm.full[grp][c]);
            }
        }
    }
    k1_modswitch(args, e, sm.bar, threadIdx.x, 192);  // K1
    __syncthreads();
    acc_init(q == 0 ? sm.acc : nullptr, q == 0 ? nullptr : sm.acc, sm.bar[n], args.mu, threadIdx.x, 192);  // ACC_q
    cluster.sync();  // peer smem live (DSMEM), ACC initialised

    double max_err = 0.0;
#if HB_TRACE
    long long tr[12];
#define HB_TR(k) do { if (pm == 100) tr[k] = clock64(); } while (0)
#else
#define HB_TR(k) do { } while (0)
#endif
    for (int pm = 0; pm < pairs; pm++) {
        HB_TR(0);
        const int ai = sm.bar[2 * pm], aj = sm.bar[2 * pm + 1];
        int ex[3];
        double2 base[3];  // issued before the FFT: the table loads' L2 latency overlaps it
#pragma unroll
        for (int c = 0; c < 3; c++) {
            ex[c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            base[c] = __ldg(&args.PSI[(ex[c] * (4 * t + 1)) & (2 * kN - 1)]);
        }
        double2 x[1][8];
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const int j = t + 64 * m;
            x[0][m] = make_double2(small_int_to_double(gadget_digit(sm.acc[j], p)),
                                   small_int_to_double(gadget_digit(sm.acc[j + kNH], p)));
        }
        if (pm > 0) cluster_wait();  // the peer has read our previous partials (relaxed arrive below)
        HB_TR(1);
        nega_fft_fwd_n<1, true>(x, xch, t, sm.tws[t], bar_id);
        HB_TR(2);
        double2 f0[8], f1[8];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const int ec = ex[c];
            double2 F[8];
            {
                const long long flip = (long long)(ec & 1) << 63;
                double2 pw[4];
#pragma unroll
                for (int m = 0; m < 4; m++) pw[m] = m == 0 ? base[c] : cmul(base[c], c_w8[(ec * m) & 7]);
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    F[m] = make_double2(pw[m].x - 1.0, pw[m].y);
                    F[m + 4] = make_double2(__longlong_as_double(__double_as_longlong(pw[m].x) ^ flip) - 1.0,
                                            __longlong_as_double(__double_as_longlong(pw[m].y) ^ flip));
                }
            }
            mbar_wait(&sm.full[grp][c], pm & 1);
            const double2 *bk0 = sm.bk[grp][c];
            const double2 *bk1 = sm.bk[grp][c] + kNH;
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const double2 y = cmul(x[0][m], F[m]);
                if (c == 0) {
                    f0[m] = cmul(y, bk0[t + 64 * m]);
                    f1[m] = cmul(y, bk1[t + 64 * m]);
                } else {
                    cmac(f0[m], y, bk0[t + 64 * m]);
                    cmac(f1[m], y, bk1[t + 64 * m]);
                }
            }
        }
        HB_TR(9);
        group_bar(bar_id);  // both warps done with the three slots (and with the FFT's xch reads)
        HB_TR(10);
        if (t == 0 && pm + 1 < pairs) {  // the next pair's stages load during reduce / inverse / FFT
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int c = 0; c < 3; c++) {
                mbar_arrive_expect_tx(&sm.full[grp][c], kRowBytes);
                bulk_g2s(sm.bk[grp][c], stage_src(pm + 1, c), kRowBytes, &sm.full[grp][c]);
            }
        }
        // partial of our output q into this group's exchange buffer (its FFT readers are
        // done: the group barrier of the last stage above); the partial of the peer's
        // output goes straight into the upper half of the peer group's buffer (unused by
        // its single-poly FFT; its previous contents were consumed before the peer's
        // relaxed arrive that our cluster_wait matched)
        {
            double2 *remote = &peer.xch[grp][1][0];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                xch[t + 64 * m] = q ? f1[m] : f0[m];
                remote[t + 64 * m] = q ? f0[m] : f1[m];
            }
        }
        HB_TR(3);
        cluster_sync_acq_rel();  // all six groups' partials visible cluster-wide
        HB_TR(4);
        if (grp != 0) cluster_arrive_relaxed();
        if (grp == 0) {
            double2 y[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int k = t + 64 * m;  // own partials in [g][0], the peer's in [g][1]
                double2 v = cadd(cadd(sm.xch[0][0][k], sm.xch[1][0][k]), sm.xch[2][0][k]);
                v = cadd(v, cadd(cadd(sm.xch[0][1][k], sm.xch[1][1][k]), sm.xch[2][1][k]));
                y[0][m] = v;
            }
            cluster_arrive_relaxed();  // received partials consumed (values are in registers)
            HB_TR(5);
            nega_fft_inv_n<1, true>(y, sm.inv, t, sm.tws[t], bar_id);
            HB_TR(6);
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const double lo = y[0][m].x, hi = y[0][m].y;
                if (kDebug) {
                    max_err = fmax(max_err, fabs(lo - rint(lo)));
                    max_err = fmax(max_err, fabs(hi - rint(hi)));
                }
                const int j = t + 64 * m;
                sm.acc[j] += round_to_torus(lo);
                sm.acc[j + kNH] += round_to_torus(hi);
            }
        }
        HB_TR(7);
        __syncthreads();  // ACC_q updated
        HB_TR(8);
#if HB_TRACE
        if (pm == 100 && blockIdx.x == 0 && threadIdx.x == 0)
            printf("clu trace: digits %lld fwd %lld mac %lld bar %lld partials %lld sync1 %lld reduce %lld inv %lld "
                   "acc %lld sync2 %lld\n",
                   tr[1] - tr[0], tr[2] - tr[1], tr[9] - tr[2], tr[10] - tr[9], tr[3] - tr[10], tr[4] - tr[3],
                   tr[5] - tr[4], tr[6] - tr[5], tr[7] - tr[6], tr[8] - tr[7]);
#endif
    }
#undef HB_TR
    if (pairs > 0) cluster_wait();  // the peer is done reading our shared memory

    if (kDebug && args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
    if (kDebug && args.acc_dump) {
        uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN + (size_t)q * kN;
        for (int c = threadIdx.x; c < kN; c += 192) dst[c] = sm.acc[c];
    }
    uint32_t *out = args.big + (size_t)e * kBigStride;
    if (q == 0) {
        for (int c = threadIdx.x; c < kN; c += 192) out[c] = c == 0 ? sm.acc[0] : 0u - sm.acc[kN - c];
    } else if (threadIdx.x == 0) {
        out[kN] = sm.acc[0];
    }
}

// ---------------------------------------------------------------------------
// K4: batched key switch.  For coefficient i the CGGI digits are the eight
// base-4 digits of w_i = (a'_i + 2^15) >> 16.  The device KSK is laid out as a
// lookup table per 8-column chunk, T[chunk][i][j][d][8] with T[..][0][..] = 0,
// so one digit costs two LDS.128 (the 4 candidate rows of an (i, j) fill one
// 128-B line: lanes with different digits hit different banks) and 8 IADDs.
// CTA = 128 gates (one per thread) x one 8-column chunk; the chunk's 1 MiB
// table streams through a shared-memory ring fed by cp.async.bulk, so every
// table byte fetched from L2 serves 128 gates.
// ---------------------------------------------------------------------------
struct KsArgs {
    const uint32_t *big;     // [n_br_work][kBigStride]
    const KsItem *items;     // [n_items]
    uint32_t lanes;
    uint32_t n_work;         // n_items * lanes
    const uint32_t *ksk;     // [kKsChunks][kN][t][4][kKsCols] lookup table
    uint32_t *pool;
    uint32_t pool_stride;
    int32_t n;
    uint32_t *partial;       // narrow levels: [splits][n_work][kKskStride] raw sums (else null)
};

constexpr int kKsCols = 8;                               // output columns per chunk
constexpr int kKsChunks = kKskStride / kKsCols;           // 80
constexpr int kKsThreads = 128;                           // one gate per thread
constexpr int kKsIBlock = 8;                              // coefficients per ring stage
constexpr uint32_t kKsStageBytes = kKsIBlock * kKsT * 4 * kKsCols * 4;  // 8 KiB
constexpr int kKsStages = 4;
constexpr size_t kKsTableWords = (size_t)kKsChunks * kN * kKsT * 4 * kKsCols;

struct KsSmem {
    uint4 tab[kKsStages][kKsStageBytes / 16];
    uint64_t full[kKsStages], empty[kKsStages];
};

__global__ void __launch_bounds__(kKsThreads) k_keyswitch(const KsArgs args) {
    __shared__ __align__(128) KsSmem ks;
    const int lane = threadIdx.x & 31;
    const uint32_t e = blockIdx.x * kKsThreads + threadIdx.x;
    const bool active = e < args.n_work;
    const uint32_t ee = active ? e : args.n_work - 1;
    const uint32_t lanes = args.lanes;
    const KsItem it = args.items[ee / lanes];
    const uint32_t lane_id = ee % lanes;
    const uint32_t *b0 = args.big + ((size_t)it.i0 * lanes + lane_id) * kBigStride;
    const uint32_t *b1 = it.i1 != 0xFFFFFFFFu ? args.big + ((size_t)it.i1 * lanes + lane_id) * kBigStride : nullptr;
    const int chunk = blockIdx.y;
    // blockIdx.z splits the coefficient range (narrow levels: more CTAs, shorter streams)
    const int kBlocks = (kN / kKsIBlock) / gridDim.z;
    const int blk0 = blockIdx.z * kBlocks;
    const char *tab_src = reinterpret_cast<const char *>(args.ksk) + (size_t)chunk * kN * kKsT * 4 * kKsCols * 4 +
                          (size_t)blk0 * kKsStageBytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kKsStages; s++) {
            mbar_init(&ks.full[s], 1);
            mbar_init(&ks.empty[s], kKsThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int b = 0; b < kKsStages - 1 && b < kBlocks; b++) {
            mbar_arrive_expect_tx(&ks.full[b], kKsStageBytes);
            bulk_g2s(ks.tab[b], tab_src + (size_t)b * kKsStageBytes, kKsStageBytes, &ks.full[b]);
        }
    }
    __syncthreads();

    uint32_t acc[kKsCols];
#pragma unroll
    for (int c = 0; c < kKsCols; c++) acc[c] = 0;
    const uint4 *wsrc0 = reinterpret_cast<const uint4 *>(b0) + 2 * blk0;
    const uint4 *wsrc1 = b1 ? reinterpret_cast<const uint4 *>(b1) + 2 * blk0 : nullptr;
    uint4 wa = __ldg(wsrc0), wb = __ldg(wsrc0 + 1);
    if (b1) {
        const uint4 xa = __ldg(wsrc1), xb = __ldg(wsrc1 + 1);
        wa = make_uint4(wa.x + xa.x, wa.y + xa.y, wa.z + xa.z, wa.w + xa.w);
        wb = make_uint4(wb.x + xb.x, wb.y + xb.y, wb.z + xb.z, wb.w + xb.w);
    }
#pragma unroll 1
    for (int blk = 0; blk < kBlocks; blk++) {
        if (threadIdx.x == 0) {
            const int nx = blk + kKsStages - 1;
            if (nx < kBlocks) {
                const int s2 = nx % kKsStages;
                if (nx >= kKsStages) mbar_wait(&ks.empty[s2], ((nx / kKsStages) - 1) & 1);
                mbar_arrive_expect_tx(&ks.full[s2], kKsStageBytes);
                bulk_g2s(ks.tab[s2], tab_src + (size_t)nx * kKsStageBytes, kKsStageBytes, &ks.full[s2]);
            }
        }
        __syncwarp();
        const uint32_t v[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
        if (blk + 1 < kBlocks) {  // prefetch the next block's coefficients
            wa = __ldg(wsrc0 + 2 * blk + 2);
            wb = __ldg(wsrc0 + 2 * blk + 3);
            if (b1) {
                const uint4 xa = __ldg(wsrc1 + 2 * blk + 2), xb = __ldg(wsrc1 + 2 * blk + 3);
                wa = make_uint4(wa.x + xa.x, wa.y + xa.y, wa.z + xa.z, wa.w + xa.w);
                wb = make_uint4(wb.x + xb.x, wb.y + xb.y, wb.z + xb.z, wb.w + xb.w);
            }
        }
        const int s = blk % kKsStages;
        mbar_wait(&ks.full[s], (blk / kKsStages) & 1);
        const uint4 *tab = ks.tab[s];
#pragma unroll
        for (int ii = 0; ii < kKsIBlock; ii++) {
            const uint32_t word = (v[ii] + (1u << 15)) >> 16;
#pragma unroll
            for (int j = 0; j < kKsT; j++) {
                const uint32_t d = (word >> (14 - 2 * j)) & 3u;
                const uint4 *row = tab + ((ii * kKsT + j) * 4 + d) * 2;
                const uint4 lo = row[0], hi = row[1];
                acc[0] += lo.x; acc[1] += lo.y; acc[2] += lo.z; acc[3] += lo.w;
                acc[4] += hi.x; acc[5] += hi.y; acc[6] += hi.z; acc[7] += hi.w;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&ks.empty[s]);
    }
    if (!active) return;
    const int c0 = chunk * kKsCols;
    if (args.partial) {  // split sums, combined by k_keyswitch_reduce
        uint32_t *dst = args.partial + ((size_t)blockIdx.z * args.n_work + e) * kKskStride + c0;
#pragma unroll
        for (int c = 0; c < kKsCols; c++) dst[c] = acc[c];
        return;
    }
    uint32_t bval = 0;
    if (c0 + kKsCols > args.n) {
        bval = b0[kN];
        if (b1) bval += b1[kN] + it.cadd;
    }
    uint32_t *dst = args.pool + ((size_t)it.dst * lanes + lane_id) * args.pool_stride;
#pragma unroll
    for (int c = 0; c < kKsCols; c++) {
        const int col = c0 + c;
        if (col <= args.n) dst[col] = (col == args.n ? bval : 0u) - acc[c];
    }
}

// Narrow levels: out = (0.., b) - sum over the coefficient splits of k_keyswitch.
__global__ void __launch_bounds__(kKskStride) k_keyswitch_reduce(const KsArgs args, int splits) {
    const uint32_t e = blockIdx.x;
    const int col = threadIdx.x;
    if (col > args.n) return;
    const uint32_t lanes = args.lanes;
    const KsItem it = args.items[e / lanes];
    const uint32_t lane_id = e % lanes;
    uint32_t sum = 0;
    for (int sp = 0; sp < splits; sp++) sum += args.partial[((size_t)sp * args.n_work + e) * kKskStride + col];
    uint32_t bval = 0;
    if (col == args.n) {
        bval = args.big[((size_t)it.i0 * lanes + lane_id) * kBigStride + kN];
        if (it.i1 != 0xFFFFFFFFu) bval += args.big[((size_t)it.i1 * lanes + lane_id) * kBigStride + kN] + it.cadd;
    }
    args.pool[((size_t)it.dst * lanes + lane_id) * args.pool_stride + col] = bval - sum;
}

// FP64 roofline probe: 8 independent DFMA chains per thread.
__global__ void __launch_bounds__(256) k_dfma_peak(double *out, int iters, double b, double c) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = fma(a[k], b, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_gather(const uint32_t *__restrict__ pool, uint32_t stride, const uint32_t *__restrict__ slots,
                         uint32_t count, uint32_t words, uint32_t *__restrict__ out, size_t out_stride) {
    const uint32_t s = blockIdx.x;
    if (s >= count) return;
    const uint32_t *src = pool + (size_t)slots[s] * stride;
    for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) out[(size_t)s * out_stride + w] = src[w];
}

// KSK host layout [kN][t][3][n+1] -> device lookup table
// T[chunk][i][j][d][kKsCols] = KS[i][j][d] columns chunk*8 .. chunk*8+7 (d = 0 row is 0).
__global__ void k_ksk_relayout(const uint32_t *__restrict__ in, uint32_t *__restrict__ out, int n) {
    const size_t ij = blockIdx.x;  // i * t + j
    const uint32_t *src = in + ij * 3 * (size_t)(n + 1);
    for (int w = threadIdx.x; w < kKskStride * 4; w += blockDim.x) {
        const int d = w / kKskStride, col = w % kKskStride;
        const uint32_t val = (d == 0 || col > n) ? 0u : src[(size_t)(d - 1) * (n + 1) + col];
        const int chunk = col / kKsCols, cc = col % kKsCols;
        out[(((size_t)chunk * kN * kKsT + ij) * 4 + d) * kKsCols + cc] = val;
    }
}

constexpr int kBrGates = 4;  // bootstraps per CTA (64 threads each)

template <int G>
constexpr size_t br_smem_bytes() {
    return sizeof(BrSmem<G>);
}

}  // namespace

// Work items (blind rotations x lanes) per launch: bounds the extracted-LWE
// scratch (4,112 B per item) to ~4.3 GB for very wide levels.
constexpr size_t kMaxWorkPerLaunch = (size_t)1 << 20;

// ---------------------------------------------------------------------------
// engine object
// ---------------------------------------------------------------------------
struct hb_engine {
    int device = 0;
    hb_params p{};
    cudaStream_t stream = nullptr;
    cudaStream_t h2d_stream = nullptr;    // async uploads overlapping the compute stream
    cudaStream_t d2h_stream = nullptr;    // async downloads
    cudaEvent_t ev_upload = nullptr;      // last async upload (the next level waits on it)
    cudaEvent_t ev_compute = nullptr;     // compute point an async download waits on
    cudaEvent_t ev_prev_level = nullptr;  // compute stream before the most recent level
    bool pending_upload = false;
    double2 *d_W = nullptr, *d_TW = nullptr, *d_PSI = nullptr;
    int unroll = 1;  // bk_unroll of the loaded key
    double2 *d_bkf = nullptr;
    uint32_t *d_ksk = nullptr;
    uint32_t *d_pool = nullptr;
    size_t pool_cap = 0;
    uint32_t pool_stride = 0;
    uint32_t *d_big = nullptr;
    size_t big_cap = 0;  // extracted-LWE slots
    BrItem *d_br = nullptr;
    size_t br_cap = 0;
    KsItem *d_ks = nullptr;
    size_t ks_cap = 0;
    uint32_t *d_tmp = nullptr;
    size_t tmp_cap = 0;  // words
    uint32_t *d_kspart = nullptr;
    size_t kspart_cap = 0;  // words: narrow-level key-switch partial sums
    void *h_stage = nullptr;
    size_t h_stage_cap = 0;
    unsigned long long *d_margin = nullptr;
    void *d_flush = nullptr;
    size_t flush_bytes = 0;
    uint64_t flush_gen = 1;
    cudaEvent_t ev[4]{};
    cudaEvent_t ev_stage = nullptr;  // item copies out of h_stage done
    uint64_t n_br = 0, n_ks = 0, n_launch = 0;
    int num_sms = 148;
    size_t max_work = kMaxWorkPerLaunch;  // HEBNN_B200_MAX_WORK overrides (tests)
    bool latency_mode = true;             // HEBNN_B200_LATENCY_MODE=0 disables (A/B tests)
    bool cluster_mode = true;             // 2-CTA clusters for <= #SM/2 key-pair bootstraps (HEBNN_B200_CLUSTER_MODE=0)
};

namespace {

int ensure_dev(void **ptr, size_t *cap, size_t need, size_t elem, bool preserve, cudaStream_t st) {
    if (need <= *cap) return HB_OK;
    size_t ncap = std::max(need, *cap + *cap / 2);
    void *np = nullptr;
    cudaError_t err = cudaMalloc(&np, ncap * elem);
    if (err != cudaSuccess) {
        set_error(std::string("cudaMalloc(") + std::to_string(ncap * elem) + " B): " + cudaGetErrorString(err));
        return HB_ENOMEM;
    }
    if (*ptr) {
        if (preserve && *cap) {
            HB_CUDA_TRY(cudaMemcpyAsync(np, *ptr, *cap * elem, cudaMemcpyDeviceToDevice, st));
            HB_CUDA_TRY(cudaStreamSynchronize(st));
        }
        cudaFree(*ptr);
    }
    *ptr = np;
    *cap = ncap;
    return HB_OK;
}

int ensure_host_stage(hb_engine *e, size_t bytes) {
    if (bytes <= e->h_stage_cap) return HB_OK;
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (e->h_stage) cudaFreeHost(e->h_stage);
    size_t ncap = std::max(bytes, e->h_stage_cap * 2);
    HB_CUDA_TRY(cudaHostAlloc(&e->h_stage, ncap, cudaHostAllocDefault));
    e->h_stage_cap = ncap;
    return HB_OK;
}

template <int G, bool kDebug>
int launch_br(hb_engine *e, const BrArgs &a) {
    const size_t smem = br_smem_bytes<G>();
    const unsigned grid = (a.n_work + G - 1) / G;
    k_blind_rotate<G, kDebug><<<grid, 64 * G, smem, e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    return HB_OK;
}

template <int G, bool kDebug, int R = kStagesU2, int MB = 1, bool TM = false>
int launch_br_u2(hb_engine *e, const BrArgs &a) {
    const unsigned grid = (a.n_work + G - 1) / G;
    k_blind_rotate_u2<G, kDebug, R, MB, TM><<<grid, 64 * G, sizeof(BrSmemU2<G, R, TM>), e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    return HB_OK;
}

template <bool kDebug>
int launch_br_lat(hb_engine *e, const BrArgs &a) {
    k_blind_rotate_lat<kDebug><<<a.n_work, 192, sizeof(BrLatSmem), e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    return HB_OK;
}

// narrow levels (<= kKsNarrow key switches): the coefficient range is split
// over kKsSplits CTAs per column chunk and the partial sums are reduced
constexpr uint32_t kKsNarrow = 32;
constexpr int kKsSplits = 8;

int launch_ks(hb_engine *e, const KsArgs &a0) {
    KsArgs a = a0;
    const bool narrow = a.n_work <= kKsNarrow;
    if (narrow) {
        int rc = ensure_dev((void **)&e->d_kspart, &e->kspart_cap, (size_t)kKsSplits * a.n_work * kKskStride,
                            sizeof(uint32_t), false, e->stream);
        if (rc) return rc;
        a.partial = e->d_kspart;
    }
    const dim3 grid((a.n_work + kKsThreads - 1) / kKsThreads, kKsChunks, narrow ? kKsSplits : 1);
    k_keyswitch<<<grid, kKsThreads, 0, e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    if (narrow) {
        k_keyswitch_reduce<<<a.n_work, kKskStride, 0, e->stream>>>(a, kKsSplits);
        HB_CUDA_TRY(cudaGetLastError());
        e->n_launch++;
    }
    return HB_OK;
}

#ifndef HB_U2_PAIRED
#define HB_U2_PAIRED 0  // experiment: wide levels as two independent 2-gate CTAs per SM
#endif
#ifndef HB_PAIRED_RING
#define HB_PAIRED_RING 3
#endif
constexpr int kPairedRing = HB_PAIRED_RING;
#ifndef HB_U2_TMEM
#define HB_U2_TMEM 0  // wide key-pair levels: accumulators in tensor memory, deeper BK ring
#endif
#ifndef HB_TMEM_RING
#define HB_TMEM_RING 9
#endif
constexpr int kStagesU2Tmem = HB_TMEM_RING;

// Blind-rotation launch for a level of a.n_work bootstraps: narrow levels
// (latency-bound) get one bootstrap per CTA split over three thread groups
// (latency mode) or fewer bootstraps per CTA; wide levels 4 per CTA.
// force_g (debug paths): 4 = the throughput kernel regardless of width.
template <bool kDebug>
int launch_br_auto(hb_engine *e, const BrArgs &a, int force_g = 0) {
    const uint32_t sms = (uint32_t)e->num_sms;
    const int gsel = force_g ? force_g : (a.n_work <= sms ? 1 : (a.n_work <= 2u * sms ? 2 : kBrGates));
    if (e->unroll == 2) {
        if (!force_g && e->latency_mode && e->cluster_mode && 2 * a.n_work <= sms) {
            k_blind_rotate_u2_clu<kDebug><<<2 * a.n_work, 192, sizeof(BrCluSmemU2), e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
        if (!force_g && gsel == 1 && e->latency_mode) {
            k_blind_rotate_u2_lat<kDebug><<<a.n_work, 192, sizeof(BrLatSmemU2), e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
        if (gsel == 1) return launch_br_u2<1, kDebug>(e, a);
        if (gsel == 2) return launch_br_u2<2, kDebug>(e, a);
#if HB_U2_PAIRED
        if (!force_g) return launch_br_u2<2, kDebug, kPairedRing, 2>(e, a);  // two 2-gate CTAs per SM
#endif
#if HB_U2_TMEM
        return launch_br_u2<kBrGates, kDebug, kStagesU2Tmem, 1, true>(e, a);
#else
        return launch_br_u2<kBrGates, kDebug>(e, a);
#endif
    }
    if (!force_g && gsel == 1 && e->latency_mode) return launch_br_lat<kDebug>(e, a);
    if (gsel == 1) return launch_br<1, kDebug>(e, a);
    if (gsel == 2) return launch_br<2, kDebug>(e, a);
    return launch_br<kBrGates, kDebug>(e, a);
}

BrArgs br_args(hb_engine *e) {
    BrArgs a{};
    a.pool = e->d_pool;
    a.pool_stride = e->pool_stride;
    a.lanes = 1;
    a.n = e->p.n;
    a.mu = 1u << 29;
    a.bkf = e->d_bkf;
    a.big = e->d_big;
    a.W = e->d_W;
    a.TW = e->d_TW;
    a.PSI = e->d_PSI;
    a.iters = e->p.n;
    return a;
}

int32_t pack_coef(int alpha, int beta, int gamma = 0) {
    return (int32_t)((uint32_t)(uint8_t)(int8_t)alpha | ((uint32_t)(uint8_t)(int8_t)beta << 8) |
                     ((uint32_t)(uint8_t)(int8_t)gamma << 16));
}

}  // namespace

extern "C" {

int hb_engine_create(int device, const hb_params *p, const uint32_t *bk, const uint32_t *ksk, hb_engine **out) {
    if (!out || !params_ok(p) || !bk || !ksk) {
        set_error("hb_engine_create: unsupported parameters or null argument");
        return HB_EINVAL;
    }
    *out = nullptr;
    int ndev = 0;
    HB_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) {
        set_error("hb_engine_create: CUDA device " + std::to_string(device) + " not present (" +
                  std::to_string(ndev) + " visible)");
        return HB_ECUDA;
    }
    HB_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    HB_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error("hb_engine_create: kernels are built for sm_100a (B200); device is sm_" +
                  std::to_string(prop.major) + std::to_string(prop.minor));
        return HB_ECUDA;
    }
    hb_engine *e = new hb_engine();
    e->device = device;
    e->p = *p;
    e->pool_stride = (uint32_t)((p->n + 1 + 3) & ~3);
    HB_CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    for (auto &ev : e->ev) HB_CUDA_TRY(cudaEventCreate(&ev));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_stage, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaStreamCreateWithFlags(&e->h2d_stream, cudaStreamNonBlocking));
    HB_CUDA_TRY(cudaStreamCreateWithFlags(&e->d2h_stream, cudaStreamNonBlocking));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_upload, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_compute, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_prev_level, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventRecord(e->ev_prev_level, e->stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_stage, e->stream));

    // twiddle tables, computed in long double then rounded
    std::vector<double2> W(kNH), TW(kNH);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int j = 0; j < kNH; j++) {
        long double th = 2.0L * pi * j / kNH;
        W[j] = make_double2((double)cosl(th), (double)sinl(th));
        long double ph = pi * j / kN;
        TW[j] = make_double2((double)cosl(ph), (double)sinl(ph));
    }
    std::vector<double2> PSI(2 * kN);
    for (int u = 0; u < 2 * kN; u++) {
        long double ph = pi * u / kN;
        PSI[u] = make_double2((double)cosl(ph), (double)sinl(ph));
    }
    HB_CUDA_TRY(cudaMalloc(&e->d_PSI, 2 * kN * sizeof(double2)));
    HB_CUDA_TRY(cudaMemcpy(e->d_PSI, PSI.data(), 2 * kN * sizeof(double2), cudaMemcpyHostToDevice));
    e->unroll = bk_unroll(p);
    HB_CUDA_TRY(cudaMalloc(&e->d_W, kNH * sizeof(double2)));
    HB_CUDA_TRY(cudaMalloc(&e->d_TW, kNH * sizeof(double2)));
    HB_CUDA_TRY(cudaMemcpy(e->d_W, W.data(), kNH * sizeof(double2), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMemcpy(e->d_TW, TW.data(), kNH * sizeof(double2), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMalloc(&e->d_margin, sizeof(unsigned long long)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<kBrGates, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<kBrGates>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<2>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<1>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<kBrGates, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<kBrGates>()));
#if HB_U2_TMEM
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, false, kStagesU2Tmem, 1, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates, kStagesU2Tmem, true>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, true, kStagesU2Tmem, 1, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates, kStagesU2Tmem, true>)));
#endif
#if HB_U2_PAIRED
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, false, kPairedRing, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<2, kPairedRing>)));
#endif
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<2>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<1>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<2>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<1>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<2>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<1>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_clu<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrCluSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_clu<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrCluSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_lat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_lat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_lat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmem)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_lat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmem)));
    HB_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    e->num_sms = prop.multiProcessorCount;
    if (const char *mw = std::getenv("HEBNN_B200_MAX_WORK")) e->max_work = std::max<size_t>(2, std::strtoull(mw, nullptr, 10));
    if (const char *lm = std::getenv("HEBNN_B200_LATENCY_MODE")) e->latency_mode = std::atoi(lm) != 0;
    if (const char *cm = std::getenv("HEBNN_B200_CLUSTER_MODE")) e->cluster_mode = std::atoi(cm) != 0;

    // BK -> Fourier
    const size_t npoly = bk_tgsw_count(p) * kRows * 2;
    uint32_t *d_bk = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_bk, npoly * kN * sizeof(uint32_t)));
    HB_CUDA_TRY(cudaMemcpy(d_bk, bk, npoly * kN * sizeof(uint32_t), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMalloc(&e->d_bkf, npoly * kNH * sizeof(double2)));
    k_bk_to_fourier<<<(unsigned)((npoly + 1) / 2), 128, 0, e->stream>>>(d_bk, e->d_bkf, (int)npoly, e->d_W, e->d_TW,
                                                                         e->unroll);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    cudaFree(d_bk);

    // KSK
    const size_t ksk_rows = (size_t)kN * kKsT * kKsVals;
    uint32_t *d_kin = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_kin, ksk_rows * (p->n + 1) * sizeof(uint32_t)));
    HB_CUDA_TRY(cudaMemcpy(d_kin, ksk, ksk_rows * (p->n + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMalloc(&e->d_ksk, kKsTableWords * sizeof(uint32_t)));
    k_ksk_relayout<<<(unsigned)(ksk_rows / kKsVals), 256, 0, e->stream>>>(d_kin, e->d_ksk, p->n);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    cudaFree(d_kin);
    *out = e;
    return HB_OK;
}

int hb_engine_destroy(hb_engine *e) {
    if (!e) return HB_OK;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (void *ptr : {(void *)e->d_W, (void *)e->d_TW, (void *)e->d_PSI, (void *)e->d_bkf, (void *)e->d_ksk, (void *)e->d_pool,
                      (void *)e->d_big, (void *)e->d_br, (void *)e->d_ks, (void *)e->d_tmp, (void *)e->d_kspart, (void *)e->d_margin,
                      e->d_flush})
        if (ptr) cudaFree(ptr);
    if (e->h_stage) cudaFreeHost(e->h_stage);
    for (auto &ev : e->ev)
        if (ev) cudaEventDestroy(ev);
    if (e->ev_stage) cudaEventDestroy(e->ev_stage);
    for (cudaStream_t st : {e->h2d_stream, e->d2h_stream})
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    for (cudaEvent_t ev : {e->ev_upload, e->ev_compute, e->ev_prev_level})
        if (ev) cudaEventDestroy(ev);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
    return HB_OK;
}

int hb_pool_reserve(hb_engine *e, size_t slots) {
    if (!e) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    size_t cap_words = e->pool_cap * e->pool_stride;
    int rc = ensure_dev((void **)&e->d_pool, &cap_words, slots * e->pool_stride, sizeof(uint32_t), true, e->stream);
    if (rc) return rc;
    e->pool_cap = cap_words / e->pool_stride;
    return HB_OK;
}

size_t hb_pool_capacity(const hb_engine *e) { return e ? e->pool_cap : 0; }
size_t hb_pool_stride(const hb_engine *e) { return e ? e->pool_stride : 0; }

int hb_pool_upload(hb_engine *e, size_t first, size_t count, const uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_upload: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_pool + first * e->pool_stride, e->pool_stride * 4, host, host_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyHostToDevice, e->stream));
    return HB_OK;
}

int hb_pool_download(hb_engine *e, size_t first, size_t count, uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_download: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaMemcpy2DAsync(host, host_stride * 4, e->d_pool + first * e->pool_stride, e->pool_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_pool_gather_device(hb_engine *e, const uint32_t *slots, size_t count, uint32_t *dev_out, size_t dev_stride) {
    if (!e || (count && (!slots || !dev_out)) || dev_stride < (size_t)e->p.n + 1) {
        set_error("hb_pool_gather_device: bad arguments");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    for (size_t i = 0; i < count; i++)
        if (slots[i] >= e->pool_cap) {
            set_error("hb_pool_gather_device: slot beyond pool capacity");
            return HB_EINVAL;
        }
    HB_CUDA_TRY(cudaSetDevice(e->device));
    int rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, count, sizeof(uint32_t), false, e->stream);
    if (rc) return rc;
    rc = ensure_host_stage(e, count * sizeof(uint32_t));
    if (rc) return rc;
    HB_CUDA_TRY(cudaEventSynchronize(e->ev_stage));
    std::memcpy(e->h_stage, slots, count * sizeof(uint32_t));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_tmp, e->h_stage, count * sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
    k_gather<<<(unsigned)count, 256, 0, e->stream>>>(e->d_pool, e->pool_stride, e->d_tmp, (uint32_t)count,
                                                    (uint32_t)e->p.n + 1, dev_out, dev_stride);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    e->n_launch++;
    return HB_OK;
}

int hb_pool_put_device(hb_engine *e, size_t first_slot, size_t count, const uint32_t *dev_in, size_t dev_stride) {
    if (!e || (count && !dev_in) || dev_stride < (size_t)e->p.n + 1 || first_slot + count > e->pool_cap) {
        set_error("hb_pool_put_device: bad arguments or slots beyond pool capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_pool + first_slot * e->pool_stride, (size_t)e->pool_stride * 4, dev_in,
                                  dev_stride * 4, ((size_t)e->p.n + 1) * 4, count, cudaMemcpyDeviceToDevice, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_pool_gather(hb_engine *e, const uint32_t *slots, size_t count, uint32_t *host, size_t host_stride) {
    if (!e || (count && (!slots || !host)) || host_stride < (size_t)e->p.n + 1) {
        set_error("hb_pool_gather: bad arguments");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    for (size_t i = 0; i < count; i++)
        if (slots[i] >= e->pool_cap) {
            set_error("hb_pool_gather: slot beyond pool capacity");
            return HB_EINVAL;
        }
    HB_CUDA_TRY(cudaSetDevice(e->device));
    const uint32_t words = (uint32_t)e->p.n + 1;
    const size_t need = count + (count * words + 3) / 1;
    int rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, need, sizeof(uint32_t), false, e->stream);
    if (rc) return rc;
    rc = ensure_host_stage(e, count * sizeof(uint32_t));
    if (rc) return rc;
    HB_CUDA_TRY(cudaEventSynchronize(e->ev_stage));
    std::memcpy(e->h_stage, slots, count * sizeof(uint32_t));
    uint32_t *d_slots = e->d_tmp, *d_out = e->d_tmp + count;
    HB_CUDA_TRY(cudaMemcpyAsync(d_slots, e->h_stage, count * sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
    k_gather<<<(unsigned)count, 256, 0, e->stream>>>(e->d_pool, e->pool_stride, d_slots, (uint32_t)count, words, d_out,
                                                    words);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaMemcpy2DAsync(host, host_stride * 4, d_out, (size_t)words * 4, (size_t)words * 4, count,
                                  cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    e->n_launch++;
    return HB_OK;
}

static int run_gates_chunk(hb_engine *e, const hb_gate *gates, size_t n, uint32_t lanes);

int hb_run_gates(hb_engine *e, const hb_gate *gates, size_t n, uint32_t lanes) {
    if (!e || (n && !gates) || lanes == 0) {
        set_error("hb_run_gates: bad arguments");
        return HB_EINVAL;
    }
    if (!n) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    // gates of one level are independent: split very wide levels into chunks
    const size_t per_chunk = std::max<size_t>(1, e->max_work / (2 * (size_t)lanes));
    nvtxRangePushA("hb_run_gates");  // NVTX range per level (visible in nsys timelines)
    for (size_t off = 0; off < n; off += per_chunk) {
        const int rc = run_gates_chunk(e, gates + off, std::min(per_chunk, n - off), lanes);
        if (rc) {
            nvtxRangePop();
            return rc;
        }
    }
    nvtxRangePop();
    return HB_OK;
}

static int run_gates_chunk(hb_engine *e, const hb_gate *gates, size_t n, uint32_t lanes) {
    // expand records into blind-rotation and key-switch work items
    size_t nbr = 0;
    for (size_t i = 0; i < n; i++) {
        const hb_gate &g = gates[i];
        if (g.kind != HB_GATE_LIN2 && g.kind != HB_GATE_MUX && g.kind != HB_GATE_LIN3) {
            set_error("hb_run_gates: unknown gate kind " + std::to_string((int)g.kind));
            return HB_EINVAL;
        }
        const size_t top = (size_t)std::max(std::max(g.dst, g.src_a), std::max(g.src_b, g.src_c)) + 1;
        if (top * lanes > e->pool_cap) {
            set_error("hb_run_gates: slot beyond pool capacity");
            return HB_EINVAL;
        }
        nbr += (g.kind == HB_GATE_MUX) ? 2 : 1;
    }
    const size_t br_bytes = nbr * sizeof(BrItem), ks_bytes = n * sizeof(KsItem);
    int rc = ensure_host_stage(e, br_bytes + ks_bytes);
    if (rc) return rc;
    // the pinned stage fed the previous level's item copies; wait for those copies only,
    // so the host builds level k+1 while the device still runs level k
    HB_CUDA_TRY(cudaEventSynchronize(e->ev_stage));
    BrItem *hbr = reinterpret_cast<BrItem *>(e->h_stage);
    KsItem *hks = reinterpret_cast<KsItem *>(reinterpret_cast<char *>(e->h_stage) + br_bytes);
    size_t b = 0;
    const uint32_t eighth = 1u << 29;
    for (size_t i = 0; i < n; i++) {
        const hb_gate &g = gates[i];
        if (g.kind == HB_GATE_LIN2) {
            hbr[b] = BrItem{g.src_a, g.src_b, g.src_a, g.c0, pack_coef(g.alpha, g.beta)};
            hks[i] = KsItem{g.dst, (uint32_t)b, 0xFFFFFFFFu, 0u};
            b += 1;
        } else if (g.kind == HB_GATE_LIN3) {
            hbr[b] = BrItem{g.src_a, g.src_b, g.src_c, g.c0, pack_coef(g.alpha, g.beta, g.gamma)};
            hks[i] = KsItem{g.dst, (uint32_t)b, 0xFFFFFFFFu, 0u};
            b += 1;
        } else {
            hbr[b] = BrItem{g.src_a, g.src_b, g.src_a, 0u - eighth, pack_coef(1, g.alpha)};
            hbr[b + 1] = BrItem{g.src_a, g.src_c, g.src_a, 0u - eighth, pack_coef(-1, g.beta)};
            hks[i] = KsItem{g.dst, (uint32_t)b, (uint32_t)(b + 1), eighth};
            b += 2;
        }
    }
    if ((rc = ensure_dev((void **)&e->d_br, &e->br_cap, nbr, sizeof(BrItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_ks, &e->ks_cap, n, sizeof(KsItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, nbr * lanes * kBigStride, sizeof(uint32_t), false,
                         e->stream)))
        return rc;
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_br, hbr, br_bytes, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_ks, hks, ks_bytes, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_stage, e->stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_prev_level, e->stream));  // "everything before this level"
    if (e->pending_upload) {  // inputs staged by hb_pool_upload_async
        HB_CUDA_TRY(cudaStreamWaitEvent(e->stream, e->ev_upload, 0));
        e->pending_upload = false;
    }

    BrArgs a = br_args(e);
    a.lanes = lanes;
    a.items = e->d_br;
    a.n_work = (uint32_t)(nbr * lanes);
    HB_CUDA_TRY(cudaEventRecord(e->ev[0], e->stream));
    if ((rc = launch_br_auto<false>(e, a))) return rc;
    HB_CUDA_TRY(cudaEventRecord(e->ev[1], e->stream));
    KsArgs k{};
    k.big = e->d_big;
    k.items = e->d_ks;
    k.lanes = lanes;
    k.n_work = (uint32_t)(n * lanes);
    k.ksk = e->d_ksk;
    k.pool = e->d_pool;
    k.pool_stride = e->pool_stride;
    k.n = e->p.n;
    if ((rc = launch_ks(e, k))) return rc;
    HB_CUDA_TRY(cudaEventRecord(e->ev[2], e->stream));
    e->n_br += nbr * lanes;
    e->n_ks += n * lanes;
    return HB_OK;
}

int hb_sync(hb_engine *e) {
    if (!e) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->h2d_stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->d2h_stream));
    return HB_OK;
}

int hb_pool_upload_async(hb_engine *e, size_t first, size_t count, const uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_upload_async: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    // may overlap the most recently issued level, never an earlier one (double buffering)
    HB_CUDA_TRY(cudaStreamWaitEvent(e->h2d_stream, e->ev_prev_level, 0));
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_pool + first * e->pool_stride, e->pool_stride * 4, host, host_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyHostToDevice, e->h2d_stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_upload, e->h2d_stream));
    e->pending_upload = true;
    return HB_OK;
}

int hb_pool_download_async(hb_engine *e, size_t first, size_t count, uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_download_async: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    // everything issued so far on the compute stream (the levels producing these slots)
    HB_CUDA_TRY(cudaEventRecord(e->ev_compute, e->stream));
    HB_CUDA_TRY(cudaStreamWaitEvent(e->d2h_stream, e->ev_compute, 0));
    HB_CUDA_TRY(cudaMemcpy2DAsync(host, host_stride * 4, e->d_pool + first * e->pool_stride, e->pool_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyDeviceToHost, e->d2h_stream));
    return HB_OK;
}

int hb_last_timing(hb_engine *e, float *br_ms, float *ks_ms) {
    if (!e) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaEventSynchronize(e->ev[2]));
    float x = 0, y = 0;
    HB_CUDA_TRY(cudaEventElapsedTime(&x, e->ev[0], e->ev[1]));
    HB_CUDA_TRY(cudaEventElapsedTime(&y, e->ev[1], e->ev[2]));
    if (br_ms) *br_ms = x;
    if (ks_ms) *ks_ms = y;
    return HB_OK;
}

int hb_counters(hb_engine *e, uint64_t *brs, uint64_t *kss, uint64_t *launches) {
    if (!e) return HB_EINVAL;
    if (brs) *brs = e->n_br;
    if (kss) *kss = e->n_ks;
    if (launches) *launches = e->n_launch;
    return HB_OK;
}

int hb_debug_blind_rotate(hb_engine *e, const uint32_t *lwe, uint32_t mu, int32_t iters, uint32_t *acc_out) {
    if (!e || !lwe || !acc_out) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    const size_t words = e->p.n + 1;
    int rc;
    if ((rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, 2 * words + 4 * kN + 64, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_br, &e->br_cap, 1, sizeof(BrItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, kBigStride, sizeof(uint32_t), false, e->stream))) return rc;
    uint32_t *d_in = e->d_tmp, *d_acc = e->d_tmp + ((2 * words + 3) & ~size_t(3));
    BrItem it{0, 0, 0, 0, pack_coef(1, 0)};
    HB_CUDA_TRY(cudaMemcpyAsync(d_in, lwe, words * 4, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_br, &it, sizeof it, cudaMemcpyHostToDevice, e->stream));
    BrArgs a = br_args(e);
    a.pool = d_in;
    a.pool_stride = (uint32_t)words;
    a.items = e->d_br;
    a.n_work = 1;
    a.mu = mu;
    if (iters >= 100000) {  // debug A/B: BK rows read from global instead of the ring
        iters -= 100000;
        a.n_work = 2;
        a.lanes = 2;
    }
    a.iters = iters < 0 ? e->p.n : iters;
    a.acc_dump = d_acc;
    if ((rc = launch_br_auto<true>(e, a, kBrGates))) return rc;
    HB_CUDA_TRY(cudaMemcpyAsync(acc_out, d_acc, 2 * kN * 4, cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_debug_bootstrap_wo_ks(hb_engine *e, const uint32_t *lin, size_t count, uint32_t *out) {
    if (!e || (count && (!lin || !out))) return HB_EINVAL;
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    const size_t words = e->p.n + 1;
    int rc;
    if ((rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, count * words, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_br, &e->br_cap, count, sizeof(BrItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, count * kBigStride, sizeof(uint32_t), false, e->stream)))
        return rc;
    std::vector<BrItem> items(count);
    for (size_t i = 0; i < count; i++) items[i] = BrItem{(uint32_t)i, (uint32_t)i, (uint32_t)i, 0u, pack_coef(1, 0)};
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_tmp, lin, count * words * 4, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_br, items.data(), count * sizeof(BrItem), cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemsetAsync(e->d_margin, 0, sizeof(unsigned long long), e->stream));
    BrArgs a = br_args(e);
    a.pool = e->d_tmp;
    a.pool_stride = (uint32_t)words;
    a.items = e->d_br;
    a.n_work = (uint32_t)count;
    a.margin = e->d_margin;
    if ((rc = launch_br_auto<true>(e, a, kBrGates))) return rc;
    HB_CUDA_TRY(cudaMemcpy2DAsync(out, (size_t)(kN + 1) * 4, e->d_big, kBigStride * 4, (size_t)(kN + 1) * 4, count,
                                  cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_flush_l2(hb_engine *e, size_t bytes) {
    if (!e) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    if (!bytes) bytes = (size_t)256 << 20;
    if (bytes > e->flush_bytes) {
        if (e->d_flush) cudaFree(e->d_flush);
        e->d_flush = nullptr;
        HB_CUDA_TRY(cudaMalloc(&e->d_flush, bytes));
        e->flush_bytes = bytes;
    }
    HB_CUDA_TRY(cudaMemsetAsync(e->d_flush, (int)(e->flush_gen++ & 0xFF), bytes, e->stream));
    return HB_OK;
}

int hb_measure_fp64_peak(hb_engine *e, double *tflops) {
    if (!e || !tflops) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    cudaDeviceProp prop;
    HB_CUDA_TRY(cudaGetDeviceProperties(&prop, e->device));
    double *d_out = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_out, sizeof(double)));
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    k_dfma_peak<<<blocks, threads, 0, e->stream>>>(d_out, iters, 0.999999, 1e-7);  // warm-up
    HB_CUDA_TRY(cudaEventRecord(e->ev[0], e->stream));
    for (int r = 0; r < 5; r++) k_dfma_peak<<<blocks, threads, 0, e->stream>>>(d_out, iters, 0.999999, 1e-7);
    HB_CUDA_TRY(cudaEventRecord(e->ev[1], e->stream));
    HB_CUDA_TRY(cudaEventSynchronize(e->ev[1]));
    float ms = 0;
    HB_CUDA_TRY(cudaEventElapsedTime(&ms, e->ev[0], e->ev[1]));
    cudaFree(d_out);
    *tflops = 5.0 * 2.0 * 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
    return HB_OK;
}

int hb_debug_fourier(hb_engine *e, const uint32_t *polys, size_t count, double *out, int which) {
    if (!e || (count && (!polys || !out))) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    if (which == 1) {  // download rows of the device BK Fourier table
        HB_CUDA_TRY(cudaMemcpy(out, e->d_bkf, count * kNH * sizeof(double2), cudaMemcpyDeviceToHost));
        return HB_OK;
    }
    uint32_t *d_in = nullptr;
    double2 *d_out = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_in, count * kN * 4));
    HB_CUDA_TRY(cudaMalloc(&d_out, count * kNH * sizeof(double2)));
    HB_CUDA_TRY(cudaMemcpy(d_in, polys, count * kN * 4, cudaMemcpyHostToDevice));
    k_bk_to_fourier<<<(unsigned)((count + 1) / 2), 128, 0, e->stream>>>(d_in, d_out, (int)count, e->d_W, e->d_TW, 1);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    HB_CUDA_TRY(cudaMemcpy(out, d_out, count * kNH * sizeof(double2), cudaMemcpyDeviceToHost));
    cudaFree(d_in);
    cudaFree(d_out);
    return HB_OK;
}

int hb_debug_fft_margin(hb_engine *e, double *max_err) {
    if (!e || !max_err) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    unsigned long long bits = 0;
    HB_CUDA_TRY(cudaMemcpy(&bits, e->d_margin, sizeof bits, cudaMemcpyDeviceToHost));
    std::memcpy(max_err, &bits, sizeof(double));
    return HB_OK;
}

int hb_debug_keyswitch(hb_engine *e, const uint32_t *in, size_t count, uint32_t *out) {
    if (!e || (count && (!in || !out))) return HB_EINVAL;
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    int rc;
    const size_t words = e->p.n + 1;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, count * kBigStride, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, count * e->pool_stride, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_ks, &e->ks_cap, count, sizeof(KsItem), false, e->stream))) return rc;
    std::vector<KsItem> items(count);
    for (size_t i = 0; i < count; i++) items[i] = KsItem{(uint32_t)i, (uint32_t)i, 0xFFFFFFFFu, 0u};
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_big, kBigStride * 4, in, (size_t)(kN + 1) * 4, (size_t)(kN + 1) * 4, count,
                                  cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_ks, items.data(), count * sizeof(KsItem), cudaMemcpyHostToDevice, e->stream));
    KsArgs k{};
    k.big = e->d_big;
    k.items = e->d_ks;
    k.lanes = 1;
    k.n_work = (uint32_t)count;
    k.ksk = e->d_ksk;
    k.pool = e->d_tmp;
    k.pool_stride = e->pool_stride;
    k.n = e->p.n;
    if ((rc = launch_ks(e, k))) return rc;
    HB_CUDA_TRY(cudaMemcpy2DAsync(out, words * 4, e->d_tmp, e->pool_stride * 4, words * 4, count,
                                  cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

}  // extern "C"
