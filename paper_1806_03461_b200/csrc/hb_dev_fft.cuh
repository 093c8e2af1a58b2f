// hb_dev_fft.cuh: FP64 negacyclic FFT, digit/torus conversions, mbarrier and bulk-copy primitives
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once


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
// The two w8 = (1+i)/sqrt2 twiddles of the first radix-2 stage are carried
// unscaled through the second stage and applied by the FMAs of the third
// (x4 +- r (u + v)): 52 FP64 instructions instead of 56.
__device__ __forceinline__ void dft8(double2 (&x)[8]) {
    const double r = 0.70710678118654752440;
    // stage 1: a_m = x_m + x_{m+4}; odd branch b_m = (x_m - x_{m+4}) w8^m, b_1 and b_3 left unscaled by r
    double2 b[4];
#pragma unroll
    for (int m = 0; m < 4; m++) {
        const double2 a = x[m], c = x[m + 4];
        x[m] = cadd(a, c);
        b[m] = csub(a, c);
    }
    const double2 b1 = make_double2(b[1].x - b[1].y, b[1].x + b[1].y);     // sqrt2 * b_1 w8
    const double2 b3 = make_double2(-b[3].x - b[3].y, b[3].x - b[3].y);    // sqrt2 * b_3 w8^3
    const double2 b2 = make_double2(-b[2].y, b[2].x);                       // b_2 * i
    // stage 2, even half (x[0..3]) and odd half (b0, b1, b2, b3)
#pragma unroll
    for (int m = 0; m < 2; m++) {
        const double2 a = x[m], c = x[m + 2];
        x[m] = cadd(a, c);
        const double2 d = csub(a, c);
        x[m + 2] = (m == 0) ? d : make_double2(-d.y, d.x);
    }
    const double2 e0 = cadd(b[0], b2), e2 = csub(b[0], b2);
    const double2 s5 = cadd(b1, b3), d7 = csub(b1, b3);
    const double2 s7 = make_double2(-d7.y, d7.x);                           // (b1 - b3) * i, still unscaled
    // stage 3
#pragma unroll
    for (int h = 0; h < 4; h += 2) {
        const double2 a = x[h], c = x[h + 1];
        x[h] = cadd(a, c);
        x[h + 1] = csub(a, c);
    }
    x[4] = make_double2(fma(r, s5.x, e0.x), fma(r, s5.y, e0.y));
    x[5] = make_double2(fma(-r, s5.x, e0.x), fma(-r, s5.y, e0.y));
    x[6] = make_double2(fma(r, s7.x, e2.x), fma(r, s7.y, e2.y));
    x[7] = make_double2(fma(-r, s7.x, e2.x), fma(-r, s7.y, e2.y));
}

__device__ __forceinline__ constexpr int rev3(int k) { return ((k & 1) << 2) | (k & 2) | ((k >> 2) & 1); }

__device__ __forceinline__ void group_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(64) : "memory");
}
// named barrier over kBT threads (the warps of one transform group)
template <int kBT>
__device__ __forceinline__ void group_bar_n(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kBT) : "memory");
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
template <int NP, bool kSB = false, int kBT = 64>
__device__ __forceinline__ void nega_fft_fwd_n(double2 (&x)[NP][8], double2 *xch, int t, const TwSeeds &tw,
                                               int bar_id) {
    constexpr int kB0 = kSB ? 1 : 2, kB1 = kSB ? 0 : 1;  // buffer q of exchange 1 / 2: q * kB0 + kB1 * (..)
#pragma unroll
    for (int q = 0; q < NP; q++) {
#pragma unroll
        for (int m = 1; m < 8; m++) x[q][m] = cmul(x[q][m], c16(m));
        dft8(x[q]);
    }
    if (kSB) group_bar_n<kBT>(bar_id);  // previous transform's readers are done
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
    if (HB_EXP_SKIP & 64) __syncwarp(); else group_bar_n<kBT>(bar_id);
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
            group_bar_n<kBT>(bar_id);
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
    if (HB_EXP_SKIP & 32) __syncwarp(); else group_bar_n<kBT>(bar_id);
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

template <int NP, bool kSB = false, int kBT = 64>
__device__ __forceinline__ void nega_fft_inv_n(double2 (&x)[NP][8], double2 *xch, int t, const TwSeeds &tw,
                                               int bar_id) {
    constexpr int kB0 = kSB ? 1 : 2, kB1 = kSB ? 0 : 1;
#pragma unroll
    for (int q = 0; q < NP; q++) {
#pragma unroll
        for (int m = 0; m < 8; m++) x[q][m].y = -x[q][m].y;
        dft8(x[q]);
    }
    if (kSB) group_bar_n<kBT>(bar_id);
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
    if (HB_EXP_SKIP & 64) __syncwarp(); else group_bar_n<kBT>(bar_id);
    {
        const int j0 = t & 7, k2 = t >> 3;
#pragma unroll
        for (int q = 0; q < NP; q++) {
#pragma unroll
            for (int j1 = 0; j1 < 8; j1++) x[q][j1] = xch[(kB0 * q) * kXchStride + j0 * 65 + k2 * 8 + j1];
            dft8(x[q]);
        }
        if (kSB) group_bar_n<kBT>(bar_id);
        double2 T[8];
        tw_powers(tw.i_b0, tw.i_stepb, false, T);
#pragma unroll
        for (int k1 = 0; k1 < 8; k1++) {
#pragma unroll
            for (int q = 0; q < NP; q++)
                xch[(kB0 * q + kB1) * kXchStride + k2 * 65 + k1 * 8 + j0] = cmul(x[q][rev3(k1)], T[k1]);
        }
    }
    if (HB_EXP_SKIP & 32) __syncwarp(); else group_bar_n<kBT>(bar_id);
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
