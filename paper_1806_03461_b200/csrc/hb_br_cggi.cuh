// hb_br_cggi.cuh: BK -> Fourier, shared blind-rotation helpers, CGGI-key blind-rotation kernels
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once

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
    uint32_t n_work;          // n_items * lanes (end of this launch's work range)
    uint32_t e0;              // first work item of this launch (a level split over launches)
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

// HA records (hb_gate kind HA): a second extraction of the same accumulator at
// index N/2 (a'_i = A_{N/2-i} for i <= N/2, -A_{3N/2-i} above; b' = B_{N/2}) into
// big row x2 of the item (oracle/tfhe_oracle.c sample_extract_at).
__device__ __forceinline__ uint32_t *x2_row(const BrArgs &args, uint32_t e) {
    const uint32_t x2 = args.items[e / args.lanes].x2;
    return x2 == kNoItem ? nullptr : args.big + ((size_t)x2 * args.lanes + e % args.lanes) * kBigStride;
}
__device__ __forceinline__ void sample_extract_half(const uint32_t *accA, const uint32_t *accB, uint32_t *out,
                                                    int tid, int nthreads) {
    for (int c = tid; c <= kN; c += nthreads) {
        uint32_t v;
        if (c < kN) v = c <= kNH ? accA[kNH - c] : 0u - accA[kN + kNH - c];
        else v = accB[kNH];
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

// WS: warp-specialised producer warpgroup (see k_blind_rotate_u2)
template <int G, bool kDebug, bool WS = false>
__global__ void __launch_bounds__(64 * G + (WS ? 128 : 0), 1) k_blind_rotate(const BrArgs args) {
    static_assert(!WS || G == 4, "warp-specialised producer: 4 bootstraps per CTA");
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
        for (int it = 0; it < kStages && it < rows_needed && !HB_BK_LDG && !WS; it++) {
            mbar_arrive_expect_tx(&sm.full[it], kRowBytes);
            bulk_g2s(sm.bk[it], bk_src + (size_t)it * kRowBytes, kRowBytes, &sm.full[it]);
        }
    }
    __syncthreads();
    if (WS) {
        if (warp >= 2 * G) {  // producer warpgroup
            asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
            if (threadIdx.x == 64 * G) {
#pragma unroll 1
                for (int it = 0; it < rows_needed; it++) {
                    const int slot = it % kStages;
                    if (it >= kStages) mbar_wait(&sm.empty[slot], ((it / kStages) - 1) & 1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive_expect_tx(&sm.full[slot], kRowBytes);
                    bulk_g2s(sm.bk[slot], bk_src + (size_t)it * kRowBytes, kRowBytes, &sm.full[slot]);
                }
            }
            return;
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
    }

    // ---- gate groups: 64 threads (2 warps) per bootstrap ----
    const int g = warp >> 1;
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + g;
    const uint32_t e_raw = args.e0 + blockIdx.x * G + g;
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
            if (!HB_BK_LDG && !WS && threadIdx.x == 0) {
#pragma unroll 1
                for (int nx = row_it + 1; nx <= row_it + 2; nx++) {
                    if (nx < kStages || nx >= rows_needed) continue;
                    const int s2 = nx % kStages;
                    mbar_wait(&sm.empty[s2], ((nx / kStages) - 1) & 1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before its async-proxy refill
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
    if (uint32_t *o2 = x2_row(args, e)) sample_extract_half(accA, accB, o2, t, 64);
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
    const uint32_t e = args.e0 + blockIdx.x;  // one bootstrap per CTA (grid == n_work - e0)
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
    if (uint32_t *o2 = x2_row(args, e)) sample_extract_half(accA, accB, o2, threadIdx.x, 192);
}
