// hb_br_u2h.cuh: key-pair blind rotation with 128 threads per bootstrap (wide levels)
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once

// ---------------------------------------------------------------------------
// k_blind_rotate_u2h: the key-pair external product of k_blind_rotate_u2 with
// each bootstrap split over two 64-thread halves.  Half h owns accumulator
// polynomial h (A or B) and its three gadget-digit rows (q = h, p = 0..2):
// per key pair it runs three single-polynomial forward transforms of its own
// digits and, for every (p, component c), a Fourier MAC of that one row into
// partial spectra of BOTH output polynomials.  At the end of the pair the
// halves swap the partial of the polynomial they do not own through their
// exchange buffers (two 128-thread barriers), and half h inverse-transforms
// output polynomial h and adds it to its own accumulator polynomial — the
// accumulator stays thread-private (bins t + 64 m of polynomial h).
//
// Why: the 64-thread kernel holds two polynomials' transforms and both output
// spectra per thread (244 registers), which caps an SM at 8 warps (2 per
// scheduler) and leaves the FP64 pipe waiting on dependencies.  Here a thread
// carries one transform and the two partial spectra (<= 128 registers), so
// four bootstraps give 16 warps per SM with the same shared memory (ring,
// exchange buffers, accumulators) and the same BK stage stream.
//
// BK stages are the layout of k_blind_rotate_u2 (per pair: [row pair][c][row]);
// consumption order per pair is [p][c][h] (row = 3h + p), mapped back to the
// stored stage index when the producer issues the bulk copy.
// ---------------------------------------------------------------------------
#ifndef HB_U2H_RING
#define HB_U2H_RING kStagesU2
#endif

__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// consumption index j (0..17) within a pair -> stored stage index within the pair
__device__ __forceinline__ int u2h_stage_of(int j) {
    const int p = j / 6, c = (j >> 1) % 3, h = j & 1;
    const int row = 3 * h + p;
    return (row >> 1) * 6 + c * 2 + (row & 1);
}
__device__ __forceinline__ size_t u2h_src_stage(int s) {
    return (size_t)(s / kStagesPerPair) * kStagesPerPair + u2h_stage_of(s % kStagesPerPair);
}

template <int G, int R = HB_U2H_RING>
struct BrSmemU2H {
    double2 bk[R][2 * kNH];          // stage ring: [output poly][bin]
    uint64_t full[R], empty[R];
    uint32_t acc[G][2][kN];          // accumulators (polynomial h: thread-private to half h)
    double2 xch[G][2][kXchStride];   // [bootstrap][half] single-buffered FFT exchange / partial swap
    uint16_t bar[G][kMaxLweN + 1];
    TwSeeds tws[64];
};

template <int G, bool kDebug, int R = HB_U2H_RING>
__global__ void __launch_bounds__(128 * G, 1) k_blind_rotate_u2h(const BrArgs args) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrSmemU2H<G, R> &sm = *reinterpret_cast<BrSmemU2H<G, R> *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = warp >> 2;          // bootstrap of this CTA
    const int hf = (warp >> 1) & 1;   // half: accumulator polynomial / digit rows 3 hf .. 3 hf + 2
    const int t = threadIdx.x & 63;   // thread within the half
    const int ub = threadIdx.x & 127; // thread within the bootstrap
    const int bar_half = 1 + 2 * g + hf;  // 64-thread named barriers 1 .. 2G
    const int bar_boot = 1 + 2 * G + g;   // 128-thread named barriers 2G+1 .. 3G
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
    int issued = 0;  // producer (thread 0) state
    if (threadIdx.x == 0) {
        for (int s = 0; s < R; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 2 * G);  // one half (2 warps) of each bootstrap consumes a stage
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (; issued < R && issued < stages_needed; issued++) {
            mbar_arrive_expect_tx(&sm.full[issued], kRowBytes);
            bulk_g2s(sm.bk[issued], bk_src + u2h_src_stage(issued) * kRowBytes, kRowBytes, &sm.full[issued]);
        }
    }
    __syncthreads();

    const uint32_t e_raw = args.e0 + blockIdx.x * G + g;
    const bool active = e_raw < args.n_work;
    const uint32_t e = active ? e_raw : args.n_work - 1;
    uint32_t *accP = sm.acc[g][hf];  // this half's accumulator polynomial
    double2 *xch = &sm.xch[g][hf][0];
    double2 *xch_other = &sm.xch[g][hf ^ 1][0];
    uint16_t *bar = sm.bar[g];

    k1_modswitch(args, e, bar, ub, 128);  // K1
    named_bar(bar_boot, 128);
    {  // ACC = X^{-barb} (0, mu...mu): half 0 zeroes A, half 1 writes the rotated test vector
        const int barb = bar[n];
#pragma unroll
        for (int m = 0; m < 16; m++) {
            const int j = t + 64 * m;
            accP[j] = hf ? (((j + barb) & kN) ? 0u - args.mu : args.mu) : 0u;
        }
    }
    // ACC is thread-private from here on (bins t + 64 m, t + 64 m + 512 of polynomial hf)

    double max_err = 0.0;
    int st = 0;  // consumption index of this thread's next p-step (6 stages per p-step)
    for (int pm = 0; pm < pairs; pm++) {
        const int ai = bar[2 * pm], aj = bar[2 * pm + 1];
        int ex[3];
#pragma unroll
        for (int c = 0; c < 3; c++) ex[c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
        double2 f0[8], f1[8];  // partial output spectra (polynomials 0 and 1) of this half's rows
#pragma unroll
        for (int m = 0; m < 8; m++) f0[m] = f1[m] = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int p = 0; p < kL; p++, st += 6) {
            if (threadIdx.x == 0) {  // producer: keep the ring R stages ahead of this p-step
#pragma unroll 1
                for (; issued < st + R && issued < stages_needed; issued++) {
                    const int s2 = issued % R;
                    mbar_wait(&sm.empty[s2], ((issued / R) - 1) & 1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before its async-proxy refill
                    mbar_arrive_expect_tx(&sm.full[s2], kRowBytes);
                    bulk_g2s(sm.bk[s2], bk_src + u2h_src_stage(issued) * kRowBytes, kRowBytes, &sm.full[s2]);
                }
            }
            __syncwarp();
            double2 x[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int j = t + 64 * m;
                x[0][m] = make_double2(small_int_to_double(gadget_digit(accP[j], p)),
                                       small_int_to_double(gadget_digit(accP[j + kNH], p)));
            }
            nega_fft_fwd_n<1, true>(x, xch, t, sm.tws[t], bar_half);
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const int sidx = st + 2 * c + hf;
                const int s = sidx % R;
                mbar_wait(&sm.full[s], (sidx / R) & 1);
                const double2 *b0 = sm.bk[s], *b1 = sm.bk[s] + kNH;
                // F_c = psi^{e (4k+1)} - 1 at bins k = t + 64 m (loaded per p-step: fewer live registers)
                const double2 basec = __ldg(&args.PSI[(ex[c] * (4 * t + 1)) & (2 * kN - 1)]);
                const long long flip = (long long)(ex[c] & 1) << 63;
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    const double2 pmv = m == 0 ? basec : cmul(basec, c_w8[(ex[c] * m) & 7]);
                    const double2 Fm[2] = {make_double2(pmv.x - 1.0, pmv.y),
                                           make_double2(__longlong_as_double(__double_as_longlong(pmv.x) ^ flip) - 1.0,
                                                        __longlong_as_double(__double_as_longlong(pmv.y) ^ flip))};
#pragma unroll
                    for (int hi = 0; hi < 2; hi++) {
                        const int mm = m + 4 * hi;
                        const int k = t + 64 * mm;
                        const double2 y = cmul(x[0][mm], Fm[hi]);
                        cmac(f0[mm], y, b0[k]);
                        cmac(f1[mm], y, b1[k]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.empty[s]);
            }
        }
        // swap partials: half 0 keeps output polynomial 0 and sends its polynomial-1
        // partial to half 1's buffer; half 1 the converse.  Both halves are past their
        // last forward-transform reads of either buffer at the first barrier.
        named_bar(bar_boot, 128);
#pragma unroll
        for (int m = 0; m < 8; m++) xch_other[t + 64 * m] = hf ? f0[m] : f1[m];
        named_bar(bar_boot, 128);
        double2 x[1][8];
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const double2 o = xch[t + 64 * m];
            x[0][m] = hf ? cadd(f1[m], o) : cadd(f0[m], o);
        }
        // (the inverse transform's first exchange store is preceded by a half barrier:
        // every thread of the half has read its partial by then)
        nega_fft_inv_n<1, true>(x, xch, t, sm.tws[t], bar_half);
#pragma unroll
        for (int m = 0; m < 8; m++) {
            if (kDebug) {
                max_err = fmax(max_err, fabs(x[0][m].x - rint(x[0][m].x)));
                max_err = fmax(max_err, fabs(x[0][m].y - rint(x[0][m].y)));
            }
            const int j = t + 64 * m;
            accP[j] += round_to_torus(x[0][m].x);
            accP[j + kNH] += round_to_torus(x[0][m].y);
        }
    }
    named_bar(bar_boot, 128);  // both accumulator polynomials final
    if (!active) return;
    if (kDebug && args.margin) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
    const uint32_t *accA = sm.acc[g][0], *accB = sm.acc[g][1];
    if (kDebug && args.acc_dump) {
        uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN;
        for (int c = ub; c < 2 * kN; c += 128) dst[c] = (c < kN) ? accA[c] : accB[c - kN];
    }
    sample_extract(accA, accB, args.big + (size_t)e * kBigStride, ub, 128);
    if (uint32_t *o2 = x2_row(args, e)) sample_extract_half(accA, accB, o2, ub, 128);
}
