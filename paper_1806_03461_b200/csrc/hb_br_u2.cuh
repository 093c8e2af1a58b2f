// hb_br_u2.cuh: key-pair blind-rotation kernels (throughput, latency, 2-CTA cluster) and TMEM helpers
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once

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
#ifndef HB_U2_MAC2
#define HB_U2_MAC2 1  // MAC over both rows of a row pair per bin (fewer live registers; 0: row by row)
#endif
#ifndef HB_U2_BKC
#define HB_U2_BKC 1  // MAC2 with the three components combined per bin before the digit product
#endif
#ifndef HB_EXP_NO_BK_LDS
#define HB_EXP_NO_BK_LDS 0
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
// WS: warp-specialised producer.  The CTA gets a fourth warpgroup whose first
// thread alone streams the BK stages (waits for a free slot, issues the bulk
// copy), so a refill is never delayed by the compute warp that used to issue it
// at the start of each row pair; the producer warpgroup gives its registers to
// the compute warps (setmaxnreg: 24 / 240).
// Compute warps are padded to whole warpgroups (G = 3: warps 6, 7 idle) so that
// the producer is a warpgroup of its own; setmaxnreg only where the launch
// bounds cap the registers (384 threads).
template <int G, bool WS>
__host__ __device__ constexpr int u2_compute_warps() { return WS ? ((2 * G + 3) / 4) * 4 : 2 * G; }
template <int G, bool WS>
__host__ __device__ constexpr int u2_threads() { return WS ? 32 * (u2_compute_warps<G, WS>() + 4) : 64 * G; }

template <int G, bool kDebug, int R = kStagesU2, int MB = 1, bool TM = false, bool WS = false>
__global__ void __launch_bounds__(u2_threads<G, WS>(), MB) k_blind_rotate_u2(const BrArgs args) {
    static_assert(!WS || (!TM && MB == 1), "warp-specialised producer: one CTA per SM, shared-memory ACC");
    constexpr int kCW = u2_compute_warps<G, WS>();
    constexpr bool kSetMax = WS && u2_threads<G, WS>() == 384;
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
        for (; !WS && issued < R && issued < stages_needed; issued++) {
            mbar_arrive_expect_tx(&sm.full[issued], kRowBytes);
            bulk_g2s(sm.bk[issued], bk_src + u2_stage(issued) * kRowBytes, kRowBytes, &sm.full[issued]);
        }
    }
    if (TM && warp == 0) tmem_alloc(&sm.tmem_base, kTmemCols);
    if (TM) tmem_fence_before();
    __syncthreads();
    if (TM) tmem_fence_after();
    if (WS) {
        if (warp >= kCW) {  // producer warpgroup
            if (kSetMax) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
            if (threadIdx.x == 32 * kCW) {
#pragma unroll 1
                for (int s = 0; s < stages_needed; s++) {
                    const int slot = s % R;
                    if (s >= R) mbar_wait(&sm.empty[slot], ((s / R) - 1) & 1);
                    // order the consumers' generic-proxy reads of this slot (released through
                    // the empty barrier) before the async-proxy bulk copy that overwrites it;
                    // without it the refill raced reads still in flight (tests/test_gpu_exactness.py
                    // determinism: 1-3 of 16,384 ciphertexts differed per run)
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive_expect_tx(&sm.full[slot], kRowBytes);
                    bulk_g2s(sm.bk[slot], bk_src + u2_stage(s) * kRowBytes, kRowBytes, &sm.full[slot]);
                }
            }
            return;
        }
        if (kSetMax) asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
        if (warp >= 2 * G) return;  // warpgroup padding
    }
    // this thread's 32 ACC columns: A at +0..15, B at +16..31 (lo bins m, then hi bins m)
    const uint32_t tacc = TM ? sm.tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + 32u * (uint32_t)(warp >> 2) : 0u;

    const int g = warp >> 1;
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + g;
    const uint32_t e_raw = args.e0 + blockIdx.x * G + g;
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
    // WS (registers to spare): the psi table values of key pair pm + 1 are loaded
    // during pair pm, so their L2 latency never stalls the MAC
    constexpr bool kPre = WS;
    double2 pre[3];
    if (kPre && pairs > 0) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const int ai = bar[0], aj = bar[1];
            const int ec = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            pre[c] = __ldg(&args.PSI[(ec * (4 * t + 1)) & (2 * kN - 1)]);
        }
    }
    for (int pm = 0; pm < pairs; pm++) {
        const int ai = bar[2 * pm], aj = bar[2 * pm + 1];
        // F_c at this thread's bins k = t + 64 m: psi^{e (4k+1)} - 1 =
        // psi^{e (4t+1)} * w8^{e m} - 1 (the exponent is warp-uniform)
        int ex[3];
        double2 base[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            ex[c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            if (kPre) {
                base[c] = pre[c];
            } else {
                base[c] = __ldg(&args.PSI[(ex[c] * (4 * t + 1)) & (2 * kN - 1)]);
            }
        }
        if (kPre && pm + 1 < pairs) {
            const int bi = bar[2 * pm + 2], bj = bar[2 * pm + 3];
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const int ec = c == 0 ? ((bi + bj) & (2 * kN - 1)) : (c == 1 ? bi : bj);
                pre[c] = __ldg(&args.PSI[(ec * (4 * t + 1)) & (2 * kN - 1)]);
            }
        }
        double2 f0[8], f1[8];
#if HB_U2_MAC2
#pragma unroll
        for (int m = 0; m < 8; m++) f0[m] = f1[m] = make_double2(0.0, 0.0);
#endif
#pragma unroll 1
        for (int rp = 0; rp < kRows / 2; rp++) {
            // producer: refill the ring up to R stages ahead of this row pair
            if (!WS && threadIdx.x == 0) {
#pragma unroll 1
                for (; issued < st + R && issued < stages_needed; issued++) {
                    const int s2 = issued % R;
                    mbar_wait(&sm.empty[s2], ((issued / R) - 1) & 1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before its async-proxy refill
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
#if HB_U2_MAC2
            // both rows of the row pair per bin: F_c at bins m, m + 4 computed in the
            // m loop (8 live registers instead of 32), two independent products per
            // bin, accumulators zeroed at the start of the pair
            static_assert(!kMidIssue, "MAC2 consumes the row pair's two stages of a component together");
#if HB_U2_BKC
            // combined key per bin: C_{h,o} = sum_c F_c BK_{h,c,o} (12 complex products), then
            // ACC_o += x_h C_{h,o} (4): 64 FP64 instructions per bin instead of 72
            {
                int sl[6];
#pragma unroll
                for (int i = 0; i < 6; i++) {
                    sl[i] = (st + i) % R;
                    mbar_wait(&sm.full[sl[i]], ((st + i) / R) & 1);
                }
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    double2 Fm[3][2];
#pragma unroll
                    for (int c = 0; c < 3; c++) {
                        const long long flip = (long long)(ex[c] & 1) << 63;
                        const double2 pw = m == 0 ? base[c] : cmul(base[c], c_w8[(ex[c] * m) & 7]);
                        Fm[c][0] = make_double2(pw.x - 1.0, pw.y);
                        Fm[c][1] = make_double2(__longlong_as_double(__double_as_longlong(pw.x) ^ flip) - 1.0,
                                                __longlong_as_double(__double_as_longlong(pw.y) ^ flip));
                    }
#pragma unroll
                    for (int hi = 0; hi < 2; hi++) {
                        const int mm = m + 4 * hi;
                        const int k = t + 64 * mm;
                        double2 C[2][2];
#pragma unroll
                        for (int c = 0; c < 3; c++) {
#pragma unroll
                            for (int h = 0; h < 2; h++) {
                                const double2 *bk = sm.bk[sl[2 * c + h]];
                                // HB_EXP_NO_BK_LDS (timing only, wrong results): one BK value per
                                // thread and stage, i.e. 1/8 of the BK shared-memory loads
                                const int kb = HB_EXP_NO_BK_LDS ? t : k;
                                if (c == 0) {
                                    C[h][0] = cmul(Fm[c][hi], bk[kb]);
                                    C[h][1] = cmul(Fm[c][hi], bk[kNH + kb]);
                                } else {
                                    cmac(C[h][0], Fm[c][hi], bk[kb]);
                                    cmac(C[h][1], Fm[c][hi], bk[kNH + kb]);
                                }
                            }
                        }
                        cmac(f0[mm], x[0][mm], C[0][0]);
                        cmac(f1[mm], x[0][mm], C[0][1]);
                        cmac(f0[mm], x[1][mm], C[1][0]);
                        cmac(f1[mm], x[1][mm], C[1][1]);
                    }
                }
                __syncwarp();
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < 6; i++) mbar_arrive(&sm.empty[sl[i]]);
                }
                __syncwarp();
                st += 6;
            }
#else
#pragma unroll
            for (int c = 0; c < 3; c++, st += 2) {
                const long long flip = (long long)(ex[c] & 1) << 63;
                const int s0 = st % R, s1 = (st + 1) % R;
                mbar_wait(&sm.full[s0], (st / R) & 1);
                mbar_wait(&sm.full[s1], ((st + 1) / R) & 1);
                const double2 *b00 = sm.bk[s0], *b01 = sm.bk[s0] + kNH;  // row h = 0: output polys 0 / 1
                const double2 *b10 = sm.bk[s1], *b11 = sm.bk[s1] + kNH;  // row h = 1
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    const double2 pm = m == 0 ? base[c] : cmul(base[c], c_w8[(ex[c] * m) & 7]);
                    const double2 Fm[2] = {make_double2(pm.x - 1.0, pm.y),
                                           make_double2(__longlong_as_double(__double_as_longlong(pm.x) ^ flip) - 1.0,
                                                        __longlong_as_double(__double_as_longlong(pm.y) ^ flip))};
#pragma unroll
                    for (int hi = 0; hi < 2; hi++) {
                        const int mm = m + 4 * hi;
                        const int k = t + 64 * mm;
                        const double2 y0 = cmul(x[0][mm], Fm[hi]), y1 = cmul(x[1][mm], Fm[hi]);
                        cmac(f0[mm], y0, b00[k]);
                        cmac(f1[mm], y0, b01[k]);
                        cmac(f0[mm], y1, b10[k]);
                        cmac(f1[mm], y1, b11[k]);
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sm.empty[s0]);
                    mbar_arrive(&sm.empty[s1]);
                }
                __syncwarp();
            }
#endif  // HB_U2_BKC
#else
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
#if HB_EXP_NO_BK_LDS  // timing experiment only (results wrong): one BK value per thread and stage
                    const double2 b0c = bk0[t], b1c = bk1[t];
#define HB_BK0(m) b0c
#define HB_BK1(m) b1c
#else
#define HB_BK0(m) bk0[t + 64 * (m)]
#define HB_BK1(m) bk1[t + 64 * (m)]
#endif
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        const double2 y = cmul(x[h][m], F[m]);
                        if (rp == 0 && c == 0 && h == 0) {
                            f0[m] = cmul(y, HB_BK0(m));
                            f1[m] = cmul(y, HB_BK1(m));
                        } else {
                            cmac(f0[m], y, HB_BK0(m));
                            cmac(f1[m], y, HB_BK1(m));
                        }
                    }
#undef HB_BK0
#undef HB_BK1
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.empty[s]);
                    if (kMidIssue && threadIdx.x == 0) {  // shallow ring: refill behind consumption
#pragma unroll 1
                        for (; issued < st + 1 + R && issued < stages_needed; issued++) {
                            const int s2 = issued % R;
                            mbar_wait(&sm.empty[s2], ((issued / R) - 1) & 1);
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before its async-proxy refill
                            mbar_arrive_expect_tx(&sm.full[s2], kRowBytes);
                            bulk_g2s(sm.bk[s2], bk_src + u2_stage(issued) * kRowBytes, kRowBytes, &sm.full[s2]);
                        }
                    }
                    __syncwarp();
                }
            }
#endif
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
            if (uint32_t *o2 = x2_row(args, e)) {  // HA: extraction at index N/2
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const int j = t + 64 * m;  // A_j -> a'_{512-j}; A_{j+512} -> a'_{1024-j} (j > 0), -sign
                    o2[kNH - j] = v[m];
                    if (j > 0) {
                        o2[kN - j] = 0u - v[8 + m];
                    } else {
                        o2[0] = v[8];     // a'_0 = A_512
                        o2[kN] = v[24];   // b' = B_512
                    }
                }
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
    if (uint32_t *o2 = x2_row(args, e)) sample_extract_half(accA, accB, o2, t, 64);
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
    const uint32_t e = args.e0 + blockIdx.x;
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
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before its async-proxy refill
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
    if (uint32_t *o2 = x2_row(args, e)) sample_extract_half(accA, accB, o2, threadIdx.x, 192);
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
    const uint32_t e = args.e0 + (blockIdx.x >> 1);
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
    uint32_t *out2 = x2_row(args, e);  // HA: second extraction at index N/2
    if (q == 0) {
        for (int c = threadIdx.x; c < kN; c += 192) out[c] = c == 0 ? sm.acc[0] : 0u - sm.acc[kN - c];
        if (out2)
            for (int c = threadIdx.x; c < kN; c += 192) out2[c] = c <= kNH ? sm.acc[kNH - c] : 0u - sm.acc[kN + kNH - c];
    } else if (threadIdx.x == 0) {
        out[kN] = sm.acc[0];
        if (out2) out2[kN] = sm.acc[kNH];
    }
}
