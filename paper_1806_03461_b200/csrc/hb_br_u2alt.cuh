// hb_br_u2alt.cuh: key-pair blind rotation, throughput kernel with alternating halves
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once

// ---------------------------------------------------------------------------
// k_blind_rotate_u2_alt: the warp-specialised key-pair kernel (hb_br_u2.cuh,
// k_blind_rotate_u2<G, .., WS>) with its G bootstraps split into two halves that
// take turns on the shared-memory data pipe.
//
// In k_blind_rotate_u2 the 7-stage ring of 16 KiB (row, component) stages holds
// little more than one row pair, and a row pair's six stages are released only
// when its MAC is over, so the G bootstraps of a CTA run in phase: all of them
// in a forward transform (FP64-bound), then all of them in the MAC (bound by the
// BK reads from shared memory).  Neither pipe is busy for more than ~2/3 of the
// time (ncu r02_m: LSU 80%, FP64 65%).
//
// Here the BK of a row pair arrives as eight 12 KiB *bin blocks* (block j holds,
// for the 64 bins t + 64 mm, mm = (j >> 1) + 4 (j & 1), the twelve values
// BK[c][h][o]) and a block is released as soon as every bootstrap has used it.
// The leaders (groups < G/2) and the followers take strict turns at the MAC of
// each row pair (two mbarriers, `turn`): the followers' MAC(q) starts when the
// leaders' MAC(q) is over, the leaders' MAC(q + 1) when the followers' MAC(q) is
// over, so one half transforms (FP64) while the other multiplies (LSU).  A
// 9-block ring is enough: while the followers multiply they free the blocks of
// row pair q one by one and the producer refills them with row pair q + 1 for
// the leaders.
//
// Arithmetic and operation order per bootstrap are those of k_blind_rotate_u2
// (combined-key MAC, HB_U2_BKC), so the ciphertexts are bit-identical.
// ---------------------------------------------------------------------------
constexpr int kAltBlockElems = 12 * 64;                                   // double2 per bin block
constexpr uint32_t kAltBlockBytes = kAltBlockElems * sizeof(double2);     // 12 KiB
constexpr int kAltBlocksPerRowPair = 8;
constexpr int kAltBlocksPerPair = 3 * kAltBlocksPerRowPair;
#ifndef HB_ALT_RING
#define HB_ALT_RING 9
#endif
#ifndef HB_ALT_TURNS
#define HB_ALT_TURNS 1  // 0: no turn-taking (free-running halves; experiment)
#endif
constexpr int kAltRing = HB_ALT_RING;

template <int G>
struct BrAltSmem {
    double2 bk[kAltRing][kAltBlockElems];    // bin-block ring: [c][h][o][64 bins]
    uint64_t full[kAltRing], empty[kAltRing];
    uint64_t turn[2];                        // MAC turns: [0] leaders done with MAC(q), [1] followers
    uint32_t acc[G][2][kN];                  // TRLWE accumulators
    double2 xch[G][2][kXchStride];           // single-buffered dual-FFT exchange
    uint16_t bar[G][kMaxLweN + 1];
    TwSeeds tws[64];
};

// BK (Fourier, stage layout of k_bk_to_fourier with unroll 2) -> bin-block layout
__global__ void __launch_bounds__(256) k_bkf_to_blocks(const double2 *__restrict__ bkf, double2 *__restrict__ blk,
                                                       size_t n_elems) {
    const size_t i = (size_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= n_elems) return;
    const int t = (int)(i & 63);
    size_t r = i >> 6;
    const int cho = (int)(r % 12);
    r /= 12;
    const int j = (int)(r % kAltBlocksPerRowPair);
    const size_t rowpair = r / kAltBlocksPerRowPair;  // pm * 3 + rp
    const int mm = (j >> 1) + 4 * (j & 1);
    blk[i] = bkf[(rowpair * 12 + cho) * kNH + 64 * mm + t];
}

template <int G, bool kDebug>
__global__ void __launch_bounds__(u2_threads<G, true>(), 1) k_blind_rotate_u2_alt(const BrArgs args) {
    static_assert(G == 4 || G == 2, "two halves of whole groups; 384 or 256 threads");
    constexpr int kCW = u2_compute_warps<G, true>();
    constexpr bool kSetMax = u2_threads<G, true>() == 384;
    constexpr int R = kAltRing;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrAltSmem<G> &sm = *reinterpret_cast<BrAltSmem<G> *>(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = args.n;
    const int pairs = min(n, args.iters) / 2;
    const int blocks_needed = pairs * kAltBlocksPerPair;
    const char *bk_src = reinterpret_cast<const char *>(args.bkf_blk);

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
        for (int s = 0; s < R; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 2 * G);
        }
        mbar_init(&sm.turn[0], G);  // G/2 groups of two warps each
        mbar_init(&sm.turn[1], G);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp >= kCW) {  // producer warpgroup
        if (kSetMax) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
        if (threadIdx.x == 32 * kCW) {
#pragma unroll 1
            for (int s = 0; s < blocks_needed; s++) {
                const int slot = s % R;
                if (s >= R) mbar_wait(&sm.empty[slot], ((s / R) - 1) & 1);
                // consumers' generic-proxy reads of the slot before the async-proxy refill
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_expect_tx(&sm.full[slot], kAltBlockBytes);
                bulk_g2s(sm.bk[slot], bk_src + (size_t)s * kAltBlockBytes, kAltBlockBytes, &sm.full[slot]);
            }
        }
        return;
    }
    if (kSetMax) asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
    if (warp >= 2 * G) return;  // warpgroup padding

    const int g = warp >> 1;
    const bool leader = g < G / 2;
    const int t = threadIdx.x & 63;
    const int bar_id = 1 + g;
    const uint32_t e_raw = args.e0 + blockIdx.x * G + g;
    const bool active = e_raw < args.n_work;
    const uint32_t e = active ? e_raw : args.n_work - 1;
    uint32_t *accA = sm.acc[g][0];
    uint32_t *accB = sm.acc[g][1];
    double2 *xch = &sm.xch[g][0][0];
    uint16_t *bar = sm.bar[g];

    k1_modswitch(args, e, bar, t, 64);  // K1
    group_bar(bar_id);
    acc_init(accA, accB, bar[n], args.mu, t, 64);  // ACC = X^{-barb} (0, mu...mu)
    group_bar(bar_id);

    double max_err = 0.0;
    int st = 0;  // next bin block to consume
    int q = 0;   // MAC counter (row pairs done)
    double2 pre[3];
    if (pairs > 0) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const int ai = bar[0], aj = bar[1];
            const int ec = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            pre[c] = __ldg(&args.PSI[(ec * (4 * t + 1)) & (2 * kN - 1)]);
        }
    }
    for (int pm = 0; pm < pairs; pm++) {
        const int ai = bar[2 * pm], aj = bar[2 * pm + 1];
        int ex[3];
        double2 base[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            ex[c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            base[c] = pre[c];
        }
        if (pm + 1 < pairs) {
            const int bi = bar[2 * pm + 2], bj = bar[2 * pm + 3];
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const int ec = c == 0 ? ((bi + bj) & (2 * kN - 1)) : (c == 1 ? bi : bj);
                pre[c] = __ldg(&args.PSI[(ec * (4 * t + 1)) & (2 * kN - 1)]);
            }
        }
        double2 f0[8], f1[8];
#pragma unroll
        for (int m = 0; m < 8; m++) f0[m] = f1[m] = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int rp = 0; rp < kRows / 2; rp++, q++) {
            double2 x[2][8];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int row = 2 * rp + h;
                const int qq = row / kL, p = row % kL;
                const uint32_t *P = qq ? accB : accA;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const int j = t + 64 * m;
                    x[h][m] = make_double2(small_int_to_double(gadget_digit(P[j], p)),
                                           small_int_to_double(gadget_digit(P[j + kNH], p)));
                }
            }
            nega_fft_fwd_n<2, true>(x, xch, t, sm.tws[t], bar_id);
            // MAC turn: followers after the leaders' MAC(q), leaders after the followers' MAC(q - 1)
            if (HB_ALT_TURNS) {
                if (!leader) mbar_wait(&sm.turn[0], q & 1);
                else if (q > 0) mbar_wait(&sm.turn[1], (q - 1) & 1);
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
                    const int bs = st + 2 * m + hi;
                    const int slot = bs % R;
                    mbar_wait(&sm.full[slot], (bs / R) & 1);
                    const double2 *bk = sm.bk[slot] + t;
                    double2 C[2][2];
#pragma unroll
                    for (int c = 0; c < 3; c++) {
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            const double2 b0 = bk[((c * 2 + h) * 2 + 0) * 64], b1 = bk[((c * 2 + h) * 2 + 1) * 64];
                            if (c == 0) {
                                C[h][0] = cmul(Fm[c][hi], b0);
                                C[h][1] = cmul(Fm[c][hi], b1);
                            } else {
                                cmac(C[h][0], Fm[c][hi], b0);
                                cmac(C[h][1], Fm[c][hi], b1);
                            }
                        }
                    }
                    cmac(f0[mm], x[0][mm], C[0][0]);
                    cmac(f1[mm], x[0][mm], C[0][1]);
                    cmac(f0[mm], x[1][mm], C[1][0]);
                    cmac(f1[mm], x[1][mm], C[1][1]);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.empty[slot]);
                }
            }
            if (HB_ALT_TURNS) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.turn[leader ? 0 : 1]);
            }
            __syncwarp();
            st += kAltBlocksPerRowPair;
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
                for (int qq = 0; qq < 2; qq++)
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        max_err = fmax(max_err, fabs(x[qq][m].x - rint(x[qq][m].x)));
                        max_err = fmax(max_err, fabs(x[qq][m].y - rint(x[qq][m].y)));
                    }
            }
#pragma unroll
            for (int qq = 0; qq < 2; qq++) {
                uint32_t *P = qq ? accB : accA;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const int j = t + 64 * m;
                    P[j] += round_to_torus(x[qq][m].x);
                    P[j + kNH] += round_to_torus(x[qq][m].y);
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
    sample_extract(accA, accB, args.big + (size_t)e * kBigStride, t, 64);
    if (uint32_t *o2 = x2_row(args, e)) sample_extract_half(accA, accB, o2, t, 64);
}
