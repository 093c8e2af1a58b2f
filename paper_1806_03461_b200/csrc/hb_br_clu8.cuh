// hb_br_clu8.cuh: lone-bootstrap latency kernel, key pairs, one bootstrap per 8-CTA cluster,
// MAC split by Fourier bins
// (textually included by hb_engine.cu after hb_br_clu6.cuh, inside its anonymous namespace;
// not a standalone header)
#pragma once

// ---------------------------------------------------------------------------
// k_blind_rotate_u2_clu8: the lone and near-lone levels (at most one bootstrap
// per 8 SMs).  k_blind_rotate_u2_clu6 splits each key pair's external product
// by digit row: every CTA multiplies its row by the BK at all 512 bins and
// ships two 8 KiB partial spectra to the owners, so an owner receives 40 KiB
// over DSMEM per key pair (~1.8k of its ~6.6k cycles; lone level 1.06 ms).  Here the MAC is split
// by BINS instead:
//   1. CTA r < 6 (row r = 3q + p: ACC polynomial q, gadget level p): digits of
//      ACC_q, one forward FFT; thread t then holds bins t + 64 m (m = 0..7) and
//      sends bin t + 64 m to CTA m (st.async, 16 B each): every CTA receives
//      the six rows' spectra at its 64 bins (6 KiB)
//   2. CTA m, threads u < 128 (bin t = u & 63, output polynomial o = u >> 6):
//      out_o = sum_r x_r C_{r,o}, C_{r,o} = sum_c F_c BK_{r,c,o} at bin t + 64 m
//      (the combined-key MAC of k_blind_rotate_u2), and ships out_o to owner o
//      (CTA 3o): the owner receives 8 KiB, already in its inverse FFT's input
//      layout (thread t, register m)
//   3. the three row CTAs of polynomial o each receive out_o and run the same
//      inverse FFT and ACC_o += round(.) on their own copy (HB_CLU8_RD, default;
//      0: only the owner CTA 3o does, then broadcasts ACC_o to the other two as
//      clu6 does — one DSMEM hop more per key pair, 0.75 vs 0.68-0.73 ms)
// Each CTA streams only its 64 bins of the pair's 18 BK stages (36 x 1 KiB
// bulk copies per pair, issued two pairs ahead into a double buffer).  All
// receive buffers are double-buffered by pair parity; their reuse two pairs
// later is ordered by the dependency chain itself (a CTA cannot send for pair
// pm + 2 before the owners consumed pair pm + 1), so no flow-control barriers
// are needed.  Same arithmetic per (row, component, bin) as the other
// key-pair kernels; the summation order differs, so bit-exactness rests on the
// FFT rounding margin (tests/test_gpu_parity.py narrow levels, exactness test).
// ---------------------------------------------------------------------------
constexpr int kClu8 = 8;
constexpr uint32_t kClu8BinBytes = 64 * sizeof(double2);               // one (stage, poly) slice: 1 KiB
constexpr uint32_t kClu8BkBytes = kStagesPerPair * 2 * kClu8BinBytes;  // a pair's slices: 36 KiB
constexpr uint32_t kClu8SpecBytes = kRows * kClu8BinBytes;            // six rows at 64 bins: 6 KiB
constexpr uint32_t kClu8OutBytes = kClu8 * kClu8BinBytes;             // eight CTAs' 64 bins: 8 KiB

struct BrClu8Smem {
    double2 bk[2][kStagesPerPair][2][64];  // [pair parity][stage][output poly][t]: bins t + 64 m
    double2 spec[2][kRows][64];            // [pair parity][row][t]: the six rows at this CTA's bins
    double2 outp[2][kClu8][64];            // owners: [pair parity][m][t] = output bin t + 64 m
    double2 xch[kXchStride];               // group 0's FFT exchange (forward and inverse)
    uint32_t acc[kN];                      // ACC_q (owner: authoritative; siblings: broadcast copy)
    uint16_t bar[kMaxLweN + 1];
    TwSeeds tws[64];
    uint64_t bk_full[2];                   // this CTA's BK slices of a pair landed
    uint64_t spec_full[2];                 // the six rows' spectra landed (6 KiB)
    uint64_t out_full[2];                  // owners: the eight CTAs' outputs landed (8 KiB)
    uint64_t acc_full;                     // siblings: the owner's new ACC_q landed
};

#ifndef HB_CLU8_RD
#define HB_CLU8_RD 1  // every row CTA of polynomial o receives out_o and inverse-transforms it (no ACC broadcast)
#endif
template <bool kDebug>
__global__ void __cluster_dims__(kClu8, 1, 1) __launch_bounds__(192, 1) k_blind_rotate_u2_clu8(const BrArgs args) {
    constexpr bool RD = HB_CLU8_RD;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrClu8Smem &sm = *reinterpret_cast<BrClu8Smem *>(smem_raw);
    const uint32_t rank = cluster_ctarank();  // = m: this CTA's bins t + 64 m
    const bool row_cta = rank < (uint32_t)kRows;
    const int q = row_cta ? (int)rank / 3 : 0, p = row_cta ? (int)rank % 3 : 0;
    const int row = 3 * q + p;
    const bool owner = row_cta && p == 0;
    const bool inverter = RD ? row_cta : owner;  // CTAs that inverse-transform output polynomial q
    const int warp = threadIdx.x >> 5, grp = warp >> 1, t = threadIdx.x & 63;
    const int u = threadIdx.x & 127;  // MAC threads u < 128: bin t = u & 63, output polynomial u >> 6
    const int bar_id = 1 + grp;
    const int n = args.n;
    const int pairs = min(n, args.iters) / 2;
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);
    const uint32_t e = args.e0 + blockIdx.x / kClu8;
    const bool producer = threadIdx.x == 128;  // group 2: BK slices and barrier re-arming
    // pair pm's BK slices of this CTA: stage s, poly o -> 64 double2 at bins 64 m .. 64 m + 63
    auto issue_bk = [&](int pm) {
        const int b = pm & 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // previous generic reads of the buffer
        mbar_arrive_expect_tx(&sm.bk_full[b], kClu8BkBytes);
        const char *src = bk_src + (size_t)pm * kStagesPerPair * kRowBytes + (size_t)rank * kClu8BinBytes;
#pragma unroll 1
        for (int s = 0; s < kStagesPerPair; s++)
#pragma unroll
            for (int o = 0; o < 2; o++)
                bulk_g2s(&sm.bk[b][s][o][0], src + (size_t)s * kRowBytes + (size_t)o * kNH * sizeof(double2),
                         kClu8BinBytes, &sm.bk_full[b]);
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
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; b++) {
            mbar_init(&sm.bk_full[b], 1);
            mbar_init(&sm.spec_full[b], 1);
            mbar_init(&sm.out_full[b], 1);
        }
        mbar_init(&sm.acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (producer) {
        for (int pm = 0; pm < 2 && pm < pairs; pm++) {
            issue_bk(pm);
            mbar_arrive_expect_tx(&sm.spec_full[pm], kClu8SpecBytes);
            if (inverter) mbar_arrive_expect_tx(&sm.out_full[pm], kClu8OutBytes);
        }
        if (!RD && row_cta && !owner && pairs > 1) mbar_arrive_expect_tx(&sm.acc_full, kN * 4);  // pair 0's new ACC_q
    }
    if (row_cta) {
        k1_modswitch(args, e, sm.bar, threadIdx.x, 192);  // K1
        __syncthreads();
        acc_init(q == 0 ? sm.acc : nullptr, q == 0 ? nullptr : sm.acc, sm.bar[n], args.mu, threadIdx.x, 192);
    } else {
        k1_modswitch(args, e, sm.bar, threadIdx.x, 192);  // the bin CTAs need the rotation exponents too
    }
    // every CTA's barriers are initialised and armed, every ACC copy is set
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

    const uint32_t spec_off = smem_addr(&sm.spec[0][0][0]);
    const uint32_t out_off = smem_addr(&sm.outp[0][0][0]);
    const uint32_t spec_bar_off = smem_addr(&sm.spec_full[0]);
    const uint32_t out_bar_off = smem_addr(&sm.out_full[0]);
    double max_err = 0.0;
    // F_c at this thread's MAC bin k = t + 64 rank: psi^{e_c (4k+1)}; pair 0's loaded here,
    // then always one pair ahead
    double2 base[3];
    auto load_base = [&](int pm, double2 (&bs)[3]) {
        const int ai = sm.bar[2 * pm], aj = sm.bar[2 * pm + 1];
        const int kk = 4 * (t + 64 * (int)rank) + 1;
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const int ec = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            bs[c] = __ldg(&args.PSI[(ec * kk) & (2 * kN - 1)]);
        }
    };
    if (pairs > 0 && grp < 2) load_base(0, base);
    for (int pm = 0; pm < pairs; pm++) {
        const int b = pm & 1;
        // 1. row CTAs, group 0: digits + forward transform of row (q, p), scattered by bin
        if (row_cta && grp == 0) {
            if (!RD && !owner && pm > 0) {
                mbar_wait_cluster(&sm.acc_full, (pm - 1) & 1);  // the owner's ACC_q after pair pm - 1
                if (t == 0 && pm + 1 < pairs) mbar_arrive_expect_tx(&sm.acc_full, kN * 4);
            }
            double2 x[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int j = t + 64 * m;
                x[0][m] = make_double2(small_int_to_double(gadget_digit(sm.acc[j], p)),
                                       small_int_to_double(gadget_digit(sm.acc[j + kNH], p)));
            }
            nega_fft_fwd_n<1, true>(x, sm.xch, t, sm.tws[t], bar_id);
            const uint32_t loc = spec_off + (uint32_t)(((b * kRows + row) * 64 + t) * 16);
            const uint32_t lbar = spec_bar_off + (uint32_t)(b * 8);
#pragma unroll
            for (int m = 0; m < 8; m++) st_async_f64x2(mapa_u32(loc, m), x[0][m], mapa_u32(lbar, m));
        }
        // 2. threads u < 128: the combined-key MAC of all six rows at bin t + 64 rank, output o
        if (grp < 2) {
            const int o = u >> 6;
            double2 nb[3];
            if (pm + 1 < pairs) load_base(pm + 1, nb);
            mbar_wait(&sm.bk_full[b], (pm >> 1) & 1);
            mbar_wait_cluster(&sm.spec_full[b], (pm >> 1) & 1);
            double2 F[3];
#pragma unroll
            for (int c = 0; c < 3; c++) F[c] = make_double2(base[c].x - 1.0, base[c].y);
            double2 acc_o = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < kRows; r++) {
                const int rs = (r >> 1) * 6 + (r & 1);  // stage of (row r, component 0) within the pair
                double2 C = cmul(F[0], sm.bk[b][rs][o][t]);
                cmac(C, F[1], sm.bk[b][rs + 2][o][t]);
                cmac(C, F[2], sm.bk[b][rs + 4][o][t]);
                cmac(acc_o, sm.spec[b][r][t], C);
            }
            // to owner o (CTA 3 o; RD: all three row CTAs of polynomial o), slot [b][rank][t]
#pragma unroll
            for (int d = 0; d < (RD ? 3 : 1); d++) {
                const uint32_t dst = 3u * (uint32_t)o + (uint32_t)d;
                st_async_f64x2(mapa_u32(out_off + (uint32_t)(((b * kClu8 + (int)rank) * 64 + t) * 16), dst), acc_o,
                               mapa_u32(out_bar_off + (uint32_t)(b * 8), dst));
            }
            if (pm + 1 < pairs) {
#pragma unroll
                for (int c = 0; c < 3; c++) base[c] = nb[c];
            }
        }
        // 3. once the MAC threads have read this pair's BK slices and spectra: the producer
        //    (group 2, idle otherwise) re-arms the spectrum barrier for pair pm + 2 and streams
        //    its BK slices into the freed buffer.  (A spectrum of pair pm + 2 cannot arrive
        //    before the owners consumed pair pm + 1, i.e. after this CTA's next MAC; a
        //    complete-tx ahead of the re-arm would also be safe: the phase still waits for
        //    the producer's arrival.)
        asm volatile("bar.sync %0, %1;" ::"r"(5), "r"(192) : "memory");  // MAC reads of bk[b] / spec[b] done
        if (producer && pm + 2 < pairs) {
            mbar_arrive_expect_tx(&sm.spec_full[b], kClu8SpecBytes);
            issue_bk(pm + 2);
        }
        // 4. owner, group 0: the eight CTAs' outputs -> inverse transform -> ACC_q -> siblings
        if (inverter && grp == 0) {
            mbar_wait_cluster(&sm.out_full[b], (pm >> 1) & 1);
            if (t == 0 && pm + 2 < pairs) mbar_arrive_expect_tx(&sm.out_full[b], kClu8OutBytes);
            double2 y[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) y[0][m] = sm.outp[b][m][t];
            nega_fft_inv_n<1, true>(y, sm.xch, t, sm.tws[t], bar_id);
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
            if (!RD && pm + 1 < pairs) {
                group_bar(bar_id);  // ACC_q complete in shared memory
                const uint32_t acc_off = smem_addr(&sm.acc[0]), abar_off = smem_addr(&sm.acc_full);
#pragma unroll
                for (int k4 = 0; k4 < 4; k4++) {
                    const int w = 4 * (t + 64 * k4);
                    const uint4 v = *reinterpret_cast<const uint4 *>(&sm.acc[w]);
#pragma unroll
                    for (int sib = 1; sib < 3; sib++) {
                        const uint32_t r = 3 * q + sib;
                        st_async_u32x4(mapa_u32(acc_off + 4u * w, r), v, mapa_u32(abar_off, r));
                    }
                }
            }
        }
    }
    // no CTA may exit while a peer can still address its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (!owner) return;
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
