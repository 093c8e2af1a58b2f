// hb_br_binsplit.cuh: latency kernels for narrow key-pair levels: one bootstrap per C-CTA
// cluster (C = 8 or 4), the external product's MAC split by Fourier bins
// (textually included by hb_engine.cu after hb_br_clu6.cuh, inside its anonymous namespace;
// not a standalone header)
#pragma once

// ---------------------------------------------------------------------------
// k_blind_rotate_u2_binsplit<C>: the lone and narrow levels.
// k_blind_rotate_u2_clu6 splits each key pair's external product by digit
// row: every CTA multiplies its row by the BK at all 512 bins and ships two
// 8 KiB partial spectra to the owners, so an owner receives 40 KiB over DSMEM
// per key pair (~1.8k of its ~6.6k cycles; lone level 1.06 ms).  Here the MAC
// is split by BINS instead.  With RPC = 6 / (row CTAs) digit rows per row CTA
// (C = 8: CTAs 0-5 one row each, CTAs 6-7 MAC only; C = 4: CTAs 0-2 two rows
// each, CTA 3 MAC only) and MPC = 8 / C bin columns m per CTA:
//   1. group g < RPC of row CTA r takes digit row 3q + p = RPC r + g (ACC
//      polynomial q, gadget level p): digits, one forward FFT; thread t then
//      holds bins t + 64 m (m = 0..7) and sends bin t + 64 m to CTA m / MPC
//      (16-byte st.async completing on the receiver's mbarrier): every CTA
//      receives the six rows' spectra at its 64 MPC bins
//   2. CTA c, threads u < 128 (t = u & 63, output polynomial o = u >> 6), for
//      each of its MPC bin columns m: out_o = sum_r x_r C_{r,o},
//      C_{r,o} = sum_c F_c BK_{r,c,o} at bin t + 64 m (the combined-key MAC of
//      k_blind_rotate_u2), sent to every row CTA holding a row of polynomial o
//      (8 KiB per polynomial per receiver, already in the inverse FFT's input
//      layout: thread t, register m)
//   3. those CTAs each inverse-transform out_o (one group per polynomial) and
//      update their own copy of ACC_o: no ACC broadcast hop (an owner-only
//      inverse plus broadcast measured 0.75 vs 0.68-0.73 ms for C = 8)
// Each CTA streams only its bins of the pair's 18 BK stages (36 bulk copies
// of MPC KiB per pair): C = 8 double-buffers them two pairs ahead; C = 4 (twice
// the bins, no room for two buffers) refills its single buffer for pair pm + 1
// as soon as the MAC of pair pm has read it.  Receive buffers are
// double-buffered by pair parity; their reuse two pairs later is ordered by
// the dependency chain itself (no CTA can send for pair pm + 2 before every
// inverter consumed pair pm + 1), so the loop has no cluster barrier.  Same
// arithmetic per (row, component, bin) as the other key-pair kernels; the
// summation order differs, so bit-exactness rests on the FFT rounding margin
// (tests/test_gpu_parity.py narrow levels).
// ---------------------------------------------------------------------------
constexpr uint32_t kBsColBytes = 64 * sizeof(double2);  // one bin column m of one (stage, poly): 1 KiB

template <int C>
struct BsCfg {
    static constexpr int kMPC = 8 / C;                        // bin columns per CTA
    static constexpr int kRowCtas = C == 8 ? 6 : 3;           // CTAs holding digit rows
    static constexpr int kRPC = kRows / kRowCtas;             // digit rows per row CTA
    static constexpr int kBkBufs = C == 8 ? 2 : 1;            // BK slice buffers
    static constexpr uint32_t kBkBytes = kStagesPerPair * 2 * kMPC * kBsColBytes;
    static constexpr uint32_t kSpecBytes = kRows * kMPC * kBsColBytes;
};

template <int C>
struct BrBsSmem {
    using K = BsCfg<C>;
    double2 bk[K::kBkBufs][kStagesPerPair][2][K::kMPC * 64];  // [buf][stage][poly][m_local * 64 + t]
    double2 spec[2][kRows][K::kMPC * 64];                     // [pair parity][row][m_local * 64 + t]
    double2 outp[2][2][8][64];                                // [pair parity][poly][m][t]
    double2 xch[2][kXchStride];                               // group g's FFT exchange
    uint32_t acc[2][kN];                                      // ACC_0 / ACC_1 (the polynomials of this CTA's rows)
    uint16_t bar[kMaxLweN + 1];
    TwSeeds tws[64];
    uint64_t bk_full[K::kBkBufs];
    uint64_t spec_full[2];
    uint64_t out_full[2];
};

// does CTA r hold a digit row of polynomial q?
template <int C>
__host__ __device__ constexpr bool bs_has_poly(int r, int q) {
    return r < BsCfg<C>::kRowCtas && (BsCfg<C>::kRPC * r) / 3 <= q && q <= (BsCfg<C>::kRPC * r + BsCfg<C>::kRPC - 1) / 3;
}

template <int C, bool kDebug>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(192, 1) k_blind_rotate_u2_binsplit(const BrArgs args) {
    using K = BsCfg<C>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrBsSmem<C> &sm = *reinterpret_cast<BrBsSmem<C> *>(smem_raw);
    const int rank = (int)cluster_ctarank();
    const bool row_cta = rank < K::kRowCtas;
    const int warp = threadIdx.x >> 5, grp = warp >> 1, t = threadIdx.x & 63;
    const int u = threadIdx.x & 127;
    const int bar_id = 1 + grp;
    const int n = args.n;
    const int pairs = min(n, args.iters) / 2;
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);
    const uint32_t e = args.e0 + blockIdx.x / C;
    const bool producer = threadIdx.x == 128;  // group 2: BK slices and barrier re-arming
    // this CTA's polynomials (inverse transforms) and its groups' digit rows
    const bool inv0 = bs_has_poly<C>(rank, 0), inv1 = bs_has_poly<C>(rank, 1);
    const int n_inv = (int)inv0 + (int)inv1;
    const int my_row = K::kRPC * rank + grp;  // digit row of a row CTA's group grp < kRPC
    const bool fft_grp = row_cta && grp < K::kRPC;
    const int q_row = my_row / 3, p_row = my_row % 3;
    // inverse transforms: group 0 -> the first polynomial this CTA holds, group 1 -> the second
    const int inv_q = (grp == 0) ? (inv0 ? 0 : 1) : 1;
    const bool inv_grp = (grp == 0 && n_inv >= 1) || (grp == 1 && n_inv == 2);
    const uint32_t out_bytes = (uint32_t)n_inv * 8u * kBsColBytes;

    auto issue_bk = [&](int pm) {
        const int b = K::kBkBufs == 2 ? (pm & 1) : 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // previous generic reads of the buffer
        mbar_arrive_expect_tx(&sm.bk_full[b], K::kBkBytes);
        const char *src = bk_src + (size_t)pm * kStagesPerPair * kRowBytes + (size_t)rank * K::kMPC * kBsColBytes;
#pragma unroll 1
        for (int s = 0; s < kStagesPerPair; s++)
#pragma unroll
            for (int o = 0; o < 2; o++)
                bulk_g2s(&sm.bk[b][s][o][0], src + (size_t)s * kRowBytes + (size_t)o * kNH * sizeof(double2),
                         K::kMPC * kBsColBytes, &sm.bk_full[b]);
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
        for (int b = 0; b < K::kBkBufs; b++) mbar_init(&sm.bk_full[b], 1);
        for (int b = 0; b < 2; b++) {
            mbar_init(&sm.spec_full[b], 1);
            mbar_init(&sm.out_full[b], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (producer) {
        for (int pm = 0; pm < K::kBkBufs && pm < pairs; pm++) issue_bk(pm);
        for (int pm = 0; pm < 2 && pm < pairs; pm++) {
            mbar_arrive_expect_tx(&sm.spec_full[pm], K::kSpecBytes);
            if (n_inv) mbar_arrive_expect_tx(&sm.out_full[pm], out_bytes);
        }
    }
    k1_modswitch(args, e, sm.bar, threadIdx.x, 192);  // K1 (every CTA needs the rotation exponents)
    __syncthreads();
    if (n_inv) acc_init(inv0 ? sm.acc[0] : nullptr, inv1 ? sm.acc[1] : nullptr, sm.bar[n], args.mu, threadIdx.x, 192);
    // every CTA's barriers are initialised and armed, every ACC copy is set
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

    const uint32_t spec_off = smem_addr(&sm.spec[0][0][0]);
    const uint32_t out_off = smem_addr(&sm.outp[0][0][0][0]);
    const uint32_t spec_bar_off = smem_addr(&sm.spec_full[0]);
    const uint32_t out_bar_off = smem_addr(&sm.out_full[0]);
    double max_err = 0.0;
    // F_c at this thread's MAC bins k = t + 64 m: psi^{e_c (4k+1)}, one pair ahead
    double2 base[K::kMPC][3];
    auto load_base = [&](int pm, double2 (&bs)[K::kMPC][3]) {
        const int ai = sm.bar[2 * pm], aj = sm.bar[2 * pm + 1];
#pragma unroll
        for (int ml = 0; ml < K::kMPC; ml++) {
            const int kk = 4 * (t + 64 * (K::kMPC * rank + ml)) + 1;
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const int ec = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
                bs[ml][c] = __ldg(&args.PSI[(ec * kk) & (2 * kN - 1)]);
            }
        }
    };
    if (pairs > 0 && grp < 2) load_base(0, base);
    for (int pm = 0; pm < pairs; pm++) {
        const int b = pm & 1;
        // 1. digit-row groups: digits + forward transform, scattered by bin column
        if (fft_grp) {
            const uint32_t *P = sm.acc[q_row];
            double2 x[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int j = t + 64 * m;
                x[0][m] = make_double2(small_int_to_double(gadget_digit(P[j], p_row)),
                                       small_int_to_double(gadget_digit(P[j + kNH], p_row)));
            }
            nega_fft_fwd_n<1, true>(x, sm.xch[grp], t, sm.tws[t], bar_id);
            const uint32_t lbar = spec_bar_off + (uint32_t)(b * 8);
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const uint32_t dst = (uint32_t)(m / K::kMPC);
                const int ml = m % K::kMPC;
                const uint32_t loc = spec_off + (uint32_t)((((b * kRows + my_row) * K::kMPC + ml) * 64 + t) * 16);
                st_async_f64x2(mapa_u32(loc, dst), x[0][m], mapa_u32(lbar, dst));
            }
        }
        // 2. threads u < 128: the combined-key MAC of all six rows at this CTA's bins, output o
        if (grp < 2) {
            const int o = u >> 6;
            double2 nb[K::kMPC][3];
            if (pm + 1 < pairs) load_base(pm + 1, nb);
            const int bb = K::kBkBufs == 2 ? b : 0;
            const uint32_t bk_par = K::kBkBufs == 2 ? (uint32_t)((pm >> 1) & 1) : (uint32_t)(pm & 1);
            mbar_wait(&sm.bk_full[bb], bk_par);
            mbar_wait_cluster(&sm.spec_full[b], (pm >> 1) & 1);
#pragma unroll
            for (int ml = 0; ml < K::kMPC; ml++) {
                double2 F[3];
#pragma unroll
                for (int c = 0; c < 3; c++) F[c] = make_double2(base[ml][c].x - 1.0, base[ml][c].y);
                const int k = ml * 64 + t;
                double2 acc_o = make_double2(0.0, 0.0);
#pragma unroll
                for (int r = 0; r < kRows; r++) {
                    const int rs = (r >> 1) * 6 + (r & 1);  // stage of (row r, component 0) within the pair
                    double2 Cc = cmul(F[0], sm.bk[bb][rs][o][k]);
                    cmac(Cc, F[1], sm.bk[bb][rs + 2][o][k]);
                    cmac(Cc, F[2], sm.bk[bb][rs + 4][o][k]);
                    cmac(acc_o, sm.spec[b][r][k], Cc);
                }
                // to every CTA inverse-transforming polynomial o, slot [b][o][m][t]
                const int m = K::kMPC * rank + ml;
                const uint32_t loc = out_off + (uint32_t)((((b * 2 + o) * 8 + m) * 64 + t) * 16);
#pragma unroll
                for (int d = 0; d < K::kRowCtas; d++) {
                    if (!bs_has_poly<C>(d, o)) continue;
                    st_async_f64x2(mapa_u32(loc, (uint32_t)d), acc_o,
                                   mapa_u32(out_bar_off + (uint32_t)(b * 8), (uint32_t)d));
                }
            }
            if (pm + 1 < pairs) {
#pragma unroll
                for (int ml = 0; ml < K::kMPC; ml++)
#pragma unroll
                    for (int c = 0; c < 3; c++) base[ml][c] = nb[ml][c];
            }
        }
        // 3. the MAC threads have read this pair's BK slices and spectra: the producer (group
        //    2) re-arms the spectrum barrier for pair pm + 2 and refills the BK buffer (a
        //    complete-tx ahead of the re-arm would be safe: the phase also waits for the
        //    producer's arrival)
        asm volatile("bar.sync %0, %1;" ::"r"(5), "r"(192) : "memory");
        if (producer) {
            if (pm + 2 < pairs) mbar_arrive_expect_tx(&sm.spec_full[b], K::kSpecBytes);
            if (pm + K::kBkBufs < pairs) issue_bk(pm + K::kBkBufs);
        }
        // 4. inverse groups: output polynomial inv_q -> inverse transform -> this CTA's ACC copy
        if (inv_grp) {
            mbar_wait_cluster(&sm.out_full[b], (pm >> 1) & 1);
            if (grp == 0 && t == 0 && pm + 2 < pairs) mbar_arrive_expect_tx(&sm.out_full[b], out_bytes);
            double2 y[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) y[0][m] = sm.outp[b][inv_q][m][t];
            nega_fft_inv_n<1, true>(y, sm.xch[grp], t, sm.tws[t], bar_id);
            uint32_t *P = sm.acc[inv_q];
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
        // the next pair's digit rows read ACC copies another group may have updated
        if (K::kRPC > 1 || n_inv > 1) asm volatile("bar.sync %0, %1;" ::"r"(6), "r"(192) : "memory");
    }
    // no CTA may exit while a peer can still address its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // extraction by the CTA holding row 0 (ACC_0) and the CTA holding row 3 (ACC_1)
    const bool x0 = rank == 0, x1 = rank == 3 / K::kRPC;
    if (kDebug && args.margin && (x0 || x1)) atomicMax(args.margin, (unsigned long long)__double_as_longlong(max_err));
    if (kDebug && args.acc_dump) {
        uint32_t *dst = args.acc_dump + (size_t)e * 2 * kN;
        if (x0)
            for (int c = threadIdx.x; c < kN; c += 192) dst[c] = sm.acc[0][c];
        if (x1)
            for (int c = threadIdx.x; c < kN; c += 192) dst[kN + c] = sm.acc[1][c];
    }
    uint32_t *out = args.big + (size_t)e * kBigStride;
    uint32_t *out2 = x2_row(args, e);  // HA: second extraction at index N/2
    if (x0) {
        const uint32_t *A = sm.acc[0];
        for (int c = threadIdx.x; c < kN; c += 192) out[c] = c == 0 ? A[0] : 0u - A[kN - c];
        if (out2)
            for (int c = threadIdx.x; c < kN; c += 192) out2[c] = c <= kNH ? A[kNH - c] : 0u - A[kN + kNH - c];
    }
    if (x1 && threadIdx.x == 0) {
        out[kN] = sm.acc[1][0];
        if (out2) out2[kN] = sm.acc[1][kNH];
    }
}
