// hb_br_u2s.cuh: key-pair blind rotation, two bootstraps sharing every warp (wide levels)
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once

// ---------------------------------------------------------------------------
// k_blind_rotate_u2s: the external products of k_blind_rotate_u2 (same key
// layout, same stage stream, same per-(row, component, bin) arithmetic) with
// the Fourier MAC reading each bootstrapping-key value from shared memory
// ONCE for two bootstraps.
//
// Why: in k_blind_rotate_u2 every bootstrap of a CTA loads every BK stage
// value from shared memory (295 KB per bootstrap and key pair) and the FFT
// exchanges move another 262 KB: with the ring's bulk-copy writes the shared-
// memory port is ~75% busy per key pair, which bounds the kernel as much as the
// FP64 pipe does.
//
// Layout: the CTA's four bootstraps form two pairs; pair P runs on warps
// 4P .. 4P+3, bootstrap A of the pair on lanes 0-15 and bootstrap B on lanes
// 16-31 of each of those warps (t = 16 w' + (lane & 15) is the thread's index
// inside its bootstrap's 64-thread FFT group, so the transforms, digit
// extraction, ACC update and sample extraction are those of u2; a named
// barrier covers the pair's 128 threads).  After the forward transform of a
// row pair, lanes l and l ^ 16 (same t, bootstraps A and B) swap half of their
// spectra with two warp shuffles per value: the lower lane then holds bins
// t + 64 m, m = 0..3, of BOTH bootstraps and the upper lane bins m = 4..7.  The
// MAC loads each BK value once and applies it to both bootstraps (F_c of each
// bootstrap at those bins); before the inverse transforms the accumulators are
// swapped back.  Shared-memory traffic per bootstrap and key pair: 148 KB of
// BK loads instead of 295, plus 16 KB of shuffles.
// ---------------------------------------------------------------------------
constexpr int kU2sBT = 128;  // threads per bootstrap pair (named-barrier count)

__device__ __forceinline__ double2 shfl_xor_d2(double2 v, int mask) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, mask), __shfl_xor_sync(0xffffffffu, v.y, mask));
}

template <bool kDebug, bool WS = false>
__global__ void __launch_bounds__(256 + (WS ? 128 : 0), 1) k_blind_rotate_u2s(const BrArgs args) {
    constexpr int G = 4, R = kStagesU2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrSmemU2<G, R, false> &sm = *reinterpret_cast<BrSmemU2<G, R, false> *>(smem_raw);
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
            mbar_init(&sm.empty[s], 8);  // one arrival per warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (; !WS && issued < R && issued < stages_needed; issued++) {
            mbar_arrive_expect_tx(&sm.full[issued], kRowBytes);
            bulk_g2s(sm.bk[issued], bk_src + (size_t)issued * kRowBytes, kRowBytes, &sm.full[issued]);
        }
    }
    __syncthreads();
    if (WS) {
        if (warp >= 8) {  // producer warpgroup
            asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
            if (threadIdx.x == 256) {
#pragma unroll 1
                for (int s = 0; s < stages_needed; s++) {
                    const int slot = s % R;
                    if (s >= R) mbar_wait(&sm.empty[slot], ((s / R) - 1) & 1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_arrive_expect_tx(&sm.full[slot], kRowBytes);
                    bulk_g2s(sm.bk[slot], bk_src + (size_t)s * kRowBytes, kRowBytes, &sm.full[slot]);
                }
            }
            return;
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
    }

    const int P = warp >> 2;                 // bootstrap pair
    const int hb = lane >> 4;                // 0: bootstrap A of the pair, 1: B (= half of the bins after the swap)
    const int t = 16 * (warp & 3) + (lane & 15);
    const int g = 2 * P + hb;                // bootstrap of this CTA
    const int bar_id = 1 + P;
    const uint32_t e_raw = args.e0 + blockIdx.x * G + g;
    const bool active = e_raw < args.n_work;
    const uint32_t e = active ? e_raw : args.n_work - 1;
    uint32_t *accA = sm.acc[g][0];
    uint32_t *accB = sm.acc[g][1];
    double2 *xch = &sm.xch[g][0][0];
    const uint16_t *barA = sm.bar[2 * P], *barB = sm.bar[2 * P + 1];

    k1_modswitch(args, e, sm.bar[g], t, 64);  // K1
    group_bar_n<kU2sBT>(bar_id);
    acc_init(accA, accB, sm.bar[g][n], args.mu, t, 64);  // ACC = X^{-barb} (0, mu...mu)
    group_bar_n<kU2sBT>(bar_id);

    double max_err = 0.0;
    int st = 0;  // next stage to consume
    for (int pm = 0; pm < pairs; pm++) {
        // F_c of both bootstraps at this thread's MAC bins k = t + 64 (m + 4 hb), m = 0..3:
        // psi^{e (4t+1)} w8^{e m} (-1)^{e hb} - 1
        int ex[2][3];
        double2 base[2][3];
#pragma unroll
        for (int s = 0; s < 2; s++) {
            const uint16_t *bb = s ? barB : barA;
            const int ai = bb[2 * pm], aj = bb[2 * pm + 1];
#pragma unroll
            for (int c = 0; c < 3; c++) {
                ex[s][c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
                base[s][c] = __ldg(&args.PSI[(ex[s][c] * (4 * t + 1)) & (2 * kN - 1)]);
            }
        }
        double2 f0[2][4], f1[2][4];  // [bootstrap A/B][m]: output polys 0/1 at bins t + 64 (m + 4 hb)
#pragma unroll
        for (int s = 0; s < 2; s++)
#pragma unroll
            for (int m = 0; m < 4; m++) f0[s][m] = f1[s][m] = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int rp = 0; rp < kRows / 2; rp++) {
            if (!WS && threadIdx.x == 0) {  // producer: refill the ring up to R stages ahead of this row pair
#pragma unroll 1
                for (; issued < st + R && issued < stages_needed; issued++) {
                    const int s2 = issued % R;
                    mbar_wait(&sm.empty[s2], ((issued / R) - 1) & 1);
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before its async-proxy refill
                    mbar_arrive_expect_tx(&sm.full[s2], kRowBytes);
                    bulk_g2s(sm.bk[s2], bk_src + (size_t)issued * kRowBytes, kRowBytes, &sm.full[s2]);
                }
            }
            __syncwarp();
            double2 x[2][8];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int row = 2 * rp + h;
                const int q = row / kL, p = row % kL;
                const uint32_t *Pp = q ? accB : accA;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const int j = t + 64 * m;
                    x[h][m] = make_double2(small_int_to_double(gadget_digit(Pp[j], p)),
                                           small_int_to_double(gadget_digit(Pp[j + kNH], p)));
                }
            }
            nega_fft_fwd_n<2, true, kU2sBT>(x, xch, t, sm.tws[t], bar_id);
            // swap: y[h][s][m] = spectrum of row h of bootstrap s at bin t + 64 (m + 4 hb)
            double2 y[2][2][4];
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    const double2 lo = x[h][m], hi = x[h][m + 4];
                    const double2 r = shfl_xor_d2(hb ? lo : hi, 16);
                    y[h][0][m] = hb ? r : lo;
                    y[h][1][m] = hb ? hi : r;
                }
#pragma unroll
            for (int c = 0; c < 3; c++, st += 2) {
                const int s0 = st % R, s1 = (st + 1) % R;
                mbar_wait(&sm.full[s0], (st / R) & 1);
                mbar_wait(&sm.full[s1], ((st + 1) / R) & 1);
                const double2 *b00 = sm.bk[s0], *b01 = sm.bk[s0] + kNH;  // row h = 0: output polys 0 / 1
                const double2 *b10 = sm.bk[s1], *b11 = sm.bk[s1] + kNH;  // row h = 1
                long long flip[2];
#pragma unroll
                for (int s = 0; s < 2; s++) flip[s] = (long long)(ex[s][c] & hb & 1) << 63;
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    const int k = t + 64 * (m + 4 * hb);
                    const double2 B00 = b00[k], B01 = b01[k], B10 = b10[k], B11 = b11[k];
#pragma unroll
                    for (int s = 0; s < 2; s++) {
                        const double2 pw = m == 0 ? base[s][c] : cmul(base[s][c], c_w8[(ex[s][c] * m) & 7]);
                        const double2 F = make_double2(__longlong_as_double(__double_as_longlong(pw.x) ^ flip[s]) - 1.0,
                                                       __longlong_as_double(__double_as_longlong(pw.y) ^ flip[s]));
                        const double2 z0 = cmul(y[0][s][m], F), z1 = cmul(y[1][s][m], F);
                        cmac(f0[s][m], z0, B00);
                        cmac(f1[s][m], z0, B01);
                        cmac(f0[s][m], z1, B10);
                        cmac(f1[s][m], z1, B11);
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sm.empty[s0]);
                    mbar_arrive(&sm.empty[s1]);
                }
                __syncwarp();
            }
        }
        {
            // swap back: this thread's bootstrap hb at bins t + 64 m, m = 0..7
            double2 x[2][8];
#pragma unroll
            for (int m = 0; m < 4; m++) {
                const double2 r0 = shfl_xor_d2(hb ? f0[0][m] : f0[1][m], 16);
                const double2 r1 = shfl_xor_d2(hb ? f1[0][m] : f1[1][m], 16);
                x[0][m] = hb ? r0 : f0[0][m];
                x[0][m + 4] = hb ? f0[1][m] : r0;
                x[1][m] = hb ? r1 : f1[0][m];
                x[1][m + 4] = hb ? f1[1][m] : r1;
            }
            nega_fft_inv_n<2, true, kU2sBT>(x, xch, t, sm.tws[t], bar_id);
            if (kDebug) {
#pragma unroll
                for (int q = 0; q < 2; q++)
#pragma unroll
                    for (int m = 0; m < 8; m++) {
                        max_err = fmax(max_err, fabs(x[q][m].x - rint(x[q][m].x)));
                        max_err = fmax(max_err, fabs(x[q][m].y - rint(x[q][m].y)));
                    }
            }
#pragma unroll
            for (int q = 0; q < 2; q++) {
                uint32_t *Pp = q ? accB : accA;
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    const int j = t + 64 * m;
                    Pp[j] += round_to_torus(x[q][m].x);
                    Pp[j + kNH] += round_to_torus(x[q][m].y);
                }
            }
        }
        group_bar_n<kU2sBT>(bar_id);
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
