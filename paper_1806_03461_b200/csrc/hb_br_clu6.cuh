// hb_br_clu6.cuh: lone-bootstrap latency kernel, key pairs, one bootstrap per 6-CTA cluster
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once

// ---------------------------------------------------------------------------
// k_blind_rotate_u2_clu6: a level of at most one bootstrap per six SMs (the
// lone and near-lone levels at the tail of every reduce tree / comparator).
// CTA r of the cluster owns digit row r = 3q + p of every key pair (ACC
// polynomial q, gadget level p); CTA 3q ("owner" of q) also inverse-transforms
// output polynomial q and holds the authoritative ACC_q.  Per key pair:
//   1. group 0: digits of ACC_q at level p, one forward FFT -> spectrum (smem)
//   2. threads u < 128: all three components at bins u + 128 m (m = 0..3):
//      MAC of the spectrum with the component's BK stage, F_c = psi^{e_c (4k+1)}
//      - 1 applied on the fly (psi^{512 e m} = i^{e m}: one table value per
//      component), into this CTA's partials of BOTH output polynomials (no
//      shared-memory reduction: a thread owns its bins); the stages for pair
//      pm+2 are then fetched into the freed slots
//   3. the same threads send the partial of output o to owner o with st.async
//      (DSMEM stores completing on the owner's mbarrier)
//   4. owner, group 0: waits for the six partials (48 KiB of transaction bytes),
//      sums them, inverse FFT, rounds, updates ACC_q and broadcasts it to its two
//      siblings with st.async; the owner's group 2 re-arms the receive barrier and
//      frees the six senders' slots (remote release-arrives, off group 0's path)
// No cluster-wide barrier inside the loop: every consumer waits only for the
// bytes it needs (mbarrier transaction counts).  Per key pair ~6.6k cycles
// (forward FFT 1.3k, MAC 1.0k, send 0.45k, partial wait ~1.8k, sum 0.45k,
// inverse 1.0k, broadcast 0.5k; clock64 trace, HB_TRACE=1) against ~8.7k for the
// 2-CTA kernel: a lone level 1.06 ms instead of 1.43 ms.  Tried and slower:
// every CTA of q receiving all six partials and inverse-transforming redundantly
// (no broadcast hop, 3x the st.async volume: 1.14 ms) and the partials moved by
// the bulk-copy engine (cp.async.bulk shared::cta -> shared::cluster: 1.18 ms).
// Same arithmetic per (row, component, bin) as the other key-pair kernels; the
// summation order of the partials differs, so bit-exactness rests on the FFT
// rounding margin like everywhere else (tests/test_gpu_parity.py narrow levels).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64x2(uint32_t raddr, double2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "d"(v.x), "d"(v.y), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_u32x4(uint32_t raddr, uint4 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t rbar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

constexpr int kClu6 = 6;
constexpr int kClu6FreeBar = 5;  // named barrier: owner group 0 (arrive) -> group 2 (sync), 128 threads
constexpr uint32_t kPartBytes = kNH * sizeof(double2);  // one output polynomial's spectrum: 8 KiB

struct BrClu6Smem {
    double2 bk[2][3][2 * kNH];     // [pair parity][component][output poly][bin]
    double2 recv[kClu6][kNH];      // owners: the six CTAs' partials of output polynomial q
    double2 spec[kNH];             // forward spectrum of this CTA's digit row
    double2 xch[kXchStride];       // group 0's FFT exchange (forward and inverse)
    uint32_t acc[kN];              // ACC_q (owner: authoritative; siblings: broadcast copy)
    uint16_t bar[kMaxLweN + 1];
    TwSeeds tws[64];
    uint64_t full[2][3];           // BK stages landed
    uint64_t part_full;            // owners: the six partials landed (transaction bytes)
    uint64_t acc_full;             // siblings: the owner's new ACC_q landed (transaction bytes)
    uint64_t slot_free[2];         // owner o consumed this CTA's previous partial (remote arrive)
};

template <bool kDebug>
__global__ void __cluster_dims__(kClu6, 1, 1) __launch_bounds__(192, 1) k_blind_rotate_u2_clu6(const BrArgs args) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    BrClu6Smem &sm = *reinterpret_cast<BrClu6Smem *>(smem_raw);
    const uint32_t rank = cluster_ctarank();
    const int q = (int)rank / 3, p = (int)rank % 3;  // ACC polynomial and gadget level of this CTA's row
    const int row = 3 * q + p, rp = row >> 1, h = row & 1;
    const bool owner = p == 0;
    const int warp = threadIdx.x >> 5, grp = warp >> 1, t = threadIdx.x & 63;
    const int u = threadIdx.x & 127;  // MAC / send threads: u < 128 (groups 0 and 1)
    const int bar_id = 1 + grp;
    const int n = args.n;
    const int pairs = min(n, args.iters) / 2;
    const char *bk_src = reinterpret_cast<const char *>(args.bkf);
    const uint32_t e = args.e0 + blockIdx.x / kClu6;
    auto stage_src = [&](int pm, int c) {
        return bk_src + (size_t)(pm * kStagesPerPair + rp * 6 + c * 2 + h) * kRowBytes;
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
        for (int b = 0; b < 2; b++)
            for (int c = 0; c < 3; c++) mbar_init(&sm.full[b][c], 1);
        mbar_init(&sm.part_full, 1);
        mbar_init(&sm.acc_full, 1);
        mbar_init(&sm.slot_free[0], 1);
        mbar_init(&sm.slot_free[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (t == 0) {  // component grp's stages of pairs 0 and 1
        for (int pm = 0; pm < 2 && pm < pairs; pm++) {
            mbar_arrive_expect_tx(&sm.full[pm][grp], kRowBytes);
            bulk_g2s(sm.bk[pm][grp], stage_src(pm, grp), kRowBytes, &sm.full[pm][grp]);
        }
    }
    k1_modswitch(args, e, sm.bar, threadIdx.x, 192);  // K1
    __syncthreads();
    acc_init(q == 0 ? sm.acc : nullptr, q == 0 ? nullptr : sm.acc, sm.bar[n], args.mu, threadIdx.x, 192);
    if (threadIdx.x == 0 && pairs > 0) {
        if (owner) mbar_arrive_expect_tx(&sm.part_full, kClu6 * kPartBytes);    // pair 0's partials
        else if (pairs > 1) mbar_arrive_expect_tx(&sm.acc_full, kN * 4);        // pair 0's new ACC_q
    }
    // every CTA's barriers are initialised and armed, every ACC copy is set
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");

    const uint32_t recv_local = smem_addr(&sm.recv[rank][0]);  // our slot in an owner's recv (same offset)
    double max_err = 0.0;
    for (int pm = 0; pm < pairs; pm++) {
        const int ai = sm.bar[2 * pm], aj = sm.bar[2 * pm + 1];
        // the three component monomials at this thread's bins, loaded now: their L2 latency
        // overlaps step 1
        int ex[3];
        double2 base[3];
#pragma unroll
        for (int c = 0; c < 3; c++) {
            ex[c] = c == 0 ? ((ai + aj) & (2 * kN - 1)) : (c == 1 ? ai : aj);
            base[c] = __ldg(&args.PSI[(ex[c] * (4 * u + 1)) & (2 * kN - 1)]);
        }
        // 1. digits + forward transform of row (q, p)
        if (grp == 0) {
            if (!owner && pm > 0) {
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
#pragma unroll
            for (int m = 0; m < 8; m++) sm.spec[t + 64 * m] = x[0][m];
        }
        __syncthreads();  // spectrum published
        // 2. threads u < 128: all three components at bins k = u + 128 m into partials of both
        //    output polynomials
        double2 f0[4], f1[4];
        if (grp < 2) {
            double2 sp[4];
#pragma unroll
            for (int m = 0; m < 4; m++) {
                sp[m] = sm.spec[u + 128 * m];
                f0[m] = f1[m] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int c = 0; c < 3; c++) {
                mbar_wait(&sm.full[pm & 1][c], (pm >> 1) & 1);
                const double2 *b0 = sm.bk[pm & 1][c], *b1 = sm.bk[pm & 1][c] + kNH;
#pragma unroll
                for (int m = 0; m < 4; m++) {
                    const int k = u + 128 * m;
                    const double2 bs = base[c];
                    double2 pw;
                    switch ((ex[c] * m) & 3) {  // i^{e m} * base
                        case 0: pw = bs; break;
                        case 1: pw = make_double2(-bs.y, bs.x); break;
                        case 2: pw = make_double2(-bs.x, -bs.y); break;
                        default: pw = make_double2(bs.y, -bs.x); break;
                    }
                    const double2 y = cmul(sp[m], make_double2(pw.x - 1.0, pw.y));
                    cmac(f0[m], y, b0[k]);
                    cmac(f1[m], y, b1[k]);
                }
            }
        }
        __syncthreads();  // this pair's BK slots and the spectrum consumed
        if (t == 0 && pm + 2 < pairs) {  // component grp's stage of pair pm + 2 into the freed slot
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive_expect_tx(&sm.full[pm & 1][grp], kRowBytes);
            bulk_g2s(sm.bk[pm & 1][grp], stage_src(pm + 2, grp), kRowBytes, &sm.full[pm & 1][grp]);
        }
        if (owner && grp == 2) {  // frees recv for the next pair once group 0 has summed it (step 4)
            asm volatile("bar.sync %0, %1;" ::"r"(kClu6FreeBar), "r"(128) : "memory");
            if (t == 0 && pm + 1 < pairs) mbar_arrive_expect_tx(&sm.part_full, kClu6 * kPartBytes);
            if (t < kClu6) mbar_arrive_remote(mapa_u32(smem_addr(&sm.slot_free[q]), t));  // one sender each
        }
        // 3. threads u < 128: the partial of output polynomial o goes to owner o (CTA 3o)
        if (grp < 2) {
#pragma unroll
            for (int o = 0; o < 2; o++) {
                const uint32_t dst_rank = 3 * o;
                if (pm > 0) mbar_wait_cluster(&sm.slot_free[o], (pm - 1) & 1);  // owner o read our previous one
                const uint32_t raddr = mapa_u32(recv_local, dst_rank);
                const uint32_t rbar = mapa_u32(smem_addr(&sm.part_full), dst_rank);
#pragma unroll
                for (int m = 0; m < 4; m++)
                    st_async_f64x2(raddr + (uint32_t)(u + 128 * m) * 16u, o ? f1[m] : f0[m], rbar);
            }
        }
        // 4. owner: the six partials of output polynomial q -> inverse transform -> ACC_q
        if (owner && grp == 0) {
            mbar_wait_cluster(&sm.part_full, pm & 1);
            double2 y[1][8];
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int k = t + 64 * m;
                double2 v = cadd(cadd(sm.recv[0][k], sm.recv[1][k]), sm.recv[2][k]);
                y[0][m] = cadd(v, cadd(cadd(sm.recv[3][k], sm.recv[4][k]), sm.recv[5][k]));
            }
            // recv consumed: group 2 (idle) re-arms part_full and frees the senders' slots —
            // the remote release-arrives cost ~1k cycles, kept off group 0's critical path
            asm volatile("bar.arrive %0, %1;" ::"r"(kClu6FreeBar), "r"(128) : "memory");
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
            if (pm + 1 < pairs) {
                group_bar(bar_id);  // ACC_q complete in shared memory
                const uint32_t acc_off = smem_addr(&sm.acc[0]), bar_off = smem_addr(&sm.acc_full);
                // 16-byte chunks: 1024 words = 256 chunks, 4 per thread, to both siblings
#pragma unroll
                for (int k4 = 0; k4 < 4; k4++) {
                    const int w = 4 * (t + 64 * k4);
                    const uint4 v = *reinterpret_cast<const uint4 *>(&sm.acc[w]);
#pragma unroll
                    for (int sib = 1; sib < 3; sib++) {
                        const uint32_t r = 3 * q + sib;
                        st_async_u32x4(mapa_u32(acc_off + 4u * w, r), v, mapa_u32(bar_off, r));
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
