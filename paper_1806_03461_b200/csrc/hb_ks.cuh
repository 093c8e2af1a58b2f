// hb_ks.cuh: key switch, key-switch table relayout, gather and FP64 peak probe kernels
// (textually included by hb_engine.cu inside its anonymous namespace;
// not a standalone header)
#pragma once

// ---------------------------------------------------------------------------
// K4: batched key switch.  For coefficient i the CGGI digits are the eight
// base-4 digits of w_i = (a'_i + 2^15) >> 16, and the key switch subtracts
// KS[i][j][d_j] (d_j = 0 contributes nothing) from (0.., b).
//
// HB_KS_PAIR = 1 (default): digits are consumed in pairs.  The device table
// holds, per coefficient i, digit pair p and output column c, the 16 sums
//   T[chunk][i][p][c][d] = KS[i][2p][d >> 2] + KS[i][2p+1][d & 3]  (mod 2^32)
// The input is big[i0] (+ or - big[i1], KsItem flag kKsSub) formed on the fly.
// (64 B: 16 consecutive banks), so one digit pair costs one conflict-free
// LDS.32 per column (lanes with equal d broadcast, different d hit different
// banks): 8 wavefronts per warp per digit PAIR, half of the one-digit layout,
// and half the integer adds.  Sums mod 2^32 are exact in any order, so the
// result is bit-identical to the digit-by-digit key switch.
// HB_KS_PAIR = 0: T[chunk][i][j][d][8] with T[..][0][..] = 0; one digit costs
// two LDS.128 (the 4 candidate rows of an (i, j) fill one 128-B line).
// CTA = 128 gates (one per thread) x one 8-column chunk; the chunk's table
// streams through a shared-memory ring fed by cp.async.bulk, so every table
// byte fetched from L2 serves 128 gates.
// ---------------------------------------------------------------------------
#ifndef HB_KS_PAIR
#define HB_KS_PAIR 1
#endif
struct KsArgs {
    const uint32_t *big;     // [n_br_work][kBigStride]
    const KsItem *items;     // [n_items]
    uint32_t lanes;
    uint32_t n_work;         // n_items * lanes
    const uint32_t *ksk;     // device lookup table (layout above)
    uint32_t *pool;
    uint32_t pool_stride;
    int32_t n;
    uint32_t *partial;       // narrow levels: [splits][n_work][kKskStride] raw sums (else null)
};

constexpr int kKsCols = 8;                               // output columns per chunk
constexpr int kKsChunks = kKskStride / kKsCols;           // 80
#ifndef HB_KS_THREADS
#define HB_KS_THREADS 128
#endif
constexpr int kKsThreads = HB_KS_THREADS;                 // one gate per thread
constexpr int kKsRowsPerI = HB_KS_PAIR ? (kKsT / 2) * 16 : kKsT * 4;  // table rows per coefficient
constexpr int kKsIBlock = HB_KS_PAIR ? 4 : 8;             // coefficients per ring stage
constexpr uint32_t kKsStageBytes = kKsIBlock * kKsRowsPerI * kKsCols * 4;  // 8 KiB
constexpr int kKsStages = HB_KS_PAIR ? 5 : 4;
constexpr size_t kKsTableWords = (size_t)kKsChunks * kN * kKsRowsPerI * kKsCols;

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
    const bool has1 = it.i1 != kNoItem, sub = has1 && (it.i1 & kKsSub);
    const uint32_t *b1 = has1 ? args.big + ((size_t)(it.i1 & ~kKsSub) * lanes + lane_id) * kBigStride : nullptr;
    const int chunk = blockIdx.y;
    // blockIdx.z splits the coefficient range (narrow levels: more CTAs, shorter streams)
    const int kBlocks = (kN / kKsIBlock) / gridDim.z;
    const int blk0 = blockIdx.z * kBlocks;
    const char *tab_src = reinterpret_cast<const char *>(args.ksk) + (size_t)chunk * kN * kKsRowsPerI * kKsCols * 4 +
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
    // this thread's extracted-LWE coefficients, kKsIBlock per block (uint4 loads)
    constexpr int kW4 = kKsIBlock / 4;
    const uint4 *wsrc0 = reinterpret_cast<const uint4 *>(b0) + kW4 * blk0;
    const uint4 *wsrc1 = b1 ? reinterpret_cast<const uint4 *>(b1) + kW4 * blk0 : nullptr;
    uint4 w[kW4];
#pragma unroll
    for (int q = 0; q < kW4; q++) {
        w[q] = __ldg(wsrc0 + q);
        if (b1) {
            uint4 x = __ldg(wsrc1 + q);
            if (sub) x = make_uint4(0u - x.x, 0u - x.y, 0u - x.z, 0u - x.w);
            w[q] = make_uint4(w[q].x + x.x, w[q].y + x.y, w[q].z + x.z, w[q].w + x.w);
        }
    }
#pragma unroll 1
    for (int blk = 0; blk < kBlocks; blk++) {
        if (threadIdx.x == 0) {
            const int nx = blk + kKsStages - 1;
            if (nx < kBlocks) {
                const int s2 = nx % kKsStages;
                if (nx >= kKsStages) mbar_wait(&ks.empty[s2], ((nx / kKsStages) - 1) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot before its async-proxy refill
                mbar_arrive_expect_tx(&ks.full[s2], kKsStageBytes);
                bulk_g2s(ks.tab[s2], tab_src + (size_t)nx * kKsStageBytes, kKsStageBytes, &ks.full[s2]);
            }
        }
        __syncwarp();
        uint32_t v[kKsIBlock];
#pragma unroll
        for (int q = 0; q < kW4; q++) {
            v[4 * q] = w[q].x; v[4 * q + 1] = w[q].y; v[4 * q + 2] = w[q].z; v[4 * q + 3] = w[q].w;
        }
        if (blk + 1 < kBlocks) {  // prefetch the next block's coefficients
#pragma unroll
            for (int q = 0; q < kW4; q++) {
                w[q] = __ldg(wsrc0 + kW4 * (blk + 1) + q);
                if (b1) {
                    uint4 x = __ldg(wsrc1 + kW4 * (blk + 1) + q);
                    if (sub) x = make_uint4(0u - x.x, 0u - x.y, 0u - x.z, 0u - x.w);
                    w[q] = make_uint4(w[q].x + x.x, w[q].y + x.y, w[q].z + x.z, w[q].w + x.w);
                }
            }
        }
        const int s = blk % kKsStages;
        mbar_wait(&ks.full[s], (blk / kKsStages) & 1);
#if HB_KS_PAIR
        const uint32_t *tab = reinterpret_cast<const uint32_t *>(ks.tab[s]);
#pragma unroll
        for (int ii = 0; ii < kKsIBlock; ii++) {
            const uint32_t word = (v[ii] + (1u << 15)) >> 16;
#pragma unroll
            for (int jp = 0; jp < kKsT / 2; jp++) {
                const uint32_t d = (word >> (12 - 4 * jp)) & 15u;
                const uint32_t *row = tab + (ii * (kKsT / 2) + jp) * (kKsCols * 16) + d;
#pragma unroll
                for (int c = 0; c < kKsCols; c++) acc[c] += row[16 * c];
            }
        }
#else
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
#endif
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
        if (b1) bval += (sub ? 0u - b1[kN] : b1[kN]) + it.cadd;
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
        if (it.i1 != kNoItem) {
            const uint32_t v1 = args.big[((size_t)(it.i1 & ~kKsSub) * lanes + lane_id) * kBigStride + kN];
            bval += ((it.i1 & kKsSub) ? 0u - v1 : v1) + it.cadd;
        }
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

// KSK host layout [kN][t][3][n+1] -> device lookup table (layout: K4 above).
// HB_KS_PAIR: T[chunk][i][p][cc][d] = KS[i][2p][d >> 2] + KS[i][2p+1][d & 3].
// HB_KS_PAIR = 0: T[chunk][i][j][d][kKsCols] = KS[i][j][d] (d = 0 row is 0).
__global__ void k_ksk_relayout(const uint32_t *__restrict__ in, uint32_t *__restrict__ out, int n) {
#if HB_KS_PAIR
    const size_t ip = blockIdx.x;  // i * (t / 2) + p
    const size_t i = ip / (kKsT / 2), p = ip % (kKsT / 2);
    const uint32_t *src0 = in + (i * kKsT + 2 * p) * 3 * (size_t)(n + 1);
    const uint32_t *src1 = src0 + 3 * (size_t)(n + 1);
    for (int w = threadIdx.x; w < kKskStride * 16; w += blockDim.x) {
        const int d = w / kKskStride, col = w % kKskStride;
        const int d0 = d >> 2, d1 = d & 3;
        uint32_t val = 0;
        if (col <= n) {
            if (d0) val += src0[(size_t)(d0 - 1) * (n + 1) + col];
            if (d1) val += src1[(size_t)(d1 - 1) * (n + 1) + col];
        }
        const int chunk = col / kKsCols, cc = col % kKsCols;
        out[(((size_t)chunk * kN * (kKsT / 2) + ip) * kKsCols + cc) * 16 + d] = val;
    }
#else
    const size_t ij = blockIdx.x;  // i * t + j
    const uint32_t *src = in + ij * 3 * (size_t)(n + 1);
    for (int w = threadIdx.x; w < kKskStride * 4; w += blockDim.x) {
        const int d = w / kKskStride, col = w % kKskStride;
        const uint32_t val = (d == 0 || col > n) ? 0u : src[(size_t)(d - 1) * (n + 1) + col];
        const int chunk = col / kKsCols, cc = col % kKsCols;
        out[(((size_t)chunk * kN * kKsT + ij) * 4 + d) * kKsCols + cc] = val;
    }
#endif
}
constexpr unsigned kKsRelayoutBlocks = kN * (HB_KS_PAIR ? kKsT / 2 : kKsT);

constexpr int kBrGates = 4;  // bootstraps per CTA (64 threads each)

template <int G>
constexpr size_t br_smem_bytes() {
    return sizeof(BrSmem<G>);
}
