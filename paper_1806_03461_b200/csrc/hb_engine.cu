// B200 (sm_100a) gate-bootstrapping engine: the device half of the
// GateBackend drop-in (reference: /root/reference/pkg/src/hebnn/backend.py
// 205-237, where SimContext only simulates each gate in plaintext).
//
// Kernels:
//   k_bk_to_fourier        K6  BK (u32 coefficients) -> FP64 negacyclic Fourier domain
//   k_blind_rotate_u2      K1+K2+K3 fused, key-pair bootstrapping key (default):
//                          gate linear combination (2 or 3 inputs) + mod switch,
//                          315 external products with the combined TGSW
//                          sum_c (X^e_c - 1) BK_c (gadget decomposition, FP64 FFT in
//                          registers/shared memory, BK stages streamed by
//                          cp.async.bulk into a shared-memory ring and reused by
//                          every gate of the CTA), sample extraction
//   k_blind_rotate_u2_lat  the same for narrow levels: one bootstrap per CTA
//   k_blind_rotate_u2_clu  the same for very narrow levels: one bootstrap per 2-CTA cluster
//   k_blind_rotate[_lat]   CGGI bootstrapping key (bk_unroll 1): 630 CMux steps
//   k_keyswitch            K4  batched LWE key switch (uint32), KSK table chunks
//                          shared by a tile of gates
//   k_gather               pool slots -> contiguous buffer for download
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hb_internal.h"

using namespace hb;

#define HB_CUDA_TRY(expr)                                                                   \
    do {                                                                                    \
        cudaError_t _err = (expr);                                                          \
        if (_err != cudaSuccess) {                                                          \
            set_error(std::string(#expr) + ": " + cudaGetErrorString(_err));               \
            return HB_ECUDA;                                                                \
        }                                                                                   \
    } while (0)

namespace {

#include "hb_dev_fft.cuh"
#include "hb_br_cggi.cuh"
#include "hb_br_u2.cuh"
#include "hb_br_clu6.cuh"
#include "hb_br_binsplit.cuh"
#include "hb_ks.cuh"

}  // namespace

// Work items (blind rotations x lanes) per launch: bounds the extracted-LWE
// scratch (4,112 B per item) to ~4.3 GB for very wide levels.
constexpr size_t kMaxWorkPerLaunch = (size_t)1 << 20;

// ---------------------------------------------------------------------------
// engine object
// ---------------------------------------------------------------------------
struct hb_engine {
    int device = 0;
    hb_params p{};
    cudaStream_t stream = nullptr;
    cudaStream_t h2d_stream = nullptr;    // async uploads overlapping the compute stream
    cudaStream_t d2h_stream = nullptr;    // async downloads
    cudaEvent_t ev_upload = nullptr;      // last async upload (the next level waits on it)
    cudaEvent_t ev_compute = nullptr;     // compute point an async download waits on
    cudaEvent_t ev_prev_level = nullptr;  // compute stream before the most recent level
    cudaEvent_t ev_download = nullptr;    // last async download (pool writers wait on it: no WAR)
    // slot ranges [lo, hi) of the async downloads that may still be reading the pool, each with
    // the d2h-stream event recorded after it; writers wait only for the ones they overlap
    // (older entries are folded into [old_lo, old_hi), fenced by the oldest kept event: the
    // d2h stream is in order)
    static constexpr int kDl = 8;
    cudaEvent_t ev_dl[kDl]{};
    size_t dl_lo[kDl]{}, dl_hi[kDl]{};
    int n_dl = 0, dl_head = 0;            // live entries, ring index of the oldest
    size_t old_lo = 0, old_hi = 0;        // folded ranges (empty when old_lo >= old_hi)
    bool pending_upload = false;
    bool pending_download = false;
    double2 *d_W = nullptr, *d_TW = nullptr, *d_PSI = nullptr;
    int unroll = 1;  // bk_unroll of the loaded key
    double2 *d_bkf = nullptr;
    uint32_t *d_ksk = nullptr;
    uint32_t *d_pool = nullptr;
    size_t pool_cap = 0;
    uint32_t pool_stride = 0;
    uint32_t *d_big = nullptr;
    size_t big_cap = 0;  // extracted-LWE slots
    BrItem *d_br = nullptr;
    size_t br_cap = 0;
    KsItem *d_ks = nullptr;
    size_t ks_cap = 0;
    uint32_t *d_tmp = nullptr;
    size_t tmp_cap = 0;  // words
    uint32_t *d_kspart = nullptr;
    size_t kspart_cap = 0;  // words: narrow-level key-switch partial sums
    void *h_stage = nullptr;
    size_t h_stage_cap = 0;
    unsigned long long *d_margin = nullptr;
    void *d_flush = nullptr;
    size_t flush_bytes = 0;
    uint64_t flush_gen = 1;
    cudaEvent_t ev[4]{};
    cudaEvent_t ev_stage = nullptr;  // item copies out of h_stage done
    cudaEvent_t ev_grow = nullptr;   // pool growth fences between the engine and copy streams
    uint64_t n_br = 0, n_ks = 0, n_launch = 0;
    int num_sms = 148;
    size_t max_work = kMaxWorkPerLaunch;  // HEBNN_B200_MAX_WORK overrides (tests)
    bool latency_mode = true;             // HEBNN_B200_LATENCY_MODE=0 disables (A/B tests)
    bool cluster_mode = true;             // 2-CTA clusters for <= #SM/2 key-pair bootstraps (HEBNN_B200_CLUSTER_MODE=0)
    int bs8_max = 0;                      // co-resident 8-CTA bin-split clusters (lone levels); HEBNN_B200_BINSPLIT=0 off
    int bs4_max = 0;                      // co-resident 4-CTA bin-split clusters
    int clu6_max = 0;                     // co-resident 6-CTA clusters (0: kernel unavailable); HEBNN_B200_CLU6=0 off
    bool split_waves = true;              // wide levels: full 4-bootstrap waves + a faster remainder kernel
                                          // (HEBNN_B200_SPLIT_WAVES=0 off)
    bool u2ws = true;                     // wide key-pair levels: warp-specialised BK producer (HEBNN_B200_U2WS=0 off;
                                          // 31.2 -> 28.5 ms per 4,096)
};

namespace {

// Grow a device scratch buffer used only by work on stream `st`: stream-ordered
// allocation and free (the old buffer is released after the queued kernels that
// use it), so a level wider than any before does not stall the host.
int ensure_dev(void **ptr, size_t *cap, size_t need, size_t elem, bool preserve, cudaStream_t st) {
    if (need <= *cap) return HB_OK;
    size_t ncap = std::max(need, *cap + *cap / 2);
    void *np = nullptr;
    cudaError_t err = cudaMallocAsync(&np, ncap * elem, st);
    if (err != cudaSuccess) {
        set_error(std::string("cudaMallocAsync(") + std::to_string(ncap * elem) + " B): " + cudaGetErrorString(err));
        return HB_ENOMEM;
    }
    if (*ptr) {
        if (preserve && *cap) HB_CUDA_TRY(cudaMemcpyAsync(np, *ptr, *cap * elem, cudaMemcpyDeviceToDevice, st));
        HB_CUDA_TRY(cudaFreeAsync(*ptr, st));
    }
    *ptr = np;
    *cap = ncap;
    return HB_OK;
}

int ensure_host_stage(hb_engine *e, size_t bytes) {
    if (bytes <= e->h_stage_cap) return HB_OK;
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (e->h_stage) cudaFreeHost(e->h_stage);
    size_t ncap = std::max({bytes, e->h_stage_cap * 2, (size_t)32 << 20});  // >= 32 MiB: rare regrowth
    HB_CUDA_TRY(cudaHostAlloc(&e->h_stage, ncap, cudaHostAllocDefault));
    e->h_stage_cap = ncap;
    return HB_OK;
}

template <int G, bool kDebug>
int launch_br(hb_engine *e, const BrArgs &a) {
    const size_t smem = br_smem_bytes<G>();
    const unsigned grid = (a.n_work - a.e0 + G - 1) / G;
    if constexpr (G == kBrGates) {
        if (e->u2ws) {
            k_blind_rotate<G, kDebug, true><<<grid, 64 * G + 128, smem, e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
    }
    k_blind_rotate<G, kDebug><<<grid, 64 * G, smem, e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    return HB_OK;
}

template <int G, bool kDebug, int R = kStagesU2, int MB = 1, bool TM = false, bool WS = false>
int launch_br_u2(hb_engine *e, const BrArgs &a) {
    const unsigned grid = (a.n_work - a.e0 + G - 1) / G;
    k_blind_rotate_u2<G, kDebug, R, MB, TM, WS><<<grid, u2_threads<G, WS>(), sizeof(BrSmemU2<G, R, TM>), e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    return HB_OK;
}

template <bool kDebug>
int launch_br_lat(hb_engine *e, const BrArgs &a) {
    k_blind_rotate_lat<kDebug><<<a.n_work - a.e0, 192, sizeof(BrLatSmem), e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    return HB_OK;
}

// narrow levels: the coefficient range is split over `splits` CTAs per column
// chunk (8, 4 or 2, so that a level launches >= ~640 CTAs) and the partial
// sums are reduced by k_keyswitch_reduce
constexpr int kKsMaxSplits = 8;
constexpr uint32_t kKsTargetCtas = 8 * kKsChunks;

int ks_splits(uint32_t n_work) {
    const uint32_t ctas = ((n_work + kKsThreads - 1) / kKsThreads) * kKsChunks;
    int s = 1;
    while (s < kKsMaxSplits && ctas * (uint32_t)(2 * s) <= kKsTargetCtas) s *= 2;
    return s;
}

int launch_ks(hb_engine *e, const KsArgs &a0) {
    KsArgs a = a0;
    const int splits = ks_splits(a.n_work);
    const bool narrow = splits > 1;
    if (narrow) {
        int rc = ensure_dev((void **)&e->d_kspart, &e->kspart_cap, (size_t)splits * a.n_work * kKskStride,
                            sizeof(uint32_t), false, e->stream);
        if (rc) return rc;
        a.partial = e->d_kspart;
    }
    // only the chunks holding output columns 0..n (79 of 80 at n = 630)
    const uint32_t chunks = (a.n + kKsCols) / kKsCols;
    const dim3 grid((a.n_work + kKsThreads - 1) / kKsThreads, chunks, splits);
    k_keyswitch<<<grid, kKsThreads, 0, e->stream>>>(a);
    HB_CUDA_TRY(cudaGetLastError());
    e->n_launch++;
    if (narrow) {
        k_keyswitch_reduce<<<a.n_work, kKskStride, 0, e->stream>>>(a, splits);
        HB_CUDA_TRY(cudaGetLastError());
        e->n_launch++;
    }
    return HB_OK;
}

#ifndef HB_U2_PAIRED
#define HB_U2_PAIRED 0  // experiment: wide levels as two independent 2-gate CTAs per SM
#endif
#ifndef HB_PAIRED_RING
#define HB_PAIRED_RING 3
#endif
#if HB_U2_PAIRED
constexpr int kPairedRing = HB_PAIRED_RING;
#endif
#ifndef HB_U2_TMEM
#define HB_U2_TMEM 0  // wide key-pair levels: accumulators in tensor memory, deeper BK ring
#endif
#ifndef HB_TMEM_RING
#define HB_TMEM_RING 9
#endif
#if HB_U2_TMEM
constexpr int kStagesU2Tmem = HB_TMEM_RING;
#endif

// Blind-rotation launch for a level of a.n_work bootstraps: narrow levels
// (latency-bound) get one bootstrap per CTA split over three thread groups
// (latency mode) or fewer bootstraps per CTA; wide levels 4 per CTA.
// force_g (debug paths): 4 = the throughput kernel regardless of width.
template <bool kDebug>
int launch_br_auto(hb_engine *e, const BrArgs &a0, int force_g = 0) {
    const uint32_t sms = (uint32_t)e->num_sms;
    BrArgs a = a0;
    // key pairs, wide levels: whole waves of 4-bootstrap CTAs, then the remainder (< one wave)
    // on the kernel that runs it fastest (a 6-CTA cluster per bootstrap ... 3 per CTA) instead
    // of a mostly idle extra 4-bootstrap wave: e.g. 729 bootstraps 8.9 -> ~6.4 ms
    if (e->unroll == 2 && !force_g && e->split_waves) {
        const uint32_t wave = kBrGates * sms, cnt = a.n_work - a.e0;
        if (cnt > wave && cnt % wave != 0 && cnt % wave <= 3 * sms) {
            BrArgs head = a;
            head.n_work = a.e0 + (cnt / wave) * wave;
            int rc = e->u2ws ? launch_br_u2<kBrGates, kDebug, kStagesU2, 1, false, true>(e, head)
                             : launch_br_u2<kBrGates, kDebug>(e, head);
            if (rc) return rc;
            a.e0 = head.n_work;
        }
    }
    const uint32_t cnt = a.n_work - a.e0;
    const int gsel = force_g ? force_g
                             : (cnt <= sms ? 1 : (cnt <= 2u * sms ? 2 : (cnt <= 3u * sms && e->unroll == 2 ? 3 : kBrGates)));
    if (e->unroll == 2) {
        if (!force_g && e->latency_mode && e->cluster_mode && cnt <= (uint32_t)e->bs8_max) {
            k_blind_rotate_u2_binsplit<8, kDebug><<<8 * cnt, 192, sizeof(BrBsSmem<8>), e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
        if (!force_g && e->latency_mode && e->cluster_mode && cnt <= (uint32_t)e->clu6_max) {
            k_blind_rotate_u2_clu6<kDebug><<<kClu6 * cnt, 192, sizeof(BrClu6Smem), e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
        // 4-CTA bin split: 1.21 ms for <= ~32, behind the 6-CTA row split (1.06 ms) but ahead of
        // the 2-CTA kernel (1.39 ms)
        if (!force_g && e->latency_mode && e->cluster_mode && cnt <= (uint32_t)e->bs4_max) {
            k_blind_rotate_u2_binsplit<4, kDebug><<<4 * cnt, 192, sizeof(BrBsSmem<4>), e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
        if (!force_g && e->latency_mode && e->cluster_mode && 2 * cnt <= sms) {
            k_blind_rotate_u2_clu<kDebug><<<2 * cnt, 192, sizeof(BrCluSmemU2), e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
        if (!force_g && gsel == 1 && e->latency_mode) {
            k_blind_rotate_u2_lat<kDebug><<<cnt, 192, sizeof(BrLatSmemU2), e->stream>>>(a);
            HB_CUDA_TRY(cudaGetLastError());
            e->n_launch++;
            return HB_OK;
        }
        if (gsel == 1) return launch_br_u2<1, kDebug>(e, a);
        if (gsel == 2)
            return e->u2ws ? launch_br_u2<2, kDebug, kStagesU2, 1, false, true>(e, a) : launch_br_u2<2, kDebug>(e, a);
        if (gsel == 3)
            return e->u2ws ? launch_br_u2<3, kDebug, kStagesU2, 1, false, true>(e, a) : launch_br_u2<3, kDebug>(e, a);
#if HB_U2_PAIRED
        if (!force_g) return launch_br_u2<2, kDebug, kPairedRing, 2>(e, a);  // two 2-gate CTAs per SM
#endif
#if HB_U2_TMEM
        return launch_br_u2<kBrGates, kDebug, kStagesU2Tmem, 1, true>(e, a);
#else
        if (e->u2ws) return launch_br_u2<kBrGates, kDebug, kStagesU2, 1, false, true>(e, a);
        return launch_br_u2<kBrGates, kDebug>(e, a);
#endif
    }
    if (!force_g && gsel == 1 && e->latency_mode) return launch_br_lat<kDebug>(e, a);
    if (gsel == 1) return launch_br<1, kDebug>(e, a);
    if (gsel == 2) return launch_br<2, kDebug>(e, a);
    return launch_br<kBrGates, kDebug>(e, a);
}

BrArgs br_args(hb_engine *e) {
    BrArgs a{};
    a.pool = e->d_pool;
    a.pool_stride = e->pool_stride;
    a.lanes = 1;
    a.n = e->p.n;
    a.mu = 1u << 29;
    a.bkf = e->d_bkf;
    a.big = e->d_big;
    a.W = e->d_W;
    a.TW = e->d_TW;
    a.PSI = e->d_PSI;
    a.iters = e->p.n;
    return a;
}

int32_t pack_coef(int alpha, int beta, int gamma = 0) {
    return (int32_t)((uint32_t)(uint8_t)(int8_t)alpha | ((uint32_t)(uint8_t)(int8_t)beta << 8) |
                     ((uint32_t)(uint8_t)(int8_t)gamma << 16));
}

}  // namespace

extern "C" {

int hb_engine_create(int device, const hb_params *p, const uint32_t *bk, const uint32_t *ksk, hb_engine **out) {
    if (!out || !params_ok(p) || !bk || !ksk) {
        set_error("hb_engine_create: unsupported parameters or null argument");
        return HB_EINVAL;
    }
    *out = nullptr;
    int ndev = 0;
    HB_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) {
        set_error("hb_engine_create: CUDA device " + std::to_string(device) + " not present (" +
                  std::to_string(ndev) + " visible)");
        return HB_ECUDA;
    }
    HB_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    HB_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error("hb_engine_create: kernels are built for sm_100a (B200); device is sm_" +
                  std::to_string(prop.major) + std::to_string(prop.minor));
        return HB_ECUDA;
    }
    hb_engine *e = new hb_engine();
    e->device = device;
    e->p = *p;
    e->pool_stride = (uint32_t)((p->n + 1 + 3) & ~3);
    HB_CUDA_TRY(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    if (const char *k = std::getenv("HEBNN_B200_POOL_KEEP_MB")) {  // experiment: mempool release threshold
        cudaMemPool_t mp;
        HB_CUDA_TRY(cudaDeviceGetDefaultMemPool(&mp, device));
        uint64_t keep = std::strtoull(k, nullptr, 10) << 20;
        HB_CUDA_TRY(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    for (auto &ev : e->ev) HB_CUDA_TRY(cudaEventCreate(&ev));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_stage, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_grow, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaStreamCreateWithFlags(&e->h2d_stream, cudaStreamNonBlocking));
    HB_CUDA_TRY(cudaStreamCreateWithFlags(&e->d2h_stream, cudaStreamNonBlocking));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_upload, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_compute, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_prev_level, cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_download, cudaEventDisableTiming));
    for (int i = 0; i < hb_engine::kDl; i++) HB_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_dl[i], cudaEventDisableTiming));
    HB_CUDA_TRY(cudaEventRecord(e->ev_prev_level, e->stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_stage, e->stream));

    // twiddle tables, computed in long double then rounded
    std::vector<double2> W(kNH), TW(kNH);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int j = 0; j < kNH; j++) {
        long double th = 2.0L * pi * j / kNH;
        W[j] = make_double2((double)cosl(th), (double)sinl(th));
        long double ph = pi * j / kN;
        TW[j] = make_double2((double)cosl(ph), (double)sinl(ph));
    }
    std::vector<double2> PSI(2 * kN);
    for (int u = 0; u < 2 * kN; u++) {
        long double ph = pi * u / kN;
        PSI[u] = make_double2((double)cosl(ph), (double)sinl(ph));
    }
    HB_CUDA_TRY(cudaMalloc(&e->d_PSI, 2 * kN * sizeof(double2)));
    HB_CUDA_TRY(cudaMemcpy(e->d_PSI, PSI.data(), 2 * kN * sizeof(double2), cudaMemcpyHostToDevice));
    e->unroll = bk_unroll(p);
    HB_CUDA_TRY(cudaMalloc(&e->d_W, kNH * sizeof(double2)));
    HB_CUDA_TRY(cudaMalloc(&e->d_TW, kNH * sizeof(double2)));
    HB_CUDA_TRY(cudaMemcpy(e->d_W, W.data(), kNH * sizeof(double2), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMemcpy(e->d_TW, TW.data(), kNH * sizeof(double2), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMalloc(&e->d_margin, sizeof(unsigned long long)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<kBrGates, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<kBrGates>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<2>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<1>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<kBrGates, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<kBrGates>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<kBrGates, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<kBrGates>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<kBrGates, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<kBrGates>()));
#if HB_U2_TMEM
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, false, kStagesU2Tmem, 1, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates, kStagesU2Tmem, true>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, true, kStagesU2Tmem, 1, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates, kStagesU2Tmem, true>)));
#endif
#if HB_U2_PAIRED
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, false, kPairedRing, 2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<2, kPairedRing>)));
#endif
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, false, kStagesU2, 1, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BrSmemU2<kBrGates>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<3, false, kStagesU2, 1, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BrSmemU2<3>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<3, true, kStagesU2, 1, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BrSmemU2<3>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, false, kStagesU2, 1, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BrSmemU2<2>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, true, kStagesU2, 1, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BrSmemU2<2>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, true, kStagesU2, 1, false, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BrSmemU2<kBrGates>)));
    if (const char *uw = std::getenv("HEBNN_B200_U2WS")) e->u2ws = std::atoi(uw) != 0;
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_clu6<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrClu6Smem)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_clu6<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrClu6Smem)));
    {  // how many 6-CTA clusters fit at once (GPC-limited); narrower levels use them
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kClu6 * 64);
        cfg.blockDim = dim3(192);
        cfg.dynamicSmemBytes = sizeof(BrClu6Smem);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_blind_rotate_u2_clu6<false>, &cfg) != cudaSuccess) {
            cudaGetLastError();
            ncl = 0;
        }
        e->clu6_max = ncl;
        if (const char *c6 = std::getenv("HEBNN_B200_CLU6"))
            if (std::atoi(c6) == 0) e->clu6_max = 0;
    }
    {  // bin-split latency kernels: as many clusters as fit at once (GPC-limited)
        auto setup = [&](auto kern, auto kdbg, size_t smem, int csize, int *max_out) {
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
                cudaFuncSetAttribute(kdbg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
                cudaGetLastError();
                *max_out = 0;
                return;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(csize * 32);
            cfg.blockDim = dim3(192);
            cfg.dynamicSmemBytes = smem;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) {
                cudaGetLastError();
                ncl = 0;
            }
            *max_out = ncl;
        };
        setup(k_blind_rotate_u2_binsplit<8, false>, k_blind_rotate_u2_binsplit<8, true>, sizeof(BrBsSmem<8>), 8,
              &e->bs8_max);
        setup(k_blind_rotate_u2_binsplit<4, false>, k_blind_rotate_u2_binsplit<4, true>, sizeof(BrBsSmem<4>), 4,
              &e->bs4_max);
        if (const char *bs = std::getenv("HEBNN_B200_BINSPLIT")) {
            const int v = std::atoi(bs);
            if (v == 0 || v == 4) e->bs8_max = 0;  // 4: only the 4-CTA kernel (A/B)
            if (v == 0 || v == 8) e->bs4_max = 0;
        }
    }
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<kBrGates, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<kBrGates>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<2>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<3>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<3>)));
    if (const char *sw = std::getenv("HEBNN_B200_SPLIT_WAVES")) e->split_waves = std::atoi(sw) != 0;
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<1>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<2>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrSmemU2<1>)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<2>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)br_smem_bytes<1>()));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_clu<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrCluSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_clu<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrCluSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_lat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_u2_lat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmemU2)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_lat<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmem)));
    HB_CUDA_TRY(cudaFuncSetAttribute(k_blind_rotate_lat<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(BrLatSmem)));
    HB_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    e->num_sms = prop.multiProcessorCount;
    if (const char *mw = std::getenv("HEBNN_B200_MAX_WORK")) e->max_work = std::max<size_t>(2, std::strtoull(mw, nullptr, 10));
    if (const char *lm = std::getenv("HEBNN_B200_LATENCY_MODE")) e->latency_mode = std::atoi(lm) != 0;
    if (const char *cm = std::getenv("HEBNN_B200_CLUSTER_MODE")) e->cluster_mode = std::atoi(cm) != 0;

    // BK -> Fourier
    const size_t npoly = bk_tgsw_count(p) * kRows * 2;
    uint32_t *d_bk = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_bk, npoly * kN * sizeof(uint32_t)));
    HB_CUDA_TRY(cudaMemcpy(d_bk, bk, npoly * kN * sizeof(uint32_t), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMalloc(&e->d_bkf, npoly * kNH * sizeof(double2)));
    k_bk_to_fourier<<<(unsigned)((npoly + 1) / 2), 128, 0, e->stream>>>(d_bk, e->d_bkf, (int)npoly, e->d_W, e->d_TW,
                                                                         e->unroll);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    cudaFree(d_bk);

    // KSK
    const size_t ksk_rows = (size_t)kN * kKsT * kKsVals;
    uint32_t *d_kin = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_kin, ksk_rows * (p->n + 1) * sizeof(uint32_t)));
    HB_CUDA_TRY(cudaMemcpy(d_kin, ksk, ksk_rows * (p->n + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice));
    HB_CUDA_TRY(cudaMalloc(&e->d_ksk, kKsTableWords * sizeof(uint32_t)));
    k_ksk_relayout<<<kKsRelayoutBlocks, 256, 0, e->stream>>>(d_kin, e->d_ksk, p->n);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    cudaFree(d_kin);
    *out = e;
    return HB_OK;
}

int hb_engine_destroy(hb_engine *e) {
    if (!e) return HB_OK;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (void *ptr : {(void *)e->d_W, (void *)e->d_TW, (void *)e->d_PSI, (void *)e->d_bkf, (void *)e->d_ksk, (void *)e->d_pool,
                      (void *)e->d_big, (void *)e->d_br, (void *)e->d_ks, (void *)e->d_tmp, (void *)e->d_kspart, (void *)e->d_margin,
                      e->d_flush})
        if (ptr) cudaFree(ptr);
    if (e->h_stage) cudaFreeHost(e->h_stage);
    for (auto &ev : e->ev)
        if (ev) cudaEventDestroy(ev);
    if (e->ev_stage) cudaEventDestroy(e->ev_stage);
    if (e->ev_grow) cudaEventDestroy(e->ev_grow);
    for (cudaStream_t st : {e->h2d_stream, e->d2h_stream})
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    for (cudaEvent_t ev : {e->ev_upload, e->ev_compute, e->ev_prev_level, e->ev_download})
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : e->ev_dl)
        if (ev) cudaEventDestroy(ev);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
    return HB_OK;
}

// Write-after-read fence: a pool write issued after hb_pool_download_async must not
// overtake the copy still reading those slots on the d2h stream (the header's
// double-buffered pattern rewrites step k-2's output slots at step k).
static int order_after_downloads(hb_engine *e, cudaStream_t st) {
    if (e->pending_download) {
        HB_CUDA_TRY(cudaStreamWaitEvent(st, e->ev_download, 0));
        if (st == e->stream) {  // later stream-ordered writers inherit it
            e->pending_download = false;
            e->n_dl = 0;
            e->old_lo = e->old_hi = 0;
        }
    }
    return HB_OK;
}

// The same fence for a writer of physical pool slots [lo, hi) only: it waits for the
// pending downloads that read any of those slots (a double-buffered client's upload of
// step k + 1 and the key switch of level k + 1 write the other slot region than the
// download of step k, so they no longer wait for it).  Completed entries are dropped.
static int order_after_downloads_range(hb_engine *e, cudaStream_t st, size_t lo, size_t hi) {
    if (!e->pending_download) return HB_OK;
    if (lo >= hi) return HB_OK;
    // drop finished downloads from the head (oldest first)
    while (e->n_dl > 0 && cudaEventQuery(e->ev_dl[e->dl_head]) == cudaSuccess) {
        e->dl_head = (e->dl_head + 1) % hb_engine::kDl;
        e->n_dl--;
        e->old_lo = e->old_hi = 0;  // everything older than the new head completed too
    }
    cudaGetLastError();  // cudaEventQuery's cudaErrorNotReady is not an error here
    if (e->n_dl == 0) {
        e->pending_download = false;
        return HB_OK;
    }
    const bool old_hit = e->old_lo < e->old_hi && lo < e->old_hi && e->old_lo < hi;
    int last_hit = -1;  // the newest overlapping entry (waiting on it covers all older ones)
    for (int k = 0; k < e->n_dl; k++) {
        const int i = (e->dl_head + k) % hb_engine::kDl;
        if (lo < e->dl_hi[i] && e->dl_lo[i] < hi) last_hit = i;
    }
    if (last_hit >= 0) {
        HB_CUDA_TRY(cudaStreamWaitEvent(st, e->ev_dl[last_hit], 0));
    } else if (old_hit) {
        HB_CUDA_TRY(cudaStreamWaitEvent(st, e->ev_dl[e->dl_head], 0));
    }
    return HB_OK;
}

// Pool growth is stream-ordered (cudaMallocAsync / copy / cudaFreeAsync on the
// engine stream, fenced against both copy streams), so growing the pool while
// levels are queued never blocks the host: the gate DAG keeps being built while
// a background flush runs.
int hb_pool_reserve(hb_engine *e, size_t slots) {
    if (!e) return HB_EINVAL;
    if (slots <= e->pool_cap) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    const size_t ncap = std::max(slots, e->pool_cap + e->pool_cap / 2);
    uint32_t *np = nullptr;
    cudaError_t err = cudaMallocAsync((void **)&np, ncap * e->pool_stride * sizeof(uint32_t), e->stream);
    if (err != cudaSuccess) {
        set_error(std::string("cudaMallocAsync(pool, ") + std::to_string(ncap * e->pool_stride * 4) +
                  " B): " + cudaGetErrorString(err));
        return HB_ENOMEM;
    }
    if (e->d_pool) {
        // copies already queued on the copy streams read / write the old buffer: order them first
        for (cudaStream_t st : {e->h2d_stream, e->d2h_stream}) {
            HB_CUDA_TRY(cudaEventRecord(e->ev_grow, st));
            HB_CUDA_TRY(cudaStreamWaitEvent(e->stream, e->ev_grow, 0));
        }
        HB_CUDA_TRY(cudaMemcpyAsync(np, e->d_pool, e->pool_cap * e->pool_stride * sizeof(uint32_t),
                                    cudaMemcpyDeviceToDevice, e->stream));
        HB_CUDA_TRY(cudaFreeAsync(e->d_pool, e->stream));
        // later copies on the copy streams address the new buffer after its contents arrived
        HB_CUDA_TRY(cudaEventRecord(e->ev_grow, e->stream));
        for (cudaStream_t st : {e->h2d_stream, e->d2h_stream}) HB_CUDA_TRY(cudaStreamWaitEvent(st, e->ev_grow, 0));
    }
    e->d_pool = np;
    e->pool_cap = ncap;
    return HB_OK;
}

size_t hb_pool_capacity(const hb_engine *e) { return e ? e->pool_cap : 0; }
size_t hb_pool_stride(const hb_engine *e) { return e ? e->pool_stride : 0; }

int hb_pool_upload(hb_engine *e, size_t first, size_t count, const uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_upload: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = order_after_downloads(e, e->stream)) return rc;
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_pool + first * e->pool_stride, e->pool_stride * 4, host, host_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyHostToDevice, e->stream));
    return HB_OK;
}

int hb_pool_download(hb_engine *e, size_t first, size_t count, uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_download: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaMemcpy2DAsync(host, host_stride * 4, e->d_pool + first * e->pool_stride, e->pool_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_pool_gather_device(hb_engine *e, const uint32_t *slots, size_t count, uint32_t *dev_out, size_t dev_stride) {
    if (!e || (count && (!slots || !dev_out)) || dev_stride < (size_t)e->p.n + 1) {
        set_error("hb_pool_gather_device: bad arguments");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    for (size_t i = 0; i < count; i++)
        if (slots[i] >= e->pool_cap) {
            set_error("hb_pool_gather_device: slot beyond pool capacity");
            return HB_EINVAL;
        }
    HB_CUDA_TRY(cudaSetDevice(e->device));
    int rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, count, sizeof(uint32_t), false, e->stream);
    if (rc) return rc;
    rc = ensure_host_stage(e, count * sizeof(uint32_t));
    if (rc) return rc;
    HB_CUDA_TRY(cudaEventSynchronize(e->ev_stage));
    std::memcpy(e->h_stage, slots, count * sizeof(uint32_t));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_tmp, e->h_stage, count * sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
    k_gather<<<(unsigned)count, 256, 0, e->stream>>>(e->d_pool, e->pool_stride, e->d_tmp, (uint32_t)count,
                                                    (uint32_t)e->p.n + 1, dev_out, dev_stride);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    e->n_launch++;
    return HB_OK;
}

int hb_pool_put_device(hb_engine *e, size_t first_slot, size_t count, const uint32_t *dev_in, size_t dev_stride) {
    if (!e || (count && !dev_in) || dev_stride < (size_t)e->p.n + 1 || first_slot + count > e->pool_cap) {
        set_error("hb_pool_put_device: bad arguments or slots beyond pool capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = order_after_downloads(e, e->stream)) return rc;
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_pool + first_slot * e->pool_stride, (size_t)e->pool_stride * 4, dev_in,
                                  dev_stride * 4, ((size_t)e->p.n + 1) * 4, count, cudaMemcpyDeviceToDevice, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_pool_gather(hb_engine *e, const uint32_t *slots, size_t count, uint32_t *host, size_t host_stride) {
    if (!e || (count && (!slots || !host)) || host_stride < (size_t)e->p.n + 1) {
        set_error("hb_pool_gather: bad arguments");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    for (size_t i = 0; i < count; i++)
        if (slots[i] >= e->pool_cap) {
            set_error("hb_pool_gather: slot beyond pool capacity");
            return HB_EINVAL;
        }
    HB_CUDA_TRY(cudaSetDevice(e->device));
    const uint32_t words = (uint32_t)e->p.n + 1;
    const size_t need = count + (count * words + 3) / 1;
    int rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, need, sizeof(uint32_t), false, e->stream);
    if (rc) return rc;
    rc = ensure_host_stage(e, count * sizeof(uint32_t));
    if (rc) return rc;
    HB_CUDA_TRY(cudaEventSynchronize(e->ev_stage));
    std::memcpy(e->h_stage, slots, count * sizeof(uint32_t));
    uint32_t *d_slots = e->d_tmp, *d_out = e->d_tmp + count;
    HB_CUDA_TRY(cudaMemcpyAsync(d_slots, e->h_stage, count * sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
    k_gather<<<(unsigned)count, 256, 0, e->stream>>>(e->d_pool, e->pool_stride, d_slots, (uint32_t)count, words, d_out,
                                                    words);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaMemcpy2DAsync(host, host_stride * 4, d_out, (size_t)words * 4, (size_t)words * 4, count,
                                  cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    e->n_launch++;
    return HB_OK;
}

static int run_gates_chunk(hb_engine *e, const hb_gate *gates, size_t n, uint32_t lanes);

int hb_run_gates(hb_engine *e, const hb_gate *gates, size_t n, uint32_t lanes) {
    if (!e || (n && !gates) || lanes == 0) {
        set_error("hb_run_gates: bad arguments");
        return HB_EINVAL;
    }
    if (!n) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    // gates of one level are independent: split very wide levels into chunks
    const size_t per_chunk = std::max<size_t>(1, e->max_work / (2 * (size_t)lanes));
    nvtxRangePushA("hb_run_gates");  // NVTX range per level (visible in nsys timelines)
    for (size_t off = 0; off < n; off += per_chunk) {
        const int rc = run_gates_chunk(e, gates + off, std::min(per_chunk, n - off), lanes);
        if (rc) {
            nvtxRangePop();
            return rc;
        }
    }
    nvtxRangePop();
    return HB_OK;
}

static int run_gates_chunk(hb_engine *e, const hb_gate *gates, size_t n, uint32_t lanes) {
    // expand records into blind-rotation and key-switch work items
    size_t nbr = 0, nha = 0;
    size_t dst_lo = SIZE_MAX, dst_hi = 0;  // slots the key switch writes
    for (size_t i = 0; i < n; i++) {
        const hb_gate &g = gates[i];
        if (g.kind != HB_GATE_LIN2 && g.kind != HB_GATE_MUX && g.kind != HB_GATE_LIN3 && g.kind != HB_GATE_HA) {
            set_error("hb_run_gates: unknown gate kind " + std::to_string((int)g.kind));
            return HB_EINVAL;
        }
        if (g.kind == HB_GATE_HA && ((g.gamma != 1 && g.gamma != -1) || g.dst == g.src_c)) {
            set_error("hb_run_gates: HA record needs gamma = +-1 and dst != src_c");
            return HB_EINVAL;
        }
        nha += g.kind == HB_GATE_HA;
        const size_t top = (size_t)std::max(std::max(g.dst, g.src_a), std::max(g.src_b, g.src_c)) + 1;
        if (top * lanes > e->pool_cap) {
            set_error("hb_run_gates: slot beyond pool capacity");
            return HB_EINVAL;
        }
        nbr += (g.kind == HB_GATE_MUX) ? 2 : 1;
        dst_lo = std::min(dst_lo, (size_t)g.dst);
        dst_hi = std::max(dst_hi, (size_t)g.dst + 1);
        if (g.kind == HB_GATE_HA) {  // the XOR output
            dst_lo = std::min(dst_lo, (size_t)g.src_c);
            dst_hi = std::max(dst_hi, (size_t)g.src_c + 1);
        }
    }
    // big-LWE rows: one per blind rotation, then one per HA second extraction
    const size_t nks = n + nha, nbig = nbr + nha;
    const size_t br_bytes = nbr * sizeof(BrItem), ks_bytes = nks * sizeof(KsItem);
    int rc = ensure_host_stage(e, br_bytes + ks_bytes);
    if (rc) return rc;
    // the pinned stage fed the previous level's item copies; wait for those copies only,
    // so the host builds level k+1 while the device still runs level k
    HB_CUDA_TRY(cudaEventSynchronize(e->ev_stage));
    BrItem *hbr = reinterpret_cast<BrItem *>(e->h_stage);
    KsItem *hks = reinterpret_cast<KsItem *>(reinterpret_cast<char *>(e->h_stage) + br_bytes);
    size_t b = 0, h = 0;
    const uint32_t eighth = 1u << 29;
    for (size_t i = 0; i < n; i++) {
        const hb_gate &g = gates[i];
        if (g.kind == HB_GATE_LIN2) {
            hbr[b] = BrItem{g.src_a, g.src_b, g.src_a, g.c0, pack_coef(g.alpha, g.beta), kNoItem};
            hks[i] = KsItem{g.dst, (uint32_t)b, 0xFFFFFFFFu, 0u};
            b += 1;
        } else if (g.kind == HB_GATE_HA) {
            // one blind rotation, extractions S0 (row b) and S1 (row nbr + h); AND = KS(S0),
            // XOR = KS(gamma (S1 - S0) + (0, -gamma/8)) (oracle/tfhe_oracle.c or_half_adder)
            const uint32_t s0 = (uint32_t)b, s1 = (uint32_t)(nbr + h);
            hbr[b] = BrItem{g.src_a, g.src_b, g.src_a, g.c0, pack_coef(g.alpha, g.beta), s1};
            hks[i] = KsItem{g.dst, s0, 0xFFFFFFFFu, 0u};
            hks[n + h] = g.gamma > 0 ? KsItem{g.src_c, s1, s0 | kKsSub, 0u - eighth}
                                     : KsItem{g.src_c, s0, s1 | kKsSub, eighth};
            b += 1;
            h += 1;
        } else if (g.kind == HB_GATE_LIN3) {
            hbr[b] = BrItem{g.src_a, g.src_b, g.src_c, g.c0, pack_coef(g.alpha, g.beta, g.gamma), kNoItem};
            hks[i] = KsItem{g.dst, (uint32_t)b, 0xFFFFFFFFu, 0u};
            b += 1;
        } else {
            hbr[b] = BrItem{g.src_a, g.src_b, g.src_a, 0u - eighth, pack_coef(1, g.alpha), kNoItem};
            hbr[b + 1] = BrItem{g.src_a, g.src_c, g.src_a, 0u - eighth, pack_coef(-1, g.beta), kNoItem};
            hks[i] = KsItem{g.dst, (uint32_t)b, (uint32_t)(b + 1), eighth};
            b += 2;
        }
    }
    if ((rc = ensure_dev((void **)&e->d_br, &e->br_cap, nbr, sizeof(BrItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_ks, &e->ks_cap, nks, sizeof(KsItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, nbig * lanes * kBigStride, sizeof(uint32_t), false,
                         e->stream)))
        return rc;
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_br, hbr, br_bytes, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_ks, hks, ks_bytes, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_stage, e->stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_prev_level, e->stream));  // "everything before this level"
    if (e->pending_upload) {  // inputs staged by hb_pool_upload_async
        HB_CUDA_TRY(cudaStreamWaitEvent(e->stream, e->ev_upload, 0));
        e->pending_upload = false;
    }

    BrArgs a = br_args(e);
    a.lanes = lanes;
    a.items = e->d_br;
    a.n_work = (uint32_t)(nbr * lanes);
    HB_CUDA_TRY(cudaEventRecord(e->ev[0], e->stream));
    if ((rc = launch_br_auto<false>(e, a))) return rc;
    HB_CUDA_TRY(cudaEventRecord(e->ev[1], e->stream));
    KsArgs k{};
    k.big = e->d_big;
    k.items = e->d_ks;
    k.lanes = lanes;
    k.n_work = (uint32_t)(nks * lanes);
    k.ksk = e->d_ksk;
    k.pool = e->d_pool;
    k.pool_stride = e->pool_stride;
    k.n = e->p.n;
    // the key switch writes pool slots [dst_lo, dst_hi) x lanes: after any async download
    // still reading them
    if ((rc = order_after_downloads_range(e, e->stream, dst_lo * lanes, dst_hi * lanes))) return rc;
    if ((rc = launch_ks(e, k))) return rc;
    HB_CUDA_TRY(cudaEventRecord(e->ev[2], e->stream));
    e->n_br += nbr * lanes;
    e->n_ks += nks * lanes;
    return HB_OK;
}

int hb_sync(hb_engine *e) {
    if (!e) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->h2d_stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->d2h_stream));
    return HB_OK;
}

int hb_pool_upload_async(hb_engine *e, size_t first, size_t count, const uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_upload_async: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    // may overlap the most recently issued level, never an earlier one (double buffering)
    HB_CUDA_TRY(cudaStreamWaitEvent(e->h2d_stream, e->ev_prev_level, 0));
    if (int rc = order_after_downloads_range(e, e->h2d_stream, first, first + count)) return rc;
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_pool + first * e->pool_stride, e->pool_stride * 4, host, host_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyHostToDevice, e->h2d_stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_upload, e->h2d_stream));
    e->pending_upload = true;
    return HB_OK;
}

int hb_pool_download_async(hb_engine *e, size_t first, size_t count, uint32_t *host, size_t host_stride) {
    if (!e || (count && !host) || host_stride < (size_t)e->p.n + 1 || first + count > e->pool_cap) {
        set_error("hb_pool_download_async: bad arguments or slot range beyond capacity");
        return HB_EINVAL;
    }
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    // everything issued so far on the compute stream (the levels producing these slots)
    HB_CUDA_TRY(cudaEventRecord(e->ev_compute, e->stream));
    HB_CUDA_TRY(cudaStreamWaitEvent(e->d2h_stream, e->ev_compute, 0));
    HB_CUDA_TRY(cudaMemcpy2DAsync(host, host_stride * 4, e->d_pool + first * e->pool_stride, e->pool_stride * 4,
                                  (size_t)(e->p.n + 1) * 4, count, cudaMemcpyDeviceToHost, e->d2h_stream));
    HB_CUDA_TRY(cudaEventRecord(e->ev_download, e->d2h_stream));
    if (e->n_dl == hb_engine::kDl) {  // fold the oldest entry into the catch-all range
        const int i = e->dl_head;
        if (e->old_lo >= e->old_hi) {
            e->old_lo = e->dl_lo[i];
            e->old_hi = e->dl_hi[i];
        } else {
            e->old_lo = std::min(e->old_lo, e->dl_lo[i]);
            e->old_hi = std::max(e->old_hi, e->dl_hi[i]);
        }
        e->dl_head = (e->dl_head + 1) % hb_engine::kDl;
        e->n_dl--;
    }
    const int slot = (e->dl_head + e->n_dl) % hb_engine::kDl;
    HB_CUDA_TRY(cudaEventRecord(e->ev_dl[slot], e->d2h_stream));
    e->dl_lo[slot] = first;
    e->dl_hi[slot] = first + count;
    e->n_dl++;
    e->pending_download = true;
    return HB_OK;
}

int hb_last_timing(hb_engine *e, float *br_ms, float *ks_ms) {
    if (!e) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    HB_CUDA_TRY(cudaEventSynchronize(e->ev[2]));
    float x = 0, y = 0;
    HB_CUDA_TRY(cudaEventElapsedTime(&x, e->ev[0], e->ev[1]));
    HB_CUDA_TRY(cudaEventElapsedTime(&y, e->ev[1], e->ev[2]));
    if (br_ms) *br_ms = x;
    if (ks_ms) *ks_ms = y;
    return HB_OK;
}

int hb_counters(hb_engine *e, uint64_t *brs, uint64_t *kss, uint64_t *launches) {
    if (!e) return HB_EINVAL;
    if (brs) *brs = e->n_br;
    if (kss) *kss = e->n_ks;
    if (launches) *launches = e->n_launch;
    return HB_OK;
}

int hb_debug_blind_rotate(hb_engine *e, const uint32_t *lwe, uint32_t mu, int32_t iters, uint32_t *acc_out) {
    if (!e || !lwe || !acc_out) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    const size_t words = e->p.n + 1;
    int rc;
    if ((rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, 2 * words + 4 * kN + 64, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_br, &e->br_cap, 1, sizeof(BrItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, kBigStride, sizeof(uint32_t), false, e->stream))) return rc;
    uint32_t *d_in = e->d_tmp, *d_acc = e->d_tmp + ((2 * words + 3) & ~size_t(3));
    BrItem it{0, 0, 0, 0, pack_coef(1, 0)};
    HB_CUDA_TRY(cudaMemcpyAsync(d_in, lwe, words * 4, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_br, &it, sizeof it, cudaMemcpyHostToDevice, e->stream));
    BrArgs a = br_args(e);
    a.pool = d_in;
    a.pool_stride = (uint32_t)words;
    a.items = e->d_br;
    a.n_work = 1;
    a.mu = mu;
    if (iters >= 100000) {  // debug A/B: BK rows read from global instead of the ring
        iters -= 100000;
        a.n_work = 2;
        a.lanes = 2;
    }
    a.iters = iters < 0 ? e->p.n : iters;
    a.acc_dump = d_acc;
    if ((rc = launch_br_auto<true>(e, a, kBrGates))) return rc;
    HB_CUDA_TRY(cudaMemcpyAsync(acc_out, d_acc, 2 * kN * 4, cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_debug_bootstrap_wo_ks(hb_engine *e, const uint32_t *lin, size_t count, uint32_t *out) {
    if (!e || (count && (!lin || !out))) return HB_EINVAL;
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    const size_t words = e->p.n + 1;
    int rc;
    if ((rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, count * words, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_br, &e->br_cap, count, sizeof(BrItem), false, e->stream))) return rc;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, count * kBigStride, sizeof(uint32_t), false, e->stream)))
        return rc;
    std::vector<BrItem> items(count);
    for (size_t i = 0; i < count; i++) items[i] = BrItem{(uint32_t)i, (uint32_t)i, (uint32_t)i, 0u, pack_coef(1, 0), kNoItem};
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_tmp, lin, count * words * 4, cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_br, items.data(), count * sizeof(BrItem), cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemsetAsync(e->d_margin, 0, sizeof(unsigned long long), e->stream));
    BrArgs a = br_args(e);
    a.pool = e->d_tmp;
    a.pool_stride = (uint32_t)words;
    a.items = e->d_br;
    a.n_work = (uint32_t)count;
    a.margin = e->d_margin;
    if ((rc = launch_br_auto<true>(e, a, kBrGates))) return rc;
    HB_CUDA_TRY(cudaMemcpy2DAsync(out, (size_t)(kN + 1) * 4, e->d_big, kBigStride * 4, (size_t)(kN + 1) * 4, count,
                                  cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

int hb_flush_l2(hb_engine *e, size_t bytes) {
    if (!e) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    if (!bytes) bytes = (size_t)256 << 20;
    if (bytes > e->flush_bytes) {
        if (e->d_flush) cudaFree(e->d_flush);
        e->d_flush = nullptr;
        HB_CUDA_TRY(cudaMalloc(&e->d_flush, bytes));
        e->flush_bytes = bytes;
    }
    HB_CUDA_TRY(cudaMemsetAsync(e->d_flush, (int)(e->flush_gen++ & 0xFF), bytes, e->stream));
    return HB_OK;
}

int hb_measure_fp64_peak(hb_engine *e, double *tflops) {
    if (!e || !tflops) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    cudaDeviceProp prop;
    HB_CUDA_TRY(cudaGetDeviceProperties(&prop, e->device));
    double *d_out = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_out, sizeof(double)));
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    k_dfma_peak<<<blocks, threads, 0, e->stream>>>(d_out, iters, 0.999999, 1e-7);  // warm-up
    HB_CUDA_TRY(cudaEventRecord(e->ev[0], e->stream));
    for (int r = 0; r < 5; r++) k_dfma_peak<<<blocks, threads, 0, e->stream>>>(d_out, iters, 0.999999, 1e-7);
    HB_CUDA_TRY(cudaEventRecord(e->ev[1], e->stream));
    HB_CUDA_TRY(cudaEventSynchronize(e->ev[1]));
    float ms = 0;
    HB_CUDA_TRY(cudaEventElapsedTime(&ms, e->ev[0], e->ev[1]));
    cudaFree(d_out);
    *tflops = 5.0 * 2.0 * 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
    return HB_OK;
}

int hb_debug_fourier(hb_engine *e, const uint32_t *polys, size_t count, double *out, int which) {
    if (!e || (count && (!polys || !out))) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    if (which == 1) {  // download rows of the device BK Fourier table
        HB_CUDA_TRY(cudaMemcpy(out, e->d_bkf, count * kNH * sizeof(double2), cudaMemcpyDeviceToHost));
        return HB_OK;
    }
    uint32_t *d_in = nullptr;
    double2 *d_out = nullptr;
    HB_CUDA_TRY(cudaMalloc(&d_in, count * kN * 4));
    HB_CUDA_TRY(cudaMalloc(&d_out, count * kNH * sizeof(double2)));
    HB_CUDA_TRY(cudaMemcpy(d_in, polys, count * kN * 4, cudaMemcpyHostToDevice));
    k_bk_to_fourier<<<(unsigned)((count + 1) / 2), 128, 0, e->stream>>>(d_in, d_out, (int)count, e->d_W, e->d_TW, 1);
    HB_CUDA_TRY(cudaGetLastError());
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    HB_CUDA_TRY(cudaMemcpy(out, d_out, count * kNH * sizeof(double2), cudaMemcpyDeviceToHost));
    cudaFree(d_in);
    cudaFree(d_out);
    return HB_OK;
}

int hb_debug_fft_margin(hb_engine *e, double *max_err) {
    if (!e || !max_err) return HB_EINVAL;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    unsigned long long bits = 0;
    HB_CUDA_TRY(cudaMemcpy(&bits, e->d_margin, sizeof bits, cudaMemcpyDeviceToHost));
    std::memcpy(max_err, &bits, sizeof(double));
    return HB_OK;
}

int hb_debug_keyswitch(hb_engine *e, const uint32_t *in, size_t count, uint32_t *out) {
    if (!e || (count && (!in || !out))) return HB_EINVAL;
    if (!count) return HB_OK;
    HB_CUDA_TRY(cudaSetDevice(e->device));
    int rc;
    const size_t words = e->p.n + 1;
    if ((rc = ensure_dev((void **)&e->d_big, &e->big_cap, count * kBigStride, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_tmp, &e->tmp_cap, count * e->pool_stride, sizeof(uint32_t), false, e->stream)))
        return rc;
    if ((rc = ensure_dev((void **)&e->d_ks, &e->ks_cap, count, sizeof(KsItem), false, e->stream))) return rc;
    std::vector<KsItem> items(count);
    for (size_t i = 0; i < count; i++) items[i] = KsItem{(uint32_t)i, (uint32_t)i, 0xFFFFFFFFu, 0u};
    HB_CUDA_TRY(cudaMemcpy2DAsync(e->d_big, kBigStride * 4, in, (size_t)(kN + 1) * 4, (size_t)(kN + 1) * 4, count,
                                  cudaMemcpyHostToDevice, e->stream));
    HB_CUDA_TRY(cudaMemcpyAsync(e->d_ks, items.data(), count * sizeof(KsItem), cudaMemcpyHostToDevice, e->stream));
    KsArgs k{};
    k.big = e->d_big;
    k.items = e->d_ks;
    k.lanes = 1;
    k.n_work = (uint32_t)count;
    k.ksk = e->d_ksk;
    k.pool = e->d_tmp;
    k.pool_stride = e->pool_stride;
    k.n = e->p.n;
    if ((rc = launch_ks(e, k))) return rc;
    HB_CUDA_TRY(cudaMemcpy2DAsync(out, words * 4, e->d_tmp, e->pool_stride * 4, words * 4, count,
                                  cudaMemcpyDeviceToHost, e->stream));
    HB_CUDA_TRY(cudaStreamSynchronize(e->stream));
    return HB_OK;
}

}  // extern "C"
