// tcgen05.cp / tcgen05.ld probe for BK staging through tensor memory.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tmem_probe scripts/tmem_cp_probe.cu
// 1. mapping: a 64 x 16 B shared-memory column (row r at offset 16 r, no swizzle) copied with
//    tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 must land in TMEM lanes r and r + 64,
//    4 consecutive 32-bit columns; every warp reads its 32 lanes back with tcgen05.ld.32x32b.x4.
// 2. throughput: 8 warps repeatedly load 32 columns (tcgen05.ld.32x32b.x32) — bytes/clock/SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_nosw(const void *smem, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version 1 (sm100)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__global__ void __launch_bounds__(256, 1) k_probe(uint32_t *out, int mode, int iters, unsigned long long *cycles) {
    __shared__ __align__(1024) uint4 src[64 * 4];  // 4 columns of 64 rows x 16 B
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 4; i += blockDim.x) {
        const uint32_t r = i & 63, c = i >> 6;
        src[i] = make_uint4(0x1000u * c + 16u * r + 0, 0x1000u * c + 16u * r + 1, 0x1000u * c + 16u * r + 2,
                            0x1000u * c + 16u * r + 3);
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy reads
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tb = tbase;
    if (threadIdx.x == 0) {
        for (int c = 0; c < 4; c++) {
            const uint64_t d = desc_nosw(&src[64 * c], 128, 128);
            const uint32_t dst = tb + 4u * (uint32_t)c;  // lane 0, column 4c
            asm volatile("tcgen05.cp.cta_group::1.64x128b.warpx2::02_13 [%0], %1;" ::"r"(dst), "l"(d) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done)
                         : "r"(smem_u32(&bar))
                         : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    if (mode == 0) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tb + lane_base));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int k = 0; k < 16; k++) out[(threadIdx.x) * 16 + k] = v[k];
    } else {
        uint32_t acc = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; it++) {
            uint32_t v[32];
            const uint32_t col = (uint32_t)((it * 32) & 511);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                           "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                           "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                           "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                         : "r"(tb + lane_base + col));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 32; k++) acc += v[k];
        }
        const long long t1 = clock64();
        if (acc == 0x12345678u) out[0] = acc;
        if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512) : "memory");
}

int main() {
    uint32_t *d_out;
    unsigned long long *d_cyc;
    cudaMalloc(&d_out, 256 * 16 * 4);
    cudaMalloc(&d_cyc, 148 * 8);
    k_probe<<<1, 256>>>(d_out, 0, 0, d_cyc);
    cudaError_t err = cudaDeviceSynchronize();
    printf("mapping run: %s\n", cudaGetErrorString(err));
    uint32_t h[256 * 16];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    // expected: thread of warp w, lane l -> TMEM lane L = 32 (w % 4) + l; data row r = L % 64; columns 4c + j
    int bad = 0;
    for (int th = 0; th < 256; th++) {
        const int w = th >> 5, l = th & 31, L = 32 * (w & 3) + l, r = L & 63;
        for (int c = 0; c < 4; c++)
            for (int j = 0; j < 4; j++) {
                const uint32_t want = 0x1000u * c + 16u * r + j, got = h[th * 16 + 4 * c + j];
                if (want != got) {
                    if (bad < 8) printf("thread %d lane %d col %d: got %x want %x\n", th, L, 4 * c + j, got, want);
                    bad++;
                }
            }
    }
    printf("mapping 64x128b.warpx2::02_13, rows r -> lanes r, r+64: %s (%d mismatches)\n", bad ? "FAIL" : "ok", bad);
    const int iters = 4096;
    k_probe<<<148, 256>>>(d_out, 1, iters, d_cyc);
    err = cudaDeviceSynchronize();
    unsigned long long cyc[148];
    cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; i++) mx = cyc[i] > mx ? cyc[i] : mx;
    const double bytes = 8.0 * iters * 32 * 32 * 4;  // 8 warps x iters x 32 lanes x 32 cols x 4 B
    printf("throughput run: %s; tcgen05.ld 32x32b.x32 (load + wait each): %.1f B/clk/SM (%llu cycles)\n",
           cudaGetErrorString(err), bytes / mx, mx);
    return 0;
}
