// FFT-only occupancy micro-benchmark: how close does the production negacyclic
// FFT (hb_dev_fft.cuh) get to the FP64 pipe at 8 / 12 / 16 warps per SM?
// Each 64-thread group repeats forward + inverse transforms of NP polynomials
// held in registers (exchange buffers in shared memory, as in the blind rotation).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/fft_occ scripts/fft_occupancy.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1806_03461_b200/csrc/hb_internal.h"
using namespace hb;
namespace {
#include "../paper_1806_03461_b200/csrc/hb_dev_fft.cuh"

template <int G, int NP, bool SB, int MB>
__global__ void __launch_bounds__(64 * G, MB) k_fft(double *out, const double2 *W, const double2 *TW, int iters) {
    constexpr int kBufs = SB ? NP : 2 * NP;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double2 (*xch)[kBufs][kXchStride] = reinterpret_cast<double2 (*)[kBufs][kXchStride]>(smem_raw);
    TwSeeds *tws = reinterpret_cast<TwSeeds *>(smem_raw + sizeof(double2) * G * kBufs * kXchStride);
    const int g = threadIdx.x >> 6, t = threadIdx.x & 63;
    if (threadIdx.x < 64) {
        TwSeeds ts;
        ts.f_a0 = TW[t];
        ts.step_a = W[t];
        ts.step_b = W[8 * (t & 7)];
        ts.i_b0 = TW[t >> 3];
        ts.i_stepb = TW[32 * (t & 7) + 8];
        tws[t] = ts;
    }
    __syncthreads();
    double2 x[NP][8];
#pragma unroll
    for (int q = 0; q < NP; q++)
#pragma unroll
        for (int m = 0; m < 8; m++) x[q][m] = make_double2((t * 7 + m * 3 + q) % 61 - 30, (t * 5 + m) % 53 - 26);
    for (int it = 0; it < iters; it++) {
        nega_fft_fwd_n<NP, SB>(x, &xch[g][0][0], t, tws[t], 1 + g);
        nega_fft_inv_n<NP, SB>(x, &xch[g][0][0], t, tws[t], 1 + g);
#pragma unroll
        for (int q = 0; q < NP; q++)
#pragma unroll
            for (int m = 0; m < 8; m++) x[q][m] = make_double2(x[q][m].x * (1.0 / 512), x[q][m].y * (1.0 / 512));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < NP; q++)
#pragma unroll
        for (int m = 0; m < 8; m++) s += x[q][m].x + x[q][m].y;
    if (s == 1234.5) out[0] = s;
}

double2 *g_W, *g_TW;

template <int G, int NP, bool SB, int MB>
void run(const char *name, int sms) {
    double *d;
    cudaMalloc(&d, 8);
    auto k = k_fft<G, NP, SB, MB>;
    constexpr int kBufs = SB ? NP : 2 * NP;
    const size_t smem = sizeof(double2) * G * kBufs * kXchStride + 64 * sizeof(TwSeeds);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 64 * G, smem);
    if (occ > MB) occ = MB;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k);
    const int iters = 200;
    const int grid = sms * occ;
    k<<<grid, 64 * G, smem>>>(d, g_W, g_TW, 2);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<grid, 64 * G, smem>>>(d, g_W, g_TW, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ffts = (double)grid * G * NP * 2 * iters;  // forward + inverse per iteration
    printf("%-28s regs %3d ctas/SM %d warps/SM %2d  %8.3f ms  %.3f us/FFT/SM  %.1f M FFT/s  err=%s\n", name,
           fa.numRegs, occ, occ * G * 2, ms, ms * 1e3 * sms / ffts, ffts / ms / 1e3,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}
}  // namespace

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    double2 hW[512], hTW[2048];
    for (int e = 0; e < 512; e++) hW[e] = make_double2(cos(2 * M_PI * e / 512), sin(2 * M_PI * e / 512));
    for (int e = 0; e < 2048; e++) hTW[e] = make_double2(cos(M_PI * e / 1024), sin(M_PI * e / 1024));
    cudaMalloc(&g_W, sizeof(hW));
    cudaMalloc(&g_TW, sizeof(hTW));
    cudaMemcpy(g_W, hW, sizeof(hW), cudaMemcpyHostToDevice);
    cudaMemcpy(g_TW, hTW, sizeof(hTW), cudaMemcpyHostToDevice);
    printf("%s, %d SMs, clock %d MHz\n", p.name, sms, p.clockRate / 1000);
    run<4, 2, true, 1>("G4 NP2 SB (u2 layout)", sms);
    run<4, 2, false, 1>("G4 NP2 DB", sms);
    run<4, 1, true, 1>("G4 NP1 SB", sms);
    run<2, 2, true, 3>("G2x3 NP2 SB (12 warps)", sms);
    run<2, 2, true, 4>("G2x4 NP2 SB (16 warps)", sms);
    run<6, 2, true, 1>("G6 NP2 SB (12 warps)", sms);
    run<8, 2, true, 1>("G8 NP2 SB (16 warps)", sms);
    run<6, 1, true, 1>("G6 NP1 SB (12 warps)", sms);
    run<8, 1, true, 1>("G8 NP1 SB (16 warps)", sms);
    run<4, 1, true, 2>("G4x2 NP1 SB (16 warps)", sms);
    run<8, 1, true, 2>("G8x2 NP1 SB (32 warps)", sms);
    run<2, 1, true, 1>("G2 NP1 SB (4 warps)", sms);
    return 0;
}
