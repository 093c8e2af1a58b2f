// FP64 pipe micro-benchmark: vector DFMA vs DMMA (mma.sync f64) vs both at once.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_pipes scripts/fp64_pipes.cu
// Question answered: does the FP64 tensor path (DMMA) run beside the vector FP64
// pipe, i.e. can a blind-rotation kernel put its Fourier MAC / DFT blocks on it?
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma_m16n8k16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// mode 0: DFMA only; 1: DMMA m8n8k4 only; 2: both interleaved in every warp;
// 3: even warps DFMA, odd warps DMMA; 4: DMMA m16n8k16 only; 5: m16n8k16 + DFMA interleaved
template <int mode>
__global__ void __launch_bounds__(256) k_pipes(double *out, int iters, double x, double y) {
    double f[8];
    for (int i = 0; i < 8; i++) f[i] = x + threadIdx.x * 1e-9 + i;
    double m[4][2];
    for (int c = 0; c < 4; c++) m[c][0] = m[c][1] = y * c;
    double M[2][4];
    for (int c = 0; c < 2; c++) for (int i = 0; i < 4; i++) M[c][i] = y * (c + i);
    double A[8], B[4];
    for (int i = 0; i < 8; i++) A[i] = x * (i + 1) * 1e-3;
    for (int i = 0; i < 4; i++) B[i] = y * (i + 1) * 1e-3;
    const int warp = threadIdx.x >> 5;
    const bool do_f = mode == 0 || mode == 2 || mode == 5 || (mode == 3 && !(warp & 1));
    const bool do_m = mode == 1 || mode == 2 || (mode == 3 && (warp & 1));
    const bool do_M = mode == 4 || mode == 5;
    for (int it = 0; it < iters; it++) {
        if (do_f) {
#pragma unroll
            for (int i = 0; i < 8; i++) f[i] = fma(f[i], x, y);
        }
        if (do_m) {
#pragma unroll
            for (int c = 0; c < 4; c++) dmma_m8n8k4(m[c], x, y);
        }
        if (do_M) {
#pragma unroll
            for (int c = 0; c < 2; c++) dmma_m16n8k16(M[c], A, B);
        }
    }
    double s = 0;
    for (int i = 0; i < 8; i++) s += f[i];
    for (int c = 0; c < 4; c++) s += m[c][0] + m[c][1];
    for (int c = 0; c < 2; c++) for (int i = 0; i < 4; i++) s += M[c][i];
    if (s == 12345.678) out[0] = s;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double *d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[] = {"DFMA only", "DMMA m8n8k4 only", "DFMA+DMMA interleaved", "DFMA warps | DMMA warps",
                           "DMMA m16n8k16 only", "DMMA m16n8k16 + DFMA"};
    void (*kern[6])(double *, int, double, double) = {k_pipes<0>, k_pipes<1>, k_pipes<2>, k_pipes<3>, k_pipes<4>, k_pipes<5>};
    for (int threads : {256}) {
        for (int per_sm : {4, 8}) {
        for (int mode = 0; mode < 6; mode++) {
            int blocks = p.multiProcessorCount * per_sm, iters = 4096;
            kern[mode]<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
            cudaEventRecord(e0);
            for (int r = 0; r < 5; r++) kern[mode]<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double warps = (double)blocks * threads / 32 * 5 * iters;
            double ff = 0, fm = 0;
            auto fw = warps * ((mode == 3) ? 0.5 : 1.0);
            if (mode == 0 || mode == 2 || mode == 5) ff = fw * 32 * 8 * 2;
            if (mode == 3) ff = fw * 32 * 8 * 2;
            if (mode == 1 || mode == 2) fm = warps * 4 * 512;
            if (mode == 3) fm = fw * 4 * 512;
            if (mode == 4 || mode == 5) fm = warps * 2 * 4096;
            printf("ctas/SM %d threads %d %-26s %8.3f ms  vector %6.2f TF  dmma %6.2f TF  total %6.2f TF  (%s)\n", per_sm, threads,
                   names[mode], ms, ff / ms / 1e9, fm / ms / 1e9, (ff + fm) / ms / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
        }
    }
    return 0;
}
