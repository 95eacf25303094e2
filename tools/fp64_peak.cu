// FP64 throughput microbenchmarks for B200 (sm_100a).
//
// The PSCA hot path is complex128 arithmetic and tcgen05 has no f64 kind, so
// the two candidate FP64 engines are the DFMA pipe and the legacy DMMA
// (mma.sync .f64) tensor path.  This measures each alone and both together
// (alternate warps) so the kernel design and the roofline denominator rest on
// numbers taken on this hardware.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
    for (int i = 0; i < ITERS; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5) out[threadIdx.x] = s;
}

__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&c)[4], double a0, double a1, double a2, double a3,
                                        double b0, double b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}
__device__ __forceinline__ void mma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                 "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int KIND>
__global__ void dmma_kernel(double* out, double a, double b) {
    double acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] = 0.0;
    double av[8], bv[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) av[i] = a + i + threadIdx.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) bv[i] = b + i;
    for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (KIND == 0) { double c2[2] = {acc[j][0], acc[j][1]}; mma884(c2, av[j], bv[0]); acc[j][0] = c2[0]; acc[j][1] = c2[1]; }
            if (KIND == 1) { double (&c)[4] = acc[j]; mma1684(c, av[j], av[(j + 1) & 7], bv[0]); }
            if (KIND == 2) { double (&c)[4] = acc[j]; mma1688(c, av[0], av[1], av[2], av[3], bv[0], bv[1]); }
            if (KIND == 3) { double (&c)[4] = acc[j]; mma16816(c, av, bv); }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) s += acc[j][i];
    if (s == 1234.5) out[threadIdx.x] = s;
}

// even warps DFMA, odd warps DMMA m16n8k8: do the two engines add up?
__global__ void mixed_kernel(double* out, double a, double b) {
    int warp = threadIdx.x / 32;
    double s = 0;
    if (warp & 1) {
        double acc[8][4] = {};
        double av[4] = {a, a + 1, a + 2, a + 3}, bv[2] = {b, b + 1};
        for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
            for (int j = 0; j < 8; ++j) mma1688(acc[j], av[0], av[1], av[2], av[3], bv[0], bv[1]);
        }
        for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
    } else {
        double x[8];
        for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
#pragma unroll 4
        for (int i = 0; i < ITERS * 2; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
        }
        for (int k = 0; k < 8; ++k) s += x[k];
    }
    if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out;
    CK(cudaMalloc(&out, 1024 * sizeof(double)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256;
    auto time_it = [&](auto launch, double flops, const char* name) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0);
        const int reps = 10;
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double tf = flops * reps / (ms * 1e-3) / 1e12;
        printf("{\"kernel\": \"%s\", \"tflops\": %.3f, \"ms\": %.4f}\n", name, tf, ms / reps);
        fflush(stdout);
    };
    double nthreads = double(blocks) * threads;
    time_it([&] { dfma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3); },
            nthreads * ITERS * 8 * 2, "dfma");
    double nwarps = nthreads / 32;
    time_it([&] { dmma_kernel<0><<<blocks, threads>>>(out, 0.999, 1e-3); },
            nwarps * (ITERS / 4) * 8 * (8 * 8 * 4) * 2, "dmma_m8n8k4");
    time_it([&] { dmma_kernel<1><<<blocks, threads>>>(out, 0.999, 1e-3); },
            nwarps * (ITERS / 4) * 8 * (16 * 8 * 4) * 2, "dmma_m16n8k4");
    time_it([&] { dmma_kernel<2><<<blocks, threads>>>(out, 0.999, 1e-3); },
            nwarps * (ITERS / 4) * 8 * (16 * 8 * 8) * 2, "dmma_m16n8k8");
    time_it([&] { dmma_kernel<3><<<blocks, threads>>>(out, 0.999, 1e-3); },
            nwarps * (ITERS / 4) * 8 * (16 * 8 * 16) * 2, "dmma_m16n8k16");
    double half = nwarps / 2;
    time_it([&] { mixed_kernel<<<blocks, threads>>>(out, 0.999, 1e-3); },
            half * (ITERS / 4) * 8 * (16 * 8 * 8) * 2 + half * 32 * ITERS * 2 * 8 * 2, "mixed_dfma_dmma");
    CK(cudaGetLastError());
    return 0;
}
