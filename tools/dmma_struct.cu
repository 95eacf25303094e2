// DMMA m8n8k4 rate of the warp-streamed quad-form structure (experiment).
// Each warp repeats the lower-triangular row loop of one 8-column block:
// rows i = NRB-1..0, 2(i+1) k-steps, two accumulator chains (P', A'), the A
// operand pair from SMEM (LDS.128 per k-step), B from registers, and an
// epilogue FMA per row (MODE 1) or none (MODE 0), or the epilogue of row i
// deferred until row i-1's chain is issued (MODE 2).  2 CTAs x 256 threads
// per SM like column_kernel_w.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NRB = 10;
constexpr int NB = NRB * (NRB + 1);
constexpr int REPS = 64;
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int MODE>
__global__ void __launch_bounds__(256, 2) k(double* out, double seed) {
    __shared__ double2 fr[NB * 24];
    for (int e = threadIdx.x; e < NB * 24; e += 256) fr[e] = make_double2(seed + e, seed - e);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double bf[2 * NRB];
#pragma unroll
    for (int kk = 0; kk < 2 * NRB; ++kk) bf[kk] = seed * (kk + lane);
    double qa = 0, ra = 0;
    const double2* FRl = fr + (lane % 24);
    for (int rep = 0; rep < REPS; ++rep) {
        double ptc[2] = {0, 0}, puc[2] = {0, 0};
#pragma unroll
        for (int i = NRB - 1; i >= 0; --i) {
            double tc[2] = {0, 0}, uc[2] = {0, 0};
            const double2* f = FRl + i * (i + 1) * 24;
#pragma unroll
            for (int kk = 0; kk < 2 * (i + 1); ++kk) {
                const double2 pa = (MODE == 3) ? make_double2(bf[(kk + 1) % (2 * NRB)], bf[(kk + 3) % (2 * NRB)]) : f[kk * 24];
                dmma(tc, pa.x, bf[kk]);
                dmma(uc, pa.y, bf[kk]);
            }
            if (MODE == 1) {
                qa = fma(bf[2 * i], tc[0] + tc[1], qa);
                ra = fma(bf[2 * i + 1], uc[0] + uc[1], ra);
            } else if (MODE == 2) {
                qa = fma(bf[2 * i], ptc[0] + ptc[1], qa);
                ra = fma(bf[2 * i + 1], puc[0] + puc[1], ra);
                ptc[0] = tc[0]; ptc[1] = tc[1]; puc[0] = uc[0]; puc[1] = uc[1];
            } else {
                qa += tc[0] + uc[1];
                ra += tc[1] + uc[0];
            }
        }
        qa = fma(ptc[0], puc[1], qa);
        bf[rep % (2 * NRB)] += qa * 1e-30;
    }
    if (qa + ra == 1.2345) out[threadIdx.x] = qa;
}
template <int MODE>
void run(int sms, double* out) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int grid = sms * 2 * 8;
    for (int w = 0; w < 2; ++w) k<MODE><<<grid, 256>>>(out, 1e-3);
    cudaEventRecord(e0);
    k<MODE><<<grid, 256>>>(out, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dmma = double(grid) * 8 * REPS * NB * 2;
    printf("{\"mode\": %d, \"tflops\": %.2f, \"ms\": %.3f}\n", MODE, dmma * 512 / (ms * 1e-3) / 1e12, ms);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8 * 256);
    run<0>(sms, out); run<1>(sms, out); run<2>(sms, out);
    run<0>(sms, out); run<1>(sms, out); run<2>(sms, out); run<3>(sms, out);
    return 0;
}
