// DMMA m8n8k4 throughput vs independent accumulator chains and warps per SMSP.
// One CTA per SM; warps map round-robin to the 4 SMSPs.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 2048;
__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, double a, double b) {
    double c[CH][2];
    for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) mma884(c[i], a + i, b);
    }
    double s = 0;
    for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}
template <int CH>
void run(int warps_per_smsp, int sms, double* out) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int threads = 128 * warps_per_smsp;
    for (int w = 0; w < 2; ++w) k<CH><<<sms, threads>>>(out, 1.0, 1e-3);
    cudaEventRecord(e0);
    k<CH><<<sms, threads>>>(out, 1.0, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double dmma = double(sms) * threads / 32 * IT * CH;
    double per_smsp_cycles = ms * 1e-3 * 1.965e9 / (dmma / (sms * 4.0));
    printf("{\"chains\": %d, \"warps_per_smsp\": %d, \"cycles_per_dmma_per_smsp\": %.2f, \"tflops\": %.2f}\n",
           CH, warps_per_smsp, per_smsp_cycles, dmma * 512 / (ms * 1e-3) / 1e12);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    for (int w : {1, 2, 4}) {
        run<1>(w, sms, out); run<2>(w, sms, out); run<4>(w, sms, out); run<8>(w, sms, out);
    }
    return 0;
}
