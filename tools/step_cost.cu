// Microbenchmark: cost of one block-sweep-like step in a lone 512-thread CTA
// (experiment tool for the c0 factor latency work).  Each variant loops STEPS
// times over: [U phase on 40 threads] barrier [V phase on NACT threads] barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_cost tools/step_cost.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int STEPS = 2000;
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, int nact, double seed) {
    __shared__ double2 c0[48], c1[48], u0[48], u1[48];
    __shared__ double kv[4];
    const int tid = threadIdx.x;
    if (tid < 48) {
        c0[tid] = make_double2(seed * tid, 0.5);
        c1[tid] = make_double2(0.25, seed);
        u0[tid] = make_double2(seed, seed);
        u1[tid] = make_double2(seed, -seed);
    }
    if (tid == 0) { kv[0] = 2.0; kv[1] = 0.1; kv[2] = 0.2; kv[3] = 3.0; }
    double2 v[2][2];
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 2; ++j) v[i][j] = make_double2(seed + i, seed - j);
    const int i0 = (tid * 7) % 38, j0 = (tid * 3) % 38;
    __syncthreads();
    const long long t0 = clock64();
    for (int s = 0; s < STEPS; ++s) {
        if (MODE & 1) {   // U phase
            const double ka = kv[0], kbr = kv[1], kbi = kv[2], kc = kv[3];
            const double det = fma(ka, kc, -fma(kbr, kbr, kbi * kbi));
            if (!(det > 0.0)) break;
            if (tid < 40) {
                const double dinv = __drcp_rn(det);
                const double m00 = kc * dinv, m11 = ka * dinv;
                const double2 m10 = make_double2(-kbr * dinv, -kbi * dinv);
                const double2 pp = c0[tid], qq = c1[tid];
                u0[tid] = make_double2(fma(m10.x, qq.x, fma(-m10.y, qq.y, m00 * pp.x)),
                                       fma(-m10.y, qq.x, fma(-m10.x, qq.y, -m00 * pp.y)));
                u1[tid] = make_double2(fma(m11, qq.x, fma(m10.x, pp.x, m10.y * pp.y)),
                                       fma(-m11, qq.y, fma(m10.y, pp.x, -m10.x * pp.y)));
            }
        }
        if (MODE & 2) __syncthreads();
        if ((MODE & 4) && tid < nact) {   // V phase
            double2 uj[2][2], ci[2][2];
            for (int d = 0; d < 2; ++d) {
                uj[0][d] = u0[j0 + d]; uj[1][d] = u1[j0 + d];
                ci[0][d] = c0[i0 + d]; ci[1][d] = c1[i0 + d];
            }
#pragma unroll
            for (int di = 0; di < 2; ++di)
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    const double2 o = v[di][dj];
                    const double2 pp = ci[0][di], qq = ci[1][di];
                    double nx = fma(-pp.x, uj[0][dj].x, fma(pp.y, uj[0][dj].y, o.x));
                    double ny = fma(-pp.x, uj[0][dj].y, fma(-pp.y, uj[0][dj].x, o.y));
                    nx = fma(-qq.x, uj[1][dj].x, fma(qq.y, uj[1][dj].y, nx));
                    ny = fma(-qq.x, uj[1][dj].y, fma(-qq.y, uj[1][dj].x, ny));
                    v[di][dj] = make_double2(nx * 1e-3, ny * 1e-3);
                }
            if (tid < 20) {   // staging
                c0[i0] = v[0][0]; c1[i0] = v[0][1]; c0[i0 + 1] = v[1][0]; c1[i0 + 1] = v[1][1];
            }
            if (tid == 0) { kv[0] = 2.0 + 1e-9 * v[0][0].x; kv[3] = 3.0 + 1e-9 * v[1][1].x; }
        }
        if (MODE & 8) __syncthreads();
    }
    const long long t1 = clock64();
    if (tid == 0) *cyc = t1 - t0;
    out[blockIdx.x * 512 + tid] = v[0][0].x + v[1][1].y + v[0][1].x + v[1][0].y;
}
template <int MODE>
void run(const char* name, int nact) {
    double* out; long long* cyc;
    cudaMalloc(&out, 512 * 8); cudaMalloc(&cyc, 8);
    k<MODE><<<1, 512>>>(out, cyc, nact, 0.01);
    k<MODE><<<1, 512>>>(out, cyc, nact, 0.01);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s nact=%3d  cycles/step = %.1f  (%s)\n", name, nact, (double)h / STEPS, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    run<15>("U + bar + V + bar", 210);
    run<15>("U + bar + V + bar", 512);
    run<15>("U + bar + V + bar", 32);
    run<10>("two barriers only", 210);
    run<11>("U + two barriers", 210);
    run<14>("V + two barriers", 210);
    run<4>("V only, no barrier", 210);
    run<4>("V only, no barrier", 32);
    run<1>("U only, no barrier", 210);
    return 0;
}
