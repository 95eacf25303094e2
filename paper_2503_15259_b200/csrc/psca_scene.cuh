// psca_scene.cuh -- scene covariance formation on the FP64 tensor pipe
// (included by psca.cu inside its anonymous namespace).
//
//   received_kernel   Y = S[:, active] diag(sqrt(g[active])) H + Z
//                     (sysmodel.py:230-241; the scaled active pilot columns
//                     times the K x M channel, plus the noise)
//   herk_dmma_kernel  Sigma_hat = Y Y^H / M (sysmodel.py:244-248), lower
//                     4 x 8 complex tiles, mirrored
//
// Both are complex GEMMs in the real 2x2 expansion used throughout the
// library (see factor_pass): an m8n8k4 tile = 4 complex rows x 8 complex
// columns, one k-step = 2 complex k; A lanes take component (p ^ q) of the
// left operand with the sign of the [[re, -im], [im, re]] block, B lanes
// component q of the right operand.  One warp per output tile, two
// accumulator chains (even / odd k-steps); operands straight from L1/L2.

__device__ __forceinline__ void tile_of_lower(int t, int& ti, int& tj) {
    int i = 0, base = 0;
    while (base + (4 * i + 3) / 8 + 1 <= t) {
        base += (4 * i + 3) / 8 + 1;
        ++i;
    }
    ti = i;
    tj = t - base;
}

// pilots [B][L][N], act [B][K], gains [B][N], h [B][K][M], z [B][L][M] -> y [B][L][M]
__global__ void __launch_bounds__(256) received_kernel(const double2* __restrict__ pilots,
                                                       const int* __restrict__ act,
                                                       const double* __restrict__ gains,
                                                       const double2* __restrict__ h,
                                                       const double2* __restrict__ z, int L, int N,
                                                       int K, int M, double2* __restrict__ y) {
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntc = (M + 7) / 8;
    const int tile = blockIdx.x * 8 + warp;
    if (tile >= ((L + 3) / 4) * ntc) return;
    const int ti = tile / ntc, tj = tile - ti * ntc;
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1;
    const bool neg = (p == 0 && q == 1);
    const int l = 4 * ti + (r8 >> 1);
    const int mb = 8 * tj + r8;
    const double2* S = pilots + (size_t)b * L * N;
    const int* A = act + (size_t)b * K;
    const double* g = gains + (size_t)b * N;
    const double2* H = h + (size_t)b * K * M;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int nks = (K + 1) / 2;
    for (int ks = 0; ks < nks; ++ks) {
        const int kc = 2 * ks + (c4 >> 1);
        double av = 0.0, bv = 0.0;
        if (kc < K) {
            if (l < L) {
                const int n = __ldg(A + kc);
                const double2 s = __ldg(S + (size_t)l * N + n);
                const double sg = sqrt(__ldg(g + n));
                const double v = (p ^ q) ? s.y * sg : s.x * sg;   // (S_A sqrt(g))(l, kc)
                av = neg ? -v : v;
            }
            if (mb < M) {
                const double2 hv = __ldg(H + (size_t)kc * M + mb);
                bv = q ? hv.y : hv.x;
            }
        }
        dmma(acc[ks & 1], av, bv);
    }
    if (l < L) {
        const double2* Z = z + (size_t)b * L * M;
        double* Y = reinterpret_cast<double*>(y + (size_t)b * L * M);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int m = 8 * tj + 2 * c4 + hh;
            if (m < M) {
                const double2 zv = __ldg(Z + (size_t)l * M + m);
                Y[2 * ((size_t)l * M + m) + p] = (acc[0][hh] + acc[1][hh]) + (p ? zv.y : zv.x);
            }
        }
    }
}

// y [B][L][Mc] -> out [B][L][L] = y y^H / n_antennas
__global__ void __launch_bounds__(256) herk_dmma_kernel(const double2* __restrict__ y, int L,
                                                        int Mc, int n_antennas,
                                                        double2* __restrict__ out) {
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nrb = (L + 3) / 4;
    const int tile = blockIdx.x * 8 + warp;
    if (tile >= rebuild_block_count(nrb)) return;
    int ti, tj;
    tile_of_lower(tile, ti, tj);
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1;
    const bool neg = (p == 0 && q == 1);
    const int l = 4 * ti + (r8 >> 1);
    const int mb = 8 * tj + r8;
    const double2* Y = y + (size_t)b * L * Mc;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int nks = (Mc + 1) / 2;
    for (int ks = 0; ks < nks; ++ks) {
        const int kc = 2 * ks + (c4 >> 1);
        double av = 0.0, bv = 0.0;
        if (kc < Mc) {
            if (l < L) {
                const double2 u = __ldg(Y + (size_t)l * Mc + kc);
                const double v = (p ^ q) ? u.y : u.x;
                av = neg ? -v : v;
            }
            if (mb < L) {   // B = Y^H: component q of conj(Y(mb, kc))
                const double2 u = __ldg(Y + (size_t)mb * Mc + kc);
                bv = q ? -u.y : u.x;
            }
        }
        dmma(acc[ks & 1], av, bv);
    }
    if (l < L) {
        double* O = reinterpret_cast<double*>(out + (size_t)b * L * L);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int m = 8 * tj + 2 * c4 + hh;
            if (m <= l) {
                const double v = __ddiv_rn(acc[0][hh] + acc[1][hh], (double)n_antennas);
                if (m == l) {
                    O[2 * ((size_t)l * L + l) + p] = p ? 0.0 : v;
                } else {
                    O[2 * ((size_t)l * L + m) + p] = v;
                    O[2 * ((size_t)m * L + l) + p] = p ? -v : v;
                }
            }
        }
    }
}
