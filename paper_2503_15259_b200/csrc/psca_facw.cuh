// psca_facw.cuh -- the factor stage of the batched two-kernel path as two
// kernels (sm_100a; included by psca.cu after psca_fast.cuh):
//
//   fac_sweep_w<NRB>   ONE WARP PER INSTANCE, four instances per 128-thread
//                      CTA (NRB <= 10, L <= 40): finalise iteration k-1
//                      (q-floor, update norm, tol stop), the prior terms at
//                      x_k, Sigma_k assembled straight from the rebuild
//                      partials and D into DMMA accumulator fragments (the
//                      same 4 x 8 complex tile layout, no shared-memory
//                      matrix), its Frobenius norm, and the Hermitian sweep
//                      operator in those registers -- every 2x2 block-pivot
//                      step is one phase-U pass (U_j = M conj(C_j) per column)
//                      and ONE DMMA per tile (the rank-2 trailing update),
//                      synchronised by __syncwarp only.  P = Sigma^-1 leaves
//                      as lower-triangle fragments (pfrag).
//   fac_prod_t<NRB>    one CTA per instance: P from pfrag into SMEM (full
//                      Hermitian), Sigma_hat staged by cp.async,
//                      trace(P Sigma_hat), G = Sigma_hat P and A = P G on DMMA
//                      and the packed P'/A' fragments of the next column pass
//                      (products_pass, shared with factor_solve_t).
//
// Why: in factor_solve_t the sweep held 55 % of the kernel's time.  Its
// per-step chain (det, reciprocal, U, update, staging) ran with the matrix in
// shared memory or in per-thread 2x2 blocks behind CTA barriers, at most four
// instances per SM (55 KB of SMEM each), interleaved with the DMMA-heavy
// product phases of the other resident instances.  Here the sweep of an
// instance needs ~4 KB of SMEM and no CTA barrier, so 12+ instances per SM
// overlap their dependent chains, and the products run as their own
// throughput-bound launch.

// instances (warps) per CTA and CTAs per SM of fac_sweep_w.  More resident warps
// do not help (measured: 2 x 7 and 4 x 4 at 128 registers spill and lose 20 %,
// 144 / 160 registers at 14 / 12 warps are equal to 4 x 3 at 168)
#ifndef PSCA_FACW_IPC
#define PSCA_FACW_IPC 4
#endif
// fully unrolled pivot loop (every tile dispatch and pivot predicate folds): 215 KB of
// code at NRB = 10, measured slower (sweep 185 -> 219 us per 4096): off
#ifndef PSCA_FACW_UNROLL
#define PSCA_FACW_UNROLL 0
#endif
#ifndef PSCA_FACW_MINB
#define PSCA_FACW_MINB 3
#endif

template <int NRB>
struct TWS {
    static constexpr int LP = 4 * NRB;
    static constexpr int LPC = LP + ((NRB & 1) ? 0 : 4);   // staged-column stride (banks)
    static constexpr int NTL = rebuild_block_count(NRB);    // lower 4 x 8 tiles
    static constexpr int NCJ = (LP + 7) / 8;
    static constexpr int IPC = PSCA_FACW_IPC;               // instances (warps) per CTA
    // deferred rebuild: gather ring of RST stages, two listed columns [2][LPC]
    // each (it aliases the sweep scratch: the rebuild is over before the sweep)
    static constexpr int RST = 8;
    // per warp: ub [2][LPC], cs [2 phases][2][LPC] (double2), kv [2][4], -M [8]
    static constexpr size_t SWEEP_SMEM = (size_t)6 * LPC * 16 + 16 * 8;
    static constexpr size_t RING_SMEM = (size_t)RST * 2 * LPC * 16;
    // then the list itself: MOV_CAP weights and columns
    static constexpr size_t WARP_SMEM =
        (SWEEP_SMEM > RING_SMEM ? SWEEP_SMEM : RING_SMEM) + (size_t)MOV_CAP * 12;
    static constexpr size_t SMEM = IPC * WARP_SMEM;
};

// Tile loops below walk the lower tiles in row-major order with the tile's row
// / column index as running counters (ti, tj), which constant-fold after
// unrolling (a constexpr lookup per tile did not, and its loops swamped the
// kernel).
#define TILE_NEXT(ti, tj)           \
    if (++tj > (4 * ti + 3) / 8) { \
        tj = 0;                     \
        ++ti;                       \
    }

// prior terms at x (fac_prior_terms_at, one warp): the map-ur / pairwise
// gradient into a.pgrad and, when the objective is recorded, the penalty value
__device__ double warp_prior_terms(const FacArgs& a, int b, const double* xv, int lane) {
    const size_t bN = (size_t)b * a.N;
    double val = 0.0;
    if (a.kind == PSCA_MAP_K && a.c2_ptr) {
        double lin = 0.0, quad = 0.0;
        for (int n = lane; n < a.N; n += 32) {
            double s = 0.0;
            for (int j = a.c2_ptr[n]; j < a.c2_ptr[n + 1]; ++j)
                s = __dadd_rn(s, __dmul_rn(a.c2_val[j], xv[a.c2_idx[j]]));
            a.pgrad[bN + n] = __ddiv_rn(-__dadd_rn(a.c1[n], s), (double)a.n_antennas);
            lin = fma(a.c1[n], xv[n], lin);
            quad = fma(xv[n], s, quad);
        }
        if (a.record_objective) {
            for (int o = 16; o > 0; o >>= 1) {
                lin += __shfl_xor_sync(0xffffffffu, lin, o);
                quad += __shfl_xor_sync(0xffffffffu, quad, o);
            }
            val = -(lin + 0.5 * quad) / a.n_antennas;
        }
        return val;
    }
    if (a.kind == PSCA_MAP_UR || (a.kind == PSCA_MAP_K && a.record_objective)) {
        double acc = 0.0;
        for (int n = lane; n < a.N; n += 32) {
            const double x = xv[n];
            if (a.kind == PSCA_MAP_UR) {
                double dens, der;
                eff_density(x, a.prior_p[n], a.eff, dens, der);
                const double mag = a.eff.dead_zone_grad;
                double gr;
                if (dens <= 1e-300) {
                    gr = ((x <= a.eff.g_low / 2.0) ? 1.0 : -1.0) * (mag / a.n_antennas);
                } else {
                    gr = -np_clip(der / dens, -mag, mag) / a.n_antennas;
                }
                a.pgrad[bN + n] = gr;
                if (a.record_objective) acc += log(dens > 1e-300 ? dens : 1e-300);
            } else {
                acc = fma(a.prior_lin[n], x, acc);
            }
        }
        if (a.record_objective) {
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            val = (a.kind == PSCA_MAP_K) ? acc : -acc / a.n_antennas;
        }
    }
    return val;
}

template <int NRB>
__host__ __device__ constexpr int row_start(int i) {
    int s = 0;
    for (int r = 0; r < i; ++r) s += (4 * r + 3) / 8 + 1;
    return s;
}

// Per-lane constants of the sweep (fragment position and operand bases).
struct SwLane {
    int rl, c4, p;    // row within a 4-row tile, column pair, component
};

// K-row fix of row tile I after the step-k DMMA: lanes on rows K take U_m, and
// on the K block -M (nm at Ud offset NMO); rlane / dl: is the lane's row in K.
template <int NRB, int I>
__device__ __forceinline__ void fix_row(double (&acc)[rebuild_block_count(NRB)][2],
                                        const SwLane& w, bool rlane, int dl, int kcl, bool clane,
                                        const double* Ud, int LPC, int NMO) {
    constexpr int T0 = row_start<NRB>(I);
    constexpr int NJ = (4 * I + 3) / 8 + 1;
    if (!rlane) return;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = 8 * j + 2 * w.c4 + h;
            const bool kb = (j == kcl) && clane;
            acc[T0 + j][h] = kb ? Ud[NMO + 2 * (2 * dl + h) + w.p] : Ud[2 * (dl * LPC + m) + w.p];
        }
    }
}
// K-column fix of column tile J: lanes on columns K take conj(U_l) (rows in K
// are redone by fix_row)
template <int NRB, int J>
__device__ __forceinline__ void fix_col(double (&acc)[rebuild_block_count(NRB)][2],
                                        const SwLane& w, bool clane, const double* Ud, int LPC) {
    if (!clane) return;
#pragma unroll
    for (int i = 2 * J; i < NRB; ++i) {
        const int l = 4 * i + w.rl;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double u = Ud[2 * (h * LPC + l) + w.p];
            acc[row_start<NRB>(i) + J][h] = w.p ? -u : u;
        }
    }
}
// staging of pivot block K' = {k2, k2 + 1}: row tile I holds rows K'
// (C(m, dl) = conj(a_{k2+dl, m}) for m < k2, and K' itself into kd)
template <int NRB, int I>
__device__ __forceinline__ void stage_row(const double (&acc)[rebuild_block_count(NRB)][2],
                                          const SwLane& w, bool rlane, int dl, int k2, int kcl,
                                          bool clane, double* Cn, double* kd, int LPC) {
    constexpr int T0 = row_start<NRB>(I);
    constexpr int NJ = (4 * I + 3) / 8 + 1;
    if (!rlane) return;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = 8 * j + 2 * w.c4 + h;
            const double v = acc[T0 + j][h];
            if (j == kcl && clane) {   // K' block, lower entries
                const int ki = (dl == 0) ? ((h == 0 && w.p == 0) ? 0 : -1)
                                         : (h == 0 ? 1 + w.p : (w.p == 0 ? 3 : -1));
                if (ki >= 0) kd[ki] = v;
            } else if (m < k2) {
                Cn[2 * (dl * LPC + m) + w.p] = w.p ? -v : v;
            }
        }
    }
}
// column tile J holds columns K': C(l, h) = a_{l, k2+h} for rows l > k2 + 1
template <int NRB, int J>
__device__ __forceinline__ void stage_col(const double (&acc)[rebuild_block_count(NRB)][2],
                                          const SwLane& w, bool clane, int k2, double* Cn,
                                          int LPC) {
    if (!clane) return;
#pragma unroll
    for (int i = 2 * J; i < NRB; ++i) {
        const int l = 4 * i + w.rl;
        if (l > k2 + 1) {
#pragma unroll
            for (int h = 0; h < 2; ++h) Cn[2 * (h * LPC + l) + w.p] = acc[row_start<NRB>(i) + J][h];
        }
    }
}
// runtime tile index -> the compile-time instantiation (a chain of compares)
template <int NRB, int I = 0, class F>
__device__ __forceinline__ void dispatch_row(int i, F&& f) {
    if constexpr (I < NRB) {
        if (i == I) f(std::integral_constant<int, I>{});
        else dispatch_row<NRB, I + 1>(i, f);
    }
}
template <int NCJ, int J = 0, class F>
__device__ __forceinline__ void dispatch_col(int j, F&& f) {
    if constexpr (J < NCJ) {
        if (j == J) f(std::integral_constant<int, J>{});
        else dispatch_col<NCJ, J + 1>(j, f);
    }
}

// The sweep of one instance by one warp, the matrix in acc (lower 4 x 8
// complex tiles, DMMA C-fragment layout); wsm = this warp's TWS::WARP_SMEM
// bytes of shared scratch.  Returns false when a pivot block is not PD.
template <int NRB>
__device__ __forceinline__ bool warp_sweep(double (&acc)[rebuild_block_count(NRB)][2],
                                           unsigned char* wsm, int L, bool want_logdet,
                                           double& logdet) {
    using S = TWS<NRB>;
    constexpr int LP = S::LP, LPC = S::LPC, NTL = S::NTL;
    const int lane = threadIdx.x & 31;
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1, kc = c4 >> 1;
    double2* ub = reinterpret_cast<double2*>(wsm);                                // [2][LPC]
    double2* cs = ub + 2 * LPC;                                                   // [2][2][LPC]
    double* kv = reinterpret_cast<double*>(cs + 4 * LPC);                         // [2][4]
    const double* Ud = reinterpret_cast<const double*>(ub);
    const int abase = 2 * (kc * LPC + (r8 >> 1)) + (p ^ q);
    const int bbase = 2 * (kc * LPC + r8) + q;
    // Rows of the pivot block are never zeroed in the staged columns: their A
    // operand lanes are masked in the DMMA and their U_j is zero by definition.
    const int rl = r8 >> 1;
    const SwLane sw{rl, c4, p};
    auto stage = [&](int k2, int dst) {
        double* Cn = reinterpret_cast<double*>(cs + dst * 2 * LPC);
        double* kd = kv + dst * 4;
        const int dl = rl - (k2 & 3);
        const bool rlane = (unsigned)dl < 2u, clane = c4 == ((k2 & 7) >> 1);
        const int kcl = k2 >> 3;
        dispatch_col<S::NCJ>(kcl, [&](auto J) { stage_col<NRB, J.value>(acc, sw, clane, k2, Cn, LPC); });
        dispatch_row<NRB>(k2 >> 2, [&](auto I) {
            stage_row<NRB, I.value>(acc, sw, rlane, dl, k2, kcl, clane, Cn, kd, LPC);
        });
    };
    stage(0, 0);
    __syncwarp();
    logdet = 0.0;
    bool ok = true;
    const int LE = (L + 1) & ~1;
    const unsigned long long sgn = (p == 0 && q == 1) ? 0ull : 0x8000000000000000ull;
    double* nm = kv + 8;   // -M as 2x2 complex: Ud[12 LPC + 8 + 2 (2 dl + h) + p]
#if PSCA_FACW_UNROLL
#pragma unroll
    for (int k = 0; k < LP; k += 2) {
        if (k >= LE) break;
#else
    for (int k = 0; k < LE; k += 2) {
#endif
        const int ph = (k >> 1) & 1;
        const double2* cc = cs + ph * 2 * LPC;
        const double* Cd = reinterpret_cast<const double*>(cc);
        const double ka = kv[ph * 4 + 0], kbr = kv[ph * 4 + 1], kbi = kv[ph * 4 + 2],
                     kcc = kv[ph * 4 + 3];
        const double det = fma(ka, kcc, -fma(kbr, kbr, kbi * kbi));
        if (!(ka > 0.0) || !(det > 0.0)) {
            ok = false;
            break;
        }
        if (want_logdet) logdet += log(det);
        {
            const double dinv = __drcp_rn(det);
            const double m00 = kcc * dinv;
            const double m11 = ka * dinv;
            const double2 m10 = make_double2(-kbr * dinv, -kbi * dinv);
            const double2 m01 = make_double2(m10.x, -m10.y);
#pragma unroll
            for (int j = lane; j < LP; j += 32) {
                double2 u0 = make_double2(0.0, 0.0), u1 = make_double2(0.0, 0.0);
                if (j != k && j != k + 1) {   // U_K = 0 (C_K is K itself, not zeroed)
                    const double2 pp = cc[j], qq = cc[LPC + j];
                    u0 = make_double2(fma(m01.x, qq.x, fma(m01.y, qq.y, m00 * pp.x)),
                                      fma(m01.y, qq.x, fma(-m01.x, qq.y, -m00 * pp.y)));
                    u1 = make_double2(fma(m11, qq.x, fma(m10.x, pp.x, m10.y * pp.y)),
                                      fma(-m11, qq.y, fma(m10.y, pp.x, -m10.x * pp.y)));
                }
                ub[j] = u0;
                ub[LPC + j] = u1;
            }
            if (lane < 8) {   // -M: (dl, h) = (0,0) (0,1) (1,0) (1,1), component p = lane & 1
                const int e = lane >> 1, pp = lane & 1;
                const double re = e == 0 ? m00 : (e == 1 ? m01.x : (e == 2 ? m10.x : m11));
                const double im = (e == 1) ? m01.y : (e == 2 ? m10.y : 0.0);
                nm[lane] = -(pp ? im : re);
            }
        }
        __syncwarp();
        const int kr = k >> 2, kcl = k >> 3, dl = rl - (k & 3);
        const bool rlane = (unsigned)dl < 2u, clane = c4 == ((k & 7) >> 1);
        // rank-2 trailing update: one DMMA per tile (operands shared per row /
        // column tile; the K rows' A lanes masked)
        {
            double af[NRB], bfr[S::NCJ];
#pragma unroll
            for (int i = 0; i < NRB; ++i)
                af[i] = (i == kr && rlane) ? 0.0 : xsign(Cd[abase + 8 * i], sgn);
#pragma unroll
            for (int j = 0; j < S::NCJ; ++j) bfr[j] = Ud[bbase + 16 * j];
            int ti = 0, tj = 0;
#pragma unroll
            for (int t = 0; t < NTL; ++t) {
                dmma(acc[t], af[ti], bfr[tj]);
                TILE_NEXT(ti, tj)
            }
        }
        // the K columns (conj(U_l)), then the K rows (U_m) and the K block (-M)
        dispatch_col<S::NCJ>(kcl, [&](auto J) { fix_col<NRB, J.value>(acc, sw, clane, Ud, LPC); });
        dispatch_row<NRB>(kr, [&](auto I) {
            fix_row<NRB, I.value>(acc, sw, rlane, dl, kcl, clane, Ud, LPC, 12 * LPC + 8);
        });
        if (k + 2 < LE) stage(k + 2, ph ^ 1);
        __syncwarp();
    }
    return ok;
}

// Deferred covariance rebuild (covlinalg.py:55 over the moving columns only):
// the column kernel left this instance's short list (column, weight); the warp
// gathers the listed pilot columns through a cp.async ring (two columns = one
// DMMA k-step per stage, RST stages in flight, rows >= L zero-filled) and sums
// w s s^H into the accumulator fragments, one DMMA per tile per k-step:
//   A[(l, p)][(c, q)] = +-S[l][c].(p ^ q)  (minus for p & q),
//   B[(c, q)][m]      = w_c S[m][c].q
// The list is copied to the warp's shared memory first (weights lw, columns lc,
// behind the ring), so no registers are held across the prior terms.
template <int NRB>
__device__ __forceinline__ void mov_issue(const FacArgs& a, const double2* pil, int cnt,
                                          const int* lc, double2* ring, int ks, int lane) {
    using S = TWS<NRB>;
    constexpr int LP = S::LP, LPC = S::LPC;
    double2* st = ring + (size_t)(ks & (S::RST - 1)) * 2 * LPC;
#pragma unroll
    for (int u = 0; u < (2 * LP + 31) / 32; ++u) {
        const int e = lane + 32 * u;
        const int col = e >= LP ? 1 : 0;
        const int row = e - col * LP;
        const int c = 2 * ks + col;
        if (e < 2 * LP) {
            const bool ok = c < cnt && row < a.L;
#ifdef PSCA_DBG_GATHER_HOT   // probe (results invalid): gather from columns 0, 1, ...
            cp_async16(st + col * LPC + row, ok ? pil + (size_t)row * a.N + c : pil, ok ? 16 : 0);
#else
            cp_async16(st + col * LPC + row, ok ? pil + (size_t)row * a.N + lc[c] : pil,
                       ok ? 16 : 0);
#endif
        }
    }
}

template <int NRB>
__device__ __forceinline__ void mov_begin(const FacArgs& a, int b, int cnt, unsigned char* wsm,
                                          int lane) {
    using S = TWS<NRB>;
    double* lw = reinterpret_cast<double*>(wsm + S::RING_SMEM);
    int* lc = reinterpret_cast<int*>(lw + MOV_CAP);
    const size_t lo = (size_t)b * a.mov_cap;
    for (int e = lane; e < MOV_CAP; e += 32) {
        lc[e] = e < cnt ? a.mov_col[lo + e] : 0;
        lw[e] = e < cnt ? a.mov_w[lo + e] : 0.0;
    }
    __syncwarp();
    const double2* pil = a.pilots + (size_t)b * a.L * a.N;
    double2* ring = reinterpret_cast<double2*>(wsm);
    const int nks = (cnt + 1) >> 1;
#pragma unroll 1
    for (int ks = 0; ks < S::RST - 1; ++ks) {
        if (ks < nks) mov_issue<NRB>(a, pil, cnt, lc, ring, ks, lane);
        cp_async_commit();
    }
}

template <int NRB>
__device__ __forceinline__ void mov_rebuild(const FacArgs& a, int b, int cnt,
                                            double (&acc)[rebuild_block_count(NRB)][2],
                                            unsigned char* wsm, int lane) {
    using S = TWS<NRB>;
    constexpr int LPC = S::LPC, NTL = S::NTL, RST = S::RST;
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1, kc = c4 >> 1;
    const double2* pil = a.pilots + (size_t)b * a.L * a.N;
    double2* ring = reinterpret_cast<double2*>(wsm);
    const double* lw = reinterpret_cast<const double*>(wsm + S::RING_SMEM);
    const int* lc = reinterpret_cast<const int*>(lw + MOV_CAP);
    const int abase = 2 * (kc * LPC + (r8 >> 1)) + (p ^ q);
    const int bbase = 2 * (kc * LPC + r8) + q;
    const unsigned long long sgn = (p & q) ? 0x8000000000000000ull : 0ull;
    const int nks = (cnt + 1) >> 1;
#pragma unroll 1
    for (int ks = 0; ks < nks; ++ks) {
        if (ks + RST - 1 < nks) mov_issue<NRB>(a, pil, cnt, lc, ring, ks + RST - 1, lane);
        cp_async_commit();
        cp_async_wait<RST - 1>();
        __syncwarp();
        const double* Sd =
            reinterpret_cast<const double*>(ring + (size_t)(ks & (RST - 1)) * 2 * LPC);
        const double w = lw[2 * ks + kc];
        // A operands one row tile ahead of their DMMAs (the accumulators fill
        // the register file: no room for all NRB of them)
        double bfr[S::NCJ];
#pragma unroll
        for (int j = 0; j < S::NCJ; ++j) bfr[j] = w * Sd[bbase + 16 * j];
        double a_cur = xsign(Sd[abase], sgn);
#pragma unroll
        for (int i = 0; i < NRB; ++i) {
            const double a_nxt = (i + 1 < NRB) ? xsign(Sd[abase + 8 * (i + 1)], sgn) : 0.0;
#pragma unroll
            for (int j = 0; j <= (4 * i + 3) / 8; ++j) dmma(acc[row_start<NRB>(i) + j], a_cur, bfr[j]);
            a_cur = a_nxt;
        }
        __syncwarp();
    }
    cp_async_wait<0>();
}

template <int NRB>
__global__ void __launch_bounds__(32 * PSCA_FACW_IPC, PSCA_FACW_MINB) fac_sweep_w(FacArgs a) {
    using S = TWS<NRB>;
    constexpr int LP = S::LP, LPC = S::LPC, NTL = S::NTL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * S::IPC + warp;
    if (b >= a.B) return;
    if (a.status[b] != PSCA_RUNNING) return;
    const int L = a.L;
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1, kc = c4 >> 1;
    const unsigned FULL = 0xffffffffu;
    const size_t bN = (size_t)b * a.N;

    // ---- finalise iteration k_new - 1 -----------------------------------------
    if (a.k_new > 0) {
        int flag = 0;
        if (lane == 0) {
            double dx2 = 0.0, minq = INFINITY;
            const double* rp = a.red_part + (size_t)b * a.n_chunks * 4;
            for (int c = 0; c < a.n_chunks; ++c) {
                dx2 += rp[4 * c];
                minq = (rp[4 * c + 1] < minq) ? rp[4 * c + 1] : minq;
            }
            flag = fac_finalize_core(a, b, a.k_new - 1, dx2, minq, a.inst + (size_t)b * 4);
        }
        flag = __shfl_sync(FULL, flag, 0);
        if (flag == PSCA_QFLOOR) {
            for (int n = lane; n < a.N; n += 32) a.x_next[bN + n] = a.x_cur[bN + n];
            return;
        }
        if (flag != 0 || a.k_new >= a.T) return;
    }
    // deferred rebuild: the list and the first gather stages go out before the
    // prior terms, so the pilot columns arrive underneath them
    const int mcnt = (a.mov_cnt && a.k_new > 0) ? a.mov_cnt[b] : -1;
    unsigned char* wsm = smem_raw + warp * S::WARP_SMEM;
    if (mcnt >= 0) mov_begin<NRB>(a, b, mcnt, wsm, lane);
    const double prior_value =
        a.prior_ext ? 0.0 : warp_prior_terms(a, b, (a.k_new == 0 ? a.x_cur : a.x_next) + bN, lane);

    // ---- Sigma_k in accumulator fragments ---------------------------------------
    // tile t = (i, j): lane holds component p of entries (4 i + r8 / 2, 8 j + 2 c4 + h)
    double acc[NTL][2];
    {
        const bool zero_weights = a.k_new == 0;
        double2* D = a.incremental ? a.dmat + (size_t)b * dmat_stride(make_geo(L, NRB), L)
                                   : nullptr;
        const double omr =
            (a.incremental && a.k_new > 0) ? __dsub_rn(1.0, a.steps[(size_t)b * a.steps_stride + a.k_new - 1]) : 0.0;
        // one column chunk per instance on this path (use_warp_factor)
        const double2* sp = a.sig_part + (size_t)b * NTL * 32;
        const double s2 = a.noise[b];
        // entry masks of tile t = (ti, tj): zero padding and upper part, noise on
        // the real diagonal, identity padding pivot for odd L
        auto finish = [&](int t, int ti, int tj, double2 sxy) {
            const int l = 4 * ti + (r8 >> 1);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = 8 * tj + 2 * c4 + h;
                double v = h ? sxy.y : sxy.x;
                if (l >= L || m >= L || m > l) v = 0.0;
                if (m == l && l < L) v = p ? 0.0 : v + s2;
                if ((L & 1) && l == L && m == L && p == 0) v = 1.0;
                acc[t][h] = v;
            }
        };
        constexpr int GA = 6;   // tiles per load batch (bounded register pressure)
        if (mcnt >= 0) {
            // deferred rebuild: (1 - rho) D first (batched loads while the
            // accumulators are still free), the listed columns on top by DMMA
#pragma unroll
            for (int t0 = 0; t0 < NTL; t0 += GA) {
                double2 dv[GA];
#pragma unroll
                for (int u = 0; u < GA; ++u)
                    dv[u] = (t0 + u < NTL && D) ? D[(t0 + u) * 32 + lane] : make_double2(0.0, 0.0);
#pragma unroll
                for (int u = 0; u < GA; ++u)
                    if (t0 + u < NTL) {
                        acc[t0 + u][0] = omr * dv[u].x;
                        acc[t0 + u][1] = omr * dv[u].y;
                    }
            }
            mov_rebuild<NRB>(a, b, mcnt, acc, wsm, lane);
            int ti = 0, tj = 0;
#pragma unroll
            for (int t = 0; t < NTL; ++t) {
                const double2 sxy = make_double2(acc[t][0], acc[t][1]);
                if (D) D[t * 32 + lane] = sxy;
                finish(t, ti, tj, sxy);
                TILE_NEXT(ti, tj)
            }
        } else {
            int ti = 0, tj = 0;
#pragma unroll
            for (int t0 = 0; t0 < NTL; t0 += GA) {
                double2 sv[GA], dv[GA];
#pragma unroll
                for (int u = 0; u < GA; ++u) {
                    const int t = t0 + u;
                    sv[u] = make_double2(0.0, 0.0);
                    dv[u] = make_double2(0.0, 0.0);
                    if (t < NTL && !zero_weights) {
                        sv[u] = sp[t * 32 + lane];
                        if (D) dv[u] = D[t * 32 + lane];
                    }
                }
#pragma unroll
                for (int u = 0; u < GA; ++u) {
                    const int t = t0 + u;
                    if (t < NTL) {
                        double2 sxy = sv[u];
                        if (D) {
                            sxy = zero_weights ? make_double2(0.0, 0.0)
                                               : make_double2(fma(omr, dv[u].x, sxy.x),
                                                              fma(omr, dv[u].y, sxy.y));
                            D[t * 32 + lane] = sxy;
                        }
                        finish(t, ti, tj, sxy);
                        TILE_NEXT(ti, tj)
                    }
                }
            }
        }
    }
    // Frobenius norm of Sigma (lower entries twice, the diagonal once)
    double frob;
    {
        double s = 0.0;
        int ti = 0, tj = 0;
#pragma unroll
        for (int t = 0; t < NTL; ++t) {
            const int l = 4 * ti + (r8 >> 1);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = 8 * tj + 2 * c4 + h;
                const double w = (l < L && m < L) ? (m < l ? 2.0 : (m == l ? 1.0 : 0.0)) : 0.0;
                s = fma(w * acc[t][h], acc[t][h], s);
            }
            TILE_NEXT(ti, tj)
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        frob = sqrt(s);
    }

    // ---- Hermitian sweep operator, 2x2 block pivots, in the fragments ----------
    double logdet;
    const bool ok = warp_sweep<NRB>(acc, wsm, L, a.record_objective, logdet);
    if (!ok) {
        if (lane == 0) {
            a.status[b] = PSCA_CHOL_FAIL;
            if (a.cond_est) a.cond_est[b] = INFINITY;
        }
        return;
    }
    // ---- P = -(swept) lower fragments (zero padding, real diagonal) -----------
    double2* pf = a.pfrag + (size_t)b * NTL * 32;
    int ti = 0, tj = 0;
#pragma unroll
    for (int t = 0; t < NTL; ++t) {
        const int l = 4 * ti + (r8 >> 1);
        double v[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = 8 * tj + 2 * c4 + h;
            v[h] = (l < L && m < L && m <= l && !(m == l && p)) ? -acc[t][h] : 0.0;
        }
        pf[t * 32 + lane] = make_double2(v[0], v[1]);
        TILE_NEXT(ti, tj)
    }
    if (lane == 0) {
        double* in = a.inst + (size_t)b * 4;
        in[0] = frob;
        in[1] = logdet;
        in[2] = 0.0;   // trace(P Sigma_hat): fac_prod_t
        in[3] = prior_value;
    }
}

// product CTA width: a warp owns whole row tiles, so eight warps cut the
// longest warp of L = 40 from three row tiles to two (c1: 0.227 -> 0.200 ms per
// 4096 instances at 256 x 4 CTAs per SM; 320 x 3: 0.197; 256 x 3: 0.214)
template <int NRB>
__host__ __device__ constexpr int prod_threads() { return NRB >= 8 ? 256 : 128; }
template <int NRB, int NTH>
__global__ void __launch_bounds__(NTH, 4) fac_prod_t(FacArgs a) {
    constexpr int LP = 4 * NRB;
    constexpr int NTL = rebuild_block_count(NRB);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double sred[SRED];
    const int b = blockIdx.x;
    if (a.status[b] != PSCA_RUNNING || a.k_new >= a.T) return;
    const int ld = LP + 1;
    double2* X = reinterpret_cast<double2*>(smem_raw);   // [LP][ld]
    double2* G = X + (size_t)LP * ld;                    // [LP][ld], Sigma_hat staged here first
    stage_emp(a, b, G, ld);
    {   // P from the lower fragments, mirrored (every entry of the LP x LP block written)
        const double2* pf = a.pfrag + (size_t)b * NTL * 32;
        double* Xd = reinterpret_cast<double*>(X);
        for (int e = threadIdx.x; e < NTL * 32; e += NTH) {
            const int t = e >> 5, lane = e & 31;
            const int r8 = lane >> 2, c4 = lane & 3, p = r8 & 1;
            int i = 0, base = 0;
            while (base + (4 * i + 3) / 8 + 1 <= t) {
                base += (4 * i + 3) / 8 + 1;
                ++i;
            }
            const int l = 4 * i + (r8 >> 1);
            const double2 v = pf[e];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = 8 * (t - base) + 2 * c4 + h;
                const double x = h ? v.y : v.x;
                if (m < l) {
                    Xd[2 * (l * ld + m) + p] = x;
                    Xd[2 * (m * ld + l) + p] = p ? -x : x;
                } else if (m == l) {
                    Xd[2 * (l * ld + l) + p] = x;
                }
            }
        }
    }
    double trace;
    double* od = reinterpret_cast<double*>(a.frags + (size_t)b * (size_t)NRB * (NRB + 1) * FRAG_SLOTS);
    products_pass<NRB, NTH>(a, b, X, G, G, od, sred, trace);
    if (threadIdx.x == 0 && a.record_objective) a.inst[(size_t)b * 4 + 2] = trace;
}
