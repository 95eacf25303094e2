// psca_fast.cuh -- compiled-shape kernels of the PSCA hot path (sm_100a).
// Included by psca.cu inside its anonymous namespace (uses its helpers,
// ColArgs / FacArgs, assemble_sigma, fac_* and the fragment layout).
//
// Two device functions carry the work:
//   col_pass<NRB>     one column pass of one instance over a column range:
//                     quadratic forms on DMMA, fused per-device update,
//                     WS = S diag(w_new), covariance rebuild on DMMA
//   factor_pass<RT>   Hermitian PD inverse of the L x L Sigma held in SMEM
//                     (register-tiled Gauss-Jordan), A = P^H Sigma_hat P, and
//                     the packed P'/A' fragments for the next col_pass
// and three kernels use them:
//   column_kernel_t / factor_solve_t   the two-kernel-per-iteration path
//                                      (any batch, column chunks per instance)
//   psca_persistent_t                  one launch for the whole solve: each CTA
//                                      owns one instance at a time for all T
//                                      iterations; fragments never leave SMEM,
//                                      Sigma goes from the rebuild accumulators
//                                      straight into the factor's SMEM, and the
//                                      latency-bound factor phase of one CTA
//                                      overlaps the DMMA work of the other
//                                      resident CTA.

// Quad-stage shape, chosen by A/B measurement on B200 (profiles/README.md):
// one DMMA accumulator chain per matrix and the B fragments loaded from SMEM
// per k-step (2.42 ms vs 3.05 ms per launch with two chains and
// register-resident B fragments: register pressure, not the ~32-cycle DMMA
// latency, was the limit), one 8-column block per warp (2.42 vs 2.55 ms with
// two blocks and four row-block groups).
#ifndef PSCA_QCB
#define PSCA_QCB 1
#endif
#ifndef PSCA_UPD_ONE
#define PSCA_UPD_ONE 1
#endif
#ifndef PSCA_BLOCK_SWEEP
#define PSCA_BLOCK_SWEEP 1
#endif
#ifndef PSCA_DSWEEP
#define PSCA_DSWEEP 0    // 1: factor_pass sweeps in DMMA fragments (dmma_sweep); 0: USWEEP
#endif
#ifndef PSCA_USWEEP
#define PSCA_USWEEP 1    // block sweep with U_j = M conj(C_j) shared per column
#endif
#ifndef PSCA_ADJ_INV
#define PSCA_ADJ_INV 1   // 2x2 pivot block inverse as adj(K)/det(K)
#endif
constexpr int QCB = PSCA_QCB;                // 8-column blocks per warp in the quad stage
constexpr int QPARTS = NWARP / (NCB / QCB);  // row-block groups (LPT-balanced)

template <int NRB>
struct TG {
    static constexpr int LP = 4 * NRB;
    static constexpr int LP8 = (LP + 7) & ~7;
    static constexpr int NB = NRB * (NRB + 1);
    static constexpr int NBLK = rebuild_block_count(NRB);
    static constexpr int MAXBW = (NBLK + NWARP - 1) / NWARP;
    static constexpr int RPT = LP8 / 8;            // tile rows per warp (copy / WS build)
    static constexpr int RT = (LP + 15) / 16;       // factor register tile
    static constexpr int WCAP = 16;                 // packed rebuild slots per round
    static constexpr size_t S_BYTES = (size_t)LP8 * NCT * 16;
    static constexpr size_t W_BYTES = (size_t)LP8 * WCAP * 16;
    static constexpr size_t F_BYTES = (size_t)NB * FRAG_SLOTS * 16;
    static constexpr size_t SMALL = (size_t)QPARTS * NCT * 2 * 8 + NCT * 8;   // quad partials, v
    static constexpr size_t TILE_BYTES = 2 * S_BYTES + 2 * W_BYTES;
    // Fragments are staged in SMEM beside the tile buffers: lane-ready
    // (FRAG_SLOTS = 24 per block, {re, im, -im}) when that fits (NRB <= 16),
    // else compacted to {re, im} (16 per block; the -im lanes flip the sign
    // bit after the load), which still fits at NRB = 20 (L = 80).
    static constexpr bool FIT24 = TILE_BYTES + F_BYTES + SMALL <= 227 * 1024;
    static constexpr size_t F16_BYTES = (size_t)NB * 16 * 16;
    static constexpr bool FIT16 = TILE_BYTES + F16_BYTES + SMALL <= 227 * 1024;
    static constexpr bool FR_SMEM = FIT24 || FIT16;
    static constexpr int FR_SLOTS = FIT24 ? FRAG_SLOTS : (FIT16 ? 16 : FRAG_SLOTS);
    static constexpr size_t COL_SMEM =
        TILE_BYTES + (FR_SMEM ? (size_t)NB * FR_SLOTS * 16 : 0) + SMALL;
    static constexpr size_t FAC_BYTES = (size_t)4 * LP * 16 + (size_t)2 * LP * (LP + 1) * 16;
    static constexpr size_t UNION = (TILE_BYTES > FAC_BYTES) ? TILE_BYTES : FAC_BYTES;
    static constexpr size_t PERSIST_SMEM = F_BYTES + UNION + SMALL;
};

// rebuild C blocks owned by this warp: w, w+8, ... in row-major lower order,
// packed (i << 8) | j
template <int NRB>
__device__ __forceinline__ void rebuild_slots(int (&slot)[TG<NRB>::MAXBW], int& nbw) {
    const int warp = threadIdx.x >> 5;
    nbw = 0;
    int idx = 0;
#pragma unroll 1
    for (int i = 0; i < NRB; ++i) {
        const int jmax = (4 * i + 3) / 8;
        for (int j = 0; j <= jmax; ++j, ++idx) {
            if ((idx % NWARP) == warp) {
#pragma unroll
                for (int t = 0; t < TG<NRB>::MAXBW; ++t)
                    if (t == nbw) slot[t] = (i << 8) | j;
                ++nbw;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// col_pass: one PSCA column pass (estimators.py:262-276 for columns
// [n_begin, n_end)) of instance b at iteration k.
//   FR    P'/A' fragments (SMEM or global), FRAG_SLOTS double2 per block
//   S0/S1 tile double buffer (swizzled rows of 32 columns)
//   WS/SP packed rebuild operands: S diag(v) and S for the columns with v != 0
// Software pipeline over 32-column tiles, two barriers per tile:
//   [barrier; cp.async prefetch of tile t+1]
//   phase A(t)  quad forms of tile t (warp -> 8-column block x row-block half,
//               B fragments in registers, 4 DMMA chains) and the deferred
//               rebuild of tile t-1 over its packed slots (warp -> its lower
//               C blocks) -- both pure DMMA work on disjoint buffers
//   sync
//   phase B(t)  per-device update of tile t (every warp, lane = column; warp 0
//               stores), ballot-compaction of the moving columns into WS/SP,
//               then S(t)'s buffer is refilled with tile t+2
//   sync
// v = w_new (full rebuild) or rho * cand * g (incremental: the increment of
// D = Sigma - sigma^2 I).  On return acc holds the pass's rebuild C fragments,
// warp 0 holds the per-lane partial sum of (x_next - x)^2 and min q, all
// cp.async groups are retired and the CTA is synchronised.
// ---------------------------------------------------------------------------

template <int NRB, int FS = FRAG_SLOTS>
__device__ __forceinline__ void col_pass(const ColArgs& a, int b, int k,
                                         const double* __restrict__ x_cur,
                                         double* __restrict__ x_next, int n_begin, int n_end,
                                         double2* S0, double2* S1, double2* WS, double2* SP,
                                         const double2* FR,
                                         double* qr_s, double (&acc)[TG<NRB>::MAXBW][2],
                                         const int (&slot)[TG<NRB>::MAXBW], int nbw,
                                         double& p_dx2, double& p_minq) {
    using G = TG<NRB>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r8 = lane >> 2, c4 = lane & 3;
    const size_t bN = (size_t)b * a.N;
    const double2* sb = a.pilots + (size_t)b * a.L * a.N;

    // ---- per-lane constants --------------------------------------------------
    const int cp_dst = warp * NCT + (lane ^ swz(warp));   // tile slot (+ s*8*NCT)
    const int cb = (warp % (NCB / QCB)) * QCB;   // first of this warp's column blocks
    const int half = warp / (NCB / QCB);         // row-block group
    unsigned long long rowmask = 0ull;
    {
        int load[QPARTS];
        for (int h = 0; h < QPARTS; ++h) load[h] = 0;
        for (int i = NRB - 1; i >= 0; --i) {
            int h = 0;
            for (int u = 1; u < QPARTS; ++u)
                if (load[u] < load[h]) h = u;
            load[h] += 2 * (i + 1);
            if (h == half) rowmask |= (1ull << i);
        }
    }
    int qoff[2];   // quad B fragment (m = 2kk + c4/2, n = 8cb + r8), k-step parity
#pragma unroll
    for (int par = 0; par < 2; ++par) {
        const int cpr = c4 >> 1;
        const int sw = (cpr << 2) | (2 * par);
        qoff[par] = 2 * (cpr * NCT + cb * 8 + (r8 ^ sw)) + (c4 & 1);
    }
    int epoff[2];  // epilogue S at C-fragment positions (+ i*8*NCT)
    {
        const int se = swz(r8 >> 1);
#pragma unroll
        for (int j = 0; j < 2; ++j)
            epoff[j] = 2 * ((r8 >> 1) * NCT + cb * 8 + ((2 * c4 + j) ^ se)) + (r8 & 1);
    }
    // lane's fragment slot; with the compact 16-slot layout the -im lanes
    // (row parity 0, k parity 1) read im and flip its sign
    const int fslot = (FS == FRAG_SLOTS)
                          ? frag_lane_slot(lane)
                          : 2 * (2 * (r8 >> 1) + (c4 >> 1)) + ((r8 & 1) != (c4 & 1));
    const unsigned long long fsgn =
        (FS != FRAG_SLOTS && (r8 & 1) == 0 && (c4 & 1) == 1) ? 0x8000000000000000ull : 0ull;
    // rebuild fragments over the packed slots (WS / SP rows of WCAP = 16 slots,
    // slot swizzle 2*(row & 3)), k-step k2 = 4 g + h, slot n = 2 k2 + (c4>>1):
    //   A (WS):  l = 4i + (r8>>1), component p^q, sign p&q
    //            n ^ 2(l&3) = 8 g + 2 (h ^ sa) + (c4>>1),  sa = r8>>1
    //   B (SP):  m = 8j + r8, component q
    //            n ^ 2(m&3) = 8 g + 2 (h ^ sbb) + (c4>>1), sbb = r8&3
    int wa_lane[4], b_lane[4];
    unsigned long long wsgn;
    {
        const int p = r8 & 1, q = c4 & 1, cpr = c4 >> 1;
        const int sa = r8 >> 1;
        const int sbb = r8 & 3;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            wa_lane[h] = 4 * (h ^ sa) + 2 * cpr + (p ^ q);
            b_lane[h] = 4 * (h ^ sbb) + 2 * cpr + q;
        }
        wsgn = (p & q) ? 0x8000000000000000ull : 0ull;
    }
#pragma unroll
    for (int t = 0; t < G::MAXBW; ++t) acc[t][0] = acc[t][1] = 0.0;
    p_dx2 = 0.0;
    p_minq = INFINITY;

    const bool known = (a.kind == PSCA_ML_K || a.kind == PSCA_MAP_K);
    const double hi = known ? 1.0 : (a.kind == PSCA_ML_UD ? INFINITY : a.eff.g_high);
    const double rho = a.steps[(size_t)b * a.steps_stride + k];
    const double omr = __dsub_rn(1.0, rho);

    auto issue_tile = [&](double2* buf, int col0) {
        const int n = col0 + lane;
        const bool colok = n < a.N;
#pragma unroll
        for (int s2 = 0; s2 < G::RPT; ++s2) {
            const int m = warp + 8 * s2;
            const bool ok = colok && (m < a.L);
            const double2* src = ok ? (sb + (size_t)m * a.N + n) : sb;
            cp_async16(buf + cp_dst + s2 * 8 * NCT, src, ok ? 16 : 0);
        }
        cp_async_commit();
    };

    // rebuild over packed slots [0, cnt) of WS / SP (warp -> its lower C blocks)
    auto rebuild = [&](int cnt) {
        const double* Wd = reinterpret_cast<const double*>(WS);
        const double* Pd = reinterpret_cast<const double*>(SP);
        const int nk2 = (cnt + 1) >> 1;
#pragma unroll
        for (int t2 = 0; t2 < G::MAXBW; ++t2) {
            if (t2 < nbw) {
                const int bi = slot[t2] >> 8, bj = slot[t2] & 0xff;
                const int abase = 2 * (4 * bi + (r8 >> 1)) * G::WCAP;
                const int bbase = 2 * (8 * bj + r8) * G::WCAP;
                double e1[2] = {0.0, 0.0};
#pragma unroll
                for (int k2 = 0; k2 < G::WCAP / 2; ++k2) {
                    if (k2 < nk2) {
                        const int h = k2 & 3, g8 = 16 * (k2 >> 2);
                        const double av = xsign(Wd[abase + wa_lane[h] + g8], wsgn);
                        const double bv = Pd[bbase + b_lane[h] + g8];
                        if (k2 & 1) dmma(e1, av, bv);
                        else dmma(acc[t2], av, bv);
                    }
                }
                acc[t2][0] += e1[0];
                acc[t2][1] += e1[1];
            }
        }
    };

    const int ntiles = (n_end - n_begin + NCT - 1) / NCT;
    if (ntiles > 0) issue_tile(S0, n_begin);
    int pend = 0;   // packed slots of the previous tile awaiting their rebuild

    for (int t = 0; t < ntiles; ++t) {
        double2* S = (t & 1) ? S1 : S0;
        const double* Sd = reinterpret_cast<const double*>(S);
        const int col0 = n_begin + t * NCT;
        // per-device operands of this tile (lane = column), latency hidden by phase A
        const int ncol = col0 + lane;
        const bool cvalid = ncol < n_end;
        double x = 0.0, g = 1.0, pg = 0.0;
        if (cvalid && (!PSCA_UPD_ONE || warp == 0)) {
            x = x_cur[ncol];
            if (known) g = a.gains[bN + ncol];
            if (a.kind == PSCA_MAP_UR || (a.kind == PSCA_MAP_K && a.pairwise))
                pg = a.pgrad[bN + ncol];
            else if (a.kind == PSCA_MAP_K) pg = a.prior_lin[ncol];
        }
        cp_async_wait<0>();
        __syncthreads();
        // prefetch tile t+1 into the other buffer (its tile t-1 was consumed in B(t-1))
        if (t + 1 < ntiles) issue_tile((t & 1) ? S0 : S1, col0 + NCT);

        // ---- phase A: deferred rebuild of tile t-1, quad forms of tile t -----
        if (pend > 0) rebuild(pend);
        {
            double qa[QCB][2], ra[QCB][2];
#pragma unroll
            for (int j = 0; j < QCB; ++j) qa[j][0] = qa[j][1] = ra[j][0] = ra[j][1] = 0.0;
#pragma unroll
            for (int i = 0; i < NRB; ++i) {
                if ((rowmask >> i) & 1ull) {
                    double tc[QCB][2], uc[QCB][2];
#pragma unroll
                    for (int j = 0; j < QCB; ++j) tc[j][0] = tc[j][1] = uc[j][0] = uc[j][1] = 0.0;
                    const double2* f = FR + i * (i + 1) * FS + fslot;
#pragma unroll
                    for (int kk = 0; kk < 2 * (i + 1); ++kk) {
                        const double2 pa = f[kk * FS];
                        const double pv = (FS == FRAG_SLOTS) ? pa.x : xsign(pa.x, fsgn);
                        const double av = (FS == FRAG_SLOTS) ? pa.y : xsign(pa.y, fsgn);
#pragma unroll
                        for (int j = 0; j < QCB; ++j) {
                            const double bv = Sd[qoff[kk & 1] + kk * 4 * NCT + 16 * j];
                            dmma(tc[j], pv, bv);
                            dmma(uc[j], av, bv);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < QCB; ++j) {
                        const double s0 = Sd[epoff[0] + i * 8 * NCT + 16 * j];
                        const double s1 = Sd[epoff[1] + i * 8 * NCT + 16 * j];
                        qa[j][0] = fma(s0, tc[j][0], qa[j][0]);
                        qa[j][1] = fma(s1, tc[j][1], qa[j][1]);
                        ra[j][0] = fma(s0, uc[j][0], ra[j][0]);
                        ra[j][1] = fma(s1, uc[j][1], ra[j][1]);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < QCB; ++j) {
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    qa[j][0] += __shfl_xor_sync(0xffffffffu, qa[j][0], o);
                    qa[j][1] += __shfl_xor_sync(0xffffffffu, qa[j][1], o);
                    ra[j][0] += __shfl_xor_sync(0xffffffffu, ra[j][0], o);
                    ra[j][1] += __shfl_xor_sync(0xffffffffu, ra[j][1], o);
                }
                if (r8 == 0) {
                    const int n0 = (cb + j) * 8 + 2 * c4;
                    double* d = qr_s + half * NCT * 2;
                    d[2 * n0] = qa[j][0];
                    d[2 * n0 + 1] = ra[j][0];
                    d[2 * (n0 + 1)] = qa[j][1];
                    d[2 * (n0 + 1) + 1] = ra[j][1];
                }
            }
        }
        __syncthreads();

        // ---- phase B: update (estimators.py:272-276) + packed WS / SP --------
        // The per-device update runs in warp 0 only (lane = column) and is
        // broadcast through SMEM: its DDIV/DMUL chain shares the FP64 pipe
        // with the other CTA's DMMAs, so it is not replicated per warp.
        {
            double v = 0.0;
#if PSCA_UPD_ONE
            double* v_s = qr_s + QPARTS * NCT * 2;
            if (warp == 0) {
#endif
            if (cvalid) {
                double q = qr_s[2 * lane], r = qr_s[2 * lane + 1];
#pragma unroll
                for (int h = 1; h < QPARTS; ++h) {
                    q += qr_s[h * NCT * 2 + 2 * lane];
                    r += qr_s[h * NCT * 2 + 2 * lane + 1];
                }
                const double diff = __dsub_rn(q, r);
                double grad;
                if (a.kind == PSCA_ML_K) grad = __dmul_rn(g, diff);
                else if (a.kind == PSCA_MAP_K) grad = __dadd_rn(__dmul_rn(g, diff), pg);
                else if (a.kind == PSCA_ML_UD) grad = diff;
                else grad = __dadd_rn(diff, pg);
                const double gq = known ? __dmul_rn(g, q) : q;
                const double coef = __dmul_rn(gq, gq);
                const double cand = np_clip(__dsub_rn(x, __ddiv_rn(grad, coef)), 0.0, hi);
                const double rc = __dmul_rn(rho, cand);
                const double xn = __dadd_rn(__dmul_rn(omr, x), rc);
                if (a.incremental) v = known ? __dmul_rn(rc, g) : rc;
                else v = known ? __dmul_rn(xn, g) : xn;
                if (warp == 0) {
                    x_next[ncol] = xn;
                    if (a.iterates)
                        a.iterates[((size_t)b * (a.T + 1) + k + 1) * a.N + ncol] = xn;
                    const double dx = __dsub_rn(xn, x);
                    p_dx2 = fma(dx, dx, p_dx2);
                    p_minq = (q < p_minq) ? q : p_minq;
                }
            }
#if PSCA_UPD_ONE
                v_s[lane] = v;
            }
            __syncthreads();
            v = v_s[lane];
#endif
            const unsigned mask = __ballot_sync(0xffffffffu, v != 0.0);
            const int nnz = __popc(mask);
            const int pos = __popc(mask & ((1u << lane) - 1u));
            const int sw = 2 * (warp & 3);
            // WCAP slots per round; a tile with more than 16 moving columns
            // (early iterations only) rebuilds its first 16 here, the rest in A(t+1)
            int lo = 0;
            for (;;) {
                const int cnt = min(nnz - lo, G::WCAP);
#pragma unroll
                for (int s2 = 0; s2 < G::RPT; ++s2) {
                    const int l = warp + 8 * s2;
                    if (v != 0.0 && pos >= lo && pos < lo + G::WCAP) {
                        const double2 sv = S[cp_dst + s2 * 8 * NCT];
                        const int o = l * G::WCAP + ((pos - lo) ^ sw);
                        WS[o] = make_double2(v * sv.x, v * sv.y);
                        SP[o] = sv;
                    }
                    if (lane == 0 && (cnt & 1)) {   // zero slot after an odd count
                        const int o = l * G::WCAP + (cnt ^ sw);
                        WS[o] = make_double2(0.0, 0.0);
                        SP[o] = make_double2(0.0, 0.0);
                    }
                }
                if (nnz - lo <= G::WCAP) {
                    pend = cnt > 0 ? cnt : 0;
                    break;
                }
                __syncthreads();
                rebuild(G::WCAP);
                __syncthreads();
                lo += G::WCAP;
            }
        }
    }
    __syncthreads();
    if (pend > 0) rebuild(pend);
    cp_async_wait<0>();
    __syncthreads();
}

// Reduce warp 0's per-lane (dx2, min q) partials; result valid in thread 0.
__device__ __forceinline__ void reduce_pass_partials(double& dx2, double& minq) {
    if ((threadIdx.x >> 5) == 0) {
        for (int o = 16; o > 0; o >>= 1) {
            dx2 += __shfl_xor_sync(0xffffffffu, dx2, o);
            const double mq = __shfl_xor_sync(0xffffffffu, minq, o);
            minq = (mq < minq) ? mq : minq;
        }
    }
}

// Rebuild C fragments -> lower triangle of Sigma in X (rows / cols < L).
// Incremental mode (Dd != nullptr): D_{k+1} = omr * D_k + acc, kept in Dd.
template <int NRB>
__device__ __forceinline__ void acc_to_sigma(const double (&acc)[TG<NRB>::MAXBW][2],
                                             const int (&slot)[TG<NRB>::MAXBW], int nbw,
                                             double2* X, int ld, int L, double* Dd, double omr) {
    const int lane = threadIdx.x & 31;
    const int r8 = lane >> 2, c4 = lane & 3;
    double* Xd = reinterpret_cast<double*>(X);
#pragma unroll
    for (int t = 0; t < TG<NRB>::MAXBW; ++t) {
        if (t < nbw) {
            const int i = slot[t] >> 8, j = slot[t] & 0xff;
            const int l = 4 * i + (r8 >> 1), p = r8 & 1;
            const int m0 = 8 * j + 2 * c4;
            if (l < L) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = m0 + h;
                    if (m <= l) {
                        double val = acc[t][h];
                        if (Dd) {
                            const size_t o = 2 * ((size_t)l * L + m) + p;
                            val = fma(omr, Dd[o], val);
                            Dd[o] = val;
                        }
                        Xd[2 * (l * ld + m) + p] = val;
                    }
                }
            }
        }
    }
}

// Upper triangle by conjugation, sigma^2 on the (real) diagonal.
__device__ __forceinline__ void finish_sigma(double2* X, int ld, int L, double s2) {
    __syncthreads();
    for (int e = threadIdx.x; e < L * L; e += blockDim.x) {
        const int i = e / L, j = e - i * L;
        if (i < j) {
            const double2 v = X[j * ld + i];
            X[i * ld + j] = make_double2(v.x, -v.y);
        } else if (i == j) {
            X[i * ld + i] = make_double2(X[i * ld + i].x + s2, 0.0);
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// factor_pass: X holds Sigma (L x L Hermitian, row stride ld = LP + 1) on
// entry.  Thread (ty, tx) = (tid/16, tid%16) owns the RT x RT entries
// (ty + 16u, tx + 16v).  Gauss-Jordan sweep in registers (pivot row / column
// ping-pong staged in SMEM, one barrier per pivot; pivots = LDL^H pivots),
// symmetrisation (covlinalg.py:107, 112-114), trace(P Sigma_hat) when the
// objective is recorded, G = Sigma_hat P and A = P^H G register-tiled, and
// the packed P'/A' fragments written to od (SMEM or global).  Returns false
// (uniformly) when a pivot is not positive.  Ends synchronised.
// ---------------------------------------------------------------------------
// Issue the cp.async copy of Sigma_hat (L x L, row stride ld) into Es.
// (t0, nt > 0: issued by the nt threads from t0 on only)
__device__ __forceinline__ void stage_emp(const FacArgs& a, int b, double2* Es, int ld, int t0 = 0,
                                          int nt = 0) {
    const double2* E = a.emp_cov + (size_t)b * a.L * a.L;
    const int L = a.L;
    if (nt <= 0) nt = blockDim.x;
    if ((int)threadIdx.x < t0 || (int)threadIdx.x >= t0 + nt) {
        cp_async_commit();
        return;
    }
    for (int e = threadIdx.x - t0; e < L * L; e += nt) {
        const int i = e / L, j = e - i * L;
        cp_async16(Es + i * ld + j, E + e, 16);
    }
    cp_async_commit();
}

template <int NRB, int NTH>
struct TF {
    static constexpr int LP = 4 * NRB;
    static constexpr int NBL = LP / 2;                 // 2x2 block rows
    static constexpr int NLB = NBL * (NBL + 1) / 2;    // lower 2x2 blocks (incl. diagonal)
    static constexpr int SL = (NLB + NTH - 1) / NTH;   // lower-block slots per thread
    static constexpr int NFB = NBL * NBL;              // all 2x2 blocks
    static constexpr int SG = (NFB + NTH - 1) / NTH;   // full-block slots per thread
};
// factor CTA size of the two-kernel path: 128 threads, Sigma_hat read from L2,
// so four instances share an SM and hide each other's pivot-barrier latency
constexpr int NT_FAC = 128;
// L >= 64: the register-tiled products need more threads (128 spill at L = 80)
// and the CTA is alone on its SM anyway (SMEM: 212 KB at L = 80), so use 512
// threads: two lower 2x2 blocks per thread in the block sweep instead of four
// (c3 L = 80 factor 3.14 -> 2.96 ms per 1024 instances vs 256 threads).
#ifndef PSCA_FAC_WIDE
#define PSCA_FAC_WIDE 512
#endif
template <int NRB>
__host__ __device__ constexpr int fac_threads() { return NRB >= 16 ? PSCA_FAC_WIDE : NT_FAC; }
// dynamic SMEM of factor_solve_t: pivot buffers, X, G
template <int NRB>
__host__ __device__ constexpr size_t fac_smem() {
    return (size_t)4 * (4 * NRB) * 16 + (size_t)2 * (4 * NRB) * (4 * NRB + 1) * 16;
}

// (bi, bj), bi >= bj, of lower 2x2 block number t (row-major)
__device__ __forceinline__ void lower_block(int t, int& bi, int& bj) {
    int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) / 2 > t) --i;
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    bi = i;
    bj = t - i * (i + 1) / 2;
}

// ---------------------------------------------------------------------------
// dmma_sweep: the Hermitian sweep operator (2x2 block pivots, the same pivots
// as LDL^H) with the matrix held in DMMA accumulator fragments.
//
// The lower triangle of the LP x LP matrix is tiled like the rebuild blocks:
// tile (bi, bj) = 4 complex rows x 8 complex columns, stored as one m8n8k4 C
// fragment in the real 2x2 expansion (lane (r8, c4) holds component r8 & 1 of
// entries (4 bi + r8 / 2, 8 bj + 2 c4 + h), h = 0, 1).  Warp w owns the tiles
// w, w + NW, ... (row-major lower order).  Step K = {k, k+1}:
//   phase U  thread j < LP forms U_j = M conj(C_j) (M = K^-1 = adj(K)/det(K),
//            C_j = (a_jk, a_j,k+1), K entries zeroed) into SMEM;
//   phase V  every owned tile takes ONE DMMA: acc += (-C^) U with C^ the real
//            expansion of the two staged columns (A operand, k = 4 = 2
//            complex) and U as B operand -- the rank-2 trailing update
//            a_ij -= C_i U_j; lanes on the K rows / columns are replaced by
//            U_j (row K), conj(U_i) (column K) and -M (the K block); the next
//            pivot block's columns and K' itself are staged from the
//            fragments.
// Compared with per-thread 2x2 blocks (8 shared-memory loads of 16 bytes per
// block per step, the factor kernel's limiter), a tile costs two 8-byte
// operand loads and one DMMA per step.  SMEM scratch (ub, cs) lives in X,
// which is free while the matrix is in registers; on return X holds
// P = Sigma^-1 (full Hermitian, zero padding) unless a pivot failed.
// ---------------------------------------------------------------------------
template <int NRB, int NTH>
struct TSW {
    static constexpr int LP = 4 * NRB;
    static constexpr int LPC = LP + ((NRB & 1) ? 0 : 4);   // staged-column stride (banks)
    static constexpr int NTL = rebuild_block_count(NRB);    // lower tiles
    static constexpr int NW = NTH / 32;
    static constexpr int TPW = (NTL + NW - 1) / NW;         // tiles per warp (max)
};

template <int NRB, int NTH>
__device__ __forceinline__ bool dmma_sweep(double2* X, int ld, int L, bool want_logdet,
                                           double& logdet) {
    using S = TSW<NRB, NTH>;
    constexpr int LP = S::LP, LPC = S::LPC;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1, kc = c4 >> 1;
    __shared__ double kv[2][4];
    __shared__ double msh[4];
    // owned tiles: row / column tile, and the step-independent operand offsets
    // (doubles) of this lane's A (staged columns) and B (U) fragment elements;
    // slots past the warp's count point at offset 0 and never match a pivot
    int tbi[S::TPW], tbj[S::TPW], aoff[S::TPW], boff[S::TPW];
#pragma unroll
    for (int t = 0; t < S::TPW; ++t) {
        tbi[t] = -64;
        tbj[t] = -64;
        aoff[t] = 0;
        boff[t] = 0;
    }
    {
        int idx = 0, nt = 0;
#pragma unroll 1
        for (int i = 0; i < NRB; ++i) {
            const int jmax = (4 * i + 3) / 8;
            for (int j = 0; j <= jmax; ++j, ++idx) {
                if ((idx % S::NW) == warp) {
#pragma unroll
                    for (int t = 0; t < S::TPW; ++t)
                        if (t == nt) {
                            tbi[t] = i;
                            tbj[t] = j;
                            aoff[t] = 2 * (kc * LPC + 4 * i + (r8 >> 1)) + (p ^ q);
                            boff[t] = 2 * (kc * LPC + 8 * j + r8) + q;
                        }
                    ++nt;
                }
            }
        }
    }
    // load the lower triangle (zero above the diagonal and in the padding;
    // odd L: the padding pivot L is an identity row, no effect on the L x L part)
    double acc[S::TPW][2];
    const double* Xd = reinterpret_cast<const double*>(X);
#pragma unroll
    for (int t = 0; t < S::TPW; ++t) {
        const int l = 4 * tbi[t] + (r8 >> 1);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = 8 * tbj[t] + 2 * c4 + h;
            double v = 0.0;
            if (tbi[t] >= 0 && l < L && m < L && m <= l) v = Xd[2 * (l * ld + m) + p];
            if ((L & 1) && l == L && m == L && p == 0) v = 1.0;
            acc[t][h] = v;
        }
    }
    __syncthreads();   // X is scratch from here on
    double2* ub = X;                  // [2][LPC]: U(kc, j)
    double2* cs = X + 2 * LPC;        // [2 phases][2][LPC]: C(l, kc)
    const double* Ud = reinterpret_cast<const double*>(ub);
    const double* Csd = reinterpret_cast<const double*>(cs);
    // stage the columns of pivot block {k2, k2 + 1} from the fragments into
    // phase dst (and K' into kv[dst]); only tiles holding those rows / columns
    auto stage = [&](int k2, int dst) {
        double* Cn = reinterpret_cast<double*>(cs + dst * 2 * LPC);
        const int kr = k2 >> 2, kcl = k2 >> 3;
#pragma unroll
        for (int t = 0; t < S::TPW; ++t) {
            if (tbi[t] == kr || tbj[t] == kcl) {
                const int l = 4 * tbi[t] + (r8 >> 1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = 8 * tbj[t] + 2 * c4 + h;
                    const double v = acc[t][h];
                    const bool il = (l == k2 || l == k2 + 1), im = (m == k2 || m == k2 + 1);
                    if (il && im) {
                        if (m <= l) {
                            if (l == k2 && m == k2 && p == 0) kv[dst][0] = v;
                            if (l == k2 + 1 && m == k2) kv[dst][1 + p] = v;
                            if (l == k2 + 1 && m == k2 + 1 && p == 0) kv[dst][3] = v;
                            if (m == l && p == 0) {   // K' rows of the staged columns: zero
                                reinterpret_cast<double2*>(Cn)[l] = make_double2(0.0, 0.0);
                                reinterpret_cast<double2*>(Cn)[LPC + l] = make_double2(0.0, 0.0);
                            }
                        }
                    } else if (im && l > k2 + 1) {
                        Cn[2 * ((m - k2) * LPC + l) + p] = v;              // a_lm
                    } else if (il && m < k2) {
                        Cn[2 * ((l - k2) * LPC + m) + p] = p ? -v : v;     // conj(a_lm)
                    }
                }
            }
        }
    };
    stage(0, 0);
    __syncthreads();
    logdet = 0.0;
    bool ok = true;
    const int LE = (L + 1) & ~1;
    const unsigned long long sgn = (p == 0 && q == 1) ? 0ull : 0x8000000000000000ull;
    for (int k = 0; k < LE; k += 2) {
        const int ph = (k >> 1) & 1;
        const double2* cc = cs + ph * 2 * LPC;
        const double* Cd = Csd + ph * 4 * LPC;
        PROBE(10 + (k >> 1));
        const double ka = kv[ph][0], kbr = kv[ph][1], kbi = kv[ph][2], kcc = kv[ph][3];
        const double det = fma(ka, kcc, -fma(kbr, kbr, kbi * kbi));
        if (!(ka > 0.0) || !(det > 0.0)) {
            ok = false;
            break;
        }
        if (want_logdet) logdet += log(det);
        if (tid < LP) {
            const double dinv = __drcp_rn(det);
            const double m00 = kcc * dinv;
            const double m11 = ka * dinv;
            const double2 m10 = make_double2(-kbr * dinv, -kbi * dinv);
            const double2 m01 = make_double2(m10.x, -m10.y);
            const double2 pp = cc[tid], qq = cc[LPC + tid];
            ub[tid] = make_double2(fma(m01.x, qq.x, fma(m01.y, qq.y, m00 * pp.x)),
                                   fma(m01.y, qq.x, fma(-m01.x, qq.y, -m00 * pp.y)));
            ub[LPC + tid] = make_double2(fma(m11, qq.x, fma(m10.x, pp.x, m10.y * pp.y)),
                                         fma(-m11, qq.y, fma(m10.y, pp.x, -m10.x * pp.y)));
            if (tid == 0) {
                msh[0] = m00;
                msh[1] = m11;
                msh[2] = m10.x;
                msh[3] = m10.y;
            }
        }
        __syncthreads();
        // rank-2 trailing update: one DMMA per tile
#pragma unroll
        for (int t = 0; t < S::TPW; ++t) dmma(acc[t], xsign(Cd[aoff[t]], sgn), Ud[boff[t]]);
        // the K rows / columns
        const int kr = k >> 2, kcl = k >> 3;
#pragma unroll
        for (int t = 0; t < S::TPW; ++t) {
            if (tbi[t] == kr || tbj[t] == kcl) {
                const int l = 4 * tbi[t] + (r8 >> 1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = 8 * tbj[t] + 2 * c4 + h;
                    const bool il = (l == k || l == k + 1), im = (m == k || m == k + 1);
                    if (il && im) {
                        if (m <= l) {
                            double v;
                            if (l == k) v = p ? 0.0 : -msh[0];
                            else if (m == k) v = p ? -msh[3] : -msh[2];
                            else v = p ? 0.0 : -msh[1];
                            acc[t][h] = v;
                        }
                    } else if (il) {
                        acc[t][h] = Ud[2 * ((l - k) * LPC + m) + p];          // U_m
                    } else if (im) {
                        const double u = Ud[2 * ((m - k) * LPC + l) + p];     // conj(U_l)
                        acc[t][h] = p ? -u : u;
                    }
                }
            }
        }
        if (k + 2 < LE) stage(k + 2, ph ^ 1);
        __syncthreads();
    }
    if (!ok) return false;
    // P = -(swept): full Hermitian into X (zero padding rows / columns)
    double* Xw = reinterpret_cast<double*>(X);
#pragma unroll
    for (int t = 0; t < S::TPW; ++t) {
        if (tbi[t] >= 0) {
            const int l = 4 * tbi[t] + (r8 >> 1);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = 8 * tbj[t] + 2 * c4 + h;
                if (m <= l && l < LP) {
                    double v = (l < L && m < L) ? -acc[t][h] : 0.0;
                    if (m == l) {
                        Xw[2 * (l * ld + m) + p] = p ? 0.0 : v;
                    } else {
                        Xw[2 * (l * ld + m) + p] = v;
                        Xw[2 * (m * ld + l) + p] = p ? -v : v;
                    }
                }
            }
        }
    }
    return true;
}

// ---------------------------------------------------------------------------
// products_pass: X holds P = Sigma^-1 (full Hermitian, zero padding, row
// stride LP + 1) and Sigma_hat is being staged into G (cp.async, or Es null:
// read from L2).  trace(P Sigma_hat) when the objective is recorded, then
// G = Sigma_hat P and A = P G on DMMA and the packed P'/A' fragments of the
// next column pass into od.  Ends synchronised.
// ---------------------------------------------------------------------------
template <int NRB, int NTH>
__device__ __forceinline__ void products_pass(const FacArgs& a, int b, double2* X, double2* G,
                                              const double2* Es, double* od, double* sred,
                                              double& trace, int jr = 0, int js = 1) {
    const int tid = threadIdx.x;
    const int L = a.L;
    constexpr int LP = 4 * NRB;
    const int ld = LP + 1;
    cp_async_wait<0>();   // Sigma_hat staged by the caller (stage_emp), if in SMEM
    __syncthreads();
    PROBE(7);
    const double2* Eg = a.emp_cov + (size_t)b * L * L;   // used when Es == nullptr
    auto Ev = [&](int i, int c) -> double2 {
        return Es ? Es[i * ld + c] : __ldg(Eg + (size_t)i * L + c);
    };
    // (jr, js): this CTA forms the column tiles j = jr (mod js) of G and A only
    // (factor_cluster_t splits the products over the CTAs of a cluster)
    trace = 0.0;
    if (a.record_objective && jr == 0) {
        double s = 0.0;
        for (int e = tid; e < L * L; e += NTH) {
            const int i = e / L, j = e - i * L;
            const double2 pv = X[i * ld + j], ev = Ev(j, i);
            s = fma(pv.x, ev.x, fma(-pv.y, ev.y, s));
        }
        trace = block_sum(s, sred);
    }
    // ---- G = Sigma_hat P and A = P G on DMMA ----------------------------------
    // Complex products in the real 2x2 expansion, first real column of each
    // complex column only: C^[2l+p][m] = sum_{kc,q} A^[2l+p][2kc+q] Bc[2kc+q][m]
    // with A^ = [[re,-im],[im,re]] and Bc[2kc+q][m] = component q of B(kc,m),
    // so C^[2l+p][m] = component p of (A B)(l,m).  Tile = 8 real rows (4
    // complex rows, ri) x 8 complex columns (cj), k-step = 2 complex columns.
    // A warp owns a row tile and keeps one accumulator chain per column tile
    // (the A fragment is shared), reading A^ from Sigma_hat (L2) or P (SMEM)
    // and Bc from SMEM.
    {
        constexpr int NCJ = (LP + 7) / 8;
        constexpr int NKS = LP / 2;
        constexpr int NWF = NTH / 32;
        const int lane = tid & 31, warp = tid >> 5;
        const int r8 = lane >> 2, c4 = lane & 3;
        const int p = r8 & 1, q = c4 & 1;
        const unsigned long long sg = (p == 0 && q == 1) ? 0x8000000000000000ull : 0ull;
        const double* Xd = reinterpret_cast<const double*>(X);
        double* Gd = reinterpret_cast<double*>(G);
        // G = Sigma_hat P, all tiles
        for (int ri = warp; ri < NRB; ri += NWF) {
            const int l = 4 * ri + (r8 >> 1);
            double acc[NCJ][2];
#pragma unroll
            for (int j = 0; j < NCJ; ++j) acc[j][0] = acc[j][1] = 0.0;
            const double* erow = Es ? reinterpret_cast<const double*>(Es + (size_t)l * ld)
                                    : reinterpret_cast<const double*>(Eg + (size_t)l * L);
#pragma unroll 4
            for (int ks = 0; ks < NKS; ++ks) {
                const int kc = 2 * ks + (c4 >> 1);
                const double av = (l < L && kc < L) ? xsign(erow[2 * kc + (p ^ q)], sg) : 0.0;
                const double* brow = Xd + 2 * (kc * ld) + q;
#pragma unroll
                for (int j = 0; j < NCJ; ++j) {
                    if (js == 1 || j % js == jr) {
                        const int m = 8 * j + r8;
                        const double bv = (m < LP) ? brow[2 * m] : 0.0;
                        dmma(acc[j], av, bv);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < NCJ; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = 8 * j + 2 * c4 + h;
                    if (m < LP && (js == 1 || j % js == jr)) Gd[2 * (l * ld + m) + p] = acc[j][h];
                }
        }
        __syncthreads();
        // A = P G, lower tiles only (column tiles cj with 8 cj <= 4 ri + 3), and
        // the fragment pack: entry (l, m), m <= 4 ri + 3, gets P'/A' = 2x the
        // lower values, the real diagonal, zero above the diagonal
        PROBE(8);
        const double* Gc = reinterpret_cast<const double*>(G);
        for (int t = warp; t < NRB; t += NWF) {
            const int ri = NRB - 1 - t;             // longest rows first
            const int ncj = (4 * ri + 3) / 8 + 1;
            const int l = 4 * ri + (r8 >> 1);
            double acc[NCJ][2];
#pragma unroll
            for (int j = 0; j < NCJ; ++j) acc[j][0] = acc[j][1] = 0.0;
            const double* prow = Xd + 2 * (l * ld);
#pragma unroll 4
            for (int ks = 0; ks < NKS; ++ks) {
                const int kc = 2 * ks + (c4 >> 1);
                const double av = xsign(prow[2 * kc + (p ^ q)], sg);
                const double* brow = Gc + 2 * (kc * ld) + q;
#pragma unroll
                for (int j = 0; j < NCJ; ++j) {
                    if (j < ncj && (js == 1 || j % js == jr)) {
                        const int m = 8 * j + r8;
                        const double bv = (m < LP) ? brow[2 * m] : 0.0;
                        dmma(acc[j], av, bv);
                    }
                }
            }
            const int i4 = l >> 2;
#pragma unroll
            for (int j = 0; j < NCJ; ++j) {
                if (j < ncj && (js == 1 || j % js == jr)) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int m = 8 * j + 2 * c4 + h;
                        if (m <= 4 * ri + 3) {
                            const double f = (m < l) ? 2.0 : ((m == l && p == 0) ? 1.0 : 0.0);
                            const double pv = f * Xd[2 * (l * ld + m) + p];
                            const double avv = f * acc[j][h];
                            const int blk = i4 * (i4 + 1) + (m >> 1);
                            const int ent = (l & 3) * 2 + (m & 1);
                            double2* o = reinterpret_cast<double2*>(od) + (size_t)blk * FRAG_SLOTS + 3 * ent;
                            if (p == 0) {
                                o[0] = make_double2(pv, avv);
                            } else {
                                o[1] = make_double2(pv, avv);
                                o[2] = make_double2(-pv, -avv);
                            }
                        }
                    }
                }
            }
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// factor_pass: X holds Sigma (L x L Hermitian, row stride ld = LP + 1) on
// entry.  Hermitian sweep-operator Gauss-Jordan on the lower triangle only:
// sweeping pivot k maps a_kk -> -1/d, a_ik, a_kj -> a/d, a_ij -> a_ij -
// c_i conj(c_j) / d with c = column k, so the matrix stays exactly Hermitian
// and the sweep over all pivots yields -Sigma^-1 (same pivots as LDL^H /
// Cholesky: log|Sigma| = sum log d).  Each thread owns whole 2x2 blocks of
// the lower triangle (registers); the pivot column is staged in SMEM by its
// owners (ping-pong, one barrier per pivot).  Then trace(P Sigma_hat) when the
// objective is recorded, G = Sigma_hat P (all 2x2 blocks), A = P G (lower
// blocks only, P Hermitian), and the P'/A' fragments written to od (SMEM or
// global).  Returns false (uniformly) when a pivot is not positive.  Ends
// synchronised.
// ---------------------------------------------------------------------------
template <int NRB, int NTH>
__device__ __forceinline__ bool factor_pass(const FacArgs& a, const Geo& geo, int b, double2* X,
                                            double2* G, double2* cbuf, double2* /*unused*/,
                                            const double2* Es, double* od, double* sred,
                                            double& frob, double& logdet, double& trace,
                                            int cs = 1, int* cflag = nullptr) {
    using F = TF<NRB, NTH>;
    const int tid = threadIdx.x;
    const int L = a.L;
    constexpr int LP = F::LP;
    const int ld = LP + 1;
    if (cs == 1) {   // (the cluster kernel sums the squares while it assembles Sigma)
        double s = 0.0;
        for (int e = tid; e < L * L; e += NTH) {
            const int i = e / L, j = e - i * L;
            const double2 v = X[i * ld + j];
            s = fma(v.x, v.x, fma(v.y, v.y, s));
        }
        frob = sqrt(block_sum(s, sred));
    }
    PROBE(4);
#if PSCA_DSWEEP
    {
        const bool ok = dmma_sweep<NRB, NTH>(X, ld, L, a.record_objective, logdet);
        PROBE(5);
        if (!ok) {
            __syncthreads();
            return false;
        }
    }
#else
    // ---- lower 2x2 blocks of this thread ---------------------------------------
    int bi[F::SL], bj[F::SL];
    double2 v[F::SL][2][2];
#pragma unroll
    for (int u = 0; u < F::SL; ++u) {
        const int t = tid + NTH * u;
        if (t < F::NLB) lower_block(t, bi[u], bj[u]); else { bi[u] = -1; bj[u] = 0; }
#pragma unroll
        for (int di = 0; di < 2; ++di)
#pragma unroll
            for (int dj = 0; dj < 2; ++dj) {
                const int i = 2 * bi[u] + di, j = 2 * bj[u] + dj;
                v[u][di][dj] = (bi[u] >= 0 && i < L && j < L && i >= j) ? X[i * ld + j]
                                                                       : make_double2(0.0, 0.0);
                // odd L: the padding pivot L is an identity row (no effect on
                // the L x L part, log 1 = 0), so pivots pair up as 2x2 blocks
                if ((L & 1) && i == L && j == L) v[u][di][dj] = make_double2(1.0, 0.0);
            }
    }
#if PSCA_BLOCK_SWEEP && PSCA_USWEEP
    // ---- 2x2 block pivots K = {k, k+1} (k even), pivot-column products shared.
    // Staged per step (ping-pong): the two columns of K for every row with the
    // K entries zeroed (cs0, cs1), and K itself (kv: a = a_kk, b = a_k+1,k,
    // c = a_k+1,k+1).  With M = K^-1 and C_j = (a_jk, a_j,k+1):
    //   phase U  thread j < LP forms U_j = M conj(C_j) once per column into
    //            SMEM (ub0 / ub1; X is free during the sweep) -- 12 FP64
    //            operations per column instead of 24 per owned 2x2 block;
    //   phase V  every owned block is updated a_ij -= C_i U_j (8 DFMA per
    //            entry); the K rows become U_j, the K columns conj(U_i), the
    //            K block -M; the next pivot block's columns are staged.
    // The pivots are those of the scalar sweep (a, then c - |b|^2 / a), so
    // PD-ness and log|Sigma| are unchanged.  Two barriers per step.
    __shared__ double kv[2][4];
    __shared__ double msh[4];
    double2* ub0 = X;
    double2* ub1 = X + LP;
    {
        double2* cs0 = cbuf;
        double2* cs1 = cbuf + LP;
        for (int e = tid; e < LP; e += NTH) {
            cs0[e] = (e < L && e >= 2) ? X[e * ld] : make_double2(0.0, 0.0);
            cs1[e] = (e < L && e >= 2) ? X[e * ld + 1] : make_double2(0.0, 0.0);
        }
        if (tid == 0) {
            kv[0][0] = X[0].x;
            const double2 bb = (L > 1) ? X[ld] : make_double2(0.0, 0.0);
            kv[0][1] = bb.x;
            kv[0][2] = bb.y;
            kv[0][3] = (L > 1) ? X[ld + 1].x : 1.0;
        }
    }
    __syncthreads();   // X (Sigma) is in registers now; ub0 / ub1 may reuse it
    logdet = 0.0;
    bool ok = true;
    const bool want_logdet = a.record_objective;
    const int LE = (L + 1) & ~1;
    for (int k = 0; k < LE; k += 2) {
        const int ph = (k >> 1) & 1;
        const double2* c0 = cbuf + ph * 2 * LP;
        const double2* c1 = c0 + LP;
        double2* n0 = cbuf + (ph ^ 1) * 2 * LP;
        double2* n1 = n0 + LP;
        if (k == 10) PROBE(10);
        const double ka = kv[ph][0], kbr = kv[ph][1], kbi = kv[ph][2], kc = kv[ph][3];
        // M = K^-1 = adj(K) / det(K), det = a c - |b|^2 = a d1; K is PD iff
        // a > 0 and det > 0 (uniform: every thread reads the same kv)
        const double det = fma(ka, kc, -fma(kbr, kbr, kbi * kbi));
        if (!(ka > 0.0) || !(det > 0.0)) {
            ok = false;
            break;
        }
        if (want_logdet) logdet += log(det);
        if (k == 10) PROBE(11);
        if (tid < LP) {
            const double dinv = __drcp_rn(det);
            const double m00 = kc * dinv;
            const double m11 = ka * dinv;
            const double2 m10 = make_double2(-kbr * dinv, -kbi * dinv);
            const double2 m01 = make_double2(m10.x, -m10.y);
            const double2 pp = c0[tid], qq = c1[tid];
            ub0[tid] = make_double2(fma(m01.x, qq.x, fma(m01.y, qq.y, m00 * pp.x)),
                                    fma(m01.y, qq.x, fma(-m01.x, qq.y, -m00 * pp.y)));
            ub1[tid] = make_double2(fma(m11, qq.x, fma(m10.x, pp.x, m10.y * pp.y)),
                                    fma(-m11, qq.y, fma(m10.y, pp.x, -m10.x * pp.y)));
            if (tid == 0) {
                msh[0] = m00;
                msh[1] = m11;
                msh[2] = m10.x;
                msh[3] = m10.y;
            }
        }
        if (k == 10) PROBE(12);
        __syncthreads();
        if (k == 10) PROBE(13);
        const int kb = k >> 1;
#pragma unroll
        for (int u = 0; u < F::SL; ++u) {
            if (bi[u] < 0) continue;
            const int i0 = 2 * bi[u], j0 = 2 * bj[u];
            if (bi[u] == kb && bj[u] == kb) {
                v[u][0][0] = make_double2(-msh[0], 0.0);
                v[u][1][0] = make_double2(-msh[2], -msh[3]);
                v[u][1][1] = make_double2(-msh[1], 0.0);
            } else if (bj[u] == kb) {
                // rows i not in K, columns K: (a_ik, a_ik+1) <- C_i M = conj(U_i)
#pragma unroll
                for (int di = 0; di < 2; ++di) {
                    const double2 x0 = ub0[i0 + di], x1 = ub1[i0 + di];
                    v[u][di][0] = make_double2(x0.x, -x0.y);
                    v[u][di][1] = make_double2(x1.x, -x1.y);
                }
            } else if (bi[u] == kb) {
                // rows K, columns j < k: (a_kj, a_k+1,j) <- M conj(C_j) = U_j
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    v[u][0][dj] = ub0[j0 + dj];
                    v[u][1][dj] = ub1[j0 + dj];
                }
            } else {
                double2 ua[2], ubv[2];
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    ua[dj] = ub0[j0 + dj];
                    ubv[dj] = ub1[j0 + dj];
                }
#if PSCA_PROBE
                if (k == 10 && u == 0) PROBE(20);
                if (k == 10 && u == 0 && ua[0].x + ubv[1].y != 1.2345e300) PROBE(21);
#endif
#pragma unroll
                for (int di = 0; di < 2; ++di) {
                    const double2 pp = c0[i0 + di], qq = c1[i0 + di];   // C_i
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj) {
                        const double2 o = v[u][di][dj];
                        double nx = fma(-pp.x, ua[dj].x, fma(pp.y, ua[dj].y, o.x));
                        double ny = fma(-pp.x, ua[dj].y, fma(-pp.y, ua[dj].x, o.y));
                        nx = fma(-qq.x, ubv[dj].x, fma(qq.y, ubv[dj].y, nx));
                        ny = fma(-qq.x, ubv[dj].y, fma(-qq.y, ubv[dj].x, ny));
                        v[u][di][dj] = make_double2(nx, ny);
                    }
                }
#if PSCA_PROBE
                if (k == 10 && u == 0 && v[u][0][0].x + v[u][1][1].y != 1.2345e300) PROBE(22);
#endif
            }
#if PSCA_PROBE
            if (k == 10 && u == 0) PROBE(23);
#endif
            // stage K' = {k+2, k+3}: its columns for every row, K' zeroed
            if (bi[u] == kb + 1 && bj[u] == kb + 1) {
                kv[ph ^ 1][0] = v[u][0][0].x;
                kv[ph ^ 1][1] = v[u][1][0].x;
                kv[ph ^ 1][2] = v[u][1][0].y;
                kv[ph ^ 1][3] = v[u][1][1].x;
#pragma unroll
                for (int di = 0; di < 2; ++di) {
                    n0[i0 + di] = make_double2(0.0, 0.0);
                    n1[i0 + di] = make_double2(0.0, 0.0);
                }
            } else if (bj[u] == kb + 1) {
#pragma unroll
                for (int di = 0; di < 2; ++di) {
                    n0[i0 + di] = v[u][di][0];
                    n1[i0 + di] = v[u][di][1];
                }
            } else if (bi[u] == kb + 1) {
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    n0[j0 + dj] = make_double2(v[u][0][dj].x, -v[u][0][dj].y);
                    n1[j0 + dj] = make_double2(v[u][1][dj].x, -v[u][1][dj].y);
                }
            }
        }
        if (k == 10) PROBE(14);
        __syncthreads();
        if (k == 10) PROBE(15);
    }
#elif PSCA_BLOCK_SWEEP
    // ---- 2x2 block pivots K = {k, k+1} (k even): one barrier per two pivots.
    // Staged per step (ping-pong): the two columns of K for every row with the
    // K entries zeroed (cs0, cs1), and K itself (kv: a = a_kk, b = a_k+1,k,
    // c = a_k+1,k+1).  The sweep of K: a_ij -= C_i M C_j^H (i, j not in K,
    // M = K^-1, C_i = (a_ik, a_i,k+1)), rows / columns of K -> M-scaled,
    // a_KK -> -M; the pivots are those of the scalar sweep (a, then
    // c - |b|^2 / a), so PD-ness and log|Sigma| are unchanged.
    __shared__ double kv[2][4];
    {
        double2* cs0 = cbuf;
        double2* cs1 = cbuf + LP;
        for (int e = tid; e < LP; e += NTH) {
            cs0[e] = (e < L && e >= 2) ? X[e * ld] : make_double2(0.0, 0.0);
            cs1[e] = (e < L && e >= 2) ? X[e * ld + 1] : make_double2(0.0, 0.0);
        }
        if (tid == 0) {
            kv[0][0] = X[0].x;
            const double2 bb = (L > 1) ? X[ld] : make_double2(0.0, 0.0);
            kv[0][1] = bb.x;
            kv[0][2] = bb.y;
            kv[0][3] = (L > 1) ? X[ld + 1].x : 1.0;
        }
    }
    __syncthreads();
    logdet = 0.0;
    bool ok = true;
    const bool want_logdet = a.record_objective;
    const int LE = (L + 1) & ~1;
    for (int k = 0; k < LE; k += 2) {
        const int ph = (k >> 1) & 1;
        const double2* c0 = cbuf + ph * 2 * LP;
        const double2* c1 = c0 + LP;
        double2* n0 = cbuf + (ph ^ 1) * 2 * LP;
        double2* n1 = n0 + LP;
        const double ka = kv[ph][0], kbr = kv[ph][1], kbi = kv[ph][2], kc = kv[ph][3];
        if (!(ka > 0.0)) {
            ok = false;
            break;
        }
#if PSCA_ADJ_INV
        // M = K^-1 = adj(K) / det(K), det = a c - |b|^2 = a d1 (d1 = the
        // second scalar-sweep pivot): one reciprocal per step instead of two
        // dependent ones; K is PD iff a > 0 and det > 0
        const double det = fma(ka, kc, -fma(kbr, kbr, kbi * kbi));
        if (!(det > 0.0)) {
            ok = false;
            break;
        }
        if (want_logdet) logdet += log(det);
        const double dinv = __drcp_rn(det);
        const double m00 = kc * dinv;
        const double m11 = ka * dinv;
        const double2 m10 = make_double2(-kbr * dinv, -kbi * dinv);
        const double2 m01 = make_double2(m10.x, -m10.y);
#else
        const double ainv = __drcp_rn(ka);
        const double d1 = kc - (kbr * kbr + kbi * kbi) * ainv;
        if (!(d1 > 0.0)) {
            ok = false;
            break;
        }
        if (want_logdet) logdet += log(ka) + log(d1);
        const double d1inv = __drcp_rn(d1);
        // M = K^-1 = [[1/a + |b|^2/(a^2 d1), -conj(b)/(a d1)], [-b/(a d1), 1/d1]]
        const double m00 = fma((kbr * kbr + kbi * kbi) * ainv * ainv, d1inv, ainv);
        const double m11 = d1inv;
        const double2 m10 = make_double2(-kbr * ainv * d1inv, -kbi * ainv * d1inv);
        const double2 m01 = make_double2(m10.x, -m10.y);
#endif
        const int kb = k >> 1;
#pragma unroll
        for (int u = 0; u < F::SL; ++u) {
            if (bi[u] < 0) continue;
            const int i0 = 2 * bi[u], j0 = 2 * bj[u];
            double2 ua[2], ub[2];   // U_j = M conj(C_j) for the block's columns
#pragma unroll
            for (int dj = 0; dj < 2; ++dj) {
                const double2 p = c0[j0 + dj], q = c1[j0 + dj];   // C_j = (p, q)
                // conj(p), conj(q)
                ua[dj] = make_double2(fma(m01.x, q.x, fma(m01.y, q.y, m00 * p.x)),
                                      fma(m01.y, q.x, fma(-m01.x, q.y, -m00 * p.y)));
                ub[dj] = make_double2(fma(m11, q.x, fma(m10.x, p.x, m10.y * p.y)),
                                      fma(-m11, q.y, fma(m10.y, p.x, -m10.x * p.y)));
            }
#pragma unroll
            for (int di = 0; di < 2; ++di) {
                const double2 p = c0[i0 + di], q = c1[i0 + di];   // C_i = (p, q)
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    const double2 o = v[u][di][dj];
                    // a_ij - (p ua + q ub)
                    double nx = fma(-p.x, ua[dj].x, fma(p.y, ua[dj].y, o.x));
                    double ny = fma(-p.x, ua[dj].y, fma(-p.y, ua[dj].x, o.y));
                    nx = fma(-q.x, ub[dj].x, fma(q.y, ub[dj].y, nx));
                    ny = fma(-q.x, ub[dj].y, fma(-q.y, ub[dj].x, ny));
                    v[u][di][dj] = make_double2(nx, ny);
                }
            }
            if (bi[u] == kb || bj[u] == kb || bi[u] == kb + 1 || bj[u] == kb + 1) {
                if (bi[u] == kb && bj[u] == kb) {
                    v[u][0][0] = make_double2(-m00, 0.0);
                    v[u][1][0] = make_double2(-m10.x, -m10.y);
                    v[u][1][1] = make_double2(-m11, 0.0);
                } else if (bj[u] == kb) {
                    // rows i not in K, columns K: (a_ik, a_ik+1) <- (a_ik, a_ik+1) M
#pragma unroll
                    for (int di = 0; di < 2; ++di) {
                        const double2 x0 = v[u][di][0], x1 = v[u][di][1];
                        v[u][di][0] = make_double2(fma(x1.x, m10.x, fma(-x1.y, m10.y, x0.x * m00)),
                                                   fma(x1.x, m10.y, fma(x1.y, m10.x, x0.y * m00)));
                        v[u][di][1] = make_double2(fma(x0.x, m01.x, fma(-x0.y, m01.y, x1.x * m11)),
                                                   fma(x0.x, m01.y, fma(x0.y, m01.x, x1.y * m11)));
                    }
                } else if (bi[u] == kb) {
                    // rows K, columns j not in K: (a_kj, a_k+1,j) <- M (a_kj, a_k+1,j)
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj) {
                        const double2 x0 = v[u][0][dj], x1 = v[u][1][dj];
                        v[u][0][dj] = make_double2(fma(m01.x, x1.x, fma(-m01.y, x1.y, m00 * x0.x)),
                                                   fma(m01.x, x1.y, fma(m01.y, x1.x, m00 * x0.y)));
                        v[u][1][dj] = make_double2(fma(m10.x, x0.x, fma(-m10.y, x0.y, m11 * x1.x)),
                                                   fma(m10.x, x0.y, fma(m10.y, x0.x, m11 * x1.y)));
                    }
                }
                // stage K' = {k+2, k+3}: its columns for every row, K' zeroed
                if (bi[u] == kb + 1 && bj[u] == kb + 1) {
                    kv[ph ^ 1][0] = v[u][0][0].x;
                    kv[ph ^ 1][1] = v[u][1][0].x;
                    kv[ph ^ 1][2] = v[u][1][0].y;
                    kv[ph ^ 1][3] = v[u][1][1].x;
#pragma unroll
                    for (int di = 0; di < 2; ++di) {
                        n0[i0 + di] = make_double2(0.0, 0.0);
                        n1[i0 + di] = make_double2(0.0, 0.0);
                    }
                } else if (bj[u] == kb + 1) {
#pragma unroll
                    for (int di = 0; di < 2; ++di) {
                        n0[i0 + di] = v[u][di][0];
                        n1[i0 + di] = v[u][di][1];
                    }
                } else if (bi[u] == kb + 1) {
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj) {
                        n0[j0 + dj] = make_double2(v[u][0][dj].x, -v[u][0][dj].y);
                        n1[j0 + dj] = make_double2(v[u][1][dj].x, -v[u][1][dj].y);
                    }
                }
            }
        }
        __syncthreads();
    }
#else
    for (int e = tid; e < 2 * LP; e += NTH)
        cbuf[e] = (e < L) ? X[e * ld] : make_double2(0.0, 0.0);   // padding stays zero
    __syncthreads();

    logdet = 0.0;
    bool ok = true;
    const bool want_logdet = a.record_objective;
    for (int k = 0; k < L; ++k) {
        const double2* cb = cbuf + (k & 1) * LP;
        double2* cn = cbuf + ((k + 1) & 1) * LP;
        const double d = cb[k].x;
        if (!(d > 0.0)) {
            ok = false;
            break;
        }
        if (want_logdet) logdet += log(d);
        const double dinv = __drcp_rn(d);
#pragma unroll
        for (int u = 0; u < F::SL; ++u) {
            if (bi[u] < 0) continue;
            const int i0 = 2 * bi[u], j0 = 2 * bj[u];
            const double2 ci[2] = {cb[i0], cb[i0 + 1]};
            const double2 cj[2] = {cb[j0], cb[j0 + 1]};
            // u_j = conj(c_j) / d (also the new row-k entries a_kj / d, since
            // a_kj = conj(c_j)); w_i = c_i / d (new column-k entries), only for
            // the blocks holding column k
            double2 uj[2], wi[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
            for (int dj = 0; dj < 2; ++dj) uj[dj] = make_double2(cj[dj].x * dinv, -cj[dj].y * dinv);
            if (j0 == (k & ~1)) {
#pragma unroll
                for (int di = 0; di < 2; ++di) wi[di] = make_double2(ci[di].x * dinv, ci[di].y * dinv);
            }
#pragma unroll
            for (int di = 0; di < 2; ++di)
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    const int i = i0 + di, j = j0 + dj;
                    const double2 o = v[u][di][dj];
                    // a_ij - c_i u_j
                    double nx = fma(-ci[di].x, uj[dj].x, fma(ci[di].y, uj[dj].y, o.x));
                    double ny = fma(-ci[di].x, uj[dj].y, fma(-ci[di].y, uj[dj].x, o.y));
                    nx = (i == k) ? uj[dj].x : nx;
                    ny = (i == k) ? uj[dj].y : ny;
                    nx = (j == k) ? wi[di].x : nx;
                    ny = (j == k) ? wi[di].y : ny;
                    nx = (i == k && j == k) ? -dinv : nx;
                    ny = (i == k && j == k) ? 0.0 : ny;
                    if (i < j) { nx = 0.0; ny = 0.0; }
                    v[u][di][dj] = make_double2(nx, ny);
                    // stage column k+1 of the swept matrix
                    if (j == k + 1 && i >= j && i < L) cn[i] = make_double2(nx, ny);
                    if (i == k + 1 && j < i) cn[j] = make_double2(nx, -ny);
                }
        }
        __syncthreads();
    }
#endif
    PROBE(5);
    // packed lower triangle of P for the cluster's other CTAs: the instance's
    // chunk partials are dead once Sigma is assembled (LP (LP + 1) / 2 entries
    // fit in the lower tiles of one chunk)
    double2* pshare = const_cast<double2*>(a.sig_part) + (size_t)b * a.n_chunks * geo.NBLK * 32;
    if (cs > 1) {
        // cluster factor (factor_cluster_t): the sweep's outcome goes to every
        // CTA's flag before the cluster barrier they wait at
        namespace cg = cooperative_groups;
        auto cl = cg::this_cluster();
        if (tid < cs) *cl.map_shared_rank(cflag, tid) = ok ? 1 : 2;
        if (!ok) {
            cl.sync();
            return false;
        }
    }
    if (!ok) {
        __syncthreads();
        return false;
    }
    // ---- P = -(swept): full Hermitian into X (of every CTA of the cluster) -----
#pragma unroll
    for (int u = 0; u < F::SL; ++u) {
        if (bi[u] < 0) continue;
#pragma unroll
        for (int di = 0; di < 2; ++di)
#pragma unroll
            for (int dj = 0; dj < 2; ++dj) {
                const int i = 2 * bi[u] + di, j = 2 * bj[u] + dj;
                if (i >= j) {
                    const double2 pv = (i < L && j < L) ? make_double2(-v[u][di][dj].x, -v[u][di][dj].y)
                                                        : make_double2(0.0, 0.0);
                    const double2 dv = (i == j) ? make_double2(pv.x, 0.0) : pv;
                    const double2 mv = make_double2(pv.x, -pv.y);
                    X[i * ld + j] = dv;
                    if (i != j) X[j * ld + i] = mv;
                    // the other CTAs of the cluster fetch P through L2 (DSMEM
                    // moves ~20 B / cycle out of one SM: 8.8 us for 7 copies)
                    if (cs > 1) pshare[i * (i + 1) / 2 + j] = dv;
                }
            }
    }
#endif  // PSCA_DSWEEP
    PROBE(6);
    if (cs > 1) cooperative_groups::this_cluster().sync();
    products_pass<NRB, NTH>(a, b, X, G, Es, od, sred, trace, 0, cs);
    return true;
}

// ===========================================================================
// two-kernel path
// ===========================================================================
template <int NRB>
__global__ void __launch_bounds__(NT, (NRB <= 12) ? 2 : 1) column_kernel_t(ColArgs a) {
    using G = TG<NRB>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.y;
    const int chunk = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t bN = (size_t)b * a.N;
    const int n_begin = chunk * a.chunk_cols;
    const int n_end = min(a.N, n_begin + a.chunk_cols);

    if (a.status[b] != PSCA_RUNNING) {
        for (int n = n_begin + tid; n < n_end; n += NT) a.x_next[bN + n] = a.x_cur[bN + n];
        return;
    }
    double2* S0 = reinterpret_cast<double2*>(smem_raw);
    double2* S1 = S0 + G::LP8 * NCT;
    double2* WS = S1 + G::LP8 * NCT;
    double2* SP = WS + G::LP8 * G::WCAP;
    double2* FRs = SP + G::LP8 * G::WCAP;                            // [NB][24] if staged
    constexpr int FS = G::FR_SLOTS;
    double* qr_s = reinterpret_cast<double*>(FRs + (G::FR_SMEM ? G::NB * FS : 0));
    const double2* FR;
    if (G::FR_SMEM) {   // stage the instance's P'/A' fragments (one cp.async group)
        const double2* src = a.frags + (size_t)b * G::NB * FRAG_SLOTS;
        for (int e = tid; e < G::NB * FS; e += NT) {
            // compact layout: slot 2 ent + var of a block <- 3 ent + var (var < 2)
            const int se = (FS == FRAG_SLOTS) ? e : (e >> 4) * FRAG_SLOTS + 3 * ((e & 15) >> 1) + (e & 1);
            cp_async16(FRs + e, src + se, 16);
        }
        cp_async_commit();
        FR = FRs;
    } else {
        FR = a.frags + (size_t)b * G::NB * FRAG_SLOTS;
    }
    int slot[G::MAXBW];
    int nbw;
    rebuild_slots<NRB>(slot, nbw);
    if (a.dbg_delay_ns > 0 && (b & 1)) __nanosleep(a.dbg_delay_ns);
    double acc[G::MAXBW][2];
    double dx2, minq;
    col_pass<NRB, FS>(a, b, a.k, a.x_cur + bN, a.x_next + bN, n_begin, n_end, S0, S1, WS, SP,
                      FR, qr_s, acc, slot, nbw, dx2, minq);

    {
        double2* sp = a.sig_part + ((size_t)b * a.n_chunks + chunk) * G::NBLK * 32;
        int idx = 0, t2 = 0;
        for (int i = 0; i < NRB; ++i) {
            const int jmax = (4 * i + 3) / 8;
            for (int j = 0; j <= jmax; ++j, ++idx) {
                if ((idx % NWARP) == warp) {
#pragma unroll
                    for (int u = 0; u < G::MAXBW; ++u)
                        if (u == t2) sp[(size_t)idx * 32 + lane] = make_double2(acc[u][0], acc[u][1]);
                    ++t2;
                }
            }
        }
    }
    reduce_pass_partials(dx2, minq);
    if (tid == 0) {
        double* rp = a.red_part + ((size_t)b * a.n_chunks + chunk) * 4;
        rp[0] = dx2;
        rp[1] = minq;
        rp[2] = 0.0;
        rp[3] = 0.0;
    }
}

template <int NRB, int NTH>
__global__ void __launch_bounds__(NTH, (NTH == 128 && NRB <= 10) ? 4 : 1) factor_solve_t(FacArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double sred[SRED];
    __shared__ int s_flag;
    const Geo geo = make_geo(a.L, a.nrb);
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int LP = geo.LP;
    const int ld = LP + 1;
    if (a.status[b] != PSCA_RUNNING) return;
    PROBE(0);
    if (a.k_new > 0) {
        if (fac_finalize(a, b, &s_flag)) return;
    }
    PROBE(1);
    const double prior_value = fac_prior_terms(a, b, sred);
    PROBE(2);
    double2* sm = reinterpret_cast<double2*>(smem_raw);
    double2* rowb = sm;             // [2][LP] pivot column ping-pong
    double2* colb = sm + 2 * LP;    // (unused)
    double2* X = sm + 4 * LP;       // [LP][ld]
    double2* G = X + (size_t)LP * ld;
    // Sigma_hat is staged (cp.async, landing during the assembly and the sweep)
    // into the G buffer itself: G = Sigma_hat P is computed by row tiles, and
    // the warp that writes G's row tile ri is the only reader of Sigma_hat's
    // rows of that tile, so the product can overwrite its operand in place
    // (no extra SMEM, so 4 CTAs per SM still fit)
    const double2* Es = G;
    stage_emp(a, b, G, ld);
    if (NTH >= 512) assemble_sigma_seq(a, geo, b, X, ld, a.k_new == 0);
    else assemble_sigma<8, 1>(a, geo, b, X, ld, a.k_new == 0);
    PROBE(3);
    double frob, logdet, trace;
    double* od = reinterpret_cast<double*>(a.frags + (size_t)b * geo.NB * FRAG_SLOTS);
    if (!factor_pass<NRB, NTH>(a, geo, b, X, G, rowb, colb, Es, od, sred, frob, logdet,
                                  trace)) {
        if (tid == 0) {
            a.status[b] = PSCA_CHOL_FAIL;
            if (a.cond_est) a.cond_est[b] = INFINITY;
        }
        return;
    }
    PROBE(9);
    if (tid == 0) {
        double* in = a.inst + (size_t)b * 4;
        in[0] = frob;
        in[1] = logdet;
        in[2] = trace;
        in[3] = prior_value;
    }
}

// ---------------------------------------------------------------------------
// factor_cluster_t: the factor stage of a lone instance (or a handful) spread
// over a cluster of FCS CTAs -- the latency-bound small-batch case (BASELINE
// c0: B = 1), where one CTA spent 4.4 us summing the 32 chunk partials
// (0.9 MB through one SM) and 7.2 us in the two DMMA products:
//   * every CTA sums the chunk partials of the fragment blocks
//     blk = rank (mod FCS) and stores its Sigma entries into CTA 0's X through
//     distributed shared memory;                          [cluster barrier]
//   * CTA 0 alone runs the pivot sweep (a dependent chain), then stores
//     P = Sigma^-1 into every CTA's X and the sweep's outcome into every
//     CTA's flag;                                          [cluster barrier]
//   * CTA r forms the column tiles j = r (mod FCS) of G = Sigma_hat P and
//     A = P G (both are column-local given all of P and Sigma_hat) and packs
//     their P'/A' fragments.
// CTA 0 finalises the previous iteration before a first cluster barrier and
// the others read its outcome (status[b]) after it, so all CTAs stop or go on
// together.  No CTA touches another's shared memory after the last barrier,
// and CTA 0 (the only remote-store target before it) outlives all of them.
// ---------------------------------------------------------------------------
constexpr int FCS = 8;
template <int NRB>
__global__ void __cluster_dims__(FCS, 1, 1) __launch_bounds__(512, 1) factor_cluster_t(FacArgs a) {
    namespace cg = cooperative_groups;
    constexpr int NTH = 512;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double sred[SRED];
    __shared__ int s_flag;
    __shared__ int s_cflag;
    __shared__ double s_ssq[FCS];
    auto cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const Geo geo = make_geo(a.L, a.nrb);
    const int b = blockIdx.x / FCS;
    const int tid = threadIdx.x;
    const int LP = geo.LP;
    const int ld = LP + 1;
    // CTA 0 finalises the previous iteration (the only writer of status[b] in
    // this launch) before the first barrier; the others read the outcome after it
    bool stop = false;
#if PSCA_PROBE
    const long long probe_t0 = clock64();
#endif
    if (rank == 0) {
        if (a.status[b] != PSCA_RUNNING) stop = true;
        else if (a.k_new > 0) stop = fac_finalize(a, b, &s_flag);
    }
    if (tid == 0) s_cflag = 0;
    cl.sync();   // every CTA of the cluster is running: remote stores may start
    if (rank != 0) stop = a.status[b] != PSCA_RUNNING || (a.k_new > 0 && a.k_new >= a.T);
    if (stop) return;
#if PSCA_PROBE
    if (blockIdx.x == PSCA_PROBE_BLOCK && tid == 0) g_probe[0] = probe_t0;
#endif
    PROBE(1);
    double2* sm = reinterpret_cast<double2*>(smem_raw);
    double2* rowb = sm;
    double2* colb = sm + 2 * LP;
    double2* X = sm + 4 * LP;
    double2* G = X + (size_t)LP * ld;
    const double2* Es = G;
    // (CTA 0's copy is issued later, by the warps that own no block of the sweep)
    if (rank > 0 && rank < (LP + 7) / 8) stage_emp(a, b, G, ld);   // the CTAs that own a column tile
    double prior_value = 0.0;
    if (rank == 0) prior_value = fac_prior_terms(a, b, sred);
    PROBE(2);
    double ssq;
    assemble_sigma_seq(a, geo, b, cl.map_shared_rank(X, 0), ld, a.k_new == 0, rank, FCS, &ssq);
    ssq = block_sum(ssq, sred);
    if (tid == 0) *cl.map_shared_rank(&s_ssq[rank], 0) = ssq;
    cl.sync();
    double frob = 0.0, logdet = 0.0, trace = 0.0;
    if (rank == 0) {
        double t = 0.0;
#pragma unroll
        for (int r = 0; r < FCS; ++r) t += s_ssq[r];   // rank order: deterministic
        frob = sqrt(t);
    }
    PROBE(3);
    PROBE(4);
    double* od = reinterpret_cast<double*>(a.frags + (size_t)b * geo.NB * FRAG_SLOTS);
    if (rank == 0) {
        stage_emp(a, b, G, ld, NTH / 2, NTH / 2);   // lands during the sweep
        if (!factor_pass<NRB, NTH>(a, geo, b, X, G, rowb, colb, Es, od, sred, frob, logdet, trace,
                                    FCS, &s_cflag)) {
            if (tid == 0) {
                a.status[b] = PSCA_CHOL_FAIL;
                if (a.cond_est) a.cond_est[b] = INFINITY;
            }
            return;
        }
        PROBE(9);
        if (tid == 0) {
            double* in = a.inst + (size_t)b * 4;
            in[0] = frob;
            in[1] = logdet;
            in[2] = trace;
            in[3] = prior_value;
        }
    } else {
        cl.sync();
        if (s_cflag != 1) return;
        if (rank < (LP + 7) / 8) {   // CTAs that own a column tile
            const double2* pshare = a.sig_part + (size_t)b * a.n_chunks * geo.NBLK * 32;
            for (int e = tid; e < LP * (LP + 1) / 2; e += NTH) {
                int i, j;
                lower_block(e, i, j);   // (i, j), i >= j, of packed entry e
                const double2 pv = __ldcg(pshare + e);
                X[i * ld + j] = pv;
                if (i != j) X[j * ld + i] = make_double2(pv.x, -pv.y);
            }
            products_pass<NRB, NTH>(a, b, X, G, Es, od, sred, trace, rank, FCS);
        }
    }
}

// ===========================================================================
// persistent path: one launch for the whole solve
// ===========================================================================
template <int NRB>
__global__ void __launch_bounds__(NT, 2) psca_persistent_t(ColArgs ca, FacArgs fa, int* counter) {
    using G = TG<NRB>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double sred[SRED];
    __shared__ double s_inst[4];
    __shared__ int s_b, s_flag;
    const Geo geo = make_geo(fa.L, fa.nrb);
    const int tid = threadIdx.x;
    const int L = fa.L, LP = geo.LP, ld = LP + 1;

    double2* FR = reinterpret_cast<double2*>(smem_raw);                    // [NB][24]
    unsigned char* U = smem_raw + G::F_BYTES;                                 // union
    double2* S0 = reinterpret_cast<double2*>(U);
    double2* S1 = S0 + G::LP8 * NCT;
    double2* WS = S1 + G::LP8 * NCT;
    double2* SP = WS + G::LP8 * G::WCAP;
    double2* rowb = reinterpret_cast<double2*>(U);
    double2* colb = rowb + 2 * LP;
    double2* X = rowb + 4 * LP;
    double2* Gm = X + (size_t)LP * ld;
    const double2* Es = nullptr;   // Sigma_hat read through L1/L2 (keeps 2 CTAs / SM)
    double* qr_s = reinterpret_cast<double*>(U + G::UNION);

    int slot[G::MAXBW];
    int nbw;
    rebuild_slots<NRB>(slot, nbw);

    for (;;) {
        if (tid == 0) s_b = atomicAdd(counter, 1);
        __syncthreads();
        const int b = s_b;
        if (b >= fa.B) break;
        const size_t bN = (size_t)b * fa.N;
        double* xc = const_cast<double*>(fa.x_cur) + bN;   // x_out slice (zeroed by psca_solve)
        double* xn = fa.x_next + bN;  // workspace slice
        double* final_x = xc;

        // ---- iterate 0: prior terms at x = 0, Sigma_0 = sigma^2 I, D_0 = 0 --
        if (fa.incremental) {
            double2* D = fa.dmat + (size_t)b * dmat_stride(geo, L);
            for (int e = tid; e < L * L; e += NT) D[e] = make_double2(0.0, 0.0);
        }
        double pv = fac_prior_terms_at(fa, b, xc, sred);
        {
            const double s2 = fa.noise[b];
            for (int e = tid; e < L * L; e += NT) {
                const int i = e / L, j = e - i * L;
                X[i * ld + j] = make_double2(i == j ? s2 : 0.0, 0.0);
            }
            __syncthreads();
        }
        double frob, logdet, trace;
        bool ok = factor_pass<NRB, NT>(fa, geo, b, X, Gm, rowb, colb, Es, reinterpret_cast<double*>(FR),
                                  sred, frob, logdet, trace);
        if (!ok) {
            if (tid == 0) {
                fa.status[b] = PSCA_CHOL_FAIL;
                if (fa.cond_est) fa.cond_est[b] = INFINITY;
            }
        } else {
            if (tid == 0) {
                s_inst[0] = frob; s_inst[1] = logdet; s_inst[2] = trace; s_inst[3] = pv;
            }
            for (int k = 0; k < fa.T; ++k) {
                double acc[G::MAXBW][2];
                double dx2, minq;
                col_pass<NRB>(ca, b, k, xc, xn, 0, fa.N, S0, S1, WS, SP, FR, qr_s, acc, slot,
                              nbw, dx2, minq);
                reduce_pass_partials(dx2, minq);
                if (tid == 0) s_flag = fac_finalize_core(fa, b, k, dx2, minq, s_inst);
                __syncthreads();
                const int flag = s_flag;
                if (flag == PSCA_QFLOOR) { final_x = xc; break; }
                final_x = xn;
                if (flag == PSCA_CONVERGED || k + 1 == fa.T) break;
                // ---- factorisation at x_{k+1} ---------------------------------
                pv = fac_prior_terms_at(fa, b, xn, sred);
                acc_to_sigma<NRB>(acc, slot, nbw, X, ld, L,
                                  fa.incremental ? reinterpret_cast<double*>(fa.dmat + (size_t)b * dmat_stride(geo, L))
                                                 : nullptr,
                                  __dsub_rn(1.0, fa.steps[(size_t)b * fa.steps_stride + k]));
                finish_sigma(X, ld, L, fa.noise[b]);
                ok = factor_pass<NRB, NT>(fa, geo, b, X, Gm, rowb, colb, Es, reinterpret_cast<double*>(FR),
                                     sred, frob, logdet, trace);
                if (!ok) {
                    if (tid == 0) {
                        fa.status[b] = PSCA_CHOL_FAIL;
                        if (fa.cond_est) fa.cond_est[b] = INFINITY;
                    }
                    break;
                }
                if (tid == 0) {
                    s_inst[0] = frob; s_inst[1] = logdet; s_inst[2] = trace; s_inst[3] = pv;
                }
                double* tsw = xc; xc = xn; xn = tsw;
            }
        }
        if (final_x != fa.x_cur + bN) {
            double* out = const_cast<double*>(fa.x_cur) + bN;
            for (int n = tid; n < fa.N; n += NT) out[n] = final_x[n];
        }
        __syncthreads();
    }
}
