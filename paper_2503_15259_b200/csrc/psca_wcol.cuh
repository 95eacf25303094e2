// psca_wcol.cuh -- warp-streamed column kernel (sm_100a), compiled shapes NRB <= 20
// (L <= 80).  Included by psca.cu after psca_fast.cuh (uses TG, rebuild_slots,
// ColArgs, dmma, the fragment layout and the packed rebuild layout).
//
// One CTA owns one (instance, column chunk) like column_kernel_t, but the
// column pass (estimators.py:262-276 for the chunk's devices) runs without
// CTA barriers: every warp streams its own 8-column blocks (w, w + 8, ...)
//
//   B fragments   the block's pilot columns go straight from HBM into
//                 registers (2 NRB doubles per lane, one LDG.64 per k-step:
//                 two 128-byte lines per instruction); the next block's
//                 fragments are loaded while this block computes
//   quad forms    q_n = s^H P s and r_n = s^H A s on DMMA over the lower
//                 block triangle (A = P' / A' fragments from SMEM, the
//                 same packed layout the factor kernel writes); the whole
//                 triangle per warp, so q and r are complete in the warp
//   epilogue      S at the C-fragment positions comes from the B registers
//                 by shuffles; the 8 column updates (gradient, surrogate,
//                 clip, relaxed step) run on lanes 0..7
//   moving list   columns with a non-zero rebuild weight are appended to the
//                 warp's list in SMEM (column, weight)
//
// and only the covariance rebuild, Sigma += S diag(v) S^H over the listed
// columns (covlinalg.py:55; incremental weights), is a CTA
// phase at the end of the pass: the listed columns are gathered 16 at a time
// from HBM / L2 into the packed WS / SP layout and summed on DMMA into the
// same C fragments column_kernel_t produces, so the factor kernel is shared.
// Reduction orders are fixed (rows in descending block order, the shuffle
// tree, lists in warp order), so reruns are bit-identical.

#ifndef PSCA_WCOL_MINB
#define PSCA_WCOL_MINB 2
#endif
#ifndef PSCA_WCOL_KDESC
#define PSCA_WCOL_KDESC 0
#endif
// B fragments of the next block through a per-warp cp.async landing zone in
// SMEM (aliased on the rebuild gather buffers, which are idle during the pass)
// instead of LDG into registers: NRB <= 10 only (the zone needs 2 gather buffers)
#ifndef PSCA_WCOL_STAGEB
#define PSCA_WCOL_STAGEB 1
#endif
// blocks per update group (4: 32 columns per update; 1: the update after every block)
#ifndef PSCA_WCOL_UGRP
#define PSCA_WCOL_UGRP 4
#endif
// rebuild gather buffers (2: the next round's loads overlap this round's DMMAs)
#ifndef PSCA_WCOL_GBUF
#define PSCA_WCOL_GBUF 2
#endif

// CTAs per SM for L <= 20: with ten B fragments per lane the kernel fits 85
// registers, and a third resident CTA covers the relatively longer per-block
// epilogue (c3 L = 20: column launch 0.728 -> 0.703 ms per 2048 instances,
// 26.46 -> 25.72 ms per 30 iterations; four CTAs at 64 registers: 0.819)
#ifndef PSCA_WCOL_MINB_SMALL
#define PSCA_WCOL_MINB_SMALL 3
#endif

template <int NRB>
struct TWC {
    using G = TG<NRB>;
    static constexpr int NKK = 2 * NRB;   // k-steps = B fragments per lane per block
    static constexpr size_t FR_BYTES = (size_t)G::NB * FRAG_SLOTS * 16;
    static constexpr size_t W_BYTES = (size_t)G::LP8 * G::WCAP * 16;
    static constexpr size_t W_BYTES_ = W_BYTES;
    static constexpr int GPT = (G::LP8 * G::WCAP + NT - 1) / NT;   // gather elements per thread
    // L > 40: the 24-slot fragments of the whole triangle fill most of SMEM
    // (L = 80: 161 KB), so one gather buffer and one CTA (up to 255 registers)
    // per SM
    static constexpr int NGB = NRB <= 10 ? PSCA_WCOL_GBUF : 1;
    // per-warp landing zone [LP rows][8 columns] double2; fits the gather buffers
    static constexpr bool STAGEB =
        PSCA_WCOL_STAGEB && NRB <= 10 &&
        (size_t)NWARP * G::LP * 8 * 16 <= (size_t)2 * (NRB <= 10 ? PSCA_WCOL_GBUF : 1) * W_BYTES_;
    static constexpr int MINB = NRB <= 5 ? PSCA_WCOL_MINB_SMALL : (NRB <= 10 ? PSCA_WCOL_MINB : 1);
    // dynamic SMEM: fragments, NGB x (WS, SP), per-warp partials, then the lists
    static constexpr size_t FIXED = FR_BYTES + 2 * NGB * W_BYTES + (size_t)NWARP * 2 * 8 + 16 * 8;
    static __host__ __device__ constexpr int list_cap(int chunk_cols) {
        return ((chunk_cols / 8 + NWARP - 1) / NWARP) * 8;
    }
    static __host__ __device__ constexpr size_t smem(int chunk_cols) {
        return FIXED + (size_t)NWARP * list_cap(chunk_cols) * 12;
    }
};

// B fragments of one 8-column block: lane (r8, c4) holds component (c4 & 1)
// of S[2 kk + (c4 >> 1)][col0 + r8] for k-step kk
template <int NRB>
__device__ __forceinline__ void wc_load_b(double (&bf)[2 * NRB], const double* __restrict__ sbd,
                                          size_t row2, int L, bool ok, int c4) {
#pragma unroll
    for (int kk = 0; kk < 2 * NRB; ++kk) {
        const int m = 2 * kk + (c4 >> 1);
        bf[kk] = (ok && m < L) ? __ldg(sbd + (size_t)m * row2) : 0.0;
    }
}

// Quadratic forms of one block; on return every lane holds, for the columns
// 2 c4 and 2 c4 + 1 of the block, q (qa) and r (ra) summed over all rows.
// Rows run in descending order, so after row i only k-steps < 2i are still
// needed: its two B fragments are then reloaded with the next block's
// (nsrc != nullptr), which keeps one fragment set per lane in registers.
// With zsrc != nullptr the next block's fragments come from the warp's SMEM
// landing zone (lane-resolved pointer: component c4 & 1 of row c4 >> 1, column
// r8; row stride 16 doubles) after its cp.async group has landed.
template <int NRB, class Mid>
__device__ __forceinline__ void wc_quad(double (&bf)[2 * NRB], const double2* __restrict__ FRl,
                                        double (&qa)[2], double (&ra)[2], int r8, int c4,
                                        const double* __restrict__ nsrc, size_t row2, int L,
                                        bool nok, Mid&& mid, const double* zsrc = nullptr) {
    qa[0] = qa[1] = ra[0] = ra[1] = 0.0;
    const int src0 = 8 * c4 + (r8 & 3);
    const bool hi = (r8 >> 2) != 0;
#pragma unroll
    for (int i = NRB - 1; i >= 0; --i) {
        double tc[2] = {0.0, 0.0}, uc[2] = {0.0, 0.0};
        const double2* f = FRl + i * (i + 1) * FRAG_SLOTS;
        // PSCA_WCOL_KDESC=1 walks the k-steps in descending order, so the fragments
        // reloaded last are consumed last: measured equal (the other warps already
        // cover that load), off
#if PSCA_WCOL_KDESC
#pragma unroll
        for (int kk = 2 * (i + 1) - 1; kk >= 0; --kk) {
#else
#pragma unroll
        for (int kk = 0; kk < 2 * (i + 1); ++kk) {
#endif
            const double2 pa = f[kk * FRAG_SLOTS];
            dmma(tc, pa.x, bf[kk]);
            dmma(uc, pa.y, bf[kk]);
        }
        // the previous block's column updates run under the longest chain
        if (i == NRB - 1) mid();
        // S[4i + (r8 >> 1)][2 c4 + h], component r8 & 1, lives in B fragment
        // 2i + (r8 >> 2) of lane (2 c4 + h) * 4 + (r8 & 3)
#ifdef PSCA_DBG_NO_EPI   // probe (results invalid): no shuffles for the epilogue operands
        const double a0 = bf[2 * i], a1 = bf[2 * i + 1], b0 = a0, b1 = a1;
#else
        const double a0 = __shfl_sync(0xffffffffu, bf[2 * i], src0);
        const double a1 = __shfl_sync(0xffffffffu, bf[2 * i + 1], src0);
        const double b0 = __shfl_sync(0xffffffffu, bf[2 * i], src0 + 4);
        const double b1 = __shfl_sync(0xffffffffu, bf[2 * i + 1], src0 + 4);
#endif
#ifdef PSCA_DBG_NO_BLOAD   // probe (results invalid): B fragments never reloaded
        if (false) {
#else
        if (zsrc) {
            if (i == NRB - 1) {   // the zone was filled during the previous block
                cp_async_wait<0>();
                __syncwarp();
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) bf[2 * i + u] = zsrc[(2 * (2 * i + u)) * 16];
        } else if (nsrc) {
#endif
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int m = 2 * (2 * i + u) + (c4 >> 1);
                bf[2 * i + u] = (nok && m < L) ? __ldg(nsrc + (size_t)m * row2) : 0.0;
            }
        }
        const double s0 = hi ? a1 : a0;
        const double s1 = hi ? b1 : b0;
        qa[0] = fma(s0, tc[0], qa[0]);
        qa[1] = fma(s1, tc[1], qa[1]);
        ra[0] = fma(s0, uc[0], ra[0]);
        ra[1] = fma(s1, uc[1], ra[1]);
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        qa[0] += __shfl_xor_sync(0xffffffffu, qa[0], o);
        qa[1] += __shfl_xor_sync(0xffffffffu, qa[1], o);
        ra[0] += __shfl_xor_sync(0xffffffffu, ra[0], o);
        ra[1] += __shfl_xor_sync(0xffffffffu, ra[1], o);
    }
}

// rebuild over packed slots [0, cnt) of WS / SP into this warp's C blocks
// (same operand layout as col_pass's rebuild)
template <int NRB>
__device__ __forceinline__ void wc_rebuild(const double2* WS, const double2* SP, int cnt,
                                           double (&acc)[TG<NRB>::MAXBW][2],
                                           const int (&slot)[TG<NRB>::MAXBW], int nbw, int lane) {
    using G = TG<NRB>;
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1, cpr = c4 >> 1;
    const int sa = r8 >> 1, sbb = r8 & 3;
    int wa_lane[4], b_lane[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        wa_lane[h] = 4 * (h ^ sa) + 2 * cpr + (p ^ q);
        b_lane[h] = 4 * (h ^ sbb) + 2 * cpr + q;
    }
    const unsigned long long wsgn = (p & q) ? 0x8000000000000000ull : 0ull;
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
}

// CTA-phase stagger (experiment, PSCA_DBG_DELAY_NS): the second CTA to arrive on
// an SM in a launch starts that much later, so the co-resident pair's start /
// rebuild phases fall into each other's column pass
__device__ int g_sm_slot[1024];

template <int NRB>
__global__ void __launch_bounds__(NT, TWC<NRB>::MINB) column_kernel_w(ColArgs a) {
    using G = TG<NRB>;
    using W = TWC<NRB>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int b = blockIdx.y;
    const int chunk = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r8 = lane >> 2, c4 = lane & 3;
    const size_t bN = (size_t)b * a.N;
    const int n_begin = chunk * a.chunk_cols;
    const int n_end = min(a.N, n_begin + a.chunk_cols);

    if (a.status[b] != PSCA_RUNNING) {
        for (int n = n_begin + tid; n < n_end; n += NT) a.x_next[bN + n] = a.x_cur[bN + n];
        return;
    }
    double2* FR = reinterpret_cast<double2*>(smem_raw);
    double2* WS = FR + G::NB * FRAG_SLOTS;
    // WS / SP gather buffers: [WS0 SP0 (WS1 SP1)], LP8 x WCAP slots each
    double* wpart = reinterpret_cast<double*>(WS + 2 * W::NGB * G::LP8 * G::WCAP);   // [NWARP][2]
    int* s_cnt = reinterpret_cast<int*>(wpart + 2 * NWARP);               // [NWARP + 1] prefix
    const int cap = W::list_cap(a.chunk_cols);
    double* lv = wpart + 2 * NWARP + 16;                                  // [NWARP][cap]
    int* lcol = reinterpret_cast<int*>(lv + (size_t)NWARP * cap);          // [NWARP][cap]

    // the instance's P'/A' fragments: one TMA bulk copy, completion on s_bar
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ int s_slot;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        if (a.dbg_delay_ns > 0) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            s_slot = atomicAdd(&g_sm_slot[smid], 1);
        }
    }
    __syncthreads();
    if (a.dbg_delay_ns > 0 && s_slot == 1) {
        if (tid == 0) {
            unsigned long long t0, t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            do {
                __nanosleep(2000);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            } while (t1 - t0 < (unsigned long long)a.dbg_delay_ns);
        }
        __syncthreads();
    }
    if (tid == 0)
        bulk_g2s(FR, a.frags + (size_t)b * G::NB * FRAG_SLOTS, (unsigned)W::FR_BYTES, &s_bar);

    const bool known = (a.kind == PSCA_ML_K || a.kind == PSCA_MAP_K);
    const double hi = known ? 1.0 : (a.kind == PSCA_ML_UD ? INFINITY : a.eff.g_high);
    const int k = a.k;
    const double rho = a.steps[(size_t)b * a.steps_stride + k];
    const double omr = __dsub_rn(1.0, rho);
    const double* x_cur = a.x_cur + bN;
    double* x_next = a.x_next + bN;
    const double2* sb = a.pilots + (size_t)b * a.L * a.N;
    const double* sbd = reinterpret_cast<const double*>(sb);
    const size_t row2 = (size_t)2 * a.N;   // doubles per pilot row
    const double2* FRl = FR + frag_lane_slot(lane);

    const int nblk = (n_end - n_begin + 7) >> 3;
    double p_dx2 = 0.0, p_minq = INFINITY;
    int cnt = 0;
    double* my_v = lv + (size_t)warp * cap;
    int* my_c = lcol + (size_t)warp * cap;

    double bf[2 * NRB];
    auto bsrc = [&](int jb) {
        const int n = n_begin + 8 * jb + r8;
        return sbd + 2 * (size_t)n + (c4 & 1);
    };
    int jb = warp;
    // landing zone of this warp: [LP rows][8 columns] double2 (rows >= L and
    // columns >= n_end zero-filled by the copy)
    double* zone = reinterpret_cast<double*>(WS) + (size_t)warp * G::LP * 16;
    const double* zlane = zone + ((c4 >> 1) * 8 + r8) * 2 + (c4 & 1);
    auto zone_issue = [&](int jblk) {
#pragma unroll
        for (int u = 0; u < (G::LP * 8 + 31) / 32; ++u) {
            const int e = lane + 32 * u;
            const int row = e >> 3, c = e & 7;
            const int n = n_begin + 8 * jblk + c;
            if (e < G::LP * 8) {
                const bool ok = row < a.L && n < n_end;
                cp_async16(zone + e * 2, ok ? sb + (size_t)row * a.N + n : sb, ok ? 16 : 0);
            }
        }
        cp_async_commit();
    };
    if (W::STAGEB) {
        if (jb < nblk) {
            zone_issue(jb);
            cp_async_wait<0>();
            __syncwarp();
#pragma unroll
            for (int kk = 0; kk < 2 * NRB; ++kk) bf[kk] = zlane[(2 * kk) * 16];
            __syncwarp();
            if (jb + NWARP < nblk) zone_issue(jb + NWARP);
        }
    } else if (jb < nblk) {
        wc_load_b<NRB>(bf, bsrc(jb), row2, a.L, n_begin + 8 * jb + r8 < n_end, c4);
    }
    mbar_wait(&s_bar, 0);   // fragments staged
    // per-device update (estimators.py:272-276) of one block's columns, lane
    // j < 8 -> column j; appends the moving columns to the warp's list and
    // asks L2 to keep their pilot lines for the rebuild gather
    auto update = [&](double q, double r, double x, double g, double pg, int ncol, bool cvalid) {
        double v = 0.0;
        if (cvalid) {
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
            x_next[ncol] = xn;
            if (a.iterates) a.iterates[((size_t)b * (a.T + 1) + k + 1) * a.N + ncol] = xn;
            const double dx = __dsub_rn(xn, x);
            p_dx2 = fma(dx, dx, p_dx2);
            p_minq = (q < p_minq) ? q : p_minq;
        }
        unsigned mv = __ballot_sync(0xffffffffu, v != 0.0);
        if (v != 0.0) {
            const int pos = cnt + __popc(mv & ((1u << lane) - 1u));
            my_v[pos] = v;
            my_c[pos] = ncol;
        }
        cnt += __popc(mv);
        while (mv) {
            const int j = __ffs(mv) - 1;
            mv &= mv - 1;
            const int cj = __shfl_sync(0xffffffffu, ncol, j);
            for (int m = lane; m < a.L; m += 32)
                asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(sb + (size_t)m * a.N + cj));
        }
    };

    // software pipeline: the updates of four blocks (32 columns, one per lane:
    // lanes 8 s .. 8 s + 7 hold the s-th block of the group) run together inside
    // the quad forms of the following block, after its longest row's DMMAs are
    // issued -- every FP64 instruction of the update then works on 32 columns
    // instead of 8 (the FP64 pipe is the one the DMMAs use)
    bool pend = false;
    double pq = 0.0, pr = 0.0, px = 0.0, pgn = 1.0, ppg = 0.0;
    int pcol = 0;
    bool pvalid = false;
    const int grp = lane >> 3;
    int slot_in_group = 0;
    for (; jb < nblk; jb += NWARP) {
        const int jn = jb + NWARP;
        {   // L2 prefetch of the block after the next one (40 lines of 128 B)
            const int jp = jb + 2 * NWARP;
            if (jp < nblk) {
                const char* base = reinterpret_cast<const char*>(sb + n_begin + 8 * jp);
                for (int m = lane; m < a.L; m += 32)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)m * a.N * 16));
            }
        }
        // the block's 8 columns go to the lanes of group slot_in_group
        const bool mine = grp == slot_in_group;
        const int ncol = n_begin + 8 * jb + (lane & 7);
        const bool cvalid = mine && ncol < n_end;
        double x = 0.0, g = 1.0, pg = 0.0;
        if (cvalid) {
            x = x_cur[ncol];
            if (known) g = a.gains[bN + ncol];
            if (a.kind == PSCA_MAP_UR || (a.kind == PSCA_MAP_K && a.pairwise))
                pg = a.pgrad[bN + ncol];
            else if (a.kind == PSCA_MAP_K) pg = a.prior_lin[ncol];
        }
        double qa[2], ra[2];
        wc_quad<NRB>(bf, FRl, qa, ra, r8, c4,
                     (!W::STAGEB && jn < nblk) ? bsrc(jn) : nullptr, row2, a.L,
                     n_begin + 8 * jn + r8 < n_end, [&] {
                         if (pend) {
                             update(pq, pr, px, pgn, ppg, pcol, pvalid);
                             pend = false;
                             pvalid = false;
                         }
                     }, (W::STAGEB && jn < nblk) ? zlane : nullptr);
        if (W::STAGEB && jn < nblk) {
            // every lane has read the zone: refill it with the block after the next
            __syncwarp();
            if (jn + NWARP < nblk) zone_issue(jn + NWARP);
        }
        // lane l takes column j = l & 7 = 2 c4' + h from lane c4' = j >> 1
        const int srcl = (lane >> 1) & 3;
        const double q0 = __shfl_sync(0xffffffffu, qa[0], srcl);
        const double q1 = __shfl_sync(0xffffffffu, qa[1], srcl);
        const double r0 = __shfl_sync(0xffffffffu, ra[0], srcl);
        const double r1 = __shfl_sync(0xffffffffu, ra[1], srcl);
        if (mine) {
            pq = (lane & 1) ? q1 : q0;
            pr = (lane & 1) ? r1 : r0;
            px = x; pgn = g; ppg = pg; pcol = ncol; pvalid = cvalid;
        }
        if (++slot_in_group == PSCA_WCOL_UGRP) {
            slot_in_group = 0;
            pend = true;
        }
    }
    if (pend || slot_in_group > 0) update(pq, pr, px, pgn, ppg, pcol, pvalid);

    // ---- per-warp partials of (sum dx^2, min q), list counts -----------------
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        p_dx2 += __shfl_xor_sync(0xffffffffu, p_dx2, o);
        const double mq = __shfl_xor_sync(0xffffffffu, p_minq, o);
        p_minq = (mq < p_minq) ? mq : p_minq;
    }
    if (lane == 0) {
        wpart[2 * warp] = p_dx2;
        wpart[2 * warp + 1] = p_minq;
        s_cnt[warp + 1] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
        s_cnt[0] = 0;
        double dx2 = 0.0, minq = INFINITY;
        for (int w = 0; w < NWARP; ++w) {
            s_cnt[w + 1] += s_cnt[w];
            dx2 += wpart[2 * w];
            minq = (wpart[2 * w + 1] < minq) ? wpart[2 * w + 1] : minq;
        }
        double* rp = a.red_part + ((size_t)b * a.n_chunks + chunk) * 4;
        rp[0] = dx2;
        rp[1] = minq;
        rp[2] = 0.0;
        rp[3] = 0.0;
    }
    __syncthreads();

    // ---- short lists: the factor warp of this instance sums the increment ----
    // (fac_sweep_w gathers the listed columns itself, psca_facw.cuh); the list
    // goes out in warp order, the order the CTA rebuild below would use
    if (a.mov_cnt) {
        const int total_mov = s_cnt[NWARP];
        if (total_mov <= a.mov_cap) {
            const size_t o = (size_t)b * a.mov_cap + s_cnt[warp];
            for (int i = lane; i < cnt; i += 32) {
                a.mov_col[o + i] = my_c[i];
                a.mov_w[o + i] = my_v[i];
            }
            if (tid == 0) a.mov_cnt[b] = total_mov;
            return;
        }
        if (tid == 0) a.mov_cnt[b] = -1;
    }

    // ---- rebuild over the moving columns, 16 per round -----------------------
    int slot[G::MAXBW];
    int nbw;
    rebuild_slots<NRB>(slot, nbw);
    double acc[G::MAXBW][2];
#pragma unroll
    for (int t = 0; t < G::MAXBW; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int total = s_cnt[NWARP];
    // gather of round r (16 listed columns x LP8 rows) into registers, then
    // into WS / SP buffer r & 1; the next round's loads are in flight while
    // the current round's DMMAs run
    double2 gs[W::GPT];
    double gv[W::GPT];
    auto gather_load = [&](int base) {
        const int rc = min(total - base, G::WCAP);
#pragma unroll
        for (int u = 0; u < W::GPT; ++u) {
            const int e = tid + u * NT;
            const int l = e / G::WCAP, s = e - l * G::WCAP;
            gs[u] = make_double2(0.0, 0.0);
            gv[u] = 0.0;
            if (e < G::LP8 * G::WCAP && s < rc && l < a.L) {
                const int gi = base + s;
                int w = 0;
                while (gi >= s_cnt[w + 1]) ++w;
                const int li = gi - s_cnt[w];
                gv[u] = lv[(size_t)w * cap + li];
                gs[u] = __ldg(sb + (size_t)l * a.N + lcol[(size_t)w * cap + li]);
            }
        }
    };
    auto gather_store = [&](int buf) {
        double2* WSb = WS + (size_t)buf * 2 * G::LP8 * G::WCAP;
        double2* SPb = WSb + G::LP8 * G::WCAP;
#pragma unroll
        for (int u = 0; u < W::GPT; ++u) {
            const int e = tid + u * NT;
            if (e < G::LP8 * G::WCAP) {
                const int l = e / G::WCAP, s = e - l * G::WCAP;
                const int o = l * G::WCAP + (s ^ (2 * (l & 3)));
                WSb[o] = make_double2(gv[u] * gs[u].x, gv[u] * gs[u].y);
                SPb[o] = gs[u];
            }
        }
    };
    const int rounds = (total + G::WCAP - 1) / G::WCAP;
    if (W::NGB == 1) {
        for (int r = 0; r < rounds; ++r) {
            gather_load(r * G::WCAP);
            gather_store(0);
            __syncthreads();
            wc_rebuild<NRB>(WS, WS + G::LP8 * G::WCAP, min(total - r * G::WCAP, G::WCAP), acc, slot,
                            nbw, lane);
            __syncthreads();
        }
    } else {
    if (rounds > 0) {
        gather_load(0);
        gather_store(0);
    }
    __syncthreads();
    for (int r = 0; r < rounds; ++r) {
        if (r + 1 < rounds) gather_load((r + 1) * G::WCAP);
        const double2* WSb = WS + (size_t)(r & 1) * 2 * G::LP8 * G::WCAP;
        wc_rebuild<NRB>(WSb, WSb + G::LP8 * G::WCAP, min(total - r * G::WCAP, G::WCAP), acc, slot,
                        nbw, lane);
        if (r + 1 < rounds) gather_store((r + 1) & 1);
        __syncthreads();
    }
    }
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
}
