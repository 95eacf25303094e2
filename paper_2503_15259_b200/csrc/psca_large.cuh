// psca_large.cuh -- large pilot length (80 < L <= 256) PSCA path, host-driven
// step loop (included by psca.cu inside its anonymous namespace).
//
// At L = 256 (BASELINE config 4: N = 100,000, one instance) neither the P'/A'
// fragments (1.6 MB) nor a useful S tile fit in SMEM, so the column pass is a
// GEMM-tiled pipeline:
//   quad_large     output tile = 32 complex rows (8 row blocks, one per warp) x
//                  64 columns; K chunks of 16 complex rows of S and the matching
//                  fragment blocks are cp.async double-buffered; fused epilogue
//                  s^T T over the tile's rows -> per-row-tile partial q, r
//   update_large   per column: q, r = fixed-order sum of the row-tile partials,
//                  the fused per-device update, rebuild weight v, per-CTA
//                  (dx2, min q) reductions
//   rebuild_large  lower C-block tiles (8 row blocks x 8 column blocks) x column
//                  splits; per 32-column chunk the moving columns (v != 0) are
//                  ballot-compacted into SMEM and multiplied on DMMA
//   reduce_large   fixed-order sums of the split partials (the rank-local Sigma
//                  increment, in C-fragment form) and of the (dx2, min q)
//                  partials -> the exchange buffer that multi-GPU column
//                  sharding all-reduces (NCCL) between psca_large_columns and
//                  psca_large_factor
// and the factorisation:
//   finalize_large one thread: q-floor guard, update norm, objective, tol stop
//   assemble_large D_{k+1} = (1 - rho_k) D_k + increment; Sigma = D + sigma^2 I
//   gj_cluster     Hermitian sweep Gauss-Jordan over an 8-CTA thread-block
//                  cluster: lower 2x2 blocks in registers across 8 x 1024
//                  threads, the pivot column broadcast into every CTA's SMEM
//                  through DSMEM, one cluster barrier per pivot
//   gemm_large     G = Sigma_hat P and A = P G (lower 2x2 blocks)
//   pack_large     P'/A' fragments (same layout as the small-L path)

constexpr int QL_NC = 64;    // columns per quad tile
constexpr int QL_KC = 16;    // complex rows per K chunk (8 k-steps)
constexpr int QL_RT = 32;    // complex rows per row tile (8 row blocks)
constexpr int RL_NC = 32;    // columns per rebuild chunk
constexpr int GJ_CL = 8;     // CTAs per GJ cluster
constexpr int GJ_NT = 512;   // threads per GJ CTA

constexpr int FROB_CTAS = 64;   // frob_large partial sums

struct LargeArgs {
    int kind, N, L, LP, NRB, T, n_antennas, record_objective, k;
    double tol, noise;
    const double2* pilots;      // [L][N] (this rank's columns)
    const double* gains;        // [N]
    const double2* emp_cov;     // [L][L]
    const double* steps;        // [T]
    const double* prior_lin;    // [N]
    const double* prior_p;      // [N]
    const double* c1;           // pairwise map-k: [N], CSR c2 (null: independent prior)
    const int* c2_ptr;
    const int* c2_idx;
    const double* c2_val;
    psca_eff_prior eff;
    const double* x_cur;
    double* x_next;
    double* iterates;           // [T+1][N] or null
    double* update_norm;        // [T]
    double* objective;          // [T] or null
    int* status;                // [1]
    int* n_iter;                // [1]
    double* cond_est;           // [1]
    // workspace
    double2* frags;             // [NB][24]
    double* q_part;             // [LP/32][N]
    double* r_part;             // [LP/32][N]
    double* v;                  // [N]
    double* pgrad;              // [N]
    double* red_part;           // [n_red][2]
    int n_red;
    double2* dsig_part;         // [ks][NBLK][32]
    int ks, n_rtiles_lower;
    double2* dsig;              // [NBLK][32]   exchange buffer (all-reduced over ranks)
    double* red;                // [4] exchange: dx2 (sum), prior partial (sum), min q (min)
    double2* dmat;              // [L][L] D
    double2* Xg;                // [LP][LP] Sigma, then P
    double2* Gg;                // [LP][LP]
    double2* Ag;                // [LP][LP]
    double* inst;               // [4] frob, logdet, trace, prior value
    int* flag;                  // [1] finalize decision
    double* frob_part;          // [FROB_CTAS] partial sums of |Sigma_ij|^2
    // moving columns of the iteration, compacted in device order (stable):
    int* mcnt;                  // [n_red + 1] per update block, then the total
    int* mcol_t;                // [n_red][NT] block-local lists (update_large)
    double* mv_t;
    int* mcol;                  // [N] dense list (compact_large)
    double* mv;
};

__device__ __forceinline__ int lblock_base(int i) {   // rebuild C-block index of (i, 0)
    int s = 0;
    for (int t = 0; t < i; ++t) s += (4 * t + 3) / 8 + 1;
    return s;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT, 2) quad_large(LargeArgs a) {
    if (a.flag[0]) return;   // stopped: the step loop may run on without a host check
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* sm = reinterpret_cast<double2*>(smem_raw);
    constexpr int SB = QL_KC * QL_NC;          // S chunk
    constexpr int FB = 8 * 8 * FRAG_SLOTS;     // fragment chunk
    constexpr int STAGE = SB + FB;
    double* qr = reinterpret_cast<double*>(sm + 2 * STAGE);   // [8 warps][64][2]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r8 = lane >> 2, c4 = lane & 3;
    const int rt = blockIdx.y, col0 = blockIdx.x * QL_NC;
    const int i = 8 * rt + warp;              // this warp's row block
    const int nkk = 2 * (i + 1);
    const int nchunks = 2 * rt + 2;
    const int fslot = frag_lane_slot(lane);

    auto stage = [&](int c, double2* buf) {
        double2* Sb = buf;
        double2* Fb = buf + SB;
        for (int e = tid; e < SB; e += NT) {
            const int m = e / QL_NC, n = e % QL_NC;
            const int gm = QL_KC * c + m, col = col0 + n;
            const bool ok = gm < a.L && col < a.N;
            const double2* src = ok ? a.pilots + (size_t)gm * a.N + col : a.pilots;
            cp_async16(Sb + m * QL_NC + (n ^ swz(m)), src, ok ? 16 : 0);
        }
        for (int e = tid; e < FB; e += NT) {
            const int rb = e / (8 * FRAG_SLOTS), rem = e % (8 * FRAG_SLOTS);
            const int kl = rem / FRAG_SLOTS, sl = rem % FRAG_SLOTS;
            const int ib = 8 * rt + rb, kk = 8 * c + kl;
            const bool ok = ib < a.NRB && kk < 2 * (ib + 1);
            const double2* src = ok ? a.frags + ((size_t)ib * (ib + 1) + kk) * FRAG_SLOTS + sl
                                    : a.frags;
            cp_async16(Fb + e, src, ok ? 16 : 0);
        }
        cp_async_commit();
    };

    double T[8][2], U[8][2];
#pragma unroll
    for (int cb = 0; cb < 8; ++cb) T[cb][0] = T[cb][1] = U[cb][0] = U[cb][1] = 0.0;

    stage(0, sm);
    for (int c = 0; c < nchunks; ++c) {
        double2* buf = sm + (c & 1) * STAGE;
        if (c + 1 < nchunks) {
            stage(c + 1, sm + ((c + 1) & 1) * STAGE);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* Sd = reinterpret_cast<const double*>(buf);
        const double2* Fb = buf + SB + warp * 8 * FRAG_SLOTS + fslot;
#pragma unroll
        for (int kl = 0; kl < 8; ++kl) {
            if (8 * c + kl < nkk) {
                const double2 pa = Fb[kl * FRAG_SLOTS];
                const int m = 2 * kl + (c4 >> 1);
#pragma unroll
                for (int cb = 0; cb < 8; ++cb) {
                    const int n = 8 * cb + r8;
                    const double bv = Sd[2 * (m * QL_NC + (n ^ swz(m))) + (c4 & 1)];
                    dmma(T[cb], pa.x, bv);
                    dmma(U[cb], pa.y, bv);
                }
            }
        }
        __syncthreads();
    }
    // ---- epilogue: q += sum_rows S_real * T over this tile's rows ------------
    double2* Se = sm;   // [32][64] rows 32 rt ..
    for (int e = tid; e < QL_RT * QL_NC; e += NT) {
        const int m = e / QL_NC, n = e % QL_NC;
        const int gm = QL_RT * rt + m, col = col0 + n;
        const bool ok = gm < a.L && col < a.N;
        const double2* src = ok ? a.pilots + (size_t)gm * a.N + col : a.pilots;
        cp_async16(Se + m * QL_NC + (n ^ swz(m)), src, ok ? 16 : 0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    {
        const double* Sd = reinterpret_cast<const double*>(Se);
        const int lr = 4 * warp + (r8 >> 1), p = r8 & 1;
#pragma unroll
        for (int cb = 0; cb < 8; ++cb) {
            const int n0 = 8 * cb + 2 * c4;
            const double s0 = Sd[2 * (lr * QL_NC + (n0 ^ swz(lr))) + p];
            const double s1 = Sd[2 * (lr * QL_NC + ((n0 + 1) ^ swz(lr))) + p];
            double q0 = s0 * T[cb][0], q1 = s1 * T[cb][1];
            double r0 = s0 * U[cb][0], r1 = s1 * U[cb][1];
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                q0 += __shfl_xor_sync(0xffffffffu, q0, o);
                q1 += __shfl_xor_sync(0xffffffffu, q1, o);
                r0 += __shfl_xor_sync(0xffffffffu, r0, o);
                r1 += __shfl_xor_sync(0xffffffffu, r1, o);
            }
            if (r8 == 0) {
                double* d = qr + (warp * QL_NC + n0) * 2;
                d[0] = q0; d[1] = r0; d[2] = q1; d[3] = r1;
            }
        }
    }
    __syncthreads();
    if (tid < QL_NC) {
        const int col = col0 + tid;
        if (col < a.N) {
            double q = 0.0, r = 0.0;
            for (int w = 0; w < NWARP; ++w) {
                q += qr[(w * QL_NC + tid) * 2];
                r += qr[(w * QL_NC + tid) * 2 + 1];
            }
            a.q_part[(size_t)rt * a.N + col] = q;
            a.r_part[(size_t)rt * a.N + col] = r;
        }
    }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) update_large(LargeArgs a) {
    if (a.flag[0]) return;   // stopped: the step loop may run on without a host check
    __shared__ double sred[2 * NWARP];
    __shared__ int wcnt[NWARP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = blockIdx.x * NT + tid;
    double vmov = 0.0;
    const bool known = (a.kind == PSCA_ML_K || a.kind == PSCA_MAP_K);
    const double hi = known ? 1.0 : (a.kind == PSCA_ML_UD ? INFINITY : a.eff.g_high);
    const double rho = a.steps[a.k];
    const double omr = __dsub_rn(1.0, rho);
    double dx2 = 0.0, mq = INFINITY;
    if (n < a.N) {
        double q = 0.0, r = 0.0;
        for (int t = 0; t < a.LP / QL_RT; ++t) {
            q += a.q_part[(size_t)t * a.N + n];
            r += a.r_part[(size_t)t * a.N + n];
        }
        const double x = a.x_cur[n];
        const double g = known ? a.gains[n] : 1.0;
        const double diff = __dsub_rn(q, r);
        double grad;
        if (a.kind == PSCA_ML_K) grad = __dmul_rn(g, diff);
        else if (a.kind == PSCA_MAP_K)
            grad = __dadd_rn(__dmul_rn(g, diff), a.c2_ptr ? a.pgrad[n] : a.prior_lin[n]);
        else if (a.kind == PSCA_ML_UD) grad = diff;
        else grad = __dadd_rn(diff, a.pgrad[n]);
        const double gq = known ? __dmul_rn(g, q) : q;
        const double coef = __dmul_rn(gq, gq);
        const double cand = np_clip(__dsub_rn(x, __ddiv_rn(grad, coef)), 0.0, hi);
        const double rc = __dmul_rn(rho, cand);
        const double xn = __dadd_rn(__dmul_rn(omr, x), rc);
        a.x_next[n] = xn;
        if (a.iterates) a.iterates[(size_t)(a.k + 1) * a.N + n] = xn;
        vmov = known ? __dmul_rn(rc, g) : rc;
        a.v[n] = vmov;
        const double d = __dsub_rn(xn, x);
        dx2 = d * d;
        mq = q;
    }
    for (int o = 16; o > 0; o >>= 1) {
        dx2 += __shfl_xor_sync(0xffffffffu, dx2, o);
        const double t = __shfl_xor_sync(0xffffffffu, mq, o);
        mq = (t < mq) ? t : mq;
    }
    // moving columns (non-zero rebuild weight) of this block, in device order
    const unsigned mvm = __ballot_sync(0xffffffffu, vmov != 0.0);
    if (lane == 0) {
        sred[2 * warp] = dx2;
        sred[2 * warp + 1] = mq;
        wcnt[warp] = __popc(mvm);
    }
    __syncthreads();
    {
        int off = 0, tot = 0;
        for (int w = 0; w < NWARP; ++w) {
            if (w < warp) off += wcnt[w];
            tot += wcnt[w];
        }
        if (vmov != 0.0) {
            const size_t o = (size_t)blockIdx.x * NT + off + __popc(mvm & ((1u << lane) - 1u));
            a.mcol_t[o] = n;
            a.mv_t[o] = vmov;
        }
        if (tid == 0) a.mcnt[blockIdx.x] = tot;
    }
    if (tid == 0) {
        double s = 0.0, m = INFINITY;
        for (int w = 0; w < NWARP; ++w) {
            s += sred[2 * w];
            m = (sred[2 * w + 1] < m) ? sred[2 * w + 1] : m;
        }
        a.red_part[2 * blockIdx.x] = s;
        a.red_part[2 * blockIdx.x + 1] = m;
    }
}

// ---------------------------------------------------------------------------
// One CTA: exclusive prefix of the per-block counts (fixed order), then the
// block-local lists concatenated into the dense list the rebuild walks, so its
// chunks of 32 columns are full (with 2.5 % of the devices moving, scanning v
// in device order found one or two columns per chunk).
__global__ void __launch_bounds__(1024) compact_large(LargeArgs a) {
    if (a.flag[0]) return;
    __shared__ int s_off[1025];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int carry = 0;
    for (int b0 = 0; b0 < a.n_red; b0 += 1024) {
        const int nb = min(1024, a.n_red - b0);
        if (warp == 0) {
            for (int c = 0; c < nb; c += 32) {
                const int v = (c + lane < nb) ? a.mcnt[b0 + c + lane] : 0;
                int inc = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += t;
                }
                if (c + lane < nb) s_off[c + lane] = carry + inc - v;
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (lane == 0) s_off[nb] = carry;
        }
        __syncthreads();
        for (int b = warp; b < nb; b += 32) {
            const int o = s_off[b], c = s_off[b + 1] - o;
            const size_t src = (size_t)(b0 + b) * NT;
            for (int i = lane; i < c; i += 32) {
                a.mcol[o + i] = a.mcol_t[src + i];
                a.mv[o + i] = a.mv_t[src + i];
            }
        }
        carry = s_off[nb];
        __syncthreads();
    }
    if (tid == 0) a.mcnt[a.n_red] = carry;
}

// ---------------------------------------------------------------------------
// rebuild: blockIdx.x = lower tile (row tile rt of 8 row blocks, column group
// cg of 8 column blocks, 64 cg <= 32 rt + 31), blockIdx.y = column split
__global__ void __launch_bounds__(NT) rebuild_large(LargeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* WS = reinterpret_cast<double2*>(smem_raw);   // [32 rows][32 slots]
    double2* SP = WS + 32 * RL_NC;                         // [64 rows][32 slots]
    if (a.flag[0]) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r8 = lane >> 2, c4 = lane & 3;
    int rt = 0, cg = 0;
    {
        int t = blockIdx.x;
        for (rt = 0;; ++rt) {
            const int ncg = (32 * rt + 31) / 64 + 1;
            if (t < ncg) { cg = t; break; }
            t -= ncg;
        }
    }
    const int i = 8 * rt + warp;
    // this split's share of the dense moving list, in whole chunks of RL_NC
    const int total = a.mcnt[a.n_red];
    const int nchunk = (total + RL_NC - 1) / RL_NC;
    const int per = ((nchunk + gridDim.y - 1) / gridDim.y) * RL_NC;
    const int c_begin = min(total, (int)blockIdx.y * per), c_end = min(total, c_begin + per);
    double acc[8][2];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) acc[jj][0] = acc[jj][1] = 0.0;
    const int p = r8 & 1, q = c4 & 1, cpr = c4 >> 1;
    const unsigned long long wsgn = (p & q) ? 0x8000000000000000ull : 0ull;
    const int la = 4 * warp + (r8 >> 1);   // local WS row of the A fragment

    for (int c0 = c_begin; c0 < c_end; c0 += RL_NC) {
        const int li = c0 + lane;
        const int col = (li < c_end) ? a.mcol[li] : 0;
        const double v = (li < c_end) ? a.mv[li] : 0.0;
        const unsigned mask = __ballot_sync(0xffffffffu, v != 0.0);
        if (mask == 0u) continue;                          // CTA-uniform (same v)
        const int nnz = __popc(mask);
        const int pos = __popc(mask & ((1u << lane) - 1u));
        __syncthreads();                                   // previous chunk consumed
        for (int r = warp; r < 32; r += NWARP) {
            const int gl = 32 * rt + r;
            const int o = r * RL_NC + (pos ^ (2 * (r & 3)));
            if (v != 0.0) {
                const double2 s = (gl < a.L) ? a.pilots[(size_t)gl * a.N + col] : make_double2(0.0, 0.0);
                WS[o] = make_double2(v * s.x, v * s.y);
            }
            if (lane == 0 && (nnz & 1)) WS[r * RL_NC + (nnz ^ (2 * (r & 3)))] = make_double2(0.0, 0.0);
        }
        for (int r = warp; r < 64; r += NWARP) {
            const int gm = 64 * cg + r;
            const int o = r * RL_NC + (pos ^ (2 * (r & 3)));
            if (v != 0.0)
                SP[o] = (gm < a.L) ? a.pilots[(size_t)gm * a.N + col] : make_double2(0.0, 0.0);
            if (lane == 0 && (nnz & 1)) SP[r * RL_NC + (nnz ^ (2 * (r & 3)))] = make_double2(0.0, 0.0);
        }
        __syncthreads();
        const double* Wd = reinterpret_cast<const double*>(WS);
        const double* Pd = reinterpret_cast<const double*>(SP);
        const int nk2 = (nnz + 1) >> 1;
        for (int k2 = 0; k2 < nk2; ++k2) {
            const int sa = la & 3;
            const int na = (2 * k2 + cpr) ^ (2 * sa);
            const double av = xsign(Wd[2 * (la * RL_NC + na) + (p ^ q)], wsgn);
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int lm = 8 * jj + r8;            // local SP row (m = 64 cg + lm)
                const int nb = (2 * k2 + cpr) ^ (2 * (lm & 3));
                const double bv = Pd[2 * (lm * RL_NC + nb) + q];
                dmma(acc[jj], av, bv);
            }
        }
    }
    // ---- C fragments -> dsig_part[split][block][lane] -------------------------
    const int base = lblock_base(i);
    const int jmax = (4 * i + 3) / 8;
    double2* out = a.dsig_part + (size_t)blockIdx.y * rebuild_block_count(a.NRB) * 32;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const int j = 8 * cg + jj;
        if (i < a.NRB && j <= jmax) out[(size_t)(base + j) * 32 + lane] = make_double2(acc[jj][0], acc[jj][1]);
    }
}

// sums of the split partials -> exchange buffers (fixed orders)
__global__ void __launch_bounds__(NT) reduce_large(LargeArgs a) {
    if (a.flag[0]) return;   // stopped: the step loop may run on without a host check
    const int nblk32 = rebuild_block_count(a.NRB) * 32;
    const int e = blockIdx.x * NT + threadIdx.x;
    if (e < nblk32) {
        double2 s = make_double2(0.0, 0.0);
        for (int sp = 0; sp < a.ks; ++sp) {
            const double2 v = a.dsig_part[(size_t)sp * nblk32 + e];
            s.x += v.x;
            s.y += v.y;
        }
        a.dsig[e] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double s = 0.0, m = INFINITY;
        for (int b = 0; b < a.n_red; ++b) {
            s += a.red_part[2 * b];
            m = (a.red_part[2 * b + 1] < m) ? a.red_part[2 * b + 1] : m;
        }
        a.red[0] = s;   // red[1] (prior partial) is left to prior_large
        a.red[2] = m;
    }
}

// ---------------------------------------------------------------------------
// factorisation
// ---------------------------------------------------------------------------
__global__ void finalize_large(LargeArgs a) {
    // flag: 0 continue, 1 stop (frozen / done)
    const int k = a.k;
    double* in = a.inst;
    {
        double s = 0.0;
        for (int c = 0; c < FROB_CTAS; ++c) s += a.frob_part[c];
        in[0] = sqrt(s);
    }
    int flag = 0;
    if (a.status[0] != PSCA_RUNNING) {
        flag = 1;
    } else if (a.red[2] < 0.5 * a.L / in[0]) {
        a.status[0] = PSCA_QFLOOR;
        a.n_iter[0] = k;
        flag = 1;
    } else {
        const double un = sqrt(a.red[0]);
        a.update_norm[k] = un;
        // the prior penalty at x_k is the all-reduced red[1] (sum over column shards)
        if (a.objective) a.objective[k] = in[1] + in[2] + a.red[1];
        a.n_iter[0] = k + 1;
        if (un < a.tol) {
            a.status[0] = PSCA_CONVERGED;
            flag = 1;
        } else if (k + 1 >= a.T) {
            flag = 1;
        }
    }
    a.flag[0] = flag;
}

// D_{k+1} = (1 - rho) D_k + increment (k >= 0), Sigma = D + sigma^2 I -> Xg
// (a.k = -1: D = 0, Sigma = sigma^2 I)
__global__ void __launch_bounds__(NT) assemble_large(LargeArgs a) {
    if (a.flag[0]) return;
    const int L = a.L, LP = a.LP;
    const int nblk32 = rebuild_block_count(a.NRB) * 32;
    const int e = blockIdx.x * NT + threadIdx.x;
    const double omr = (a.k >= 0) ? __dsub_rn(1.0, a.steps[a.k]) : 0.0;
    double* Dd = reinterpret_cast<double*>(a.dmat);
    double* Xd = reinterpret_cast<double*>(a.Xg);
    if (e < nblk32) {
        const int blk = e >> 5, lane = e & 31;
        int i = 0, base = 0;
        while (base + (4 * i + 3) / 8 + 1 <= blk) { base += (4 * i + 3) / 8 + 1; ++i; }
        const int j = blk - base;
        const double2 s = (a.k >= 0) ? a.dsig[e] : make_double2(0.0, 0.0);
        const int r8 = lane >> 2, c4 = lane & 3;
        const int l = 4 * i + (r8 >> 1), p = r8 & 1;
        const int m0 = 8 * j + 2 * c4;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = m0 + h;
            if (l < L && m <= l) {
                const size_t o = 2 * ((size_t)l * L + m) + p;
                const double val = (a.k >= 0) ? fma(omr, Dd[o], h ? s.y : s.x) : 0.0;
                Dd[o] = val;
                Xd[2 * ((size_t)l * LP + m) + p] = val;
            }
        }
    }
}

__global__ void __launch_bounds__(NT) finish_sigma_large(LargeArgs a) {
    if (a.flag[0]) return;
    const int L = a.L, LP = a.LP;
    const int e = blockIdx.x * NT + threadIdx.x;
    if (e >= LP * LP) return;
    const int i = e / LP, j = e % LP;
    double2* X = a.Xg;
    if (i >= L || j >= L) {
        X[e] = make_double2(0.0, 0.0);
    } else if (i < j) {
        const double2 v = X[(size_t)j * LP + i];
        X[e] = make_double2(v.x, -v.y);
    } else if (i == j) {
        X[e] = make_double2(X[e].x + a.noise, 0.0);
    }
}

// Frobenius norm of Sigma and (optionally) the prior terms; one CTA
// ||Sigma||_F: FROB_CTAS partial sums (row slices), combined in fixed order by
// finalize_large of the next iteration (the q-floor is its only reader)
__global__ void __launch_bounds__(NT) frob_large(LargeArgs a) {
    __shared__ double sred[SRED];
    if (a.flag[0]) return;
    double s = 0.0;
    const int rows = (a.L + FROB_CTAS - 1) / FROB_CTAS;
    const int r0 = blockIdx.x * rows, r1 = min(a.L, r0 + rows);
    for (int e = threadIdx.x; e < (r1 - r0) * a.L; e += NT) {
        const int i = r0 + e / a.L, j = e % a.L;
        const double2 v = a.Xg[(size_t)i * a.LP + j];
        s = fma(v.x, v.x, fma(v.y, v.y, s));
    }
    s = block_sum(s, sred);
    if (threadIdx.x == 0) a.frob_part[blockIdx.x] = s;
}

// Sweep-operator Gauss-Jordan on an 8-CTA cluster (see header comment).
__global__ void __cluster_dims__(GJ_CL, 1, 1) __launch_bounds__(GJ_NT, 1)
gj_cluster(LargeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* cbuf = reinterpret_cast<double2*>(smem_raw);   // [2 phases][4 columns][LP]
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    if (a.flag[0]) return;   // uniform across the cluster
    const int L = a.L, LP = a.LP;
    const int rank = (int)cl.block_rank();
    const int gtid = rank * GJ_NT + threadIdx.x;
    constexpr int GT = GJ_CL * GJ_NT;
    const int nbl = LP / 2, nlb = nbl * (nbl + 1) / 2;
    constexpr int SLMAX = (256 / 2) * (256 / 2 + 1) / 2 / (GJ_CL * GJ_NT) + 1;   // LP <= 256
    int bi[SLMAX], bj[SLMAX];
    double2 v[SLMAX][2][2];
#pragma unroll
    for (int u = 0; u < SLMAX; ++u) {
        const int t = gtid + GT * u;
        if (t < nlb) lower_block(t, bi[u], bj[u]); else { bi[u] = -1; bj[u] = 0; }
#pragma unroll
        for (int di = 0; di < 2; ++di)
#pragma unroll
            for (int dj = 0; dj < 2; ++dj) {
                const int i = 2 * bi[u] + di, j = 2 * bj[u] + dj;
                v[u][di][dj] = (bi[u] >= 0 && i < L && j < L && i >= j) ? a.Xg[(size_t)i * LP + j]
                                                                       : make_double2(0.0, 0.0);
            }
    }
    // 4x4 block pivots K = {k, .., k+3}: one cluster barrier per four pivots.
    // Per step every CTA holds (ping-pong) the four columns of K for all rows
    // with the K rows zeroed (cs[q][i] = a_i,k+q) and K itself (kr, full
    // 4 x 4); the owners of the next block's rows / columns broadcast them into
    // all CTAs through DSMEM.  Every thread inverts K redundantly by 2 x 2
    // blocks (pivots = those of the scalar sweep), then a_ij -= C_i M C_j^H
    // (i, j not in K), the K rows / columns become M-scaled (from the staged
    // pre-step values) and a_KK -> -M.
    __shared__ double2 kr[2][16];
    constexpr int PB = 4;
    const int LE = (L + PB - 1) / PB * PB;   // identity padding pivots L..LE-1 (LE <= LP)
#pragma unroll
    for (int u = 0; u < SLMAX; ++u)
#pragma unroll
        for (int di = 0; di < 2; ++di)
#pragma unroll
            for (int dj = 0; dj < 2; ++dj) {
                const int i = 2 * bi[u] + di, j = 2 * bj[u] + dj;
                if (i == j && i >= L && i < LE) v[u][di][dj] = make_double2(1.0, 0.0);
            }
    auto xval = [&](int i, int j) -> double2 {   // initial Sigma with the padding pivots
        if (i < L && j < L) return a.Xg[(size_t)i * LP + j];
        return (i == j && i < LE) ? make_double2(1.0, 0.0) : make_double2(0.0, 0.0);
    };
    for (int e = threadIdx.x; e < LP; e += GJ_NT) {
#pragma unroll
        for (int q = 0; q < PB; ++q)
            cbuf[q * LP + e] = (e >= PB) ? xval(e, q) : make_double2(0.0, 0.0);
    }
    if (threadIdx.x < 16) kr[0][threadIdx.x] = xval(threadIdx.x >> 2, threadIdx.x & 3);
    cl.sync();
    double logdet = 0.0;
    bool ok = true;
    for (int k = 0; k < LE; k += PB) {
        const int ph = (k / PB) & 1;
        const double2* cs = cbuf + ph * PB * LP;
        const int nbase = (ph ^ 1) * PB * LP;
        // ---- M = K^-1 by 2 x 2 blocks K = [[A, B^H], [B, C]] ------------------
        const double2* K = kr[ph];
        __shared__ double2 msm[16];   // M = K^-1 (row-major)
        __shared__ double spiv[4];
        if (threadIdx.x == 0) {
            double piv[4];
            // A^-1 (a = K00, b = K10, c = K11)
            const double a0 = K[0].x, br = K[4].x, bi_ = K[4].y, c0 = K[5].x;
            const double ainv = __drcp_rn(a0);
            const double d1 = c0 - (br * br + bi_ * bi_) * ainv;
            const double d1inv = __drcp_rn(d1);
            piv[0] = a0;
            piv[1] = d1;
            // Ai = [[p, conj(r)], [r, s]]
            const double ap = fma((br * br + bi_ * bi_) * ainv * ainv, d1inv, ainv);
            const double as = d1inv;
            const double arx = -br * ainv * d1inv, ary = -bi_ * ainv * d1inv;
            // T = B Ai (2 x 2), B rows 2,3 cols 0,1 of K
            double tx[2][2], ty[2][2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const double2 b0 = K[(2 + r) * 4 + 0], b1 = K[(2 + r) * 4 + 1];
                // col 0: b0 * p + b1 * r
                tx[r][0] = fma(b0.x, ap, b1.x * arx - b1.y * ary);
                ty[r][0] = fma(b0.y, ap, b1.x * ary + b1.y * arx);
                // col 1: b0 * conj(r) + b1 * s
                tx[r][1] = fma(b1.x, as, b0.x * arx + b0.y * ary);
                ty[r][1] = fma(b1.y, as, b0.y * arx - b0.x * ary);
            }
            // S = C - T B^H  (Hermitian 2 x 2): S[r][c] = C[r][c] - sum_p T[r][p] conj(B[c][p])
            double sx[2][2], sy[2][2];
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const double2 cc = K[(2 + r) * 4 + 2 + c];
                    double x = cc.x, y = cc.y;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const double2 bb = K[(2 + c) * 4 + q];   // B[c][q]
                        // T[r][q] * conj(bb)
                        x -= tx[r][q] * bb.x + ty[r][q] * bb.y;
                        y -= ty[r][q] * bb.x - tx[r][q] * bb.y;
                    }
                    sx[r][c] = x;
                    sy[r][c] = y;
                }
            const double s0 = sx[0][0], sbr = sx[1][0], sbi = sy[1][0], s1 = sx[1][1];
            const double sinv0 = __drcp_rn(s0);
            const double d3 = s1 - (sbr * sbr + sbi * sbi) * sinv0;
            const double d3inv = __drcp_rn(d3);
            piv[2] = s0;
            piv[3] = d3;
            // Si = [[sp, conj(sr)], [sr, ss]]
            const double sp = fma((sbr * sbr + sbi * sbi) * sinv0 * sinv0, d3inv, sinv0);
            const double ss = d3inv;
            const double srx = -sbr * sinv0 * d3inv, sry = -sbi * sinv0 * d3inv;
            const double six[2][2] = {{sp, srx}, {srx, ss}};
            const double siy[2][2] = {{0.0, -sry}, {sry, 0.0}};
            // M22 = Si; M21 = -Si T; M11 = Ai + T^H Si T
            double nx[2][2], ny[2][2];   // Si T
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    double x = 0.0, y = 0.0;
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        x += six[r][q] * tx[q][c] - siy[r][q] * ty[q][c];
                        y += six[r][q] * ty[q][c] + siy[r][q] * tx[q][c];
                    }
                    nx[r][c] = x;
                    ny[r][c] = y;
                }
            const double aix[2][2] = {{ap, arx}, {arx, as}};
            const double aiy[2][2] = {{0.0, -ary}, {ary, 0.0}};
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    msm[(2 + r) * 4 + 2 + c] = make_double2(six[r][c], siy[r][c]);
                    msm[(2 + r) * 4 + c] = make_double2(-nx[r][c], -ny[r][c]);
                    msm[c * 4 + 2 + r] = make_double2(-nx[r][c], ny[r][c]);   // M12 = M21^H
                    // (T^H Si T)[r][c] = sum_q conj(T[q][r]) (Si T)[q][c]
                    double x = aix[r][c], y = aiy[r][c];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        x += tx[q][r] * nx[q][c] + ty[q][r] * ny[q][c];
                        y += tx[q][r] * ny[q][c] - ty[q][r] * nx[q][c];
                    }
                    msm[r * 4 + c] = make_double2(x, y);
                }
#pragma unroll
            for (int r = 0; r < 4; ++r) spiv[r] = piv[r];
        }
        __syncthreads();
        const double piv[4] = {spiv[0], spiv[1], spiv[2], spiv[3]};
        auto M = [&](int r, int c) { return msm[r * 4 + c]; };
        // a failed pivot is identical in every thread (same staged K)
        if (!(piv[0] > 0.0) || !(piv[1] > 0.0) || !(piv[2] > 0.0) || !(piv[3] > 0.0)) {
            ok = false;
            break;
        }
        if (a.record_objective) logdet += log(piv[0]) + log(piv[1]) + log(piv[2]) + log(piv[3]);
        const int kb = k >> 1;
        auto bcast = [&](int idx, double2 val) {
#pragma unroll
            for (int r = 0; r < GJ_CL; ++r) cl.map_shared_rank(cbuf, r)[idx] = val;
        };
        auto in_k = [&](int bb) { return bb == kb || bb == kb + 1; };
        auto in_kn = [&](int bb) { return bb == kb + 2 || bb == kb + 3; };
#pragma unroll
        for (int u = 0; u < SLMAX; ++u) {
            if (bi[u] < 0) continue;
            const int i0 = 2 * bi[u], j0 = 2 * bj[u];
            if (!in_k(bi[u]) && !in_k(bj[u])) {
                // generic: a_ij -= sum_p c_p[i] U_j[p], U_j = M conj(C_j); one
                // column of the block at a time (register pressure)
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    double2 uu[PB];
                    {
                        double2 cj[PB];
#pragma unroll
                        for (int q = 0; q < PB; ++q) cj[q] = cs[q * LP + j0 + dj];
#pragma unroll
                        for (int p = 0; p < PB; ++p) {
                            double x = 0.0, y = 0.0;
#pragma unroll
                            for (int q = 0; q < PB; ++q) {   // M[p][q] * conj(cj[q])
                                const double2 mv = M(p, q);
                                x = fma(mv.x, cj[q].x, fma(mv.y, cj[q].y, x));
                                y = fma(mv.y, cj[q].x, fma(-mv.x, cj[q].y, y));
                            }
                            uu[p] = make_double2(x, y);
                        }
                    }
#pragma unroll
                    for (int di = 0; di < 2; ++di) {
                        double nx = v[u][di][dj].x, ny = v[u][di][dj].y;
#pragma unroll
                        for (int p = 0; p < PB; ++p) {
                            const double2 c = cs[p * LP + i0 + di];
                            nx = fma(-c.x, uu[p].x, fma(c.y, uu[p].y, nx));
                            ny = fma(-c.x, uu[p].y, fma(-c.y, uu[p].x, ny));
                        }
                        v[u][di][dj] = make_double2(nx, ny);
                    }
                }
            } else if (in_k(bi[u]) && in_k(bj[u])) {
#pragma unroll
                for (int di = 0; di < 2; ++di)
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj) {
                        const int p = i0 + di - k, q = j0 + dj - k;
                        v[u][di][dj] = make_double2(-M(p, q).x, -M(p, q).y);
                    }
            } else if (in_k(bj[u])) {
                // rows i not in K, columns K: a_i,k+q <- sum_p a_i,k+p M[p][q]
#pragma unroll
                for (int di = 0; di < 2; ++di) {
                    double2 ci[PB];
#pragma unroll
                    for (int p = 0; p < PB; ++p) ci[p] = cs[p * LP + i0 + di];
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj) {
                        const int q = j0 + dj - k;
                        double x = 0.0, y = 0.0;
#pragma unroll
                        for (int p = 0; p < PB; ++p) {
                            x = fma(ci[p].x, M(p, q).x, fma(-ci[p].y, M(p, q).y, x));
                            y = fma(ci[p].x, M(p, q).y, fma(ci[p].y, M(p, q).x, y));
                        }
                        v[u][di][dj] = make_double2(x, y);
                    }
                }
            } else {
                // rows K, columns j not in K: a_k+p,j <- sum_q M[p][q] a_k+q,j
                //   with a_k+q,j = conj(c_q[j])
#pragma unroll
                for (int dj = 0; dj < 2; ++dj) {
                    double2 cj[PB];
#pragma unroll
                    for (int q = 0; q < PB; ++q) cj[q] = cs[q * LP + j0 + dj];
#pragma unroll
                    for (int di = 0; di < 2; ++di) {
                        const int p = i0 + di - k;
                        double x = 0.0, y = 0.0;
#pragma unroll
                        for (int q = 0; q < PB; ++q) {
                            x = fma(M(p, q).x, cj[q].x, fma(M(p, q).y, cj[q].y, x));
                            y = fma(M(p, q).y, cj[q].x, fma(-M(p, q).x, cj[q].y, y));
                        }
                        v[u][di][dj] = make_double2(x, y);
                    }
                }
            }
            // ---- stage the next pivot block K' = {k+4, .., k+7} ----------------
            if (in_kn(bi[u]) && in_kn(bj[u])) {
#pragma unroll
                for (int di = 0; di < 2; ++di)
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj) {
                        const int p = i0 + di - k - PB, q = j0 + dj - k - PB;
                        if (p >= q) {
                            const double2 val = v[u][di][dj];
#pragma unroll
                            for (int r = 0; r < GJ_CL; ++r) {
                                double2* rk = cl.map_shared_rank(&kr[0][0], r) + (ph ^ 1) * 16;
                                rk[p * 4 + q] = val;
                                rk[q * 4 + p] = make_double2(val.x, -val.y);
                            }
                        }
                    }
                if (bi[u] == bj[u]) {   // the diagonal owners zero K' rows in the staged columns
#pragma unroll
                    for (int di = 0; di < 2; ++di)
#pragma unroll
                        for (int q = 0; q < PB; ++q) bcast(nbase + q * LP + i0 + di, make_double2(0.0, 0.0));
                }
            } else if (in_kn(bj[u])) {
#pragma unroll
                for (int di = 0; di < 2; ++di)
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj)
                        bcast(nbase + (j0 + dj - k - PB) * LP + i0 + di, v[u][di][dj]);
            } else if (in_kn(bi[u])) {
#pragma unroll
                for (int di = 0; di < 2; ++di)
#pragma unroll
                    for (int dj = 0; dj < 2; ++dj)
                        bcast(nbase + (i0 + di - k - PB) * LP + j0 + dj,
                              make_double2(v[u][di][dj].x, -v[u][di][dj].y));
            }
        }
        cl.sync();
    }
    // a failed pivot is seen identically by every thread of every CTA
    if (!ok) {
        if (rank == 0 && threadIdx.x == 0) {
            a.status[0] = PSCA_CHOL_FAIL;
            if (a.cond_est) a.cond_est[0] = INFINITY;
        }
        return;
    }
    if (rank == 0 && threadIdx.x == 0) a.inst[1] = logdet;
    // P = -(swept), full Hermitian, into Xg
#pragma unroll
    for (int u = 0; u < SLMAX; ++u) {
        if (bi[u] < 0) continue;
#pragma unroll
        for (int di = 0; di < 2; ++di)
#pragma unroll
            for (int dj = 0; dj < 2; ++dj) {
                const int i = 2 * bi[u] + di, j = 2 * bj[u] + dj;
                if (i >= j) {
                    const double2 pv = (i < L && j < L) ? make_double2(-v[u][di][dj].x, -v[u][di][dj].y)
                                                        : make_double2(0.0, 0.0);
                    a.Xg[(size_t)i * LP + j] = (i == j) ? make_double2(pv.x, 0.0) : pv;
                    if (i != j) a.Xg[(size_t)j * LP + i] = make_double2(pv.x, -pv.y);
                }
            }
    }
}

// G = Sigma_hat P (all 2x2 blocks, MODE 0) or A = P G (lower 2x2 blocks, MODE 1)
// G = Sigma_hat P (MODE 0, all tiles) and A = P G (MODE 1, lower tiles) on
// DMMA: one warp per 4 x 8 complex output tile in the real 2x2 expansion
// (see factor_pass), k-steps of 2 complex columns, two accumulator chains
template <int MODE>
__global__ void __launch_bounds__(NT) gemm_large(LargeArgs a) {
    if (a.flag[0] || a.status[0] != PSCA_RUNNING) return;
    const int L = a.L, LP = a.LP;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x * NWARP + warp;
    const int nrt = LP / 4, nct = LP / 8;
    int ti, tj;
    if (MODE == 0) {
        if (tile >= nrt * nct) return;
        ti = tile / nct;
        tj = tile - ti * nct;
    } else {
        if (tile >= rebuild_block_count(nrt)) return;
        int i = 0, base = 0;
        while (base + (4 * i + 3) / 8 + 1 <= tile) {
            base += (4 * i + 3) / 8 + 1;
            ++i;
        }
        ti = i;
        tj = tile - base;
    }
    const int r8 = lane >> 2, c4 = lane & 3;
    const int p = r8 & 1, q = c4 & 1;
    const unsigned long long sg = (p == 0 && q == 1) ? 0x8000000000000000ull : 0ull;
    const int l = 4 * ti + (r8 >> 1);
    const int mb = 8 * tj + r8;
    const double* Ad = reinterpret_cast<const double*>(MODE == 0 ? a.emp_cov : a.Xg);
    const int lda = (MODE == 0) ? L : LP;
    const double* Bd = reinterpret_cast<const double*>(MODE == 0 ? a.Xg : a.Gg);
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    const int kmax = (MODE == 0) ? L : LP;
    const int nks = (kmax + 1) / 2;
    // operands of GK k-steps are loaded together before their DMMAs: with the
    // loads issued one k-step at a time the warp waited out a full L2 latency
    // per k-step (ncu: 85 % long-scoreboard stalls, 73 us per launch at L = 256)
    constexpr int GK = 8;
    for (int ks0 = 0; ks0 < nks; ks0 += GK) {
        double av[GK], bv[GK];
#pragma unroll
        for (int u = 0; u < GK; ++u) {
            const int kc = 2 * (ks0 + u) + (c4 >> 1);
            const bool kin = ks0 + u < nks && kc < kmax;
            av[u] = (kin && l < (MODE == 0 ? L : LP))
                        ? __ldg(Ad + 2 * ((size_t)l * lda + kc) + (p ^ q)) : 0.0;
            bv[u] = kin ? Bd[2 * ((size_t)kc * LP + mb) + q] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GK; ++u) dmma(acc[u & 1], xsign(av[u], sg), bv[u]);
    }
    double* out = reinterpret_cast<double*>(MODE == 0 ? a.Gg : a.Ag);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int m = 8 * tj + 2 * c4 + h;
        out[2 * ((size_t)l * LP + m) + p] = acc[0][h] + acc[1][h];
    }
}

// trace(P Sigma_hat) for the objective; one CTA
__global__ void __launch_bounds__(NT) trace_large(LargeArgs a) {
    __shared__ double sred[SRED];
    if (a.flag[0] || a.status[0] != PSCA_RUNNING) return;
    double s = 0.0;
    for (int e = threadIdx.x; e < a.L * a.L; e += NT) {
        const int i = e / a.L, j = e % a.L;
        const double2 pv = a.Xg[(size_t)i * a.LP + j];
        const double2 ev = a.emp_cov[(size_t)j * a.L + i];
        s = fma(pv.x, ev.x, fma(-pv.y, ev.y, s));
    }
    s = block_sum(s, sred);
    if (threadIdx.x == 0) a.inst[2] = s;
}

// prior terms at the new iterate (x_next of the finalised iteration, or 0)
__global__ void __launch_bounds__(NT) prior_large(LargeArgs a, const double* xv) {
    __shared__ double sred[SRED];
    if (a.flag[0]) return;
    double acc = 0.0, quad = 0.0;
    const int n = blockIdx.x * NT + threadIdx.x;   // grid-stride not needed: one pass
    for (int m = n; m < a.N; m += gridDim.x * NT) {
        const double x = xv[m];
        if (a.kind == PSCA_MAP_K && a.c2_ptr) {
            // pairwise MVB prior (priors.py:145-159): -(c1 + c2 x)/M, CSR row order
            double s = 0.0;
            for (int j = a.c2_ptr[m]; j < a.c2_ptr[m + 1]; ++j)
                s = __dadd_rn(s, __dmul_rn(a.c2_val[j], xv[a.c2_idx[j]]));
            a.pgrad[m] = __ddiv_rn(-__dadd_rn(a.c1[m], s), (double)a.n_antennas);
            acc = fma(a.c1[m], x, acc);
            quad = fma(x, s, quad);
        } else if (a.kind == PSCA_MAP_UR) {
            double dens, der;
            eff_density(x, a.prior_p[m], a.eff, dens, der);
            const double mag = a.eff.dead_zone_grad;
            a.pgrad[m] = (dens <= 1e-300) ? ((x <= a.eff.g_low / 2.0) ? 1.0 : -1.0) * (mag / a.n_antennas)
                                          : -np_clip(der / dens, -mag, mag) / a.n_antennas;
            if (a.record_objective) acc += log(dens > 1e-300 ? dens : 1e-300);
        } else if (a.kind == PSCA_MAP_K) {
            acc = fma(a.prior_lin[m], x, acc);
        }
    }
    if (gridDim.x == 1 && a.record_objective) {
        acc = block_sum(acc, sred);
        if (a.kind == PSCA_MAP_K && a.c2_ptr) {
            quad = block_sum(quad, sred);
            acc = -(acc + 0.5 * quad) / a.n_antennas;
        }
        // this shard's penalty: summed over the ranks with the next exchange
        if (threadIdx.x == 0)
            a.red[1] = (a.kind == PSCA_MAP_K) ? acc : (a.kind == PSCA_MAP_UR ? -acc / a.n_antennas : 0.0);
    }
}

__global__ void __launch_bounds__(NT) pack_large(LargeArgs a) {
    if (a.flag[0] || a.status[0] != PSCA_RUNNING) return;
    const int NB = a.NRB * (a.NRB + 1);
    const int e = blockIdx.x * NT + threadIdx.x;
    if (e >= NB * 8) return;
    const int blk = e >> 3, a4 = (e >> 1) & 3, cc = e & 1;
    int i = (int)((sqrt(4.0 * blk + 1.0) - 1.0) * 0.5);
    while (i * (i + 1) > blk) --i;
    while ((i + 1) * (i + 2) <= blk) ++i;
    const int kk = blk - i * (i + 1);
    const int l = 4 * i + a4, m = 2 * kk + cc;
    double2 pv = make_double2(0.0, 0.0), av = make_double2(0.0, 0.0);
    if (l < a.L && m <= l) {
        pv = a.Xg[(size_t)l * a.LP + m];
        av = a.Ag[(size_t)l * a.LP + m];
        if (m < l) {
            pv.x *= 2.0; pv.y *= 2.0; av.x *= 2.0; av.y *= 2.0;
        } else {
            pv.y = 0.0; av.y = 0.0;
        }
    }
    const int ent = a4 * 2 + cc;
    double* o = reinterpret_cast<double*>(a.frags) + ((size_t)blk * FRAG_SLOTS + 3 * ent) * 2;
    o[0] = pv.x; o[1] = av.x;
    o[2] = pv.y; o[3] = av.y;
    o[4] = -pv.y; o[5] = -av.y;
}
