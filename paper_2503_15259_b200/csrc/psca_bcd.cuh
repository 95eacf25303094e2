// psca_bcd.cuh -- block coordinate descent sweep (baselines.py:54-150), the
// sequential comparison detector.  Included by psca.cu inside its anonymous
// namespace.
//
// One CTA per instance walks the devices in ascending order; per device:
//   u = Sigma^-1 s, q = Re s^H u, r = Re u^H Sigma_hat u     (rows on threads)
//   exact coordinate minimiser of the 1-D objective             (thread 0)
//   Sigma^-1 -= (dw / (1 + dw q)) u u^H  (Sherman-Morrison, covlinalg.py:118-131)
// Sigma^-1 and Sigma_hat stay in SMEM for the whole sweep (row stride L + 1:
// thread-per-row reads are bank-conflict free), the iterate x in SMEM; four
// barriers per device.  The sweep is inherently sequential over devices, so
// parallelism comes from the batch (one CTA per instance).

constexpr int BCD_NT = 128;

__device__ double bcd_coord_objective(double x_new, double x_old, double gq, double gr,
                                      double slope) {   // baselines.py:25-35
    const double delta = x_new - x_old;
    const double u = 1.0 + delta * gq;
    return log(u) - delta * gr / u + slope * x_new;
}

__device__ double bcd_stationary_root(double gq, double gr, double slope) {   // :38-47
    const double disc = gq * gq + 4.0 * slope * gr;
    return 2.0 * gr / (gq + sqrt(disc));
}

// exact minimiser of one coordinate problem on [0, hi] (baselines.py:121-139)
__device__ double bcd_coordinate(double x_old, double gq, double gr, double slope, double hi) {
    if (slope >= 0.0) {
        const double u_star = slope > 0.0 ? bcd_stationary_root(gq, gr, slope) : gr / gq;
        return np_clip(x_old + (u_star - 1.0) / gq, 0.0, hi);
    }
    const double disc = gq * gq + 4.0 * slope * gr;
    const double top = hi < 1.0 ? hi : 1.0;
    if (disc <= 0.0) return top;
    const double root =
        np_clip(x_old + (bcd_stationary_root(gq, gr, slope) - 1.0) / gq, 0.0, hi);
    const double cand[3] = {root, 0.0, top};
    int best = 0;
    double bv = bcd_coord_objective(cand[0], x_old, gq, gr, slope);
    if (!(bv == bv)) return cand[0];   // np.argmin returns the first NaN
    for (int c = 1; c < 3; ++c) {
        const double v = bcd_coord_objective(cand[c], x_old, gq, gr, slope);
        if (!(v == v)) return cand[c];
        if (v < bv) {
            bv = v;
            best = c;
        }
    }
    return cand[best];
}

__global__ void __launch_bounds__(BCD_NT) bcd_sweep_kernel(psca_bcd_args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double qpart[128], rpart[128];
    __shared__ double s_coef;
    __shared__ int s_stop;
    const int b = blockIdx.x, tid = threadIdx.x;
    const int L = a.L, N = a.N, ld = L + 1;
    if (a.status[b] != 0) return;
    double2* P = reinterpret_cast<double2*>(smem_raw);    // [L][ld] Sigma^-1
    double2* E = P + (size_t)L * ld;                       // [L][ld] Sigma_hat
    double2* s = E + (size_t)L * ld;                       // [2][L] pilot column ping-pong
    double2* u = s + 2 * L;                                // [L]
    double* xs = reinterpret_cast<double*>(u + L);         // [N]
    const double2* Pg = reinterpret_cast<const double2*>(a.sigma_inv) + (size_t)b * L * L;
    const double2* Eg = reinterpret_cast<const double2*>(a.emp_cov) + (size_t)b * L * L;
    const double2* Sg = reinterpret_cast<const double2*>(a.pilots) + (size_t)b * L * N;
    double* xg = a.x + (size_t)b * N;
    const bool known = a.kind != PSCA_ML_UD;
    const double hi = known ? 1.0 : INFINITY;
    const double inv_s2 = 1.0 / a.noise[b];
    for (int e = tid; e < L * L; e += BCD_NT) {
        const int i = e / L, j = e - i * L;
        E[i * ld + j] = Eg[e];
        P[i * ld + j] = a.init ? make_double2(i == j ? inv_s2 : 0.0, 0.0) : Pg[e];
    }
    for (int n = tid; n < N; n += BCD_NT) xs[n] = a.init ? 0.0 : xg[n];
    if (tid < L) s[tid] = Sg[(size_t)tid * N];
    if (tid == 0) s_stop = 0;
    __syncthreads();

    for (int n = 0; n < N; ++n) {
        const double2* sc = s + (n & 1) * L;
        // u = Sigma^-1 s, q partials
        if (tid < L) {
            double ux = 0.0, uy = 0.0;
            const double2* prow = P + tid * ld;
            for (int k = 0; k < L; ++k) {
                const double2 pv = prow[k], sv = sc[k];
                ux = fma(pv.x, sv.x, fma(-pv.y, sv.y, ux));
                uy = fma(pv.x, sv.y, fma(pv.y, sv.x, uy));
            }
            u[tid] = make_double2(ux, uy);
            qpart[tid] = sc[tid].x * ux + sc[tid].y * uy;   // Re conj(s_t) u_t
        }
        __syncthreads();
        // Sigma_hat u, r partials
        if (tid < L) {
            double vx = 0.0, vy = 0.0;
            const double2* erow = E + tid * ld;
            for (int k = 0; k < L; ++k) {
                const double2 ev = erow[k], uv = u[k];
                vx = fma(ev.x, uv.x, fma(-ev.y, uv.y, vx));
                vy = fma(ev.x, uv.y, fma(ev.y, uv.x, vy));
            }
            rpart[tid] = u[tid].x * vx + u[tid].y * vy;      // Re conj(u_t) v_t
        }
        __syncthreads();
        if (tid == 0) {
            double q = 0.0, r = 0.0;
            for (int t = 0; t < L; ++t) q += qpart[t];
            for (int t = 0; t < L; ++t) r += rpart[t];
            const double g = known ? a.gains[(size_t)b * N + n] : 1.0;
            const double gq = g * q, gr = g * r;
            double slope = 0.0;
            if (a.kind == PSCA_MAP_K) {
                if (a.prior_c2_indptr) {   // -(c1 + c2 x)/M at the current iterate
                    double acc = 0.0;
                    for (int j = a.prior_c2_indptr[n]; j < a.prior_c2_indptr[n + 1]; ++j)
                        acc += a.prior_c2_data[j] * xs[a.prior_c2_indices[j]];
                    slope = -(a.prior_c1[n] + acc) / a.n_antennas;
                } else {
                    slope = a.prior_lin[n];
                }
            }
            const double x_old = xs[n];
            const double x_new = bcd_coordinate(x_old, gq, gr, slope, hi);
            const double dw = (x_new - x_old) * g;
            double coef = 0.0;
            if (dw != 0.0) {
                const double denom = 1.0 + dw * q;
                if (denom <= 1e-14) {
                    a.status[b] = 1;
                    s_stop = 1;
                } else {
                    coef = dw / denom;
                }
            }
            if (!s_stop) xs[n] = x_new;
            s_coef = coef;
        }
        // the next pilot column, consumed after the next barrier
        if (tid < L && n + 1 < N) s[((n + 1) & 1) * L + tid] = Sg[(size_t)tid * N + n + 1];
        __syncthreads();
        if (s_stop) break;
        const double coef = s_coef;
        if (coef != 0.0) {
            for (int e = tid; e < L * L; e += BCD_NT) {
                const int i = e / L, j = e - i * L;
                const double2 ui = u[i], uj = u[j];
                const double ox = ui.x * uj.x + ui.y * uj.y;   // u_i conj(u_j)
                const double oy = ui.y * uj.x - ui.x * uj.y;
                double2& pv = P[i * ld + j];
                pv = make_double2(pv.x - coef * ox, pv.y - coef * oy);
            }
        }
        __syncthreads();
    }
    double2* Po = reinterpret_cast<double2*>(a.sigma_inv) + (size_t)b * L * L;
    for (int e = tid; e < L * L; e += BCD_NT) {
        const int i = e / L, j = e - i * L;
        Po[e] = P[i * ld + j];
    }
    for (int n = tid; n < N; n += BCD_NT) xg[n] = xs[n];
}

size_t bcd_smem_bytes(int L, int N) {
    return (size_t)2 * L * (L + 1) * 16 + (size_t)3 * L * 16 + (size_t)N * 8;
}
