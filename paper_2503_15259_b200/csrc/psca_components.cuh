// psca_components.cuh -- standalone per-instance entry points of the pieces
// the fused solver runs inside its kernels (included by psca.cu):
//
//   prior_terms_kernel   psca_prior_terms: the prior gradient / value /
//                        smoothed density at a given x, through the SAME
//                        device function (fac_prior_terms_at) the factor
//                        kernel evaluates at every iterate
//                        (priors.py:145-159, 313-399)
//   coord_step_kernel    psca_coord_step: q-floor guard, gradient, surrogate
//                        coefficient, clipped coordinate minimiser, relaxed
//                        update and update norm (estimators.py:176-200,
//                        233-236, 267-284)
//   fault_kernel         the fault-injection seam of psca_solve
//
// One CTA per instance, grid-stride over the N devices; reductions are the
// deterministic block_sum (fixed order, no atomics).

__global__ void __launch_bounds__(NT) prior_terms_kernel(FacArgs a, const double* __restrict__ x,
                                                         double* value, double* density) {
    __shared__ double sred[SRED];
    const int b = blockIdx.x;
    const size_t bN = (size_t)b * a.N;
    const double v = fac_prior_terms_at(a, b, x + bN, sred);
    if (a.kind == PSCA_MAP_K && !a.c2_ptr) {
        // independent prior: the gradient is the constant -log(p/(1-p))/M
        for (int n = threadIdx.x; n < a.N; n += NT) a.pgrad[bN + n] = a.prior_lin[n];
    }
    if (density && a.kind == PSCA_MAP_UR) {
        for (int n = threadIdx.x; n < a.N; n += NT) {
            double dens, der;
            eff_density(x[bN + n], a.prior_p[n], a.eff, dens, der);
            density[bN + n] = dens;
        }
    }
    if (value && threadIdx.x == 0) value[b] = v;
}

__global__ void __launch_bounds__(NT) coord_step_kernel(psca_coord_args a) {
    __shared__ double sred[SRED];
    const int b = blockIdx.x;
    const size_t bN = (size_t)b * a.N;
    const bool known = a.kind == PSCA_ML_K || a.kind == PSCA_MAP_K;
    double minq = INFINITY, dx2 = 0.0;
    for (int n = threadIdx.x; n < a.N; n += NT) {
        const double q = a.q[bN + n], r = a.r[bN + n], x = a.x[bN + n];
        minq = (q < minq) ? q : minq;
        const double diff = __dsub_rn(q, r);
        double gr = known ? __dmul_rn(a.gains[bN + n], diff) : diff;
        if (a.prior_grad) gr = __dadd_rn(gr, a.prior_grad[bN + n]);
        const double gq = known ? __dmul_rn(a.gains[bN + n], q) : q;
        const double cf = __dmul_rn(gq, gq);
        const double cand = np_clip(__dsub_rn(x, __ddiv_rn(gr, cf)), 0.0, a.hi);
        const double xn = __dadd_rn(__dmul_rn(__dsub_rn(1.0, a.rho), x), __dmul_rn(a.rho, cand));
        const double d = __dsub_rn(xn, x);
        dx2 = fma(d, d, dx2);
        if (a.grad) a.grad[bN + n] = gr;
        if (a.coef) a.coef[bN + n] = cf;
        if (a.cand) a.cand[bN + n] = cand;
        if (a.x_new) a.x_new[bN + n] = xn;
    }
    dx2 = block_sum(dx2, sred);
    // block minimum of q (fixed order)
    for (int o = 16; o > 0; o >>= 1) {
        const double m = __shfl_xor_sync(0xffffffffu, minq, o);
        minq = (m < minq) ? m : minq;
    }
    __shared__ double smin[NT / 32];
    if ((threadIdx.x & 31) == 0) smin[threadIdx.x >> 5] = minq;
    double frob2 = 0.0;
    if (a.sigma) {
        const double2* S = reinterpret_cast<const double2*>(a.sigma) + (size_t)b * a.L * a.L;
        for (int e = threadIdx.x; e < a.L * a.L; e += NT) {
            const double2 v = S[e];
            frob2 = fma(v.x, v.x, fma(v.y, v.y, frob2));
        }
    }
    frob2 = block_sum(frob2, sred);   // synchronises, so smin is complete
    if (threadIdx.x == 0) {
        double mq = smin[0];
        for (int w = 1; w < NT / 32; ++w) mq = (smin[w] < mq) ? smin[w] : mq;
        if (a.update_norm) a.update_norm[b] = sqrt(dx2);
        if (a.status) {
            int st = PSCA_RUNNING;
            if (a.sigma && mq < 0.5 * a.L / sqrt(frob2)) st = PSCA_QFLOOR;
            a.status[b] = st;
        }
    }
}

// psca_solve fault seam: every instance still running reports a failed
// factorisation (as a non-positive pivot would)
__global__ void fault_kernel(int* status, double* cond_est, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B && status[b] == PSCA_RUNNING) {
        status[b] = PSCA_CHOL_FAIL;
        if (cond_est) cond_est[b] = INFINITY;
    }
}
