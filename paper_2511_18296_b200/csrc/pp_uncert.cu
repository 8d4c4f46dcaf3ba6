// pp_uncert.cu -- uncertainty_factors (uncertainty.py:276-321) on the device: sigma[S][T] of a
// grade matrix, with Moran's I over the rook weights (pp_set_rook: the directed pairs of
// rook_weights, uncertainty.py:50-76, unit weights) and the local coefficient of variation.
//
// One CTA per scenario, every sum a numpy pairwise sum in numpy's order (s2_pairwise_f): the mean
// (np.mean), the squared deviations (np.std, np.var's reduction) and the Moran numerator
// np.sum(w * dev[i] * dev[j]) over the pairs in rook order.  One term is not numpy's own: the Moran
// denominator `dev @ dev` is a BLAS dot product, whose summation order belongs to the BLAS build;
// here it is the same pairwise sum of dev^2, so sigma agrees with the reference to rounding (the
// tests: relative 1e-12), not bit for bit -- which is why the drop-ins keep taking sigma as an
// input and this is an ingestion path (the refresh of colgen.py:477-478 without the host).
#include "pp_internal.cuh"

namespace {

constexpr int UT = 1024;

// psi, phi[T] from the host (np.exp and the feature blend); out: sigma[S][T], moran[S] (NaN when the
// field is degenerate), local[S]
__global__ void __launch_bounds__(UT) k_uncertainty(const double *__restrict__ grades, int B, int T,
                                                    const int32_t *__restrict__ rpi, const int32_t *__restrict__ ridx,
                                                    int E, const double *__restrict__ phi, double psi,
                                                    int *__restrict__ leaf_s, int *__restrict__ leaf_l,
                                                    double *__restrict__ leaf_v, int cap, double *__restrict__ sigma,
                                                    double *__restrict__ moran_out, double *__restrict__ local_out) {
    const int s = blockIdx.x;
    const double *x = grades + (size_t)s * B;
    int *ls = leaf_s + (size_t)s * cap, *ll = leaf_l + (size_t)s * cap;
    double *lv = leaf_v + (size_t)s * cap;
    __shared__ double s_mean;
    const double sum = s2_pairwise_f([&](int k) { return x[k]; }, B, ls, ll, lv);
    if (threadIdx.x == 0) s_mean = f64_div(sum, (double)B);
    __syncthreads();
    const double mean = s_mean;
    // np.std: the deviations squared, their pairwise sum / n, sqrt; the same sum stands in for the
    // BLAS dot product of the Moran denominator
    const double ssq = s2_pairwise_f(
        [&](int k) {
            const double d = f64_sub(x[k], mean);
            return f64_mul(d, d);
        },
        B, ls, ll, lv);
    // Moran numerator over the directed rook pairs (i ascending, j in rook order): (w * dev[i]) * dev[j]
    const double num = s2_pairwise_f(
        [&](int k) { return f64_mul(f64_mul(1.0, f64_sub(x[rpi[k]], mean)), f64_sub(x[ridx[k]], mean)); }, E, ls, ll,
        lv);
    if (threadIdx.x == 0) {
        const double var = f64_div(ssq, (double)B);
        const double std_ = __dsqrt_rn(var);
        const double local = mean > 0 ? f64_div(std_, mean) : 0.0;
        const bool degenerate = !(ssq > 0);
        double f;
        if (degenerate) {
            f = f64_add(1.0, local);
            moran_out[s] = __longlong_as_double(0x7ff8000000000000ll);  // NaN, as the reference's array
        } else {
            const double mi = f64_div(f64_mul((double)B, num), f64_mul((double)E, ssq));
            moran_out[s] = mi;
            f = f64_add(f64_sub(1.0, mi), local);
        }
        local_out[s] = local;
        for (int t = 0; t < T; t++) {
            double r = f64_mul(f64_mul(f, phi[t]), psi);
            r = r < 1e-6 ? 1e-6 : (r > 2.0 ? 2.0 : r);  // np.clip(raw, SIGMA_FLOOR, SIGMA_CEIL)
            sigma[(size_t)s * T + t] = r;
        }
    }
}

}  // namespace

extern "C" {

int pp_uncertainty_sigma(pp_ctx *c, int32_t n_scen, const double *grades, const double *phi, double psi,
                         double *sigma_out, double *moran_out, double *local_out, int32_t mem, void *stream) {
    if (!c || !c->have_instance || !c->have_rook) return fail(PP_ERR_STATE, "pp_set_instance and pp_set_rook first");
    if (n_scen < 1 || !grades || !phi || !sigma_out) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if (mem != PP_MEM_HOST && mem != PP_MEM_DEVICE) return fail(PP_ERR_INVALID_ARGS, "unknown memory kind %d", mem);
    if (c->B < 2) return fail(PP_ERR_INVALID_ARGS, "need at least 2 blocks");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int S = n_scen, B = c->B, T = c->T;
    const int E = c->rook_pairs;
    if (E <= 0) return fail(PP_ERR_INVALID_ARGS, "weights must have positive total");
    const int cap = std::max(B, E) / 64 + 4;
    DevBuf leaves, io;
    TRY(leaves.ensure((size_t)S * cap * (4 + 4 + 8)));
    const size_t n_in = mem == PP_MEM_HOST ? (size_t)S * B : 0;
    TRY(io.ensure(sizeof(double) * (n_in + T + (size_t)S * T + 2 * (size_t)S)));
    double *dg = const_cast<double *>(grades), *dphi = io.as<double>() + n_in, *dsig = dphi + T, *dmo = dsig + (size_t)S * T,
           *dlo = dmo + S;
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(io.ptr, grades, sizeof(double) * n_in, cudaMemcpyHostToDevice, st));
        dg = io.as<double>();
    }
    CUDA_TRY(cudaMemcpyAsync(dphi, phi, sizeof(double) * T, mem == PP_MEM_HOST ? cudaMemcpyHostToDevice
                                                                                : cudaMemcpyDeviceToDevice, st));
    int *ls = leaves.as<int>(), *ll = ls + (size_t)S * cap;
    double *lv = reinterpret_cast<double *>(ll + (size_t)S * cap);
    k_uncertainty<<<S, UT, 0, st>>>(dg, B, T, c->lns_rpi.as<int32_t>(), c->lns_ridx.as<int32_t>(), E, dphi, psi, ls, ll,
                                    lv, cap, dsig, dmo, dlo);
    CUDA_TRY(cudaGetLastError());
    const cudaMemcpyKind k = mem == PP_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    CUDA_TRY(cudaMemcpyAsync(sigma_out, dsig, sizeof(double) * (size_t)S * T, k, st));
    if (moran_out) CUDA_TRY(cudaMemcpyAsync(moran_out, dmo, sizeof(double) * S, k, st));
    if (local_out) CUDA_TRY(cudaMemcpyAsync(local_out, dlo, sizeof(double) * S, k, st));
    CUDA_TRY(cudaStreamSynchronize(st));  // (the scratch is released on return)
    return PP_OK;
}

}  // extern "C"
