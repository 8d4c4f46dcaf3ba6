// pp_vae.cu -- the VAE scenario decode on the device (§8(f) row 4, ingestion): prior samples
// z[S][latent] through the decoder MLP of vae.py:91-93 (nn.py:42-53: dense layers, relu between
// them, the last one linear), de-normalised (yn * norm_std + norm_mean) and clamped at zero
// (vae.py:284-292), giving grades[S][B] -- optionally bound straight into the scenario value table
// (pp_set_scenarios_vae) so the generated set never visits the host.
//
// Each layer is Y[S][O] = X[S][I] W^T + b (W stored [O][I] as the reference's Dense) as a tiled f64
// GEMM: 64x64 output tiles, 16-deep k steps through shared memory, 4x4 outputs per thread,
// accumulated with fused multiply-adds.  The reference's numpy matmul goes through BLAS, whose
// blocking and FMA use are its own, so the decode agrees to rounding (relative 1e-12 in the tests),
// not bit for bit -- unlike the evaluation path, whose arithmetic is the reference's own scalar
// order.  The decode is dense work with no reuse problem: the output layer's W (B x 256 doubles,
// 102 MB at 50k blocks) is read once per 64-scenario tile.
#include "pp_internal.cuh"

namespace {

constexpr int VT = 64;   // output tile (scenarios x outputs)
constexpr int VK = 16;   // k step
constexpr int VTHREADS = 256;

// act: 1 = relu, 0 = linear; denorm: final layer (y * std + mean, then max(0, .))
__global__ void __launch_bounds__(VTHREADS) k_dense(const double *__restrict__ X, int S, int I,
                                                    const double *__restrict__ W, const double *__restrict__ bias, int O,
                                                    double *__restrict__ Y, int act, const double *__restrict__ nmean,
                                                    const double *__restrict__ nstd) {
    __shared__ double sx[VK][VT + 1];  // X tile, k-major (scenario fastest)
    __shared__ double sw[VK][VT + 1];  // W tile, k-major (output fastest)
    const int tid = threadIdx.x;
    const int s0 = blockIdx.y * VT, o0 = blockIdx.x * VT;
    const int ts = (tid / 16) * 4, to = (tid % 16) * 4;  // this thread's 4x4 outputs
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < I; k0 += VK) {
        // coalesced tile loads: 64 rows x 16 k each, 4 elements per thread
        for (int e = tid; e < VT * VK; e += VTHREADS) {
            const int r = e / VK, k = e % VK;
            const int s = s0 + r, o = o0 + r, kk = k0 + k;
            sx[k][r] = (s < S && kk < I) ? X[(size_t)s * I + kk] : 0.0;
            sw[k][r] = (o < O && kk < I) ? W[(size_t)o * I + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < VK; k++) {
            double xv[4], wv[4];
#pragma unroll
            for (int a = 0; a < 4; a++) xv[a] = sx[k][ts + a];
#pragma unroll
            for (int b = 0; b < 4; b++) wv[b] = sw[k][to + b];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] = __fma_rn(xv[a], wv[b], acc[a][b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int s = s0 + ts + a;
        if (s >= S) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int o = o0 + to + b;
            if (o >= O) continue;
            double y = f64_add(acc[a][b], bias[o]);
            if (act) y = y > 0.0 ? y : 0.0;
            if (nmean) {
                y = f64_add(f64_mul(y, nstd[o]), nmean[o]);
                y = y > 0.0 ? y : 0.0;
            }
            Y[(size_t)s * O + o] = y;
        }
    }
}

}  // namespace

// decode z[S][latent] (device) into grades[S][B] (device), scratch in c->vae_h
static int vae_decode_dev(pp_ctx *c, int S, const double *dz, double *dgrades, cudaStream_t st) {
    const int L = (int)c->vae_widths.size() - 1;
    size_t hmax = 0;
    for (int l = 1; l < L; l++) hmax = std::max(hmax, (size_t)c->vae_widths[l]);
    TRY(c->vae_h.ensure(sizeof(double) * 2 * (size_t)S * std::max<size_t>(hmax, 1)));
    double *h0 = c->vae_h.as<double>(), *h1 = h0 + (size_t)S * hmax;
    const double *x = dz;
    const double *params = c->vae_params.as<double>();
    size_t off = 0;
    for (int l = 0; l < L; l++) {
        const int I = c->vae_widths[l], O = c->vae_widths[l + 1];
        const double *W = params + off, *b = W + (size_t)O * I;
        off += (size_t)O * I + O;
        const bool last = l == L - 1;
        double *y = last ? dgrades : (l % 2 == 0 ? h0 : h1);
        dim3 grid((O + VT - 1) / VT, (S + VT - 1) / VT);
        k_dense<<<grid, VTHREADS, 0, st>>>(x, S, I, W, b, O, y, last ? 0 : 1,
                                           last ? c->vae_norm.as<double>() : nullptr,
                                           last ? c->vae_norm.as<double>() + c->B : nullptr);
        CUDA_TRY(cudaGetLastError());
        x = y;
    }
    return PP_OK;
}

// defined in pp_schedule.cu: bind grades[S][B] already on the device as the scenario set
int set_scenarios_from_device_grades(pp_ctx *c, int32_t S, const double *dgrades, int32_t n_modes, double price,
                                     const double *recovery, int32_t n_recovery, const double *proc_cost,
                                     int32_t n_proc_cost, const double *sigma_st);

extern "C" {

int pp_set_vae_decoder(pp_ctx *c, int32_t n_layers, const int32_t *widths, const double *params,
                       const double *norm_mean, const double *norm_std) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (n_layers < 1 || !widths || !params || !norm_mean || !norm_std) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    for (int l = 0; l <= n_layers; l++)
        if (widths[l] < 1) return fail(PP_ERR_INVALID_ARGS, "layer width %d < 1", widths[l]);
    if (widths[n_layers] != c->B)
        return fail(PP_ERR_SHAPE, "the decoder's output width %d differs from the instance's %d blocks", widths[n_layers], c->B);
    size_t n = 0;
    for (int l = 0; l < n_layers; l++) n += (size_t)widths[l] * widths[l + 1] + widths[l + 1];
    TRY(use_device(c));
    TRY(c->vae_params.ensure(sizeof(double) * n));
    TRY(c->vae_norm.ensure(sizeof(double) * 2 * (size_t)c->B));
    CUDA_TRY(dev_upload(c, c->vae_params.ptr, params, sizeof(double) * n));
    CUDA_TRY(dev_upload(c, c->vae_norm.ptr, norm_mean, sizeof(double) * c->B));
    CUDA_TRY(dev_upload(c, c->vae_norm.as<double>() + c->B, norm_std, sizeof(double) * c->B));
    c->vae_widths.assign(widths, widths + n_layers + 1);
    return PP_OK;
}

int pp_vae_decode(pp_ctx *c, int32_t n_scen, const double *z, double *grades_out, int32_t mem, void *stream) {
    if (!c || c->vae_widths.empty()) return fail(PP_ERR_STATE, "pp_set_vae_decoder first");
    if (n_scen < 1 || !z || !grades_out) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if (mem != PP_MEM_HOST && mem != PP_MEM_DEVICE) return fail(PP_ERR_INVALID_ARGS, "unknown memory kind %d", mem);
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int S = n_scen, D = c->vae_widths[0], B = c->B;
    const double *dz = z;
    double *dg = grades_out;
    if (mem == PP_MEM_HOST) {
        TRY(c->vae_io.ensure(sizeof(double) * ((size_t)S * D + (size_t)S * B)));
        CUDA_TRY(cudaMemcpyAsync(c->vae_io.ptr, z, sizeof(double) * (size_t)S * D, cudaMemcpyHostToDevice, st));
        dz = c->vae_io.as<double>();
        dg = c->vae_io.as<double>() + (size_t)S * D;
    }
    TRY(vae_decode_dev(c, S, dz, dg, st));
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(grades_out, dg, sizeof(double) * (size_t)S * B, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return PP_OK;
}

int pp_set_scenarios_vae(pp_ctx *c, int32_t n_scen, const double *z, int32_t n_modes, double price,
                         const double *recovery, int32_t n_recovery, const double *proc_cost, int32_t n_proc_cost,
                         const double *sigma_st) {
    if (!c || c->vae_widths.empty()) return fail(PP_ERR_STATE, "pp_set_vae_decoder first");
    if (n_scen < 1 || !z) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    TRY(use_device(c));
    const int S = n_scen, D = c->vae_widths[0], B = c->B;
    DevBuf buf;
    TRY(buf.ensure(sizeof(double) * ((size_t)S * D + (size_t)S * B)));
    CUDA_TRY(cudaMemcpyAsync(buf.ptr, z, sizeof(double) * (size_t)S * D, cudaMemcpyHostToDevice, c->stream));
    double *dg = buf.as<double>() + (size_t)S * D;
    int rc = vae_decode_dev(c, S, buf.as<double>(), dg, c->stream);
    if (rc == PP_OK)
        rc = set_scenarios_from_device_grades(c, S, dg, n_modes, price, recovery, n_recovery, proc_cost, n_proc_cost,
                                              sigma_st);
    buf.release();
    return rc;
}

}  // extern "C"
