// approx_kmeans over an explicit value array (quantize.cpp:256-325) and the
// entry points that are not implemented on the device yet.
#include "engine.h"
#include "hist.cuh"
#include "kmeans_api.h"
#include "quantize_api.h"

namespace dqtg {

__global__ void __launch_bounds__(256) value_sketch_kernel(const float* x, uint64_t n,
                                                           BucketTab tab, unsigned long long* gh,
                                                           uint32_t* err) {
    extern __shared__ uint32_t sh[];
    hist_clear(sh);
    __syncthreads();
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = per * blockIdx.x, b1 = b0 + per < n ? b0 + per : n;
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) hist_add(sh, gh, x[i], tab, err);
    __syncthreads();
    hist_flush(sh, gh, tab);
}

void approx_kmeans(Engine& e, const float* values_any, uint64_t n, uint32_t k, double sigma,
                   double alpha, uint64_t seed, float* cb, uint32_t* len) {
    DQTG_REQUIRE(k >= 1, DQTG_ERROR, "k must be >= 1");
    *len = 0;
    if (n == 0) return;
    DQTG_REQUIRE(sigma >= 0.0 && sigma <= 1.0, DQTG_ERROR, "sigma must be in [0, 1]");
    AlphaTables& T = e.alpha_tables(alpha);
    const float* x = values_any;
    if (!is_device_ptr(values_any)) {
        float* d = (float*)e.buf("ak.x", n * 4);
        e.to_device(d, values_any, n * 4);
        x = d;
    }
    auto* gh = (unsigned long long*)e.buf("ak.gh", T.HS * 8);
    DQTG_CUDA(cudaMemsetAsync(gh, 0, T.HS * 8, e.stream));
    int grid = (int)std::min<uint64_t>((uint64_t)e.num_sms * 4, (n + 4095) / 4096);
    { DQTG_SPAN(e, "value_sketch_kernel"); value_sketch_kernel<<<grid, 256, kWinSlots * 4, e.stream>>>(x, n, e.bucket_tab(T), gh, e.d_err); }
    e.launched();
    auto* pts = (double*)e.buf("ak.pts", T.HS * 8);
    auto* kw = (double*)e.buf("ak.kw", T.HS * 8);
    auto* kc = (unsigned long long*)e.buf("ak.kc", T.HS * 8);
    auto* nk = (int*)e.buf("ak.nk", 16);
    compact_keys(e, gh, T.HS, T.HS, T.d_key, sigma, 1, pts, kc, kw, T.HS, nk);
    int h_nk = 0;
    e.d2h(&h_nk, nk, 4);
    e.check_err();
    float* d_cb = (float*)e.buf("ak.cb", (size_t)k * 4 + 4);
    uint32_t* d_len = (uint32_t*)e.buf("ak.len", 16);
    DQTG_CUDA(cudaMemsetAsync(d_len, 0, 4, e.stream));
    if ((uint32_t)h_nk < k) {
        distinct_value_codebook_array(e, x, n, k, sigma, seed, d_cb, d_len);
    } else {
        std::vector<KProblem> probs(1);
        probs[0] = KProblem{};
        probs[0].pts = pts;
        probs[0].w = kw;
        probs[0].n = h_nk;
        probs[0].k = (int)k;
        probs[0].seed = seed;
        probs[0].slot = 0;
        run_kmeans(e, probs, d_cb, (int)k, d_len);
    }
    e.d2h(len, d_len, 4);
    e.sync();
    if (*len) e.from_device(cb, d_cb, (size_t)*len * 4);
    e.check_err();
}


}  // namespace dqtg
