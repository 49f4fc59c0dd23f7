// Stand-alone device primitives behind the C ABI: sketch_build over a float
// array (sketch.cpp:131-148), ema_update (ranker.cpp:21-37), compute_scores
// (ranker.cpp:79-101), delta_compute/apply (codec.cpp:12-37).
#include "engine.h"
#include "hist.cuh"

namespace dqtg {

__global__ void __launch_bounds__(256) sketch_kernel(const float* x, uint64_t n, BucketTab tab,
                                                     unsigned long long* gh, uint32_t* err) {
    extern __shared__ uint32_t sh[];
    hist_clear(sh);
    __syncthreads();
    const uint64_t per = (n + gridDim.x - 1) / gridDim.x;
    const uint64_t b0 = per * blockIdx.x, b1 = b0 + per < n ? b0 + per : n;
    for (uint64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) hist_add(sh, gh, x[i], tab, err);
    __syncthreads();
    hist_flush(sh, gh, tab);
}

void sketch_build(Engine& e, const float* x_any, uint64_t n, double alpha, uint64_t* zero,
                  uint64_t* pos, uint64_t* neg) {
    AlphaTables& T = e.alpha_tables(alpha);
    const float* x = x_any;
    if (n && !is_device_ptr(x_any)) {
        float* d = (float*)e.buf("sk.x", n * 4);
        e.to_device(d, x_any, n * 4);
        x = d;
    }
    auto* gh = (unsigned long long*)e.buf("sk.gh", T.HS * 8);
    DQTG_CUDA(cudaMemsetAsync(gh, 0, T.HS * 8, e.stream));
    if (n) {
        int grid = (int)std::min<uint64_t>((uint64_t)e.num_sms * 4, (n + 4095) / 4096);
        { DQTG_SPAN(e, "sketch_kernel"); sketch_kernel<<<grid, 256, kWinSlots * 4, e.stream>>>(x, n, e.bucket_tab(T), gh, e.d_err); }
        e.launched();
    }
    std::vector<unsigned long long> h(T.HS);
    e.d2h(h.data(), gh, T.HS * 8);
    e.check_err();
    *zero = h[T.NB];
    for (int64_t k = T.kmin; k <= T.kmax; ++k) {
        pos[k - T.kmin] = h[T.NB + 1 + k - T.kmin];
        neg[k - T.kmin] = h[T.kmax - k];
    }
}

__global__ void ema_kernel(float* e, const float* g, uint64_t n, float b) {
    const float ob = __fsub_rn(1.0f, b);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        e[i] = __fadd_rn(__fmul_rn(b, g[i]), __fmul_rn(ob, e[i]));
}

void ema_update(Engine& e, float* ema_dev, const float* g_dev, uint64_t n, float beta) {
    if (!n) return;
    int grid = (int)std::min<uint64_t>((uint64_t)e.num_sms * 8, (n + 255) / 256);
    { DQTG_SPAN(e, "ema_kernel"); ema_kernel<<<grid, 256, 0, e.stream>>>(ema_dev, g_dev, n, beta); }
    e.launched();
    DQTG_CUDA(cudaGetLastError());
}

__global__ void scores_kernel(const float* w, const float* ema, uint64_t n, float* mag,
                              float* sens) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        float x = w[i];
        if (mag) mag[i] = fabsf(x);
        if (sens) sens[i] = fabsf(__fmul_rn(ema[i], x));
    }
}

void compute_scores(Engine& e, const float* w, const float* ema, uint64_t n, float* mag,
                    float* sens) {
    if (!n) return;
    int grid = (int)std::min<uint64_t>((uint64_t)e.num_sms * 8, (n + 255) / 256);
    { DQTG_SPAN(e, "scores_kernel"); scores_kernel<<<grid, 256, 0, e.stream>>>(w, ema, n, mag, sens); }
    e.launched();
    DQTG_CUDA(cudaGetLastError());
}

__global__ void delta_kernel(const uint16_t* prev, const uint16_t* x, uint64_t n, uint32_t B,
                             uint16_t* out, bool apply, uint32_t* err) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t p = prev[i], c = x[i];
        if (p >= B || c >= B) {
            atomicOr(err, kErrCorruptIndex);
            continue;
        }
        out[i] = (uint16_t)(p >= c ? p - c : p + B - c);  // same formula both ways
    }
    (void)apply;
}

void delta_kernel_api(Engine& e, const uint16_t* prev, const uint16_t* x, uint64_t n, uint32_t B,
                      uint16_t* out, bool apply) {
    DQTG_REQUIRE(B > 0, DQTG_ERROR, "cyclic alphabet size must be positive");
    if (!n) return;
    auto* dp = (uint16_t*)e.buf("dl.p", n * 2);
    auto* dx = (uint16_t*)e.buf("dl.x", n * 2);
    auto* dout = (uint16_t*)e.buf("dl.o", n * 2);
    e.to_device(dp, prev, n * 2);
    e.to_device(dx, x, n * 2);
    int grid = (int)std::min<uint64_t>((uint64_t)e.num_sms * 8, (n + 255) / 256);
    { DQTG_SPAN(e, "delta_kernel"); delta_kernel<<<grid, 256, 0, e.stream>>>(dp, dx, n, B, dout, apply, e.d_err); }
    e.launched();
    e.from_device(out, dout, n * 2);
    e.check_err();
}

}  // namespace dqtg
