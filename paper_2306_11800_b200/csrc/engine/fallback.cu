// Distinct-value fallback of approx_kmeans (quantize.cpp:280-300): used when the
// QUANTIZE values of a layer type occupy fewer sketch buckets than k (e.g.
// LayerNorm weights that are all 1.0).  Values are gathered in element order,
// sorted on the device, de-duplicated with the reference's double compare, and
// either returned directly (<= k distinct) or clustered by the device k-means.
#include <cub/device/device_radix_sort.cuh>

#include "engine.h"
#include "kmeans.cuh"
#include "kmeans_api.h"
#include "quantize_api.h"

namespace dqtg {

__device__ __forceinline__ int classify_fb(float mag, float sens, bool has_sens, int metric,
                                           const LtParams& p) {
    bool prot = (p.flags & kProtectAll) ||
                ((p.flags & kDoProtect) && (mag > p.t_mag || (has_sens && sens > p.t_sens)));
    if (prot) return 2;
    float ps = metric ? sens : mag;
    if ((p.flags & kDoPrune) && ps <= p.t_prune) return 1;
    return 0;
}

__device__ __forceinline__ void scores_fb(const PassIn& a, bool expl, uint64_t idx, float w,
                                          float& m, float& s) {
    if (expl) {
        m = a.mag[idx];
        s = a.has_sens ? a.sens[idx] : 0.0f;
    } else {
        m = fabsf(w);
        s = a.has_sens ? fabsf(__fmul_rn(a.ema[idx], w)) : 0.0f;
    }
}

// mode 0: count per tile, mode 1: write values at tile offsets (element order)
__global__ void gather_q_kernel(PassIn a, bool expl, const LtParams* lp, int lt, int mode,
                                uint32_t* tile_cnt, const unsigned long long* tile_off,
                                float* out) {
    __shared__ unsigned long long s_scan[33];
    const Tile T = a.tiles[blockIdx.x];
    const int tl = a.types[T.tensor];
    if (tl != lt) {
        if (mode == 0 && threadIdx.x == 0) tile_cnt[blockIdx.x] = 0;
        return;
    }
    const LtParams P = lp[lt];
    unsigned long long base = mode ? tile_off[blockIdx.x] : 0ull;
    for (uint32_t i0 = 0; i0 < T.count; i0 += blockDim.x) {
        uint32_t i = i0 + threadIdx.x;
        float w = 0.0f;
        unsigned long long f = 0;
        if (i < T.count) {
            uint64_t idx = T.start + i;
            w = a.w[idx];
            float m, s;
            scores_fb(a, expl, idx, w, m, s);
            f = classify_fb(m, s, a.has_sens, a.metric, P) == 0;
        }
        unsigned long long tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(f, s_scan, &tot);
        if (mode && f) out[base + ex] = w;
        base += tot;
    }
    if (mode == 0 && threadIdx.x == 0) tile_cnt[blockIdx.x] = (uint32_t)base;
}

__global__ void zero_signs_kernel(const float* v, uint64_t n, uint32_t* flags) {
    uint32_t f = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t b = __float_as_uint(v[i]);
        if (b == 0u) f |= 1u;
        if (b == 0x80000000u) f |= 2u;
    }
    if (f) atomicOr(flags, f);
}

// libstdc++ std::sort of the gathered values (single thread) to learn which
// signed zero heads the zero run (quantize.cpp:282-288 keeps the first one).
__global__ void first_zero_kernel(float* tmp, uint64_t n, uint32_t* sign_out) {
    if (threadIdx.x || blockIdx.x) return;
    IntroSort<float, LessF>{}.sort(tmp, (long)n);
    uint32_t s = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (tmp[i] == 0.0f) {
            s = __float_as_uint(tmp[i]) >> 31;
            break;
        }
    *sign_out = s;
}

__global__ void __launch_bounds__(1024) unique_kernel(const float* sorted, uint64_t n,
                                                      const uint32_t* zflags,
                                                      const uint32_t* zsign, double* keys,
                                                      unsigned long long* counts,
                                                      unsigned long long* n_out) {
    __shared__ unsigned long long s_scan[33];
    unsigned long long base = 0;
    // pass 1: heads + key values; head index stored in counts temporarily
    for (uint64_t c0 = 0; c0 < n; c0 += blockDim.x) {
        uint64_t i = c0 + threadIdx.x;
        unsigned long long h = 0;
        if (i < n) h = (i == 0 || sorted[i] != sorted[i - 1]) ? 1ull : 0ull;
        unsigned long long tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(h, s_scan, &tot);
        if (h) {
            float v = sorted[i];
            if (v == 0.0f) {
                uint32_t both = (*zflags == 3u);
                uint32_t neg = both ? *zsign : (*zflags == 2u);
                v = __uint_as_float(neg << 31);
            }
            keys[base + ex] = (double)v;
            counts[base + ex] = i;
        }
        base += tot;
    }
    if (threadIdx.x == 0) *n_out = base;
}

__global__ void counts_from_heads_kernel(unsigned long long* heads, unsigned long long nd,
                                         uint64_t n, unsigned long long* counts) {
    unsigned long long j = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (j >= nd) return;
    unsigned long long next = j + 1 < nd ? heads[j + 1] : n;
    counts[j] = next - heads[j];
}

__global__ void __launch_bounds__(1024) mix_weights_kernel(const double* keys,
                                                           const unsigned long long* counts,
                                                           unsigned long long n, double sigma,
                                                           double* w) {
    __shared__ unsigned long long s_maxc;
    __shared__ unsigned long long s_maxk;
    if (threadIdx.x == 0) s_maxc = 1, s_maxk = 0;
    __syncthreads();
    unsigned long long lc = 1;
    double lk = 0.0;
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) {
        lc = counts[i] > lc ? counts[i] : lc;
        lk = fmax(lk, fabs(keys[i]));
    }
    atomicMax(&s_maxc, lc);
    atomicMax(&s_maxk, (unsigned long long)__double_as_longlong(lk));
    __syncthreads();
    const double maxc = (double)s_maxc, maxk = __longlong_as_double((long long)s_maxk);
    for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) {
        double nc = __ddiv_rn((double)counts[i], maxc);
        double nx = maxk > 0.0 ? __ddiv_rn(fabs(keys[i]), maxk) : 0.0;
        w[i] = __dadd_rn(__dmul_rn(sigma, nc), __dmul_rn(__dsub_rn(1.0, sigma), nx));
    }
}

__global__ void write_distinct_cb_kernel(const double* keys, unsigned long long nd, float* cb,
                                         uint32_t* cb_len) {
    if (threadIdx.x || blockIdx.x) return;
    for (unsigned long long i = 0; i < nd; ++i) cb[i] = __double2float_rn(keys[i]);
    *cb_len = (uint32_t)nd;
}

// values (device, element order) -> codebook slot
static void codebook_from_values(Engine& e, float* vals, uint64_t m, uint32_t k, double sigma,
                                 uint64_t seed, float* cb, uint32_t* cb_len_dev) {
    cudaStream_t st = e.stream;
    auto* flags = (uint32_t*)e.buf("fb.flags", 8);
    DQTG_CUDA(cudaMemsetAsync(flags, 0, 8, st));
    { DQTG_SPAN(e, "zero_signs_kernel"); zero_signs_kernel<<<(unsigned)std::min<uint64_t>(1024, (m + 255) / 256 + 1), 256, 0, st>>>(
        vals, m, flags); }
    uint32_t hf = 0;
    e.d2h(&hf, flags, 4);
    e.sync();
    if (hf == 3u) {  // both signed zeros present: sign of the zero key follows std::sort
        float* tmp = (float*)e.buf("fb.tmp", m * 4);
        DQTG_CUDA(cudaMemcpyAsync(tmp, vals, m * 4, cudaMemcpyDeviceToDevice, st));
        { DQTG_SPAN(e, "first_zero_kernel"); first_zero_kernel<<<1, 1, 0, st>>>(tmp, m, flags + 1); }
        e.launched();
    }
    float* sorted = (float*)e.buf("fb.sorted", m * 4);
    size_t tb = 0;
    DQTG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, vals, sorted, (int64_t)m, 0, 32, st));
    void* temp = e.buf("fb.cubtmp", tb + 16);
    DQTG_CUDA(cub::DeviceRadixSort::SortKeys(temp, tb, vals, sorted, (int64_t)m, 0, 32, st));
    auto* keys = (double*)e.buf("fb.keys", m * 8);
    auto* heads = (unsigned long long*)e.buf("fb.heads", m * 8);
    auto* counts = (unsigned long long*)e.buf("fb.counts", m * 8);
    auto* nd_d = (unsigned long long*)e.buf("fb.nd", 8);
    { DQTG_SPAN(e, "unique_kernel"); unique_kernel<<<1, 1024, 0, st>>>(sorted, m, flags, flags + 1, keys, heads, nd_d); }
    unsigned long long nd = 0;
    e.d2h(&nd, nd_d, 8);
    e.sync();
    { DQTG_SPAN(e, "counts_from_heads_kernel"); counts_from_heads_kernel<<<(unsigned)((nd + 255) / 256 + 1), 256, 0, st>>>(heads, nd, m,
                                                                               counts); }
    e.launched(3);
    if (nd <= k) {  // quantize.cpp:294-297
        { DQTG_SPAN(e, "write_distinct_cb_kernel"); write_distinct_cb_kernel<<<1, 1, 0, st>>>(keys, nd, cb, cb_len_dev); }
        e.launched();
        return;
    }
    auto* w = (double*)e.buf("fb.w", nd * 8);
    { DQTG_SPAN(e, "mix_weights_kernel"); mix_weights_kernel<<<1, 1024, 0, st>>>(keys, counts, nd, sigma, w); }
    e.launched();
    // the k-means writes the codebook through slot 0 of a one-slot view
    std::vector<KProblem> probs(1);
    probs[0] = KProblem{};
    probs[0].pts = keys;
    probs[0].w = w;
    probs[0].n = (int)nd;
    probs[0].k = (int)k;
    probs[0].seed = seed;
    probs[0].slot = 0;
    run_kmeans(e, probs, cb, (int)k, cb_len_dev);
}

void distinct_value_codebook(Engine& e, const PassIn& a, const LtParams* d_lp, int lt, uint32_t k,
                             const dqtg_config& cfg, uint64_t seed, float* cb, int cb_stride,
                             uint32_t* cb_len_dev) {
    const int ntiles = a.ntiles;
    auto* tile_cnt = (uint32_t*)e.buf("fb.tcnt", (size_t)ntiles * 4 + 4);
    auto* tile_off = (unsigned long long*)e.buf("fb.toff", (size_t)(ntiles + 1) * 8);
    bool expl = a.mag != nullptr;
    { DQTG_SPAN(e, "gather_q_kernel"); gather_q_kernel<<<ntiles, 256, 0, e.stream>>>(a, expl, d_lp, lt, 0, tile_cnt, tile_off,
                                                  nullptr); }
    scan_tiles(e, tile_cnt, ntiles, tile_off);
    unsigned long long m = 0;
    e.d2h(&m, tile_off + ntiles, 8);
    e.sync();
    float* vals = (float*)e.buf("fb.vals", m * 4 + 4);
    { DQTG_SPAN(e, "gather_q_kernel"); gather_q_kernel<<<ntiles, 256, 0, e.stream>>>(a, expl, d_lp, lt, 1, tile_cnt, tile_off, vals); }
    e.launched(2);
    codebook_from_values(e, vals, m, k, cfg.sigma, seed, cb + (size_t)lt * cb_stride,
                         cb_len_dev + lt);
}

void distinct_value_codebook_array(Engine& e, const float* vals_dev, uint64_t n, uint32_t k,
                                   double sigma, uint64_t seed, float* cb, uint32_t* cb_len_dev) {
    float* vals = (float*)e.buf("fb.vals_arr", n * 4 + 4);
    DQTG_CUDA(cudaMemcpyAsync(vals, vals_dev, n * 4, cudaMemcpyDeviceToDevice, e.stream));
    codebook_from_values(e, vals, n, k, sigma, seed, cb, cb_len_dev);
}

__global__ void count_protected_kernel(const Tile* tiles, const uint8_t* types,
                                       const uint16_t* levels, const uint32_t* cb_len,
                                       uint32_t* tile_prot) {
    __shared__ uint32_t s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const Tile T = tiles[blockIdx.x];
    const uint32_t pl = cb_len[types[T.tensor]] + 1;
    uint32_t c = 0;
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x) c += levels[T.start + i] == pl;
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&s, c);
    __syncthreads();
    if (threadIdx.x == 0) tile_prot[blockIdx.x] = s;
}

void count_protected(Engine& e, const Layout& L, const uint16_t* levels, const uint32_t* cb_len,
                     uint32_t* tile_prot) {
    { DQTG_SPAN(e, "count_protected_kernel"); count_protected_kernel<<<(unsigned)L.tiles.size(), 256, 0, e.stream>>>(
        L.d_tiles, L.d_types, levels, cb_len, tile_prot); }
    e.launched();
}

}  // namespace dqtg
