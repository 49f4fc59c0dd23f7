// quantize_checkpoint on the device (quantize.cpp:34-92, 373-425).
//
//   pass A  score histograms per layer type (magnitude / sensitivity), scores
//           derived in registers from w (+EMA) or read from explicit ScoreSets
//   quantile thresholds on device (sketch.cpp:59-77), float round-down (§7 H2)
//   pass B  partition + QUANTIZE-value histogram + protected counts per tile
//   keys    histogram -> ascending keys + mixed weights (quantize.cpp:263-279)
//   k-means 8 restarts per layer type (kmeans.cu)
//   pass C  partition + nearest-centre levels + protected (pos, bf16) compaction
#include <float.h>
#include <math.h>

#include <algorithm>

#include "engine.h"
#include "hist.cuh"
#include "kmeans_api.h"
#include "quantize_api.h"

namespace dqtg {

constexpr int kPB = 256;  // threads per streaming CTA

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg((const float4*)p); }

__device__ __forceinline__ int classify(float mag, float sens, bool has_sens, int metric,
                                        const LtParams& p) {
    // quantize.cpp:82-87
    bool prot = (p.flags & kProtectAll) ||
                ((p.flags & kDoProtect) && (mag > p.t_mag || (has_sens && sens > p.t_sens)));
    if (prot) return 2;
    float ps = metric ? sens : mag;
    if ((p.flags & kDoPrune) && ps <= p.t_prune) return 1;
    return 0;
}

template <bool EXPL>
__device__ __forceinline__ void load_scores(const PassIn& a, uint64_t idx, const float4& w,
                                            float (&m)[4], float (&s)[4]) {
    if (EXPL) {
        float4 mv = ld4(a.mag + idx);
        m[0] = mv.x, m[1] = mv.y, m[2] = mv.z, m[3] = mv.w;
        if (a.has_sens) {
            float4 sv = ld4(a.sens + idx);
            s[0] = sv.x, s[1] = sv.y, s[2] = sv.z, s[3] = sv.w;
        }
    } else {
        m[0] = fabsf(w.x), m[1] = fabsf(w.y), m[2] = fabsf(w.z), m[3] = fabsf(w.w);
        if (a.has_sens) {  // ranker.cpp:96: fabs(e * w) in float
            float4 ev = ld4(a.ema + idx);
            s[0] = fabsf(__fmul_rn(ev.x, w.x)), s[1] = fabsf(__fmul_rn(ev.y, w.y));
            s[2] = fabsf(__fmul_rn(ev.z, w.z)), s[3] = fabsf(__fmul_rn(ev.w, w.w));
        }
    }
}

// ---- pass A: score histograms ----------------------------------------------
template <bool EXPL>
__global__ void __launch_bounds__(kPB) pass_a_kernel(PassIn a, unsigned long long* gh_mag,
                                                     unsigned long long* gh_sens,
                                                     uint32_t mask_mag, uint32_t mask_sens) {
    extern __shared__ uint32_t sh[];
    uint32_t* shm = sh;
    uint32_t* shs = sh + kWinSlots;
    hist_clear(shm);
    hist_clear(shs);
    __syncthreads();
    const int t0 = (int)((int64_t)blockIdx.x * a.ntiles / gridDim.x);
    const int t1 = (int)((int64_t)(blockIdx.x + 1) * a.ntiles / gridDim.x);
    int cur = -1;
    for (int ti = t0; ti < t1; ++ti) {
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        if (lt != cur) {
            __syncthreads();
            if (cur >= 0) {
                hist_flush(shm, gh_mag + cur * a.HS, a.tab);
                hist_flush(shs, gh_sens + cur * a.HS, a.tab);
            }
            __syncthreads();
            cur = lt;
        }
        const bool dm = (mask_mag >> lt) & 1, ds = (mask_sens >> lt) & 1;
        if (!dm && !ds) continue;
        for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 4) {
            const uint64_t idx = T.start + i;
            float4 wv = ld4(a.w + idx);
            float m[4], s[4];
            load_scores<EXPL>(a, idx, wv, m, s);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (i + j >= T.count) break;
                if (dm) hist_add(shm, gh_mag + lt * a.HS, m[j], a.tab, a.err);
                if (ds) hist_add(shs, gh_sens + lt * a.HS, s[j], a.tab, a.err);
            }
        }
    }
    __syncthreads();
    if (cur >= 0) {
        hist_flush(shm, gh_mag + cur * a.HS, a.tab);
        hist_flush(shs, gh_sens + cur * a.HS, a.tab);
    }
}

// ---- quantile thresholds (sketch.cpp:59-77) --------------------------------
__global__ void __launch_bounds__(1024) quantile_kernel(const QJob* jobs, int64_t HS,
                                                        const float* keyf, LtParams* lp) {
    __shared__ unsigned long long s_scan[33];
    __shared__ unsigned long long s_tot;
    __shared__ int64_t s_hit;
    const QJob J = jobs[blockIdx.x];
    unsigned long long loc = 0;
    for (int64_t i = threadIdx.x; i < HS; i += blockDim.x) loc += J.hist[i];
    unsigned long long total;
    block_exclusive_scan<unsigned long long>(loc, s_scan, &total);
    if (threadIdx.x == 0) {
        s_tot = total;
        s_hit = HS - 1;
    }
    __syncthreads();
    if (total == 0) return;  // empty sketch: rejected on the host beforehand
    unsigned long long rank =
        (unsigned long long)ceil(__dmul_rn(J.q, (double)(total - 1))) + 1ull;
    if (rank > total) rank = total;
    unsigned long long seen = 0;
    for (int64_t c0 = 0; c0 < HS; c0 += blockDim.x) {
        int64_t i = c0 + threadIdx.x;
        unsigned long long c = i < HS ? J.hist[i] : 0ull, tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(c, s_scan, &tot);
        if (c && seen + ex < rank && seen + ex + c >= rank) s_hit = i;
        __syncthreads();
        if (seen + tot >= rank) break;
        seen += tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = keyf[s_hit];
        if (J.which == 0) lp[J.lt].t_mag = t;
        else if (J.which == 1) lp[J.lt].t_sens = t;
        else lp[J.lt].t_prune = t;
    }
}

// ---- pass B: partition + QUANTIZE value histogram + protected counts --------
template <bool EXPL>
__global__ void __launch_bounds__(kPB) pass_b_kernel(PassIn a, const LtParams* lp,
                                                     unsigned long long* gh_val,
                                                     uint32_t* tile_prot,
                                                     unsigned long long* tensor_prot) {
    extern __shared__ uint32_t sh[];
    __shared__ uint32_t s_red[kPB / 32];
    hist_clear(sh);
    __syncthreads();
    const int t0 = (int)((int64_t)blockIdx.x * a.ntiles / gridDim.x);
    const int t1 = (int)((int64_t)(blockIdx.x + 1) * a.ntiles / gridDim.x);
    int cur = -1;
    LtParams P{};
    for (int ti = t0; ti < t1; ++ti) {
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        if (lt != cur) {
            __syncthreads();
            if (cur >= 0) hist_flush(sh, gh_val + cur * a.HS, a.tab);
            __syncthreads();
            cur = lt;
            P = lp[lt];
        }
        uint32_t np = 0;
        for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 4) {
            const uint64_t idx = T.start + i;
            float4 wv = ld4(a.w + idx);
            float m[4], s[4];
            load_scores<EXPL>(a, idx, wv, m, s);
            const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (i + j >= T.count) break;
                int part = classify(m[j], s[j], a.has_sens, a.metric, P);
                np += part == 2;
                if (part == 0) hist_add(sh, gh_val + lt * a.HS, wa[j], a.tab, a.err);
            }
        }
        np = warp_sum(np);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = np;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int wi = 0; wi < kPB / 32; ++wi) t += s_red[wi];
            tile_prot[ti] = t;
            if (t) atomicAdd(tensor_prot + T.tensor, (unsigned long long)t);
        }
    }
    __syncthreads();
    if (cur >= 0) hist_flush(sh, gh_val + cur * a.HS, a.tab);
}

// ---- exclusive scan of per-tile counts (single CTA) --------------------------
__global__ void __launch_bounds__(1024) scan_u32_kernel(const uint32_t* in, int n,
                                                        unsigned long long* out) {
    __shared__ unsigned long long s[33];
    unsigned long long base = 0;
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        int i = c0 + threadIdx.x;
        unsigned long long v = i < n ? in[i] : 0ull, tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(v, s, &tot);
        if (i < n) out[i] = base + ex;
        base += tot;
    }
    if (threadIdx.x == 0) out[n] = base;
}

// ---- pass C: levels + protected entries --------------------------------------
__device__ __forceinline__ uint32_t nearest_center(const float* c, uint32_t k, float v) {
    // quantize.cpp:327-335: lower_bound, then float half-gap, ties to the lower index
    uint32_t lo = 0, n = k;
    while (n > 0) {
        uint32_t h = n >> 1;
        if (c[lo + h] < v) {
            lo += h + 1;
            n -= h + 1;
        } else {
            n = h;
        }
    }
    if (lo == 0) return 0;
    if (lo == k) return k - 1;
    return (__fsub_rn(c[lo], v) < __fsub_rn(v, c[lo - 1])) ? lo : lo - 1;
}

__device__ __forceinline__ uint16_t bf16_rne(float v) {  // quantize.cpp:337-342
    uint32_t bits = __float_as_uint(v);
    bits += 0x7fffu + ((bits >> 16) & 1u);
    return (uint16_t)(bits >> 16);
}

template <bool EXPL>
__global__ void __launch_bounds__(kPB) pass_c_kernel(PassIn a, const LtParams* lp,
                                                     const float* cb, int cb_stride,
                                                     const uint32_t* cb_len,
                                                     const unsigned long long* tile_prot_off,
                                                     uint16_t* levels, uint64_t* ppos,
                                                     uint16_t* pval) {
    extern __shared__ float s_cb[];
    __shared__ unsigned long long s_scan[33];
    const int ti = blockIdx.x;
    const Tile T = a.tiles[ti];
    const int lt = a.types[T.tensor];
    const uint32_t k = cb_len[lt];
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) s_cb[j] = cb[lt * cb_stride + j];
    const LtParams P = lp[lt];
    const uint64_t tensor_base = a.tensor_off[T.tensor];
    __syncthreads();
    unsigned long long out = tile_prot_off[ti];
    for (uint32_t i0 = 0; i0 < T.count; i0 += kPB * 4) {
        const uint32_t i = i0 + threadIdx.x * 4;
        uint16_t lv[4] = {0, 0, 0, 0};
        unsigned long long flags = 0;
        float wa[4] = {0, 0, 0, 0};
        if (i < T.count) {
            const uint64_t idx = T.start + i;
            float4 wv = ld4(a.w + idx);
            float m[4], s[4];
            load_scores<EXPL>(a, idx, wv, m, s);
            wa[0] = wv.x, wa[1] = wv.y, wa[2] = wv.z, wa[3] = wv.w;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (i + j >= T.count) break;
                int part = classify(m[j], s[j], a.has_sens, a.metric, P);
                if (part == 0) lv[j] = (uint16_t)nearest_center(s_cb, k, wa[j]);
                else if (part == 1) lv[j] = (uint16_t)k;
                else {
                    lv[j] = (uint16_t)(k + 1);
                    flags |= 1ull << j;
                }
            }
            uint2 pk;
            pk.x = (uint32_t)lv[0] | ((uint32_t)lv[1] << 16);
            pk.y = (uint32_t)lv[2] | ((uint32_t)lv[3] << 16);
            *(uint2*)(levels + idx) = pk;
        }
        unsigned long long cnt = __popcll(flags), tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(cnt, s_scan, &tot);
        if (flags) {
            unsigned long long o = out + ex;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (flags >> j & 1) {
                    ppos[o] = (T.start - tensor_base) + i + j;
                    pval[o] = bf16_rne(wa[j]);
                    ++o;
                }
        }
        out += tot;
    }
}

// ---- dequantize (quantize.cpp:427-462) ----------------------------------------
__global__ void dequant_kernel(const Tile* tiles, const uint8_t* types, const uint64_t* tensor_off,
                               const float* cb, int cb_stride, const uint32_t* cb_len,
                               const uint16_t* levels, const unsigned long long* tile_prot_off,
                               const uint16_t* pval, float* out, uint32_t* err) {
    __shared__ unsigned long long s_scan[33];
    const Tile T = tiles[blockIdx.x];
    const int lt = types[T.tensor];
    const uint32_t k = cb_len[lt];
    const float* c = cb + lt * cb_stride;
    unsigned long long o = tile_prot_off[blockIdx.x];
    for (uint32_t i0 = 0; i0 < T.count; i0 += blockDim.x) {
        uint32_t i = i0 + threadIdx.x;
        uint16_t l = i < T.count ? levels[T.start + i] : 0;
        unsigned long long isp = (i < T.count && l == k + 1) ? 1ull : 0ull, tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(isp, s_scan, &tot);
        if (i < T.count) {
            float v;
            if (l < k) v = c[l];
            else if (l == k) v = 0.0f;
            else if (l == k + 1) v = __uint_as_float((uint32_t)pval[o + ex] << 16);
            else {
                atomicOr(err, kErrCorruptIndex);
                v = 0.0f;
            }
            out[T.start + i] = v;
        }
        o += tot;
    }
}

// ---- host orchestration ---------------------------------------------------------
static PassIn pass_in(Engine& e, const DevCkpt& c, const AlphaTables& T, int metric) {
    const Layout& L = *c.L;
    PassIn a{};
    a.tiles = L.d_tiles;
    a.ntiles = (int)L.tiles.size();
    a.types = L.d_types;
    a.tensor_off = L.d_off;
    a.w = c.w;
    a.ema = c.ema;
    a.mag = c.mag;
    a.sens = c.sens;
    a.has_sens = c.has_sens;
    a.metric = metric;
    a.tab = e.bucket_tab(T);
    a.HS = T.HS;
    a.err = e.d_err;
    return a;
}

static int stream_grid(Engine& e, int ntiles, int per_sm) {
    int g = e.num_sms * per_sm;
    return std::max(1, std::min(g, ntiles));
}

void quantize_plan(const Layout& L, const dqtg_config& cfg, bool has_sens, QuantPlan& plan) {
    // Validation in the reference's order (quantize.cpp:375, :35-38, :46-74).
    DQTG_REQUIRE(cfg.bins >= 1 && cfg.embed_bins >= 1, DQTG_ERROR, "bins must be >= 1");
    DQTG_REQUIRE(!(cfg.metric == 1 && !has_sens), DQTG_MISSING_SCORES,
                 "sensitivity prune metric requested without gradient history");
    plan = QuantPlan{};
    for (uint32_t i = 0; i < L.nt; ++i) {
        plan.present[L.types[i]] = true;
        plan.lt_n[L.types[i]] += L.numel[i];
    }
    const bool alpha_ok = cfg.alpha > 0.0 && cfg.alpha < 1.0;
    for (int lt = 0; lt < kLayerTypes; ++lt) {
        LtParams& p = plan.lp[lt];
        p.t_mag = p.t_sens = p.t_prune = FLT_MAX;
        p.flags = 0;
        if (!plan.present[lt]) continue;
        bool do_prune = cfg.prune_frac > 0.0 && lt != kEmbedding;
        if (do_prune) {
            DQTG_REQUIRE(alpha_ok, DQTG_ALPHA_OUT_OF_RANGE, "alpha must be in (0, 1)");
            DQTG_REQUIRE(cfg.prune_frac >= 0.0 && cfg.prune_frac <= 1.0, DQTG_ALPHA_OUT_OF_RANGE,
                         "quantile q must be in [0, 1]");
            DQTG_REQUIRE(plan.lt_n[lt] > 0, DQTG_EMPTY_SKETCH, "quantile of empty sketch");
            p.flags |= kDoPrune;
            plan.jobs.push_back(QJob{lt, 2, cfg.prune_frac, nullptr});
            if (cfg.metric == 1) plan.mask_sens |= 1u << lt;
            else plan.mask_mag |= 1u << lt;
        }
        bool do_protect = cfg.protect_frac > 0.0;
        double q_prot = 1.0 - cfg.protect_frac / 2.0;
        bool protect_all = do_protect && q_prot <= 0.0;
        if (do_protect) p.flags |= kDoProtect;
        if (protect_all) p.flags |= kProtectAll;
        if (do_protect && !protect_all) {
            DQTG_REQUIRE(alpha_ok, DQTG_ALPHA_OUT_OF_RANGE, "alpha must be in (0, 1)");
            DQTG_REQUIRE(plan.lt_n[lt] > 0, DQTG_EMPTY_SKETCH, "quantile of empty sketch");
            plan.jobs.push_back(QJob{lt, 0, q_prot, nullptr});
            plan.mask_mag |= 1u << lt;
            if (has_sens) {
                plan.jobs.push_back(QJob{lt, 1, q_prot, nullptr});
                plan.mask_sens |= 1u << lt;
            }
        }
    }
}

std::unique_ptr<QState> quantize(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                                 uint64_t seed, uint64_t step) {
    const Layout& L = *c.L;
    QuantPlan plan;
    quantize_plan(L, cfg, c.has_sens, plan);
    auto q = std::make_unique<QState>();
    q->eng = &e;
    q->L = c.L;
    q->step = step;
    q->cfg = cfg;
    const uint32_t kmax_bins = std::max(cfg.bins, cfg.embed_bins);
    q->cb_stride = kmax_bins;
    DQTG_CUDA(cudaMalloc(&q->d_levels, L.Np * 2));
    DQTG_CUDA(cudaMalloc(&q->d_cb, (size_t)kLayerTypes * kmax_bins * 4));
    q->prot_count.assign(L.nt, 0);
    q->prot_off.assign(L.nt + 1, 0);
    const int ntiles = (int)L.tiles.size();
    if (L.N == 0) {
        DQTG_CUDA(cudaMemsetAsync(q->d_levels, 0, L.Np * 2, e.stream));
        return q;
    }
    DQTG_REQUIRE(cfg.alpha > 0.0 && cfg.alpha < 1.0, DQTG_ALPHA_OUT_OF_RANGE,
                 "alpha must be in (0, 1)");
    AlphaTables& T = e.alpha_tables(cfg.alpha);
    const int64_t HS = T.HS;
    PassIn a = pass_in(e, c, T, (int)cfg.metric);
    cudaStream_t st = e.stream;

    // device parameters
    LtParams* d_lp = (LtParams*)e.buf("q.lp", sizeof(LtParams) * kLayerTypes);
    DQTG_CUDA(cudaMemcpyAsync(d_lp, plan.lp, sizeof(plan.lp), cudaMemcpyHostToDevice, st));

    // pass A + thresholds
    if (!plan.jobs.empty()) {
        auto* gh = (unsigned long long*)e.buf("q.gh_scores", (size_t)2 * kLayerTypes * HS * 8);
        DQTG_CUDA(cudaMemsetAsync(gh, 0, (size_t)2 * kLayerTypes * HS * 8, st));
        unsigned long long* gh_mag = gh;
        unsigned long long* gh_sens = gh + (size_t)kLayerTypes * HS;
        const size_t smem = (size_t)2 * kWinSlots * 4;
        int grid = stream_grid(e, ntiles, 3);
        if (c.explicit_scores) {
            DQTG_CUDA(cudaFuncSetAttribute(pass_a_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            pass_a_kernel<true><<<grid, kPB, smem, st>>>(a, gh_mag, gh_sens, plan.mask_mag,
                                                         plan.mask_sens);
        } else {
            DQTG_CUDA(cudaFuncSetAttribute(pass_a_kernel<false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            pass_a_kernel<false><<<grid, kPB, smem, st>>>(a, gh_mag, gh_sens, plan.mask_mag,
                                                          plan.mask_sens);
        }
        for (auto& j : plan.jobs) {
            bool sens_hist = (j.which == 1) || (j.which == 2 && cfg.metric == 1);
            j.hist = (sens_hist ? gh_sens : gh_mag) + (size_t)j.lt * HS;
        }
        QJob* d_jobs = (QJob*)e.buf("q.jobs", sizeof(QJob) * plan.jobs.size());
        DQTG_CUDA(cudaMemcpyAsync(d_jobs, plan.jobs.data(), sizeof(QJob) * plan.jobs.size(),
                                  cudaMemcpyHostToDevice, st));
        quantile_kernel<<<(unsigned)plan.jobs.size(), 1024, 0, st>>>(d_jobs, HS, T.d_keyf, d_lp);
        e.launched(2);
    }

    // pass B
    auto* gh_val = (unsigned long long*)e.buf("q.gh_val", (size_t)kLayerTypes * HS * 8);
    auto* tile_prot = (uint32_t*)e.buf("q.tile_prot", (size_t)ntiles * 4 + 4);
    auto* tile_off = (unsigned long long*)e.buf("q.tile_off", (size_t)(ntiles + 1) * 8);
    auto* tensor_prot = (unsigned long long*)e.buf("q.tensor_prot", (size_t)(L.nt + 1) * 8);
    DQTG_CUDA(cudaMemsetAsync(gh_val, 0, (size_t)kLayerTypes * HS * 8, st));
    DQTG_CUDA(cudaMemsetAsync(tensor_prot, 0, (size_t)(L.nt + 1) * 8, st));
    {
        const size_t smem = (size_t)kWinSlots * 4;
        int grid = stream_grid(e, ntiles, 6);
        if (c.explicit_scores)
            pass_b_kernel<true><<<grid, kPB, smem, st>>>(a, d_lp, gh_val, tile_prot, tensor_prot);
        else
            pass_b_kernel<false><<<grid, kPB, smem, st>>>(a, d_lp, gh_val, tile_prot, tensor_prot);
        scan_u32_kernel<<<1, 1024, 0, st>>>(tile_prot, ntiles, tile_off);
        e.launched(2);
    }

    // keys + weights per layer type
    auto* pts = (double*)e.buf("q.pts", (size_t)kLayerTypes * HS * 8);
    auto* kw = (double*)e.buf("q.kw", (size_t)kLayerTypes * HS * 8);
    auto* kc = (unsigned long long*)e.buf("q.kc", (size_t)kLayerTypes * HS * 8);
    auto* n_keys = (int*)e.buf("q.nkeys", kLayerTypes * 4);
    compact_keys(e, gh_val, HS, HS, T.d_key, cfg.sigma, kLayerTypes, pts, kc, kw, HS, n_keys);

    int h_nkeys[kLayerTypes];
    std::vector<unsigned long long> h_tprot(L.nt + 1);
    DQTG_CUDA(cudaMemcpyAsync(h_nkeys, n_keys, sizeof(h_nkeys), cudaMemcpyDeviceToHost, st));
    DQTG_CUDA(cudaMemcpyAsync(h_tprot.data(), tensor_prot, (L.nt + 1) * 8,
                              cudaMemcpyDeviceToHost, st));
    e.check_err();  // syncs

    auto* cb_len_d = (uint32_t*)e.buf("q.cblen", kLayerTypes * 4);
    DQTG_CUDA(cudaMemsetAsync(cb_len_d, 0, kLayerTypes * 4, st));
    std::vector<KProblem> probs;
    for (int lt = 0; lt < kLayerTypes; ++lt) {
        if (h_nkeys[lt] == 0) continue;  // no QUANTIZE values: empty codebook
        DQTG_REQUIRE(cfg.sigma >= 0.0 && cfg.sigma <= 1.0, DQTG_ERROR, "sigma must be in [0, 1]");
        const uint32_t k = lt == kEmbedding ? cfg.embed_bins : cfg.bins;
        if ((uint32_t)h_nkeys[lt] < k) {
            distinct_value_codebook(e, a, d_lp, lt, k, cfg, mix_seed(seed, (uint64_t)lt), q->d_cb,
                                    (int)q->cb_stride, cb_len_d);
            continue;
        }
        KProblem p{};
        p.pts = pts + (size_t)lt * HS;
        p.w = kw + (size_t)lt * HS;
        p.n = h_nkeys[lt];
        p.k = (int)k;
        p.seed = mix_seed(seed, (uint64_t)lt);  // quantize.cpp:393
        p.slot = lt;
        probs.push_back(p);
    }
    run_kmeans(e, probs, q->d_cb, (int)q->cb_stride, cb_len_d);

    // pass C
    q->prot_total = h_tprot[0];
    uint64_t acc = 0;
    for (uint32_t i = 0; i < L.nt; ++i) {
        q->prot_off[i] = acc;
        q->prot_count[i] = h_tprot[i];
        acc += h_tprot[i];
    }
    q->prot_off[L.nt] = acc;
    q->prot_total = acc;
    DQTG_CUDA(cudaMalloc(&q->d_ppos, (acc + 1) * 8));
    DQTG_CUDA(cudaMalloc(&q->d_pval, (acc + 1) * 2));
    {
        const size_t smem = (size_t)q->cb_stride * 4 + 16;
        if (c.explicit_scores)
            pass_c_kernel<true><<<ntiles, kPB, smem, st>>>(a, d_lp, q->d_cb, (int)q->cb_stride,
                                                           cb_len_d, tile_off, q->d_levels,
                                                           q->d_ppos, q->d_pval);
        else
            pass_c_kernel<false><<<ntiles, kPB, smem, st>>>(a, d_lp, q->d_cb, (int)q->cb_stride,
                                                            cb_len_d, tile_off, q->d_levels,
                                                            q->d_ppos, q->d_pval);
        e.launched();
        DQTG_CUDA(cudaGetLastError());
    }
    // codebooks to host
    std::vector<float> hcb((size_t)kLayerTypes * q->cb_stride);
    DQTG_CUDA(cudaMemcpyAsync(q->cb_len, cb_len_d, sizeof(q->cb_len), cudaMemcpyDeviceToHost, st));
    DQTG_CUDA(cudaMemcpyAsync(hcb.data(), q->d_cb, hcb.size() * 4, cudaMemcpyDeviceToHost, st));
    e.check_err();
    for (int lt = 0; lt < kLayerTypes; ++lt)
        q->cb[lt].assign(hcb.begin() + (size_t)lt * q->cb_stride,
                         hcb.begin() + (size_t)lt * q->cb_stride + q->cb_len[lt]);
    return q;
}

void dequantize(Engine& e, const QState& q, float* out_dev) {
    const Layout& L = *q.L;
    const int ntiles = (int)L.tiles.size();
    if (!ntiles) return;
    // per-tile protected offsets from the levels themselves
    auto* tile_prot = (uint32_t*)e.buf("dq.tile_prot", (size_t)ntiles * 4 + 4);
    auto* tile_off = (unsigned long long*)e.buf("dq.tile_off", (size_t)(ntiles + 1) * 8);
    auto* cb_len_d = (uint32_t*)e.buf("dq.cblen", kLayerTypes * 4);
    DQTG_CUDA(cudaMemcpyAsync(cb_len_d, q.cb_len, sizeof(q.cb_len), cudaMemcpyHostToDevice,
                              e.stream));
    count_protected(e, L, q.d_levels, cb_len_d, tile_prot);
    scan_u32_kernel<<<1, 1024, 0, e.stream>>>(tile_prot, ntiles, tile_off);
    dequant_kernel<<<ntiles, 256, 0, e.stream>>>(L.d_tiles, L.d_types, L.d_off, q.d_cb,
                                                 (int)q.cb_stride, cb_len_d, q.d_levels, tile_off,
                                                 q.d_pval, out_dev, e.d_err);
    e.launched(2);
    DQTG_CUDA(cudaGetLastError());
}

void scan_tiles(Engine& e, const uint32_t* in, int n, unsigned long long* out) {
    scan_u32_kernel<<<1, 1024, 0, e.stream>>>(in, n, out);
    e.launched();
}

}  // namespace dqtg
