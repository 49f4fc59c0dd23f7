// Shared types of the quantize pipeline (quantize.cu, fallback.cu, eval.cu).
#pragma once

#include <vector>

#include "engine.h"

namespace dqtg {

enum LtFlags : uint32_t { kDoPrune = 1, kDoProtect = 2, kProtectAll = 4 };

// Per-layer-type partition parameters; thresholds are the float round-down of
// the reference's double quantiles so float>double compares are preserved.
struct LtParams {
    float t_mag, t_sens, t_prune;
    uint32_t flags;
};

// One quantile (sketch.cpp:59-77): which = 0 magnitude-protect, 1 sensitivity-
// protect, 2 prune (metric histogram).
struct QJob {
    int lt;
    int which;
    double q;
    const unsigned long long* hist;
};

struct PassIn {
    const Tile* tiles;
    int ntiles;
    const uint8_t* types;
    const uint64_t* tensor_off;
    const float* w;
    const float* ema;
    const float* mag;
    const float* sens;
    int has_sens;
    int metric;
    BucketTab tab;
    int64_t HS;
    uint32_t* err;
    unsigned int* tile_ctr;  // dynamic tile scheduling of persistent passes (zeroed per launch)
};

struct QuantPlan {
    bool present[kLayerTypes] = {false};
    uint64_t lt_n[kLayerTypes] = {0};
    LtParams lp[kLayerTypes];
    std::vector<QJob> jobs;
    uint32_t mask_mag = 0, mask_sens = 0;
};

void quantize_plan(const Layout& L, const dqtg_config& cfg, bool has_sens, QuantPlan& plan);

inline uint64_t mix_seed(uint64_t seed, uint64_t salt) {  // quantize.cpp:13-18
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// Distinct-value fallback of approx_kmeans (quantize.cpp:280-300) for a layer
// type whose QUANTIZE values occupy fewer than k sketch buckets.
void distinct_value_codebook(Engine& e, const PassIn& a, const LtParams* d_lp, int lt, uint32_t k,
                             const dqtg_config& cfg, uint64_t seed, float* cb, int cb_stride,
                             uint32_t* cb_len_dev);
// Same fallback for an explicit value array (dqtg_approx_kmeans).
void distinct_value_codebook_array(Engine& e, const float* vals_dev, uint64_t n, uint32_t k,
                                   double sigma, uint64_t seed, float* cb, uint32_t* cb_len_dev);
void count_protected(Engine& e, const Layout& L, const uint16_t* levels, const uint32_t* cb_len,
                     uint32_t* tile_prot);
void scan_tiles(Engine& e, const uint32_t* in, int n, unsigned long long* out);

}  // namespace dqtg
