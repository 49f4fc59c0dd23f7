// Quantizer API (reference src/quantize.cpp).  partition_params,
// quantize_checkpoint, dequantize_checkpoint, approx_kmeans and the k-means
// primitives execute on the B200 engine; this file converts value types.
#include "dqt/quantize.hpp"

#include <algorithm>
#include <cstring>

#include "dqtg.h"
#include "gpu.h"

namespace dqt {

uint64_t mix_seed(uint64_t seed, uint64_t salt) {  // splitmix64 finaliser
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

uint64_t PartitionMasks::count(Part p) const {
    uint64_t n = 0;
    for (const auto& v : part) n += uint64_t(std::count(v.begin(), v.end(), uint8_t(p)));
    return n;
}

static void check_scores(const Checkpoint& c, const ScoreSet& s, const QuantConfig& cfg) {
    if (s.magnitude.size() != c.tensors.size())
        throw MissingScores("score set does not match checkpoint");
    if (cfg.metric == PruneMetric::Sensitivity && !s.has_sensitivity)
        throw MissingScores("sensitivity prune metric requested without gradient history");
    if (s.has_sensitivity && s.sensitivity.size() != c.tensors.size())
        throw MissingScores("score set does not match checkpoint");
}

PartitionMasks partition_params(const Checkpoint& c, const ScoreSet& s, const QuantConfig& cfg) {
    check_scores(c, s, cfg);
    auto ck = gpu::upload_checkpoint(c, &s.magnitude, s.has_sensitivity ? &s.sensitivity : nullptr);
    PartitionMasks m;
    m.part.resize(c.tensors.size());
    std::vector<uint8_t*> ptrs;
    for (size_t i = 0; i < c.tensors.size(); ++i) {
        m.part[i].resize(c.tensors[i].data.size());
        ptrs.push_back(m.part[i].data());
    }
    dqtg_config cc = gpu::to_c(cfg);
    gpu::check(dqtg_partition(gpu::engine(), ck->h, &cc, ptrs.data()));
    return m;
}

std::vector<double> weighted_kmeanspp_init(const std::vector<double>& points,
                                           const std::vector<double>& weights, uint32_t k,
                                           uint64_t seed) {
    if (k == 0) throw Error("k must be >= 1");
    if (weights.size() != points.size()) throw Error("points/weights size mismatch");
    std::vector<double> out(k);
    gpu::check(dqtg_kmeanspp_init(gpu::engine(), points.data(), weights.data(), points.size(), k,
                                  seed, out.data()));
    return out;
}

LloydResult weighted_lloyd(const std::vector<double>& points, const std::vector<double>& weights,
                           std::vector<double> centers, double tol, uint32_t max_iter) {
    if (centers.empty()) throw Error("no initial centers");
    if (weights.size() != points.size()) throw Error("points/weights size mismatch");
    LloydResult r;
    gpu::check(dqtg_lloyd(gpu::engine(), points.data(), weights.data(), points.size(),
                          centers.data(), uint32_t(centers.size()), tol, max_iter, &r.iterations));
    r.centers = std::move(centers);
    return r;
}

double weighted_sq_loss(const std::vector<double>& points, const std::vector<double>& weights,
                        const std::vector<double>& centers) {
    double loss = 0.0;
    gpu::check(dqtg_sq_loss(gpu::engine(), points.data(), weights.data(), points.size(),
                            centers.data(), uint32_t(centers.size()), &loss));
    return loss;
}

std::vector<float> approx_kmeans(const std::vector<float>& values, uint32_t k, double sigma,
                                 double alpha, uint64_t seed) {
    if (k == 0) throw Error("k must be >= 1");
    std::vector<float> cb(k);
    uint32_t len = 0;
    gpu::check(dqtg_approx_kmeans(gpu::engine(), values.data(), values.size(), k, sigma, alpha,
                                  seed, cb.data(), &len));
    cb.resize(len);
    return cb;
}

uint32_t nearest_center(const std::vector<float>& c, float v) {
    auto it = std::lower_bound(c.begin(), c.end(), v);
    if (it == c.begin()) return 0;
    if (it == c.end()) return uint32_t(c.size() - 1);
    uint32_t hi = uint32_t(it - c.begin()), lo = hi - 1;
    return (c[hi] - v < v - c[lo]) ? hi : lo;  // tie -> lower index
}

uint16_t bf16_from_f32(float v) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    return uint16_t((b + 0x7fffu + ((b >> 16) & 1u)) >> 16);
}

float bf16_to_f32(uint16_t v) {
    uint32_t b = uint32_t(v) << 16;
    float f;
    std::memcpy(&f, &b, 4);
    return f;
}

uint64_t QuantizedTensor::size() const {
    uint64_t n = 1;
    for (uint64_t d : shape) n *= d;
    return n;
}

uint32_t QuantizedCheckpoint::levels_for(LayerType t) const {
    return uint32_t(codebooks[size_t(t)].size()) + 2;
}

uint32_t QuantizedCheckpoint::max_levels() const {
    uint32_t m = 0;
    for (const auto& t : tensors) m = std::max(m, levels_for(t.type));
    return m;
}

uint64_t QuantizedCheckpoint::param_count() const {
    uint64_t n = 0;
    for (const auto& t : tensors) n += t.size();
    return n;
}

QuantizedCheckpoint quantize_checkpoint(const Checkpoint& c, const ScoreSet& s,
                                        const QuantConfig& cfg, uint64_t seed) {
    if (cfg.bins < 1 || cfg.embed_bins < 1) throw Error("bins must be >= 1");
    check_scores(c, s, cfg);
    auto ck = gpu::upload_checkpoint(c, &s.magnitude, s.has_sensitivity ? &s.sensitivity : nullptr);
    gpu::StateHandle st;
    dqtg_config cc = gpu::to_c(cfg);
    gpu::check(dqtg_quantize(gpu::engine(), ck->h, &cc, seed, c.step, &st.h));
    std::vector<std::string> names;
    std::vector<LayerType> types;
    std::vector<std::vector<uint64_t>> shapes;
    for (const auto& t : c.tensors) {
        names.push_back(t.name);
        types.push_back(t.type);
        shapes.push_back(t.shape);
    }
    return gpu::download_state_layout(st.h, names, types, shapes);
}

Checkpoint dequantize_checkpoint(const QuantizedCheckpoint& q) {
    auto st = gpu::upload_state(q);
    Checkpoint c;
    c.step = q.step;
    std::vector<float*> outs;
    c.tensors.resize(q.tensors.size());
    for (size_t i = 0; i < q.tensors.size(); ++i) {
        auto& t = c.tensors[i];
        t.name = q.tensors[i].name;
        t.type = q.tensors[i].type;
        t.shape = q.tensors[i].shape;
        t.data.resize(q.tensors[i].levels.size());
        outs.push_back(t.data.data());
    }
    gpu::check(dqtg_dequantize(gpu::engine(), st.h, outs.data()));
    return c;
}

}  // namespace dqt
