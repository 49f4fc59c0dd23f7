#include "gpu.h"

#include <cstdlib>
#include <mutex>

#include "dqt/errors.hpp"

namespace dqt::gpu {

dqtg_engine* engine() {
    static std::once_flag once;
    static dqtg_engine* eng = nullptr;
    static dqtg_status st = DQTG_OK;
    std::call_once(once, [] {
        const char* dev = std::getenv("DQT_DEVICE");
        st = dqtg_engine_create(dev ? std::atoi(dev) : 0, nullptr, &eng);
    });
    if (st != DQTG_OK) raise(st);
    return eng;
}

void raise(dqtg_status st) {
    std::string m = dqtg_last_error();
    switch (st) {
        case DQTG_BAD_MAGIC: throw BadMagic(m);
        case DQTG_TRUNCATED: throw TruncatedFile(m);
        case DQTG_SHAPE_MISMATCH: throw ShapeMismatch(m);
        case DQTG_NON_FINITE: throw NonFiniteData(m);
        case DQTG_IO: throw IoError(m);
        case DQTG_ALPHA_OUT_OF_RANGE: throw AlphaOutOfRange(m);
        case DQTG_ALPHA_MISMATCH: throw AlphaMismatch(m);
        case DQTG_EMPTY_SKETCH: throw EmptySketch(m);
        case DQTG_MISSING_GRADIENTS: throw MissingGradients(m);
        case DQTG_MISSING_SCORES: throw MissingScores(m);
        case DQTG_TOO_FEW_DISTINCT: throw TooFewDistinctPoints(m);
        case DQTG_CORRUPT_INDEX: throw CorruptIndex(m);
        case DQTG_CORRUPT_BITSTREAM: throw CorruptBitstream(m);
        case DQTG_CHECKSUM_MISMATCH: throw ChecksumMismatch(m);
        case DQTG_CHAIN_CORRUPT: throw ChainCorrupt(m);
        case DQTG_CUDA: throw Error("CUDA: " + m);
        default: throw Error(m);
    }
}

dqtg_config to_c(const QuantConfig& c) {
    dqtg_config o{};
    o.bins = c.bins;
    o.embed_bins = c.embed_bins;
    o.prune_frac = c.prune_frac;
    o.protect_frac = c.protect_frac;
    o.metric = uint32_t(c.metric);
    o.sigma = c.sigma;
    o.alpha = c.alpha;
    return o;
}

QuantConfig from_c(const dqtg_config& c) {
    QuantConfig o;
    o.bins = c.bins;
    o.embed_bins = c.embed_bins;
    o.prune_frac = c.prune_frac;
    o.protect_frac = c.protect_frac;
    o.metric = PruneMetric(c.metric);
    o.sigma = c.sigma;
    o.alpha = c.alpha;
    return o;
}

std::unique_ptr<CkptHandle> upload_checkpoint(const Checkpoint& c,
                                              const std::vector<std::vector<float>>* mag,
                                              const std::vector<std::vector<float>>* sens) {
    for (const auto& t : c.tensors)
        if (t.data.size() != t.size())
            throw ShapeMismatch("tensor " + t.name + " has " + std::to_string(t.data.size()) +
                                " elements, shape implies " + std::to_string(t.size()));
    LayoutView lv(c.tensors);
    auto h = std::make_unique<CkptHandle>();
    check(dqtg_ckpt_create(engine(), &lv.c, &h->h));
    std::vector<const float*> ptrs;
    for (const auto& t : c.tensors) ptrs.push_back(t.data.data());
    check(dqtg_ckpt_set_weights(h->h, ptrs.data()));
    if (mag) {
        std::vector<const float*> mp, sp;
        for (size_t i = 0; i < mag->size(); ++i) {
            if ((*mag)[i].size() != c.tensors[i].data.size())
                throw MissingScores("score set does not match checkpoint");
            mp.push_back((*mag)[i].data());
        }
        if (sens)
            for (size_t i = 0; i < sens->size(); ++i) {
                if ((*sens)[i].size() != c.tensors[i].data.size())
                    throw MissingScores("score set does not match checkpoint");
                sp.push_back((*sens)[i].data());
            }
        check(dqtg_ckpt_set_scores(h->h, mp.data(), sens ? sp.data() : nullptr));
    }
    return h;
}

StateHandle upload_state(const QuantizedCheckpoint& q) {
    LayoutView lv(q.tensors);
    dqtg_config cfg = to_c(q.config);
    uint32_t cbl[kLayerTypeCount];
    const float* cbs[kLayerTypeCount];
    for (int lt = 0; lt < kLayerTypeCount; ++lt) {
        cbl[lt] = uint32_t(q.codebooks[lt].size());
        cbs[lt] = q.codebooks[lt].data();
    }
    std::vector<const uint16_t*> levels;
    std::vector<uint64_t> counts;
    std::vector<std::vector<uint64_t>> pos(q.tensors.size());
    std::vector<std::vector<uint16_t>> val(q.tensors.size());
    std::vector<const uint64_t*> pp;
    std::vector<const uint16_t*> pv;
    for (size_t i = 0; i < q.tensors.size(); ++i) {
        const auto& t = q.tensors[i];
        if (t.levels.size() != t.size())
            throw ShapeMismatch("level count does not match shape of " + t.name);
        levels.push_back(t.levels.data());
        counts.push_back(t.protected_values.size());
        for (const auto& e : t.protected_values) {
            pos[i].push_back(e.pos);
            val[i].push_back(e.value);
        }
        pp.push_back(pos[i].data());
        pv.push_back(val[i].data());
    }
    StateHandle s;
    check(dqtg_qstate_upload(engine(), &lv.c, q.step, &cfg, cbl, cbs, levels.data(), counts.data(),
                             pp.data(), pv.data(), &s.h));
    return s;
}

QuantizedCheckpoint download_state_layout(dqtg_qstate* s, const std::vector<std::string>& names,
                                          const std::vector<LayerType>& types,
                                          const std::vector<std::vector<uint64_t>>& shapes) {
    dqtg_qstate_info info{};
    check(dqtg_qstate_info_get(s, &info));
    QuantizedCheckpoint q;
    q.step = info.step;
    q.config = from_c(info.config);
    const size_t nt = names.size();
    std::vector<uint64_t> counts(nt);
    if (nt) check(dqtg_qstate_protected_counts(s, counts.data()));
    q.tensors.resize(nt);
    std::vector<uint16_t*> lv(nt);
    std::vector<std::vector<uint64_t>> pos(nt);
    std::vector<std::vector<uint16_t>> val(nt);
    std::vector<uint64_t*> pp(nt);
    std::vector<uint16_t*> pv(nt);
    for (size_t i = 0; i < nt; ++i) {
        auto& t = q.tensors[i];
        t.name = names[i];
        t.type = types[i];
        t.shape = shapes[i];
        t.levels.resize(t.size());
        lv[i] = t.levels.data();
        pos[i].resize(counts[i]);
        val[i].resize(counts[i]);
        pp[i] = pos[i].data();
        pv[i] = val[i].data();
    }
    float* cbp[kLayerTypeCount];
    for (int lt = 0; lt < kLayerTypeCount; ++lt) {
        q.codebooks[lt].resize(info.codebook_len[lt]);
        cbp[lt] = q.codebooks[lt].data();
    }
    check(dqtg_qstate_download(s, lv.data(), pp.data(), pv.data(), cbp));
    for (size_t i = 0; i < nt; ++i) {
        auto& pe = q.tensors[i].protected_values;
        pe.resize(counts[i]);
        for (size_t j = 0; j < counts[i]; ++j) pe[j] = ProtectedEntry{pos[i][j], val[i][j]};
    }
    return q;
}

QuantizedCheckpoint download_state(dqtg_qstate* s, const std::vector<QuantizedTensor>& src) {
    std::vector<std::string> names;
    std::vector<LayerType> types;
    std::vector<std::vector<uint64_t>> shapes;
    for (const auto& t : src) {
        names.push_back(t.name);
        types.push_back(t.type);
        shapes.push_back(t.shape);
    }
    return download_state_layout(s, names, types, shapes);
}

}  // namespace dqt::gpu
