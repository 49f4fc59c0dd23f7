// TEST INFRASTRUCTURE ONLY (never linked into the product): C entry points into the
// reference library compiled from its sources (oracle/_ref, namespace renamed to
// dqtref by -Ddqt=dqtref) for functions its Python module does not bind.
//   ref_payload_bytes: payload_bytes_pe / _rle / _he (src/codec.cpp:615-646) of two
//   states given as plain arrays (levels per tensor, layer types, codebook lengths).
#include <cstdint>
#include <string>

#include "dqt/codec.hpp"
#include "dqt/quantize.hpp"

namespace {

dqt::QuantizedCheckpoint make_state(uint32_t nt, const uint8_t* types, const uint64_t* numel,
                                    const uint16_t* const* levels, const uint32_t* cb_len) {
    dqt::QuantizedCheckpoint q;
    for (int lt = 0; lt < dqt::kLayerTypeCount; ++lt) q.codebooks[lt].assign(cb_len[lt], 0.0f);
    for (uint32_t i = 0; i < nt; ++i) {
        dqt::QuantizedTensor t;
        t.name = "t" + std::to_string(i);
        t.type = dqt::LayerType(types[i]);
        t.shape = {numel[i]};
        t.levels.assign(levels[i], levels[i] + numel[i]);
        q.tensors.push_back(std::move(t));
    }
    return q;
}

}  // namespace

extern "C" uint64_t ref_payload_bytes(int variant, uint32_t nt, const uint8_t* types,
                                      const uint64_t* numel, const uint16_t* const* base_levels,
                                      const uint32_t* base_cb_len,
                                      const uint16_t* const* target_levels,
                                      const uint32_t* target_cb_len) {
    const auto b = make_state(nt, types, numel, base_levels, base_cb_len);
    const auto t = make_state(nt, types, numel, target_levels, target_cb_len);
    if (variant == 0) return dqt::payload_bytes_pe(b, t);
    if (variant == 1) return dqt::payload_bytes_rle(b, t);
    return dqt::payload_bytes_he(b, t);
}
