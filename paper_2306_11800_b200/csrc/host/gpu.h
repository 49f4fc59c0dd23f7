// Bridge from the value-semantic dqt API to the B200 engine C ABI (dqtg.h).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "dqt/quantize.hpp"
#include "dqtg.h"

namespace dqt::gpu {

dqtg_engine* engine();           // process-wide engine on $DQT_DEVICE (default 0)
[[noreturn]] void raise(dqtg_status st);  // rethrow as the matching dqt:: exception
inline void check(dqtg_status st) {
    if (st != DQTG_OK) raise(st);
}

dqtg_config to_c(const QuantConfig& c);
QuantConfig from_c(const dqtg_config& c);

// Keeps the arrays a dqtg_layout points into alive.
struct LayoutView {
    std::vector<const char*> names;
    std::vector<uint8_t> types, ranks;
    std::vector<uint64_t> dims;
    dqtg_layout c{};
    template <typename T>
    explicit LayoutView(const std::vector<T>& tensors) {
        for (const auto& t : tensors) {
            names.push_back(t.name.c_str());
            types.push_back(uint8_t(t.type));
            ranks.push_back(uint8_t(t.shape.size()));
            dims.insert(dims.end(), t.shape.begin(), t.shape.end());
        }
        c.n_tensors = uint32_t(tensors.size());
        c.names = names.data();
        c.types = types.data();
        c.ranks = ranks.data();
        c.dims = dims.data();
    }
};

struct CkptHandle {
    dqtg_ckpt* h = nullptr;
    CkptHandle() = default;
    CkptHandle(const CkptHandle&) = delete;
    ~CkptHandle() {
        if (h) dqtg_ckpt_destroy(h);
    }
};
struct StateHandle {
    dqtg_qstate* h = nullptr;
    StateHandle() = default;
    StateHandle(const StateHandle&) = delete;
    StateHandle(StateHandle&& o) noexcept : h(o.h) { o.h = nullptr; }
    StateHandle& operator=(StateHandle&& o) noexcept {
        std::swap(h, o.h);
        return *this;
    }
    ~StateHandle() {
        if (h) dqtg_qstate_destroy(h);
    }
};

// Upload weights (and explicit scores when given) of a checkpoint.
std::unique_ptr<CkptHandle> upload_checkpoint(const Checkpoint& c,
                                              const std::vector<std::vector<float>>* mag,
                                              const std::vector<std::vector<float>>* sens);
StateHandle upload_state(const QuantizedCheckpoint& q);
QuantizedCheckpoint download_state(dqtg_qstate* s, const std::vector<QuantizedTensor>& shape_src);
QuantizedCheckpoint download_state_layout(dqtg_qstate* s, const std::vector<std::string>& names,
                                          const std::vector<LayerType>& types,
                                          const std::vector<std::vector<uint64_t>>& shapes);

}  // namespace dqt::gpu
