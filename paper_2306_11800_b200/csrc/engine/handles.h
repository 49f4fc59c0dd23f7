// Opaque C-ABI handles (include/dqtg.h) shared by the C entry points.
#pragma once

#include <memory>
#include <string>

#include "engine.h"

struct dqtg_engine {
    dqtg::Engine e;
};
struct dqtg_ckpt {
    dqtg::DevCkpt c;
};
struct dqtg_qstate {
    std::unique_ptr<dqtg::QState> q;
};
struct dqtg_record {
    std::unique_ptr<dqtg::Record> r;
};

namespace dqtg {
void init_engine(Engine& e, int device, void* stream);  // device check, stream, pool (capi.cu)
void set_last_error(const std::string& m);             // dqtg_last_error() of this thread
}  // namespace dqtg
