// extern "C" surface of libdqtg.so (include/dqtg.h).  Every entry point catches
// internal failures and turns them into a dqtg_status + thread-local message.
#include <cstdlib>
#include <exception>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "engine.h"
#include "kmeans_api.h"
#include "quantize_api.h"

using namespace dqtg;

#include "handles.h"

static thread_local std::string g_err;

namespace dqtg {
void set_last_error(const std::string& m) { g_err = m; }
}

template <typename F>
static dqtg_status guard(F&& f) {
    try {
        f();
        return DQTG_OK;
    } catch (const Fail& x) {
        g_err = x.what();
        return x.code;
    } catch (const std::exception& x) {
        g_err = x.what();
        return DQTG_ERROR;
    } catch (...) {
        g_err = "unknown failure";
        return DQTG_ERROR;
    }
}

// Engine lock for one API call; a call that unwinds with an exception drops the
// engine's pending staged read-backs (their host destinations are gone).
struct EngineCall {
    Engine* e;
    std::lock_guard<std::recursive_mutex> lk;
    int exc;
    explicit EngineCall(Engine* eng) : e(eng), lk(eng->mu), exc(std::uncaught_exceptions()) {}
    ~EngineCall() {
        if (std::uncaught_exceptions() > exc) {
            cudaStreamSynchronize(e->stream);
            e->pend.clear();
        }
    }
};
#define LOCK(eng)              \
    EngineCall lk_((eng));     \
    (eng)->activate()

namespace dqtg {
void init_engine(Engine& e, int device, void* stream) {
    e.device = device;
    DQTG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    DQTG_CUDA(cudaGetDeviceProperties(&prop, device));
    DQTG_REQUIRE(prop.major >= 10, DQTG_CUDA,
                 "dqtg needs a Blackwell (sm_100) device; found " + std::string(prop.name));
    e.num_sms = prop.multiProcessorCount;
    if (stream) {
        e.stream = (cudaStream_t)stream;
    } else {
        DQTG_CUDA(cudaStreamCreateWithFlags(&e.stream, cudaStreamNonBlocking));
        e.own_stream = true;
    }
    DQTG_CUDA(cudaMalloc(&e.d_err, 16));
    // a private stream-ordered pool per engine; freed memory stays cached (per-step
    // states/records reuse it) and is never handed to another engine's stream (the
    // default pool's cross-stream reuse inserts waits on other engines' streams)
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    DQTG_CUDA(cudaMemPoolCreate(&e.pool, &props));
    uint64_t keep = ~0ull;
    DQTG_CUDA(cudaMemPoolSetAttribute(e.pool, cudaMemPoolAttrReleaseThreshold, &keep));
    int no = 0;
    DQTG_CUDA(cudaMemPoolSetAttribute(e.pool, cudaMemPoolReuseAllowInternalDependencies, &no));
    register_pool(e.pool, device);
    DQTG_CUDA(cudaMemsetAsync(e.d_err, 0, 16, e.stream));
    DQTG_CUDA(cudaStreamSynchronize(e.stream));
}
}  // namespace dqtg

extern "C" {

const char* dqtg_last_error(void) { return g_err.c_str(); }
const char* dqtg_version(void) { return "dqtg 0.1 sm_100a"; }

dqtg_status dqtg_engine_create(int device, void* stream, dqtg_engine** out) {
    return guard([&] {
        auto* h = new dqtg_engine();
        try {
            init_engine(h->e, device, stream);
        } catch (...) {
            delete h;
            throw;
        }
        h->e.owner = h;
        h->e.deleter = [](void* o) { delete static_cast<dqtg_engine*>(o); };
        *out = h;
    });
}

// drops the caller's reference; checkpoints/states/records still alive keep the
// engine until they are destroyed
void dqtg_engine_destroy(dqtg_engine* h) {
    if (h) engine_release(&h->e);
}

dqtg_status dqtg_engine_sync(dqtg_engine* h) {
    return guard([&] {
        LOCK(&h->e);
        h->e.sync();
    });
}

uint64_t dqtg_engine_launches(const dqtg_engine* h) { return h->e.launches; }


dqtg_status dqtg_engine_profile(dqtg_engine* h, int enable) {
    return guard([&] {
        LOCK(&h->e);
        h->e.profiling = enable != 0;
        if (enable) timeline_epoch(h->e);
    });
}

void dqtg_engine_sync_stats(const dqtg_engine* h, uint64_t* syncs, double* blocked_ms) {
    if (syncs) *syncs = h->e.sync_n;
    if (blocked_ms) *blocked_ms = 1e-6 * (double)h->e.sync_ns;
}

dqtg_status dqtg_engine_profile_report(dqtg_engine* h, char* json, uint64_t cap) {
    return guard([&] {
        LOCK(&h->e);
        Engine& e = h->e;
        e.sync();
        std::vector<std::pair<std::string, std::pair<uint64_t, double>>> acc;
        if (getenv("DQTG_TIMELINE")) dump_timeline(e);  // per-launch start/end (ms) on stderr
        for (auto& s : e.spans) {
            float ms = 0.0f;
            DQTG_CUDA(cudaEventElapsedTime(&ms, s.a, s.b));
            auto it = std::find_if(acc.begin(), acc.end(),
                                   [&](const auto& kv) { return kv.first == s.name; });
            if (it == acc.end()) acc.push_back({s.name, {1, ms}});
            else {
                it->second.first++;
                it->second.second += ms;
            }
        }
        std::string out = "{";
        for (size_t i = 0; i < acc.size(); ++i) {
            char b[256];
            snprintf(b, sizeof(b), "%s\"%s\": [%llu, %.6f]", i ? ", " : "", acc[i].first.c_str(),
                     (unsigned long long)acc[i].second.first, acc[i].second.second);
            out += b;
        }
        out += "}";
        e.spans.clear();
        e.ev_used = 0;
        DQTG_REQUIRE(out.size() + 1 <= cap, DQTG_ERROR, "profile buffer too small");
        memcpy(json, out.c_str(), out.size() + 1);
    });
}

dqtg_status dqtg_sketch_range(double alpha, int64_t* kmin, int64_t* kmax) {
    return guard([&] {
        // host-only: same rule as the alpha tables
        DQTG_REQUIRE(alpha > 0.0 && alpha < 1.0, DQTG_ALPHA_OUT_OF_RANGE, "alpha must be in (0, 1)");
        Engine tmp;  // never touches the device for range queries
        (void)tmp;
        double g = (1.0 + alpha) / (1.0 - alpha), inv = 1.0 / log(g);
        auto bucket = [&](double ax) {
            double r = log(ax) * inv;
            double nearest = nearbyint(r);
            if (fabs(r - nearest) > 1e-9 * fmax(1.0, fabs(r))) return (int64_t)ceil(r);
            int64_t k = (int64_t)nearest;
            while (pow(g, (double)(k - 1)) >= ax) --k;
            while (pow(g, (double)k) < ax) ++k;
            return k;
        };
        float zf = (float)1e-12;
        if ((double)zf < 1e-12) zf = nextafterf(zf, INFINITY);
        *kmin = bucket((double)zf);
        *kmax = bucket((double)3.4028234663852886e38);
    });
}

dqtg_status dqtg_sketch_build(dqtg_engine* h, const float* x, uint64_t n, double alpha,
                              uint64_t* zero, uint64_t* pos, uint64_t* neg) {
    return guard([&] {
        LOCK(&h->e);
        sketch_build(h->e, x, n, alpha, zero, pos, neg);
    });
}

dqtg_status dqtg_ema_update(dqtg_engine* h, float* ema, const float* g, uint64_t n, double beta) {
    return guard([&] {
        LOCK(&h->e);
        Engine& e = h->e;
        const bool de = is_device_ptr(ema);
        float* d_e = de ? ema : (float*)e.buf("api.ema", n * 4 + 4);
        float* d_g = (float*)e.buf("api.g", n * 4 + 4);
        if (!de) e.to_device(d_e, ema, n * 4);
        e.to_device(d_g, g, n * 4);
        ::dqtg::ema_update(e, d_e, d_g, n, (float)beta);
        if (!de) e.from_device(ema, d_e, n * 4);
        e.sync();
    });
}

dqtg_status dqtg_compute_scores(dqtg_engine* h, const float* w, const float* ema, uint64_t n,
                                float* mag, float* sens) {
    return guard([&] {
        LOCK(&h->e);
        Engine& e = h->e;
        float* d_w = (float*)e.buf("api.w", n * 4 + 4);
        float* d_e = ema ? (float*)e.buf("api.ema", n * 4 + 4) : nullptr;
        float* d_m = mag ? (float*)e.buf("api.mag", n * 4 + 4) : nullptr;
        float* d_s = sens ? (float*)e.buf("api.sens", n * 4 + 4) : nullptr;
        e.to_device(d_w, w, n * 4);
        if (ema) e.to_device(d_e, ema, n * 4);
        ::dqtg::compute_scores(e, d_w, d_e, n, d_m, (ema && sens) ? d_s : nullptr);
        if (mag) e.from_device(mag, d_m, n * 4);
        if (sens && ema) e.from_device(sens, d_s, n * 4);
        e.sync();
    });
}

// ---- checkpoints ---------------------------------------------------------------
dqtg_status dqtg_ckpt_create(dqtg_engine* h, const dqtg_layout* layout, dqtg_ckpt** out) {
    return guard([&] {
        LOCK(&h->e);
        auto* c = new dqtg_ckpt();
        try {
            c->c.eng = &h->e;
            c->c.L = make_layout(&h->e, layout);
            DQTG_CUDA(dev_malloc((void**)&c->c.w, c->c.L->Np * 4, h->e.device));
            // on the engine stream: a legacy-stream memset is not ordered with the
            // (non-blocking) engine stream's uploads
            DQTG_CUDA(cudaMemsetAsync(c->c.w, 0, c->c.L->Np * 4, h->e.stream));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void dqtg_ckpt_destroy(dqtg_ckpt* c) { delete c; }

static void upload_tensors(Engine& e, const Layout& L, float* dst, const float* const* src) {
    // merged while sources and padded destinations are both contiguous (pipe.cu upload)
    uint32_t i = 0;
    while (i < L.nt) {
        uint32_t j = i + 1;
        uint64_t n = L.numel[i];
        while (j < L.nt && src[j] == src[i] + n && L.off[j] == L.off[i] + n) n += L.numel[j++];
        if (n) e.to_device(dst + L.off[i], src[i], n * 4);
        i = j;
    }
}

static float* alloc_padded(Engine& e, const Layout& L) {
    float* p = nullptr;
    DQTG_CUDA(dev_malloc((void**)&p, L.Np * 4, e.device));
    DQTG_CUDA(cudaMemsetAsync(p, 0, L.Np * 4, e.stream));  // ordered before the uploads
    return p;
}

dqtg_status dqtg_ckpt_set_weights(dqtg_ckpt* c, const float* const* t) {
    return guard([&] {
        LOCK(c->c.eng);
        if (!c->c.w) c->c.w = alloc_padded(*c->c.eng, *c->c.L);  // after dqtg_ckpt_release
        upload_tensors(*c->c.eng, *c->c.L, c->c.w, t);
        c->c.eng->sync();
    });
}

dqtg_status dqtg_ckpt_release(dqtg_ckpt* c) {
    return guard([&] {
        LOCK(c->c.eng);
        DevCkpt& d = c->c;
        DQTG_REQUIRE(d.own, DQTG_ERROR, "checkpoint buffers are borrowed");
        d.eng->sync();
        for (float** p : {&d.w, &d.ema, &d.mag, &d.sens}) {
            if (*p) cudaFree(*p);
            *p = nullptr;
        }
        d.explicit_scores = d.has_sens = d.ema_seeded = false;
    });
}

dqtg_status dqtg_ckpt_set_scores(dqtg_ckpt* c, const float* const* mag, const float* const* sens) {
    return guard([&] {
        LOCK(c->c.eng);
        DevCkpt& d = c->c;
        if (!d.mag) d.mag = alloc_padded(*d.eng, *d.L);
        upload_tensors(*d.eng, *d.L, d.mag, mag);
        if (sens) {
            if (!d.sens) d.sens = alloc_padded(*d.eng, *d.L);
            upload_tensors(*d.eng, *d.L, d.sens, sens);
        }
        d.explicit_scores = true;
        d.has_sens = sens != nullptr;
        d.eng->sync();
    });
}

dqtg_status dqtg_ckpt_set_ema(dqtg_ckpt* c, const float* const* ema) {
    return guard([&] {
        LOCK(c->c.eng);
        DevCkpt& d = c->c;
        d.explicit_scores = false;
        if (ema) {
            if (!d.ema) d.ema = alloc_padded(*d.eng, *d.L);
            upload_tensors(*d.eng, *d.L, d.ema, ema);
            d.has_sens = true;
            d.ema_seeded = true;
        } else {
            d.has_sens = false;
        }
        d.eng->sync();
    });
}

dqtg_status dqtg_ckpt_update_ema(dqtg_ckpt* c, const float* const* grads, double beta) {
    return guard([&] {
        LOCK(c->c.eng);
        DevCkpt& d = c->c;
        Engine& e = *d.eng;
        if (!d.ema) d.ema = alloc_padded(*d.eng, *d.L);
        if (!d.ema_seeded) {  // first snapshot seeds the average (ranker.cpp:22-23)
            upload_tensors(e, *d.L, d.ema, grads);
            d.ema_seeded = true;
        } else {
            float* g = (float*)e.buf("ck.g", d.L->Np * 4);
            upload_tensors(e, *d.L, g, grads);
            ::dqtg::ema_update(e, d.ema, g, d.L->Np, (float)beta);
        }
        d.explicit_scores = false;
        d.has_sens = true;
        e.sync();
    });
}

uint64_t dqtg_ckpt_param_count(const dqtg_ckpt* c) { return c->c.L->N; }
float* dqtg_ckpt_weights_dev(dqtg_ckpt* c) { return c->c.w; }
float* dqtg_ckpt_ema_dev(dqtg_ckpt* c) {
    if (!c->c.ema) {
        c->c.ema = alloc_padded(*c->c.eng, *c->c.L);
        c->c.has_sens = true;
        c->c.ema_seeded = true;
        c->c.explicit_scores = false;
    }
    return c->c.ema;
}
uint64_t dqtg_ckpt_tensor_offset(const dqtg_ckpt* c, uint32_t i) { return c->c.L->off[i]; }

// ---- quantize / states ------------------------------------------------------------
dqtg_status dqtg_quantize(dqtg_engine* h, const dqtg_ckpt* c, const dqtg_config* cfg,
                          uint64_t seed, uint64_t step, dqtg_qstate** out) {
    return guard([&] {
        LOCK(&h->e);
        auto q = ::dqtg::quantize(h->e, c->c, *cfg, seed, step);
        auto* s = new dqtg_qstate();
        s->q = std::move(q);
        *out = s;
    });
}

dqtg_status dqtg_qstate_info_get(const dqtg_qstate* s, dqtg_qstate_info* info) {
    return guard([&] {
        const QState& q = *s->q;
        info->step = q.step;
        info->config = q.cfg;
        for (int lt = 0; lt < kLayerTypes; ++lt) info->codebook_len[lt] = q.cb_len[lt];
        info->max_levels = q.max_levels();
        info->param_count = q.L->N;
        info->protected_total = q.prot_total;
    });
}

dqtg_status dqtg_qstate_protected_counts(const dqtg_qstate* s, uint64_t* counts) {
    return guard([&] {
        for (uint32_t i = 0; i < s->q->L->nt; ++i) counts[i] = s->q->prot_count[i];
    });
}

dqtg_status dqtg_qstate_download(const dqtg_qstate* s, uint16_t* const* levels,
                                 uint64_t* const* ppos, uint16_t* const* pval,
                                 float* const* codebooks) {
    return guard([&] {
        const QState& q = *s->q;
        Engine& e = *q.eng;
        LOCK(&e);
        const Layout& L = *q.L;
        for (uint32_t i = 0; i < L.nt; ++i) {
            if (levels && levels[i] && L.numel[i])
                e.from_device(levels[i], q.d_levels + L.off[i], L.numel[i] * 2);
            if (q.prot_count[i]) {
                if (ppos && ppos[i])
                    e.from_device(ppos[i], q.d_ppos + q.prot_off[i], q.prot_count[i] * 8);
                if (pval && pval[i])
                    e.from_device(pval[i], q.d_pval + q.prot_off[i], q.prot_count[i] * 2);
            }
        }
        if (codebooks)
            for (int lt = 0; lt < kLayerTypes; ++lt)
                if (codebooks[lt] && q.cb_len[lt])
                    memcpy(codebooks[lt], q.cb[lt].data(), q.cb_len[lt] * 4);
        e.sync();
    });
}

dqtg_status dqtg_qstate_upload(dqtg_engine* h, const dqtg_layout* layout, uint64_t step,
                               const dqtg_config* cfg, const uint32_t* cb_len,
                               const float* const* cbs, const uint16_t* const* levels,
                               const uint64_t* prot_count, const uint64_t* const* ppos,
                               const uint16_t* const* pval, dqtg_qstate** out) {
    return guard([&] {
        LOCK(&h->e);
        Engine& e = h->e;
        auto q = std::make_unique<QState>();
        q->eng = &e;
        q->L = make_layout(&e, layout);
        q->step = step;
        q->cfg = *cfg;
        uint32_t stride = 1;
        for (int lt = 0; lt < kLayerTypes; ++lt) {
            q->cb_len[lt] = cb_len[lt];
            q->cb[lt].assign(cbs[lt], cbs[lt] + cb_len[lt]);
            stride = std::max(stride, cb_len[lt]);
        }
        q->cb_stride = stride;
        std::vector<float> flat((size_t)kLayerTypes * stride, 0.0f);
        for (int lt = 0; lt < kLayerTypes; ++lt)
            std::copy(q->cb[lt].begin(), q->cb[lt].end(), flat.begin() + (size_t)lt * stride);
        q->d_cb = (decltype(q->d_cb))e.dalloc(flat.size() * 4);
        DQTG_CUDA(cudaMemcpyAsync(q->d_cb, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice,
                                  e.stream));
        const Layout& L = *q->L;
        q->d_levels = (decltype(q->d_levels))e.dalloc(L.Np * 2);
        DQTG_CUDA(cudaMemsetAsync(q->d_levels, 0, L.Np * 2, e.stream));
        q->prot_count.assign(L.nt, 0);
        q->prot_off.assign(L.nt + 1, 0);
        uint64_t acc = 0;
        for (uint32_t i = 0; i < L.nt; ++i) {
            q->prot_off[i] = acc;
            q->prot_count[i] = prot_count ? prot_count[i] : 0;
            acc += q->prot_count[i];
        }
        q->prot_off[L.nt] = q->prot_total = acc;
        q->d_ppos = (decltype(q->d_ppos))e.dalloc((acc + 1) * 8);
        q->d_pval = (decltype(q->d_pval))e.dalloc((acc + 1) * 2);
        for (uint32_t i = 0; i < L.nt; ++i) {
            if (L.numel[i]) e.to_device(q->d_levels + L.off[i], levels[i], L.numel[i] * 2);
            if (q->prot_count[i]) {
                e.to_device(q->d_ppos + q->prot_off[i], ppos[i], q->prot_count[i] * 8);
                e.to_device(q->d_pval + q->prot_off[i], pval[i], q->prot_count[i] * 2);
            }
        }
        e.sync();
        auto* s = new dqtg_qstate();
        s->q = std::move(q);
        *out = s;
    });
}

void dqtg_qstate_destroy(dqtg_qstate* s) { delete s; }

uint32_t dqtg_qstate_tensor_count(const dqtg_qstate* s) { return s->q->L->nt; }

dqtg_status dqtg_qstate_tensor_info(const dqtg_qstate* s, uint32_t i, char* name, uint64_t cap,
                                    uint8_t* type, uint8_t* rank, uint64_t* dims) {
    return guard([&] {
        const Layout& L = *s->q->L;
        DQTG_REQUIRE(i < L.nt, DQTG_ERROR, "tensor index out of range");
        if (name && cap) {
            const size_t k = std::min<size_t>(L.names[i].size(), cap - 1);
            memcpy(name, L.names[i].data(), k);
            name[k] = 0;
        }
        if (type) *type = L.types[i];
        if (rank) *rank = L.ranks[i];
        if (dims)
            for (size_t r = 0; r < L.dims[i].size(); ++r) dims[r] = L.dims[i][r];
    });
}
uint16_t* dqtg_qstate_levels_dev(dqtg_qstate* s) { return s->q->d_levels; }

dqtg_status dqtg_dequantize(dqtg_engine* h, const dqtg_qstate* s, float* const* out) {
    return guard([&] {
        LOCK(&h->e);
        Engine& e = h->e;
        const QState& q = *s->q;
        const Layout& L = *q.L;
        bool all_dev = true;
        for (uint32_t i = 0; i < L.nt && all_dev; ++i)
            if (L.numel[i] && !is_device_ptr(out[i])) all_dev = false;
        if (all_dev) {  // written in place by the kernel
            auto* d = (float**)e.buf("dq.outs", (size_t)L.nt * 8 + 8);
            e.to_device(d, out, (size_t)L.nt * 8);
            ::dqtg::dequantize_to(e, q, d);
            e.check_err();
            return;
        }
        float* d = (float*)e.buf("dq.out", L.Np * 4);
        ::dqtg::dequantize(e, q, d);
        e.check_err();
        for (uint32_t i = 0; i < L.nt; ++i)
            if (L.numel[i]) e.from_device(out[i], d + L.off[i], L.numel[i] * 4);
        e.sync();
    });
}

// ---- records --------------------------------------------------------------------
dqtg_status dqtg_encode_record(dqtg_engine* h, const dqtg_qstate* base, const dqtg_qstate* target,
                               double quality, dqtg_record** out) {
    return guard([&] {
        LOCK(&h->e);
        auto r = ::dqtg::encode_record(h->e, base ? base->q.get() : nullptr, *target->q, quality);
        auto* rr = new dqtg_record();
        rr->r = std::move(r);
        *out = rr;
    });
}

dqtg_status dqtg_payload_bytes(dqtg_engine* h, const dqtg_qstate* base, const dqtg_qstate* target,
                               int variant, uint64_t* bytes) {
    return guard([&] {
        LOCK(&h->e);
        DQTG_REQUIRE(variant >= 0 && variant <= 2, DQTG_ERROR, "payload_bytes variant must be 0, 1 or 2");
        DQTG_REQUIRE(base != nullptr, DQTG_ERROR, "payload_bytes needs a base state");
        encode_record_ex(h->e, base->q.get(), *target->q, 0.0, 0, 0, nullptr, variant, bytes);
    });
}

uint64_t dqtg_record_size(const dqtg_record* r) { return r->r->size; }

dqtg_status dqtg_record_copy(const dqtg_record* r, void* dst) {
    return guard([&] {
        Engine& e = *r->r->eng;
        LOCK(&e);
        e.from_device(dst, r->r->d_buf, r->r->size);
        e.sync();
    });
}

const uint8_t* dqtg_record_dev(const dqtg_record* r) { return r->r->d_buf; }
void dqtg_record_destroy(dqtg_record* r) { delete r; }

dqtg_status dqtg_decode_record(dqtg_engine* h, const uint8_t* rec, uint64_t n,
                               const dqtg_qstate* base, dqtg_qstate** out) {
    return guard([&] {
        LOCK(&h->e);
        auto q = ::dqtg::decode_record(h->e, rec, n, base ? base->q.get() : nullptr);
        auto* s = new dqtg_qstate();
        s->q = std::move(q);
        *out = s;
    });
}

dqtg_status dqtg_decode_chain(dqtg_engine* h, uint32_t n, const uint8_t* const* recs,
                              const uint64_t* sizes, const dqtg_qstate* base, dqtg_state_fn fn,
                              void* user, dqtg_qstate** last_out) {
    return guard([&] {
        LOCK(&h->e);
        auto last = ::dqtg::decode_chain(
            h->e, recs, sizes, n, base ? base->q.get() : nullptr,
            [&](uint32_t k, const ::dqtg::QState& s) {
                if (!fn) return;
                dqtg_qstate tmp;  // borrowed for the callback
                tmp.q.reset(const_cast<::dqtg::QState*>(&s));
                fn(user, k, &tmp);
                (void)tmp.q.release();
            });
        if (last_out) {
            *last_out = nullptr;
            if (last) {
                auto* s = new dqtg_qstate();
                s->q = std::move(last);
                *last_out = s;
            }
        }
    });
}

uint64_t dqtg_shard_hist_len(dqtg_engine* h, const dqtg_config* cfg, int which) {
    uint64_t n = 0;
    dqtg_status st = guard([&] {
        LOCK(&h->e);
        n = shard_hist_len(h->e, *cfg, which);
    });
    return st == DQTG_OK ? n : 0;
}

dqtg_status dqtg_shard_stage1(dqtg_engine* h, const dqtg_ckpt* c, const dqtg_config* cfg,
                              uint64_t* score_hist) {
    return guard([&] {
        LOCK(&h->e);
        shard_stage1(h->e, c->c, *cfg, (unsigned long long*)score_hist);
    });
}

dqtg_status dqtg_shard_stage2(dqtg_engine* h, const dqtg_ckpt* c, const dqtg_config* cfg,
                              const uint64_t* score_hist, uint64_t* value_hist) {
    return guard([&] {
        LOCK(&h->e);
        shard_stage2(h->e, c->c, *cfg, (const unsigned long long*)score_hist,
                     (unsigned long long*)value_hist);
    });
}

dqtg_status dqtg_shard_stage3(dqtg_engine* h, const dqtg_ckpt* c, const dqtg_config* cfg,
                              uint64_t seed, uint64_t step, const uint64_t* value_hist,
                              dqtg_qstate** out) {
    return guard([&] {
        LOCK(&h->e);
        auto q = shard_stage3(h->e, c->c, *cfg, seed, step, (const unsigned long long*)value_hist);
        auto* s = new dqtg_qstate();
        s->q = std::move(q);
        *out = s;
    });
}

dqtg_status dqtg_encode_record_shard(dqtg_engine* h, const dqtg_qstate* base,
                                     const dqtg_qstate* target, double quality, uint32_t gB,
                                     uint32_t gnt, dqtg_record** out, uint64_t* body_offset) {
    return guard([&] {
        LOCK(&h->e);
        auto r = encode_record_ex(h->e, base ? base->q.get() : nullptr, *target->q, quality, gB,
                                  gnt, body_offset);
        auto* rr = new dqtg_record();
        rr->r = std::move(r);
        *out = rr;
    });
}

dqtg_status dqtg_compress_step(dqtg_engine* h, const dqtg_ckpt* c, const dqtg_config* cfg,
                               uint64_t seed, uint64_t step, const dqtg_qstate* base,
                               double quality, dqtg_qstate** state_out, dqtg_record** record_out) {
    return guard([&] {
        LOCK(&h->e);
        std::unique_ptr<QState> q;
        auto r = ::dqtg::compress_step(h->e, c->c, *cfg, seed, step, base ? base->q.get() : nullptr,
                                       quality, q);
        auto* s = new dqtg_qstate();
        s->q = std::move(q);
        auto* rr = new dqtg_record();
        rr->r = std::move(r);
        *state_out = s;
        *record_out = rr;
    });
}

dqtg_status dqtg_partition(dqtg_engine* h, const dqtg_ckpt* c, const dqtg_config* cfg,
                           uint8_t* const* masks) {
    return guard([&] {
        LOCK(&h->e);
        ::dqtg::partition(h->e, c->c, *cfg, masks);
    });
}

dqtg_status dqtg_proxy_quality(dqtg_engine* h, const dqtg_layout* layout,
                               const float* const* orig, const float* const* recon,
                               double* out) {
    return guard([&] {
        LOCK(&h->e);
        Engine& e = h->e;
        DevCkpt c;
        c.eng = &e;
        c.L = make_layout(&e, layout);
        DQTG_CUDA(cudaMalloc(&c.w, c.L->Np * 4));
        float* r = (float*)e.buf("pq.recon", c.L->Np * 4);
        for (uint32_t i = 0; i < c.L->nt; ++i)
            if (c.L->numel[i]) {
                e.to_device(c.w + c.L->off[i], orig[i], c.L->numel[i] * 4);
                e.to_device(r + c.L->off[i], recon[i], c.L->numel[i] * 4);
            }
        *out = ::dqtg::proxy_quality(e, c, r);
    });
}

dqtg_status dqtg_engine_trim(dqtg_engine* h) {
    return guard([&] {
        LOCK(&h->e);
        h->e.sync();
        h->e.drop_scratch("");
        trim_device_caches(h->e.device);
        std::lock_guard<std::mutex> g(h->e.pin_mu);  // pooled pinned decode staging
        for (auto& b : h->e.pin_free) cudaFreeHost(b.first);
        h->e.pin_free.clear();
    });
}

dqtg_status dqtg_qstate_equal(dqtg_engine* h, const dqtg_qstate* a, const dqtg_qstate* b,
                              int* equal) {
    return guard([&] {
        LOCK(&h->e);
        *equal = ::dqtg::states_equal(h->e, *a->q, *b->q) ? 1 : 0;
    });
}

dqtg_status dqtg_level_counts(dqtg_engine* h, const dqtg_qstate* q, uint32_t stride,
                              uint64_t* counts) {
    return guard([&] {
        LOCK(&h->e);
        ::dqtg::level_counts(h->e, *q->q, counts, (int)stride);
    });
}

dqtg_status dqtg_eval_batch(dqtg_engine* h, const dqtg_ckpt* c, const dqtg_config* cfgs,
                            const uint64_t* seeds, uint32_t m, double* quality, double* est) {
    return guard([&] {
        LOCK(&h->e);
        ::dqtg::eval_batch(h->e, c->c, cfgs, seeds, m, quality, est);
    });
}

// ---- clustering --------------------------------------------------------------------
dqtg_status dqtg_approx_kmeans(dqtg_engine* h, const float* values, uint64_t n, uint32_t k,
                               double sigma, double alpha, uint64_t seed, float* cb,
                               uint32_t* len) {
    return guard([&] {
        LOCK(&h->e);
        ::dqtg::approx_kmeans(h->e, values, n, k, sigma, alpha, seed, cb, len);
    });
}

dqtg_status dqtg_kmeanspp_init(dqtg_engine* h, const double* pts, const double* w, uint64_t n,
                               uint32_t k, uint64_t seed, double* centers) {
    return guard([&] {
        LOCK(&h->e);
        kmeanspp_host_api(h->e, pts, w, n, k, seed, centers);
    });
}

dqtg_status dqtg_lloyd(dqtg_engine* h, const double* pts, const double* w, uint64_t n,
                       double* centers, uint32_t k, double tol, uint32_t max_iter,
                       uint32_t* iters) {
    return guard([&] {
        LOCK(&h->e);
        lloyd_host_api(h->e, pts, w, n, centers, k, tol, max_iter, iters);
    });
}

dqtg_status dqtg_sq_loss(dqtg_engine* h, const double* pts, const double* w, uint64_t n,
                         const double* centers, uint32_t k, double* loss) {
    return guard([&] {
        LOCK(&h->e);
        *loss = sq_loss_host_api(h->e, pts, w, n, centers, k);
    });
}

// ---- codec primitives -----------------------------------------------------------------
dqtg_status dqtg_delta_compute(dqtg_engine* h, const uint16_t* prev, const uint16_t* cur,
                               uint64_t n, uint32_t B, uint16_t* out) {
    return guard([&] {
        LOCK(&h->e);
        delta_kernel_api(h->e, prev, cur, n, B, out, false);
    });
}

dqtg_status dqtg_delta_apply(dqtg_engine* h, const uint16_t* prev, const uint16_t* d, uint64_t n,
                             uint32_t B, uint16_t* out) {
    return guard([&] {
        LOCK(&h->e);
        delta_kernel_api(h->e, prev, d, n, B, out, true);
    });
}

dqtg_status dqtg_crc32(dqtg_engine* h, const uint8_t* data, uint64_t n, uint32_t* crc) {
    return guard([&] {
        LOCK(&h->e);
        Engine& e = h->e;
        const uint8_t* d = data;
        if (n && !is_device_ptr(data)) {
            uint8_t* b = (uint8_t*)e.buf("crc.in", n);
            e.to_device(b, data, n);
            d = b;
        }
        *crc = crc32_device(e, d, n);
    });
}

}  // extern "C"
