// Pipelined delta chain (dqtg_pipe_*, include/dqtg.h): the native runtime behind
// Chain::append over a series of snapshots (chain.cpp:86-129).
//
// W workers, each an engine with its own non-blocking CUDA stream and a host
// thread.  Snapshot k runs on worker k mod W:
//
//   weights(k), EMA(k) -> worker checkpoint   (device snapshots in the padded
//                                             layout are read in place; others
//                                             are copied H2D / D2D)
//   quantize(k)                               (passes A/B, k-means, pass C)
//   record event q[k]; publish state k
//   wait state k-1 published; stream waits on q[k-1]
//   encode(k | k-1); on_record(k); stream sync
//   release k-1 and k once both encodes that read them are done
//
// While one worker blocks on a host read-back (record size, overflow counts) or
// a copy, the others keep the GPU fed, and the few-CTA phases (k-means restarts,
// per-group Huffman) overlap the streaming passes of the other workers.
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.h"
#include "handles.h"

using namespace dqtg;

struct dqtg_pipe {
    int device = 0;
    // optional caller stream (dqtg_pipe_set_stream): every run's device work is
    // ordered after the work queued on it before the run, and work queued on it
    // after the run waits for every worker, so events on it time the whole chain
    cudaStream_t join = nullptr;
    // optional (dqtg_pipe_set_comms): one NCCL communicator per worker -- worker w runs
    // the tensor-sharded step of snapshots k = w mod W on its own communicator, so every
    // communicator sees the same sequence of collectives on every rank
    std::vector<dqtg_comm*> comms;
    uint32_t nt_total = 0;
    // worker engines: released (not deleted) so states handed out stay valid
    struct Release {
        void operator()(Engine* e) const { engine_release(e); }
    };
    std::vector<std::unique_ptr<Engine, Release>> eng;
    // per worker: a borrowing checkpoint view + owned staging buffers for snapshots
    // that are not device-resident in the padded layout (rebuilt when the layout changes)
    struct Slot {
        std::unique_ptr<DevCkpt> ck;
        float* wbuf = nullptr;
        float* ebuf = nullptr;
        const float* ebuf_src = nullptr;  // EMA currently in ebuf (per run)
        ~Slot() {
            cudaFree(wbuf);
            cudaFree(ebuf);
        }
    };
    std::vector<std::unique_ptr<Slot>> ck;
};

namespace {

bool same_layout(const Layout& a, const dqtg_layout* l) {
    if (a.nt != l->n_tensors) return false;
    size_t d = 0;
    for (uint32_t i = 0; i < a.nt; ++i) {
        if (a.types[i] != (l->types ? l->types[i] : 6) || a.ranks[i] != l->ranks[i]) return false;
        for (uint32_t r = 0; r < a.ranks[i]; ++r)
            if (a.dims[i][r] != l->dims[d + r]) return false;
        d += l->ranks[i];
        if (l->names && a.names[i] != l->names[i]) return false;
    }
    return true;
}

// per-tensor copies, merged while both the sources and the padded destinations are
// contiguous (C2: every tensor is a multiple of 64 elements -> one copy per snapshot)
void upload(Engine& e, const Layout& L, float* dst, const float* const* src) {
    uint32_t i = 0;
    while (i < L.nt) {
        uint32_t j = i + 1;
        uint64_t n = L.numel[i];
        while (j < L.nt && src[j] == src[i] + n && L.off[j] == L.off[i] + n) n += L.numel[j++];
        if (n) e.to_device(dst + L.off[i], src[i], n * 4);
        i = j;
    }
}

// The tensors of one snapshot form a device buffer in the engine's padded layout
// (tensor i at base + off[i], e.g. a dqtg_ckpt): the passes read it in place.
const float* padded_view(const Layout& L, const float* const* src) {
    if (!L.nt || !is_device_ptr(src[0])) return nullptr;
    const float* base = src[0] - L.off[0];
    for (uint32_t i = 1; i < L.nt; ++i)
        if (src[i] != base + L.off[i]) return nullptr;
    return base;
}

// weights / EMA of snapshot k for the worker: in place or staged
float* stage(Engine& e, const Layout& L, const float* const* src, float*& buf) {
    if (const float* v = padded_view(L, src)) return const_cast<float*>(v);
    if (!buf) {
        DQTG_CUDA(cudaMalloc(&buf, L.Np * 4));
        DQTG_CUDA(cudaMemsetAsync(buf, 0, L.Np * 4, e.stream));
    }
    upload(e, L, buf, src);
    return buf;
}

struct Run {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<std::unique_ptr<QState>> states;
    std::vector<cudaEvent_t> qev;
    std::vector<char> ready;
    std::vector<int> users;
    bool failed = false;
    dqtg_status code = DQTG_OK;
    std::string msg;

    void fail(dqtg_status c, const std::string& m) {
        std::lock_guard<std::mutex> g(mu);
        if (!failed) failed = true, code = c, msg = m;
        cv.notify_all();
    }
};

}  // namespace

extern "C" {

dqtg_status dqtg_pipe_create(int device, int workers, dqtg_pipe** out) {
    try {
        DQTG_REQUIRE(workers >= 1 && workers <= 16, DQTG_ERROR, "workers must be in [1, 16]");
        auto p = std::make_unique<dqtg_pipe>();
        p->device = device;
        for (int w = 0; w < workers; ++w) {
            p->eng.push_back(std::unique_ptr<Engine, dqtg_pipe::Release>(new Engine()));
            init_engine(*p->eng.back(), device, nullptr);
        }
        p->ck.resize(workers);
        *out = p.release();
        return DQTG_OK;
    } catch (const Fail& x) {
        set_last_error(x.what());
        return x.code;
    } catch (const std::exception& x) {
        set_last_error(x.what());
        return DQTG_ERROR;
    }
}

void dqtg_pipe_destroy(dqtg_pipe* p) {
    if (!p) return;
    for (auto& e : p->eng) cudaStreamSynchronize(e->stream);
    p->ck.clear();
    p->eng.clear();
    delete p;
}

void dqtg_pipe_set_stream(dqtg_pipe* p, void* stream) { p->join = (cudaStream_t)stream; }

dqtg_status dqtg_pipe_set_comms(dqtg_pipe* p, dqtg_comm* const* comms, int n,
                                uint32_t n_tensors_total) {
    if (n != 0 && n != (int)p->eng.size()) {
        set_last_error("one communicator per worker");
        return DQTG_ERROR;
    }
    p->comms.assign(comms, comms + n);
    p->nt_total = n_tensors_total;
    return DQTG_OK;
}

uint64_t dqtg_pipe_launches(const dqtg_pipe* p) {
    uint64_t n = 0;
    for (auto& e : p->eng) n += e->launches;
    return n;
}

dqtg_status dqtg_pipe_run(dqtg_pipe* p, const dqtg_layout* layout, const float* const* weights,
                          uint64_t n, const uint64_t* steps, const float* const* ema,
                          const dqtg_config* cfg, uint64_t seed, const dqtg_qstate* base,
                          double quality, dqtg_record_fn on_record, void* user,
                          dqtg_qstate** last_out) {
    try {
        const int W = (int)p->eng.size();
        DQTG_CUDA(cudaSetDevice(p->device));
        // worker checkpoint views for this layout
        for (int w = 0; w < W; ++w) {
            Engine& e = *p->eng[w];
            auto& sl = p->ck[w];
            if (!sl || !same_layout(*sl->ck->L, layout)) {
                sl = std::make_unique<dqtg_pipe::Slot>();
                sl->ck = std::make_unique<DevCkpt>();
                sl->ck->eng = &e;
                sl->ck->own = false;
                sl->ck->L = make_layout(&e, layout);
            }
            sl->ebuf_src = nullptr;
            DevCkpt& c = *sl->ck;
            c.explicit_scores = false;
            c.has_sens = ema != nullptr;
            c.ema_seeded = ema != nullptr;
        }
        if (p->join) {  // fork: the workers start after the caller stream's prior work
            cudaEvent_t ev;
            DQTG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            DQTG_CUDA(cudaEventRecord(ev, p->join));
            for (auto& e : p->eng) DQTG_CUDA(cudaStreamWaitEvent(e->stream, ev, 0));
            cudaEventDestroy(ev);
        }
        const uint32_t nt = layout->n_tensors;
        const bool tl = getenv("DQTG_TIMELINE") != nullptr;
        for (auto& e : p->eng) {
            e->profiling = tl;
            if (tl) timeline_epoch(*e);
        }
        Run R;
        const bool trace = getenv("DQTG_PIPE_TRACE") != nullptr;
        const auto t_start = std::chrono::steady_clock::now();
        std::vector<double> t_q(n, 0.0), t_e(n, 0.0), t_u(n, 0.0), t_w(n, 0.0), t_c(n, 0.0), t_0(n, 0.0);
        auto now_ms = [&] {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        };
        R.states.resize(n);
        R.qev.assign(n, nullptr);
        R.ready.assign(n, 0);
        R.users.assign(n, 0);
        for (uint64_t k = 0; k < n; ++k) DQTG_CUDA(cudaEventCreateWithFlags(&R.qev[k], cudaEventDisableTiming));

        auto release = [&](uint64_t k) {  // caller holds R.mu
            if (++R.users[k] == 2 && k + 1 != n) R.states[k].reset();
        };
        auto worker = [&](int w) {
            Engine& e = *p->eng[w];
            dqtg_pipe::Slot& sl = *p->ck[w];
            DevCkpt& c = *sl.ck;
            try {
                e.activate();
                for (uint64_t k = (uint64_t)w; k < n; k += (uint64_t)W) {
                    {
                        std::lock_guard<std::mutex> g(R.mu);
                        if (R.failed) return;
                    }
                    if (trace) t_0[k] = now_ms();
                    c.w = stage(e, *c.L, weights + k * nt, sl.wbuf);
                    if (ema) {  // snapshot k's own EMA (the scores of step k)
                        const float* const* ek = ema + k * nt;
                        if (const float* v = padded_view(*c.L, ek)) {
                            c.ema = const_cast<float*>(v);
                        } else {
                            if (sl.ebuf_src != ek[0]) stage(e, *c.L, ek, sl.ebuf);
                            sl.ebuf_src = ek[0];
                            c.ema = sl.ebuf;
                        }
                    }
                    if (trace) t_u[k] = now_ms();
                    dqtg_comm* cm = p->comms.empty() ? nullptr : p->comms[w];
                    const uint64_t sk = steps ? steps[k] : k;
                    // publish state k (its levels are enqueued on this stream)
                    auto publish = [&](std::unique_ptr<QState> q) {
                        DQTG_CUDA(cudaEventRecord(R.qev[k], e.stream));
                        std::lock_guard<std::mutex> g(R.mu);
                        R.states[k] = std::move(q);
                        R.ready[k] = 1;
                        R.cv.notify_all();
                    };
                    // state k-1 (the delta base): wait until it is published
                    auto wait_prev = [&]() -> const QState* {
                        if (k == 0) return base ? base->q.get() : nullptr;
                        std::unique_lock<std::mutex> g(R.mu);
                        R.cv.wait(g, [&] { return R.failed || R.ready[k - 1]; });
                        if (R.failed) return nullptr;
                        return R.states[k - 1].get();
                    };
                    dqtg_record rec;
                    if (cm) {
                        auto q = sharded_quantize(e, cm, c, *cfg, seed, sk);
                        if (trace) t_q[k] = now_ms();
                        const QState* target = q.get();
                        publish(std::move(q));
                        const QState* prev = wait_prev();
                        if (k > 0 && !prev) return;
                        if (k > 0) DQTG_CUDA(cudaStreamWaitEvent(e.stream, R.qev[k - 1], 0));
                        if (trace) t_w[k] = now_ms();
                        rec.r = sharded_encode(e, cm, prev, *target, quality, p->nt_total);
                    } else {
                        // quantize + encode with pass C fused into the DELTA encoder: the
                        // state is published once its levels are enqueued (mid-encode), and
                        // the base must be published before this step's encode starts
                        const QState* prev = nullptr;
                        bool have_prev = false;
                        std::unique_ptr<QState> q;
                        const uint32_t kt = std::max(cfg->bins, cfg->embed_bins) + 2;
                        const bool fuse = (k > 0 || base) && fused_c_enabled() && kt <= 64;
                        FuseC fc;
                        q = quantize(e, c, *cfg, seed, sk, fuse ? &fc : nullptr);
                        if (trace) t_q[k] = now_ms();
                        QState* target = q.get();
                        if (!fuse || !fc.w) {
                            publish(std::move(q));
                            q.reset();
                        }
                        prev = wait_prev();
                        have_prev = prev != nullptr;
                        if (k > 0 && !have_prev) return;
                        if (k > 0) DQTG_CUDA(cudaStreamWaitEvent(e.stream, R.qev[k - 1], 0));
                        if (trace) t_w[k] = now_ms();
                        if (q && prev && prev->max_levels() <= 64) {
                            QState* tq = q.get();
                            rec.r = encode_record_ex(e, prev, *tq, quality, 0, 0, nullptr, 0, nullptr, &fc,
                                                     [&] { publish(std::move(q)); });
                        } else {
                            if (q) {  // could not fuse after all: pass C, then publish
                                run_pass_c(e, c, fc, *target);
                                publish(std::move(q));
                            }
                            rec.r = encode_record(e, prev, *target, quality);
                        }
                    }
                    if (trace) t_c[k] = now_ms();
                    if (on_record && rec.r) on_record(user, k, &rec);
                    rec.r.reset();
                    e.sync();  // encode(k) complete: its inputs may be released
                    if (trace) t_e[k] = now_ms();
                    std::lock_guard<std::mutex> g(R.mu);
                    release(k);
                    if (k > 0) release(k - 1);
                }
            } catch (const Fail& x) {
                R.fail(x.code, x.what());
            } catch (const std::exception& x) {
                R.fail(DQTG_ERROR, x.what());
            }
        };
        std::vector<std::thread> th;
        for (int w = 0; w < W; ++w) th.emplace_back(worker, w);
        for (auto& t : th) t.join();
        for (auto ev : R.qev) cudaEventDestroy(ev);
        if (p->join) {  // join: the caller stream waits for every worker's last work
            for (auto& e : p->eng) {
                cudaEvent_t ev;
                DQTG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                DQTG_CUDA(cudaEventRecord(ev, e->stream));
                DQTG_CUDA(cudaStreamWaitEvent(p->join, ev, 0));
                cudaEventDestroy(ev);
            }
        }
        if (trace)
            for (uint64_t k = 0; k < n; ++k)
                fprintf(stderr, "pipe k=%llu worker=%d start %.3f uploaded %.3f quantized %.3f waited %.3f encode-call %.3f encoded %.3f ms\n",
                        (unsigned long long)k, (int)(k % W), t_0[k], t_u[k], t_q[k], t_w[k], t_c[k], t_e[k]);
        if (tl)
            for (auto& e : p->eng) {
                e->sync();
                dump_timeline(*e);
                e->spans.clear();
                e->ev_used = 0;
            }
        if (R.failed) throw Fail(R.code, R.msg);
        if (last_out) {
            *last_out = nullptr;
            if (n) {
                auto* s = new dqtg_qstate();
                s->q = std::move(R.states[n - 1]);
                *last_out = s;
            }
        }
        return DQTG_OK;
    } catch (const Fail& x) {
        set_last_error(x.what());
        return x.code;
    } catch (const std::exception& x) {
        set_last_error(x.what());
        return DQTG_ERROR;
    }
}

}  // extern "C"
