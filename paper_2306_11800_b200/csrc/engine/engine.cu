#include <chrono>
// Engine plumbing: device/stream, scratch, alpha tables, layouts, object lifetimes.
#include <algorithm>
#include <cstdlib>
#include <float.h>
#include <math.h>
#include <string.h>

#include <cstdio>
#include <cstring>

#include "engine.h"

namespace dqtg {

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaEvent_t Engine::take_event() {
    if (ev_used == event_pool.size()) {
        cudaEvent_t ev;
        DQTG_CUDA(cudaEventCreate(&ev));
        event_pool.push_back(ev);
    }
    return event_pool[ev_used++];
}

cudaStream_t Engine::hi() {
    if (!hi_stream) {
        int lo = 0, hi_p = 0;
        DQTG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi_p));
        DQTG_CUDA(cudaStreamCreateWithPriority(&hi_stream, cudaStreamNonBlocking, hi_p));
        DQTG_CUDA(cudaEventCreateWithFlags(&hi_fork, cudaEventDisableTiming));
        DQTG_CUDA(cudaEventCreateWithFlags(&hi_join, cudaEventDisableTiming));
    }
    DQTG_CUDA(cudaEventRecord(hi_fork, stream));
    DQTG_CUDA(cudaStreamWaitEvent(hi_stream, hi_fork, 0));
    return hi_stream;
}

void Engine::hi_done() {
    DQTG_CUDA(cudaEventRecord(hi_join, hi_stream));
    DQTG_CUDA(cudaStreamWaitEvent(stream, hi_join, 0));
}

// ---- launch timeline (DQTG_TIMELINE): spans relative to a process-wide epoch ----
static cudaEvent_t g_epoch = nullptr;
static std::mutex g_epoch_mu;

void timeline_epoch(Engine& e) {
    std::lock_guard<std::mutex> g(g_epoch_mu);
    if (g_epoch) return;
    e.activate();
    DQTG_CUDA(cudaEventCreate(&g_epoch));
    DQTG_CUDA(cudaEventRecord(g_epoch, e.stream));
}

void dump_timeline(Engine& e) {
    if (!g_epoch) return;
    for (auto& s : e.spans) {
        float a = 0.0f, b = 0.0f;
        if (cudaEventElapsedTime(&a, g_epoch, s.a) != cudaSuccess) continue;
        if (cudaEventElapsedTime(&b, g_epoch, s.b) != cudaSuccess) continue;
        fprintf(stderr, "timeline %9.3f %9.3f %8.3f %p %s\n", a, b, b - a, (void*)e.stream, s.name);
    }
}

void engine_retain(Engine* e) { e->refs.fetch_add(1, std::memory_order_relaxed); }

void engine_release(Engine* e) {
    if (e->refs.fetch_sub(1, std::memory_order_acq_rel) != 1) return;
    if (e->deleter) e->deleter(e->owner);
    else delete e;
}

Engine::~Engine() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (hi_stream) {
        cudaStreamSynchronize(hi_stream);
        cudaStreamDestroy(hi_stream);
        cudaEventDestroy(hi_fork);
        cudaEventDestroy(hi_join);
    }
    for (auto ev : event_pool) cudaEventDestroy(ev);
    for (auto& kv : scratch) cudaFreeAsync(kv.second.first, stream);
    cudaStreamSynchronize(stream);
    for (auto& kv : tables) {
        cudaFree(kv.second->d_U);
        cudaFree(kv.second->d_cell);
        cudaFree(kv.second->d_slot);
        cudaFree(kv.second->d_ctab);
        cudaFree(kv.second->d_key);
        cudaFree(kv.second->d_keyf);
    }
    if (d_err) cudaFree(d_err);
    if (pinned) cudaFreeHost(pinned);
    for (auto& b : pin_free) cudaFreeHost(b.first);
    for (auto& b : stage_blocks) cudaFreeHost(b.first);
    if (own_stream && stream) cudaStreamDestroy(stream);
    if (pool) {
        unregister_pool(pool);
        cudaMemPoolDestroy(pool);  // blocks still owned by live states keep it alive
    }
}

// ---- out-of-memory recovery --------------------------------------------------------
// Freed memory stays cached (engine pools keep everything, BigCache keeps freed level
// arrays and records): right for a steady chain, but a workload that moves between
// very different sizes (C4 then C5 in one process) can find HBM held by caches.  On
// an allocation failure every cache of the device is dropped and the pools trimmed,
// then the allocation is retried once.
namespace {
std::mutex g_pools_mu;
std::map<cudaMemPool_t, int> g_pools;  // live engine pools -> device
}  // namespace

void register_pool(cudaMemPool_t p, int device) {
    std::lock_guard<std::mutex> g(g_pools_mu);
    g_pools[p] = device;
}
void unregister_pool(cudaMemPool_t p) {
    std::lock_guard<std::mutex> g(g_pools_mu);
    g_pools.erase(p);
}

static void drop_big_cache(int device);

void trim_device_caches(int device) {
    cudaGetLastError();  // the failed allocation's error
    cudaDeviceSynchronize();
    drop_big_cache(device);
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> g(g_pools_mu);
    for (auto& kv : g_pools)
        if (kv.second == device) cudaMemPoolTrimTo(kv.first, 0);
}

template <typename F>
static cudaError_t alloc_retry(int device, F f) {
    cudaError_t r = f();
    if (r == cudaErrorMemoryAllocation) {
        trim_device_caches(device);
        r = f();
    }
    return r;
}

cudaError_t dev_malloc(void** p, size_t bytes, int device) {
    return alloc_retry(device, [&] { return cudaMalloc(p, bytes); });
}

void* Engine::buf(const std::string& name, size_t bytes) {
    auto& slot = scratch[name];
    if (slot.second < bytes) {
        // stream-ordered: scratch is only touched by this engine's stream, so the
        // old block is released after its last use without a device-wide sync
        if (getenv("DQTG_SYNC_BUF")) {  // debug: synchronous growth
            if (slot.first) {
                DQTG_CUDA(cudaStreamSynchronize(stream));
                DQTG_CUDA(cudaFree(slot.first));
            }
            size_t cap = bytes < 256 ? 256 : bytes + bytes / 4;
            DQTG_CUDA(cudaMalloc(&slot.first, cap));
            slot.second = cap;
            return slot.first;
        }
        // at least double on growth: data-dependent scratch (overflow runs, protected
        // entries, k-means keys) would otherwise grow by small steps, and every growth
        // maps pool memory on the host thread mid-step
        size_t cap = pool_size_class(std::max(bytes < 256 ? 256 : bytes + bytes / 4, 2 * slot.second));
        if (slot.first) DQTG_CUDA(cudaFreeAsync(slot.first, stream));
        slot.first = nullptr;
        DQTG_CUDA(alloc_retry(device, [&] { return cudaMallocFromPoolAsync(&slot.first, cap, pool, stream); }));
        slot.second = cap;
    }
    return slot.first;
}

void Engine::drop_scratch(const std::string& prefix) {
    for (auto it = scratch.begin(); it != scratch.end();) {
        if (it->first.compare(0, prefix.size(), prefix) == 0) {
            if (it->second.first) cudaFreeAsync(it->second.first, stream);
            it = scratch.erase(it);
        } else {
            ++it;
        }
    }
}

// Pool requests are rounded to size classes (powers of two up to 1 MiB, then eighths
// of the next power of two): steps whose record / protected-entry sizes wobble then
// reuse the blocks the previous steps freed instead of growing the pool, which maps
// new physical memory on the host thread (measured: 1-68 ms stalls mid-step).
size_t pool_size_class(size_t n) {
    if (n <= 256) return 256;
    if (n <= (1u << 20)) {
        size_t p = 256;
        while (p < n) p <<= 1;
        return p;
    }
    size_t p = 1;
    while ((p << 1) <= n) p <<= 1;
    const size_t step = p / 8;
    return (n + step - 1) / step * step;
}

constexpr size_t kBigBlock = 1u << 20;  // level arrays, records, protected entries
constexpr size_t kBigKeep = 12;  // cached blocks per (device, size class)

namespace {
struct BigBlock {
    void* p;
    size_t cls;
    int device;
    cudaEvent_t ev;  // recorded on the freeing stream
};
struct BigCache {
    std::mutex mu;
    std::map<void*, std::pair<size_t, int>> live;  // block -> (size class, device)
    std::vector<BigBlock> free;
};
BigCache& big_cache() {
    static BigCache* c = new BigCache();  // process lifetime (blocks outlive engines)
    return *c;
}
}  // namespace

static void drop_big_cache(int device) {
    BigCache& bc = big_cache();
    std::lock_guard<std::mutex> g(bc.mu);
    for (size_t i = bc.free.size(); i-- > 0;) {
        BigBlock& b = bc.free[i];
        if (b.device != device) continue;
        cudaEventSynchronize(b.ev);
        cudaEventDestroy(b.ev);
        cudaFree(b.p);  // returns the block to its pool (synchronous)
        bc.free.erase(bc.free.begin() + (long)i);
    }
}

void* Engine::dalloc(size_t bytes) {
    void* p = nullptr;
    const size_t cls = pool_size_class(bytes ? bytes : 16);
    if (cls >= kBigBlock) {
        BigCache& bc = big_cache();
        std::lock_guard<std::mutex> g(bc.mu);
        // best fit among cached blocks of this class up to 1.25x (record and
        // protected-entry sizes wobble across class edges from step to step)
        size_t best = bc.free.size();
        for (size_t i = bc.free.size(); i-- > 0;) {
            const BigBlock& b = bc.free[i];
            if (b.device == device && b.cls >= cls && b.cls <= cls + cls / 4 &&
                (best == bc.free.size() || b.cls < bc.free[best].cls))
                best = i;
        }
        if (best != bc.free.size()) {
            BigBlock b = bc.free[best];
            bc.free.erase(bc.free.begin() + (long)best);
            DQTG_CUDA(cudaStreamWaitEvent(stream, b.ev, 0));
            cudaEventDestroy(b.ev);
            bc.live[b.p] = {b.cls, device};
            return b.p;
        }
    }
    DQTG_CUDA(alloc_retry(device, [&] { return cudaMallocFromPoolAsync(&p, cls, pool, stream); }));
    if (cls >= kBigBlock) {
        BigCache& bc = big_cache();
        std::lock_guard<std::mutex> g(bc.mu);
        bc.live[p] = {cls, device};
    }
    return p;
}

void Engine::dfree(void* p) {
    if (!p) return;
    BigCache& bc = big_cache();
    {
        std::lock_guard<std::mutex> g(bc.mu);
        auto it = bc.live.find(p);
        if (it != bc.live.end()) {
            const size_t cls = it->second.first;
            bc.live.erase(it);
            size_t same = 0;
            for (auto& b : bc.free) same += b.cls == cls && b.device == device;
            cudaEvent_t ev;
            if (same < kBigKeep && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
                if (cudaEventRecord(ev, stream) == cudaSuccess) {
                    bc.free.push_back(BigBlock{p, cls, device, ev});
                    return;
                }
                cudaEventDestroy(ev);
            }
        }
    }
    cudaFreeAsync(p, stream);
}

void* Engine::pin_acquire(size_t bytes, size_t* cap) {
    {
        std::lock_guard<std::mutex> g(pin_mu);
        size_t best = pin_free.size();
        for (size_t i = 0; i < pin_free.size(); ++i)  // smallest block that fits
            if (pin_free[i].second >= bytes && (best == pin_free.size() || pin_free[i].second < pin_free[best].second))
                best = i;
        if (best < pin_free.size()) {
            auto b = pin_free[best];
            pin_free.erase(pin_free.begin() + (long)best);
            *cap = b.second;
            return b.first;
        }
    }
    void* p = nullptr;
    size_t c = 1u << 20;  // power-of-two classes: records of a chain wobble in size
    while (c < bytes + bytes / 4) c <<= 1;
    activate();  // may run on a helper thread: the engine's device, not device 0
    DQTG_CUDA(cudaHostAlloc(&p, c, cudaHostAllocPortable));
    *cap = c;
    return p;
}

void Engine::pin_release(void* p, size_t cap) {
    if (!p) return;
    std::lock_guard<std::mutex> g(pin_mu);
    pin_free.emplace_back(p, cap);
}

void* Engine::host_pinned(size_t bytes) {
    if (pinned_cap < bytes) {
        if (pinned) {
            DQTG_CUDA(cudaStreamSynchronize(stream));
            cudaFreeHost(pinned);
        }
        pinned_cap = bytes + bytes / 4 + 4096;
        DQTG_CUDA(cudaMallocHost(&pinned, pinned_cap));
    }
    return pinned;
}

void Engine::d2h(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    const size_t need = (bytes + 15) & ~(size_t)15;
    if (stage_blocks.empty() || stage_used + need > stage_blocks.back().second) {
        const size_t cap = std::max<size_t>(need, stage_blocks.empty() ? (1u << 20)
                                                                       : 2 * stage_blocks.back().second);
        uint8_t* p = nullptr;
        DQTG_CUDA(cudaMallocHost(&p, cap));
        stage_blocks.push_back({p, cap});
        stage_used = 0;
    }
    uint8_t* at = stage_blocks.back().first + stage_used;
    stage_used += need;
    DQTG_CUDA(cudaMemcpyAsync(at, src, bytes, cudaMemcpyDeviceToHost, stream));
    pend.push_back({dst, at, bytes});
}

static thread_local std::chrono::steady_clock::time_point g_last_tp{};

void Engine::tp(int line) {
    static const bool trace = getenv("DQTG_SYNC_TRACE") != nullptr;
    if (!trace) return;
    const auto t = std::chrono::steady_clock::now();
    const double us = g_last_tp.time_since_epoch().count()
                          ? std::chrono::duration<double, std::micro>(t - g_last_tp).count() : -1.0;
    fprintf(stderr, "tp %d %.1f us %p\n", line, us, (void*)this);
    g_last_tp = std::chrono::steady_clock::now();
}

void Engine::sync(const char* fn, int line) {
    static const bool trace = getenv("DQTG_SYNC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    DQTG_CUDA(cudaStreamSynchronize(stream));
    const auto t1 = std::chrono::steady_clock::now();
    sync_n++;
    sync_ns += (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    if (trace) {
        static thread_local std::chrono::steady_clock::time_point last{};
        const double host = last.time_since_epoch().count()
                                ? std::chrono::duration<double, std::micro>(t0 - last).count() : 0.0;
        fprintf(stderr, "sync %-28s:%-5d host %8.1f us blocked %8.1f us\n", fn, line, host,
                std::chrono::duration<double, std::micro>(t1 - t0).count());
        last = std::chrono::steady_clock::now();
        g_last_tp = last;
    }
    for (auto& p : pend) memcpy(p.dst, p.staged, p.n);
    pend.clear();
    while (stage_blocks.size() > 1) {  // keep the largest (last) block
        cudaFreeHost(stage_blocks.front().first);
        stage_blocks.erase(stage_blocks.begin());
    }
    stage_used = 0;
}

void Engine::check_err(const char* fn, int line) {
    uint32_t h = 0;
    d2h(&h, d_err, 4);
    sync(fn, line);
    if (!h) return;
    DQTG_CUDA(cudaMemsetAsync(d_err, 0, 4, stream));
    throw_err_bits(h);
}

void throw_err_bits(uint32_t h) {
    if (!h) return;
    if (h & kErrNonFinite) throw Fail(DQTG_NON_FINITE, "input contains NaN/Inf");
    if (h & kErrEmptySketch) throw Fail(DQTG_EMPTY_SKETCH, "quantile of empty sketch");
    if (h & kErrCorruptIndex) throw Fail(DQTG_CORRUPT_INDEX, "level outside cyclic alphabet");
    if (h & kErrHuffmanDepth) throw Fail(DQTG_ERROR, "huffman code length overflow");
    if (h & kErrKmeansWeights) throw Fail(DQTG_ERROR, "total weight must be positive");
    if (h & kErrCorruptBitstream) throw Fail(DQTG_CORRUPT_BITSTREAM, "corrupt bitstream");
    throw Fail(DQTG_ERROR, "device error");
}

void Engine::to_device(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    DQTG_CUDA(cudaMemcpyAsync(dst, src, bytes,
                              is_device_ptr(src) ? cudaMemcpyDeviceToDevice
                                                 : cudaMemcpyHostToDevice,
                              stream));
}

void Engine::from_device(void* dst, const void* src, size_t bytes) {
    if (!bytes) return;
    DQTG_CUDA(cudaMemcpyAsync(dst, src, bytes,
                              is_device_ptr(dst) ? cudaMemcpyDeviceToDevice
                                                 : cudaMemcpyDeviceToHost,
                              stream));
}

// ---- alpha tables ----------------------------------------------------------
// Host restatement of the reference bucket rule, used only to build and verify
// the integer boundary tables (sketch.cpp:21-31).
static int64_t ref_bucket(double gamma, double inv_ln_gamma, double ax) {
    double r = log(ax) * inv_ln_gamma;
    double nearest = nearbyint(r);
    if (fabs(r - nearest) > 1e-9 * fmax(1.0, fabs(r))) return (int64_t)ceil(r);
    int64_t k = (int64_t)nearest;
    while (pow(gamma, (double)(k - 1)) >= ax) --k;
    while (pow(gamma, (double)k) < ax) ++k;
    return k;
}

static float round_down_f(double v) {
    if (v >= (double)FLT_MAX) return FLT_MAX;
    if (v <= -(double)FLT_MAX) return -FLT_MAX;
    float f = (float)v;
    if ((double)f > v) f = nextafterf(f, -INFINITY);
    return f;
}

static uint32_t fbits(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

AlphaTables& Engine::alpha_tables(double alpha) {
    if (!(alpha > 0.0) || !(alpha < 1.0))
        throw Fail(DQTG_ALPHA_OUT_OF_RANGE, "alpha must be in (0, 1)");
    uint64_t key;
    memcpy(&key, &alpha, 8);
    auto it = tables.find(key);
    if (it != tables.end()) return *it->second;
    auto t = std::make_unique<AlphaTables>();
    t->alpha = alpha;
    t->gamma = (1.0 + alpha) / (1.0 - alpha);  // sketch.cpp:16-18
    t->inv_ln_gamma = 1.0 / log(t->gamma);
    t->rep_scale = 2.0 / (1.0 + t->gamma);
    float zf = (float)1e-12;
    if ((double)zf < 1e-12) zf = nextafterf(zf, INFINITY);
    t->zbits = fbits(zf);
    t->kmin = ref_bucket(t->gamma, t->inv_ln_gamma, (double)zf);
    t->kmax = ref_bucket(t->gamma, t->inv_ln_gamma, (double)FLT_MAX);
    t->NB = t->kmax - t->kmin + 1;
    t->HS = 2 * t->NB + 1;
    std::vector<uint32_t> U((size_t)t->NB + 1);
    for (int64_t k = t->kmin - 1; k <= t->kmax; ++k)
        U[(size_t)(k - t->kmin + 1)] = fbits(round_down_f(pow(t->gamma, (double)k)));
    // Verify the table against the reference rule at every bucket boundary; the
    // rule is monotone, so agreement at all boundaries is agreement everywhere.
    for (int64_t k = t->kmin; k <= t->kmax; ++k) {
        uint32_t u = U[(size_t)(k - t->kmin + 1)];
        float f;
        memcpy(&f, &u, 4);
        if (u >= t->zbits && ref_bucket(t->gamma, t->inv_ln_gamma, (double)f) != k)
            throw Fail(DQTG_ERROR, "bucket table disagrees with reference rule at k=" +
                                       std::to_string(k));
        if (k < t->kmax) {
            float g = nextafterf(f, INFINITY);
            if (fbits(g) >= t->zbits && ref_bucket(t->gamma, t->inv_ln_gamma, (double)g) != k + 1)
                throw Fail(DQTG_ERROR, "bucket table boundary mismatch at k=" + std::to_string(k));
        }
    }
    t->h_key.resize((size_t)t->HS);
    std::vector<float> keyf((size_t)t->HS);
    for (int64_t k = t->kmin; k <= t->kmax; ++k) {
        double rep = t->rep_scale * pow(t->gamma, (double)k);  // sketch.cpp:33-37
        t->h_key[(size_t)(t->kmax - k)] = -rep;
        t->h_key[(size_t)(t->NB + 1 + k - t->kmin)] = rep;
    }
    t->h_key[(size_t)t->NB] = 0.0;
    for (size_t i = 0; i < keyf.size(); ++i) keyf[i] = round_down_f(t->h_key[i]);
    if (t->NB <= kWin) {
        t->kw_lo = t->kmin;
    } else {
        int64_t top = ref_bucket(t->gamma, t->inv_ln_gamma, 10.0);
        int64_t lo = top - kWin + 1;
        if (lo > t->kmax - kWin + 1) lo = t->kmax - kWin + 1;
        if (lo < t->kmin) lo = t->kmin;
        t->kw_lo = lo;
    }
    t->inv_log2_gamma = (float)(1.0 / log2(t->gamma));
    // Cell table (see AlphaTables): the coarsest cell width whose cells all span
    // at most two buckets, each cell checked against U (exact integer compares).
    std::vector<uint2> cells;
    auto ubits = [&](int64_t k) { return U[(size_t)(k - t->kmin + 1)]; };
    auto host_bucket = [&](uint32_t a) {  // smallest k in [kmin, kmax] with U(k) >= a
        int64_t lo = t->kmin, hi = t->kmax;
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if (ubits(mid) >= a) hi = mid;
            else lo = mid + 1;
        }
        return lo;
    };
    // Slot table on the same cells: the shared-memory window slot of |x| directly
    // (0 zero bucket, 1..kWin window bucket kw_lo + p - 1, kSlotSpill outside the
    // window, kSlotBad non-finite); entry = (lo | hi << 16, split bits).
    std::vector<uint2> slots;
    auto pslot = [&](int64_t k) -> uint32_t {
        const int64_t d = k - t->kw_lo;
        return (d >= 0 && d < kWin) ? (uint32_t)(d + 1) : kSlotSpill;
    };
    for (uint32_t m = 4; m <= 12 && !t->cell_shift; ++m) {
        const uint32_t shift = 23 - m, ncell = 0x7f800000u >> shift;
        cells.assign(ncell, uint2{0, 0xffffffffu});
        slots.assign(0x80000000u >> shift, uint2{kSlotBad | (kSlotBad << 16), 0xffffffffu});
        bool ok = true;
        for (uint32_t c = 0; c < ncell && ok; ++c) {
            const uint32_t c0 = c << shift, a0 = std::max(c0, t->zbits), a1 = ((c + 1) << shift) - 1;
            if (a1 < t->zbits) {  // zero bucket
                slots[c] = uint2{0u, 0xffffffffu};
                continue;
            }
            const int64_t k0 = host_bucket(a0), k1 = host_bucket(a1);
            if (k1 > k0 + 1) ok = false;
            cells[c].x = (uint32_t)(int32_t)k0;
            cells[c].y = k1 == k0 ? 0xffffffffu : ubits(k0);
            if (c0 < t->zbits) {  // zero bucket below zbits, then one bucket
                if (k1 != k0) ok = false;
                slots[c] = uint2{0u | (pslot(k0) << 16), t->zbits - 1};
            } else {
                slots[c] = uint2{pslot(k0) | (pslot(k1) << 16), k1 == k0 ? 0xffffffffu : ubits(k0)};
            }
        }
        if (ok) t->cell_shift = shift;
    }
    activate();
    if (t->cell_shift) {
        DQTG_CUDA(cudaMalloc(&t->d_cell, cells.size() * sizeof(uint2)));
        DQTG_CUDA(cudaMemcpy(t->d_cell, cells.data(), cells.size() * sizeof(uint2),
                             cudaMemcpyHostToDevice));
        DQTG_CUDA(cudaMalloc(&t->d_slot, slots.size() * sizeof(uint2)));
        DQTG_CUDA(cudaMemcpy(t->d_slot, slots.data(), slots.size() * sizeof(uint2),
                             cudaMemcpyHostToDevice));
        const uint32_t m = 23 - t->cell_shift;
        if (t->cell_shift <= 17 && m <= 7) {  // 32 binades [2^-32, 1) in <= 16 KB
            t->ctab_lo = (95u << 23) >> t->cell_shift;
            t->ctab_n = 32u << m;
            std::vector<uint32_t> ct(t->ctab_n);
            for (uint32_t r = 0; r < t->ctab_n; ++r) {
                const uint32_t cell = t->ctab_lo + r, a0 = cell << t->cell_shift;
                const uint2 e = slots[cell];
                const uint32_t lo = e.x & 0xffffu, hi = e.x >> 16;
                const bool split = e.y != 0xffffffffu;
                const uint32_t off = split ? e.y - a0 : (1u << 17) - 1u;
                const bool lo_sp = lo > (uint32_t)kWin;
                const bool hi_sp = split ? (hi != lo + 1 || hi > (uint32_t)kWin) : lo_sp;
                ct[r] = (lo & 0x1fffu) | (off << 13) | ((uint32_t)hi_sp << 30) | ((uint32_t)lo_sp << 31);
            }
            DQTG_CUDA(cudaMalloc(&t->d_ctab, ct.size() * 4));
            DQTG_CUDA(cudaMemcpy(t->d_ctab, ct.data(), ct.size() * 4, cudaMemcpyHostToDevice));
        }
    }
    DQTG_CUDA(cudaMalloc(&t->d_U, U.size() * 4));
    DQTG_CUDA(cudaMalloc(&t->d_key, t->h_key.size() * 8));
    DQTG_CUDA(cudaMalloc(&t->d_keyf, keyf.size() * 4));
    DQTG_CUDA(cudaMemcpy(t->d_U, U.data(), U.size() * 4, cudaMemcpyHostToDevice));
    DQTG_CUDA(cudaMemcpy(t->d_key, t->h_key.data(), t->h_key.size() * 8, cudaMemcpyHostToDevice));
    DQTG_CUDA(cudaMemcpy(t->d_keyf, keyf.data(), keyf.size() * 4, cudaMemcpyHostToDevice));
    // pageable H2D copies may return before their DMA lands, on the legacy stream
    // that the (non-blocking) engine streams do not wait for
    DQTG_CUDA(cudaStreamSynchronize(0));
    auto& ref = *t;
    tables[key] = std::move(t);
    return ref;
}

void ensure_dyn_smem(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<const void*, size_t> set;
    std::lock_guard<std::mutex> g(mu);
    size_t& cur = set[func];
    if (bytes <= cur) return;
    DQTG_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
}

// ---- layouts --------------------------------------------------------------
Layout::~Layout() {
    cudaFree(d_tiles);
    cudaFree(d_types);
    cudaFree(d_off);
    cudaFree(d_numel);
    cudaFree(d_tile0);
    cudaFree(d_stream_off);
    cudaFree(d_crc_shift);
    cudaFree(d_sample);
}

bool Layout::same_shape(const Layout& o) const {
    if (nt != o.nt) return false;
    for (uint32_t i = 0; i < nt; ++i) {
        if (types[i] != o.types[i] || dims[i] != o.dims[i]) return false;
        if (has_names && o.has_names && names[i] != o.names[i]) return false;
    }
    return true;
}

template <typename T>
static T* upload_vec(const std::vector<T>& v) {
    T* d = nullptr;
    size_t bytes = (v.size() ? v.size() : 1) * sizeof(T);
    DQTG_CUDA(cudaMalloc(&d, bytes));
    if (!v.empty()) DQTG_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    DQTG_CUDA(cudaStreamSynchronize(0));  // see alpha_tables: the DMA may still be in flight
    return d;
}

std::shared_ptr<Layout> make_layout(Engine* e, const dqtg_layout* l) {
    auto L = std::make_shared<Layout>();
    L->eng = e;
    L->nt = l->n_tensors;
    L->has_names = l->names != nullptr;
    size_t d = 0;
    std::vector<uint64_t> soff;
    for (uint32_t i = 0; i < L->nt; ++i) {
        uint8_t ty = l->types ? l->types[i] : 6;
        DQTG_REQUIRE(ty < kLayerTypes, DQTG_CORRUPT_INDEX, "bad tensor layer type");
        L->types.push_back(ty);
        uint8_t r = l->ranks[i];
        L->ranks.push_back(r);
        std::vector<uint64_t> dm(l->dims + d, l->dims + d + r);
        d += r;
        uint64_t n = 1;
        for (uint64_t x : dm) n *= x;
        L->dims.push_back(dm);
        L->numel.push_back(n);
        L->names.push_back(L->has_names ? std::string(l->names[i]) : std::string());
        L->off.push_back(L->Np);
        soff.push_back(L->N);
        L->Np += round_up(n, kAlign);
        L->N += n;
        L->tile0.push_back((uint32_t)L->tiles.size());
        for (uint64_t s = 0; s < n; s += kTile) {
            DQTG_REQUIRE(L->tiles.size() < 0xffffffffull, DQTG_ERROR, "checkpoint too large");
            L->tiles.push_back(Tile{i, (uint32_t)((n - s) < kTile ? (n - s) : kTile), L->off[i] + s});
        }
    }
    L->tile0.push_back((uint32_t)L->tiles.size());
    if (L->Np == 0) L->Np = kAlign;
    {
        constexpr size_t kSampleTiles = 192;
        std::vector<size_t> per(kLayerTypes, 0), seen(kLayerTypes, 0);
        for (const Tile& t : L->tiles) ++per[L->types[t.tensor]];
        for (const Tile& t : L->tiles) {
            const int lt = L->types[t.tensor];
            const size_t stride = std::max<size_t>(1, per[lt] / kSampleTiles);
            if (seen[lt]++ % stride == 0) L->sample_tiles.push_back(t);
        }
    }
    e->activate();
    L->d_tiles = upload_vec(L->tiles);
    L->d_sample = upload_vec(L->sample_tiles);
    L->d_types = upload_vec(L->types);
    L->d_off = upload_vec(L->off);
    L->d_numel = upload_vec(L->numel);
    L->d_tile0 = upload_vec(L->tile0);
    L->d_stream_off = upload_vec(soff);
    layout_crc_shift(*L);
    return L;
}

DevCkpt::~DevCkpt() {
    if (!own) return;
    cudaFree(w);
    cudaFree(ema);
    cudaFree(mag);
    cudaFree(sens);
}

uint32_t QState::max_levels() const {  // quantize.cpp:357-365
    uint32_t m = 0;
    for (uint32_t i = 0; i < L->nt; ++i) {
        uint32_t l = cb_len[L->types[i]] + 2;
        m = l > m ? l : m;
    }
    return m;
}

QState::~QState() {
    if (!eng) return;
    eng->dfree(d_cb);
    eng->dfree(d_levels);
    eng->dfree(d_ppos);
    eng->dfree(d_pval);
    eng->dfree(d_tile_hist);
}

Record::~Record() {
    if (eng) eng->dfree(d_buf);
}

}  // namespace dqtg
