// Host-side objects of the dqtg engine: engine/stream, alpha tables, layouts,
// device checkpoints, quantized states and records.
#pragma once

#include <atomic>
#include <map>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"

struct dqtg_comm;

namespace dqtg {

// Shared-memory histogram window: kWin buckets per sign plus the zero bucket.
constexpr int kWin = 2048;
constexpr int kWinSlots = 2 * kWin + 1;
// slot-table sentinels (AlphaTables::d_slot)
constexpr uint32_t kSlotSpill = 0xffffu, kSlotBad = 0xfffeu;
// Elements per tile of every streaming pass (a tile never crosses a tensor).
constexpr uint32_t kTile = 4096;

struct Tile {
    uint32_t tensor;
    uint32_t count;  // valid elements (<= kTile)
    uint64_t start;  // padded element offset of the first element
};

// Exact log-bucket tables for one alpha: the reference's
// bucket_index(x) (sketch.cpp:21-31) equals "smallest k with gamma^k >= x";
// with U[k] = largest float <= gamma^k this is an integer compare on float bits.
struct AlphaTables {
    double alpha, gamma, inv_ln_gamma, rep_scale;
    int64_t kmin, kmax, NB, HS;  // HS = 2*NB + 1 signed slots (neg desc, zero, pos asc)
    int64_t kw_lo;               // shared-memory window covers k in [kw_lo, kw_lo + kWin)
    uint32_t zbits;              // bits of the smallest float >= 1e-12 (zero bucket bound)
    float inv_log2_gamma;
    uint32_t* d_U = nullptr;     // U(k) for k in [kmin-1, kmax]
    double* d_key = nullptr;     // representative value per signed slot (sketch.cpp:33-37)
    float* d_keyf = nullptr;     // largest float <= key (threshold compare, §7 H2)
    std::vector<double> h_key;
    // Cell table: |x| bits >> cell_shift index cells of 2^cell_shift floats, each
    // spanning at most two buckets; entry = {k of the cell's first float, last
    // float bits of that bucket inside the cell (0xffffffff: whole cell)}.
    // bucket(a) = k + (a > split), one load instead of log2 + table probes.
    uint32_t cell_shift = 0;     // 0: no table (alpha too small), probe U instead
    uint2* d_cell = nullptr;
    uint2* d_slot = nullptr;     // same cells: window slot of |x| (lo | hi << 16, split)
    // compact slot table for |x| in [2^-32, 1): 4-byte entries staged in shared memory
    // by the streaming passes (lo slot | split offset << 13 | hi special << 30 |
    // lo special << 31; hi = lo + 1); null when the cells are too fine
    uint32_t* d_ctab = nullptr;
    uint32_t ctab_lo = 0, ctab_n = 0;
};

// Device view of the bucket tables passed by value to kernels.
struct BucketTab {
    const uint32_t* U;
    int64_t kmin, kmax, NB, kw_lo;
    uint32_t zbits;
    float inv_log2_gamma;
    const uint2* cell;  // null: probe U
    uint32_t cell_shift;
    const uint2* slot;  // window-slot table (null with cell)
    const uint32_t* ctab;  // compact table (global copy; kernels stage it in shared)
    uint32_t ctab_lo, ctab_n;
};

struct Engine;

// Counted reference to an engine.  Checkpoints, states and records keep their
// engine alive (their destructors free through its stream-ordered pool), so the
// owner may destroy the engine handle in any order relative to them (Python's
// cycle collector finalises objects in arbitrary order).
void engine_retain(Engine* e);
void engine_release(Engine* e);
class EngineRef {
    Engine* p_ = nullptr;

public:
    EngineRef() = default;
    EngineRef(Engine* e) : p_(e) {  // NOLINT: implicit by design
        if (p_) engine_retain(p_);
    }
    EngineRef(const EngineRef& o) : EngineRef(o.p_) {}
    EngineRef& operator=(Engine* e) {
        if (e) engine_retain(e);
        if (p_) engine_release(p_);
        p_ = e;
        return *this;
    }
    EngineRef& operator=(const EngineRef& o) { return *this = o.p_; }
    ~EngineRef() {
        if (p_) engine_release(p_);
    }
    Engine* get() const { return p_; }
    Engine* operator->() const { return p_; }
    Engine& operator*() const { return *p_; }
    operator Engine*() const { return p_; }  // NOLINT
    explicit operator bool() const { return p_ != nullptr; }
};

struct Layout {
    uint32_t nt = 0;
    std::vector<std::string> names;
    std::vector<uint8_t> types, ranks;
    std::vector<std::vector<uint64_t>> dims;
    std::vector<uint64_t> numel, off;  // off = padded element offset
    uint64_t N = 0, Np = 0;            // real / padded element totals
    bool has_names = false;
    std::vector<Tile> tiles;
    std::vector<uint32_t> tile0;  // first tile of each tensor (size nt+1)
    // every layer type's tiles, thinned to ~kSampleTiles (192) per type (threshold guess
    // of the fused score/partition pass, quantize.cu)
    std::vector<Tile> sample_tiles;
    Tile* d_sample = nullptr;
    // device copies
    Tile* d_tiles = nullptr;
    uint8_t* d_types = nullptr;      // per tensor
    uint64_t* d_off = nullptr;       // per tensor padded offset
    uint64_t* d_numel = nullptr;     // per tensor
    uint32_t* d_tile0 = nullptr;     // per tensor first tile (nt+1)
    uint64_t* d_stream_off = nullptr;  // per tensor unpadded element offset (CRC stream position)
    uint32_t* d_crc_shift = nullptr;   // per tile x^(8*bytes after the tile) mod P (lazily built)
    Engine* eng = nullptr;
    ~Layout();
    bool same_shape(const Layout& o) const;
};

std::shared_ptr<Layout> make_layout(Engine* e, const dqtg_layout* l);
void layout_crc_shift(Layout& L);  // per-tile CRC shift constants (codec.cu)
size_t pool_size_class(size_t n);   // rounding of stream-ordered pool requests

struct DevCkpt {
    EngineRef eng;
    std::shared_ptr<Layout> L;
    float* w = nullptr;
    float* ema = nullptr;  // derived-score mode
    float* mag = nullptr;  // explicit-score mode
    float* sens = nullptr;
    bool explicit_scores = false;
    bool has_sens = false;
    bool ema_seeded = false;
    bool own = true;  // false: w / ema are borrowed (the worker pool aliases caller buffers)
    ~DevCkpt();
};

struct QState {
    EngineRef eng;
    std::shared_ptr<Layout> L;
    uint64_t step = 0;
    dqtg_config cfg{};
    uint32_t cb_len[kLayerTypes] = {0};
    std::vector<float> cb[kLayerTypes];
    float* d_cb = nullptr;  // [7][cb_stride]
    uint32_t cb_stride = 0;
    uint16_t* d_levels = nullptr;  // padded flat
    uint64_t* d_ppos = nullptr;    // protected positions (tensor-local), tensor order
    uint16_t* d_pval = nullptr;
    // decoded states (alphabet <= 64): per tile, counts of each level value 0..63 -- the
    // next record's per-tile key counts, so its decode skips a pass over these levels
    uint32_t* d_tile_hist = nullptr;
    std::vector<uint64_t> prot_count, prot_off;  // per tensor
    uint64_t prot_total = 0;
    uint32_t max_levels() const;
    ~QState();
};

struct Record {
    EngineRef eng;
    uint8_t* d_buf = nullptr;
    uint64_t size = 0, cap = 0;
    std::vector<uint8_t> host;  // filled by decode-free host copies
    ~Record();
};

struct Engine {
    int device = 0;
    // intrusive count (EngineRef): the creator holds one reference; the last release
    // runs `deleter(owner)` (the C handle or the engine itself)
    std::atomic<int> refs{1};
    void* owner = nullptr;
    void (*deleter)(void*) = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // the engine's own stream-ordered pool: blocks freed by this engine are reused
    // by it alone, so engines on other streams never wait on this stream's work
    cudaMemPool_t pool = nullptr;
    // high-priority side stream for latency-critical few-CTA phases (k-means):
    // its CTAs are scheduled ahead of other streams' streaming passes
    cudaStream_t hi_stream = nullptr;
    cudaEvent_t hi_fork = nullptr, hi_join = nullptr;
    cudaStream_t hi();      // forks: hi_stream waits for `stream`
    void hi_done();         // joins: `stream` waits for hi_stream
    std::recursive_mutex mu;
    uint64_t launches = 0;
    uint64_t sync_n = 0, sync_ns = 0;  // host syncs and time blocked in them
    uint32_t* d_err = nullptr;
    std::map<uint64_t, std::unique_ptr<AlphaTables>> tables;
    // grow-only scratch buffers keyed by name
    std::map<std::string, std::pair<void*, size_t>> scratch;
    void* pinned = nullptr;
    size_t pinned_cap = 0;
    int num_sms = 148;
    // optional per-kernel CUDA-event timing (dqtg_engine_profile)
    bool profiling = false;
    struct Span {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Span> spans;
    std::vector<cudaEvent_t> event_pool;
    size_t ev_used = 0;
    cudaEvent_t take_event();
    // sharded quantize: per-checkpoint state between stage 2 and 3
    std::map<const void*, std::shared_ptr<void>> pending;

    ~Engine();
    void activate() const { DQTG_CUDA(cudaSetDevice(device)); }
    AlphaTables& alpha_tables(double alpha);
    BucketTab bucket_tab(const AlphaTables& t) const {
        return BucketTab{t.d_U, t.kmin, t.kmax, t.NB, t.kw_lo, t.zbits, t.inv_log2_gamma, t.d_cell,
                         t.cell_shift, t.d_slot, t.d_ctab, t.ctab_lo, t.ctab_n};
    }
    void* buf(const std::string& name, size_t bytes);  // scratch, contents undefined
    // release the scratch buffers whose names start with prefix ("" = all)
    void drop_scratch(const std::string& prefix);
    // stream-ordered pool allocations for per-step objects (states, records)
    void* dalloc(size_t bytes);
    void dfree(void* p);
    // Large per-step blocks (quantized level arrays) are recycled through a per-device
    // cache shared by all engines (engine.cu: BigCache): a freed block is kept with an
    // event on the freeing stream and handed to the next request of its size class
    // after the requesting stream waits on that event.  Growing the stream-ordered
    // pools mid-step mapped new memory on the host thread (measured 11-470 ms stalls
    // in the worker pool).
    void* host_pinned(size_t bytes);
    // Thread-safe pool of pinned host blocks (decode staging: a record's uploads are
    // packed into one block by the walk thread, so the device decode issues
    // asynchronous copies from pinned memory instead of staged pageable ones).
    std::mutex pin_mu;
    std::vector<std::pair<void*, size_t>> pin_free;
    void* pin_acquire(size_t bytes, size_t* cap);
    void pin_release(void* p, size_t cap);
    // Device->host read-back through a pinned staging arena: the copy is queued on
    // the engine stream and lands in `dst` at the next sync()/check_err().  (A
    // pageable destination would make the driver stage the copy synchronously,
    // which serialises host threads driving other engines.)
    void d2h(void* dst, const void* src, size_t bytes);
    // stream sync + pending read-backs (DQTG_SYNC_TRACE=1: call site, host time since
    // the previous sync returned, time blocked, on stderr)
    void sync(const char* fn = __builtin_FUNCTION(), int line = __builtin_LINE());
    // DQTG_SYNC_TRACE: host time since the previous sync / trace point (diagnostics)
    void tp(int line = __builtin_LINE());
    struct PendingD2H {
        void* dst;
        const void* staged;
        size_t n;
    };
    std::vector<PendingD2H> pend;
    std::vector<std::pair<uint8_t*, size_t>> stage_blocks;  // pinned; last = current
    size_t stage_used = 0;
    void launched(int n = 1) { launches += n; }
    void check_err(const char* fn = __builtin_FUNCTION(), int line = __builtin_LINE());  // reads + clears the device error word (syncs)
    // copy host-or-device memory into a device destination
    void to_device(void* dst, const void* src_any, size_t bytes);
    void from_device(void* dst_any, const void* src_dev, size_t bytes);
};

bool is_device_ptr(const void* p);
void throw_err_bits(uint32_t h);  // the Fail that check_err raises for device error bits h

void timeline_epoch(Engine& e);  // DQTG_TIMELINE reference event (first call records it)
void dump_timeline(Engine& e);   // recorded spans on stderr, relative to the epoch

// Raises a kernel's dynamic shared-memory limit to at least `bytes` and never
// lowers it: engines on several host threads launch the same kernels with
// different sizes, and a lowered limit would fail a concurrent launch.
void ensure_dyn_smem(const void* func, size_t bytes);

// Scoped CUDA-event span around one kernel launch (only when profiling).
struct KSpan {
    Engine& e;
    int idx = -1;
    KSpan(Engine& eng, const char* name) : e(eng) {
        if (!e.profiling) return;
        Engine::Span s{name, e.take_event(), e.take_event()};
        cudaEventRecord(s.a, e.stream);
        idx = (int)e.spans.size();
        e.spans.push_back(s);
    }
    ~KSpan() {
        if (idx >= 0) cudaEventRecord(e.spans[idx].b, e.stream);
    }
};
#define DQTG_SPAN(e, name) ::dqtg::KSpan dqtg_span_##__LINE__((e), (name))

// Fused pass C (codec.cu enc_tile_delta_kernel<true>): quantize(..., defer) stops
// before pass C and hands its inputs here; encode_record_ex then computes the target
// levels inside the DELTA tile pass (written to target.d_levels once, never re-read).
struct LtParams;
struct FuseC {
    const float* w = nullptr;
    const uint8_t* parts = nullptr;                     // 2 bits per element, element order
    const uint32_t* pbits = nullptr;                    // or: protected-element bitmap (no pruning)
    const float* lb = nullptr;                          // [7][lb_stride] level boundaries
    int lb_stride = 0;
    const uint32_t* cb_len = nullptr;                   // [7] (device)
    const unsigned long long* tile_prot_off = nullptr;  // first protected entry per tile
    uint16_t* levels = nullptr;                         // out: target levels
    uint64_t* ppos = nullptr;
    uint16_t* pval = nullptr;
    const LtParams* lp = nullptr;                       // [7] partition parameters (pass C kernel)
};
void run_pass_c(Engine& e, const DevCkpt& c, const FuseC& f, QState& q);
// whether compress_step may fuse pass C into the DELTA encoder (sparse encoder, B <= 64)
bool fused_c_enabled();

// memory: engine pools register for out-of-memory trimming (engine.cu)
void register_pool(cudaMemPool_t p, int device);
void unregister_pool(cudaMemPool_t p);
void trim_device_caches(int device);
cudaError_t dev_malloc(void** p, size_t bytes, int device);

// ---- pipeline entry points implemented across the .cu files ---------------
void sketch_build(Engine& e, const float* x_any, uint64_t n, double alpha, uint64_t* zero,
                  uint64_t* pos, uint64_t* neg);
// defer: pass C is not run; its inputs go to *defer (levels / protected entries of the
// returned state are written by the fused encoder, encode_record_ex(..., defer))
std::unique_ptr<QState> quantize(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                                 uint64_t seed, uint64_t step, FuseC* defer = nullptr);
std::unique_ptr<Record> encode_record(Engine& e, const QState* base, const QState& target,
                                      double quality);
std::unique_ptr<QState> decode_record(Engine& e, const uint8_t* rec, uint64_t n,
                                      const QState* base);
// records of a chain decoded in order (host walk of k+1 overlapping the device decode of k)
std::unique_ptr<QState> decode_chain(Engine& e, const uint8_t* const* recs, const uint64_t* sizes,
                                     uint32_t n, const QState* base,
                                     const std::function<void(uint32_t, const QState&)>& on_state);
void dequantize(Engine& e, const QState& q, float* out_dev_padded);
void dequantize_to(Engine& e, const QState& q, float* const* outs_dev);  // device array of nt outputs
// same step, layout, codebooks, levels and protected entries (compared on the device)
bool states_equal(Engine& e, const QState& a, const QState& b);
// crc32 (codec.cpp:275-306) of a state's level stream (u16 LE, tensor order)
uint32_t level_stream_crc(Engine& e, const Layout& L, const uint16_t* levels_dev);
void partition(Engine& e, const DevCkpt& c, const dqtg_config& cfg, uint8_t* const* masks);
double proxy_quality(Engine& e, const DevCkpt& orig, const float* recon_dev_padded);
void level_counts(Engine& e, const QState& q, uint64_t* counts, int lstride);
uint64_t shard_hist_len(Engine& e, const dqtg_config& cfg, int which);
void shard_stage1(Engine& e, const DevCkpt& c, const dqtg_config& cfg, unsigned long long* score_hist);
void shard_stage2(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                  const unsigned long long* score_hist, unsigned long long* value_hist);
std::unique_ptr<QState> shard_stage3(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                                     uint64_t seed, uint64_t step,
                                     const unsigned long long* value_hist);
// mode / payload_total: payload_bytes_* ablation sizes instead of a record (codec.cu)
std::unique_ptr<Record> encode_record_ex(Engine& e, const QState* base, const QState& target,
                                         double quality, uint32_t B_override, uint32_t nt_total,
                                         uint64_t* body_offset, int mode = 0,
                                         uint64_t* payload_total = nullptr,
                                         const FuseC* fc = nullptr,
                                         const std::function<void()>& on_levels = {});
// quantize + encode_delta_record against base (Chain::append): pass C fused into the
// DELTA encoder when possible; on_levels runs once the target levels are enqueued
std::unique_ptr<Record> compress_step(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                                      uint64_t seed, uint64_t step, const QState* base,
                                      double quality, std::unique_ptr<QState>& state_out,
                                      const std::function<void(QState*)>& on_levels = {});
void eval_batch(Engine& e, const DevCkpt& c, const dqtg_config* cfgs, const uint64_t* seeds,
                uint32_t m, double* quality, double* est);
void approx_kmeans(Engine& e, const float* values_any, uint64_t n, uint32_t k, double sigma,
                   double alpha, uint64_t seed, float* cb, uint32_t* len);
void kmeanspp_host_api(Engine& e, const double* pts, const double* w, uint64_t n, uint32_t k,
                       uint64_t seed, double* centers);
void lloyd_host_api(Engine& e, const double* pts, const double* w, uint64_t n, double* centers,
                    uint32_t k, double tol, uint32_t max_iter, uint32_t* iters);
double sq_loss_host_api(Engine& e, const double* pts, const double* w, uint64_t n,
                        const double* centers, uint32_t k);
void ema_update(Engine& e, float* ema_dev, const float* g_dev, uint64_t n, float beta);
void compute_scores(Engine& e, const float* w_dev, const float* ema_dev, uint64_t n, float* mag,
                    float* sens);
uint32_t crc32_device(Engine& e, const uint8_t* data_dev, uint64_t n);
void delta_kernel_api(Engine& e, const uint16_t* prev, const uint16_t* x, uint64_t n, uint32_t B,
                      uint16_t* out, bool apply);
// tensor-sharded step over an NCCL communicator (comm.cu)
std::unique_ptr<QState> sharded_quantize(Engine& e, dqtg_comm* comm, const DevCkpt& ck,
                                         const dqtg_config& cfg, uint64_t seed, uint64_t step);
std::unique_ptr<Record> sharded_encode(Engine& e, dqtg_comm* comm, const QState* base,
                                       const QState& target, double quality, uint32_t n_tensors_total);

}  // namespace dqtg
