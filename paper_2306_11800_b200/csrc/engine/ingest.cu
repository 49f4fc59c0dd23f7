// DQT1 checkpoint ingest straight into HBM: replaces read_checkpoint
// (src/tensor.cpp:110-149) + validate (src/tensor.cpp:63-75) on the compress path,
// where the reference parses the whole file into host vectors and the engine would
// then copy every tensor again.
//
// The tensor headers are parsed on the host with buffered preads (the data sections
// are skipped, not read), so every parse error of the reference surfaces before any
// tensor byte moves.  The data sections are then streamed file -> pinned staging ->
// HBM by T reader threads, each owning two staging chunks and a CUDA stream:
//
//   thread t:  pread chunk t      | H2D chunk t       |
//                     pread chunk t+T | H2D chunk t+T     | ...
//
// Chunks are 4 KiB-aligned file ranges, so the same loop runs with O_DIRECT (DMA from
// the device into pinned memory, no page-cache copy) when DQTG_INGEST_DIRECT is
// requested and the filesystem supports it.  A chunk's bytes are scattered to the
// padded per-tensor offsets of the device checkpoint with one cudaMemcpyAsync per
// tensor piece.  Finiteness (validate's NaN/Inf check) runs as one streaming kernel
// over the device copy; the first failing tensor is reported in the reference's
// validation order (name checks of earlier tensors first).
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstring>
#include <set>
#include <thread>

#include "handles.h"

namespace dqtg {
namespace {

constexpr uint64_t kIoAlign = 4096;

// buffered little-endian reader over a file descriptor (header fields only)
struct FileRd {
    int fd;
    uint64_t size, at = 0;
    std::vector<uint8_t> win;
    uint64_t win_off = 0, win_len = 0;
    FileRd(int f, uint64_t s) : fd(f), size(s), win(1 << 16) {}
    void need(uint64_t n) const {
        if (n > size - at) throw Fail(DQTG_TRUNCATED, "unexpected end of DQT1 file");
    }
    void raw(void* out, uint64_t n) {
        need(n);
        auto* o = static_cast<uint8_t*>(out);
        while (n) {
            if (at < win_off || at >= win_off + win_len) {
                win_off = at;
                ssize_t r = pread(fd, win.data(), win.size(), (off_t)at);
                if (r <= 0) throw Fail(DQTG_IO, std::string("read failed: ") + strerror(errno));
                win_len = (uint64_t)r;
            }
            uint64_t k = std::min<uint64_t>(n, win_off + win_len - at);
            memcpy(o, win.data() + (at - win_off), k);
            o += k;
            at += k;
            n -= k;
        }
    }
    template <class T>
    T le() {
        uint8_t b[sizeof(T)];
        raw(b, sizeof(T));
        uint64_t v = 0;
        for (size_t i = 0; i < sizeof(T); ++i) v |= uint64_t(b[i]) << (8 * i);
        return T(v);
    }
    std::string str() {
        uint16_t k = le<uint16_t>();
        std::string s(k, '\0');
        raw(s.data(), k);
        return s;
    }
};

struct Seg {
    uint64_t file_off, bytes, dev_off;  // dev_off in bytes from the checkpoint base
};

// first tensor (by index) holding a NaN/Inf; tiles are 16-B aligned and padded with
// zeros, so whole float4s are read
__global__ void __launch_bounds__(256) nonfinite_kernel(const float* __restrict__ w,
                                                         const Tile* __restrict__ tiles,
                                                         uint32_t ntiles, uint32_t* first) {
    for (uint32_t ti = blockIdx.x; ti < ntiles; ti += gridDim.x) {
        const Tile t = tiles[ti];
        const float4* p = reinterpret_cast<const float4*>(w + t.start);
        const uint32_t n4 = (t.count + 3) / 4;
        bool bad = false;
        for (uint32_t i = threadIdx.x; i < n4; i += blockDim.x) {
            float4 v = __ldcs(p + i);
            const uint32_t m = 0x7f800000u;
            bad |= ((__float_as_uint(v.x) & m) == m) | ((__float_as_uint(v.y) & m) == m) |
                   ((__float_as_uint(v.z) & m) == m) | ((__float_as_uint(v.w) & m) == m);
        }
        if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMin(first, t.tensor);
    }
}

void pread_full(int fd, uint8_t* dst, uint64_t n, uint64_t off, bool direct, uint64_t fsize) {
    // O_DIRECT reads stop at EOF with a short count; buffered reads loop until n
    while (n) {
        ssize_t r = pread(fd, dst, n, (off_t)off);
        if (r < 0) {
            if (errno == EINTR) continue;
            throw Fail(DQTG_IO, std::string("read failed: ") + strerror(errno));
        }
        if (r == 0) {
            if (direct && off >= fsize) return;
            throw Fail(DQTG_TRUNCATED, "DQT1 file shrank while reading");
        }
        dst += r;
        off += (uint64_t)r;
        n -= (uint64_t)r;
    }
}

}  // namespace

struct Dqt1Info {
    uint64_t step = 0;
    std::vector<uint8_t> meta;  // raw meta section: u32 nmeta | {str key | u32 len | bytes}
};

// Parses + uploads `path`; returns the new device checkpoint.
static dqtg_ckpt* ingest_dqt1(Engine& e, const char* path, int threads, bool direct,
                              Dqt1Info& info) {
    e.activate();
    int fd = open(path, O_RDONLY | O_CLOEXEC);
    if (fd < 0) throw Fail(DQTG_IO, std::string("cannot open ") + path + ": " + strerror(errno));
    struct Closer {
        int fd;
        ~Closer() { close(fd); }
    } closer{fd};
    struct stat st;
    if (fstat(fd, &st) != 0) throw Fail(DQTG_IO, std::string("cannot stat ") + path);
    const uint64_t fsize = (uint64_t)st.st_size;

    // ---- header parse (read_checkpoint order of checks) ----
    FileRd r(fd, fsize);
    char magic[4];
    r.raw(magic, 4);
    if (memcmp(magic, "DQT1", 4) != 0) throw Fail(DQTG_BAD_MAGIC, std::string("not a DQT1 file: ") + path);
    uint32_t version = r.le<uint32_t>();
    if (version != 1) throw Fail(DQTG_IO, "unsupported DQT1 version " + std::to_string(version));
    info.step = r.le<uint64_t>();
    const uint64_t meta0 = r.at;
    uint32_t nmeta = r.le<uint32_t>();
    for (uint32_t i = 0; i < nmeta; ++i) {
        r.str();
        uint32_t n = r.le<uint32_t>();
        r.need(n);
        r.at += n;
    }
    info.meta.resize(r.at - meta0);
    {
        uint64_t save = r.at;
        r.at = meta0;
        r.raw(info.meta.data(), info.meta.size());
        r.at = save;
    }
    uint32_t nt = r.le<uint32_t>();
    std::vector<std::string> names;
    std::vector<uint8_t> types, ranks;
    std::vector<uint64_t> dims, file_off, numel;
    for (uint32_t i = 0; i < nt; ++i) {
        std::string name = r.str();
        uint8_t lt = r.le<uint8_t>();
        if (lt >= kLayerTypes) throw Fail(DQTG_IO, "bad layer type " + std::to_string(lt));
        uint8_t rank = r.le<uint8_t>();
        if (rank == 0) throw Fail(DQTG_SHAPE_MISMATCH, "tensor " + name + " has rank 0");
        uint64_t n = 1;
        for (uint8_t k = 0; k < rank; ++k) {
            uint64_t d = r.le<uint64_t>();
            dims.push_back(d);
            n *= d;  // wraps like NamedTensor::size()
        }
        const uint64_t rem = fsize - r.at;
        if (n > rem / 4 + 1 || n * 4 > rem)
            throw Fail(DQTG_TRUNCATED, "tensor " + name + " exceeds file size");
        names.push_back(std::move(name));
        types.push_back(lt);
        ranks.push_back(rank);
        numel.push_back(n);
        file_off.push_back(r.at);
        r.at += n * 4;
    }
    if (r.at != fsize) throw Fail(DQTG_IO, std::string("trailing bytes after last tensor in ") + path);
    // validate(): first name problem in tensor order (data checked on the device)
    uint32_t name_bad = nt;
    std::string name_msg;
    {
        std::set<std::string> seen;
        for (uint32_t i = 0; i < nt && name_bad == nt; ++i) {
            if (names[i].empty()) {
                name_bad = i;
                name_msg = "tensor with empty name";
            } else if (!seen.insert(names[i]).second) {
                name_bad = i;
                name_msg = "duplicate tensor name: " + names[i];
            }
        }
    }

    // ---- device checkpoint ----
    std::vector<const char*> cn(nt);
    for (uint32_t i = 0; i < nt; ++i) cn[i] = names[i].c_str();
    dqtg_layout lay{nt, cn.data(), types.data(), ranks.data(), dims.data()};
    auto* c = new dqtg_ckpt();
    std::unique_ptr<dqtg_ckpt> own(c);
    c->c.eng = &e;
    c->c.L = make_layout(&e, &lay);
    const Layout& L = *c->c.L;
    DQTG_CUDA(cudaMalloc(&c->c.w, L.Np * 4));
    DQTG_CUDA(cudaMemsetAsync(c->c.w, 0, L.Np * 4, e.stream));  // tensor padding stays zero
    cudaEvent_t zeroed;
    DQTG_CUDA(cudaEventCreateWithFlags(&zeroed, cudaEventDisableTiming));
    DQTG_CUDA(cudaEventRecord(zeroed, e.stream));

    std::vector<Seg> segs;
    for (uint32_t i = 0; i < nt; ++i)
        if (numel[i]) segs.push_back(Seg{file_off[i], numel[i] * 4, L.off[i] * 4});

    uint64_t chunk = 4ull << 20;
    if (const char* s = getenv("DQTG_INGEST_CHUNK_MB")) chunk = std::max<uint64_t>(1, atoll(s)) << 20;
    const uint64_t lo = segs.empty() ? 0 : segs.front().file_off / kIoAlign * kIoAlign;
    const uint64_t hi = segs.empty() ? 0 : segs.back().file_off + segs.back().bytes;
    const uint64_t nchunks = (hi - lo + chunk - 1) / chunk;
    if (threads <= 0) threads = 8;
    threads = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)threads, nchunks));

    int dfd = -1;
    if (direct && nchunks) dfd = open(path, O_RDONLY | O_CLOEXEC | O_DIRECT);
    struct Closer2 {
        int fd;
        ~Closer2() {
            if (fd >= 0) close(fd);
        }
    } closer2{dfd};

    // 2 staging chunks per reader thread (+ one alignment page for O_DIRECT tails)
    const uint64_t slot = chunk + kIoAlign;
    uint8_t* pin = nchunks ? static_cast<uint8_t*>(e.host_pinned(slot * 2 * threads)) : nullptr;
    uint8_t* base = reinterpret_cast<uint8_t*>(c->c.w);

    std::atomic<bool> failed{false};
    std::string err_msg;
    dqtg_status err_code = DQTG_OK;
    std::mutex err_mu;
    std::vector<cudaStream_t> streams(threads);
    std::vector<cudaEvent_t> done(threads * 2);
    for (int t = 0; t < threads; ++t) {
        DQTG_CUDA(cudaStreamCreateWithFlags(&streams[t], cudaStreamNonBlocking));
        DQTG_CUDA(cudaStreamWaitEvent(streams[t], zeroed, 0));
        for (int b = 0; b < 2; ++b) DQTG_CUDA(cudaEventCreateWithFlags(&done[t * 2 + b], cudaEventDisableTiming));
    }
    auto reader = [&](int t) {
        try {
            cudaSetDevice(e.device);
            bool use_direct = dfd >= 0;
            uint64_t local = 0;
            for (uint64_t ci = (uint64_t)t; ci < nchunks && !failed.load(); ci += threads, ++local) {
                const int b = (int)(local & 1);
                uint8_t* buf = pin + slot * (2 * t + b);
                if (local >= 2) DQTG_CUDA(cudaEventSynchronize(done[t * 2 + b]));
                const uint64_t a = lo + ci * chunk, z = std::min(hi, a + chunk);
                if (use_direct) {
                    const uint64_t zz = (z + kIoAlign - 1) / kIoAlign * kIoAlign;
                    ssize_t probe = pread(dfd, buf, zz - a, (off_t)a);
                    if (probe < 0 && errno == EINVAL) {
                        use_direct = false;  // filesystem without O_DIRECT support
                    } else {
                        if (probe < 0) throw Fail(DQTG_IO, std::string("read failed: ") + strerror(errno));
                        if ((uint64_t)probe < z - a)
                            pread_full(fd, buf + probe, z - a - probe, a + probe, false, fsize);
                    }
                }
                if (!use_direct) pread_full(fd, buf, z - a, a, false, fsize);
                // scatter the chunk's tensor pieces
                auto it = std::upper_bound(segs.begin(), segs.end(), a,
                                           [](uint64_t x, const Seg& s) { return x < s.file_off + s.bytes; });
                for (; it != segs.end() && it->file_off < z; ++it) {
                    const uint64_t s0 = std::max(a, it->file_off);
                    const uint64_t s1 = std::min(z, it->file_off + it->bytes);
                    DQTG_CUDA(cudaMemcpyAsync(base + it->dev_off + (s0 - it->file_off), buf + (s0 - a), s1 - s0,
                                              cudaMemcpyHostToDevice, streams[t]));
                }
                DQTG_CUDA(cudaEventRecord(done[t * 2 + b], streams[t]));
            }
        } catch (const Fail& x) {
            std::lock_guard<std::mutex> g(err_mu);
            if (!failed.exchange(true)) {
                err_code = x.code;
                err_msg = x.what();
            }
        } catch (const std::exception& x) {
            std::lock_guard<std::mutex> g(err_mu);
            if (!failed.exchange(true)) {
                err_code = DQTG_ERROR;
                err_msg = x.what();
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(reader, t);
    if (nchunks) reader(0);
    for (auto& th : pool) th.join();
    for (int t = 0; t < threads; ++t) {
        cudaEvent_t j;
        cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
        cudaEventRecord(j, streams[t]);
        cudaStreamWaitEvent(e.stream, j, 0);
        cudaEventDestroy(j);
    }
    // the staging chunks must not be reused before the copies drained
    for (int t = 0; t < threads; ++t) {
        cudaStreamSynchronize(streams[t]);
        cudaStreamDestroy(streams[t]);
        cudaEventDestroy(done[t * 2]);
        cudaEventDestroy(done[t * 2 + 1]);
    }
    cudaEventDestroy(zeroed);
    if (failed) throw Fail(err_code, err_msg);

    // ---- validate(): finiteness on the device ----
    uint32_t first = nt;
    if (!L.tiles.empty()) {
        auto* d_first = static_cast<uint32_t*>(e.buf("ingest.first", 4));
        DQTG_CUDA(cudaMemcpyAsync(d_first, &first, 4, cudaMemcpyHostToDevice, e.stream));
        const uint32_t ntiles = (uint32_t)L.tiles.size();
        const uint32_t grid = std::min<uint32_t>(ntiles, (uint32_t)e.num_sms * 8);
        {
            DQTG_SPAN(e, "nonfinite");
            nonfinite_kernel<<<grid, 256, 0, e.stream>>>(c->c.w, L.d_tiles, ntiles, d_first);
        }
        e.launched();
        DQTG_CUDA(cudaGetLastError());
        e.d2h(&first, d_first, 4);
    }
    e.sync();
    if (name_bad < nt && name_bad <= first) throw Fail(DQTG_IO, name_msg);
    if (first < nt) throw Fail(DQTG_NON_FINITE, "tensor " + names[first] + " contains NaN/Inf");
    return own.release();
}

}  // namespace dqtg

using namespace dqtg;

extern "C" dqtg_status dqtg_ckpt_read_dqt1(dqtg_engine* h, const char* path, int flags, int threads,
                                           dqtg_ckpt** out, uint64_t* step, uint8_t* meta,
                                           uint64_t meta_cap, uint64_t* meta_len) {
    try {
        std::lock_guard<std::recursive_mutex> lk(h->e.mu);
        Dqt1Info info;
        const bool direct = (flags & DQTG_INGEST_DIRECT) != 0;
        dqtg_ckpt* c = ingest_dqt1(h->e, path, threads, direct, info);
        if (step) *step = info.step;
        if (meta_len) *meta_len = info.meta.size();
        if (meta && meta_cap) memcpy(meta, info.meta.data(), std::min<uint64_t>(meta_cap, info.meta.size()));
        *out = c;
        return DQTG_OK;
    } catch (const Fail& x) {
        set_last_error(x.what());
        return x.code;
    } catch (const std::exception& x) {
        set_last_error(x.what());
        return DQTG_ERROR;
    }
}

extern "C" uint32_t dqtg_ckpt_tensor_count(const dqtg_ckpt* c) { return c->c.L->nt; }

extern "C" dqtg_status dqtg_ckpt_tensor_info(const dqtg_ckpt* c, uint32_t i, char* name, uint64_t cap,
                                             uint8_t* type, uint8_t* rank, uint64_t* dims) {
    const Layout& L = *c->c.L;
    if (i >= L.nt) {
        set_last_error("tensor index out of range");
        return DQTG_ERROR;
    }
    if (name && cap) {
        const size_t k = std::min<size_t>(L.names[i].size(), cap - 1);
        memcpy(name, L.names[i].data(), k);
        name[k] = 0;
    }
    if (type) *type = L.types[i];
    if (rank) *rank = L.ranks[i];
    if (dims)
        for (size_t r = 0; r < L.dims[i].size(); ++r) dims[r] = L.dims[i][r];
    return DQTG_OK;
}

extern "C" dqtg_status dqtg_ckpt_download(dqtg_ckpt* c, float* const* out_any) {
    try {
        Engine& e = *c->c.eng;
        std::lock_guard<std::recursive_mutex> lk(e.mu);
        e.activate();
        const Layout& L = *c->c.L;
        for (uint32_t i = 0; i < L.nt; ++i)
            if (L.numel[i] && out_any[i]) e.from_device(out_any[i], c->c.w + L.off[i], L.numel[i] * 4);
        e.sync();
        return DQTG_OK;
    } catch (const Fail& x) {
        set_last_error(x.what());
        return x.code;
    } catch (const std::exception& x) {
        set_last_error(x.what());
        return DQTG_ERROR;
    }
}

// apply_layer_rules (src/tensor.cpp:225-227) on a device checkpoint: same tensors and
// offsets, new layer types (states already quantized keep their own layout)
extern "C" dqtg_status dqtg_ckpt_set_types(dqtg_ckpt* c, const uint8_t* types) {
    try {
        Engine& e = *c->c.eng;
        std::lock_guard<std::recursive_mutex> lk(e.mu);
        const Layout& L = *c->c.L;
        std::vector<const char*> cn(L.nt);
        std::vector<uint64_t> dims;
        for (uint32_t i = 0; i < L.nt; ++i) {
            cn[i] = L.names[i].c_str();
            dims.insert(dims.end(), L.dims[i].begin(), L.dims[i].end());
        }
        dqtg_layout lay{L.nt, L.has_names ? cn.data() : nullptr, types, L.ranks.data(), dims.data()};
        auto L2 = make_layout(&e, &lay);
        c->c.L = std::move(L2);
        return DQTG_OK;
    } catch (const Fail& x) {
        set_last_error(x.what());
        return x.code;
    } catch (const std::exception& x) {
        set_last_error(x.what());
        return DQTG_ERROR;
    }
}
