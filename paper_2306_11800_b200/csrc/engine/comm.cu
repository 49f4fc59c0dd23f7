// Multi-GPU data plane of the sharded compress step:
// an NCCL communicator owned by the engine library and one C-ABI call that runs a
// whole tensor-sharded Chain::append step (chain.cpp:86-129) on this rank:
//
//   stage 1  pass A of this rank's tensors      -> ncclAllReduce(u64 sum) score histograms
//   stage 2  pass B with the global thresholds  -> ncclAllReduce(u64 sum) value histograms
//   stage 3  codebooks from the global histograms (identical on every rank), pass C
//   encode   this rank's tensor blocks with the global alphabet and tensor count
//   gather   per-rank (body bytes, CRC, level-stream bytes) by ncclAllGather; the
//            bodies by ncclSend/ncclRecv straight into rank 0's record buffer; rank 0
//            combines the CRCs (crc32_combine) -> the single-GPU record, byte for byte
//
// Every collective is queued on the engine's stream: no host synchronisation between
// the stages (the host reads back only what sizes buffers: the global alphabet and
// the body lengths).  NCCL is loaded at run time (dlopen of libnccl.so.2): inside a
// PyTorch process that is the library torch already mapped; elsewhere the system one.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "crc.cuh"
#include "engine.h"
#include "handles.h"

using namespace dqtg;

namespace {

struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp && n.why.empty()) n.why = std::string("libnccl lacks ") + name;
        };
        sym(n.GetUniqueId, "ncclGetUniqueId");
        sym(n.CommInitRank, "ncclCommInitRank");
        sym(n.CommDestroy, "ncclCommDestroy");
        sym(n.AllReduce, "ncclAllReduce");
        sym(n.AllGather, "ncclAllGather");
        sym(n.Send, "ncclSend");
        sym(n.Recv, "ncclRecv");
        sym(n.GroupStart, "ncclGroupStart");
        sym(n.GroupEnd, "ncclGroupEnd");
        sym(n.GetErrorString, "ncclGetErrorString");
        n.ok = n.why.empty();
    });
    if (!n.ok) throw Fail(DQTG_ERROR, n.why);
    return n;
}

#define DQTG_NCCL(call)                                                                  \
    do {                                                                                 \
        const ncclResult_t r_ = (call);                                                  \
        if (r_ != ncclSuccess)                                                           \
            throw Fail(DQTG_ERROR, std::string("NCCL: ") + #call + ": " +                \
                                       nccl().GetErrorString(r_));                       \
    } while (0)

template <typename F>
dqtg_status guarded(F&& f) {
    try {
        f();
        return DQTG_OK;
    } catch (const Fail& x) {
        set_last_error(x.what());
        return x.code;
    } catch (const std::exception& x) {
        set_last_error(x.what());
        return DQTG_ERROR;
    }
}

uint32_t crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {  // zlib rule
    static const CrcX2N x2n = crc_x2n_table();
    return len2 ? crc_multmodp(crc_x2nmodp(x2n.t, len2, 3), crc1) ^ crc2 : crc1;
}

}  // namespace

struct dqtg_comm {
    ncclComm_t c = nullptr;
    int nranks = 1, rank = 0, device = 0;
};

namespace dqtg {

// stages 1-3 of the sharded quantize with the two histogram all-reduces on the
// engine stream (caller holds the engine lock)
std::unique_ptr<QState> sharded_quantize(Engine& e, dqtg_comm* comm, const DevCkpt& ck,
                                         const dqtg_config& cfg, uint64_t seed, uint64_t step) {
    const Nccl& N = nccl();
    cudaStream_t st = e.stream;
    const int R = comm->nranks;
    const uint64_t ns = shard_hist_len(e, cfg, 0), nv = shard_hist_len(e, cfg, 1);
    auto* score = (unsigned long long*)e.buf("cm.score", ns * 8);
    auto* value = (unsigned long long*)e.buf("cm.value", nv * 8);
    shard_stage1(e, ck, cfg, score);
    if (R > 1) DQTG_NCCL(N.AllReduce(score, score, ns, ncclUint64, ncclSum, comm->c, st));
    shard_stage2(e, ck, cfg, score, value);
    if (R > 1) DQTG_NCCL(N.AllReduce(value, value, nv, ncclUint64, ncclSum, comm->c, st));
    return shard_stage3(e, ck, cfg, seed, step, value);
}

// this rank's blocks with the global alphabet and tensor count; rank 0 gets the
// whole record (bodies by ncclSend/Recv, CRCs combined), other ranks null
std::unique_ptr<Record> sharded_encode(Engine& e, dqtg_comm* comm, const QState* bq,
                                       const QState& q, double quality, uint32_t n_tensors_total) {
    const Nccl& N = nccl();
    cudaStream_t st = e.stream;
    const int R = comm->nranks, me = comm->rank;
    // global alphabet (max over ranks, codec.cpp:416-417) and tensor count
    auto* meta = (unsigned long long*)e.buf("cm.meta", 32);
    unsigned long long hm[2] = {std::max<unsigned long long>(q.max_levels(), bq ? bq->max_levels() : 0),
                                q.L->nt};
    DQTG_CUDA(cudaMemcpyAsync(meta, hm, 16, cudaMemcpyHostToDevice, st));
    if (R > 1) {
        DQTG_NCCL(N.AllReduce(meta, meta, 1, ncclUint64, ncclMax, comm->c, st));
        DQTG_NCCL(N.AllReduce(meta + 1, meta + 1, 1, ncclUint64, ncclSum, comm->c, st));
    }
    e.from_device(hm, meta, 16);
    e.sync();
    const uint32_t gB = (uint32_t)std::max<unsigned long long>(2, hm[0]);
    const uint32_t gnt = n_tensors_total ? n_tensors_total : (uint32_t)hm[1];
    uint64_t body_off = 0;
    auto rec = encode_record_ex(e, bq, q, quality, gB, gnt, &body_off);
    // per rank: body bytes, CRC of its level stream, level-stream bytes
    const uint64_t body = rec->size - body_off - 4;
    uint32_t crc = 0;
    e.from_device(&crc, rec->d_buf + rec->size - 4, 4);
    e.sync();
    auto* info = (unsigned long long*)e.buf("cm.info", (size_t)R * 24 + 24);
    unsigned long long mine[3] = {body, crc, 2ull * q.L->N};
    DQTG_CUDA(cudaMemcpyAsync(info + (size_t)me * 3, mine, 24, cudaMemcpyHostToDevice, st));
    if (R > 1) DQTG_NCCL(N.AllGather(info + (size_t)me * 3, info, 3, ncclUint64, comm->c, st));
    std::vector<unsigned long long> all((size_t)R * 3);
    e.from_device(all.data(), info, all.size() * 8);
    e.sync();
    std::unique_ptr<Record> full;
    if (me == 0) {
        uint64_t total = body_off + 4;
        for (int r = 0; r < R; ++r) total += all[(size_t)r * 3];
        full = std::make_unique<Record>();
        full->eng = &e;
        full->size = total;
        full->cap = round_up(total, 16) + 16;
        full->d_buf = (uint8_t*)e.dalloc(full->cap);
        DQTG_CUDA(cudaMemcpyAsync(full->d_buf, rec->d_buf, body_off + body, cudaMemcpyDeviceToDevice, st));
    }
    if (R > 1) {  // bodies in rank order behind rank 0's prefix and body
        DQTG_NCCL(N.GroupStart());
        if (me == 0) {
            uint64_t at = body_off + body;
            for (int r = 1; r < R; ++r) {
                const uint64_t n = all[(size_t)r * 3];
                if (n) DQTG_NCCL(N.Recv(full->d_buf + at, n, ncclUint8, r, comm->c, st));
                at += n;
            }
        } else if (body) {
            DQTG_NCCL(N.Send(rec->d_buf + body_off, body, ncclUint8, 0, comm->c, st));
        }
        DQTG_NCCL(N.GroupEnd());
    }
    if (me == 0) {  // crc32 of the whole level stream, combined in rank order
        uint32_t c = (uint32_t)all[1];
        for (int r = 1; r < R; ++r)
            c = crc32_combine(c, (uint32_t)all[(size_t)r * 3 + 1], all[(size_t)r * 3 + 2]);
        const uint8_t b[4] = {(uint8_t)c, (uint8_t)(c >> 8), (uint8_t)(c >> 16), (uint8_t)(c >> 24)};
        DQTG_CUDA(cudaMemcpyAsync(full->d_buf + full->size - 4, b, 4, cudaMemcpyHostToDevice, st));
    }
    e.sync();  // the local record's memory returns to the pool after the sends
    return full;
}

}  // namespace dqtg

extern "C" {

dqtg_status dqtg_comm_unique_id(uint8_t* id_out) {
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == DQTG_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        DQTG_NCCL(nccl().GetUniqueId(&id));
        memcpy(id_out, &id, sizeof(id));
    });
}

dqtg_status dqtg_comm_init(dqtg_engine* h, const uint8_t* id, int nranks, int rank,
                           dqtg_comm** out) {
    return guarded([&] {
        DQTG_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, DQTG_ERROR, "bad rank / size");
        h->e.activate();
        ncclUniqueId uid;
        memcpy(&uid, id, sizeof(uid));
        auto c = std::make_unique<dqtg_comm>();
        c->nranks = nranks;
        c->rank = rank;
        c->device = h->e.device;
        DQTG_NCCL(nccl().CommInitRank(&c->c, nranks, uid, rank));
        *out = c.release();
    });
}

void dqtg_comm_destroy(dqtg_comm* c) {
    if (!c) return;
    if (c->c) {
        cudaSetDevice(c->device);
        nccl().CommDestroy(c->c);
    }
    delete c;
}

int dqtg_comm_rank(const dqtg_comm* c) { return c->rank; }
int dqtg_comm_size(const dqtg_comm* c) { return c->nranks; }

dqtg_status dqtg_comm_allreduce_u64(dqtg_engine* h, dqtg_comm* c, uint64_t* buf_dev, uint64_t n) {
    return guarded([&] {
        std::lock_guard<std::recursive_mutex> lk(h->e.mu);
        h->e.activate();
        DQTG_NCCL(nccl().AllReduce(buf_dev, buf_dev, n, ncclUint64, ncclSum, c->c, h->e.stream));
    });
}

dqtg_status dqtg_compress_sharded(dqtg_engine* h, dqtg_comm* comm, const dqtg_ckpt* ck,
                                  const dqtg_config* cfg, uint64_t seed, uint64_t step,
                                  const dqtg_qstate* base, double quality,
                                  uint32_t n_tensors_total, dqtg_qstate** state_out,
                                  dqtg_record** record_out) {
    return guarded([&] {
        Engine& e = h->e;
        std::lock_guard<std::recursive_mutex> lk(e.mu);
        e.activate();
        auto q = sharded_quantize(e, comm, ck->c, *cfg, seed, step);
        auto full = sharded_encode(e, comm, base ? base->q.get() : nullptr, *q, quality, n_tensors_total);
        auto* s = new dqtg_qstate();
        s->q = std::move(q);
        *state_out = s;
        *record_out = nullptr;
        if (full) {
            auto* rr = new dqtg_record();
            rr->r = std::move(full);
            *record_out = rr;
        }
    });
}

}  // extern "C"
