// decode_delta_record on the device (reference codec.cpp:459-597, DQDR v1 layout in
// SURVEY.md Appendix B).
//
//   host   walk the record structure: header, codebooks, per tensor the static
//          prefix, protected entries and the (bucket, elems, nsyms, table, bytes)
//          header of every group; canonical decode limits per group
//   H1     every group's bitstream is cut into 4096-bit chunks, one thread per
//          chunk.  Threads start decoding at their chunk's nominal start; a chunk's
//          true start is the first codeword boundary the previous chunk's decode
//          reaches at or past it.  Canonical Huffman codes self-synchronise within
//          a few codewords, so a handful of passes (each re-decoding only chunks
//          whose start moved) converge; symbols per chunk -> scan -> symbol index
//   H2     decode again, writing symbols (-v run values, run lengths) in order
//   R      RLE expansion (codec.cpp:91-107): symbols -> element counts -> scan ->
//          run heads marked, max-scan fills every element with its run's value
//   U      unrearrange (codec.cpp:56-77): stable rank of every element among the
//          elements with the same previous level (per-tile match ranks + per-key
//          prefixes over tiles) indexes its group's delta; cur = (prev - d) mod B
//   C      CRC-32 of the decoded level stream against the stored one
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"

namespace dqtg {

constexpr uint32_t kChunkBits = 512;
constexpr int kBnd = 24;  // codeword starts recorded per chunk (sync shortcut)
constexpr int kMaxCodeLen = 64;

struct GroupDesc {
    uint64_t elem_off;  // dense rearranged position of the group's first element
    uint64_t elems;
    uint64_t nsyms;
    uint64_t sym_off;   // first symbol in the symbol array
    uint64_t bit_off;   // absolute bit offset of the stream in the device record
    uint64_t nbits;
    uint32_t tab_off, tsize;
    uint32_t chunk0, nchunks;
    uint32_t minlen, maxlen;
    uint32_t lim_off;   // decode tables: entries for code lengths minlen..maxlen
    uint32_t lut;       // the group's index: its 1024-entry first-10-bits table
};

struct ChunkDesc {
    uint32_t group;
    uint32_t local;  // chunk index inside its group
};

// the delta base as the host walk needs it: its step and tensor table
struct BaseInfo {
    uint64_t step = 0;
    std::vector<std::string> names;
    std::vector<uint8_t> types, ranks;
    std::vector<std::vector<uint64_t>> dims;
};

constexpr size_t kPinStageMax = (size_t)96 << 20;

// a record after the host walk (decode_plan), before the device decode (decode_run)
struct DecodePlan {
    std::vector<uint8_t> host_copy;  // the record, when it was handed over in device memory
    const uint8_t* h = nullptr;
    uint64_t n = 0;
    bool has_base = false;
    uint64_t target_step = 0;
    uint32_t B = 0, nt = 0;
    std::unique_ptr<QState> q;  // step, config, codebooks
    std::vector<std::string> names;
    std::vector<uint8_t> types, ranks;
    std::vector<uint64_t> dims;
    std::vector<uint64_t> ppos;  // protected entries of all tensors, flat (one upload)
    std::vector<uint16_t> pval;
    std::vector<uint64_t> pcount;  // per tensor
    std::vector<GroupDesc> groups;
    std::vector<ChunkDesc> chunks;
    std::vector<int64_t> tab_sym;
    std::vector<uint8_t> tab_len;
    std::vector<unsigned long long> rec_elems, gstart_h;
    std::vector<uint64_t> lim, first;
    std::vector<uint32_t> lbase;
    uint64_t sym_total = 0;
    std::string deferred_index;
    uint32_t stored_crc = 0;
    // the device decode's uploads packed into one pinned block by the walk
    Engine* eng = nullptr;
    void* pin = nullptr;
    size_t pin_cap = 0;
    size_t o_rec = 0, o_groups = 0, o_chunks = 0, o_sym = 0, o_lim = 0, o_first = 0, o_lbase = 0,
           o_relems = 0, o_gstart = 0, o_ppos = 0, o_pval = 0;
    ~DecodePlan() {
        if (pin) eng->pin_release(pin, pin_cap);
    }
    void stage() {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t at = o;
            o += (bytes + 15) & ~(size_t)15;
            return at;
        };
        o_rec = take(n);
        o_groups = take(groups.size() * sizeof(GroupDesc));
        o_chunks = take(chunks.size() * sizeof(ChunkDesc));
        o_sym = take(tab_sym.size() * 8);
        o_lim = take(lim.size() * 8);
        o_first = take(first.size() * 8);
        o_lbase = take(lbase.size() * 4);
        o_relems = take(rec_elems.size() * 8);
        o_gstart = take(gstart_h.size() * 8);
        o_ppos = take(ppos.size() * 8);
        o_pval = take(pval.size() * 2);
        // very large records (billion-element shards) upload from the walk's own
        // vectors: packing hundreds of MB into fresh pinned blocks costs more than the
        // pageable copies save
        if (o > kPinStageMax) return;
        pin = eng->pin_acquire(o + 16, &pin_cap);
        uint8_t* S = (uint8_t*)pin;
        auto put = [&](size_t at, const void* src, size_t bytes) {
            if (bytes) memcpy(S + at, src, bytes);
        };
        put(o_rec, h, n);
        put(o_groups, groups.data(), groups.size() * sizeof(GroupDesc));
        put(o_chunks, chunks.data(), chunks.size() * sizeof(ChunkDesc));
        put(o_sym, tab_sym.data(), tab_sym.size() * 8);
        put(o_lim, lim.data(), lim.size() * 8);
        put(o_first, first.data(), first.size() * 8);
        put(o_lbase, lbase.data(), lbase.size() * 4);
        put(o_relems, rec_elems.data(), rec_elems.size() * 8);
        put(o_gstart, gstart_h.data(), gstart_h.size() * 8);
        put(o_ppos, ppos.data(), ppos.size() * 8);
        put(o_pval, pval.data(), pval.size() * 2);
    }
};

// ---- bit access: MSB-first stream (codec.cpp:111-122) -------------------------
__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
}
// 64 bits starting at absolute bit position p (record padded by 16 zero bytes)
__device__ __forceinline__ uint64_t peek64(const uint64_t* rec64, uint64_t p) {
    const uint64_t w = p >> 6;
    const uint32_t s = (uint32_t)(p & 63);
    const uint64_t a = bswap64(__ldg(rec64 + w)), b = bswap64(__ldg(rec64 + w + 1));
    return s ? (a << s) | (b >> (64 - s)) : a;
}

struct DecTabs {
    const uint64_t* lim;    // left-aligned exclusive limit of codes of length <= L
    const uint64_t* first;  // canonical first code of length L
    const uint32_t* base;   // table index of the first symbol of length L
    const int64_t* syms;
    const uint32_t* lut;    // per group, indexed by the next 10 bits: idx << 8 | length
                            // for codes of <= 10 bits, 0 otherwise
};
constexpr int kLutBits = 10;

// Decodes the codeword at bit p (relative to the group stream); returns its length
// and the table index, or length 0 for an invalid code.
__device__ __forceinline__ uint32_t decode_one(const uint64_t* rec64, const GroupDesc& G,
                                               const DecTabs& T, uint64_t p, uint32_t& idx) {
    const uint64_t x = peek64(rec64, G.bit_off + p);
    const uint32_t ent = T.lut[(size_t)G.lut << kLutBits | (uint32_t)(x >> (64 - kLutBits))];
    if (ent & 0xffu) {  // a code of at most kLutBits bits: one lookup
        idx = ent >> 8;
        return ent & 0xffu;
    }
    // longer codes: the canonical limits from length kLutBits + 1 (every shorter
    // length's limit is <= x, which is what a zero table entry records)
    const uint64_t* lim = T.lim + G.lim_off;
    uint32_t L = max(G.minlen, (uint32_t)kLutBits + 1);
    while (L <= G.maxlen && x >= lim[L - G.minlen]) ++L;
    if (L > G.maxlen) return 0;
    const uint64_t code = x >> (64 - L);
    idx = T.base[G.lim_off + L - G.minlen] + (uint32_t)(code - T.first[G.lim_off + L - G.minlen]);
    return L;
}

// The first-kLutBits table of every group with symbols (one CTA per group): entry e
// is the canonical decode of the bits e followed by zeros when its code is at most
// kLutBits long (codes of length L are decided by their first L bits alone).
__global__ void huff_lut_kernel(const GroupDesc* groups, DecTabs T, uint32_t* lut) {
    const GroupDesc G = groups[blockIdx.x];
    uint32_t* out = lut + ((size_t)blockIdx.x << kLutBits);
    const uint64_t* lim = T.lim + G.lim_off;
    const uint32_t top = min(G.maxlen, (uint32_t)kLutBits);
    for (uint32_t e = threadIdx.x; e < (1u << kLutBits); e += blockDim.x) {
        uint32_t ent = 0;
        if (G.nsyms) {
            const uint64_t x = (uint64_t)e << (64 - kLutBits);
            uint32_t L = G.minlen;
            while (L <= top && x >= lim[L - G.minlen]) ++L;
            if (L <= top) {
                const uint64_t code = x >> (64 - L);
                const uint32_t idx = T.base[G.lim_off + L - G.minlen] +
                                     (uint32_t)(code - T.first[G.lim_off + L - G.minlen]);
                if (idx < (1u << 24)) ent = idx << 8 | L;
            }
        }
        out[e] = ent;
    }
}

// Decodes chunk c from start[c] to its nominal end: end position, symbol count and
// the first kBnd codeword starts (relative to the chunk's nominal start).
__device__ __forceinline__ void decode_chunk(const uint64_t* rec64, const GroupDesc& G,
                                             const ChunkDesc& C, const DecTabs& T, uint32_t c,
                                             const uint64_t* start, uint64_t* out_pos,
                                             uint32_t* count, uint16_t* bounds) {
    const uint64_t end = min((uint64_t)(C.local + 1) * kChunkBits, G.nbits);
    const uint64_t nom = (uint64_t)C.local * kChunkBits;
    uint64_t p = start[c];
    uint32_t n = 0;
    uint16_t* bnd = bounds + (size_t)c * kBnd;
    while (p < end) {
        if (n < kBnd) bnd[n] = (uint16_t)(p - nom);
        uint32_t idx;
        const uint32_t L = decode_one(rec64, G, T, p, idx);
        p += L ? L : 1;  // invalid code: resynchronise (corrupt streams fail in H2)
        ++n;
    }
    for (uint32_t k = n; k < kBnd; ++k) bnd[k] = 0xffff;
    out_pos[c] = p;
    count[c] = n;
}

// Moves chunk c's start to `s` (where the previous chunk's decode ended).  When `s`
// is one of the codeword starts the chunk's own (speculative) decode went through,
// its end position is already right and only its symbol count shrinks: returns
// false.  Otherwise the chunk must be decoded again: returns true.
__device__ __forceinline__ bool restart_chunk(uint32_t c, uint32_t local, uint64_t s,
                                              uint64_t* start, uint32_t* count, uint16_t* bounds) {
    start[c] = s;
    const uint64_t rel = s - (uint64_t)local * kChunkBits;
    uint16_t* bnd = bounds + (size_t)c * kBnd;
    int hit = -1;
    for (int k = 0; k < kBnd && hit < 0; ++k)
        if (bnd[k] == rel) hit = k;
    if (hit < 0) return true;
    count[c] -= (uint32_t)hit;
    for (int k = 0; k + hit < kBnd; ++k) bnd[k] = bnd[k + hit];
    for (int k = kBnd - hit; k < kBnd; ++k) bnd[k] = 0xffff;
    return false;
}

// H1: decode chunk c from start[c] to its nominal end (dirty chunks only)
// gate: null, or the previous pass's "some start moved" flag (0: converged, nothing to do)
__global__ void __launch_bounds__(256) huff_sync_kernel(const uint64_t* rec64, const GroupDesc* groups,
                                                        const ChunkDesc* chunks, uint32_t nchunks,
                                                        DecTabs T, const uint64_t* start,
                                                        uint64_t* out_pos, uint32_t* count,
                                                        const uint8_t* dirty, uint16_t* bounds,
                                                        const uint32_t* gate) {
    if (gate && !*gate) return;
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks || !dirty[c]) return;
    const ChunkDesc C = chunks[c];
    decode_chunk(rec64, groups[C.group], C, T, c, start, out_pos, count, bounds);
}

// H1 update: every chunk takes the previous chunk's end as its start (in parallel)
__global__ void huff_update_kernel(const ChunkDesc* chunks, uint32_t nchunks, uint64_t* start,
                                   const uint64_t* out_pos, uint32_t* count, uint8_t* dirty,
                                   uint16_t* bounds, uint32_t* any, const uint32_t* gate) {
    if (gate && !*gate) return;
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    uint8_t d = 0;
    const uint32_t local = chunks[c].local;
    if (local > 0) {
        const uint64_t s = out_pos[c - 1];
        if (s != start[c]) d = restart_chunk(c, local, s, start, count, bounds);
    }
    dirty[c] = d;
    if (d) *any = 1;
}

// H1 fallback when the parallel passes have not converged: one thread per group walks
// its chunks in order, so every start is final after one sweep.  Codes whose lengths
// share a common factor that does not divide the chunk size (e.g. a complete table of
// 3-bit codes) never fall back into step from a wrong phase: the parallel passes
// would fix one chunk per pass.  Costs at most one sequential decode of the group.
__global__ void huff_serial_sync_kernel(const uint64_t* rec64, const GroupDesc* groups, uint32_t ngroups,
                                        const ChunkDesc* chunks, DecTabs T, uint64_t* start,
                                        uint64_t* out_pos, uint32_t* count, uint16_t* bounds,
                                        const uint8_t* dirty, const uint32_t* gate) {
    if (gate && !*gate) return;
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const GroupDesc G = groups[g];
    for (uint32_t l = 1; l < G.nchunks; ++l) {
        const uint32_t c = G.chunk0 + l;
        const uint64_t s = out_pos[c - 1];
        // dirty: start already moved by the last update, decode still pending
        bool redo = dirty[c] != 0;
        if (s != start[c]) redo = restart_chunk(c, l, s, start, count, bounds);
        if (redo) decode_chunk(rec64, G, chunks[c], T, c, start, out_pos, count, bounds);
    }
}

__global__ void group_flags_kernel(const GroupDesc* groups, uint32_t ng, uint8_t* f) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ng) return;
    const GroupDesc G = groups[g];
    if (!G.nsyms) return;
    if (G.nsyms == 1) {
        f[G.sym_off] = 3;
    } else {
        f[G.sym_off] = 1;
        f[G.sym_off + G.nsyms - 1] = 2;
    }
}

__global__ void chunk_init_kernel(const ChunkDesc* chunks, uint32_t nc, uint64_t* start) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nc) start[c] = (uint64_t)chunks[c].local * kChunkBits;
}

// H2: decode again, writing symbols at their index inside the group
__global__ void __launch_bounds__(256) huff_write_kernel(const uint64_t* rec64, const GroupDesc* groups,
                                                         const ChunkDesc* chunks, uint32_t nchunks,
                                                         DecTabs T, const uint64_t* start,
                                                         const unsigned long long* sym_scan,
                                                         int32_t* syms, uint32_t* err) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const ChunkDesc C = chunks[c];
    const GroupDesc G = groups[C.group];
    const uint64_t end = min((uint64_t)(C.local + 1) * kChunkBits, G.nbits);
    uint64_t k = sym_scan[c] - sym_scan[G.chunk0];
    uint64_t p = start[c];
    while (p < end && k < G.nsyms) {
        uint32_t idx;
        const uint32_t L = decode_one(rec64, G, T, p, idx);
        // invalid code, or a code running past the group's bytes (the reference's
        // BitReader runs out: codec.cpp:258-266)
        if (!L || idx >= G.tsize || p + L > G.nbits) {
            atomicOr(err, kErrCorruptBitstream);
            return;
        }
        syms[G.sym_off + k] = (int32_t)T.syms[G.tab_off + idx];
        p += L;
        ++k;
    }
}

// per group: the chunks' symbol total must cover nsyms (codec.cpp:250 overrun)
__global__ void huff_check_kernel(const GroupDesc* groups, uint32_t ngroups,
                                  const unsigned long long* sym_scan, uint32_t* err) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const GroupDesc G = groups[g];
    if (!G.nsyms) return;
    const uint64_t got = sym_scan[G.chunk0 + G.nchunks] - sym_scan[G.chunk0];
    if (got < G.nsyms) atomicOr(err, kErrCorruptBitstream);
}

// R1: elements produced by every symbol; run lengths need a preceding value
// (codec.cpp:91-107).  flags: bit0 first symbol of its group, bit1 last.
__global__ void rle_count_kernel(const int32_t* syms, const uint8_t* sflags, uint64_t n,
                                 unsigned long long* cnt, uint32_t err_bits, uint32_t* err) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t v = syms[s];
        const uint8_t f = sflags[s];
        unsigned long long c = 0;
        if (v > 0) {
            if ((f & 1) || syms[s - 1] > 0) atomicOr(err, err_bits);  // length without value
        } else {
            c = 1;
            if (!(f & 2) && syms[s + 1] > 0) c = (unsigned long long)syms[s + 1];
        }
        cnt[s] = c;
    }
}

// per group: the runs must produce exactly `elems` elements
__global__ void rle_total_kernel(const GroupDesc* groups, uint32_t ngroups,
                                 const unsigned long long* off, const unsigned long long* cnt,
                                 uint32_t* err) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const GroupDesc G = groups[g];
    if (!G.nsyms) {
        if (G.elems) atomicOr(err, kErrCorruptBitstream);
        return;
    }
    const uint64_t last = G.sym_off + G.nsyms - 1;
    const uint64_t total = off[last] + cnt[last] - off[G.sym_off];
    if (total != G.elems || off[G.sym_off] != G.elem_off) atomicOr(err, kErrCorruptBitstream);
}

struct Widen {
    __device__ __forceinline__ unsigned long long operator()(uint32_t x) const { return x; }
};

// R2+R3 (sparse): the delta stream starts zeroed; every value symbol writes its run's
// non-zero value over [off, off + cnt) -- the work follows the non-zero runs, not the
// elements (DELTA records are mostly zero runs).  Runs longer than kLongRun are queued
// for a block each.  Values outside the alphabet are CorruptIndex (codec.cpp:96-99,
// as rle_fill_kernel reported them).
constexpr unsigned long long kLongRun = 256;
__global__ void rle_fill_sparse_kernel(const int32_t* syms, uint64_t n, const unsigned long long* off,
                                       const unsigned long long* cnt, uint32_t B, uint8_t* d,
                                       uint64_t nd, unsigned long long* longs, unsigned int* nlong,
                                       uint32_t cap, uint32_t* err) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long c = cnt[s];
        if (!c) continue;  // a length symbol
        const int32_t x = syms[s];
        if (-x >= (int32_t)B) {
            atomicOr(err, kErrCorruptIndex);
            continue;
        }
        if (x == 0) continue;
        const uint8_t v = (uint8_t)(-x);
        const unsigned long long o = off[s];
        if (o + c > nd || o + c < o) {  // corrupt counts (flagged by rle_total too)
            atomicOr(err, kErrCorruptBitstream);
            continue;
        }
        if (c <= kLongRun) {
            for (unsigned long long j = 0; j < c; ++j) d[o + j] = v;
        } else {
            const unsigned int k = atomicAdd(nlong, 1u);
            if (k < cap) longs[k] = s;
            else atomicOr(err, kErrCorruptBitstream);  // cannot happen: cap bounds the list
        }
    }
}

__global__ void rle_fill_long_kernel(const int32_t* syms, const unsigned long long* off,
                                     const unsigned long long* cnt, const unsigned long long* longs,
                                     const unsigned int* nlong, uint32_t cap, uint8_t* d) {
    const unsigned int n = min(*nlong, cap);
    for (unsigned int k = blockIdx.x; k < n; k += gridDim.x) {
        const unsigned long long s = longs[k];
        const uint8_t v = (uint8_t)(-syms[s]);
        const unsigned long long o = off[s], c = cnt[s];
        for (unsigned long long j = threadIdx.x; j < c; j += blockDim.x) d[o + j] = v;
    }
}

// ---- U: unrearrange ------------------------------------------------------------
// U1: per tile, count of elements per previous level
template <int KB>
__global__ void __launch_bounds__(256) prev_count_kernel(const Tile* tiles, const uint16_t* prev,
                                                         uint32_t B, uint32_t* tile_cnt, uint32_t* err) {
    __shared__ uint32_t s_c[KB];
    const Tile T = tiles[blockIdx.x];
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) s_c[b] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x) {
        const uint32_t p = prev ? prev[T.start + i] : 0u;
        if (p >= B) atomicOr(err, kErrCorruptIndex);
        else atomicAdd(&s_c[p], 1u);
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) tile_cnt[(size_t)blockIdx.x * B + b] = s_c[b];
}

// U2: one block per (tensor, key): exclusive prefix of the tile counts over the
// tensor's tiles; key totals must match the record's group sizes
// (tile_in: the counts, row stride in_stride -- the U1 counts, or the base state's
// per-tile level histogram; tile_cnt: the prefixes, row stride B)
__global__ void __launch_bounds__(256) prev_scan_kernel(const uint32_t* tile0, uint32_t B,
                                                        const uint32_t* tile_in, uint32_t in_stride,
                                                        uint32_t* tile_cnt,
                                                        const unsigned long long* rec_elems,
                                                        unsigned long long* totals, uint32_t* err) {
    __shared__ unsigned long long s_scan[33];
    const uint32_t t = blockIdx.x / B, b = blockIdx.x % B;
    const uint32_t t0 = tile0[t], t1 = tile0[t + 1];
    unsigned long long run = 0;
    for (uint32_t c0 = t0; c0 < t1; c0 += blockDim.x) {
        const uint32_t ti = c0 + threadIdx.x;
        const unsigned long long v = ti < t1 ? tile_in[(size_t)ti * in_stride + b] : 0ull;
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_scan<unsigned long long>(v, s_scan, &tot);
        if (ti < t1) tile_cnt[(size_t)ti * B + b] = (uint32_t)(run + ex);
        run += tot;
    }
    if (threadIdx.x == 0) {
        totals[(size_t)t * B + b] = run;
        if (run != rec_elems[(size_t)t * B + b]) atomicOr(err, kErrCorruptIndex);
    }
}

// U3: per tile, stable rank of every element among equal previous levels (warp
// ranges of 512 elements, 32-element chunks matched on the key), delta gathered
// from the element's rearranged position, cur = (prev - d) mod B, range checks
template <int KB>
__global__ void __launch_bounds__(256) unrearrange_kernel(const Tile* tiles, const uint8_t* types,
                                                          const uint64_t* stream_off,
                                                          const uint64_t* off, const uint16_t* prev,
                                                          uint32_t B, const uint32_t* tile_base,
                                                          const unsigned long long* gstart,
                                                          const uint8_t* d, uint64_t nd,
                                                          const uint32_t* cb_len,
                                                          uint16_t* cur, uint32_t* err) {
    __shared__ uint32_t s_wc[8][KB];  // per-warp key counts -> per-warp key bases
    __shared__ uint32_t s_base[KB];
    const Tile T = tiles[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    for (int i = tid; i < 8 * KB; i += 256) (&s_wc[0][0])[i] = 0;
    __syncthreads();
    uint32_t rk[16], ky[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t e = wid * 512 + j * 32 + lane;
        const bool valid = e < T.count;
        uint32_t key = valid ? (prev ? prev[T.start + e] : 0u) : 0xffffu;
        if (key >= B && valid) key = 0;  // flagged in U1
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (lane == leader && valid) {
            old = s_wc[wid][key];
            s_wc[wid][key] = old + __popc(peers);
        }
        __syncwarp();
        old = __shfl_sync(0xffffffffu, old, leader);
        rk[j] = old + __popc(peers & lt_mask);
        ky[j] = key;
    }
    __syncthreads();
    const uint32_t t = T.tensor;
    for (uint32_t b = tid; b < B; b += 256) {
        uint32_t acc = 0;
        for (int w = 0; w < 8; ++w) {
            const uint32_t c = s_wc[w][b];
            s_wc[w][b] = acc;
            acc += c;
        }
        s_base[b] = (uint32_t)gstart[(size_t)t * B + b] + tile_base[(size_t)blockIdx.x * B + b];
    }
    __syncthreads();
    const uint64_t so = stream_off[t];
    const uint32_t maxl = cb_len[types[t]] + 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t e = wid * 512 + j * 32 + lane;
        if (e >= T.count) continue;
        const uint32_t key = ky[j];
        const uint64_t pos = (uint64_t)s_base[key] + s_wc[wid][key] + rk[j];
        const uint32_t dv = so + pos < nd ? d[so + pos] : 0u;  // see unrearrange16_kernel
        const uint32_t c = key >= dv ? key - dv : key + B - dv;
        if (c > maxl) atomicOr(err, kErrCorruptIndex);
        cur[T.start + e] = (uint16_t)c;
    }
}

// U3 for alphabets of at most 64 keys: every thread owns 16 contiguous elements (its
// count block).  Per (key, block) counts (u16, one column per thread), an exclusive
// prefix per key over the 256 blocks, and the element's rank among the equal keys of
// its own block from byte compares of its registers: the stable rank inside the tile
// without match / per-chunk serial counters.
__global__ void __launch_bounds__(256) unrearrange16_kernel(const Tile* tiles, const uint8_t* types,
                                                            const uint64_t* stream_off,
                                                            const uint16_t* prev, uint32_t B,
                                                            const uint32_t* tile_base,
                                                            const unsigned long long* gstart,
                                                            const uint8_t* d, uint64_t nd,
                                                            const uint32_t* cb_len,
                                                            uint16_t* cur, uint32_t* hist_out,
                                                            uint32_t* err) {
    __shared__ __align__(16) uint16_t s_hc[64 * 256];
    __shared__ unsigned long long s_base[64];
    const Tile T = tiles[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (uint32_t i = tid; i < B * 32; i += 256) ((uint4*)s_hc)[i] = make_uint4(0, 0, 0, 0);
    const uint32_t t = T.tensor;
    for (uint32_t b = tid; b < B; b += 256)
        s_base[b] = gstart[(size_t)t * B + b] + tile_base[(size_t)blockIdx.x * B + b];
    const uint32_t e0 = tid * 16;
    const uint32_t nv = e0 < T.count ? min(T.count - e0, 16u) : 0u;
    uint32_t kw[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};  // keys as bytes
    if (nv) {
        uint4 x = make_uint4(0, 0, 0, 0), y = x;
        if (prev) {
            const uint4* pp = (const uint4*)(prev + T.start + e0);
            x = pp[0], y = pp[1];
        }
        const uint32_t hi = x.x | x.y | x.z | x.w | y.x | y.y | y.z | y.w;
        kw[0] = __byte_perm(x.x, x.y, 0x6420);
        kw[1] = __byte_perm(x.z, x.w, 0x6420);
        kw[2] = __byte_perm(y.x, y.y, 0x6420);
        kw[3] = __byte_perm(y.z, y.w, 0x6420);
        // keys >= B (or >= 256) were flagged by U1; they count as key 0 here
        const uint32_t Brep = B * 0x01010101u;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int keep = (int)nv - 4 * w;
            const uint32_t m = keep >= 4 ? 0xffffffffu : (keep <= 0 ? 0u : (1u << (8 * keep)) - 1u);
            uint32_t v = kw[w] & ~__vcmpgeu4(kw[w], Brep);  // out of range -> 0
            kw[w] = (v & m) | ~m;                          // no element: 0xff
        }
        (void)hi;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t k = (kw[j >> 2] >> (8 * (j & 3))) & 0xffu;
        if (k < 64) ++s_hc[k * 256 + tid];
    }
    __syncthreads();
    for (uint32_t k = wid; k < B; k += 8) {  // per key: exclusive prefix over the 256 blocks
        uint4* row = (uint4*)(s_hc + k * 256 + 8 * lane);
        const uint4 v = *row;
        const uint32_t c0 = v.x & 0xffffu, c1 = v.x >> 16, c2 = v.y & 0xffffu, c3 = v.y >> 16;
        const uint32_t c4 = v.z & 0xffffu, c5 = v.z >> 16, c6 = v.w & 0xffffu, c7 = v.w >> 16;
        const uint32_t p1 = c0, p2 = p1 + c1, p3 = p2 + c2, p4 = p3 + c3, p5 = p4 + c4, p6 = p5 + c5,
                       p7 = p6 + c6, s8 = p7 + c7;
        uint32_t x = s8;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t ex = x - s8;
        *row = make_uint4(ex | ((ex + p1) << 16), (ex + p2) | ((ex + p3) << 16), (ex + p4) | ((ex + p5) << 16),
                          (ex + p6) | ((ex + p7) << 16));
    }
    __syncthreads();
    const uint64_t so = stream_off[t];
    const uint32_t maxl = cb_len[types[t]] + 1;
    uint32_t out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        uint32_t c = 0;
        if ((uint32_t)j < nv) {
            const uint32_t k = (kw[j >> 2] >> (8 * (j & 3))) & 0xffu;
            const uint32_t krep = k * 0x01010101u;
            uint32_t r = 0;  // equal keys of this block before j
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const int keep = j - 4 * w;
                const uint32_t m = keep >= 4 ? 0xffffffffu : (keep <= 0 ? 0u : (1u << (8 * keep)) - 1u);
                r += __popc(__vcmpeq4(kw[w], krep) & m);
            }
            r >>= 3;
            const unsigned long long pos = s_base[k] + s_hc[k * 256 + tid] + r;
            // a key count that disagrees with the record's groups is flagged by U2;
            // its positions may leave the stream
            const uint32_t dv = so + pos < nd ? d[so + pos] : 0u;
            c = k >= dv ? k - dv : k + B - dv;
            bad |= c > maxl;
        }
        if (j & 1) out[j >> 1] |= c << 16;
        else out[j >> 1] = c;
    }
    if (bad) atomicOr(err, kErrCorruptIndex);
    if (nv) {
        uint4* cp = (uint4*)(cur + T.start + e0);
        cp[0] = make_uint4(out[0], out[1], out[2], out[3]);
        cp[1] = make_uint4(out[4], out[5], out[6], out[7]);
    }
    if (!hist_out) return;
    // per-tile counts of the decoded levels (< B <= 64), for the next record's decode:
    // the count blocks again, one column per thread, then a sum per level
    __syncthreads();  // every prefix of s_hc has been read
    for (uint32_t i = tid; i < 64 * 32; i += 256) ((uint4*)s_hc)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j)
        if ((uint32_t)j < nv) ++s_hc[((out[j >> 1] >> (16 * (j & 1))) & 63u) * 256 + tid];
    __syncthreads();
    for (uint32_t v = wid; v < 64; v += 8) {
        const uint4 x = ((const uint4*)(s_hc + v * 256))[lane];
        uint32_t c = (x.x & 0xffffu) + (x.x >> 16) + (x.y & 0xffffu) + (x.y >> 16) + (x.z & 0xffffu) +
                     (x.z >> 16) + (x.w & 0xffffu) + (x.w >> 16);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) hist_out[(size_t)blockIdx.x * 64 + v] = c;
    }
}

// the base's level histogram as key counts: levels >= B are outside the alphabet
// (U1 reports them when it counts the levels itself)
__global__ void hist_range_check_kernel(const uint32_t* hist, int ntiles, uint32_t B, uint32_t* err) {
    const int ti = blockIdx.x * blockDim.x + threadIdx.x;
    if (ti >= ntiles) return;
    uint32_t any = 0;
    for (uint32_t v = B; v < 64; ++v) any |= hist[(size_t)ti * 64 + v];
    if (any) atomicOr(err, kErrCorruptIndex);
}

// ---- host ----------------------------------------------------------------------
namespace {

struct Rd {
    const uint8_t* p;
    uint64_t n, at = 0;
    void need(uint64_t k) const {
        if (n - at < k) throw Fail(DQTG_TRUNCATED, "DQDR record truncated");
    }
    uint8_t u8() {
        need(1);
        return p[at++];
    }
    template <typename T>
    T le() {
        need(sizeof(T));
        T v = 0;
        for (size_t i = 0; i < sizeof(T); ++i) v |= (T)p[at + i] << (8 * i);
        at += sizeof(T);
        return v;
    }
    double f64() {
        uint64_t u = le<uint64_t>();
        double d;
        memcpy(&d, &u, 8);
        return d;
    }
    float f32() {
        uint32_t u = le<uint32_t>();
        float f;
        memcpy(&f, &u, 4);
        return f;
    }
    uint64_t uv() {  // LEB128 (bytes.hpp:36-41)
        uint64_t v = 0;
        for (int sh = 0;; sh += 7) {
            const uint8_t b = u8();
            if (sh >= 64) throw Fail(DQTG_CORRUPT_BITSTREAM, "varint overflow");
            v |= (uint64_t)(b & 0x7f) << sh;
            if (!(b & 0x80)) return v;
        }
    }
    int64_t sv() {  // zig-zag (bytes.hpp:43-47)
        const uint64_t u = uv();
        return (int64_t)(u >> 1) ^ -(int64_t)(u & 1);
    }
    std::string str() {
        const uint16_t len = le<uint16_t>();
        need(len);
        std::string s((const char*)p + at, len);
        at += len;
        return s;
    }
};

}  // namespace

// Host walk of a record (decode_delta_record's parse, codec.cpp:513-597): everything
// that does not need the base's levels, in the reference's validation order.  `base`
// describes the delta base (step + tensor table) -- a decoded state, or the plan of
// the previous record of a chain, so the walk of record k+1 can overlap the device
// decode of record k (decode_chain).
std::unique_ptr<DecodePlan> decode_plan(Engine& e, const uint8_t* rec, uint64_t n, const BaseInfo* base) {
    auto P = std::make_unique<DecodePlan>();
    cudaStream_t st = e.stream;
    const bool trace = getenv("DQTG_DECODE_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (trace)
            fprintf(stderr, "decode %-12s %8.3f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    };
    // the record may live in device memory: decode from a host copy of its structure
    auto& host_copy = P->host_copy;
    const uint8_t* h = rec;
    if (is_device_ptr(rec)) {
        host_copy.resize(n);
        e.from_device(host_copy.data(), rec, n);
        e.sync();
        h = host_copy.data();
    }
    P->h = h;
    P->n = n;
    Rd r{h, n};
    {
        r.need(4);
        if (memcmp(h, "DQDR", 4) != 0) throw Fail(DQTG_BAD_MAGIC, "not a DQDR record");
        r.at = 4;
        const uint32_t v = r.le<uint32_t>();
        if (v != 1) throw Fail(DQTG_IO, "unsupported DQDR version " + std::to_string(v));
    }
    const bool has_base = r.u8() != 0;
    const uint64_t base_step = r.le<uint64_t>(), target_step = r.le<uint64_t>();
    const uint32_t B = r.le<uint32_t>();
    P->has_base = has_base;
    P->target_step = target_step;
    P->B = B;
    if (has_base && !base) throw Fail(DQTG_CHAIN_CORRUPT, "delta record requires its base state");
    if (!has_base) base = nullptr;
    if (base && base->step != base_step)
        throw Fail(DQTG_CHAIN_CORRUPT, "base step mismatch: record expects " +
                                           std::to_string(base_step) + ", got " +
                                           std::to_string(base->step));
    // deltas are staged as bytes and keys index per-tile shared arrays: B <= 255
    DQTG_REQUIRE(B >= 1 && B <= 255, DQTG_CORRUPT_INDEX, "cyclic alphabet outside the device decoder's range");
    P->q = std::make_unique<QState>();
    QState* q = P->q.get();
    q->eng = &e;
    q->step = target_step;
    dqtg_config& cfg = q->cfg;
    cfg.bins = r.le<uint32_t>();
    cfg.embed_bins = r.le<uint32_t>();
    cfg.prune_frac = r.f64();
    cfg.protect_frac = r.f64();
    cfg.metric = r.u8();
    cfg.sigma = r.f64();
    cfg.alpha = r.f64();
    r.f64();  // quality
    const uint8_t nlt = r.u8();
    for (uint8_t i = 0; i < nlt; ++i) {
        const uint8_t lt = r.u8();
        if (lt >= kLayerTypes) throw Fail(DQTG_CORRUPT_INDEX, "bad codebook layer type");
        const uint32_t len = r.le<uint32_t>();
        r.need((uint64_t)len * 4);
        q->cb[lt].resize(len);
        for (auto& v : q->cb[lt]) v = r.f32();
        q->cb_len[lt] = len;
    }
    const uint32_t nt = r.le<uint32_t>();
    P->nt = nt;
    if (base && base->names.size() != nt) throw Fail(DQTG_CHAIN_CORRUPT, "base tensor count mismatch");
    std::string& deferred_index = P->deferred_index;  // CorruptIndex found while parsing, reported after H/R
    // a corrupt count must not size host tables: every tensor takes >= 6 record bytes
    // (the reference's reserve() would throw std::length_error / bad_alloc here)
    if (nt > (r.n - r.at) / 6) throw Fail(DQTG_TRUNCATED, "tensor count exceeds the record size");
    // tensors
    auto& names = P->names;
    auto& types = P->types;
    auto& ranks = P->ranks;
    auto& dims = P->dims;
    auto& ppos = P->ppos;
    auto& pval = P->pval;
    auto& groups = P->groups;
    auto& chunks = P->chunks;
    auto& tab_sym = P->tab_sym;
    auto& tab_len = P->tab_len;
    auto& rec_elems = P->rec_elems;
    auto& gstart_h = P->gstart_h;
    auto& lim = P->lim;
    auto& first = P->first;
    auto& lbase = P->lbase;
    names.resize(nt);
    types.resize(nt);
    ranks.resize(nt);
    P->pcount.assign(nt, 0);
    rec_elems.assign((size_t)nt * B, 0);
    gstart_h.assign((size_t)nt * B, 0);
    uint64_t stream_pos = 0, sym_total = 0;
    for (uint32_t i = 0; i < nt; ++i) {
        names[i] = r.str();
        types[i] = r.u8();
        if (types[i] >= kLayerTypes) throw Fail(DQTG_CORRUPT_INDEX, "bad tensor layer type");
        ranks[i] = r.u8();
        uint64_t numel = 1;
        for (uint8_t k = 0; k < ranks[i]; ++k) {
            dims.push_back(r.le<uint64_t>());
            numel *= dims.back();
        }
        // device codec limit (2^31 elements per tensor, see encode_record_ex); also keeps
        // a corrupt shape from sizing host tables and device buffers
        if (numel >= (1ull << 31))
            throw Fail(DQTG_ERROR, "tensor " + names[i] + " has 2^31 or more elements (device codec limit)");
        const uint64_t np = r.uv();
        if (np > numel) throw Fail(DQTG_CORRUPT_INDEX, "too many protected entries in " + names[i]);
        if (np > (r.n - r.at) / 3) throw Fail(DQTG_TRUNCATED, "protected entries exceed the record size");
        P->pcount[i] = np;
        const size_t pb = ppos.size();
        ppos.resize(pb + np);
        pval.resize(pb + np);
        uint64_t pos = 0;
        for (uint64_t k = 0; k < np; ++k) {
            uint64_t dd;
            if (r.n - r.at >= 12) {  // fast path: no per-byte bounds checks
                const uint8_t* q8 = r.p + r.at;
                dd = q8[0] & 0x7f;
                int len = 1;
                if (q8[0] & 0x80) {
                    for (int sh = 7;; sh += 7) {
                        const uint8_t b = q8[len++];
                        dd |= (uint64_t)(b & 0x7f) << sh;
                        if (!(b & 0x80)) break;
                        if (len >= 10) throw Fail(DQTG_CORRUPT_BITSTREAM, "varint overflow");
                    }
                }
                r.at += len;
                pval[pb + k] = (uint16_t)(r.p[r.at] | (r.p[r.at + 1] << 8));
                r.at += 2;
            } else {
                dd = r.uv();
                pval[pb + k] = r.le<uint16_t>();
            }
            pos = k == 0 ? dd : pos + dd;
            if (pos >= numel || (k > 0 && dd == 0))
                throw Fail(DQTG_CORRUPT_INDEX, "protected positions not ascending in " + names[i]);
            ppos[pb + k] = pos;
        }
        if (base) {
            if (base->names[i] != names[i] || base->types[i] != types[i] || base->ranks[i] != ranks[i] ||
                !std::equal(base->dims[i].begin(), base->dims[i].end(), dims.end() - ranks[i]))
                throw Fail(DQTG_CHAIN_CORRUPT, "base tensor layout mismatch at " + names[i]);
        }
        // groups of the payload (codec.cpp:283-300)
        const uint64_t ng = r.uv();
        uint64_t total = 0;
        std::vector<uint8_t> seen_bucket(B, 0);
        for (uint64_t k = 0; k < ng; ++k) {
            GroupDesc G{};
            const uint64_t bucket = r.uv();
            G.elems = r.uv();
            G.nsyms = r.uv();
            const uint64_t tsize = r.uv();
            // the reference finds a bad bucket only in unrearrange, after the group
            // bitstreams decoded (codec.cpp:330-355): reported after the Huffman and
            // RLE stages so that their CorruptBitstream wins, as there
            // unrearrange (codec.cpp:56-64) takes the groups in any order but rejects
            // out-of-range and duplicate buckets
            if (bucket >= B || seen_bucket[bucket]) {
                if (deferred_index.empty())
                    deferred_index = std::string(bucket >= B ? "group bucket outside cyclic alphabet"
                                                             : "duplicate group bucket") + " in " + names[i];
            } else {
                seen_bucket[bucket] = 1;
            }
            // every table entry takes >= 2 bytes: a larger count runs out of record
            if (tsize > (r.n - r.at) / 2) throw Fail(DQTG_TRUNCATED, "huffman table exceeds the record");
            G.tab_off = (uint32_t)tab_sym.size();
            G.tsize = (uint32_t)tsize;
            for (uint64_t j = 0; j < tsize; ++j) {
                int64_t s = r.sv();
                // a symbol only matters once decoded: values beyond u16 and run lengths
                // beyond any group are clamped to sentinels the RLE stage rejects
                // (codec.cpp:96-99), as the reference rejects them only when read
                if (s > INT32_MAX) s = INT32_MAX;
                if (s < -(int64_t)0x10000) s = -(int64_t)0x10000;
                tab_sym.push_back(s);
                tab_len.push_back(r.u8());
            }
            const uint64_t nb = r.uv();
            r.need(nb);
            G.bit_off = r.at * 8;
            G.nbits = nb * 8;
            r.at += nb;
            G.lim_off = (uint32_t)lim.size();
            // huffman_decode (codec.cpp:234-250) validates the table only when the group
            // has symbols: empty table, canonical order, lengths and the Kraft sum of
            // assign_codes (codec.cpp:196-214)
            if (G.nsyms) {
                if (!tsize) throw Fail(DQTG_CORRUPT_BITSTREAM, "empty huffman table");
                for (uint64_t j = 1; j < tsize; ++j) {
                    const uint32_t a = G.tab_off + (uint32_t)j;
                    if (tab_len[a] < tab_len[a - 1] || (tab_len[a] == tab_len[a - 1] && tab_sym[a] <= tab_sym[a - 1]))
                        throw Fail(DQTG_CORRUPT_BITSTREAM, "huffman table not canonical");
                }
                for (uint64_t j = 0; j < tsize; ++j) {
                    const uint8_t l = tab_len[G.tab_off + j];
                    if (l == 0 || l > kMaxCodeLen - 1) throw Fail(DQTG_CORRUPT_BITSTREAM, "bad huffman table");
                }
                if (G.nsyms > G.nbits) throw Fail(DQTG_CORRUPT_BITSTREAM, "more symbols than bits");
                // canonical decode limits
                G.minlen = tab_len[G.tab_off];
                G.maxlen = tab_len[G.tab_off + tsize - 1];
                const size_t span = G.maxlen - G.minlen + 1;  // tables for minlen..maxlen only
                lim.resize(lim.size() + span, ~0ull);
                first.resize(first.size() + span, 0);
                lbase.resize(lbase.size() + span, 0);
                uint64_t code = 0;
                uint32_t j = 0, prev_len = G.minlen;
                for (uint32_t L = G.minlen; L <= G.maxlen; ++L) {
                    if (L > prev_len) code <<= (L - prev_len);
                    prev_len = L;
                    const size_t at = G.lim_off + (L - G.minlen);
                    first[at] = code;
                    lbase[at] = j;
                    uint32_t cntL = 0;
                    while (j < tsize && tab_len[G.tab_off + j] == L) ++j, ++cntL;
                    code += cntL;
                    // Kraft sum > 1 <=> the next canonical code passes 2^L (L <= 63)
                    if (code > (1ull << L)) throw Fail(DQTG_CORRUPT_BITSTREAM, "huffman table overfull");
                    lim[at] = code << (64 - L);
                    if (code == (1ull << L)) lim[at] = ~0ull;  // complete code
                }
            }
            G.elem_off = stream_pos + total;
            G.sym_off = sym_total;
            sym_total += G.nsyms;
            G.chunk0 = (uint32_t)chunks.size();
            G.nchunks = G.nsyms ? (uint32_t)((G.nbits + kChunkBits - 1) / kChunkBits) : 0;
            if (G.nsyms && !G.nchunks) throw Fail(DQTG_CORRUPT_BITSTREAM, "bitstream overrun");
            for (uint32_t c = 0; c < G.nchunks; ++c) chunks.push_back(ChunkDesc{(uint32_t)groups.size(), c});
            if (bucket < B) {  // the group's place in the dense rearranged stream (record order)
                rec_elems[(size_t)i * B + bucket] = G.elems;
                gstart_h[(size_t)i * B + bucket] = total;
            }
            total += G.elems;
            G.lut = (uint32_t)groups.size();
            groups.push_back(G);
        }
        if (total != numel) throw Fail(DQTG_CORRUPT_INDEX, "group totals do not cover the tensor");
        stream_pos += numel;
    }
    P->stored_crc = r.le<uint32_t>();
    if (r.at != n) throw Fail(DQTG_IO, "trailing bytes after DQDR record");
    P->sym_total = sym_total;
    P->eng = &e;
    mark("walked");
    P->stage();
    mark("staged");
    return P;
}

// Device decode of a planned record against its base state (the base's levels are
// only read here).
// base_hist: the base's per-tile level histogram may replace the key count pass (a
// state decoded within the same chain restore, never handed to the caller in between)
// want_hist: the decoded state will be the base of the next record of the chain
std::unique_ptr<QState> decode_run(Engine& e, DecodePlan& P, const QState* base, bool base_hist = false,
                                   bool want_hist = false) {
    cudaStream_t st = e.stream;
    const bool trace = getenv("DQTG_DECODE_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (trace)
            fprintf(stderr, "decode %-12s %8.3f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    };
    if (!P.has_base) base = nullptr;
    std::unique_ptr<QState> q = std::move(P.q);
    const uint32_t B = P.B, nt = P.nt;
    const uint64_t n = P.n, target_step = P.target_step, sym_total = P.sym_total;
    const uint8_t* rec = P.h;
    auto& names = P.names;
    auto& types = P.types;
    auto& ranks = P.ranks;
    auto& dims = P.dims;
    auto& ppos = P.ppos;
    auto& pval = P.pval;
    auto& groups = P.groups;
    auto& chunks = P.chunks;
    auto& tab_sym = P.tab_sym;
    auto& lim = P.lim;
    auto& first = P.first;
    auto& lbase = P.lbase;
    auto& rec_elems = P.rec_elems;
    auto& gstart_h = P.gstart_h;
    const std::string& deferred_index = P.deferred_index;
    const uint32_t stored_crc = P.stored_crc;

    // state layout from the record
    dqtg_layout dl{};
    std::vector<const char*> cn(nt);
    for (uint32_t i = 0; i < nt; ++i) cn[i] = names[i].c_str();
    dl.n_tensors = nt;
    dl.names = cn.data();
    dl.types = types.data();
    dl.ranks = ranks.data();
    dl.dims = dims.data();
    // a delta record has the base's tensor table (checked above): share its layout
    // (no per-record layout uploads / frees)
    q->L = base ? base->L : make_layout(&e, &dl);
    const Layout& L = *q->L;
    const uint64_t N = L.N;
    const int ntiles = (int)L.tiles.size();
    uint32_t stride = 1;
    for (int lt = 0; lt < kLayerTypes; ++lt) stride = std::max(stride, q->cb_len[lt]);
    q->cb_stride = stride;
    {
        std::vector<float> flat((size_t)kLayerTypes * stride, 0.0f);
        for (int lt = 0; lt < kLayerTypes; ++lt)
            std::copy(q->cb[lt].begin(), q->cb[lt].end(), flat.begin() + (size_t)lt * stride);
        q->d_cb = (float*)e.dalloc(flat.size() * 4);
        // pageable source: staged by the call, free to go out of scope on return
        DQTG_CUDA(cudaMemcpyAsync(q->d_cb, flat.data(), flat.size() * 4, cudaMemcpyHostToDevice, st));
    }
    // protected entries
    q->prot_count.assign(nt, 0);
    q->prot_off.assign(nt + 1, 0);
    uint64_t acc = 0;
    for (uint32_t i = 0; i < nt; ++i) {
        q->prot_off[i] = acc;
        q->prot_count[i] = P.pcount[i];
        acc += P.pcount[i];
    }
    q->prot_off[nt] = q->prot_total = acc;
    q->d_ppos = (uint64_t*)e.dalloc((acc + 1) * 8);
    q->d_pval = (uint16_t*)e.dalloc((acc + 1) * 2);
    const uint8_t* S = (const uint8_t*)P.pin;  // pinned staging of the walk, if packed
    auto up = [&](void* dst, size_t off, size_t bytes, const void* src) {
        if (!bytes) return;
        if (S) DQTG_CUDA(cudaMemcpyAsync(dst, S + off, bytes, cudaMemcpyHostToDevice, st));
        else e.to_device(dst, src, bytes);
    };
    if (acc) {
        up(q->d_ppos, P.o_ppos, acc * 8, ppos.data());
        up(q->d_pval, P.o_pval, acc * 2, pval.data());
    }
    q->d_levels = (uint16_t*)e.dalloc(L.Np * 2);
    DQTG_CUDA(cudaMemsetAsync(q->d_levels, 0, L.Np * 2, st));

    // device copies: record (+16 zero bytes), groups, chunks, tables
    const uint32_t ng = (uint32_t)groups.size(), nc = (uint32_t)chunks.size();
    auto* d_rec = (uint8_t*)e.buf("d.rec", n + 32);
    DQTG_CUDA(cudaMemsetAsync(d_rec + n, 0, 32, st));
    up(d_rec, P.o_rec, n, rec);
    auto* d_groups = (GroupDesc*)e.buf("d.groups", (size_t)(ng + 1) * sizeof(GroupDesc));
    auto* d_chunks = (ChunkDesc*)e.buf("d.chunks", (size_t)(nc + 1) * sizeof(ChunkDesc));
    auto* d_sym = (int64_t*)e.buf("d.tsym", (tab_sym.size() + 1) * 8);
    auto* d_lim = (uint64_t*)e.buf("d.lim", (lim.size() + 1) * 8);
    auto* d_first = (uint64_t*)e.buf("d.first", (first.size() + 1) * 8);
    auto* d_lbase = (uint32_t*)e.buf("d.lbase", (lbase.size() + 1) * 4);
    auto* d_relems = (unsigned long long*)e.buf("d.relems", rec_elems.size() * 8 + 8);
    up(d_groups, P.o_groups, ng * sizeof(GroupDesc), groups.data());
    up(d_chunks, P.o_chunks, nc * sizeof(ChunkDesc), chunks.data());
    up(d_sym, P.o_sym, tab_sym.size() * 8, tab_sym.data());
    up(d_lim, P.o_lim, lim.size() * 8, lim.data());
    up(d_first, P.o_first, first.size() * 8, first.data());
    up(d_lbase, P.o_lbase, lbase.size() * 4, lbase.data());
    up(d_relems, P.o_relems, rec_elems.size() * 8, rec_elems.data());
    auto* d_lut = (uint32_t*)e.buf("d.lut", ((size_t)ng << kLutBits) * 4 + 4);
    DecTabs T{d_lim, d_first, d_lbase, d_sym, d_lut};
    if (ng) { DQTG_SPAN(e, "huff_lut_kernel"); huff_lut_kernel<<<ng, 256, 0, st>>>(d_groups, T, d_lut); }
    mark("uploaded");
    const uint64_t* rec64 = (const uint64_t*)d_rec;

    // symbol flags (first / last of each group)
    auto* d_sflags = (uint8_t*)e.buf("d.sflags", sym_total + 16);
    DQTG_CUDA(cudaMemsetAsync(d_sflags, 0, sym_total + 1, st));
    if (ng) { DQTG_SPAN(e, "group_flags_kernel"); group_flags_kernel<<<(ng + 255) / 256, 256, 0, st>>>(d_groups, ng, d_sflags); }

    // ---- H1: self-synchronising chunk decode
    auto* d_start = (uint64_t*)e.buf("d.start", (size_t)(nc + 1) * 8);
    auto* d_out = (uint64_t*)e.buf("d.outpos", (size_t)(nc + 1) * 8);
    auto* d_cnt = (uint32_t*)e.buf("d.cnt", (size_t)(nc + 1) * 4);
    auto* d_dirty = (uint8_t*)e.buf("d.dirty", (size_t)nc + 16);
    auto* d_any = (uint32_t*)e.buf("d.any", 64);
    auto* d_bnd = (uint16_t*)e.buf("d.bounds", (size_t)(nc + 1) * kBnd * 2);
    uint32_t* d_err2 = nullptr;  // error word of the stages after the RLE counts
    {
        if (nc) { DQTG_SPAN(e, "chunk_init_kernel"); chunk_init_kernel<<<(nc + 255) / 256, 256, 0, st>>>(d_chunks, nc, d_start); }
        DQTG_CUDA(cudaMemsetAsync(d_dirty, 1, nc, st));
        const unsigned gb = (nc + 255) / 256;
        // a few parallel passes converge for Huffman tables in practice; what is still
        // out of step after them is finished by the sequential per-group sweep.  Every
        // pass is gated on the previous pass's flag on the device (no host round trip):
        // passes after convergence exit at once
        constexpr int kParallelPasses = 4;
        if (nc) {
            DQTG_CUDA(cudaMemsetAsync(d_any, 0, 4 * kParallelPasses, st));
            for (int it = 0; it < kParallelPasses; ++it) {
                const uint32_t* gate = it ? d_any + it - 1 : nullptr;
                { DQTG_SPAN(e, "huff_sync_kernel"); huff_sync_kernel<<<gb, 256, 0, st>>>(rec64, d_groups, d_chunks, nc, T, d_start, d_out, d_cnt, d_dirty, d_bnd, gate); }
                { DQTG_SPAN(e, "huff_update_kernel"); huff_update_kernel<<<gb, 256, 0, st>>>(d_chunks, nc, d_start, d_out, d_cnt, d_dirty, d_bnd, d_any + it, gate); }
                e.launched(2);
            }
            { DQTG_SPAN(e, "huff_serial_sync_kernel");
              huff_serial_sync_kernel<<<(ng + 127) / 128, 128, 0, st>>>(rec64, d_groups, ng, d_chunks, T, d_start, d_out, d_cnt, d_bnd, d_dirty, d_any + kParallelPasses - 1); }
            e.launched(1);
        }
        mark("synced");
        // chunks' symbol counts -> scan (u64)
        auto* d_scan = (unsigned long long*)e.buf("d.scan", (size_t)(nc + 2) * 8);
        cub::TransformInputIterator<unsigned long long, Widen, const uint32_t*> it(d_cnt, Widen{});
        size_t tb = 0;
        DQTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, d_scan, (int64_t)nc + 1, st));
        DQTG_CUDA(cudaMemsetAsync(d_cnt + nc, 0, 4, st));
        void* tmp = e.buf("d.cubtmp", tb + 16);
        DQTG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, it, d_scan, (int64_t)nc + 1, st));
        { DQTG_SPAN(e, "huff_check_kernel"); huff_check_kernel<<<(ng + 255) / 256 + 1, 256, 0, st>>>(d_groups, ng, d_scan, e.d_err); }
        auto* d_syms = (int32_t*)e.buf("d.syms", (sym_total + 1) * 4);
        { DQTG_SPAN(e, "huff_write_kernel"); huff_write_kernel<<<(nc + 255) / 256 + 1, 256, 0, st>>>(rec64, d_groups, d_chunks, nc, T, d_start, d_scan, d_syms, e.d_err); }
        e.launched(2);
        // Huffman and RLE-count errors are both CorruptBitstream: one check after both
        // (the RLE kernels only read and write within the symbol arrays)

        mark("huffman");
        // ---- R: RLE expansion into the dense rearranged delta stream
        auto* d_ecnt = (unsigned long long*)e.buf("d.ecnt", (sym_total + 1) * 8);
        auto* d_eoff = (unsigned long long*)e.buf("d.eoff", (sym_total + 1) * 8);
        const unsigned rg = (unsigned)std::min<uint64_t>((sym_total + 255) / 256 + 1, (uint64_t)e.num_sms * 16);
        { DQTG_SPAN(e, "rle_count_kernel"); rle_count_kernel<<<rg, 256, 0, st>>>(d_syms, d_sflags, sym_total, d_ecnt, kErrCorruptBitstream, e.d_err); }
        size_t tb2 = 0;
        DQTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, d_ecnt, d_eoff, (int64_t)std::max<uint64_t>(sym_total, 1), st));
        void* tmp2 = e.buf("d.cubtmp2", tb2 + 16);
        DQTG_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, tb2, d_ecnt, d_eoff, (int64_t)std::max<uint64_t>(sym_total, 1), st));
        { DQTG_SPAN(e, "rle_total_kernel"); rle_total_kernel<<<(ng + 255) / 256 + 1, 256, 0, st>>>(d_groups, ng, d_eoff, d_ecnt, e.d_err); }
        e.launched(2);
        // The later stages report into a second error word, read with the first one at
        // the end (one synchronisation per record): bitstream errors of the Huffman /
        // RLE-count stages first, then a bad group bucket found by the walk, then the
        // later stages' index errors -- the reference's order.  The later kernels stay
        // inside their buffers on corrupt input.
        d_err2 = (uint32_t*)e.buf("d.err2", 16);
        DQTG_CUDA(cudaMemsetAsync(d_err2, 0, 4, st));
        auto* d_d = (uint8_t*)e.buf("d.delta", N + 16);
        DQTG_CUDA(cudaMemsetAsync(d_d, 0, N + 16, st));
        // long runs: at most N / kLongRun of them
        const uint32_t lcap = (uint32_t)std::min<uint64_t>(N / kLongRun + 16, 0xffffffffull);
        auto* d_long = (unsigned long long*)e.buf("d.longruns", (size_t)lcap * 8 + 8);
        auto* d_nlong = (unsigned int*)e.buf("d.nlong", 16);
        DQTG_CUDA(cudaMemsetAsync(d_nlong, 0, 4, st));
        { DQTG_SPAN(e, "rle_fill_kernel"); rle_fill_sparse_kernel<<<rg, 256, 0, st>>>(d_syms, sym_total, d_eoff, d_ecnt, B, d_d, N, d_long, d_nlong, lcap, d_err2); }
        { DQTG_SPAN(e, "rle_fill_long_kernel"); rle_fill_long_kernel<<<e.num_sms * 4, 256, 0, st>>>(d_syms, d_eoff, d_ecnt, d_long, d_nlong, lcap, d_d); }
        e.launched(2);

        // ---- U: unrearrange against the previous levels
        auto* d_tc = (uint32_t*)e.buf("d.tilecnt", (size_t)ntiles * B * 4 + 4);
        auto* d_gs = (unsigned long long*)e.buf("d.gstart", (size_t)nt * B * 8 + 8);
        up(d_gs, P.o_gstart, gstart_h.size() * 8, gstart_h.data());
        auto* d_cbl = (uint32_t*)e.buf("d.cblen", kLayerTypes * 4);
        e.to_device(d_cbl, q->cb_len, sizeof(q->cb_len));
        const uint16_t* prev = base ? base->d_levels : nullptr;
        if (ntiles) {
            const bool fast = B <= 64 && !getenv("DQTG_UNREARRANGE_MATCH");
            const uint32_t* tin = d_tc;
            uint32_t in_stride = B;
            if (fast && base && base_hist && base->d_tile_hist && !getenv("DQTG_NO_TILE_HIST")) {
                tin = base->d_tile_hist;  // U1 from the previous decode
                in_stride = 64;
                { DQTG_SPAN(e, "hist_range_check_kernel"); hist_range_check_kernel<<<(ntiles + 255) / 256, 256, 0, st>>>(tin, ntiles, B, d_err2); }
            } else {
                DQTG_SPAN(e, "prev_count_kernel");
                (B <= 64 ? prev_count_kernel<64> : prev_count_kernel<256>)<<<ntiles, 256, 0, st>>>(L.d_tiles, prev, B, d_tc, d_err2);
            }
            auto* d_tot = (unsigned long long*)e.buf("d.ktot", (size_t)nt * B * 8 + 8);
            { DQTG_SPAN(e, "prev_scan_kernel"); prev_scan_kernel<<<nt * B, 256, 0, st>>>(L.d_tile0, B, tin, in_stride, d_tc, d_relems, d_tot, d_err2); }
            if (fast) {
                if (want_hist) q->d_tile_hist = (uint32_t*)e.dalloc((size_t)ntiles * 64 * 4);
                DQTG_SPAN(e, "unrearrange_kernel");
                unrearrange16_kernel<<<ntiles, 256, 0, st>>>(L.d_tiles, L.d_types, L.d_stream_off, prev, B, d_tc, d_gs, d_d, N, d_cbl, q->d_levels, q->d_tile_hist, d_err2);
            } else {
                DQTG_SPAN(e, "unrearrange_kernel");
                (B <= 64 ? unrearrange_kernel<64> : unrearrange_kernel<256>)<<<ntiles, 256, 0, st>>>(L.d_tiles, L.d_types, L.d_stream_off, L.d_off, prev, B, d_tc, d_gs, d_d, N, d_cbl, q->d_levels, d_err2);
            }
            e.launched(3);
        }
    }
    mark("unrearranged");
    // ---- C: stream checksum (queued behind the unrearrange; the error words are read
    // with it and checked first, in stage order)
    uint32_t h1 = 0, h2 = 0;
    e.d2h(&h1, e.d_err, 4);
    if (d_err2) e.d2h(&h2, d_err2, 4);
    const uint32_t crc = level_stream_crc(e, L, q->d_levels);
    if (h1 | h2) {
        DQTG_CUDA(cudaMemsetAsync(e.d_err, 0, 4, st));
        throw_err_bits(h1);
    }
    if (!deferred_index.empty()) throw Fail(DQTG_CORRUPT_INDEX, deferred_index);
    throw_err_bits(h2);
    mark("crc");
    if (P.pin) e.pin_release(P.pin, P.pin_cap);  // every upload has completed (the CRC read synced)
    P.pin = nullptr;
    if (crc != stored_crc)
        throw Fail(DQTG_CHECKSUM_MISMATCH, "record checksum mismatch at step " + std::to_string(target_step));
    return q;
}

BaseInfo base_info(const QState& s) {
    BaseInfo b;
    b.step = s.step;
    b.names = s.L->names;
    b.types = s.L->types;
    b.ranks = s.L->ranks;
    b.dims = s.L->dims;
    return b;
}

// the target of a planned record as the base of the next record of a chain
BaseInfo base_info(const DecodePlan& p) {
    BaseInfo b;
    b.step = p.target_step;
    b.names = p.names;
    b.types = p.types;
    b.ranks = p.ranks;
    size_t o = 0;
    for (uint32_t i = 0; i < p.nt; ++i) {
        b.dims.emplace_back(p.dims.begin() + (long)o, p.dims.begin() + (long)(o + p.ranks[i]));
        o += p.ranks[i];
    }
    return b;
}

// Chain::restore (chain.cpp:131-154) over host records.  The host walks of the next
// records run on helper threads (up to kPlanAhead at a time) while the device decodes
// record k.  A walk needs only its base's step and tensor table, not its levels, so
// record j is walked speculatively against the step in record j-1's header and the
// tensor table of record 0; once record j-1's own walk is known, a different table or
// step re-walks record j against it, so every record is checked against its true base
// (the walk is a pure function of the record and the base description).  Errors
// surface in record order: an error in record k+1 after record k is decoded, as in
// the reference's sequential restore.  on_state(k, state) sees every decoded state;
// the last one is returned.
namespace {
bool same_base(const BaseInfo& a, const BaseInfo& b) {
    return a.step == b.step && a.names == b.names && a.types == b.types && a.ranks == b.ranks &&
           a.dims == b.dims;
}
}  // namespace

std::unique_ptr<QState> decode_chain(Engine& e, const uint8_t* const* recs, const uint64_t* sizes,
                                     uint32_t n, const QState* base,
                                     const std::function<void(uint32_t, const QState&)>& on_state) {
    if (!n) return nullptr;
    for (uint32_t k = 0; k < n; ++k)
        DQTG_REQUIRE(!is_device_ptr(recs[k]), DQTG_ERROR, "decode_chain takes host records");
    constexpr uint32_t kPlanAhead = 8;
    BaseInfo b0;
    if (base) b0 = base_info(*base);
    BaseInfo table0;  // speculative tensor table of every later base
    std::unique_ptr<DecodePlan> cur;
    struct Walk {
        std::thread th;
        BaseInfo spec;
        std::unique_ptr<DecodePlan> plan;
        std::exception_ptr err;
    };
    std::vector<Walk> walks(n);
    struct Joiner {  // no helper thread outlives the call (they reference `walks`)
        std::vector<Walk>& w;
        ~Joiner() {
            for (auto& x : w)
                if (x.th.joinable()) x.th.join();
        }
    } joiner{walks};
    auto header_step = [&](uint32_t j) -> uint64_t {  // target step in record j's header
        if (sizes[j] < 25) return ~0ull;  // truncated: its own walk reports it
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= (uint64_t)recs[j][17 + i] << (8 * i);
        return v;
    };
    uint32_t launched = 1;
    auto launch = [&](uint32_t j) {  // table0 is set
        Walk& W = walks[j];
        W.spec = table0;
        W.spec.step = header_step(j - 1);
        W.th = std::thread([&e, &W, recs, sizes, j] {
            try {
                W.plan = decode_plan(e, recs[j], sizes[j], &W.spec);
            } catch (...) {
                W.err = std::current_exception();
            }
        });
    };
    // With a base state, its tensor table is the speculation and the later walks start
    // together with record 0's; otherwise they start from record 0's table
    if (base) {
        table0 = b0;
        while (launched < n && launched <= kPlanAhead) launch(launched++);
    }
    cur = decode_plan(e, recs[0], sizes[0], base ? &b0 : nullptr);
    if (!base) {
        table0 = base_info(*cur);
        while (launched < n && launched <= kPlanAhead) launch(launched++);
    }
    std::unique_ptr<QState> prev;
    const QState* pb = base;
    for (uint32_t k = 0; k < n; ++k) {
        BaseInfo actual;
        if (k + 1 < n) actual = base_info(*cur);  // the true base of record k+1
        std::unique_ptr<QState> s = decode_run(e, *cur, pb, k > 0, k + 1 < n);
        if (on_state) on_state(k, *s);
        cur.reset();
        prev = std::move(s);
        pb = prev.get();
        if (k + 1 == n) break;
        Walk& W = walks[k + 1];
        W.th.join();
        if (!same_base(actual, W.spec)) {  // mis-speculated base: walk again
            W.plan.reset();
            W.err = nullptr;
            try {
                W.plan = decode_plan(e, recs[k + 1], sizes[k + 1], &actual);
            } catch (...) {
                W.err = std::current_exception();
            }
        }
        if (W.err) std::rethrow_exception(W.err);
        cur = std::move(W.plan);
        if (launched < n) launch(launched++);
    }
    return prev;
}

std::unique_ptr<QState> decode_record(Engine& e, const uint8_t* rec, uint64_t n, const QState* base) {
    BaseInfo bi;
    if (base) bi = base_info(*base);
    auto plan = decode_plan(e, rec, n, base ? &bi : nullptr);
    return decode_run(e, *plan, base);
}

}  // namespace dqtg
