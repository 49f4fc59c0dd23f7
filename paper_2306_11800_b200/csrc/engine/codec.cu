// encode_delta_record on the device (codec.cpp:12-460).
//
// Per 4096-element tile of a tensor (one CTA):
//   E1  cyclic delta (codec.cpp:12-24), stable group-by of the deltas on the
//       previous level inside the tile (rearrange, codec.cpp:39-54) with a
//       ballot-based radix rank, run detection inside each group segment
//       (rle_encode, codec.cpp:79-90), symbol frequencies of runs that are
//       interior to the segment, CRC-32 of the target levels (combine algebra)
//   S   per (tensor, group): resolves runs that cross tile boundaries with a
//       forward "last value" scan and a backward run-monoid suffix scan
//   H   per (tensor, group): canonical Huffman (codec.cpp:137-214) with the
//       reference's (frequency, insertion order) tie-break via two queues
//   E2a bits per (tile, group); S2 scans them across tiles
//   L   record layout (varint sizes, protected entries, group headers)
//   W   header/table/protected writers; E2b MSB-first bit emission into the
//       final record buffer (codec.cpp:111-122)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "crc.cuh"
#include "engine.h"
#include "quantize_api.h"

namespace dqtg {

constexpr int kCB = 256;   // threads per codec CTA
constexpr int kLD = 64;    // dense run-length slots: lengths 2..63
constexpr int kMaxB = 64;  // cyclic alphabet of the shared-memory fast path (sparse DELTA, fused)
// Larger alphabets (quantize.cpp:400-401: u16 levels, B = max levels + 2, codec.cpp:416)
// run the dense tile kernel with 8-bit ballot keys, the symbol frequencies accumulated
// in global memory, and the tail kernels' per-group arrays sized for kMaxBLarge; the
// byte-packed tile codec keeps one byte per key and per delta, with 0xff reserved for
// "no element", so B <= 255.
constexpr int kMaxBLarge = 255;
constexpr int kIt = kTile / kCB;  // 16 elements per thread

__constant__ uint32_t c_crc_pw[kCB];   // x^(8*32*(255-t)) mod P
__constant__ uint32_t c_crc_x2n[32];

struct Seg {
    uint32_t n, lead, trail, run_begin, run_end;
    uint16_t fv, lv;
    uint32_t cont;
    uint32_t pad;
    unsigned long long lead_total, trail_total;
};

struct EncArgs {
    int ntiles;
    unsigned int* tile_ctr;  // dynamic tile scheduling (zeroed per launch)
    const uint32_t* crc_shift;  // per tile
    uint32_t n_tb;              // tensors * B
    const Tile* tiles;
    const uint8_t* types;
    const uint64_t* off;
    const uint64_t* stream_off;
    const uint32_t* tile0;
    uint64_t N;
    uint32_t B, NS;
    const uint16_t* prev;  // null: FULL record (all-zero base)
    const uint16_t* cur;
    Seg* segs;                       // [tile][B]
    unsigned long long* runs;        // [tile][kTile]: v | b<<16 | len<<32
    uint32_t* tile_nruns;
    uint32_t* freq;                  // [tensor][B][NS]
    unsigned long long* ov;          // overflow run lengths: (tensor*B+b)<<32 | len
    unsigned long long* ov_count;
    unsigned long long ov_cap;
    uint32_t* crc_acc;
    uint32_t* tile_crc;  // per tile, zero register, ending at the tile's last byte
    uint32_t* err;
    uint32_t* zs;        // enc_tile_delta_kernel: per-CTA kTile words for dense tiles
    // payload_bytes ablations (codec.cpp:601-646): 0 = record (rearranged groups),
    // 1 = one group per tensor (no rearrange), 2 = one group and no RLE (every
    // element its own run)
    uint32_t mode;
};

__device__ __forceinline__ uint32_t uvlen(unsigned long long v) {
    uint32_t n = 1;
    while (v >= 0x80) {
        v >>= 7;
        ++n;
    }
    return n;
}
__device__ __forceinline__ unsigned long long zigzag(long long v) {
    return ((unsigned long long)v << 1) ^ (unsigned long long)(v >> 63);
}
__device__ __forceinline__ uint32_t put_uv(uint8_t* p, unsigned long long v) {
    uint32_t n = 0;
    while (v >= 0x80) {
        p[n++] = (uint8_t)(v | 0x80);
        v >>= 7;
    }
    p[n++] = (uint8_t)v;
    return n;
}

__device__ __forceinline__ void add_symbol(uint32_t* f, uint32_t NS, uint32_t B, uint32_t tb,
                                           uint32_t v, unsigned long long L, const EncArgs& A) {
    atomicAdd(f + v, 1u);
    if (L > 1) {
        if (L < (unsigned long long)kLD) {
            atomicAdd(f + B + (uint32_t)L, 1u);
        } else {
            unsigned long long slot = atomicAdd(A.ov_count, 1ull);
            if (slot < A.ov_cap) A.ov[slot] = ((unsigned long long)tb << 32) | L;
            else atomicOr(A.err, kErrCorruptIndex);
        }
    }
}

// ---- E1 --------------------------------------------------------------------
// Persistent CTAs walk contiguous tile ranges.  Per tile (4096 elements):
//   L  16 contiguous elements per thread, packed as bytes (levels < 64):
//      key = previous level, d = cyclic delta (codec.cpp:12-24) with SIMD byte
//      ops; CRC-32 of the thread's 32 level-stream bytes (zero-skipping
//      slice-by-16, the high byte of every level is 0), moved to the tile end
//      with nibble tables of x^(8n) mod P (lane, then warp); the tile value is
//      moved to its stream position later (crc_tiles_kernel)
//   M  warp w owns elements [512w, 512w+512) in 32-element chunks:
//      __match_any_sync on the key gives the rank inside the chunk; per-chunk
//      key counts -> per-key prefix over chunks (stable group-by,
//      codec.cpp:39-54)
//   P  per key: prefix over warps, group starts
//   S  d scattered to its rearranged position (bytes)
//   D  run heads (rle_encode, codec.cpp:79-90) = group starts | byte changes
//      of the rearranged stream (SIMD compare), block scan -> run starts
//   R  runs (value, group, length), first/last run per group, interior-run
//      symbol frequencies (accumulated per tensor in shared memory)
constexpr int kCrcTabs = 10;  // T1,T3,T5,T7,T9,T11,T12,T13,T14,T15 (T_n: byte + n zero bytes)
constexpr int kChunks = 512 / 32;  // chunks per warp range
__device__ uint32_t g_crc_slice[kCrcTabs][256];
// g_crc_nib[s][i][n]: nibble n at position i times x^(8m) mod P for the combine
// constant s: s < 8 lane r of a group of 8 lanes (m = 32 * (7 - r) bytes), s = 8, 9
// groups of a warp (m = 256, 512), s = 10..12 warps of the tile (m = 1024 * 2^(s-10))
constexpr int kNibConsts = 13;
__device__ uint32_t g_crc_nib[kNibConsts][8][16];

// 8 levels (16 stream bytes, odd bytes 0) through the CRC register
__device__ __forceinline__ uint32_t crc_block8(const uint32_t* T, uint32_t r, uint32_t l03,
                                               uint32_t l47) {
    // l03 / l47: levels 0..3 / 4..7 as bytes
    const uint32_t x = r ^ ((l03 & 0xff) | ((l03 & 0xff00) << 8));
    return T[9 * 256 + (x & 0xff)] ^ T[8 * 256 + ((x >> 8) & 0xff)] ^
           T[7 * 256 + ((x >> 16) & 0xff)] ^ T[6 * 256 + (x >> 24)] ^
           T[5 * 256 + ((l03 >> 16) & 0xff)] ^ T[4 * 256 + (l03 >> 24)] ^
           T[3 * 256 + (l47 & 0xff)] ^ T[2 * 256 + ((l47 >> 8) & 0xff)] ^
           T[1 * 256 + ((l47 >> 16) & 0xff)] ^ T[0 * 256 + (l47 >> 24)];
}
// v * (shift of combine level s) mod P from the nibble tables (16 consecutive words
// per nibble position: conflict-free)
__device__ __forceinline__ uint32_t crc_mul_nib(const uint32_t* N, uint32_t v, int s) {
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= N[(s * 8 + i) * 16 + ((v >> (4 * i)) & 15u)];
    return r;
}

// Binary-tree combine of per-lane values over `levels` levels with constants
// s0, s0+1, ..., lanes at multiples of `stride`: the left value of every pair
// moves past the right one.  Lane 0 returns the combined value.
__device__ __forceinline__ uint32_t crc_tree(const uint32_t* N, uint32_t v, int s0, int levels,
                                             int stride = 1) {
    const int lane = threadIdx.x & 31;
    for (int l = 0; l < levels; ++l) {
        const int d = stride << l;
        const uint32_t o = __shfl_down_sync(0xffffffffu, v, d);
        const uint32_t m = crc_mul_nib(N, v, s0 + l) ^ o;
        if ((lane & (2 * d - 1)) == 0) v = m;
    }
    return v;
}

// Warp combine of 32 consecutive 32-byte chunk CRCs: each lane moves its chunk to
// the end of its 8-lane group (one table multiply), XOR within the group, then a
// two-level tree over the four groups.  Lane 0 returns the warp's 1 KiB CRC.
__device__ __forceinline__ uint32_t crc_warp(const uint32_t* N, uint32_t v) {
    const int lane = threadIdx.x & 31;
    v = crc_mul_nib(N, v, lane & 7);
    v ^= __shfl_down_sync(0xffffffffu, v, 1);
    v ^= __shfl_down_sync(0xffffffffu, v, 2);
    v ^= __shfl_down_sync(0xffffffffu, v, 4);
    return crc_tree(N, v, 8, 2, 8);
}

struct E1Smem {
    uint32_t* freq;   // B*NS, per tensor
    uint32_t* crc;    // kCrcTabs*256
    uint32_t* nib;    // kNibConsts*8*16
    uint32_t* wcnt;   // 8*B: per-warp key counts -> per-warp key bases
    uint16_t* cc;     // 8*kChunks*B: per-chunk key counts -> prefix over chunks
    uint32_t* part;   // 8 warp CRCs
    uint32_t* gs;     // kTile/32 group-start bitmap
    uint16_t* kd;     // kTile: key | d << 8      (aliased by hp after M)
    uint16_t* hp;     // kTile + 1 run starts
    uint8_t* sd;      // kTile: rearranged deltas (sd[-1] readable)
};

__host__ __device__ inline size_t e1_smem_bytes(uint32_t B, uint32_t NS) {
    return (B > (uint32_t)kMaxB ? 16 : (((size_t)B * NS * 4 + 15) & ~(size_t)15)) + (size_t)kCrcTabs * 256 * 4 +
           (size_t)kNibConsts * 8 * 16 * 4 + (((size_t)8 * B * 4 + 15) & ~(size_t)15) +
           (((size_t)8 * kChunks * B * 2 + 15) & ~(size_t)15) + 32 + kTile / 8 +
           (2 * (size_t)kTile + 16) + (kTile + 32);
}

__device__ inline E1Smem e1_carve(uint8_t* base, uint32_t B, uint32_t NS) {
    E1Smem S;
    size_t o = 0;
    S.freq = (uint32_t*)(base + o);  // KB > kMaxB: unused (frequencies in global memory)
    o += B > (uint32_t)kMaxB ? 16 : (((size_t)B * NS * 4 + 15) & ~(size_t)15);
    S.crc = (uint32_t*)(base + o);  o += (size_t)kCrcTabs * 256 * 4;
    S.nib = (uint32_t*)(base + o);  o += (size_t)kNibConsts * 8 * 16 * 4;
    S.wcnt = (uint32_t*)(base + o); o += ((size_t)8 * B * 4 + 15) & ~(size_t)15;
    S.cc = (uint16_t*)(base + o);   o += ((size_t)8 * kChunks * B * 2 + 15) & ~(size_t)15;
    S.part = (uint32_t*)(base + o); o += 32;
    S.gs = (uint32_t*)(base + o);   o += kTile / 8;
    S.kd = (uint16_t*)(base + o);
    S.hp = (uint16_t*)(base + o);   o += 2 * (size_t)kTile + 16;
    S.sd = base + o + 16;
    return S;
}

// bit j (j = 0..3) = top bit of byte j
__device__ __forceinline__ uint32_t byte_msbs(uint32_t x) {
    return (((x >> 7) & 0x01010101u) * 0x10204080u) >> 28;
}

__device__ __forceinline__ uint32_t keep_mask(int keep) {  // low `keep` bytes
    return keep >= 4 ? 0xffffffffu : (keep <= 0 ? 0u : (1u << (8 * keep)) - 1u);
}

// lanes of the warp holding the same NB-bit key: one ballot per key bit (keys are
// < 2^NB; invalid elements carry 2^NB - 1, which no valid key reaches)
template <int NB>
__device__ __forceinline__ uint32_t peers_of(uint32_t key) {
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int bit = 0; bit < NB; ++bit) {
        const bool on = (key >> bit) & 1u;
        const uint32_t b = __ballot_sync(0xffffffffu, on);
        peers &= on ? b : ~b;
    }
    return peers;
}

// MATCH.ANY is one instruction, but its unit is throughput-limited: the rank phase
// stalled on its results.  Every third chunk ranks with ballots instead, which run
// on the ALU/vote pipes (all-ballot ranks were slower, 0.785 vs 0.745 ms; one third:
// 0.716 ms at C2).
constexpr int kBallotEvery = 3;

template <bool HAS_BASE, int NB, int KB>
__global__ void __launch_bounds__(kCB, 4) enc_tile_kernel(EncArgs A) {
    extern __shared__ __align__(16) uint8_t e1_dyn[];
    const uint32_t B = A.B, NS = A.NS;
    const E1Smem S = e1_carve(e1_dyn, B, NS);
    constexpr bool GF = KB > kMaxB;  // symbol frequencies straight into global memory
    __shared__ uint32_t s_cnt[KB], s_start[KB + 1], s_run0[KB], s_run1[KB];
    __shared__ unsigned long long s_scan[33];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    const uint32_t Brep = B * 0x01010101u;

    for (uint32_t i = tid; i < kCrcTabs * 256; i += kCB) S.crc[i] = (&g_crc_slice[0][0])[i];
    for (uint32_t i = tid; i < kNibConsts * 8 * 16; i += kCB) S.nib[i] = (&g_crc_nib[0][0][0])[i];
    if (!GF)
        for (uint32_t i = tid; i < B * NS; i += kCB) S.freq[i] = 0;
    if (tid < 16) S.sd[tid - 16] = 0;
    __shared__ int s_base;
    uint32_t cur_tensor = 0xffffffffu;

    for (int base; (base = grab_tiles(A.tile_ctr, 4, &s_base)) < A.ntiles;)
    for (int ti = base; ti < min(base + 4, A.ntiles); ++ti) {
        const Tile T = A.tiles[ti];
        const uint32_t cnt = T.count;
        if (tid == 0 && ti + 1 < min(base + 4, A.ntiles)) {  // next tile's levels into L2
            const Tile N = A.tiles[ti + 1];
            const uint32_t bytes = ((N.count + 7u) & ~7u) * 2u;
            prefetch_l2(A.cur + N.start, bytes);
            if (HAS_BASE) prefetch_l2(A.prev + N.start, bytes);
        }
        if (T.tensor != cur_tensor) {  // flush the previous tensor's symbol counts
            __syncthreads();
            if (!GF && cur_tensor != 0xffffffffu) {
                uint32_t* gf = A.freq + (size_t)cur_tensor * B * NS;
                for (uint32_t i = tid; i < B * NS; i += kCB) {
                    const uint32_t c = S.freq[i];
                    if (c) {
                        atomicAdd(gf + i, c);
                        S.freq[i] = 0;
                    }
                }
            }
            cur_tensor = T.tensor;
        }
        // ---- L
        if (tid < kTile / 32) S.gs[tid] = 0;
        {
            uint32_t* cc = (uint32_t*)(S.cc + wid * kChunks * B);
            for (uint32_t i = lane; i < kChunks * B / 2; i += 32) cc[i] = 0;
        }
        {
            const uint32_t e0 = tid * kIt;
            uint32_t cw[4] = {0, 0, 0, 0}, pw[4] = {0, 0, 0, 0};
            const uint32_t nv = e0 < cnt ? min(cnt - e0, (uint32_t)kIt) : 0u;  // valid here
            if (nv) {
                const uint4* cp = (const uint4*)(A.cur + T.start + e0);
                const uint4 a0 = cp[0], a1 = cp[1];
                uint32_t hi[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                cw[0] = __byte_perm(a0.x, a0.y, 0x6420);
                cw[1] = __byte_perm(a0.z, a0.w, 0x6420);
                cw[2] = __byte_perm(a1.x, a1.y, 0x6420);
                cw[3] = __byte_perm(a1.z, a1.w, 0x6420);
                uint32_t hp_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                if (HAS_BASE) {
                    const uint4* pp = (const uint4*)(A.prev + T.start + e0);
                    const uint4 b0 = pp[0], b1 = pp[1];
                    hp_[0] = b0.x, hp_[1] = b0.y, hp_[2] = b0.z, hp_[3] = b0.w;
                    hp_[4] = b1.x, hp_[5] = b1.y, hp_[6] = b1.z, hp_[7] = b1.w;
                    pw[0] = __byte_perm(b0.x, b0.y, 0x6420);
                    pw[1] = __byte_perm(b0.z, b0.w, 0x6420);
                    pw[2] = __byte_perm(b1.x, b1.y, 0x6420);
                    pw[3] = __byte_perm(b1.z, b1.w, 0x6420);
                }
                // high bytes of the u16 levels (must be 0) of the valid elements
                uint32_t bad = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int keep = (int)nv - 2 * j;
                    const uint32_t m = keep >= 2 ? 0xff00ff00u : (keep == 1 ? 0x0000ff00u : 0u);
                    bad |= (hi[j] | hp_[j]) & m;
                }
                uint32_t big = 0;
                const bool full = nv == (uint32_t)kIt;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t m = full ? 0xffffffffu : keep_mask((int)nv - 4 * j);
                    cw[j] &= m;
                    pw[j] &= m;
                    big |= __vcmpgeu4(cw[j], Brep) | __vcmpgeu4(pw[j], Brep);
                }
                if (bad | big) atomicOr(A.err, kErrCorruptIndex);
            }
            // d = (p - c) mod B per byte
            uint32_t kd[8];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t lt = __vcmpltu4(pw[j], cw[j]);
                const uint32_t dw = __vadd4(__vsub4(pw[j], cw[j]), lt & Brep);
                const uint32_t vm = keep_mask((int)nv - 4 * j);
                // invalid elements: key 0xff; ablation modes group by nothing (key 0)
                const uint32_t key = ((A.mode ? 0u : pw[j]) & vm) | ~vm;
                kd[2 * j] = __byte_perm(key, dw, 0x5140);
                kd[2 * j + 1] = __byte_perm(key, dw, 0x7362);
            }
            *(uint4*)(S.kd + e0) = make_uint4(kd[0], kd[1], kd[2], kd[3]);
            *(uint4*)(S.kd + e0 + 8) = make_uint4(kd[4], kd[5], kd[6], kd[7]);
            // CRC of this thread's levels (zero register), right-aligned in its
            // 32-byte chunk when the tile ends inside it (leading zero levels are neutral)
            uint32_t c0 = cw[0], c1 = cw[1], c2 = cw[2], c3 = cw[3];
            if (nv && nv < (uint32_t)kIt) {
                const int sh = kIt - (int)nv;  // bytes to move up
                uint32_t w[8] = {0, 0, 0, 0, cw[0], cw[1], cw[2], cw[3]};
                // shift the 16-byte little-endian value left by sh bytes
                uint32_t o[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int src = 4 + j - (sh >> 2);
                    const uint32_t lo_w = src - 1 >= 0 ? w[src - 1] : 0u;
                    o[j] = (sh & 3) ? __funnelshift_l(lo_w, w[src], 8 * (sh & 3)) : w[src];
                }
                c0 = o[0], c1 = o[1], c2 = o[2], c3 = o[3];
            }
            uint32_t r = 0;
            if (nv) r = crc_block8(S.crc, crc_block8(S.crc, 0u, c0, c1), c2, c3);
            if (cnt == kTile) {
                r = crc_warp(S.nib, r);  // lane 0: CRC of the warp's 1 KiB
                if (lane == 0) S.part[wid] = r;
            } else {  // ragged tile: shift by the bytes after this chunk inside the tile
                if (r) r = crc_shift(c_crc_x2n, r, 2ull * (cnt - (e0 + nv)));
                r = warp_xor(r);
                if (lane == 0) S.part[wid] = r;
            }
        }
        __syncthreads();

        // ---- M: rank inside the chunk (match), per-chunk key counts
        uint32_t pk[kIt];  // rank-in-chunk | key << 8 | d << 16 (key 0xff: no element)
        uint16_t* cc = S.cc + wid * kChunks * B;
        {
#pragma unroll
            for (int j = 0; j < kIt; ++j) {
                const uint32_t e = wid * 512 + j * 32 + lane;
                const uint32_t kdv = S.kd[e];
                const uint32_t key = kdv & 0xffu;
                const bool valid = key != 0xffu;
                const uint32_t peers = (j % kBallotEvery) == kBallotEvery - 1
                                           ? peers_of<NB>(key) : __match_any_sync(0xffffffffu, key);
                if (valid && (peers & lt_mask) == 0) cc[j * B + key] = (uint16_t)__popc(peers);
                pk[j] = __popc(peers & lt_mask) | (kdv << 8);  // rank | key << 8 | d << 16
            }
        }
        __syncwarp();
        for (uint32_t b = lane; b < B; b += 32) {  // prefix over chunks per key
            uint32_t acc = 0;
#pragma unroll
            for (int j = 0; j < kChunks; ++j) {
                const uint32_t c = cc[j * B + b];
                cc[j * B + b] = (uint16_t)acc;
                acc += c;
            }
            S.wcnt[wid * B + b] = acc;
        }
        __syncthreads();
        // ---- P: per key prefix over warps; group starts
        for (uint32_t b = tid; b < B; b += kCB) {
            uint32_t acc = 0;
#pragma unroll
            for (int w = 0; w < kCB / 32; ++w) {
                const uint32_t c = S.wcnt[w * B + b];
                S.wcnt[w * B + b] = acc;
                acc += c;
            }
            s_cnt[b] = acc;
        }
        if (wid == kCB / 32 - 1) {  // tile CRC (moved to its stream position by crc_tiles_kernel)
            uint32_t r = lane < kCB / 32 ? S.part[lane] : 0u;
            if (cnt == kTile) r = crc_tree(S.nib, r, 10, 3);  // warps: 1 KiB chunks
            else r = warp_xor(r);                              // ragged: already at the tile end
            if (lane == 0) A.tile_crc[ti] = r;
        }
        __syncthreads();
        if (wid == 0) {
            uint32_t run = 0;
            for (uint32_t b0 = 0; b0 < B; b0 += 32) {
                const uint32_t b = b0 + lane;
                const uint32_t v = b < B ? s_cnt[b] : 0;
                uint32_t x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (b < B) {
                    const uint32_t st = run + x - v;
                    s_start[b] = st;
                    if (v) atomicOr(S.gs + (st >> 5), 1u << (st & 31));
                }
                run += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) s_start[B] = run;
        }
        __syncthreads();
        // ---- S: scatter deltas to their rearranged positions
        {
            const uint32_t* wb = S.wcnt + wid * B;
#pragma unroll
            for (int j = 0; j < kIt; ++j) {
                const uint32_t q = pk[j];
                const uint32_t key = (q >> 8) & 0xffu;
                if (key != 0xffu) S.sd[s_start[key] + wb[key] + cc[j * B + key] + (q & 31u)] = (uint8_t)(q >> 16);
            }
        }
        __syncthreads();
        // ---- D: run heads = group starts | changes of the rearranged stream
        uint32_t R;
        {
            const uint32_t p0 = tid * kIt;
            const uint4 x = *(const uint4*)(S.sd + p0);
            const uint32_t prevw = (uint32_t)S.sd[(int)p0 - 1] << 24;
            uint32_t m = byte_msbs(__vcmpne4(x.x, __funnelshift_l(prevw, x.x, 8))) |
                         (byte_msbs(__vcmpne4(x.y, __funnelshift_l(x.x, x.y, 8))) << 4) |
                         (byte_msbs(__vcmpne4(x.z, __funnelshift_l(x.y, x.z, 8))) << 8) |
                         (byte_msbs(__vcmpne4(x.w, __funnelshift_l(x.z, x.w, 8))) << 12);
            m |= (S.gs[tid >> 1] >> ((tid & 1) * 16)) & 0xffffu;
            if (A.mode == 2) m = 0xffffu;  // no RLE: every element starts a run
            if (p0 + kIt > cnt) m &= p0 >= cnt ? 0u : (1u << (cnt - p0)) - 1u;
            unsigned long long tot;
            uint32_t r = (uint32_t)block_exclusive_scan<unsigned long long>(__popc(m), s_scan, &tot);
            R = (uint32_t)tot;
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                S.hp[r++] = (uint16_t)(p0 + j);
            }
            if (tid == 0) S.hp[R] = (uint16_t)cnt;
        }
        __syncthreads();
        // ---- R: runs, first/last run of every group, interior-run symbols
        unsigned long long* runs = A.runs + (size_t)ti * kTile;
        for (uint32_t r = tid; r < R; r += kCB) {
            const uint32_t p = S.hp[r], L = S.hp[r + 1] - p;
            const uint32_t v = S.sd[p];
            uint32_t lo = 0, n = B + 1;  // last b with s_start[b] <= p (a non-empty group)
            while (n > 1) {
                const uint32_t h = n >> 1;
                if (s_start[lo + h] <= p) lo += h, n -= h;
                else n = h;
            }
            const uint32_t b = lo;
            runs[r] = (unsigned long long)v | ((unsigned long long)b << 16) |
                      ((unsigned long long)L << 32);
            const bool first = p == s_start[b], last = p + L == s_start[b] + s_cnt[b];
            if (first) s_run0[b] = r;
            if (last) s_run1[b] = r;
            if (!first && !last)
                add_symbol((GF ? A.freq + (size_t)cur_tensor * B * NS : S.freq) + b * NS, NS, B,
                           cur_tensor * B + b, v, L, A);
        }
        if (tid == 0) A.tile_nruns[ti] = R;
        __syncthreads();
        for (uint32_t b = tid; b < B; b += kCB) {
            Seg G{};
            G.n = s_cnt[b];
            if (G.n) {
                G.run_begin = s_run0[b];
                G.run_end = s_run1[b] + 1;
                const uint32_t pb = S.hp[G.run_begin], pe = S.hp[G.run_end - 1];
                G.fv = S.sd[pb];
                G.lv = S.sd[pe];
                G.lead = S.hp[G.run_begin + 1] - pb;
                G.trail = S.hp[G.run_end] - pe;
            }
            A.segs[(size_t)ti * B + b] = G;
        }
        __syncthreads();
    }
    if (!GF && cur_tensor != 0xffffffffu) {
        uint32_t* gf = A.freq + (size_t)cur_tensor * B * NS;
        for (uint32_t i = tid; i < B * NS; i += kCB) {
            const uint32_t c = S.freq[i];
            if (c) atomicAdd(gf + i, c);
        }
    }
}

// ---- E1 for DELTA records: sparse formulation -----------------------------------
// Between consecutive checkpoints most levels do not move, so most cyclic deltas are
// zero (96 % at C2).  A group's RLE stream (codec.cpp:79-90) is then zero runs
// between a few non-zero deltas, and the only per-element work needed is
//   * the key (previous level) histogram of the tile: group sizes, and
//   * for the non-zero elements only, the rank inside their group (the number of
//     same-key elements before them in the tile) and among the non-zero ones.
// Per tile (4096 elements, thread t owns elements 16t..16t+15):
//   L  levels -> key / delta bytes (SIMD), validation, CRC (as enc_tile_kernel);
//      per 32-element block (a thread pair) and key: element and non-zero counts
//      (shared atomics)
//   H  one warp scan per key over the 128 blocks -> block prefixes; key offsets
//      of the non-zero elements
//   Z  every non-zero element (by its owning thread): rank r in its group = block
//      prefix + same-key bytes before it in its block (SIMD compares), slot among
//      the key's non-zero elements likewise -> Z[key-sorted slot] = (r, v, key)
//   R  runs from Z: a zero run before an entry whose predecessor in the group is
//      not adjacent, a value run at every head (new value or after a gap), a
//      trailing zero run; run positions by one packed block scan; groups without
//      non-zero elements are one zero run.  Output (runs, segments, interior-run
//      symbol frequencies, tile CRC) is the format enc_tile_kernel writes.
// Seven block barriers per tile (single-barrier scans); Z lives in shared memory
// up to kZCap non-zero elements, in a per-CTA global slice for denser tiles.
constexpr int kNBlk = kCB;                // count blocks per tile: one per thread (16 elements)
constexpr int kZCap = 2048;               // non-zero elements held in shared memory

// Exclusive block scan with one barrier: warp totals in slots[kCB / 32]; the slots
// must not be reused before every thread has passed a later barrier.
template <typename T>
__device__ __forceinline__ T block_exscan1(T v, T* slots, T* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) slots[wid] = x;
    __syncthreads();
    T base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kCB / 32; ++w) {
        const T s = slots[w];
        base += w < wid ? s : T(0);
        tot += s;
    }
    *total = tot;
    return base + x - v;
}

struct DSmem {
    uint32_t* freq;   // B*NS per tensor
    uint32_t* crc;    // kCrcTabs*256
    uint32_t* nib;    // kNibConsts*8*16
    uint32_t* hc;     // [B][kNBlk]: counts (lo 16) | non-zero counts (hi 16) -> exclusive prefixes
    uint16_t* hp;     // kTile + 1: slots of run heads (aliases hc after Z)
    uint32_t* z;      // kZCap: r | v << 16 | key << 24, key-sorted
};

__host__ __device__ inline size_t dsm_hc_bytes(uint32_t B) {
    const size_t a = ((size_t)kNBlk * B * 4 + 15) & ~(size_t)15, b = (size_t)(kTile + 8) * 2;
    return a > b ? a : b;
}

__host__ __device__ inline size_t dsm_bytes(uint32_t B, uint32_t NS) {
    return (((size_t)B * NS * 4 + 15) & ~(size_t)15) + (size_t)kCrcTabs * 256 * 4 +
           (size_t)kNibConsts * 8 * 16 * 4 + dsm_hc_bytes(B) + (size_t)kZCap * 4;
}

__device__ inline DSmem dsm_carve(uint8_t* base, uint32_t B, uint32_t NS) {
    DSmem S;
    size_t o = 0;
    S.freq = (uint32_t*)(base + o); o += ((size_t)B * NS * 4 + 15) & ~(size_t)15;
    S.crc = (uint32_t*)(base + o);  o += (size_t)kCrcTabs * 256 * 4;
    S.nib = (uint32_t*)(base + o);  o += (size_t)kNibConsts * 8 * 16 * 4;
    S.hc = (uint32_t*)(base + o);
    S.hp = (uint16_t*)(base + o);
    o += dsm_hc_bytes(B);
    S.z = (uint32_t*)(base + o);
    return S;
}

// Per-tile run state shared by the R phase helpers.
struct DRun {
    uint32_t *n, *nz, *zoff, *gruns, *gbase, *fv, *lv, *lead, *trail, *aux;
};

// R1: up to PER key-sorted entries per thread (consecutive slots): run counts
// (zero run before, value run at a head, trailing zero run) and flags.
template <int PER>
__device__ __forceinline__ void r_count(const uint32_t* Z, const DRun& D, uint32_t nzt, uint32_t j0,
                                        uint32_t (&zc)[PER], uint32_t (&fl)[PER],
                                        uint32_t& cnt_runs, uint32_t& cnt_heads) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        zc[u] = 0;
        fl[u] = 0;
        const uint32_t j = j0 + u;
        if (j >= nzt) continue;
        const uint32_t z = Z[j];
        const uint32_t r = z & 0xffffu, v = (z >> 16) & 0xffu, k = z >> 24;
        const bool first = j == D.zoff[k], last = j + 1 == D.zoff[k + 1];
        uint32_t pr = 0, pv = 0;
        if (!first) {
            const uint32_t p = Z[j - 1];
            pr = p & 0xffffu;
            pv = (p >> 16) & 0xffu;
        }
        const bool zb = first ? r > 0 : pr + 1 < r;
        const bool head = first || pr + 1 < r || pv != v;
        const bool tail = last && r + 1 < D.n[k];
        zc[u] = z;
        fl[u] = (zb ? 1u : 0u) | (head ? 2u : 0u) | (tail ? 4u : 0u) | (first ? 8u : 0u) | 16u;
        const uint32_t c = (zb ? 1u : 0u) + (head ? 1u : 0u) + (tail ? 1u : 0u);
        cnt_runs += c;
        cnt_heads += head ? 1u : 0u;
        atomicAdd(&D.gruns[k], c);
        if (tail) D.aux[k] = 1;
    }
}

template <int PER>
__device__ __forceinline__ void r_heads(const DSmem& S, uint32_t j0, const uint32_t (&fl)[PER],
                                        uint32_t h) {
#pragma unroll
    for (int u = 0; u < PER; ++u)
        if (fl[u] & 2u) S.hp[h++] = (uint16_t)(j0 + u);
}

// R2: the runs of the thread's entries at their tile positions; first / last runs
// of a group go to the segment, interior ones to the symbol frequencies.
template <int PER>
__device__ __forceinline__ void r_emit(const EncArgs& A, const DSmem& S, const uint32_t* Z, const DRun& D,
                                       uint32_t tensor, uint32_t j0, const uint32_t (&zc)[PER],
                                       const uint32_t (&fl)[PER], uint32_t xr, uint32_t h,
                                       unsigned long long* runs) {
    const uint32_t B = A.B, NS = A.NS;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        if (!fl[u]) continue;
        const uint32_t z = zc[u], f = fl[u];
        const uint32_t r = z & 0xffffu, v = (z >> 16) & 0xffu, k = z >> 24;
        const uint32_t j = j0 + u;
        const uint32_t p0 = xr + (D.aux[k] >> 1);  // + one run per empty group before k
        uint32_t p = p0;
        uint32_t* fk = S.freq + k * NS;
        const uint32_t tb = tensor * B + k;
        const bool gtail = D.aux[k] & 1u;
        if (f & 1u) {  // zero run before the entry
            const uint32_t pr = (f & 8u) ? 0u : (Z[j - 1] & 0xffffu) + 1u;
            const uint32_t L = r - pr;
            runs[p++] = ((unsigned long long)k << 16) | ((unsigned long long)L << 32);
            if (f & 8u) {
                D.fv[k] = 0;
                D.lead[k] = L;
            } else {
                add_symbol(fk, NS, B, tb, 0u, L, A);
            }
        }
        if (f & 2u) {  // value run: up to the next head of the group
            const uint32_t nxt = min((uint32_t)S.hp[h + 1], D.zoff[k + 1]);
            const uint32_t L = nxt - j;
            runs[p++] = (unsigned long long)v | ((unsigned long long)k << 16) |
                        ((unsigned long long)L << 32);
            const bool is_first = (f & 8u) && !(f & 1u);
            const bool is_last = !gtail && nxt == D.zoff[k + 1];
            if (is_first) {
                D.fv[k] = v;
                D.lead[k] = L;
            }
            if (is_last) {
                D.lv[k] = v;
                D.trail[k] = L;
            }
            if (!is_first && !is_last) add_symbol(fk, NS, B, tb, v, L, A);
            ++h;
        }
        if (f & 4u) {  // trailing zero run
            const uint32_t L = D.n[k] - r - 1;
            runs[p++] = ((unsigned long long)k << 16) | ((unsigned long long)L << 32);
            D.lv[k] = 0;
            D.trail[k] = L;
        }
        xr += p - p0;
    }
}

template <int PER>
__device__ __forceinline__ void r_phase(const EncArgs& A, const DSmem& S, const uint32_t* Z,
                                        const DRun& D, uint32_t tensor, uint32_t nzt,
                                        unsigned long long* slots, unsigned long long* runs) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t B = A.B;
    const uint32_t j0 = tid * PER;
    uint32_t zc[PER], fl[PER];
    uint32_t cnt_runs = 0, cnt_heads = 0;
    r_count<PER>(Z, D, nzt, j0, zc, fl, cnt_runs, cnt_heads);
    unsigned long long tot;
    const unsigned long long ex = block_exscan1<unsigned long long>(
        (unsigned long long)cnt_runs | ((unsigned long long)cnt_heads << 32), slots, &tot);
    const uint32_t xr = (uint32_t)ex, xh = (uint32_t)(ex >> 32);
    r_heads<PER>(S, j0, fl, xh);
    if (tid == 0) S.hp[tot >> 32] = (uint16_t)nzt;
    if (wid == 0) {  // per key: run base (an empty group is one zero run)
        uint32_t run = 0, erun = 0;
        for (uint32_t b0 = 0; b0 < B; b0 += 32) {
            const uint32_t b = b0 + lane;
            const uint32_t empty = (b < B && D.n[b] && !D.nz[b]) ? 1u : 0u;
            const uint32_t v = b < B ? D.gruns[b] + empty : 0u;
            const uint32_t vx = v | (empty << 16);  // runs (lo 16) | empty groups (hi 16)
            uint32_t x = vx;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (b < B) {
                D.gbase[b] = run + ((x - vx) & 0xffffu);
                D.gruns[b] = v;
                D.aux[b] |= (erun + ((x - vx) >> 16)) << 1;
            }
            const uint32_t last = __shfl_sync(0xffffffffu, x, 31);
            run += last & 0xffffu;
            erun += last >> 16;
        }
        if (lane == 0) D.gbase[B] = run;
    }
    __syncthreads();
    for (uint32_t b = tid; b < B; b += kCB)  // empty groups: one zero run covering the group
        if (D.n[b] && !D.nz[b]) {
            runs[D.gbase[b]] = ((unsigned long long)b << 16) | ((unsigned long long)D.n[b] << 32);
            D.fv[b] = D.lv[b] = 0;
            D.lead[b] = D.trail[b] = D.n[b];
        }
    r_emit<PER>(A, S, Z, D, tensor, j0, zc, fl, xr, xh, runs);
}

// ---- fused pass C (quantize.cpp:396-423) ------------------------------------------
// compress_step with a base: the target levels are computed inside the DELTA tile
// pass from w and pass B's 2-bit partition codes, written once, and encoded from
// registers (no level read-back); protected (pos, bf16) entries are compacted per
// tile at pass B's per-tile offsets, in element order.

// 16 levels of one thread (elements e0..e0+15 of the tile, nv valid) as bytes, and
// the protected-element mask: nearest-centre level by branch-free bisection over the
// boundaries (pass_c_tile), PRUNED = k, PROTECTED = k + 1.
template <int LOGP>
__device__ __forceinline__ void fused_levels(const float* s_lb, const float4 (&wv)[4], uint32_t pw,
                                             uint32_t k, uint32_t (&cw)[4], uint32_t& pmask) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float4 v = wv[q];
        const float a[4] = {v.x, v.y, v.z, v.w};
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            // the search walks a shared-memory pointer: one load with an immediate
            // offset, one compare and one predicated add per step
            const float* p = s_lb;
#pragma unroll
            for (int st = (1 << LOGP) >> 1; st > 0; st >>= 1)
                if (a[j] >= p[st]) p += st;
            const uint32_t pos = (uint32_t)(p - s_lb);
            const uint32_t part = (pw >> (2 * (4 * q + j))) & 3u;
            const uint32_t lv = part ? k + (part >> 1) : pos;  // PRUNED = k, PROTECTED = k + 1
            word |= lv << (8 * j);
            pmask |= (part >> 1) << (4 * q + j);
        }
        cw[q] = word;
    }
}

template <bool FUSED>
__global__ void __launch_bounds__(kCB, 3) enc_tile_delta_kernel(EncArgs A, FuseC F) {
    extern __shared__ __align__(16) uint8_t e1_dyn[];
    const uint32_t B = A.B, NS = A.NS;
    const DSmem S = dsm_carve(e1_dyn, B, NS);
    __shared__ uint32_t s_n[kMaxB], s_nz[kMaxB], s_zoff[kMaxB + 1], s_gruns[kMaxB], s_gbase[kMaxB + 1];
    __shared__ uint32_t s_fv[kMaxB], s_lv[kMaxB], s_lead[kMaxB], s_trail[kMaxB], s_aux[kMaxB];
    __shared__ uint32_t s_part[kCB / 32];
    __shared__ unsigned long long s_slots[kCB / 32];
    __shared__ uint32_t s_pslots[kCB / 32];
    __shared__ float s_lb[64];  // FUSED: level boundaries of the current layer type
    __shared__ uint32_t s_k, s_logp;
    __shared__ int s_base;
    const DRun D{s_n, s_nz, s_zoff, s_gruns, s_gbase, s_fv, s_lv, s_lead, s_trail, s_aux};
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t Brep = B * 0x01010101u;

    for (uint32_t i = tid; i < kCrcTabs * 256; i += kCB) S.crc[i] = (&g_crc_slice[0][0])[i];
    for (uint32_t i = tid; i < kNibConsts * 8 * 16; i += kCB) S.nib[i] = (&g_crc_nib[0][0][0])[i];
    for (uint32_t i = tid; i < B * NS; i += kCB) S.freq[i] = 0;
    for (uint32_t i = tid; i < kNBlk * B / 4; i += kCB) ((uint4*)S.hc)[i] = make_uint4(0, 0, 0, 0);
    for (uint32_t b = tid; b < B; b += kCB) s_nz[b] = s_gruns[b] = s_aux[b] = 0;
    uint32_t* zg = A.zs + (size_t)blockIdx.x * kTile;  // Z of tiles denser than kZCap
    uint32_t cur_tensor = 0xffffffffu;

    for (int base; (base = grab_tiles(A.tile_ctr, 4, &s_base)) < A.ntiles;)
    for (int ti = base; ti < min(base + 4, A.ntiles); ++ti) {
        const Tile T = A.tiles[ti];
        const uint32_t cnt = T.count;
        if (tid == 0 && ti + 1 < min(base + 4, A.ntiles)) {  // next tile's levels into L2
            const Tile N = A.tiles[ti + 1];
            const uint32_t bytes = ((N.count + 7u) & ~7u) * 2u;
            if (FUSED) {
                prefetch_l2(F.w + N.start, ((N.count + 3u) & ~3u) * 4u);
                if (!F.pbits) prefetch_l2(F.parts + (N.start >> 2), ((N.count + 15u) & ~15u) >> 2);
            } else {
                prefetch_l2(A.cur + N.start, bytes);
            }
            prefetch_l2(A.prev + N.start, bytes);
        }
        if (T.tensor != cur_tensor) {  // flush the previous tensor's symbol counts
            __syncthreads();
            if (cur_tensor != 0xffffffffu) {
                uint32_t* gf = A.freq + (size_t)cur_tensor * B * NS;
                for (uint32_t i = tid; i < B * NS; i += kCB) {
                    const uint32_t c = S.freq[i];
                    if (c) {
                        atomicAdd(gf + i, c);
                        S.freq[i] = 0;
                    }
                }
            }
            cur_tensor = T.tensor;
            if (FUSED) {  // level boundaries of the tensor's layer type (+inf padded to 64)
                const int lt = A.types[T.tensor];
                const uint32_t k = F.cb_len[lt];
                uint32_t kp = 1, lg = 0;
                while (kp < k) kp <<= 1, ++lg;
                if (tid < 64) s_lb[tid] = tid < (int)kp ? F.lb[lt * F.lb_stride + tid]
                                                        : __int_as_float(0x7f800000);
                if (tid == 0) s_k = k, s_logp = lg;
                __syncthreads();
            }
        }
        // ---- L: 16 levels per thread, deltas, validation, CRC; block key counts
        const uint32_t e0 = tid * kIt;
        const uint32_t nv = e0 < cnt ? min(cnt - e0, (uint32_t)kIt) : 0u;
        uint32_t kw[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu}, dwv[4] = {0, 0, 0, 0};
        uint32_t nzm = 0;  // non-zero delta bits of the 16 elements
        uint32_t pmask = 0;  // FUSED: protected elements
        {
            uint32_t cw[4] = {0, 0, 0, 0}, pw[4] = {0, 0, 0, 0};
            if (nv) {
                const uint4* pp = (const uint4*)(A.prev + T.start + e0);
                const uint4 b0 = pp[0], b1 = pp[1];
                uint4 a0 = make_uint4(0, 0, 0, 0), a1 = a0;
                if (FUSED) {
                    // w's loads first: their latency overlaps the partition word's
                    const float* wp = F.w + T.start + e0;
                    float4 wv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        wv[q] = (uint32_t)(4 * q) < nv ? __ldg((const float4*)(wp + 4 * q))
                                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                    uint32_t pc;  // 2-bit partition codes of the 16 elements
                    if (F.pbits) {  // protected bitmap (no pruning): bit -> code 2
                        uint32_t x = (F.pbits[(T.start + e0) >> 5] >> ((T.start + e0) & 31)) & 0xffffu;
                        x = (x | (x << 8)) & 0x00ff00ffu;
                        x = (x | (x << 4)) & 0x0f0f0f0fu;
                        x = (x | (x << 2)) & 0x33333333u;
                        x = (x | (x << 1)) & 0x55555555u;
                        pc = x << 1;
                    } else {
                        pc = *(const uint32_t*)(F.parts + ((T.start + e0) >> 2));
                    }
                    switch (s_logp) {
#define DQTG_FL(L) case L: fused_levels<L>(s_lb, wv, pc, s_k, cw, pmask); break;
                        DQTG_FL(0) DQTG_FL(1) DQTG_FL(2) DQTG_FL(3) DQTG_FL(4) DQTG_FL(5)
                        default: fused_levels<6>(s_lb, wv, pc, s_k, cw, pmask);
#undef DQTG_FL
                    }
                    if (nv < (uint32_t)kIt) {
                        pmask &= (1u << nv) - 1u;
#pragma unroll
                        for (int j = 0; j < 4; ++j) cw[j] &= keep_mask((int)nv - 4 * j);
                    }
                    // u16 levels (little-endian: level, 0); the tile's padding gets 0
                    uint16_t* lp = F.levels + T.start + e0;
                    *(uint4*)lp = make_uint4(__byte_perm(cw[0], 0, 0x4140), __byte_perm(cw[0], 0, 0x4342),
                                             __byte_perm(cw[1], 0, 0x4140), __byte_perm(cw[1], 0, 0x4342));
                    *(uint4*)(lp + 8) = make_uint4(__byte_perm(cw[2], 0, 0x4140), __byte_perm(cw[2], 0, 0x4342),
                                                   __byte_perm(cw[3], 0, 0x4140), __byte_perm(cw[3], 0, 0x4342));
                } else {
                    const uint4* cp = (const uint4*)(A.cur + T.start + e0);
                    a0 = cp[0], a1 = cp[1];
                    cw[0] = __byte_perm(a0.x, a0.y, 0x6420);
                    cw[1] = __byte_perm(a0.z, a0.w, 0x6420);
                    cw[2] = __byte_perm(a1.x, a1.y, 0x6420);
                    cw[3] = __byte_perm(a1.z, a1.w, 0x6420);
                }
                const uint32_t hi[8] = {a0.x | b0.x, a0.y | b0.y, a0.z | b0.z, a0.w | b0.w,
                                        a1.x | b1.x, a1.y | b1.y, a1.z | b1.z, a1.w | b1.w};
                pw[0] = __byte_perm(b0.x, b0.y, 0x6420);
                pw[1] = __byte_perm(b0.z, b0.w, 0x6420);
                pw[2] = __byte_perm(b1.x, b1.y, 0x6420);
                pw[3] = __byte_perm(b1.z, b1.w, 0x6420);
                uint32_t bad = 0;
                if (nv == (uint32_t)kIt) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) bad |= hi[j];
                    bad &= 0xff00ff00u;
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int keep = (int)nv - 2 * j;
                        const uint32_t m = keep >= 2 ? 0xff00ff00u : (keep == 1 ? 0x0000ff00u : 0u);
                        bad |= hi[j] & m;
                    }
                }
                uint32_t big = 0;
                const bool full = nv == (uint32_t)kIt;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t m = full ? 0xffffffffu : keep_mask((int)nv - 4 * j);
                    cw[j] &= m;
                    pw[j] &= m;
                    big |= __vcmpgeu4(cw[j], Brep) | __vcmpgeu4(pw[j], Brep);
                    const uint32_t lt = __vcmpltu4(pw[j], cw[j]);
                    dwv[j] = __vadd4(__vsub4(pw[j], cw[j]), lt & Brep) & m;
                    kw[j] = pw[j] | ~m;  // no element: key 0xff
                    nzm |= byte_msbs(__vcmpne4(dwv[j], 0u)) << (4 * j);
                }
                if (bad | big) atomicOr(A.err, kErrCorruptIndex);
            }
            // CRC of this thread's levels (zero register), right-aligned in its 32-byte chunk
            uint32_t c0 = cw[0], c1 = cw[1], c2 = cw[2], c3 = cw[3];
            if (nv && nv < (uint32_t)kIt) {
                const int sh = kIt - (int)nv;
                uint32_t w[8] = {0, 0, 0, 0, cw[0], cw[1], cw[2], cw[3]};
                uint32_t o[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int src = 4 + j - (sh >> 2);
                    const uint32_t lo_w = src - 1 >= 0 ? w[src - 1] : 0u;
                    o[j] = (sh & 3) ? __funnelshift_l(lo_w, w[src], 8 * (sh & 3)) : w[src];
                }
                c0 = o[0], c1 = o[1], c2 = o[2], c3 = o[3];
            }
            uint32_t r = 0;
            if (nv) r = crc_block8(S.crc, crc_block8(S.crc, 0u, c0, c1), c2, c3);
            if (cnt == kTile) {
                r = crc_warp(S.nib, r);
                if (lane == 0) s_part[wid] = r;
            } else {
                if (r) r = crc_shift(c_crc_x2n, r, 2ull * (cnt - (e0 + nv)));
                r = warp_xor(r);
                if (lane == 0) s_part[wid] = r;
            }
            // block (= thread) counts: elements (lo 16 bits) and non-zero elements (hi
            // 16 bits), conflict-free (one column per thread); per key: non-zero elements
            uint32_t* hb = S.hc + tid;
            if (nv == (uint32_t)kIt) {  // full threads: no per-element bound checks
#pragma unroll
                for (int j = 0; j < kIt; ++j) {
                    const uint32_t k = (kw[j >> 2] >> (8 * (j & 3))) & 0xffu;
                    atomicAdd(hb + k * kNBlk, 1u + ((nzm >> j & 1u) << 16));
                }
            } else {
#pragma unroll
                for (int j = 0; j < kIt; ++j) {
                    if ((uint32_t)j >= nv) break;
                    const uint32_t k = (kw[j >> 2] >> (8 * (j & 3))) & 0xffu;
                    atomicAdd(hb + k * kNBlk, (nzm >> j & 1u) ? 0x10001u : 1u);
                }
            }
            for (uint32_t m = nzm; m; m &= m - 1) {
                const uint32_t j = __ffs(m) - 1;
                atomicAdd(&s_nz[(kw[j >> 2] >> (8 * (j & 3))) & 0xffu], 1u);
            }
        }
        if (FUSED) {  // protected entries in element order (the scan's barrier ends L)
            uint32_t ptot;
            const uint32_t pex = block_exscan1<uint32_t>(__popc(pmask), s_pslots, &ptot);
            unsigned long long o = F.tile_prot_off[ti] + pex;
            const uint64_t tbase = A.off[T.tensor];
            for (uint32_t m = pmask; m; m &= m - 1) {
                const uint32_t j = __ffs(m) - 1;
                F.ppos[o] = (T.start - tbase) + e0 + j;
                F.pval[o] = bf16_rne(F.w[T.start + e0 + j]);
                ++o;
            }
        } else {
            __syncthreads();
        }
        // ---- H: per key, exclusive prefix over the 256 blocks (one warp per key)
        for (uint32_t k = wid; k < B; k += kCB / 32) {
            uint4* row = (uint4*)(S.hc + k * kNBlk + 8 * lane);
            const uint4 v = row[0], u = row[1];
            const uint32_t s1 = v.x + v.y, s2 = s1 + v.z, s3 = s2 + v.w, s4 = s3 + u.x,
                           s5 = s4 + u.y, s6 = s5 + u.z, s7 = s6 + u.w;
            uint32_t x = s7;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            const uint32_t ex = x - s7;
            row[0] = make_uint4(ex, ex + v.x, ex + s1, ex + s2);
            row[1] = make_uint4(ex + s3, ex + s4, ex + s5, ex + s6);
            if (lane == 31) s_n[k] = x & 0xffffu;
        }
        if (wid == 0) {  // slot offsets of the keys' non-zero elements in Z
            uint32_t run = 0;
            for (uint32_t b0 = 0; b0 < B; b0 += 32) {
                const uint32_t b = b0 + lane;
                const uint32_t v = b < B ? s_nz[b] : 0u;
                uint32_t x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (b < B) s_zoff[b] = run + x - v;
                run += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) s_zoff[B] = run;
        }
        if (wid == kCB / 32 - 1) {  // tile CRC (moved to its stream position by crc_tiles_kernel)
            uint32_t r = lane < kCB / 32 ? s_part[lane] : 0u;
            if (cnt == kTile) r = crc_tree(S.nib, r, 10, 3);
            else r = warp_xor(r);
            if (lane == 0) A.tile_crc[ti] = r;
        }
        __syncthreads();
        // ---- Z: every non-zero element, by its owning thread
        const uint32_t nzt = s_zoff[B];
        uint32_t* Z = nzt <= (uint32_t)kZCap ? S.z : zg;
        // the thread's own 16 keys / deltas are its count block: ranks from registers
        // (16-bit mask of the equal keys, counted below j)
        for (uint32_t m = nzm; m; m &= m - 1) {
            const uint32_t j = __ffs(m) - 1;
            const uint32_t wj = j >> 2, sh = 8 * (j & 3);
            const uint32_t kwj = wj == 0 ? kw[0] : wj == 1 ? kw[1] : wj == 2 ? kw[2] : kw[3];
            const uint32_t dwj = wj == 0 ? dwv[0] : wj == 1 ? dwv[1] : wj == 2 ? dwv[2] : dwv[3];
            const uint32_t k = (kwj >> sh) & 0xffu, v = (dwj >> sh) & 0xffu;
            const uint32_t krep = k * 0x01010101u;
            uint32_t em = 0;
#pragma unroll
            for (int w = 0; w < 4; ++w) em |= byte_msbs(__vcmpeq4(kw[w], krep)) << (4 * w);
            const uint32_t below = em & ((1u << j) - 1u);
            const uint32_t acc = __popc(below), accnz = __popc(below & nzm);  // same key before j
            const uint32_t pre = S.hc[k * kNBlk + tid];
            Z[s_zoff[k] + (pre >> 16) + accnz] = ((pre & 0xffffu) + acc) | (v << 16) | (k << 24);
        }
        __syncthreads();
        // ---- R: runs (key-sorted entries, consecutive slots per thread)
        unsigned long long* runs = A.runs + (size_t)ti * kTile;
        if (nzt <= (uint32_t)kCB) r_phase<1>(A, S, Z, D, cur_tensor, nzt, s_slots, runs);
        else if (nzt <= 4u * kCB) r_phase<4>(A, S, Z, D, cur_tensor, nzt, s_slots, runs);
        else r_phase<kTile / kCB>(A, S, Z, D, cur_tensor, nzt, s_slots, runs);
        if (tid == 0) A.tile_nruns[ti] = s_gbase[B];
        __syncthreads();
        for (uint32_t b = tid; b < B; b += kCB) {
            Seg G{};
            G.n = s_n[b];
            if (G.n) {
                G.run_begin = s_gbase[b];
                G.run_end = s_gbase[b + 1];  // groups' runs are contiguous, in key order
                G.fv = (uint16_t)s_fv[b];
                G.lv = (uint16_t)s_lv[b];
                G.lead = s_lead[b];
                G.trail = s_trail[b];
            }
            A.segs[(size_t)ti * B + b] = G;
            s_nz[b] = s_gruns[b] = s_aux[b] = 0;
        }
        for (uint32_t i = tid; i < kNBlk * B / 4; i += kCB) ((uint4*)S.hc)[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
    }
    if (cur_tensor != 0xffffffffu) {
        uint32_t* gf = A.freq + (size_t)cur_tensor * B * NS;
        for (uint32_t i = tid; i < B * NS; i += kCB) {
            const uint32_t c = S.freq[i];
            if (c) atomicAdd(gf + i, c);
        }
    }
}

// CRC of one tile of a level array (zero register, ending at the tile's last byte),
// 16 levels per thread (levels must be < 256: validated by the caller).
__global__ void __launch_bounds__(kCB) level_crc_tile_kernel(const Tile* tiles, const uint16_t* levels,
                                                             uint32_t* tile_crc) {
    __shared__ uint32_t s_crc[kCrcTabs * 256];
    __shared__ uint32_t s_nib[kNibConsts * 8 * 16];
    __shared__ uint32_t s_part[kCB / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (uint32_t i = tid; i < kCrcTabs * 256; i += kCB) s_crc[i] = (&g_crc_slice[0][0])[i];
    for (uint32_t i = tid; i < kNibConsts * 8 * 16; i += kCB) s_nib[i] = (&g_crc_nib[0][0][0])[i];
    __syncthreads();
    const Tile T = tiles[blockIdx.x];
    const uint32_t cnt = T.count, e0 = tid * kIt;
    const uint32_t nv = e0 < cnt ? min(cnt - e0, (uint32_t)kIt) : 0u;
    uint32_t cw[4] = {0, 0, 0, 0};
    if (nv) {
        const uint4* cp = (const uint4*)(levels + T.start + e0);
        const uint4 a0 = cp[0], a1 = cp[1];
        cw[0] = __byte_perm(a0.x, a0.y, 0x6420);
        cw[1] = __byte_perm(a0.z, a0.w, 0x6420);
        cw[2] = __byte_perm(a1.x, a1.y, 0x6420);
        cw[3] = __byte_perm(a1.z, a1.w, 0x6420);
#pragma unroll
        for (int j = 0; j < 4; ++j) cw[j] &= keep_mask((int)nv - 4 * j);
    }
    uint32_t c0 = cw[0], c1 = cw[1], c2 = cw[2], c3 = cw[3];
    if (nv && nv < (uint32_t)kIt) {  // right-align the tail chunk (leading zeros are neutral)
        const int sh = kIt - (int)nv;
        uint32_t w[8] = {0, 0, 0, 0, cw[0], cw[1], cw[2], cw[3]};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int src = 4 + j - (sh >> 2);
            const uint32_t lo_w = src - 1 >= 0 ? w[src - 1] : 0u;
            o[j] = (sh & 3) ? __funnelshift_l(lo_w, w[src], 8 * (sh & 3)) : w[src];
        }
        c0 = o[0], c1 = o[1], c2 = o[2], c3 = o[3];
    }
    uint32_t r = 0;
    if (nv) r = crc_block8(s_crc, crc_block8(s_crc, 0u, c0, c1), c2, c3);
    if (cnt == kTile) {
        r = crc_warp(s_nib, r);
        if (lane == 0) s_part[wid] = r;
    } else {
        if (r) r = crc_shift(c_crc_x2n, r, 2ull * (cnt - (e0 + nv)));
        r = warp_xor(r);
        if (lane == 0) s_part[wid] = r;
    }
    __syncthreads();
    if (wid == 0) {
        uint32_t v = lane < kCB / 32 ? s_part[lane] : 0u;
        if (cnt == kTile) v = crc_tree(s_nib, v, 10, 3);
        else v = warp_xor(v);
        if (lane == 0) tile_crc[blockIdx.x] = v;
    }
}

// Tile CRCs (each ending at its tile's last byte) moved to the end of the level
// stream and XOR-combined (crc32 linearity, crc.cuh).
__global__ void __launch_bounds__(256) crc_tiles_kernel(const uint32_t* tile_crc,
                                                        const uint32_t* shift, int ntiles,
                                                        uint32_t* acc) {
    uint32_t r = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        const uint32_t v = tile_crc[t];
        if (v) r ^= crc_multmodp(shift[t], v);
    }
    r = warp_xor(r);
    if ((threadIdx.x & 31) == 0 && r) atomicXor(acc, r);
}

// ---- S: cross-tile run resolution per (tensor, group) --------------------------
struct RunM {  // run-length monoid over a concatenation of segments
    unsigned long long n, lead;
    uint32_t fv, lv;
    uint32_t single;  // whole concatenation is one run
};

__device__ __forceinline__ RunM runm_combine(const RunM& a, const RunM& b) {
    if (!a.n) return b;
    if (!b.n) return a;
    RunM r;
    r.n = a.n + b.n;
    r.fv = a.fv;
    r.lv = b.lv;
    const bool join = a.single && a.lv == b.fv;
    r.single = join && b.single;
    r.lead = join ? a.n + b.lead : a.lead;
    return r;
}

__device__ __forceinline__ RunM shfl_down_runm(const RunM& m, int o);

// Tensors with many tiles: chunks of kResChunk tiles, three launches.
//   R1 (block per (chunk, group)): the chunk's aggregates -- the last non-empty
//      segment (forward) and the run monoid of its segments (backward);
//   R2 (thread per (tensor, group)): carries over the tensor's chunks -- the last
//      non-empty segment before each chunk, the monoid of the segments after it;
//   R3 (block per (chunk, group)): the forward continuation flags and the backward
//      run extensions of the chunk's segments with those carries, symbol counts
//      added to the tensor's frequencies.
// Every chunk works in parallel (the run across tiles, codec.cpp:79-90, of one
// 38.6 M-element tensor used to be walked by a single block).
constexpr int kResPer = 4;                       // tiles per thread
constexpr uint32_t kResChunk = kCB * kResPer;    // tiles per chunk
struct ResChunk {
    uint32_t t, c0, c1, k;  // tensor, tile range [c0, c1), chunk index within the tensor
    uint32_t first;         // index of the tensor's first chunk in the chunk list
};

__device__ __forceinline__ RunM seg_runm(const Seg& S) {
    RunM m{};
    if (S.n) {
        m.n = S.n;
        m.fv = S.fv;
        m.lv = S.lv;
        m.single = S.lead == S.n;
        m.lead = S.lead;
    }
    return m;
}

__global__ void __launch_bounds__(kCB) enc_resolve_agg_kernel(EncArgs A, const ResChunk* chunks,
                                                              int* fwd_last, RunM* bwd_agg) {
    __shared__ int s_wmax[kCB / 32];
    __shared__ RunM s_wm[kCB / 32];
    const uint32_t B = A.B;
    const ResChunk C = chunks[blockIdx.x / B];
    const uint32_t b = blockIdx.x % B;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t i0 = C.c0 + tid * kResPer;
    int x = -1;
    RunM m[kResPer];
#pragma unroll
    for (int u = 0; u < kResPer; ++u) {
        m[u] = RunM{};
        if (i0 + u < C.c1) {
            const Seg S = A.segs[(size_t)(i0 + u) * B + b];
            m[u] = seg_runm(S);
            if (S.n) x = (int)(i0 + u);
        }
    }
    RunM r = m[kResPer - 1];
#pragma unroll
    for (int u = kResPer - 2; u >= 0; --u) r = runm_combine(m[u], r);
    for (int o = 16; o > 0; o >>= 1) {
        x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // warp suffix: lane 0 holds the warp's monoid
        const RunM y = shfl_down_runm(r, o);
        if (lane + o < 32) r = runm_combine(r, y);
    }
    if (lane == 0) s_wmax[wid] = x, s_wm[wid] = r;
    __syncthreads();
    if (tid == 0) {
        int mx = -1;
        RunM agg{};
        for (int w = kCB / 32 - 1; w >= 0; --w) {
            mx = max(mx, s_wmax[w]);
            agg = runm_combine(s_wm[w], agg);
        }
        fwd_last[blockIdx.x] = mx;
        bwd_agg[blockIdx.x] = agg;
    }
}

__global__ void enc_resolve_carry_kernel(const ResChunk* chunks, uint32_t nchunks, uint32_t B,
                                         int* fwd_last, RunM* bwd_agg) {
    // one thread per (tensor, group): chunk indices of its tensor are consecutive
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nchunks * B) return;
    const uint32_t ci = g / B, b = g % B;
    const ResChunk C = chunks[ci];
    if (C.k != 0) return;  // the tensor's first chunk drives its tensor
    uint32_t n = 0;
    while (ci + n < nchunks && chunks[ci + n].t == C.t) ++n;
    int carry = -1;  // exclusive: last non-empty segment before each chunk
    for (uint32_t j = 0; j < n; ++j) {
        const size_t s = (size_t)(ci + j) * B + b;
        const int v = fwd_last[s];
        fwd_last[s] = carry;
        carry = max(carry, v);
    }
    RunM after{};  // exclusive: monoid of the segments after each chunk
    for (uint32_t j = n; j-- > 0;) {
        const size_t s = (size_t)(ci + j) * B + b;
        const RunM v = bwd_agg[s];
        bwd_agg[s] = after;
        after = runm_combine(v, after);
    }
}

__global__ void __launch_bounds__(kCB) enc_resolve_big_kernel(EncArgs A, const ResChunk* chunks,
                                                              const int* fwd_carry,
                                                              const RunM* bwd_carry) {
    extern __shared__ uint32_t s_f[];  // NS
    __shared__ int s_wmax[kCB / 32];
    __shared__ RunM s_wm[kCB / 32];
    const uint32_t B = A.B, NS = A.NS;
    const ResChunk C = chunks[blockIdx.x / B];
    const uint32_t t = C.t, b = blockIdx.x % B;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t a1 = C.c1;
    for (uint32_t i = tid; i < NS; i += kCB) s_f[i] = 0;
    // forward: lv of the nearest earlier non-empty segment (inclusive max-scan)
    {
        const int carry_last = fwd_carry[blockIdx.x];
        const uint32_t i0 = C.c0 + tid * kResPer;
        int idx[kResPer];
        uint32_t fv[kResPer];
        int x = -1;
#pragma unroll
        for (int u = 0; u < kResPer; ++u) {
            idx[u] = -1;
            fv[u] = 0;
            if (i0 + u < a1) {
                const Seg& S = A.segs[(size_t)(i0 + u) * B + b];
                if (S.n) {
                    idx[u] = (int)(i0 + u);
                    fv[u] = S.fv;
                }
            }
            x = max(x, idx[u]);
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o && y > x) x = y;
        }
        if (lane == 31) s_wmax[wid] = x;
        __syncthreads();
        int before = carry_last;
        for (int w = 0; w < wid; ++w) before = max(before, s_wmax[w]);
        int excl = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) excl = -1;
        int prev = max(before, excl);
#pragma unroll
        for (int u = 0; u < kResPer; ++u)
            if (idx[u] >= 0) {
                A.segs[(size_t)idx[u] * B + b].cont =
                    A.mode != 2 && prev >= 0 && A.segs[(size_t)prev * B + b].lv == fv[u];
                prev = idx[u];
            }
    }
    __syncthreads();
    // backward: suffix run monoid gives the extension of each trailing run
    {
        const RunM carry = bwd_carry[blockIdx.x];
        uint32_t* f = s_f;
        const uint32_t tb = t * B + b;
        const uint32_t i0 = C.c0 + tid * kResPer;
        RunM m[kResPer];
        Seg S[kResPer];
#pragma unroll
        for (int u = 0; u < kResPer; ++u) {
            m[u] = RunM{};
            S[u] = Seg{};
            if (i0 + u < a1) {
                S[u] = A.segs[(size_t)(i0 + u) * B + b];
                m[u] = seg_runm(S[u]);
            }
        }
        RunM x = m[kResPer - 1];
#pragma unroll
        for (int u = kResPer - 2; u >= 0; --u) x = runm_combine(m[u], x);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const RunM y = shfl_down_runm(x, o);
            if (lane + o < 32) x = runm_combine(x, y);
        }
        if (lane == 0) s_wm[wid] = x;
        __syncthreads();
        RunM later = carry;  // suffix of the warps after this one, then the carry
        for (int w = kCB / 32 - 1; w > wid; --w) later = runm_combine(s_wm[w], later);
        RunM nxt = shfl_down_runm(x, 1);  // suffix starting at the next lane
        RunM after = lane < 31 ? runm_combine(nxt, later) : later;
#pragma unroll
        for (int u = kResPer - 1; u >= 0; --u) {  // items of this thread, last first
            if (i0 + u < a1 && S[u].n) {
                unsigned long long E = (A.mode != 2 && after.n && after.fv == S[u].lv) ? after.lead : 0ull;
                const bool single = S[u].lead == S[u].n;
                Seg& G = A.segs[(size_t)(i0 + u) * B + b];
                if (single) {
                    G.lead_total = G.trail_total = S[u].n + E;
                    if (!S[u].cont) add_symbol(f, NS, B, tb, S[u].fv, S[u].n + E, A);
                } else {
                    G.lead_total = S[u].lead;
                    G.trail_total = S[u].trail + E;
                    if (!S[u].cont) add_symbol(f, NS, B, tb, S[u].fv, S[u].lead, A);
                    add_symbol(f, NS, B, tb, S[u].lv, S[u].trail + E, A);
                }
            }
            after = runm_combine(m[u], after);
        }
    }
    __syncthreads();
    uint32_t* gf = A.freq + (size_t)(t * B + b) * NS;
    for (uint32_t i = tid; i < NS; i += kCB)
        if (s_f[i]) atomicAdd(gf + i, s_f[i]);
}

constexpr int kResolveWarps = 8;

__device__ __forceinline__ RunM shfl_down_runm(const RunM& m, int o) {
    RunM r;
    r.n = __shfl_down_sync(0xffffffffu, m.n, o);
    r.lead = __shfl_down_sync(0xffffffffu, m.lead, o);
    r.fv = __shfl_down_sync(0xffffffffu, m.fv, o);
    r.lv = __shfl_down_sync(0xffffffffu, m.lv, o);
    r.single = __shfl_down_sync(0xffffffffu, m.single, o);
    return r;
}

// One warp per (tensor, group): forward "last non-empty value" scan and a
// backward run-monoid suffix scan over the tensor's tiles, 32 tiles at a time.
__global__ void __launch_bounds__(kResolveWarps * 32) enc_resolve_kernel(EncArgs A,
                                                                         const uint32_t* tensors,
                                                                         uint32_t n_pairs) {
    extern __shared__ uint32_t s_f_all[];  // kResolveWarps * NS
    const uint32_t B = A.B, NS = A.NS;
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t pair = blockIdx.x * kResolveWarps + wid;
    if (pair >= n_pairs) return;
    const uint32_t t = tensors[pair / B], b = pair % B;
    const uint32_t tb = t * B + b;
    const uint32_t a0 = A.tile0[t], a1 = A.tile0[t + 1];
    uint32_t* f = s_f_all + wid * NS;
    for (uint32_t i = lane; i < NS; i += 32) f[i] = 0;
    __syncwarp();
    // forward: cont = leading run continues the nearest earlier non-empty segment
    int carry_last = -1;
    bool any = false;
    for (uint32_t c0 = a0; c0 < a1; c0 += 32) {
        const uint32_t i = c0 + lane;
        Seg* S = i < a1 ? &A.segs[(size_t)i * B + b] : nullptr;
        const int idx = (S && S->n) ? (int)i : -1;
        int x = idx;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = max(x, y);
        }
        int prev = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) prev = -1;
        prev = max(prev, carry_last);
        if (idx >= 0) {
            S->cont = A.mode != 2 && prev >= 0 && A.segs[(size_t)prev * B + b].lv == S->fv;
            any = true;
        }
        carry_last = max(carry_last, __shfl_sync(0xffffffffu, x, 31));
    }
    if (!__any_sync(0xffffffffu, any)) return;
    __syncwarp();
    // backward: suffix run monoid gives each trailing run's extension
    RunM carry{};
    for (int64_t c0 = (int64_t)a1 - 32; c0 > (int64_t)a0 - 32; c0 -= 32) {
        const int64_t ii = c0 + lane;
        const bool in = ii >= (int64_t)a0 && ii < (int64_t)a1;
        RunM m{};
        Seg S{};
        if (in) {
            S = A.segs[(size_t)ii * B + b];
            if (S.n) {
                m.n = S.n;
                m.fv = S.fv;
                m.lv = S.lv;
                m.single = S.lead == S.n;
                m.lead = S.lead;
            }
        }
        // inclusive suffix scan over the 32 lanes (lane i combines with later lanes)
        RunM x = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            RunM y = shfl_down_runm(x, o);
            if (lane + o < 32) x = runm_combine(x, y);
        }
        RunM nxt = shfl_down_runm(x, 1);
        RunM after = lane < 31 ? runm_combine(nxt, carry) : carry;
        if (in && S.n) {
            const unsigned long long E = (A.mode != 2 && after.n && after.fv == S.lv) ? after.lead : 0ull;
            Seg& G = A.segs[(size_t)ii * B + b];
            if (S.lead == S.n) {
                G.lead_total = G.trail_total = S.n + E;
                if (!S.cont) add_symbol(f, NS, B, tb, S.fv, S.n + E, A);
            } else {
                G.lead_total = S.lead;
                G.trail_total = S.trail + E;
                if (!S.cont) add_symbol(f, NS, B, tb, S.fv, S.lead, A);
                add_symbol(f, NS, B, tb, S.lv, S.trail + E, A);
            }
        }
        RunM head = shfl_down_runm(x, 0);
        head.n = __shfl_sync(0xffffffffu, x.n, 0);
        head.lead = __shfl_sync(0xffffffffu, x.lead, 0);
        head.fv = __shfl_sync(0xffffffffu, x.fv, 0);
        head.lv = __shfl_sync(0xffffffffu, x.lv, 0);
        head.single = __shfl_sync(0xffffffffu, x.single, 0);
        carry = runm_combine(head, carry);
    }
    __syncwarp();
    uint32_t* gf = A.freq + (size_t)tb * NS;
    for (uint32_t i = lane; i < NS; i += 32)
        if (f[i]) gf[i] += f[i];
}

// ---- overflow run lengths: sorted unique (key, count) ------------------------------
__global__ void ov_unique_kernel(const unsigned long long* sorted, unsigned long long n,
                                 unsigned long long* ukey, unsigned long long* uhead,
                                 unsigned long long* nu) {
    __shared__ unsigned long long s_scan[33];
    unsigned long long base = 0;
    for (unsigned long long c0 = 0; c0 < n; c0 += blockDim.x) {
        unsigned long long i = c0 + threadIdx.x;
        unsigned long long h = (i < n && (i == 0 || sorted[i] != sorted[i - 1])) ? 1ull : 0ull;
        unsigned long long tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(h, s_scan, &tot);
        if (h) {
            ukey[base + ex] = sorted[i];
            uhead[base + ex] = i;
        }
        base += tot;
    }
    if (threadIdx.x == 0) *nu = base;
}

__global__ void ov_counts_kernel(const unsigned long long* uhead, const unsigned long long* nu_p,
                                 unsigned long long n, unsigned long long* ucnt) {
    const unsigned long long nu = *nu_p;
    for (unsigned long long j = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; j < nu;
         j += (unsigned long long)gridDim.x * blockDim.x)
        ucnt[j] = (j + 1 < nu ? uhead[j + 1] : n) - uhead[j];
}

// ---- H: canonical Huffman per (tensor, group) -------------------------------------
struct GroupInfo {
    unsigned long long n_elems, nsyms, bits, nbytes;
    unsigned long long tab_base;  // first table entry
    uint32_t tsize, hdr;          // hdr: header bytes excluding uvarint(nbytes)
    unsigned long long ov_begin, ov_end;
    unsigned long long pay;       // record byte offset of the bitstream
    unsigned long long gbytes;    // full group size in the record
};

__device__ __forceinline__ unsigned long long lb_u64(const unsigned long long* a,
                                                     unsigned long long n,
                                                     unsigned long long key) {
    unsigned long long lo = 0, hi = n;
    while (lo < hi) {
        unsigned long long m = (lo + hi) >> 1;
        if (a[m] < key) lo = m + 1;
        else hi = m;
    }
    return lo;
}

struct HufWork {
    unsigned long long* ovh;    // overflow-length hash: [2 ov_begin, 2 ov_end) per group
    long long* sym;             // [tab_base + i]
    unsigned long long* f;      // [tab_base + i]
    uint32_t* perm;             // [tab_base + i]
    unsigned long long* nodef;  // [2*tab_base + 2*tb + j]
    uint32_t* parent;
    uint32_t* depth;
};

__global__ void ov_group_max_kernel(const unsigned long long* ukey, const unsigned long long* nu_p,
                                    uint32_t ngroups, uint32_t* max_nov,
                                    unsigned long long* ov_range /*[ngroups][2]*/) {
    const unsigned long long nu = *nu_p;
    for (uint32_t tb = blockIdx.x * blockDim.x + threadIdx.x; tb < ngroups;
         tb += gridDim.x * blockDim.x) {
        unsigned long long a = lb_u64(ukey, nu, (unsigned long long)tb << 32);
        unsigned long long b = lb_u64(ukey, nu, (unsigned long long)(tb + 1) << 32);
        ov_range[2 * tb] = a;
        ov_range[2 * tb + 1] = b;
        if (b > a) atomicMax(max_nov, (uint32_t)(b - a));
    }
}

// Groups are launched in tiers by their symbol-count bound (host: (B + kLD) + distinct
// overflow lengths): small and medium tiers keep the working set in shared memory
// (one warp per group, sized for the tier); BIG groups (tens of thousands of
// distinct run lengths in billion-element tensors, C5) keep it in global memory and
// sort with 1024 threads, then continue on warp 0.  glist: the tier's groups;
// gws/goff (BIG): per group (byte offset, n_pad) of its global working set.
template <bool GWS, int NT>  // GWS: working set in global memory (gws/goff); NT threads per group
__global__ void __launch_bounds__(NT) enc_huffman_kernel(EncArgs A, const unsigned long long* elems,
                                                          const unsigned long long* ukey,
                                                          const unsigned long long* ucnt,
                                                          const unsigned long long* nu_p,
                                                          GroupInfo* gi, long long* tab_sym,
                                                          uint8_t* tab_len,
                                                          unsigned long long* code_dense,
                                                          uint8_t* len_dense,
                                                          unsigned long long* code_ov,
                                                          uint8_t* len_ov, HufWork W,
                                                          uint32_t n_pad,
                                                          const unsigned long long* ov_range,
                                                          const uint32_t* glist,
                                                          const unsigned long long* goff,
                                                          uint8_t* gws) {
    // working set (the tree build is a serial chain): n_pad >= n.  32-bit frequencies
    // / node weights / symbols (the host guarantees tensors below 2^31 elements) and
    // 8-bit depths (saturated; >= 63 is an error anyway) keep it at 38 B per slot, so
    // more single-warp CTAs stay resident per SM.
    extern __shared__ unsigned long long s_dyn[];
    unsigned long long* s_keys = s_dyn;
    if (GWS) {
        s_keys = (unsigned long long*)(gws + goff[2 * blockIdx.x]);
        n_pad = (uint32_t)goff[2 * blockIdx.x + 1];
    }
    __shared__ uint32_t s_hist[65], s_at[65], s_n;
    uint32_t* nodef = (uint32_t*)(s_keys + n_pad);   // 2 n_pad
    uint32_t* parent = nodef + 2 * n_pad;            // 2 n_pad
    uint32_t* f = parent + 2 * n_pad;                // n_pad
    int32_t* sym = (int32_t*)(f + n_pad);            // n_pad
    uint32_t* perm = (uint32_t*)(sym + n_pad);       // n_pad
    uint8_t* depth = (uint8_t*)(perm + n_pad);       // 2 n_pad
    const uint32_t B = A.B, NS = A.NS;
    const uint32_t tb = glist[blockIdx.x], b = tb % B;
    GroupInfo G{};
    G.n_elems = elems[tb];
    (void)nu_p;
    G.ov_begin = ov_range[2 * tb];
    G.ov_end = ov_range[2 * tb + 1];
    const uint32_t nov = (uint32_t)(G.ov_end - G.ov_begin);
    G.tab_base = (unsigned long long)tb * NS + G.ov_begin;
    (void)W;
    // symbols in ascending order (the reference's std::map): values -(B-1)..0, dense
    // run lengths 2..63, overflow lengths; compacted warp-wide with ballots
    const uint32_t* fr = A.freq + (size_t)tb * NS;
    const int lane = threadIdx.x & 31;
    uint32_t n = 0;
    if (G.n_elems && threadIdx.x < 32) {
        for (uint32_t i0 = 0; i0 < B + kLD; i0 += 32) {
            const uint32_t i = i0 + lane;
            int32_t sv = 0;
            uint32_t fv = 0;
            if (i < B) {  // value -(B-1-i)
                fv = fr[B - 1 - i];
                sv = -(int32_t)(B - 1 - i);
            } else if (i < B + kLD && i - B >= 2) {
                fv = fr[i];
                sv = (int32_t)(i - B);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, fv != 0);
            if (fv) {
                const uint32_t o = n + __popc(m & ((1u << lane) - 1u));
                sym[o] = sv;
                f[o] = fv;
            }
            n += __popc(m);
        }
        for (unsigned long long j0 = G.ov_begin; j0 < G.ov_end; j0 += 32) {
            const unsigned long long j = j0 + lane;
            if (j < G.ov_end) {
                sym[n + lane] = (int32_t)(ukey[j] & 0x7fffffffull);
                f[n + lane] = (uint32_t)ucnt[j];
            }
            n += (uint32_t)min(32ull, G.ov_end - j0);
        }
    }
    if (NT > 32) {  // n from warp 0
        if (threadIdx.x == 0) s_n = n;
        __syncthreads();
        n = s_n;
    }
    __syncwarp();
    if (n == 0) {
        if (threadIdx.x == 0) gi[tb] = G;
        return;
    }
    // stable order by (frequency, insertion order): bitonic sort of f<<24|index
    uint32_t np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x)
        s_keys[i] = i < n ? (((unsigned long long)f[i] << 24) | i) : ~0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= np2; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    unsigned long long a = s_keys[i], c = s_keys[ixj];
                    bool up = (i & k) == 0;
                    if ((a > c) == up) {
                        s_keys[i] = c;
                        s_keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) perm[r] = (uint32_t)(s_keys[r] & 0xffffffu);
    if (NT > 32) {  // the rest is warp 0's
        __syncthreads();
        if (threadIdx.x >= 32) return;
    }
    {  // symbols in the group's stream (warp reduction)
        unsigned long long ns = 0;
        for (uint32_t i = lane; i < n; i += 32) ns += f[i];
        for (int o = 16; o > 0; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        G.nsyms = ns;
    }
    __syncwarp();
    uint32_t made = n;
    if (threadIdx.x == 0 && n > 1) {
        // two queues == the reference's priority queue on (f, order): a serial chain.
        // Leaves come in sorted-key order (frequency in the key's high bits, index in
        // the low 24); a leaf always precedes an internal node of equal weight (its
        // insertion index is smaller), so the queue compare is fl <= internal weight.
        // Both queue fronts stay in registers (the next leaf key; the oldest unmerged
        // internal weight f2), so the chain per merge is compares and selects; the
        // loads that refill them do not depend on the node being built (the internal
        // queue's next weight was written merges ago, except when the queue empties).
        uint32_t q1 = 0, q2 = n;
        unsigned long long k1 = s_keys[0];
        uint32_t f2 = 0;  // nodef[q2] when q2 < made
        auto take = [&](uint32_t& idx) -> uint32_t {
            const uint32_t fl = (uint32_t)(k1 >> 24);
            if (q1 < n && (q2 >= made || fl <= f2)) {
                idx = (uint32_t)(k1 & 0xffffffu);
                if (++q1 < n) k1 = s_keys[q1];
                return fl;
            }
            idx = q2;
            const uint32_t f = f2;
            if (++q2 < made) f2 = nodef[q2];
            return f;
        };
        for (uint32_t st = 0; st + 1 < n; ++st) {
            uint32_t x, y;
            const uint32_t fx = take(x), fy = take(y);
            const uint32_t w = fx + fy;
            nodef[made] = w;
            if (q2 == made) f2 = w;  // the internal queue was empty: its new front
            parent[x] = parent[y] = made;
            ++made;
        }
    }
    made = __shfl_sync(0xffffffffu, made, 0);
    __syncwarp();
    // leaf depths by pointer jumping (6 rounds reach every depth <= 64; deeper leaves
    // are a code-length overflow): ancestors in parent/nodef, distances in depth/s_keys
    bool overflow = false;
    if (n == 1) {
        if (lane == 0) depth[0] = 1;
    } else {
        const uint32_t root = made - 1;
        uint32_t* anc[2] = {parent, nodef};
        uint8_t* dist[2] = {depth, (uint8_t*)s_keys};
        for (uint32_t i = lane; i < made; i += 32) {
            if (i == root) parent[i] = root;
            depth[i] = i == root ? 0 : 1;
        }
        __syncwarp();
        int cur = 0;
        for (int round = 0; round < 6; ++round) {
            const uint32_t* ac = anc[cur];
            const uint8_t* dc = dist[cur];
            uint32_t* an = anc[cur ^ 1];
            uint8_t* dn = dist[cur ^ 1];
            for (uint32_t i = lane; i < made; i += 32) {
                const uint32_t a = ac[i];
                const uint32_t d = (uint32_t)dc[i] + dc[a];
                dn[i] = (uint8_t)(d < 255u ? d : 255u);
                an[i] = ac[a];
            }
            __syncwarp();
            cur ^= 1;
        }
        // cur == 0 after an even number of rounds: results are in parent/depth
        for (uint32_t i = lane; i < n; i += 32)
            if (anc[cur][i] != root || dist[cur][i] >= 64) overflow = true;
    }
    if (__any_sync(0xffffffffu, overflow) && lane == 0) atomicOr(A.err, kErrHuffmanDepth);
    __syncwarp();
    // table sorted by (len, sym): counting sort over lengths, stable in sym order
    uint32_t* hist = s_hist;
    uint32_t* at = s_at;
    __shared__ unsigned long long s_first[65];
    for (int l = lane; l < 65; l += 32) hist[l] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) atomicAdd(&hist[depth[i] < 64 ? depth[i] : 64], 1u);
    __syncwarp();
    if (lane == 0) {
        // canonical first code per length (codec.cpp:184-214): the o-th entry in
        // (len, sym) order gets first[len] + (o - start[len])
        uint32_t acc = 0;
        unsigned long long code = 0;
        int prev = -1;
        for (int l = 0; l < 65; ++l) {
            at[l] = acc;
            if (hist[l]) {
                if (prev >= 0) code <<= (l - prev);
                s_first[l] = code;
                code += hist[l];
                prev = l;
            }
            acc += hist[l];
        }
    }
    __syncwarp();
    // stable placement by length, 32 symbols at a time: lanes of equal length take
    // consecutive slots in lane (= symbol) order
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const uint32_t d = i < n ? (depth[i] < 64 ? depth[i] : 64u) : 65u;
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t base = 0;
        if (lane == leader && d < 65) base = at[d];
        base = __shfl_sync(0xffffffffu, base, leader);
        if (d < 65) perm[base + __popc(peers & ((1u << lane) - 1u))] = i;
        __syncwarp();
        if (lane == leader && d < 65) at[d] = base + __popc(peers);
        __syncwarp();
    }
    if (lane == 0) {
        uint32_t acc = 0;
        for (int l = 0; l < 65; ++l) {  // starts again
            at[l] = acc;
            acc += hist[l];
        }
    }
    __syncwarp();
    uint32_t hdr = 0;
    for (uint32_t o = lane; o < n; o += 32) {
        const uint32_t i = perm[o];
        const uint32_t len = depth[i];
        const uint32_t lc = len < 64 ? len : 64;
        const unsigned long long code = s_first[lc] + (o - at[lc]);
        tab_sym[G.tab_base + o] = sym[i];
        tab_len[G.tab_base + o] = (uint8_t)len;
        hdr += uvlen(zigzag(sym[i])) + 1;
        const long long sv = (long long)sym[i];
        if (sv <= 0) {
            code_dense[(size_t)tb * NS + (uint32_t)(-sv)] = code;
            len_dense[(size_t)tb * NS + (uint32_t)(-sv)] = (uint8_t)len;
        } else if (sv < kLD) {
            code_dense[(size_t)tb * NS + B + (uint32_t)sv] = code;
            len_dense[(size_t)tb * NS + B + (uint32_t)sv] = (uint8_t)len;
        } else {
            // overflow leaves were appended last, in ukey order: leaf i <-> ov_begin + i - n_dense
            const unsigned long long j = G.ov_begin + (i - (n - nov));
            code_ov[j] = code;
            len_ov[j] = (uint8_t)len;
            // hash slot for the emission's lookup: (length, local index), linear probing
            // in 2 nov slots (lengths >= kLD, so 0 marks an empty slot)
            unsigned long long* H = W.ovh + 2 * G.ov_begin;
            const uint32_t m = 2 * nov;
            uint32_t h = (uint32_t)(((unsigned long long)(uint32_t)sv * 2654435761ull) % m);
            const unsigned long long ent = ((unsigned long long)(uint32_t)sv << 32) | (uint32_t)(j - G.ov_begin);
            while (atomicCAS(H + h, 0ull, ent) != 0ull) h = h + 1 == m ? 0 : h + 1;
        }
    }
    for (int o = 16; o > 0; o >>= 1) hdr += __shfl_xor_sync(0xffffffffu, hdr, o);
    if (lane == 0) {
        G.tsize = n;
        G.hdr = hdr + uvlen(b) + uvlen(G.n_elems) + uvlen(G.nsyms) + uvlen(n);
        gi[tb] = G;
    }
}

// ---- symbol walk shared by E2a / E2b ---------------------------------------------
struct CodeTabs {
    const unsigned long long* ovh;  // overflow-length hash (enc_huffman_kernel)
    const unsigned long long* code_dense;
    const uint8_t* len_dense;
    const unsigned long long* ukey;
    const unsigned long long* code_ov;
    const uint8_t* len_ov;
    const GroupInfo* gi;
};

__device__ __forceinline__ void code_of(const CodeTabs& C, uint32_t tb, uint32_t NS, uint32_t slot,
                                        unsigned long long& code, uint32_t& len) {
    code = C.code_dense[(size_t)tb * NS + slot];
    len = C.len_dense[(size_t)tb * NS + slot];
}

__device__ __forceinline__ void code_of_len(const CodeTabs& C, uint32_t tb, uint32_t NS,
                                            uint32_t B, unsigned long long L,
                                            unsigned long long& code, uint32_t& len) {
    if (L < (unsigned long long)kLD) {
        code_of(C, tb, NS, B + (uint32_t)L, code, len);
    } else {
        const GroupInfo& G = C.gi[tb];
        const unsigned long long* H = C.ovh + 2 * G.ov_begin;
        const uint32_t m = 2 * (uint32_t)(G.ov_end - G.ov_begin);
        uint32_t h = (uint32_t)((L * 2654435761ull) % m);
        unsigned long long ent;
        while (((ent = H[h]) >> 32) != L) h = h + 1 == m ? 0 : h + 1;  // present by construction
        const unsigned long long j = G.ov_begin + (uint32_t)ent;
        code = C.code_ov[j];
        len = C.len_ov[j];
    }
}

// Owned (value, length) of run r of the tile, or L = 0 when the run continues an
// earlier one.
__device__ __forceinline__ void owned_run(const EncArgs& A, const Seg* segs, unsigned long long rw,
                                          uint32_t r, uint32_t& v, uint32_t& b,
                                          unsigned long long& L) {
    v = (uint32_t)(rw & 0xffff);
    b = (uint32_t)((rw >> 16) & 0xffff);
    L = rw >> 32;
    const Seg& S = segs[b];
    if (r == S.run_begin) {
        if (S.cont) {
            L = 0;
            return;
        }
        if (S.run_end == S.run_begin + 1) L = S.lead_total;
    } else if (r + 1 == S.run_end) {
        L = S.trail_total;
    }
}

// E2a: bits per (tile, group), one warp per tile
// Resolved codes per run (enc_bits_kernel -> enc_emit_kernel): the run's value code
// and length code concatenated, its group and its bit count, so the emission reads one
// word per run instead of the segment, two code tables and -- for long runs -- a
// binary search in the group's overflow-length list.  Bit counts above kRcMaxBits are
// marked kRcSlow and resolved again by the emission.
constexpr uint32_t kRcMaxBits = 49, kRcSlow = 127;
__device__ __forceinline__ unsigned long long rc_pack(unsigned long long code, uint32_t b, uint32_t bits) {
    return bits > kRcMaxBits ? (unsigned long long)kRcSlow : (code << 15) | ((unsigned long long)b << 7) | bits;
}

template <int KB>
__global__ void __launch_bounds__(256) enc_bits_kernel(EncArgs A, CodeTabs C, int ntiles,
                                                       uint32_t* segbits, unsigned long long* rc) {
    __shared__ uint32_t s_bits[8][KB];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ti = blockIdx.x * 8 + wid;
    if (ti >= ntiles) return;
    const uint32_t B = A.B, NS = A.NS;
    const Tile T = A.tiles[ti];
    for (uint32_t b = lane; b < B; b += 32) s_bits[wid][b] = 0;
    __syncwarp();
    const uint32_t R = A.tile_nruns[ti];
    const Seg* segs = A.segs + (size_t)ti * B;
    const unsigned long long* runs = A.runs + (size_t)ti * kTile;
    unsigned long long* rct = rc + (size_t)ti * kTile;
    // four runs per lane in flight: their words, segments and code-table loads are
    // issued together before any result is stored
    constexpr int kU = 4;
    for (uint32_t r0 = lane; r0 < R; r0 += 32 * kU) {
        unsigned long long rw[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t r = r0 + 32 * u;
            rw[u] = r < R ? runs[r] : 0ull;
        }
        uint32_t v[kU], b[kU];
        unsigned long long L[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t r = r0 + 32 * u;
            if (r < R) owned_run(A, segs, rw[u], r, v[u], b[u], L[u]);
            else v[u] = b[u] = 0, L[u] = 0;
        }
        unsigned long long out[kU];
        uint32_t bits[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            out[u] = 0;
            bits[u] = 0;
            if (!L[u]) continue;
            const uint32_t tb = T.tensor * B + b[u];
            unsigned long long c1, c2 = 0;
            uint32_t l1, l2 = 0;
            code_of(C, tb, NS, v[u], c1, l1);
            if (L[u] > 1) code_of_len(C, tb, NS, B, L[u], c2, l2);
            out[u] = rc_pack(l2 ? (c1 << l2) | c2 : c1, b[u], l1 + l2);
            bits[u] = l1 + l2;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint32_t r = r0 + 32 * u;
            if (r >= R) break;
            rct[r] = out[u];
            if (bits[u]) atomicAdd(&s_bits[wid][b[u]], bits[u]);
        }
    }
    __syncwarp();
    for (uint32_t b = lane; b < B; b += 32) segbits[(size_t)ti * B + b] = s_bits[wid][b];
}

// S2: exclusive scan of segment bits across the tensor's tiles
__global__ void __launch_bounds__(kCB) enc_bitscan_kernel(EncArgs A, const uint32_t* segbits,
                                                          unsigned long long* segoff, GroupInfo* gi) {
    __shared__ unsigned long long s_scan[33];
    const uint32_t B = A.B;
    const uint32_t t = blockIdx.x / B, b = blockIdx.x % B;
    const uint32_t a0 = A.tile0[t], a1 = A.tile0[t + 1];
    // four consecutive tiles per thread: a quarter of the block scans (and barriers)
    // on the long tile ranges of the large tensors
    constexpr int kPer = 4;
    unsigned long long base = 0;
    for (uint32_t c0 = a0; c0 < a1; c0 += kCB * kPer) {
        const uint32_t i0 = c0 + threadIdx.x * kPer;
        uint32_t v[kPer];
        unsigned long long sum = 0, tot;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            v[u] = i0 + u < a1 ? segbits[(size_t)(i0 + u) * B + b] : 0u;
            sum += v[u];
        }
        unsigned long long ex = block_exclusive_scan<unsigned long long>(sum, s_scan, &tot);
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            if (i0 + u < a1) segoff[(size_t)(i0 + u) * B + b] = base + ex;
            ex += v[u];
        }
        base += tot;
    }
    if (threadIdx.x == 0) {
        GroupInfo& G = gi[blockIdx.x];
        G.bits = base;
        G.nbytes = (base + 7) / 8;
        G.gbytes = G.n_elems ? G.hdr + uvlen(G.nbytes) + G.nbytes : 0;
    }
}

// ---- record layout ---------------------------------------------------------------
struct TensorRec {
    unsigned long long static_off, static_len;  // in the host-built static blob
    unsigned long long prot_begin, prot_end;    // protected entry range
    unsigned long long size, off;               // record bytes / offset
    uint32_t ngroups, pad;
    unsigned long long payload;                 // encode_tensor_payload bytes (or ablation size)
};

__device__ __forceinline__ uint32_t tensor_of_entry(const TensorRec* tr, uint32_t nt,
                                                    unsigned long long i) {
    uint32_t lo = 0, hi = nt;  // last tensor with prot_begin <= i
    while (hi - lo > 1) {
        uint32_t m = (lo + hi) >> 1;
        if (tr[m].prot_begin <= i) lo = m;
        else hi = m;
    }
    while (lo + 1 < nt && tr[lo].prot_end <= i) ++lo;
    return lo;
}

__global__ void prot_sizes_kernel(const TensorRec* tr, uint32_t nt, unsigned long long np,
                                  const uint64_t* ppos, unsigned long long* sizes) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < np;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const TensorRec& R = tr[tensor_of_entry(tr, nt, i)];
        unsigned long long d = i == R.prot_begin ? ppos[i] : ppos[i] - ppos[i - 1];
        sizes[i] = uvlen(d) + 2;
    }
}

// protected entries of every tensor: uvarint position delta + u16 bf16
__global__ void write_prot_kernel(const TensorRec* tr, uint32_t nt, unsigned long long np,
                                  const uint64_t* ppos, const uint16_t* pval,
                                  const unsigned long long* prot_scan, uint8_t* rec) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < np;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const TensorRec& R = tr[tensor_of_entry(tr, nt, i)];
        const unsigned long long np_t = R.prot_end - R.prot_begin;
        uint8_t* q = rec + R.off + R.static_len + uvlen(np_t) + (prot_scan[i] - prot_scan[R.prot_begin]);
        unsigned long long d = i == R.prot_begin ? ppos[i] : ppos[i] - ppos[i - 1];
        uint32_t k = put_uv(q, d);
        q[k] = (uint8_t)(pval[i] & 0xff);
        q[k + 1] = (uint8_t)(pval[i] >> 8);
    }
}

__global__ void tensor_size_kernel(EncArgs A, TensorRec* tr, const unsigned long long* prot_scan,
                                   GroupInfo* gi) {
    if (threadIdx.x) return;
    const uint32_t t = blockIdx.x, B = A.B;
    TensorRec& R = tr[t];
    unsigned long long s = R.static_len;
    const unsigned long long np = R.prot_end - R.prot_begin;
    s += uvlen(np) + (prot_scan[R.prot_end] - prot_scan[R.prot_begin]);
    uint32_t ng = 0;
    unsigned long long gs = 0;
    for (uint32_t b = 0; b < B; ++b) {
        const GroupInfo& G = gi[t * B + b];
        if (!G.n_elems) continue;
        ++ng;
        gs += G.gbytes;
    }
    R.ngroups = ng;
    R.size = s + uvlen(ng) + gs;
    if (A.mode == 0) {
        R.payload = uvlen(ng) + gs;  // encode_tensor_payload (codec.cpp:308-327)
    } else {  // huffman_payload_size (codec.cpp:601-613) of the single group
        const GroupInfo& G = gi[t * B];
        R.payload = ng ? gs - 1 - uvlen(G.n_elems) : 3;  // minus uv(bucket 0), uv(n)
    }
}

__global__ void tensor_scan_kernel(TensorRec* tr, uint32_t nt, unsigned long long prefix,
                                   unsigned long long* total) {
    if (threadIdx.x || blockIdx.x) return;
    unsigned long long o = prefix;
    for (uint32_t t = 0; t < nt; ++t) {
        tr[t].off = o;
        o += tr[t].size;
    }
    *total = o + 4;
}

// W: per tensor CTA: static prefix, protected entries, group headers + tables.
template <int KB>
__global__ void __launch_bounds__(kCB) write_tensor_kernel(
    EncArgs A, const TensorRec* tr, const uint8_t* statics, const uint64_t* ppos,
    const uint16_t* pval, const unsigned long long* prot_scan, GroupInfo* gi,
    const long long* tab_sym, const uint8_t* tab_len, uint8_t* rec) {
    __shared__ uint32_t s_pre[kCB / 32];
    const uint32_t t = blockIdx.x, B = A.B;
    const TensorRec R = tr[t];
    uint8_t* p = rec + R.off;
    for (unsigned long long i = threadIdx.x; i < R.static_len; i += kCB)
        p[i] = statics[R.static_off + i];
    unsigned long long o = R.static_len;
    const unsigned long long np = R.prot_end - R.prot_begin;
    if (threadIdx.x == 0) put_uv(p + o, np);
    o += uvlen(np);
    o += prot_scan[R.prot_end] - prot_scan[R.prot_begin];  // entries: write_prot_kernel
    if (threadIdx.x == 0) put_uv(p + o, R.ngroups);
    o += uvlen(R.ngroups);
    // group offsets in ascending bucket order (codec.cpp:312-326)
    __shared__ unsigned long long s_goff[KB];
    if (threadIdx.x == 0) {
        unsigned long long g = o;
        for (uint32_t b = 0; b < B; ++b) {
            s_goff[b] = g;
            g += gi[t * B + b].gbytes;
        }
    }
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t b = wid; b < B; b += kCB / 32) {
        GroupInfo& G = gi[t * B + b];
        if (!G.n_elems) continue;
        uint8_t* q = p + s_goff[b];
        if (lane == 0) {
            uint32_t k = put_uv(q, b);
            k += put_uv(q + k, G.n_elems);
            k += put_uv(q + k, G.nsyms);
            k += put_uv(q + k, G.tsize);
            s_pre[wid] = k;
        }
        __syncwarp();
        uint32_t k = s_pre[wid];
        // table entries: sequential varints; one lane per entry with a warp scan of sizes
        for (uint32_t e0 = 0; e0 < G.tsize; e0 += 32) {
            const uint32_t e = e0 + lane;
            uint32_t sz = 0;
            unsigned long long zz = 0;
            if (e < G.tsize) {
                zz = zigzag(tab_sym[G.tab_base + e]);
                sz = uvlen(zz) + 1;
            }
            uint32_t x = sz;
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            if (e < G.tsize) {
                uint8_t* w = q + k + x - sz;
                uint32_t m = put_uv(w, zz);
                w[m] = tab_len[G.tab_base + e];
            }
            k += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) {
            k += put_uv(q + k, G.nbytes);
            G.pay = (unsigned long long)(q + k - rec);
        }
        __syncwarp();
    }
}

// E2b: emission, MSB-first, atomicOr into the zeroed record
__device__ __forceinline__ void put_bits(uint32_t* words, unsigned long long q,
                                         unsigned long long code, int len) {
    while (len > 0) {
        const unsigned long long byte = q >> 3;
        const int bo = (int)(q & 7), avail = 8 - bo, take = avail < len ? avail : len;
        const uint32_t bits = (uint32_t)((code >> (len - take)) & ((1ull << take) - 1));
        const uint32_t bv = bits << (avail - take);
        atomicOr(words + (byte >> 2), bv << (8 * (uint32_t)(byte & 3)));
        len -= take;
        q += take;
    }
}

// E2b: emission.  Each (tile, group) segment owns a contiguous bit range of its
// group's stream.  Codes are first packed MSB-first into shared-memory words
// laid out with the destination's bit phase, then copied out as whole 32-bit
// words: interior words with plain stores, the two boundary words with
// atomicOr (they may share bytes with neighbouring segments or headers).
constexpr int kEmitWarps = 8;
constexpr int kWarpStage = 512;  // staged 32-bit words per warp (2 KiB; larger tiles write directly)

__device__ __forceinline__ void stage_bits(uint32_t* st, unsigned long long q,
                                           unsigned long long code, int len) {
    while (len > 0) {
        const uint32_t w = (uint32_t)(q >> 5), off = (uint32_t)(q & 31);
        const int take = (int)min(32u - off, (uint32_t)len);
        const uint32_t piece = (uint32_t)((code >> (len - take)) & ((1ull << take) - 1));
        atomicOr(st + w, piece << (32 - off - take));
        q += take;
        len -= take;
    }
}

// bits of run r (0 when it continues an earlier run)
__device__ __forceinline__ uint32_t run_bits(const EncArgs& A, const CodeTabs& C, const Seg* segs,
                                             const unsigned long long* runs, uint32_t tensor,
                                             uint32_t r, uint32_t& b_out) {
    uint32_t v, b;
    unsigned long long L;
    owned_run(A, segs, runs[r], r, v, b, L);
    b_out = b;
    if (!L) return 0;
    const uint32_t tb = tensor * A.B + b;
    unsigned long long c;
    uint32_t l1, l2 = 0;
    code_of(C, tb, A.NS, v, c, l1);
    if (L > 1) code_of_len(C, tb, A.NS, A.B, L, c, l2);
    return l1 + l2;
}

// E2b: emission, one warp per tile, warp-synchronous.  Each (tile, group)
// segment owns a contiguous bit range of its group's stream; codes are packed
// MSB-first into per-warp shared words laid out at the destination's bit phase,
// then copied out as whole 32-bit words (the two boundary words with atomicOr,
// since they can share bytes with neighbouring segments or headers).
template <int KB, int EW = (KB > kMaxB ? 2 : kEmitWarps)>
__global__ void __launch_bounds__(EW * 32) enc_emit_kernel(EncArgs A, CodeTabs C,
                                                                   const unsigned long long* segoff,
                                                                   const uint32_t* segbits,
                                                                   const unsigned long long* rc,
                                                                   int ntiles, uint8_t* rec) {
    __shared__ uint32_t s_stage[EW][kWarpStage];
    __shared__ uint32_t s_segbits[EW][KB];
    __shared__ uint32_t s_segstart[EW][KB + 1];
    __shared__ uint32_t s_sw[EW][KB + 1];
    __shared__ uint32_t s_phase[EW][KB];
    __shared__ unsigned long long s_dw[EW][KB];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ti = blockIdx.x * EW + wid;
    if (ti >= ntiles) return;
    const uint32_t B = A.B, NS = A.NS;
    const Tile T = A.tiles[ti];
    const uint32_t R = A.tile_nruns[ti];
    const Seg* segs = A.segs + (size_t)ti * B;
    const unsigned long long* runs = A.runs + (size_t)ti * kTile;
    uint32_t* words = (uint32_t*)rec;
    uint32_t* stage = s_stage[wid];
    // bits per segment (enc_bits_kernel)
    for (uint32_t b = lane; b < B; b += 32) s_segbits[wid][b] = segbits[(size_t)ti * B + b];
    __syncwarp();
    // segment layout: tile-local start, destination word + phase, staging base
    uint32_t tile_base = 0, stage_base = 0;
    for (uint32_t b0 = 0; b0 < B; b0 += 32) {
        const uint32_t b = b0 + lane;
        uint32_t bits = 0, nw = 0;
        if (b < B) {
            bits = s_segbits[wid][b];
            unsigned long long dest = 0;
            if (bits) dest = C.gi[T.tensor * B + b].pay * 8 + segoff[(size_t)ti * B + b];
            s_phase[wid][b] = (uint32_t)(dest & 31);
            s_dw[wid][b] = dest >> 5;
            nw = bits ? ((uint32_t)(dest & 31) + bits + 31) / 32 : 0u;
        }
        uint32_t xb = bits, xw = nw;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t yb = __shfl_up_sync(0xffffffffu, xb, o), yw = __shfl_up_sync(0xffffffffu, xw, o);
            if (lane >= o) xb += yb, xw += yw;
        }
        if (b < B) {
            s_segstart[wid][b] = tile_base + xb - bits;
            s_sw[wid][b] = stage_base + xw - nw;
        }
        tile_base += __shfl_sync(0xffffffffu, xb, 31);
        stage_base += __shfl_sync(0xffffffffu, xw, 31);
    }
    if (lane == 0) s_sw[wid][B] = stage_base;
    const bool staged = stage_base <= (uint32_t)kWarpStage;
    if (staged)
        for (uint32_t i = lane; i < stage_base; i += 32) stage[i] = 0;
    __syncwarp();
    // pass 2: place codes; a warp scan over each 32-run chunk gives tile offsets
    uint32_t running = 0;
    const unsigned long long* rct = rc + (size_t)ti * kTile;
    unsigned long long wn = lane < R ? rct[lane] : 0ull;  // the next chunk's word, in flight
    for (uint32_t r0 = 0; r0 < R; r0 += 32) {
        const uint32_t r = r0 + lane;
        uint32_t b = 0, l1 = 0, l2 = 0;
        unsigned long long c1 = 0, c2 = 0;
        const unsigned long long w = wn;
        wn = r + 32 < R ? rct[r + 32] : 0ull;
        if ((w & 127) != kRcSlow) {  // resolved by enc_bits_kernel: one code of l1 bits
            l1 = (uint32_t)(w & 127);
            b = (uint32_t)((w >> 7) & 0xff);
            c1 = w >> 15;
        } else {  // more than kRcMaxBits bits: resolve again
            uint32_t v = 0;
            unsigned long long L = 0;
            owned_run(A, segs, runs[r], r, v, b, L);
            const uint32_t tb = T.tensor * B + b;
            code_of(C, tb, NS, v, c1, l1);
            if (L > 1) code_of_len(C, tb, NS, B, L, c2, l2);
        }
        const uint32_t bits = l1 + l2;
        uint32_t x = bits;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        const uint32_t tile_off = running + x - bits;
        running += __shfl_sync(0xffffffffu, x, 31);
        if (bits) {
            const uint32_t local = tile_off - s_segstart[wid][b];
            if (staged) {
                unsigned long long q = (unsigned long long)s_sw[wid][b] * 32 + s_phase[wid][b] + local;
                stage_bits(stage, q, c1, (int)l1);
                if (l2) stage_bits(stage, q + l1, c2, (int)l2);
            } else {
                unsigned long long q = s_dw[wid][b] * 32 + s_phase[wid][b] + local;
                put_bits(words, q, c1, (int)l1);
                if (l2) put_bits(words, q + l1, c2, (int)l2);
            }
        }
    }
    if (!staged) return;
    __syncwarp();
    // pass 3: copy staged words (big-endian bit order -> little-endian words)
    uint32_t b = 0;
    for (uint32_t i = lane; i < stage_base; i += 32) {
        while (b + 1 < B && s_sw[wid][b + 1] <= i) ++b;
        const uint32_t j = i - s_sw[wid][b], nw = s_sw[wid][b + 1] - s_sw[wid][b];
        const uint32_t val = __byte_perm(stage[i], 0, 0x0123);
        uint32_t* dst = words + s_dw[wid][b] + j;
        if (j == 0 || j + 1 == nw) {
            if (val) atomicOr(dst, val);
        } else {
            *dst = val;
        }
    }
}

// x^(8 * level-stream bytes after tile t) mod P, once per layout
__global__ void crc_tile_shift_kernel(const Tile* tiles, int ntiles, const uint64_t* off,
                                      const uint64_t* stream_off, uint64_t N, uint32_t* out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles; t += gridDim.x * blockDim.x) {
        const Tile T = tiles[t];
        const uint64_t end = stream_off[T.tensor] + (T.start - off[T.tensor]) + T.count;
        out[t] = crc_x2nmodp(c_crc_x2n, 2 * (N - end), 3);
    }
}

__global__ void finish_crc_kernel(const uint32_t* acc, unsigned long long total_bytes,
                                  uint8_t* dst, uint32_t* crc_out) {
    if (threadIdx.x || blockIdx.x) return;
    uint32_t c = *acc ^ crc_shift(c_crc_x2n, 0xffffffffu, total_bytes) ^ 0xffffffffu;
    if (dst) {
        dst[0] = (uint8_t)c;
        dst[1] = (uint8_t)(c >> 8);
        dst[2] = (uint8_t)(c >> 16);
        dst[3] = (uint8_t)(c >> 24);
    }
    if (crc_out) *crc_out = c;
}

// ---- host ------------------------------------------------------------------------
static void put_le(std::vector<uint8_t>& v, uint64_t x, int n) {
    for (int i = 0; i < n; ++i) v.push_back((uint8_t)(x >> (8 * i)));
}
static void put_f64(std::vector<uint8_t>& v, double d) {
    uint64_t b;
    memcpy(&b, &d, 8);
    put_le(v, b, 8);
}

void group_elems(Engine& e, const void* segs, const Layout& L, uint32_t B,
                 unsigned long long* elems);

static std::once_flag crc_consts_once;
static void init_crc_consts_impl();
static void init_crc_consts() { std::call_once(crc_consts_once, init_crc_consts_impl); }
static void init_crc_consts_impl() {
    CrcX2N x = crc_x2n_table();
    uint32_t pw[kCB];
    for (int t = 0; t < kCB; ++t) pw[t] = crc_x2nmodp(x.t, (uint64_t)32 * (kCB - 1 - t), 3);
    DQTG_CUDA(cudaMemcpyToSymbol(c_crc_pw, pw, sizeof(pw)));
    // zero-skipping slice-by-16 tables T1,T3,...,T11,T12..T15 (T_n: byte then n zero bytes)
    static uint32_t tn[16][256];
    for (uint32_t b = 0; b < 256; ++b) {
        uint32_t c = b;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xedb88320u ^ (c >> 1) : c >> 1;
        tn[0][b] = c;
    }
    for (int n = 1; n < 16; ++n)
        for (uint32_t b = 0; b < 256; ++b) tn[n][b] = (tn[n - 1][b] >> 8) ^ tn[0][tn[n - 1][b] & 0xff];
    static const int pick[kCrcTabs] = {1, 3, 5, 7, 9, 11, 12, 13, 14, 15};
    static uint32_t sl[kCrcTabs][256];
    for (int i = 0; i < kCrcTabs; ++i) memcpy(sl[i], tn[pick[i]], sizeof(sl[i]));
    DQTG_CUDA(cudaMemcpyToSymbol(g_crc_slice, sl, sizeof(sl)));
    static uint32_t nib[kNibConsts][8][16];
    for (int lv = 0; lv < kNibConsts; ++lv) {
        const uint64_t m = lv < 8 ? (uint64_t)32 * (7 - lv)
                                  : (lv < 10 ? (uint64_t)256 << (lv - 8) : (uint64_t)1024 << (lv - 10));
        const uint32_t k = crc_x2nmodp(x.t, m, 3);
        for (int i = 0; i < 8; ++i)
            for (uint32_t n = 0; n < 16; ++n) nib[lv][i][n] = m ? crc_multmodp(k, n << (4 * i)) : (n << (4 * i));
    }
    DQTG_CUDA(cudaMemcpyToSymbol(g_crc_nib, nib, sizeof(nib)));
    DQTG_CUDA(cudaMemcpyToSymbol(c_crc_x2n, x.t, sizeof(x.t)));

}

std::unique_ptr<Record> encode_record(Engine& e, const QState* base, const QState& target,
                                      double quality) {
    return encode_record_ex(e, base, target, quality, 0, 0, nullptr, 0, nullptr);
}

bool fused_c_enabled() {  // read per step: tests toggle it inside one process
    return getenv("DQTG_NO_FUSED_C") == nullptr && getenv("DQTG_DENSE_DELTA") == nullptr;
}

std::unique_ptr<Record> compress_step(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                                      uint64_t seed, uint64_t step, const QState* base,
                                      double quality, std::unique_ptr<QState>& state_out,
                                      const std::function<void(QState*)>& on_levels) {
    // the fused encoder needs the sparse DELTA path with the byte codec: a base, and
    // an alphabet the shared-memory codec holds (checked again by encode_record_ex)
    const uint32_t kt = std::max(cfg.bins, cfg.embed_bins) + 2;
    bool fuse = base && fused_c_enabled() && std::max(base->max_levels(), kt) <= (uint32_t)kMaxB;
    FuseC fc;
    state_out = quantize(e, c, cfg, seed, step, fuse ? &fc : nullptr);
    QState* q = state_out.get();
    if (fuse && !fc.w) {  // nothing deferred (no elements): levels are already set
        fuse = false;
    }
    if (!fuse) {
        if (on_levels) on_levels(q);
        return encode_record(e, base, *q, quality);
    }
    return encode_record_ex(e, base, *q, quality, 0, 0, nullptr, 0, nullptr, &fc,
                            [&] { if (on_levels) on_levels(q); });
}

// B_override / nt_total: a shard of a tensor-sharded checkpoint encodes its tensor
// blocks with the global alphabet and writes the global tensor count, so the
// bytes [body_offset, size-4) of every rank concatenate into the single-GPU record.
std::unique_ptr<Record> encode_record_ex(Engine& e, const QState* base, const QState& target,
                                         double quality, uint32_t B_override, uint32_t nt_total,
                                         uint64_t* body_offset, int mode, uint64_t* payload_total,
                                         const FuseC* fc, const std::function<void()>& on_levels) {
    const Layout& L = *target.L;
    for (uint32_t i = 0; i < L.nt; ++i)  // 32-bit run lengths / symbol counts on the device
        DQTG_REQUIRE(L.numel[i] < (1ull << 31), DQTG_ERROR,
                     "tensor " + L.names[i] + " has 2^31 or more elements (device codec limit)");
    if (base) {
        const Layout& BL = *base->L;
        DQTG_REQUIRE(BL.nt == L.nt, DQTG_SHAPE_MISMATCH, "base/target tensor count mismatch");
        for (uint32_t i = 0; i < L.nt; ++i)
            if (BL.names[i] != L.names[i] || BL.dims[i] != L.dims[i] || BL.types[i] != L.types[i])
                throw Fail(DQTG_SHAPE_MISMATCH,
                           "base/target tensor layout mismatch at " + L.names[i]);
    }
    // codec.cpp:416-417
    uint32_t B = std::max(base ? base->max_levels() : 0u, target.max_levels());
    if (B == 0) B = 2;
    if (B_override) {
        DQTG_REQUIRE(B_override >= B, DQTG_ERROR, "alphabet override below the local alphabet");
        B = B_override;
    }
    DQTG_REQUIRE(B <= (uint32_t)kMaxBLarge, DQTG_ERROR,
                 "cyclic alphabet larger than the device codec supports (255 levels)");
    const bool large = B > (uint32_t)kMaxB;  // 8-bit keys, global frequencies, larger tails
    init_crc_consts();
    cudaStream_t st = e.stream;
    const uint32_t NS = B + kLD;
    const uint32_t nt = L.nt;
    const int ntiles = (int)L.tiles.size();

    // ---- host-built static bytes: record prefix + per-tensor prefixes (codec.cpp:419-446)
    std::vector<uint8_t> pre;
    pre.insert(pre.end(), {'D', 'Q', 'D', 'R'});
    put_le(pre, 1, 4);
    pre.push_back(base ? 1 : 0);
    put_le(pre, base ? base->step : 0, 8);
    put_le(pre, target.step, 8);
    put_le(pre, B, 4);
    const dqtg_config& c = target.cfg;
    put_le(pre, c.bins, 4);
    put_le(pre, c.embed_bins, 4);
    put_f64(pre, c.prune_frac);
    put_f64(pre, c.protect_frac);
    pre.push_back((uint8_t)c.metric);
    put_f64(pre, c.sigma);
    put_f64(pre, c.alpha);
    put_f64(pre, quality);
    uint8_t nlt = 0;
    for (int lt = 0; lt < kLayerTypes; ++lt) nlt += target.cb_len[lt] != 0;
    pre.push_back(nlt);
    for (int lt = 0; lt < kLayerTypes; ++lt) {
        if (!target.cb_len[lt]) continue;
        pre.push_back((uint8_t)lt);
        put_le(pre, target.cb_len[lt], 4);
        for (float v : target.cb[lt]) {
            uint32_t u;
            memcpy(&u, &v, 4);
            put_le(pre, u, 4);
        }
    }
    put_le(pre, nt_total ? nt_total : nt, 4);
    const uint64_t prefix_len = pre.size();
    if (body_offset) *body_offset = prefix_len;
    std::vector<TensorRec> trh(nt);
    std::vector<uint8_t> statics;
    for (uint32_t i = 0; i < nt; ++i) {
        trh[i].static_off = statics.size();
        put_le(statics, L.names[i].size(), 2);
        statics.insert(statics.end(), L.names[i].begin(), L.names[i].end());
        statics.push_back(L.types[i]);
        statics.push_back(L.ranks[i]);
        for (uint64_t d : L.dims[i]) put_le(statics, d, 8);
        trh[i].static_len = statics.size() - trh[i].static_off;
        trh[i].prot_begin = target.prot_off[i];
        trh[i].prot_end = target.prot_off[i + 1];
    }

    auto rec = std::make_unique<Record>();
    rec->eng = &e;
    if (nt == 0 && payload_total) {
        *payload_total = 0;
        return nullptr;
    }
    if (nt == 0) {
        // no tensors: prefix + CRC of the empty stream
        std::vector<uint8_t> host = pre;
        put_le(host, 0, 4);  // crc32 of nothing = 0
        rec->size = host.size();
        rec->d_buf = (uint8_t*)e.dalloc(host.size());
        DQTG_CUDA(cudaMemcpyAsync(rec->d_buf, host.data(), host.size(), cudaMemcpyHostToDevice,
                                  e.stream));
        e.sync();
        return rec;
    }

    // ---- device scratch
    if (!L.d_crc_shift) {
        Layout& ML = const_cast<Layout&>(L);
        DQTG_CUDA(cudaMalloc(&ML.d_crc_shift, (size_t)ntiles * 4 + 4));
        { DQTG_SPAN(e, "crc_tile_shift_kernel"); crc_tile_shift_kernel<<<(ntiles + 255) / 256, 256, 0, st>>>(L.d_tiles, ntiles, L.d_off, L.d_stream_off, L.N, ML.d_crc_shift); }
        e.launched();
    }
    EncArgs A{};
    A.crc_shift = L.d_crc_shift;
    A.tiles = L.d_tiles;
    A.types = L.d_types;
    A.off = L.d_off;
    A.stream_off = L.d_stream_off;
    A.tile0 = L.d_tile0;
    A.N = L.N;
    A.B = B;
    A.NS = NS;
    A.n_tb = nt * B;
    A.prev = base ? base->d_levels : nullptr;
    A.cur = target.d_levels;
    A.segs = (Seg*)e.buf("e.segs", (size_t)ntiles * B * sizeof(Seg) + 64);
    A.runs = (unsigned long long*)e.buf("e.runs", (size_t)ntiles * kTile * 8);
    A.tile_nruns = (uint32_t*)e.buf("e.nruns", (size_t)ntiles * 4 + 4);
    const size_t freq_n = (size_t)nt * B * NS;
    A.freq = (uint32_t*)e.buf("e.freq", freq_n * 4);
    A.ov_cap = L.N / kLD + (unsigned long long)ntiles * B * 2 + 16;
    A.ov = (unsigned long long*)e.buf("e.ov", A.ov_cap * 8);
    auto* small = (unsigned long long*)e.buf("e.small", 64);
    A.ov_count = small;
    A.crc_acc = (uint32_t*)(small + 1);
    A.tile_crc = (uint32_t*)e.buf("e.tile_crc", (size_t)ntiles * 4 + 4);
    A.tile_ctr = (unsigned int*)(small + 5);
    A.err = e.d_err;
    A.mode = (uint32_t)mode;
    DQTG_CUDA(cudaMemsetAsync(A.freq, 0, freq_n * 4, st));
    DQTG_CUDA(cudaMemsetAsync(small, 0, 64, st));

    // E1 (persistent CTAs)
    const size_t e1_smem = e1_smem_bytes(B, NS);
    A.ntiles = ntiles;
    {
        // ballot key width: keys < B, invalid elements 0xff -> 2^NB - 1 (> every key)
        // DELTA records: the sparse formulation (work on the non-zero deltas only);
        // FULL records (every delta non-zero) and the ablation modes: dense ranks
        const bool sparse = base && mode == 0 && !large && !getenv("DQTG_DENSE_DELTA");
        if (fc) {
            FuseC* m = const_cast<FuseC*>(fc);
            m->levels = target.d_levels;
            m->ppos = target.d_ppos;
            m->pval = target.d_pval;
        }
        DQTG_REQUIRE(!fc || sparse, DQTG_ERROR, "fused pass C needs the sparse DELTA encoder");
        void (*dfn)(EncArgs, FuseC) = fc ? enc_tile_delta_kernel<true> : enc_tile_delta_kernel<false>;
        auto kfn = sparse ? (void (*)(EncArgs))nullptr
                 : base ? (B <= 63 ? enc_tile_kernel<true, 6, kMaxB>
                           : B <= 64 ? enc_tile_kernel<true, 7, kMaxB>
                           : B <= 127 ? enc_tile_kernel<true, 7, kMaxBLarge> : enc_tile_kernel<true, 8, kMaxBLarge>)
                        : (B <= 63 ? enc_tile_kernel<false, 6, kMaxB>
                           : B <= 64 ? enc_tile_kernel<false, 7, kMaxB>
                           : B <= 127 ? enc_tile_kernel<false, 7, kMaxBLarge> : enc_tile_kernel<false, 8, kMaxBLarge>);
        const void* kptr = sparse ? (const void*)dfn : (const void*)kfn;
        const size_t smem = sparse ? dsm_bytes(B, NS) : e1_smem;
        ensure_dyn_smem(kptr, smem);
        DQTG_CUDA(cudaFuncSetAttribute(kptr, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        DQTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kptr, kCB, smem));
        const int grid = std::max(1, std::min(ntiles, e.num_sms * std::max(1, per_sm)));
        if (sparse) A.zs = (uint32_t*)e.buf("e.zs", (size_t)grid * kTile * 4);
        if (sparse) {
            FuseC F{};
            if (fc) F = *fc;
            { DQTG_SPAN(e, fc ? "quant_delta_kernel" : "enc_tile_delta_kernel"); dfn<<<grid, kCB, smem, st>>>(A, F); }
        } else {
            { DQTG_SPAN(e, "enc_tile_kernel"); kfn<<<grid, kCB, smem, st>>>(A); }
        }
        if (on_levels) on_levels();  // the target levels are complete after this point
        { DQTG_SPAN(e, "crc_tiles_kernel"); crc_tiles_kernel<<<std::max(1, std::min(e.num_sms * 2, (ntiles + 255) / 256)), 256, 0, st>>>(A.tile_crc, A.crc_shift, ntiles, A.crc_acc); }
        e.launched();
    }
    // S
    {
        // tensors with few tiles: a warp per (tensor, group); many tiles: a CTA
        std::vector<uint32_t> small, big;
        for (uint32_t t = 0; t < nt; ++t)
            (L.tile0[t + 1] - L.tile0[t] <= 64 ? small : big).push_back(t);
        auto* d_list = (uint32_t*)e.buf("e.tlist", (size_t)(nt + 2) * 4);
        std::vector<uint32_t> both(small);
        both.insert(both.end(), big.begin(), big.end());
        DQTG_CUDA(cudaMemcpyAsync(d_list, both.data(), both.size() * 4, cudaMemcpyHostToDevice, st));
        const uint32_t np_small = (uint32_t)small.size() * B;
        if (np_small) { DQTG_SPAN(e, "enc_resolve_kernel"); enc_resolve_kernel<<<(np_small + kResolveWarps - 1) / kResolveWarps, kResolveWarps * 32, kResolveWarps * NS * 4, st>>>(A, d_list, np_small); }
        if (!big.empty()) {
            std::vector<ResChunk> ch;
            for (uint32_t tt : big) {
                const uint32_t first = (uint32_t)ch.size();
                uint32_t k = 0;
                for (uint32_t c0 = L.tile0[tt]; c0 < L.tile0[tt + 1]; c0 += kResChunk, ++k)
                    ch.push_back(ResChunk{tt, c0, std::min(c0 + kResChunk, L.tile0[tt + 1]), k, first});
            }
            const uint32_t nch = (uint32_t)ch.size();
            auto* d_ch = (ResChunk*)e.buf("e.reschunks", nch * sizeof(ResChunk) + 16);
            auto* d_fl = (int*)e.buf("e.resfwd", (size_t)nch * B * 4 + 16);
            auto* d_ba = (RunM*)e.buf("e.resbwd", (size_t)nch * B * sizeof(RunM) + 16);
            DQTG_CUDA(cudaMemcpyAsync(d_ch, ch.data(), nch * sizeof(ResChunk), cudaMemcpyHostToDevice, st));
            DQTG_SPAN(e, "enc_resolve_big_kernel");
            enc_resolve_agg_kernel<<<nch * B, kCB, 0, st>>>(A, d_ch, d_fl, d_ba);
            enc_resolve_carry_kernel<<<(nch * B + 255) / 256, 256, 0, st>>>(d_ch, nch, B, d_fl, d_ba);
            enc_resolve_big_kernel<<<nch * B, kCB, NS * 4, st>>>(A, d_ch, d_fl, d_ba);
            e.launched(2);  // (a pageable source is staged before cudaMemcpyAsync returns)
        }
        e.launched(2);
    }
    e.launched(2);
    DQTG_CUDA(cudaGetLastError());
    // group element counts from the segments (host-free): sum of seg.n per (t,b)
    auto* elems = (unsigned long long*)e.buf("e.elems", (size_t)nt * B * 8);
    group_elems(e, A.segs, L, B, elems);

    // overflow run lengths: sort + unique
    unsigned long long n_ov = 0;
    e.d2h(&n_ov, A.ov_count, 8);
    e.sync();
    DQTG_REQUIRE(n_ov <= A.ov_cap, DQTG_ERROR, "run-length overflow list exhausted");
    // overflow buffers sized for the layout's bound (ov_cap), not this step's count:
    // the count varies step to step and every scratch growth maps pool memory mid-step
    const unsigned long long ov_cap = A.ov_cap;
    auto* ov_sorted = (unsigned long long*)e.buf("e.ov_sorted", ov_cap * 8 + 8);
    auto* ukey = (unsigned long long*)e.buf("e.ukey", ov_cap * 8 + 8);
    auto* ucnt = (unsigned long long*)e.buf("e.ucnt", ov_cap * 8 + 8);
    auto* nu = (unsigned long long*)(small + 2);
    if (n_ov) {
        size_t tb = 0, tb_cap = 0;
        DQTG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, A.ov, ov_sorted, (int64_t)n_ov, 0, 64,
                                                 st));
        DQTG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb_cap, A.ov, ov_sorted, (int64_t)ov_cap, 0,
                                                 64, st));
        void* tmp = e.buf("e.cubtmp", std::max(tb, tb_cap) + 16);
        DQTG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, A.ov, ov_sorted, (int64_t)n_ov, 0, 64, st));
        size_t tb2 = 0, tb2_cap = 0;
        DQTG_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb2, ov_sorted, ukey, ucnt, nu,
                                                     (int64_t)n_ov, st));
        DQTG_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, tb2_cap, ov_sorted, ukey, ucnt, nu,
                                                     (int64_t)ov_cap, st));
        void* tmp2 = e.buf("e.cubtmp3", std::max(tb2, tb2_cap) + 16);
        DQTG_CUDA(cub::DeviceRunLengthEncode::Encode(tmp2, tb2, ov_sorted, ukey, ucnt, nu,
                                                     (int64_t)n_ov, st));
    } else {
        DQTG_CUDA(cudaMemsetAsync(nu, 0, 8, st));
    }
    unsigned long long n_unique = 0;
    e.d2h(&n_unique, nu, 8);
    e.sync();
    // H
    auto* gi = (GroupInfo*)e.buf("e.gi", (size_t)nt * B * sizeof(GroupInfo));
    const size_t tab_n = (size_t)nt * B * NS + ov_cap + 8;  // bound, see above
    auto* tab_sym = (long long*)e.buf("e.tabsym", tab_n * 8);
    auto* tab_len = (uint8_t*)e.buf("e.tablen", tab_n);
    auto* code_dense = (unsigned long long*)e.buf("e.cdense", (size_t)nt * B * NS * 8);
    auto* len_dense = (uint8_t*)e.buf("e.ldense", (size_t)nt * B * NS);
    auto* code_ov = (unsigned long long*)e.buf("e.cov", ov_cap * 8 + 8);
    auto* ovh = (unsigned long long*)e.buf("e.ovhash", 2 * ov_cap * 8 + 16);
    if (n_unique) DQTG_CUDA(cudaMemsetAsync(ovh, 0, 2 * n_unique * 8, st));
    auto* len_ov = (uint8_t*)e.buf("e.lov", ov_cap + 8);
    {
        auto* max_nov = (uint32_t*)(small + 4);
        auto* ov_range = (unsigned long long*)e.buf("e.ovrange", (size_t)nt * B * 16 + 16);
        DQTG_CUDA(cudaMemsetAsync(max_nov, 0, 4, st));
        if (n_unique) {
            { DQTG_SPAN(e, "ov_group_max_kernel"); ov_group_max_kernel<<<(nt * B + 255) / 256, 256, 0, st>>>(ukey, nu, nt * B, max_nov, ov_range); }
            e.launched();
        } else {
            DQTG_CUDA(cudaMemsetAsync(ov_range, 0, (size_t)nt * B * 16, st));
        }
        // symbol-count bound per group -> tiers (see enc_huffman_kernel)
        const uint32_t ng = nt * B;
        std::vector<unsigned long long> h_rng((size_t)ng * 2), h_el(ng);
        e.d2h(h_rng.data(), ov_range, (size_t)ng * 16);
        e.d2h(h_el.data(), elems, (size_t)ng * 8);
        e.sync();
        std::vector<uint32_t> tiers[3];
        std::vector<unsigned long long> big_off;
        uint32_t np_mid = 1;
        unsigned long long big_bytes = 0;
        for (uint32_t g = 0; g < ng; ++g) {
            uint32_t np2 = 1;
            const unsigned long long bound = h_el[g] ? NS + (h_rng[2 * g + 1] - h_rng[2 * g]) : 1;
            while (np2 < bound) np2 <<= 1;
            if (np2 <= 128) {
                tiers[0].push_back(g);
            } else if (np2 <= 2048) {
                tiers[1].push_back(g);
                np_mid = std::max(np_mid, np2);
            } else {
                tiers[2].push_back(g);
                big_off.push_back(big_bytes);
                big_off.push_back(np2);
                big_bytes += round_up((unsigned long long)np2 * 38 + 16, 256);
            }
        }
        auto* d_gl = (uint32_t*)e.buf("h.glist", (size_t)ng * 4 + 16);
        auto* d_goff = (unsigned long long*)e.buf("h.goff", big_off.size() * 8 + 16);
        uint8_t* d_gws = big_bytes ? (uint8_t*)e.buf("h.gws", big_bytes) : nullptr;
        {
            std::vector<uint32_t> all;
            for (auto& v : tiers) all.insert(all.end(), v.begin(), v.end());
            DQTG_CUDA(cudaMemcpyAsync(d_gl, all.data(), all.size() * 4, cudaMemcpyHostToDevice, st));
            if (!big_off.empty())
                DQTG_CUDA(cudaMemcpyAsync(d_goff, big_off.data(), big_off.size() * 8,
                                          cudaMemcpyHostToDevice, st));
            e.sync();  // host vectors
        }
        HufWork W{};  // the working sets are per tier (shared memory or h.gws)
        W.ovh = ovh;
        DQTG_SPAN(e, "enc_huffman_kernel");
        const uint32_t* gl = d_gl;
        if (!tiers[0].empty()) {
            enc_huffman_kernel<false, 32><<<(unsigned)tiers[0].size(), 32, 128 * 38 + 16, st>>>(
                A, elems, ukey, ucnt, nu, gi, tab_sym, tab_len, code_dense, len_dense, code_ov, len_ov,
                W, 128, ov_range, gl, nullptr, nullptr);
            gl += tiers[0].size();
            e.launched();
        }
        if (!tiers[1].empty()) {
            const size_t hsm = (size_t)np_mid * 38 + 16;
            // the bitonic sort of a mid-size alphabet with 256 threads, then warp 0
            ensure_dyn_smem((const void*)enc_huffman_kernel<false, 256>, hsm);
            enc_huffman_kernel<false, 256><<<(unsigned)tiers[1].size(), 256, hsm, st>>>(
                A, elems, ukey, ucnt, nu, gi, tab_sym, tab_len, code_dense, len_dense, code_ov, len_ov,
                W, np_mid, ov_range, gl, nullptr, nullptr);
            gl += tiers[1].size();
            e.launched();
        }
        if (!tiers[2].empty()) {
            enc_huffman_kernel<true, 1024><<<(unsigned)tiers[2].size(), 1024, 0, st>>>(
                A, elems, ukey, ucnt, nu, gi, tab_sym, tab_len, code_dense, len_dense, code_ov, len_ov,
                W, 0, ov_range, gl, d_goff, d_gws);
            e.launched();
        }
    }
    CodeTabs C{ovh, code_dense, len_dense, ukey, code_ov, len_ov, gi};
    auto* segbits = (uint32_t*)e.buf("e.segbits32", (size_t)ntiles * B * 4 + 4);
    auto* rcodes = (unsigned long long*)e.buf("e.rcodes", (size_t)ntiles * kTile * 8);
    auto* segoff = (unsigned long long*)e.buf("e.segoff", (size_t)ntiles * B * 8);
    {
        DQTG_SPAN(e, "enc_bits_kernel");
        if (large) enc_bits_kernel<kMaxBLarge><<<(ntiles + 7) / 8, 256, 0, st>>>(A, C, ntiles, segbits, rcodes);
        else enc_bits_kernel<kMaxB><<<(ntiles + 7) / 8, 256, 0, st>>>(A, C, ntiles, segbits, rcodes);
    }
    { DQTG_SPAN(e, "enc_bitscan_kernel"); enc_bitscan_kernel<<<nt * B, kCB, 0, st>>>(A, segbits, segoff, gi); }
    e.launched(2);

    // protected entry sizes + layout
    const uint64_t np = target.prot_total;
    auto* psz = (unsigned long long*)e.buf("e.psz", (np + 1) * 8);
    auto* pscan = (unsigned long long*)e.buf("e.pscan", (np + 1) * 8);
    auto* tr = (TensorRec*)e.buf("e.tr", nt * sizeof(TensorRec));
    DQTG_CUDA(cudaMemcpyAsync(tr, trh.data(), nt * sizeof(TensorRec), cudaMemcpyHostToDevice, st));
    DQTG_CUDA(cudaMemsetAsync(psz, 0, (np + 1) * 8, st));
    const unsigned pgrid = (unsigned)std::min<uint64_t>((uint64_t)e.num_sms * 8, (np + 255) / 256 + 1);
    if (np) { DQTG_SPAN(e, "prot_sizes_kernel"); prot_sizes_kernel<<<pgrid, 256, 0, st>>>(tr, nt, np, target.d_ppos, psz); }
    {
        size_t tb = 0;
        DQTG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, psz, pscan, (int64_t)(np + 1), st));
        void* tmp = e.buf("e.cubtmp2", tb + 16);
        DQTG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, psz, pscan, (int64_t)(np + 1), st));
    }
    { DQTG_SPAN(e, "tensor_size_kernel"); tensor_size_kernel<<<nt, 32, 0, st>>>(A, tr, pscan, gi); }
    auto* total_d = (unsigned long long*)(small + 3);
    { DQTG_SPAN(e, "tensor_scan_kernel"); tensor_scan_kernel<<<1, 1, 0, st>>>(tr, nt, prefix_len, total_d); }
    e.launched(3);
    unsigned long long total = 0;
    e.d2h(&total, total_d, 8);
    if (payload_total) {  // sizes only (payload_bytes_*): no record is written
        std::vector<TensorRec> th(nt);
        e.d2h(th.data(), tr, nt * sizeof(TensorRec));
        e.check_err();
        *payload_total = 0;
        for (auto& r : th) *payload_total += r.payload;
        return nullptr;
    }
    e.check_err();  // syncs

    // ---- writers
    rec->size = total;
    rec->cap = round_up(total, 16) + 16;
    rec->d_buf = (uint8_t*)e.dalloc(rec->cap);
    DQTG_CUDA(cudaMemsetAsync(rec->d_buf, 0, rec->cap, st));
    DQTG_CUDA(cudaMemcpyAsync(rec->d_buf, pre.data(), pre.size(), cudaMemcpyHostToDevice, st));
    auto* d_statics = (uint8_t*)e.buf("e.statics", statics.size() + 8);
    DQTG_CUDA(cudaMemcpyAsync(d_statics, statics.data(), statics.size(), cudaMemcpyHostToDevice, st));
    { DQTG_SPAN(e, "write_tensor_kernel"); (large ? write_tensor_kernel<kMaxBLarge> : write_tensor_kernel<kMaxB>)<<<nt, kCB, 0, st>>>(A, tr, d_statics, target.d_ppos, target.d_pval, pscan,
                                            gi, tab_sym, tab_len, rec->d_buf); }
    if (np) { DQTG_SPAN(e, "write_prot_kernel"); write_prot_kernel<<<pgrid, 256, 0, st>>>(tr, nt, np, target.d_ppos, target.d_pval, pscan, rec->d_buf); }
    {
        DQTG_SPAN(e, "enc_emit_kernel");
        if (large) enc_emit_kernel<kMaxBLarge><<<(ntiles + 1) / 2, 2 * 32, 0, st>>>(A, C, segoff, segbits, rcodes, ntiles, rec->d_buf);
        else enc_emit_kernel<kMaxB><<<(ntiles + kEmitWarps - 1) / kEmitWarps, kEmitWarps * 32, 0, st>>>(A, C, segoff, segbits, rcodes, ntiles, rec->d_buf);
    }
    { DQTG_SPAN(e, "finish_crc_kernel"); finish_crc_kernel<<<1, 1, 0, st>>>(A.crc_acc, 2 * L.N, rec->d_buf + total - 4, nullptr); }
    e.launched(3);
    DQTG_CUDA(cudaGetLastError());
    e.check_err();
    // keep host copies of the staging buffers alive until the copies finished
    return rec;
}

__global__ void group_elems_kernel(const Seg* segs, const uint32_t* tile0, uint32_t B,
                                   unsigned long long* elems) {
    __shared__ unsigned long long s_scan[33];
    const uint32_t t = blockIdx.x / B, b = blockIdx.x % B;
    unsigned long long acc = 0;
    for (uint32_t i = tile0[t] + threadIdx.x; i < tile0[t + 1]; i += blockDim.x)
        acc += segs[(size_t)i * B + b].n;
    unsigned long long tot;
    block_exclusive_scan<unsigned long long>(acc, s_scan, &tot);
    if (threadIdx.x == 0) elems[blockIdx.x] = tot;
}

void group_elems(Engine& e, const void* segs, const Layout& L, uint32_t B,
                 unsigned long long* elems) {
    { DQTG_SPAN(e, "group_elems_kernel"); group_elems_kernel<<<L.nt * B, 256, 0, e.stream>>>((const Seg*)segs, L.d_tile0, B, elems); }
    e.launched();
}

// ---- crc32 over an arbitrary byte buffer (codec.cpp:275-288) ---------------------
__global__ void crc_bytes_kernel(const uint8_t* data, unsigned long long n, uint32_t* acc) {
    // each thread: 64 contiguous bytes; shift by the bytes that follow
    __shared__ uint32_t s_tab[256];
    {
        uint32_t c = threadIdx.x;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xedb88320u ^ (c >> 1) : c >> 1;
        s_tab[threadIdx.x] = c;
    }
    __syncthreads();
    const unsigned long long chunk = 64;
    for (unsigned long long s = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) * chunk;
         s < n; s += (unsigned long long)gridDim.x * blockDim.x * chunk) {
        unsigned long long e = s + chunk < n ? s + chunk : n;
        uint32_t r = 0;
        for (unsigned long long i = s; i < e; ++i) r = s_tab[(r ^ data[i]) & 0xff] ^ (r >> 8);
        r = crc_shift(c_crc_x2n, r, n - e);
        if (r) atomicXor(acc, r);
    }
}

uint32_t crc32_device(Engine& e, const uint8_t* data, uint64_t n) {
    init_crc_consts();
    auto* acc = (uint32_t*)e.buf("crc.acc", 16);
    auto* out = acc + 1;
    DQTG_CUDA(cudaMemsetAsync(acc, 0, 16, e.stream));
    if (n) { DQTG_SPAN(e, "crc_bytes_kernel"); crc_bytes_kernel<<<std::min<unsigned long long>(4096, (n + 16383) / 16384), 256, 0,
                              e.stream>>>(data, n, acc); }
    { DQTG_SPAN(e, "finish_crc_kernel"); finish_crc_kernel<<<1, 1, 0, e.stream>>>(acc, n, nullptr, out); }
    e.launched(2);
    uint32_t h = 0;
    e.d2h(&h, out, 4);
    e.sync();
    return h;
}


// Per-tile CRC shift constants of a layout, built once when the layout is made
// (a lazy cudaMalloc on the first encode synchronised the device mid-step).
void layout_crc_shift(Layout& L) {
    if (L.d_crc_shift || L.tiles.empty()) return;
    init_crc_consts();
    const int ntiles = (int)L.tiles.size();
    DQTG_CUDA(cudaMalloc(&L.d_crc_shift, (size_t)ntiles * 4 + 4));
    crc_tile_shift_kernel<<<(ntiles + 255) / 256, 256>>>(L.d_tiles, ntiles, L.d_off, L.d_stream_off, L.N,
                                                         L.d_crc_shift);
    DQTG_CUDA(cudaGetLastError());
    DQTG_CUDA(cudaStreamSynchronize(0));
}

static void ensure_crc_shift(Engine& e, const Layout& L) {
    if (L.d_crc_shift || L.tiles.empty()) return;
    Layout& ML = const_cast<Layout&>(L);
    const int ntiles = (int)L.tiles.size();
    DQTG_CUDA(cudaMalloc(&ML.d_crc_shift, (size_t)ntiles * 4 + 4));
    { DQTG_SPAN(e, "crc_tile_shift_kernel"); crc_tile_shift_kernel<<<(ntiles + 255) / 256, 256, 0, e.stream>>>(L.d_tiles, ntiles, L.d_off, L.d_stream_off, L.N, ML.d_crc_shift); }
    e.launched();
}

uint32_t level_stream_crc(Engine& e, const Layout& L, const uint16_t* levels) {
    init_crc_consts();
    cudaStream_t st = e.stream;
    const int ntiles = (int)L.tiles.size();
    auto* acc = (uint32_t*)e.buf("crc.acc", 16);
    DQTG_CUDA(cudaMemsetAsync(acc, 0, 4, st));
    if (ntiles) {
        ensure_crc_shift(e, L);
        auto* tc = (uint32_t*)e.buf("crc.tiles", (size_t)ntiles * 4 + 4);
        { DQTG_SPAN(e, "level_crc_tile_kernel"); level_crc_tile_kernel<<<ntiles, kCB, 0, st>>>(L.d_tiles, levels, tc); }
        { DQTG_SPAN(e, "crc_tiles_kernel"); crc_tiles_kernel<<<std::max(1, std::min(e.num_sms * 2, (ntiles + 255) / 256)), 256, 0, st>>>(tc, L.d_crc_shift, ntiles, acc); }
        e.launched(2);
    }
    { DQTG_SPAN(e, "finish_crc_kernel"); finish_crc_kernel<<<1, 1, 0, st>>>(acc, 2 * L.N, nullptr, acc + 1); }
    e.launched();
    uint32_t h = 0;
    e.d2h(&h, acc + 1, 4);
    e.sync();
    return h;
}

}  // namespace dqtg
