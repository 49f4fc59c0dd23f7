// quantize_checkpoint on the device (quantize.cpp:34-92, 373-425).
//
//   pass A  score histograms per layer type (magnitude / sensitivity), scores
//           derived in registers from w (+EMA) or read from explicit ScoreSets
//   quantile thresholds on device (sketch.cpp:59-77), float round-down (§7 H2)
//   pass B  partition + QUANTIZE-value histogram + protected counts per tile
//   keys    histogram -> ascending keys + mixed weights (quantize.cpp:263-279)
//   k-means 8 restarts per layer type (kmeans.cu)
//   pass C  partition + nearest-centre levels + protected (pos, bf16) compaction
#include <float.h>
#include <math.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include "engine.h"
#include "hist.cuh"
#include "kmeans_api.h"
#include "quantize_api.h"

namespace dqtg {

constexpr int kPB = 256;  // threads per streaming CTA
constexpr int kGrab = 8;  // tiles per dynamic grab of the persistent passes
constexpr int kPfDist = 148 * 5;  // pass C: about one wave of resident CTAs ahead

// L2 prefetch of one tile's score inputs (w + EMA, or the explicit scores)
__device__ __forceinline__ void prefetch_tile(const PassIn& a, int ti, bool expl) {
    const Tile T = a.tiles[ti];
    const uint32_t bytes = ((T.count + 3u) & ~3u) * 4u;
    prefetch_l2(a.w + T.start, bytes);
    if (expl) {
        prefetch_l2(a.mag + T.start, bytes);
        if (a.has_sens) prefetch_l2(a.sens + T.start, bytes);
    } else if (a.has_sens) {
        prefetch_l2(a.ema + T.start, bytes);
    }
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg((const float4*)p); }

__device__ __forceinline__ int classify(float mag, float sens, bool has_sens, int metric,
                                        const LtParams& p) {
    // quantize.cpp:82-87
    bool prot = (p.flags & kProtectAll) ||
                ((p.flags & kDoProtect) && (mag > p.t_mag || (has_sens && sens > p.t_sens)));
    if (prot) return 2;
    float ps = metric ? sens : mag;
    if ((p.flags & kDoPrune) && ps <= p.t_prune) return 1;
    return 0;
}

template <bool EXPL>
__device__ __forceinline__ void load_scores(const PassIn& a, uint64_t idx, const float4& w,
                                            float (&m)[4], float (&s)[4]) {
    if (EXPL) {
        float4 mv = ld4(a.mag + idx);
        m[0] = mv.x, m[1] = mv.y, m[2] = mv.z, m[3] = mv.w;
        if (a.has_sens) {
            float4 sv = ld4(a.sens + idx);
            s[0] = sv.x, s[1] = sv.y, s[2] = sv.z, s[3] = sv.w;
        }
    } else {
        m[0] = fabsf(w.x), m[1] = fabsf(w.y), m[2] = fabsf(w.z), m[3] = fabsf(w.w);
        if (a.has_sens) {  // ranker.cpp:96: fabs(e * w) in float
            float4 ev = ld4(a.ema + idx);
            s[0] = fabsf(__fmul_rn(ev.x, w.x)), s[1] = fabsf(__fmul_rn(ev.y, w.y));
            s[2] = fabsf(__fmul_rn(ev.z, w.z)), s[3] = fabsf(__fmul_rn(ev.w, w.w));
        }
    }
}

// ---- pass A: score histograms ----------------------------------------------
// Derived scores are non-negative: half-size windows (kPosSlots) per histogram.
template <bool EXPL>
__global__ void __launch_bounds__(kPB, 5) pass_a_kernel(PassIn a, unsigned long long* gh_mag,
                                                     unsigned long long* gh_sens,
                                                     uint32_t mask_mag, uint32_t mask_sens) {
    extern __shared__ uint32_t sh[];
    constexpr int W = EXPL ? kWinSlots : kPosSlots;
    uint32_t* shm = sh;
    uint32_t* shs = sh + W;
    uint32_t* s_ctab = sh + 2 * W;  // compact slot table (a.tab.ctab_n words)
    const bool fastc = a.tab.ctab != nullptr;
    for (int i = threadIdx.x; i < 2 * W; i += blockDim.x) sh[i] = 0;
    if (fastc) {
        for (uint32_t i = threadIdx.x; i < a.tab.ctab_n; i += blockDim.x) s_ctab[i] = __ldg(a.tab.ctab + i);
        if (threadIdx.x == 0) s_ctab[a.tab.ctab_n] = 0xc0000000u;  // sentinel: exact path
    }
    __syncthreads();
    const FastPos fp = fast_pos(a.tab, s_ctab);
    const uint32_t shm_s = (uint32_t)__cvta_generic_to_shared(shm);
    const uint32_t shs_s = (uint32_t)__cvta_generic_to_shared(shs);
    __shared__ int s_base;
    int cur = -1;
    auto flush = [&](int lt) {
        if (EXPL) {
            hist_flush(shm, gh_mag + lt * a.HS, a.tab);
            hist_flush(shs, gh_sens + lt * a.HS, a.tab);
        } else {
            hist_flush_pos(shm, gh_mag + lt * a.HS, a.tab);
            hist_flush_pos(shs, gh_sens + lt * a.HS, a.tab);
        }
    };
    for (int base; (base = grab_tiles(a.tile_ctr, kGrab, &s_base)) < a.ntiles;)
    for (int ti = base; ti < min(base + kGrab, a.ntiles); ++ti) {
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        if (threadIdx.x == 0 && ti + 1 < min(base + kGrab, a.ntiles)) prefetch_tile(a, ti + 1, EXPL);
        if (lt != cur) {
            __syncthreads();
            if (cur >= 0) flush(cur);
            __syncthreads();
            cur = lt;
        }
        const bool dm = (mask_mag >> lt) & 1, ds = (mask_sens >> lt) & 1;
        if (!dm && !ds) continue;
        unsigned long long* gm = gh_mag + lt * a.HS;
        unsigned long long* gs = gh_sens + lt * a.HS;
        // two float4 groups per iteration: twice the bytes in flight per thread
        for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 8) {
            const uint32_t i2 = i + kPB * 4;
            const bool two = i2 < T.count;
            float m[8], s[8];
            {
                float4 w0 = ld4(a.w + T.start + i);
                float4 w1 = two ? ld4(a.w + T.start + i2) : make_float4(0, 0, 0, 0);
                float mm[4], ss[4];
                load_scores<EXPL>(a, T.start + i, w0, mm, ss);
#pragma unroll
                for (int j = 0; j < 4; ++j) m[j] = mm[j], s[j] = ss[j];
                if (two) {
                    load_scores<EXPL>(a, T.start + i2, w1, mm, ss);
#pragma unroll
                    for (int j = 0; j < 4; ++j) m[4 + j] = mm[j], s[4 + j] = ss[j];
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t e = (j < 4 ? i : i2) + (j & 3);
                if (e >= T.count) continue;
                if (EXPL) {
                    if (fastc) {
                        if (dm) hist_add_s(shm, gm, m[j], a.tab, a.err, s_ctab);
                        if (ds) hist_add_s(shs, gs, s[j], a.tab, a.err, s_ctab);
                    } else {
                        if (dm) hist_add(shm, gm, m[j], a.tab, a.err);
                        if (ds) hist_add(shs, gs, s[j], a.tab, a.err);
                    }
                } else if (fastc) {  // branch-free table path; exact path for the rest
                    if (dm && !hist_fast_pos(shm_s, __float_as_uint(m[j]), fp))
                        hist_add_pos(shm, gm, m[j], a.tab, a.err);
                    if (ds && !hist_fast_pos(shs_s, __float_as_uint(s[j]), fp))
                        hist_add_pos(shs, gs, s[j], a.tab, a.err);
                } else {
                    if (dm) hist_add_pos(shm, gm, m[j], a.tab, a.err);
                    if (ds) hist_add_pos(shs, gs, s[j], a.tab, a.err);
                }
            }
        }
    }
    __syncthreads();
    if (cur >= 0) flush(cur);
}

// ---- quantile thresholds (sketch.cpp:59-77) --------------------------------
__global__ void __launch_bounds__(1024) quantile_kernel(const QJob* jobs, int64_t HS,
                                                        const float* keyf, LtParams* lp,
                                                        int* slot_out) {
    __shared__ unsigned long long s_scan[33];
    __shared__ unsigned long long s_tot;
    __shared__ int64_t s_hit;
    const QJob J = jobs[blockIdx.x];
    unsigned long long loc = 0;
    for (int64_t i = threadIdx.x; i < HS; i += blockDim.x) loc += J.hist[i];
    unsigned long long total;
    block_exclusive_scan<unsigned long long>(loc, s_scan, &total);
    if (threadIdx.x == 0) {
        s_tot = total;
        s_hit = HS - 1;
    }
    __syncthreads();
    if (total == 0) return;  // empty sketch: rejected on the host beforehand
    unsigned long long rank =
        (unsigned long long)ceil(__dmul_rn(J.q, (double)(total - 1))) + 1ull;
    if (rank > total) rank = total;
    unsigned long long seen = 0;
    for (int64_t c0 = 0; c0 < HS; c0 += blockDim.x) {
        int64_t i = c0 + threadIdx.x;
        unsigned long long c = i < HS ? J.hist[i] : 0ull, tot;
        unsigned long long ex = block_exclusive_scan<unsigned long long>(c, s_scan, &tot);
        if (c && seen + ex < rank && seen + ex + c >= rank) s_hit = i;
        __syncthreads();
        if (seen + tot >= rank) break;
        seen += tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = keyf[s_hit];
        if (slot_out) slot_out[J.lt * 3 + J.which] = (int)s_hit;
        if (J.which == 0) lp[J.lt].t_mag = t;
        else if (J.which == 1) lp[J.lt].t_sens = t;
        else lp[J.lt].t_prune = t;
    }
}

// ---- pass B: partition + QUANTIZE value histogram + protected counts --------
template <bool EXPL>
__global__ void __launch_bounds__(kPB, 6) pass_b_kernel(PassIn a, const LtParams* lp,
                                                     unsigned long long* gh_val,
                                                     uint32_t* tile_prot,
                                                     unsigned long long* tensor_prot,
                                                     uint8_t* parts) {
    extern __shared__ uint32_t sh[];
    __shared__ uint32_t s_red[2][kPB / 32];  // by tile parity: warps may run ahead into the next tile
    uint32_t par = 0;
    hist_clear(sh);
    __syncthreads();
    __shared__ int s_base;
    int cur = -1;
    LtParams P{};
    for (int base; (base = grab_tiles(a.tile_ctr, kGrab, &s_base)) < a.ntiles;)
    for (int ti = base; ti < min(base + kGrab, a.ntiles); ++ti) {
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        if (threadIdx.x == 0 && ti + 1 < min(base + kGrab, a.ntiles)) prefetch_tile(a, ti + 1, EXPL);
        if (lt != cur) {
            __syncthreads();
            if (cur >= 0) hist_flush(sh, gh_val + cur * a.HS, a.tab);
            __syncthreads();
            cur = lt;
            P = lp[lt];
        }
        uint32_t np = 0;
        unsigned long long* gv = gh_val + lt * a.HS;
        int itn = 0;
        for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 8, ++itn) {
            const uint32_t i2 = i + kPB * 4;
            const bool two = i2 < T.count;
            float4 w0 = ld4(a.w + T.start + i);
            float4 w1 = two ? ld4(a.w + T.start + i2) : make_float4(0, 0, 0, 0);
            float m[8], s[8];
            {
                float mm[4], ss[4];
                load_scores<EXPL>(a, T.start + i, w0, mm, ss);
#pragma unroll
                for (int j = 0; j < 4; ++j) m[j] = mm[j], s[j] = ss[j];
                if (two) {
                    load_scores<EXPL>(a, T.start + i2, w1, mm, ss);
#pragma unroll
                    for (int j = 0; j < 4; ++j) m[4 + j] = mm[j], s[4 + j] = ss[j];
                }
            }
            const float wa[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            uint32_t pw = 0;  // 2 bits per element: the partition pass C reuses
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t e = (j < 4 ? i : i2) + (j & 3);
                if (e >= T.count) continue;
                int part = classify(m[j], s[j], a.has_sens, a.metric, P);
                np += part == 2;
                pw |= (uint32_t)part << (2 * j);
                if (part == 0) hist_add(sh, gv, wa[j], a.tab, a.err);
            }
            if (parts) {  // one byte per float4 group, element order (2 bits per element)
                parts[(T.start + i) >> 2] = (uint8_t)pw;
                if (two) parts[(T.start + i2) >> 2] = (uint8_t)(pw >> 8);
            }
        }
        np = warp_sum(np);
        if ((threadIdx.x & 31) == 0) s_red[par][threadIdx.x >> 5] = np;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int wi = 0; wi < kPB / 32; ++wi) t += s_red[par][wi];
            tile_prot[ti] = t;
            if (t) atomicAdd(tensor_prot + T.tensor, (unsigned long long)t);
        }
        par ^= 1u;
    }
    __syncthreads();
    if (cur >= 0) hist_flush(sh, gh_val + cur * a.HS, a.tab);
}

// ---- fused pass A+B (derived scores, no pruning) ------------------------------------
// Pass B only needs the thresholds pass A's histograms produce.  With a guess of the
// thresholds (the same quantiles over a thinned tile sample, Layout::sample_tiles),
// one streaming pass builds everything both passes produced: the score histograms
// (magnitude as the signed histogram of w, folded afterwards; sensitivity), and for
// the guessed partition the 2-bit codes, per-tile and per-tensor protected counts and
// the histogram of the protected values.  Elements whose score lies in a band of
// kBand buckets around a guessed threshold are listed; once the exact thresholds
// are known, the listed elements whose class differs are corrected (fixup), and
// the QUANTIZE-value histogram is w's histogram minus the protected values'.  When
// an exact threshold falls outside its band (or the list overflows) the host runs
// pass B as before, so the result is exact either way (quantize.cpp:34-92, 383-393).
constexpr int kBand = 4;

struct FuseArgs {
    const LtParams* lpg;           // guessed thresholds [7]
    const float4* band;            // [7]: magnitude (lo, hi], sensitivity (lo, hi]
    unsigned long long* gh_w;      // [7][HS] signed histogram of w
    unsigned long long* gh_sens;   // [7][HS]
    unsigned long long* prot;      // [7][HS] protected (guessed) values by signed slot
    uint8_t* parts;                // 2 bits per element, element order
    uint32_t* tile_prot;
    unsigned long long* tensor_prot;
    unsigned long long* cand;      // (tile << 32) | element
    unsigned long long* n_cand;
    unsigned long long cap;
    uint32_t* flag;                // non-zero: run pass B
};

// window slot of a signed value through the shared compact table; false: exact path
__device__ __forceinline__ bool hist_fast_signed(uint32_t win_s, uint32_t b, const FastPos& f) {
    const uint32_t a = b & 0x7fffffffu;
    const uint32_t rel = min((a >> f.shift) - f.lo, f.n);
    uint32_t c;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(c) : "r"(f.ctab_s + 4 * rel));
    const uint32_t hi = (a & f.offmask) > ((c >> 13) & 0x1ffffu) ? 1u : 0u;
    const uint32_t p = (c & 0x1fffu) + hi;
    const bool ok = !((c >> (31 - hi)) & 1u) && p <= (uint32_t)kWin;
    const uint32_t w = (b >> 31) ? (uint32_t)kWin - p : (uint32_t)kWin + p;
    if (ok) asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(win_s + 4 * w) : "memory");
    return ok;
}

__global__ void __launch_bounds__(kPB, 4) pass_ab_kernel(PassIn a, FuseArgs f) {
    extern __shared__ uint32_t sh[];
    uint32_t* shw = sh;                   // kWinSlots: signed w
    uint32_t* shs = sh + kWinSlots;       // kPosSlots: sensitivity
    uint32_t* s_ctab = shs + kPosSlots;
    __shared__ uint32_t s_red[2][kPB / 32];
    uint32_t par = 0;
    const bool fastc = a.tab.ctab != nullptr;
    for (int i = threadIdx.x; i < kWinSlots + kPosSlots; i += blockDim.x) sh[i] = 0;
    if (fastc) {
        for (uint32_t i = threadIdx.x; i < a.tab.ctab_n; i += blockDim.x) s_ctab[i] = __ldg(a.tab.ctab + i);
        if (threadIdx.x == 0) s_ctab[a.tab.ctab_n] = 0xc0000000u;
    }
    __syncthreads();
    const FastPos fp = fast_pos(a.tab, s_ctab);
    const uint32_t shw_s = (uint32_t)__cvta_generic_to_shared(shw);
    const uint32_t shs_s = (uint32_t)__cvta_generic_to_shared(shs);
    const int lane = threadIdx.x & 31;
    __shared__ int s_base;
    int cur = -1;
    LtParams P{};
    float4 band{};
    for (int base; (base = grab_tiles(a.tile_ctr, kGrab, &s_base)) < a.ntiles;)
    for (int ti = base; ti < min(base + kGrab, a.ntiles); ++ti) {
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        if (threadIdx.x == 0 && ti + 1 < min(base + kGrab, a.ntiles)) prefetch_tile(a, ti + 1, false);
        if (lt != cur) {
            __syncthreads();
            if (cur >= 0) {
                hist_flush(shw, f.gh_w + cur * a.HS, a.tab);
                hist_flush_pos(shs, f.gh_sens + cur * a.HS, a.tab);
            }
            __syncthreads();
            cur = lt;
            P = f.lpg[lt];
            band = f.band[lt];
        }
        unsigned long long* gw = f.gh_w + lt * a.HS;
        unsigned long long* gs = f.gh_sens + lt * a.HS;
        uint32_t np = 0;
        int itn = 0;
        for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 8, ++itn) {
            const uint32_t i2 = i + kPB * 4;
            const bool two = i2 < T.count;
            const float4 w0 = ld4(a.w + T.start + i);
            const float4 w1 = two ? ld4(a.w + T.start + i2) : make_float4(0, 0, 0, 0);
            float m[8], s[8];
            {
                float mm[4], ss[4];
                load_scores<false>(a, T.start + i, w0, mm, ss);
#pragma unroll
                for (int j = 0; j < 4; ++j) m[j] = mm[j], s[j] = ss[j];
                if (two) {
                    load_scores<false>(a, T.start + i2, w1, mm, ss);
#pragma unroll
                    for (int j = 0; j < 4; ++j) m[4 + j] = mm[j], s[4 + j] = ss[j];
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) m[4 + j] = s[4 + j] = 0.0f;
                }
            }
            const float wa[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            uint32_t pw = 0;
            const uint32_t act = __activemask();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t e = (j < 4 ? i : i2) + (j & 3);
                const bool valid = e < T.count;
                bool c = false;
                if (valid) {
                    if (!(fastc && hist_fast_signed(shw_s, __float_as_uint(wa[j]), fp)))
                        hist_add(shw, gw, wa[j], a.tab, a.err);
                    if (a.has_sens && !(fastc && hist_fast_pos(shs_s, __float_as_uint(s[j]), fp)))
                        hist_add_pos(shs, gs, s[j], a.tab, a.err);
                    const int part = classify(m[j], s[j], a.has_sens, a.metric, P);
                    np += part == 2;
                    pw |= (uint32_t)part << (2 * j);
                    if (part == 2 && __float_as_uint(m[j]) < 0x7f800000u)
                        atomicAdd(f.prot + lt * a.HS + slot_of(wa[j], a.tab), 1ull);
                    c = (m[j] > band.x && m[j] <= band.y) || (a.has_sens && s[j] > band.z && s[j] <= band.w);
                }
                const uint32_t bal = __ballot_sync(act, c);
                if (bal) {  // warp-aggregated append to the band list
                    const int leader = __ffs(bal) - 1;
                    unsigned long long b0 = 0;
                    if (lane == leader) b0 = atomicAdd(f.n_cand, (unsigned long long)__popc(bal));
                    b0 = __shfl_sync(act, b0, leader);
                    if (c) {
                        const unsigned long long at = b0 + __popc(bal & ((1u << lane) - 1u));
                        if (at < f.cap) f.cand[at] = ((unsigned long long)ti << 32) | e;
                        else atomicOr(f.flag, 1u);
                    }
                }
            }
            f.parts[(T.start + i) >> 2] = (uint8_t)pw;
            if (two) f.parts[(T.start + i2) >> 2] = (uint8_t)(pw >> 8);
        }
        np = warp_sum(np);
        if (lane == 0) s_red[par][threadIdx.x >> 5] = np;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int wi = 0; wi < kPB / 32; ++wi) t += s_red[par][wi];
            f.tile_prot[ti] = t;
            if (t) atomicAdd(f.tensor_prot + T.tensor, (unsigned long long)t);
        }
        par ^= 1u;
    }
    __syncthreads();
    if (cur >= 0) {
        hist_flush(shw, f.gh_w + cur * a.HS, a.tab);
        hist_flush_pos(shs, f.gh_sens + cur * a.HS, a.tab);
    }
}

// ---- pass A2: score histograms + protected candidates (replaces pass B) -----------
// For derived scores without pruning (the default QuantConfig), pass B's only jobs are
// the partition (quantize.cpp:76-89) and the QUANTIZE-value histogram (:384-393).
// The protected set is tiny (protect_frac), so pass A2 reads w + EMA once and builds
//   * the signed histogram of w (|w|'s histogram is its fold -- the magnitude scores),
//   * the sensitivity histogram, and
//   * a candidate list: every element whose magnitude or sensitivity exceeds a lower
//     bound of its threshold (the quantile of a thinned tile sample, kCandMargin
//     buckets lower).
// Once the exact thresholds are known, the candidates are classified: protected ones
// set a bit in an element bitmap (the fused encoder's partition) and are counted per
// tile and tensor; the QUANTIZE-value histogram is w's histogram minus theirs.  If an
// exact threshold lies below its bound (or the list overflows) pass B runs as before,
// so the result is exact either way.
constexpr int kCandMargin = 4;  // sketch buckets below the sample quantile (~8 % at alpha 0.01)

struct A2Args {
    const float2* lo;               // [7]: candidate lower bounds (magnitude, sensitivity)
    // [7]: bound slots; a layer type with a sensitivity bound (y >= 0) skips its
    // sensitivity histogram here: the buckets above the bound are rebuilt from the
    // candidates and everything below is one count (sens_from_cand / sens_lump)
    const int2* lo_slot;
    unsigned long long* gh_w;       // [7][HS] signed histogram of w
    unsigned long long* gh_sens;    // [7][HS]
    uint4* cand;                    // (tile, element, w bits, sensitivity bits)
    unsigned long long* n_cand;
    unsigned long long cap;
};

__global__ void __launch_bounds__(kPB, 5) pass_a2_kernel(PassIn a, A2Args f) {
    extern __shared__ uint32_t sh[];
    uint32_t* shw = sh;              // kWinSlots: signed w
    uint32_t* shs = sh + kWinSlots;  // kPosSlots: sensitivity
    uint32_t* s_ctab = shs + kPosSlots;
    const bool fastc = a.tab.ctab != nullptr;
    for (int i = threadIdx.x; i < kWinSlots + kPosSlots; i += blockDim.x) sh[i] = 0;
    if (fastc) {
        for (uint32_t i = threadIdx.x; i < a.tab.ctab_n; i += blockDim.x) s_ctab[i] = __ldg(a.tab.ctab + i);
        if (threadIdx.x == 0) s_ctab[a.tab.ctab_n] = 0xc0000000u;
    }
    __syncthreads();
    const FastPos fp = fast_pos(a.tab, s_ctab);
    const uint32_t shw_s = (uint32_t)__cvta_generic_to_shared(shw);
    const uint32_t shs_s = (uint32_t)__cvta_generic_to_shared(shs);
    const int lane = threadIdx.x & 31;
    __shared__ int s_base;
    int cur = -1;
    float2 lo = make_float2(0.f, 0.f);
    bool sens_hist = true;
    for (int base; (base = grab_tiles(a.tile_ctr, kGrab, &s_base)) < a.ntiles;)
    for (int ti = base; ti < min(base + kGrab, a.ntiles); ++ti) {
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        if (threadIdx.x == 0 && ti + 1 < min(base + kGrab, a.ntiles)) prefetch_tile(a, ti + 1, false);
        if (lt != cur) {
            __syncthreads();
            if (cur >= 0) {
                hist_flush(shw, f.gh_w + cur * a.HS, a.tab);
                hist_flush_pos(shs, f.gh_sens + cur * a.HS, a.tab);
            }
            __syncthreads();
            cur = lt;
            lo = f.lo[lt];
            sens_hist = f.lo_slot[lt].y < 0;
        }
        unsigned long long* gw = f.gh_w + lt * a.HS;
        unsigned long long* gs = f.gh_sens + lt * a.HS;
        // the whole tile's loads first (4 float4 of w and of EMA per thread: twice the
        // bytes in flight of a two-group iteration), then the 16 elements
        float4 wv[4], ev[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t i = g * kPB * 4 + threadIdx.x * 4;
            wv[g] = i < T.count ? ld4(a.w + T.start + i) : make_float4(0, 0, 0, 0);
            ev[g] = (a.has_sens && i < T.count) ? ld4(a.ema + T.start + i) : make_float4(0, 0, 0, 0);
        }
        uint32_t cm = 0;  // candidate elements of this thread (bit 4g + j)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t i = g * kPB * 4 + threadIdx.x * 4;
            const float wa[4] = {wv[g].x, wv[g].y, wv[g].z, wv[g].w};
            const float ea[4] = {ev[g].x, ev[g].y, ev[g].z, ev[g].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (i + j >= T.count) continue;
                const float m = fabsf(wa[j]);
                const float s = a.has_sens ? fabsf(__fmul_rn(ea[j], wa[j])) : 0.0f;  // ranker.cpp:96
                if (!(fastc && hist_fast_signed(shw_s, __float_as_uint(wa[j]), fp)))
                    hist_add(shw, gw, wa[j], a.tab, a.err);
                if (a.has_sens) {
                    if (sens_hist) {
                        if (!(fastc && hist_fast_pos(shs_s, __float_as_uint(s), fp)))
                            hist_add_pos(shs, gs, s, a.tab, a.err);
                    } else if (__float_as_uint(s) >= 0x7f800000u) {
                        atomicOr(a.err, kErrNonFinite);
                    }
                }
                if (m > lo.x || (a.has_sens && s > lo.y)) cm |= 1u << (4 * g + j);
            }
        }
        {
            const uint32_t act = __activemask();
            const uint32_t bal = __ballot_sync(act, cm != 0);
            if (bal) {  // warp-aggregated append (rare)
                const uint32_t cnt = __popc(cm);
                uint32_t x = cnt;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(act, x, o);
                    if (lane >= o) x += y;
                }
                const int last = 31 - __clz(act);
                unsigned long long b0 = 0;
                if (lane == last) b0 = atomicAdd(f.n_cand, (unsigned long long)x);
                b0 = __shfl_sync(act, b0, last);
                unsigned long long at = b0 + (x - cnt);
                for (uint32_t q = cm; q; q &= q - 1) {
                    const int bit = __ffs(q) - 1, g = bit >> 2, j = bit & 3;
                    const uint32_t e = g * kPB * 4 + threadIdx.x * 4 + j;
                    // re-read (cached): the register arrays stay statically indexed
                    const float w = a.w[T.start + e];
                    const float s = a.has_sens ? fabsf(__fmul_rn(a.ema[T.start + e], w)) : 0.0f;
                    if (at < f.cap)
                        f.cand[at] = make_uint4((uint32_t)ti, e, __float_as_uint(w), __float_as_uint(s));
                    ++at;
                }
            }
        }
    }
    __syncthreads();
    if (cur >= 0) {
        hist_flush(shw, f.gh_w + cur * a.HS, a.tab);
        hist_flush_pos(shs, f.gh_sens + cur * a.HS, a.tab);
    }
}

// Pass A2 with the inputs staged in shared memory by the TMA engine: half tiles
// (2048 elements of w and EMA, 16 KB) are copied with cp.async.bulk into a
// two-stage ring completed on mbarriers, the next half-tile's copy issued before the
// current one is processed, so the histogram work never waits on global loads.
constexpr uint32_t kA2Half = kTile / 2;

struct A2Stage {
    float w[kA2Half];
    float e[kA2Half];
};

__global__ void __launch_bounds__(kPB, 3) pass_a2_tma_kernel(PassIn a, A2Args f) {
    extern __shared__ __align__(16) uint8_t a2_dyn[];
    A2Stage* stg = (A2Stage*)a2_dyn;  // [2]
    uint32_t* sh = (uint32_t*)(a2_dyn + 2 * sizeof(A2Stage));
    uint32_t* shw = sh;              // kWinSlots: signed w
    uint32_t* shs = sh + kWinSlots;  // kPosSlots: sensitivity
    uint32_t* s_ctab = shs + kPosSlots;
    __shared__ __align__(8) uint64_t s_mbar[2];
    __shared__ int s_next;
    const int tid = threadIdx.x, lane = tid & 31;
    const bool fastc = a.tab.ctab != nullptr;
    for (int i = tid; i < kWinSlots + kPosSlots; i += blockDim.x) sh[i] = 0;
    if (fastc) {
        for (uint32_t i = tid; i < a.tab.ctab_n; i += blockDim.x) s_ctab[i] = __ldg(a.tab.ctab + i);
        if (tid == 0) s_ctab[a.tab.ctab_n] = 0xc0000000u;
    }
    // work items: (tile, half), 2 * tile + half; thread 0 walks them in grabs of
    // kGrab tiles and keeps one item in flight ahead of the one being processed
    int g_end = 0, g_item = 0;  // thread 0 only
    auto next_item = [&](int item) -> int {
        for (;;) {
            int n = item + 1;
            if (item >= 0 && (item & 1) == 0 && a.tiles[item >> 1].count <= kA2Half) ++n;  // no second half
            if (item >= 0 && n < g_end) return n;
            const int gb = (int)atomicAdd(a.tile_ctr, (unsigned)kGrab);
            if (gb >= a.ntiles) return 2 * a.ntiles;
            g_item = 2 * gb;
            g_end = 2 * min(gb + kGrab, a.ntiles);
            return g_item;
        }
    };
    auto issue = [&](int item, int slot) {
        const Tile T = a.tiles[item >> 1];
        const uint32_t h0 = (item & 1) * kA2Half;
        const uint32_t n = min(T.count - h0, kA2Half);
        const uint32_t bytes = ((n + 3u) & ~3u) * 4u;
        mbar_arrive_expect_tx(&s_mbar[slot], a.has_sens ? 2 * bytes : bytes);
        bulk_g2s(stg[slot].w, a.w + T.start + h0, bytes, &s_mbar[slot]);
        if (a.has_sens) bulk_g2s(stg[slot].e, a.ema + T.start + h0, bytes, &s_mbar[slot]);
    };
    if (tid == 0) {
        mbar_init(&s_mbar[0], 1);
        mbar_init(&s_mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int first = next_item(-1);
        s_next = first;
        if (first < 2 * a.ntiles) issue(first, 0);
    }
    __syncthreads();
    const FastPos fp = fast_pos(a.tab, s_ctab);
    const uint32_t shw_s = (uint32_t)__cvta_generic_to_shared(shw);
    const uint32_t shs_s = (uint32_t)__cvta_generic_to_shared(shs);
    int cur = -1;
    float2 lo = make_float2(0.f, 0.f);
    bool sens_hist = true;
    int item = s_next;
    for (uint32_t it = 0; item < 2 * a.ntiles; ++it) {
        const int slot = it & 1;
        if (tid == 0) {  // the next item's copy into the other stage (free since the last barrier)
            const int nx = next_item(item);
            s_next = nx;
            if (nx < 2 * a.ntiles) {
                fence_proxy_async_smem();
                issue(nx, slot ^ 1);
            }
        }
        const int ti = item >> 1;
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        if (lt != cur) {
            __syncthreads();
            if (cur >= 0) {
                hist_flush(shw, f.gh_w + cur * a.HS, a.tab);
                hist_flush_pos(shs, f.gh_sens + cur * a.HS, a.tab);
            }
            __syncthreads();
            cur = lt;
            lo = f.lo[lt];
            sens_hist = f.lo_slot[lt].y < 0;
        }
        unsigned long long* gw = f.gh_w + lt * a.HS;
        unsigned long long* gs = f.gh_sens + lt * a.HS;
        const uint32_t h0 = (item & 1) * kA2Half;
        const uint32_t n = min(T.count - h0, kA2Half);
        mbar_wait(&s_mbar[slot], (it >> 1) & 1);
        uint32_t cm = 0;  // candidate elements of this thread (bit 4g + j)
        if (a.has_sens && !sens_hist && fastc && n == kA2Half) {
            // the default step's path, its branches hoisted: EMA scores, the sensitivity
            // histogram left to the candidates, a full half tile; non-finite
            // sensitivities reported once per half tile
            uint32_t smax = 0;
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const uint32_t i = g * kPB * 4 + tid * 4;
                const float4 wv = *(const float4*)(stg[slot].w + i);
                const float4 ev = *(const float4*)(stg[slot].e + i);
                const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
                const float ea[4] = {ev.x, ev.y, ev.z, ev.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float m = fabsf(wa[j]);
                    const float sv = fabsf(__fmul_rn(ea[j], wa[j]));  // ranker.cpp:96
                    if (!hist_fast_signed(shw_s, __float_as_uint(wa[j]), fp))
                        hist_add(shw, gw, wa[j], a.tab, a.err);
                    smax = max(smax, __float_as_uint(sv));
                    if (m > lo.x || sv > lo.y) cm |= 1u << (4 * g + j);
                }
            }
            if (smax >= 0x7f800000u) atomicOr(a.err, kErrNonFinite);  // the histogram would have said so
        } else
#pragma unroll
        for (int g = 0; g < 2; ++g) {
            const uint32_t i = g * kPB * 4 + tid * 4;  // within the half tile
            if (i >= n) continue;
            const float4 wv = *(const float4*)(stg[slot].w + i);
            const float4 ev = a.has_sens ? *(const float4*)(stg[slot].e + i) : make_float4(0, 0, 0, 0);
            const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
            const float ea[4] = {ev.x, ev.y, ev.z, ev.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (i + j >= n) continue;
                const float m = fabsf(wa[j]);
                const float s = a.has_sens ? fabsf(__fmul_rn(ea[j], wa[j])) : 0.0f;  // ranker.cpp:96
                if (!(fastc && hist_fast_signed(shw_s, __float_as_uint(wa[j]), fp)))
                    hist_add(shw, gw, wa[j], a.tab, a.err);
                if (a.has_sens) {
                    if (sens_hist) {
                        if (!(fastc && hist_fast_pos(shs_s, __float_as_uint(s), fp)))
                            hist_add_pos(shs, gs, s, a.tab, a.err);
                    } else if (__float_as_uint(s) >= 0x7f800000u) {
                        atomicOr(a.err, kErrNonFinite);  // the histogram would have said so
                    }
                }
                if (m > lo.x || (a.has_sens && s > lo.y)) cm |= 1u << (4 * g + j);
            }
        }
        {
            const uint32_t bal = __ballot_sync(0xffffffffu, cm != 0);
            if (bal) {  // warp-aggregated append (rare)
                const uint32_t cnt = __popc(cm);
                uint32_t x = cnt;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                unsigned long long b0 = 0;
                if (lane == 31) b0 = atomicAdd(f.n_cand, (unsigned long long)x);
                b0 = __shfl_sync(0xffffffffu, b0, 31);
                unsigned long long at = b0 + (x - cnt);
                for (uint32_t qm = cm; qm; qm &= qm - 1) {
                    const int bit = __ffs(qm) - 1, g = bit >> 2, j = bit & 3;
                    const uint32_t i = g * kPB * 4 + tid * 4 + j;
                    const float w = stg[slot].w[i];
                    const float s = a.has_sens ? fabsf(__fmul_rn(stg[slot].e[i], w)) : 0.0f;
                    if (at < f.cap)
                        f.cand[at] = make_uint4((uint32_t)ti, h0 + i, __float_as_uint(w), __float_as_uint(s));
                    ++at;
                }
            }
        }
        __syncthreads();  // stage `slot` free for the copy after next; s_next visible
        item = s_next;
    }
    __syncthreads();
    if (cur >= 0) {
        hist_flush(shw, f.gh_w + cur * a.HS, a.tab);
        hist_flush_pos(shs, f.gh_sens + cur * a.HS, a.tab);
    }
}

// candidate lower bounds from the sample's quantile slots; +inf where there is no job
__global__ void cand_bounds_kernel(const int* slot_g, const float* keyf, int64_t NB, int64_t HS,
                                   float2* lo, int2* lo_slot, int shift) {
    const int lt = threadIdx.x;
    if (lt >= kLayerTypes) return;
    float2 b = make_float2(__int_as_float(0x7f800000), __int_as_float(0x7f800000));
    int2 bs = make_int2(-1, -1);
    for (int which = 0; which < 2; ++which) {
        const int g = slot_g[lt * 3 + which];
        if (g < 0) continue;
        // shift: test hook (DQTG_A2_BOUND_SHIFT) -- a bound above the exact threshold
        const int64_t l = min(HS - 1, max(NB, (int64_t)g - kCandMargin + shift));
        if (which == 0) b.x = keyf[l], bs.x = (int)l;
        else b.y = keyf[l], bs.y = (int)l;
    }
    lo[lt] = b;
    lo_slot[lt] = bs;
}

// exact threshold slots at or above the candidate bounds? (else: pass B)  The
// sensitivity threshold must lie strictly above its bound: the bound's bucket holds
// the lumped count of everything below (sens_lump_kernel)
__global__ void cand_check_kernel(const int* slot_x, const int2* lo_slot,
                                  const unsigned long long* n_cand, unsigned long long cap,
                                  uint32_t* flag) {
    const int lt = threadIdx.x;
    if (lt >= kLayerTypes) return;
    const int2 bs = lo_slot[lt];
    for (int which = 0; which < 2; ++which) {
        const int x = slot_x[lt * 3 + which];
        const int b = which ? bs.y : bs.x;
        if (x < 0 && b < 0) continue;
        if (x < 0 || b < 0 || x < b || (which == 1 && x == b)) atomicOr(flag, 2u);
    }
    if (lt == 0 && *n_cand > cap) atomicOr(flag, 4u);
}

// Sensitivity histogram of the layer types with a bound, from the candidate list: the
// buckets above the bound's bucket hold candidates only (every element of them
// exceeds the bound, the bucket's representative), so their counts are exact.
// The candidates' sensitivities crowd into the few buckets above the bound: counted
// per block in shared memory (a window of kSensWin buckets above each layer type's
// bound), flushed once per block.
constexpr int kSensWin = 512;
__global__ void __launch_bounds__(256) sens_from_cand_kernel(PassIn a, const uint4* cand,
                                                             const unsigned long long* n_cand,
                                                             unsigned long long cap,
                                                             const int2* lo_slot,
                                                             unsigned long long* gh_sens) {
    __shared__ uint32_t h[kLayerTypes * kSensWin];
    __shared__ int s_l[kLayerTypes];
    for (int i = threadIdx.x; i < kLayerTypes * kSensWin; i += blockDim.x) h[i] = 0;
    if (threadIdx.x < kLayerTypes) s_l[threadIdx.x] = lo_slot[threadIdx.x].y;
    __syncthreads();
    const unsigned long long n = min(*n_cand, cap);
    for (unsigned long long c = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; c < n;
         c += (unsigned long long)gridDim.x * blockDim.x) {
        const uint4 x = cand[c];
        const int lt = a.types[a.tiles[x.x].tensor];
        const int l = s_l[lt];
        if (l < 0 || x.w >= 0x7f800000u) continue;  // non-finite: flagged by pass A2
        const int64_t idx = slot_of(__uint_as_float(x.w), a.tab);
        if (idx <= l) continue;
        if (idx - l - 1 < kSensWin) atomicAdd(&h[lt * kSensWin + (idx - l - 1)], 1u);
        else atomicAdd(gh_sens + (int64_t)lt * a.HS + idx, 1ull);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kLayerTypes * kSensWin; i += blockDim.x) {
        const uint32_t v = h[i];
        if (!v) continue;
        const int lt = i / kSensWin;
        atomicAdd(gh_sens + (int64_t)lt * a.HS + s_l[lt] + 1 + (i % kSensWin), (unsigned long long)v);
    }
}

struct LtCounts {
    unsigned long long n[kLayerTypes];
};

// ... and everything at or below the bound's bucket as one count in that bucket
// (a quantile depends only on cumulative counts and the crossing bucket, sketch.cpp:59-78)
__global__ void sens_lump_kernel(const int2* lo_slot, unsigned long long* gh_sens, int64_t HS,
                                 LtCounts total) {
    __shared__ unsigned long long s[33];
    const int lt = blockIdx.x;
    const int l = lo_slot[lt].y;
    if (l < 0) return;
    unsigned long long* g = gh_sens + (int64_t)lt * HS;
    unsigned long long acc = 0;
    for (int64_t i = l + 1 + threadIdx.x; i < HS; i += blockDim.x) acc += g[i];
    unsigned long long tot;
    block_exclusive_scan<unsigned long long>(acc, s, &tot);
    if (threadIdx.x == 0) g[l] = total.n[lt] - tot;
}

// per-tensor sums of per-tile counts (one CTA per tensor)
__global__ void tensor_sum_kernel(const uint32_t* tile_cnt, const uint32_t* tile0,
                                  unsigned long long* out) {
    __shared__ unsigned long long s[33];
    const uint32_t t = blockIdx.x;
    unsigned long long acc = 0;
    for (uint32_t i = tile0[t] + threadIdx.x; i < tile0[t + 1]; i += blockDim.x) acc += tile_cnt[i];
    unsigned long long tot;
    block_exclusive_scan<unsigned long long>(acc, s, &tot);
    if (threadIdx.x == 0) out[t] = tot;
}

// classify the candidates with the exact thresholds: protected ones into the bitmap,
// the per-tile / per-tensor counts and the protected-value histogram
__global__ void cand_classify_kernel(PassIn a, const uint4* cand, const unsigned long long* n_cand,
                                     unsigned long long cap, const LtParams* lp, uint32_t* pbits,
                                     uint32_t* tile_prot, unsigned long long* tensor_prot,
                                     unsigned long long* prot_hist) {
    // consecutive candidates come from the same warp append, i.e. the same tile and
    // nearby elements: the atomics are aggregated over the lanes that share a target
    const unsigned long long n = min(*n_cand, cap);
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long c0 = blockIdx.x * (unsigned long long)blockDim.x; c0 < n; c0 += stride) {
        const unsigned long long c = c0 + threadIdx.x;
        bool prot = false;
        uint32_t tile = 0xffffffffu, word = 0xffffffffu, bit = 0;
        long long slot = -1;
        int lt = 0;
        if (c < n) {
            const uint4 q = cand[c];
            const Tile T = a.tiles[q.x];
            lt = a.types[T.tensor];
            const float w = __uint_as_float(q.z);
            prot = classify(fabsf(w), __uint_as_float(q.w), a.has_sens, a.metric, lp[lt]) == 2;
            if (prot) {
                const uint64_t idx = T.start + q.y;
                tile = q.x;
                word = (uint32_t)(idx >> 5);
                bit = 1u << (idx & 31);
                if (__float_as_uint(fabsf(w)) < 0x7f800000u) slot = lt * a.HS + slot_of(w, a.tab);
            }
        }
        const uint32_t act = __ballot_sync(0xffffffffu, prot);
        if (!prot) continue;
        const int lane = threadIdx.x & 31;
        const uint32_t pw = __match_any_sync(act, word);
        const uint32_t ob = __reduce_or_sync(pw, bit);
        if (lane == __ffs(pw) - 1) atomicOr(pbits + word, ob);
        const uint32_t pt = __match_any_sync(act, tile);
        if (lane == __ffs(pt) - 1) atomicAdd(tile_prot + tile, (uint32_t)__popc(pt));
        const uint32_t ps = __match_any_sync(act, (unsigned long long)slot);
        if (slot >= 0 && lane == __ffs(ps) - 1) atomicAdd(prot_hist + slot, (unsigned long long)__popc(ps));
    }
}

// magnitude histogram = |w| folded from the signed histogram of w
__global__ void fold_abs_kernel(const unsigned long long* gw, unsigned long long* gm, int64_t HS,
                                int64_t NB) {
    const int lt = blockIdx.y;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HS;
         i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long v = 0;
        if (i == NB) v = gw[lt * HS + i];
        else if (i > NB) v = gw[lt * HS + i] + gw[lt * HS + (2 * NB - i)];  // neg slot of the same k
        gm[lt * HS + i] = v;
    }
}

// band (lo, hi] around each guessed threshold: kBand buckets either side
__global__ void band_kernel(const int* slot_g, const float* keyf, int64_t NB, int64_t HS,
                            float4* band, int2* band_slots, LtParams* lpg, int shift) {
    const int lt = threadIdx.x;
    if (lt >= kLayerTypes) return;
    float4 b = make_float4(FLT_MAX, -FLT_MAX, FLT_MAX, -FLT_MAX);
    int2 bs = make_int2(-1, -1);  // per kind: packed lo | hi << 16 relative to NB
    for (int which = 0; which < 2; ++which) {
        int g = slot_g[lt * 3 + which];
        if (g < 0) continue;
        if (shift) {  // test hook (DQTG_FUSED_GUESS_SHIFT): a deliberately wrong guess
            g = (int)min(HS - 1, max((int64_t)NB, (int64_t)g + shift));
            if (which == 0) lpg[lt].t_mag = keyf[g];
            else lpg[lt].t_sens = keyf[g];
        }
        const int64_t lo = max((int64_t)NB, (int64_t)g - kBand), hi = min(HS - 1, (int64_t)g + kBand);
        if (which == 0) b.x = keyf[lo], b.y = keyf[hi], bs.x = (int)((lo - NB) | ((hi - NB) << 16));
        else b.z = keyf[lo], b.w = keyf[hi], bs.y = (int)((lo - NB) | ((hi - NB) << 16));
    }
    band[lt] = b;
    band_slots[lt] = bs;
}

// exact thresholds inside their bands?
__global__ void band_check_kernel(const int* slot_x, const int2* band_slots, int64_t NB,
                                  const unsigned long long* n_cand, unsigned long long cap,
                                  uint32_t* flag) {
    const int lt = threadIdx.x;
    if (lt >= kLayerTypes) return;
    const int2 bs = band_slots[lt];
    for (int which = 0; which < 2; ++which) {
        const int x = slot_x[lt * 3 + which];
        const int b = which ? bs.y : bs.x;
        if (x < 0 && b < 0) continue;
        if (x < 0 || b < 0) {
            atomicOr(flag, 2u);
            continue;
        }
        const int64_t lo = NB + (b & 0xffff), hi = NB + (b >> 16);
        if (x < lo || x > hi) atomicOr(flag, 2u);
    }
    if (lt == 0 && *n_cand > cap) atomicOr(flag, 4u);
}

// correct the listed elements whose exact class differs from the guessed one
__global__ void fixup_kernel(PassIn a, FuseArgs f, const LtParams* lp) {
    const unsigned long long n = min(*f.n_cand, f.cap);
    for (unsigned long long c = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; c < n;
         c += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long q = f.cand[c];
        const uint32_t ti = (uint32_t)(q >> 32), o = (uint32_t)q;
        const Tile T = a.tiles[ti];
        const int lt = a.types[T.tensor];
        const float w = a.w[T.start + o];
        const float m = fabsf(w);
        const float s = a.has_sens ? fabsf(__fmul_rn(a.ema[T.start + o], w)) : 0.0f;
        const int g = classify(m, s, a.has_sens, a.metric, f.lpg[lt]);
        const int x = classify(m, s, a.has_sens, a.metric, lp[lt]);
        if (g == x) continue;
        const bool to_prot = x == 2;  // no pruning on this path: classes 0 <-> 2
        atomicAdd(f.prot + lt * a.HS + slot_of(w, a.tab), to_prot ? 1ull : ~0ull);
        atomicAdd(f.tile_prot + ti, to_prot ? 1u : ~0u);
        atomicAdd(f.tensor_prot + T.tensor, to_prot ? 1ull : ~0ull);
        // 2-bit code of element o (element-order layout, 16 codes per word)
        const uint64_t idx = T.start + o;
        uint32_t* word = (uint32_t*)f.parts + (idx >> 4);
        const uint32_t sh = 2 * (uint32_t)(idx & 15);
        if (to_prot) atomicOr(word, 2u << sh);
        else atomicAnd(word, ~(3u << sh));
    }
}

// QUANTIZE-value histogram = w's histogram minus the protected values'
__global__ void value_hist_kernel(const unsigned long long* gw, const unsigned long long* prot,
                                  unsigned long long* gv, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        gv[i] = gw[i] - prot[i];
}

// ---- exclusive scan of per-tile counts (single CTA) --------------------------
__global__ void __launch_bounds__(1024) scan_u32_kernel(const uint32_t* in, int n,
                                                        unsigned long long* out) {
    __shared__ unsigned long long s[33];
    constexpr int kPer = 8;  // consecutive entries per thread: fewer block scans
    unsigned long long base = 0;
    for (int c0 = 0; c0 < n; c0 += blockDim.x * kPer) {
        const int i0 = c0 + threadIdx.x * kPer;
        uint32_t v[kPer];
        unsigned long long sum = 0, tot;
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            v[u] = i0 + u < n ? in[i0 + u] : 0u;
            sum += v[u];
        }
        unsigned long long ex = block_exclusive_scan<unsigned long long>(sum, s, &tot);
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            if (i0 + u < n) out[i0 + u] = base + ex;
            ex += v[u];
        }
        base += tot;
    }
    if (threadIdx.x == 0) out[n] = base;
}

// ---- pass C: levels + protected entries --------------------------------------
__device__ __forceinline__ uint32_t nearest_center(const float* c, uint32_t k, float v) {
    // quantize.cpp:327-335: lower_bound, then float half-gap, ties to the lower index
    uint32_t lo = 0, n = k;
    while (n > 0) {
        uint32_t h = n >> 1;
        if (c[lo + h] < v) {
            lo += h + 1;
            n -= h + 1;
        } else {
            n = h;
        }
    }
    if (lo == 0) return 0;
    if (lo == k) return k - 1;
    return (__fsub_rn(c[lo], v) < __fsub_rn(v, c[lo - 1])) ? lo : lo - 1;
}

// Level boundaries: nearest_center is monotone non-decreasing in v (lower_bound
// plus a half-gap compare whose two sides move in opposite directions), so it is
// fully described by T[j] = smallest float (in value order) with level >= j,
// j = 1..k-1: level(v) = #{j : v >= T[j]}.  One thread per boundary finds T[j]
// by bisection over the ordered float encoding, evaluating the reference rule
// itself; -0.0 and +0.0 get the same level (they compare equal everywhere in
// the rule), so a float compare against T[j] is exact for every finite v.
__device__ __forceinline__ uint32_t ord_of(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float float_of_ord(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

__global__ void __launch_bounds__(64) level_bounds_kernel(const float* cb, int cb_stride,
                                                          const uint32_t* cb_len, float* lb,
                                                          int lb_stride) {
    extern __shared__ float s_c[];
    const int lt = blockIdx.x;
    const uint32_t k = cb_len[lt];
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) s_c[j] = cb[lt * cb_stride + j];
    __syncthreads();
    for (int j = threadIdx.x; j < lb_stride; j += blockDim.x) {
        float t = __int_as_float(0x7f800000);  // +inf: never reached by a finite value
        if (j >= 1 && (uint32_t)j < k) {
            uint32_t lo = ord_of(-__int_as_float(0x7f800000)), hi = ord_of(__int_as_float(0x7f800000));
            while (lo < hi) {  // level(float_of_ord(hi)) >= j holds throughout
                const uint32_t mid = lo + ((hi - lo) >> 1);
                if (nearest_center(s_c, k, float_of_ord(mid)) >= (uint32_t)j) hi = mid;
                else lo = mid + 1;
            }
            t = float_of_ord(lo);
        }
        lb[lt * lb_stride + j] = t;
    }
}

// Level of a QUANTIZE value from the boundaries (P = power of two >= k, T[j] =
// +inf for j >= k): branch-free bisection, log2(P) shared loads.
__device__ __forceinline__ uint32_t level_of(const float* T, uint32_t P, float v) {
    uint32_t pos = 0;
    for (uint32_t st = P >> 1; st > 0; st >>= 1) pos += (v >= T[pos + st]) ? st : 0u;
    return pos;
}

__host__ __device__ __forceinline__ uint32_t pow2_ceil(uint32_t k) {
    uint32_t p = 1;
    while (p < k) p <<= 1;
    return p;
}

template <int LOGP>
__device__ __forceinline__ uint32_t level_fixed(const float* T, float v, uint32_t kp) {
    if (LOGP < 0) return level_of(T, kp, v);  // k > 64: runtime bisection
    uint32_t pos = 0;
#pragma unroll
    for (int st = (1 << LOGP) >> 1; st > 0; st >>= 1) pos += (v >= T[pos + st]) ? (uint32_t)st : 0u;
    return pos;
}

// One tile of pass C with the level bisection unrolled for P = 2^LOGP.
template <bool EXPL, int LOGP, bool PARTS>
__device__ __forceinline__ void pass_c_tile(const PassIn& a, const LtParams& P, const Tile& T,
                                            uint32_t k, const float* s_lb, uint64_t tensor_base,
                                            unsigned long long out,
                                            unsigned long long* s_scan, uint16_t* levels,
                                            uint64_t* ppos, uint16_t* pval, const uint8_t* parts,
                                            int ti) {
    // two float4 groups per thread and iteration; protected entries keep element
    // order: group 0 (i0..i0+1023) before group 1, one packed (lo|hi) scan
    int itn = 0;
    for (uint32_t i0 = 0; i0 < T.count; i0 += kPB * 8, ++itn) {
        uint32_t flags[2] = {0, 0};
        float wa[2][4];
        uint32_t pw = 0;
        if (PARTS) {
            const uint32_t i = i0 + threadIdx.x * 4, i2 = i + kPB * 4;
            if (i < T.count) pw = parts[(T.start + i) >> 2];
            if (i2 < T.count) pw |= (uint32_t)parts[(T.start + i2) >> 2] << 8;
        }
        for (int g = 0; g < 2; ++g) {
            const uint32_t i = i0 + g * kPB * 4 + threadIdx.x * 4;
            wa[g][0] = wa[g][1] = wa[g][2] = wa[g][3] = 0.0f;
            if (i < T.count) {
                const uint64_t idx = T.start + i;
                float4 wv = ld4(a.w + idx);
                float m[4] = {0, 0, 0, 0}, s[4] = {0, 0, 0, 0};
                if (!PARTS) load_scores<EXPL>(a, idx, wv, m, s);
                wa[g][0] = wv.x, wa[g][1] = wv.y, wa[g][2] = wv.z, wa[g][3] = wv.w;
                uint32_t lv[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    // level for every element (branch-free), then the partition decides
                    const uint32_t q = level_fixed<LOGP>(s_lb, wa[g][j], pow2_ceil(k));
                    const int part = PARTS ? (int)((pw >> (2 * (4 * g + j))) & 3u)
                                           : classify(m[j], s[j], a.has_sens, a.metric, P);
                    lv[j] = part == 0 ? q : (part == 1 ? k : k + 1);
                    if (part == 2 && i + j < T.count) flags[g] |= 1u << j;
                }
                uint2 pk;
                pk.x = lv[0] | (lv[1] << 16);
                pk.y = lv[2] | (lv[3] << 16);
                *(uint2*)(levels + idx) = pk;
            }
        }
        const unsigned long long packed =
            (unsigned long long)__popc(flags[0]) | ((unsigned long long)__popc(flags[1]) << 32);
        unsigned long long tot;
        const unsigned long long ex = block_exclusive_scan<unsigned long long>(packed, s_scan, &tot);
        const unsigned long long tot0 = tot & 0xffffffffull;
        for (int g = 0; g < 2; ++g) {
            if (!flags[g]) continue;
            const uint32_t i = i0 + g * kPB * 4 + threadIdx.x * 4;
            unsigned long long o = out + (g ? tot0 + (ex >> 32) : (ex & 0xffffffffull));
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (flags[g] >> j & 1) {
                    ppos[o] = (T.start - tensor_base) + i + j;
                    pval[o] = bf16_rne(wa[g][j]);
                    ++o;
                }
        }
        out += tot0 + (tot >> 32);
    }
}

template <bool EXPL, bool PARTS>
__global__ void __launch_bounds__(kPB) pass_c_kernel(PassIn a, const LtParams* lp,
                                                     const float* lb, int lb_stride,
                                                     const uint32_t* cb_len,
                                                     const unsigned long long* tile_prot_off,
                                                     uint16_t* levels, uint64_t* ppos,
                                                     uint16_t* pval, const uint8_t* parts) {
    extern __shared__ float s_lb[];
    __shared__ unsigned long long s_scan[33];
    const int ti = blockIdx.x;
    const Tile T = a.tiles[ti];
    const int lt = a.types[T.tensor];
    // the tile a CTA launched about one residency later will read (L2 prefetch)
    if (threadIdx.x == 0 && ti + kPfDist < a.ntiles) {
        if (PARTS) {
            const Tile N = a.tiles[ti + kPfDist];
            prefetch_l2(a.w + N.start, ((N.count + 3u) & ~3u) * 4u);
        } else {
            prefetch_tile(a, ti + kPfDist, EXPL);
        }
    }
    const uint32_t k = cb_len[lt], kp = pow2_ceil(k);
    for (uint32_t j = threadIdx.x; j < kp; j += blockDim.x) s_lb[j] = lb[lt * lb_stride + j];
    const LtParams P = lp[lt];
    const uint64_t tensor_base = a.tensor_off[T.tensor];
    __syncthreads();
    const unsigned long long out = tile_prot_off[ti];
    switch (__ffs(kp) - 1) {
#define DQTG_PC(L) \
    case L: pass_c_tile<EXPL, L, PARTS>(a, P, T, k, s_lb, tensor_base, out, s_scan, levels, ppos, pval, parts, ti); break;
        DQTG_PC(0) DQTG_PC(1) DQTG_PC(2) DQTG_PC(3) DQTG_PC(4) DQTG_PC(5) DQTG_PC(6)
#undef DQTG_PC
        default: pass_c_tile<EXPL, -1, PARTS>(a, P, T, k, s_lb, tensor_base, out, s_scan, levels, ppos, pval, parts, ti);
    }
}

// ---- dequantize (quantize.cpp:427-462) ----------------------------------------
// Protected entries of tile ti: [lo[ti], hi[ti]) by binary search of the tile's element
// range in its tensor's ascending positions (no pass over the levels).  Entries of a
// tensor outside all of its tiles (positions >= numel) are unreferenced: CorruptIndex.
__global__ void prot_tile_range_kernel(const Tile* tiles, int ntiles, const uint64_t* tensor_off,
                                       const uint32_t* tile0, const unsigned long long* prot_off,
                                       const uint64_t* ppos, unsigned long long* lo_hi,
                                       uint32_t* err) {
    const int ti = blockIdx.x * blockDim.x + threadIdx.x;
    if (ti >= ntiles) return;
    const Tile T = tiles[ti];
    const uint32_t t = T.tensor;
    const unsigned long long base = prot_off[t], cnt = prot_off[t + 1] - base;
    const uint64_t* p = ppos + base;
    const uint64_t r0 = T.start - tensor_off[t], r1 = r0 + T.count;
    auto lower = [&](uint64_t x) {
        unsigned long long lo = 0, hi = cnt;
        while (lo < hi) {
            const unsigned long long mid = (lo + hi) >> 1;
            if (p[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    };
    const unsigned long long a = lower(r0), b = lower(r1);
    lo_hi[2 * ti] = base + a;
    lo_hi[2 * ti + 1] = base + b;
    if ((uint32_t)ti + 1 == tile0[t + 1] && b != cnt) atomicOr(err, kErrCorruptIndex);
}

// out[t]: the tensor's output (device pointers); every protected level must meet its
// entry in order, and every entry of the tile a protected level.  16 contiguous
// levels per thread (two 16-byte loads), one block scan of the protected counts per
// tile, float4 stores when the output is 16-byte aligned.
__global__ void __launch_bounds__(256) dequant_kernel(const Tile* tiles, const uint8_t* types,
                                                      const uint64_t* tensor_off, const float* cb,
                                                      int cb_stride, const uint32_t* cb_len,
                                                      const uint16_t* levels,
                                                      const unsigned long long* lo_hi,
                                                      const uint64_t* ppos, const uint16_t* pval,
                                                      float* const* outs, uint32_t* err) {
    __shared__ uint32_t s_slots[8];
    const Tile T = tiles[blockIdx.x];
    const int lt = types[T.tensor];
    const uint32_t k = cb_len[lt];
    const float* c = cb + lt * cb_stride;
    const uint64_t rel0 = T.start - tensor_off[T.tensor];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t e0 = tid * 16;
    const uint32_t nv = e0 < T.count ? min(T.count - e0, 16u) : 0u;
    uint32_t lw[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // 16 levels, two per word
    if (nv) {
        const uint4* lp = (const uint4*)(levels + T.start + e0);  // tile starts are 64-aligned
        const uint4 x = lp[0], y = lp[1];
        lw[0] = x.x, lw[1] = x.y, lw[2] = x.z, lw[3] = x.w, lw[4] = y.x, lw[5] = y.y, lw[6] = y.z, lw[7] = y.w;
    }
    uint32_t pm = 0;  // protected elements of the thread
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t l = (lw[j >> 1] >> (16 * (j & 1))) & 0xffffu;
        if ((uint32_t)j < nv && l == k + 1) pm |= 1u << j;
    }
    // exclusive block scan of the protected counts (one barrier)
    const uint32_t cnt = __popc(pm);
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_slots[wid] = x;
    __syncthreads();
    uint32_t base = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint32_t sv = s_slots[w];
        base += w < wid ? sv : 0u;
        tot += sv;
    }
    const unsigned long long o0 = lo_hi[2 * blockIdx.x], o1 = lo_hi[2 * blockIdx.x + 1];
    unsigned long long o = o0 + base + (x - cnt);
    float v[16];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t l = (lw[j >> 1] >> (16 * (j & 1))) & 0xffffu;
        float f = 0.0f;
        if (l < k) {
            f = __ldg(c + l);
        } else if ((pm >> j) & 1u) {
            if (o >= o1 || ppos[o] != rel0 + e0 + j) bad = true;
            else f = __uint_as_float((uint32_t)pval[o] << 16);
            ++o;
        } else if (l != k && (uint32_t)j < nv) {
            bad = true;
        }
        v[j] = f;
    }
    if (bad) atomicOr(err, kErrCorruptIndex);
    if (tid == 0 && tot != o1 - o0) atomicOr(err, kErrCorruptIndex);  // unreferenced entries
    if (!nv) return;
    float* out = outs[T.tensor] + rel0 + e0;
    if (nv == 16 && ((uintptr_t)out & 15) == 0) {
        float4* o4 = (float4*)out;
#pragma unroll
        for (int q = 0; q < 4; ++q) o4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if ((uint32_t)j < nv) out[j] = v[j];
    }
}

// ---- partition masks (quantize.cpp:34-92 as a stand-alone entry point) --------
template <bool EXPL>
__global__ void __launch_bounds__(kPB) mask_kernel(PassIn a, const LtParams* lp, uint8_t* out) {
    const Tile T = a.tiles[blockIdx.x];
    const int lt = a.types[T.tensor];
    const LtParams P = lp[lt];
    for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 4) {
        const uint64_t idx = T.start + i;
        float4 wv = ld4(a.w + idx);
        float m[4], s[4];
        load_scores<EXPL>(a, idx, wv, m, s);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (i + j < T.count) out[idx + j] = (uint8_t)classify(m[j], s[j], a.has_sens, a.metric, P);
    }
}

// ---- candidate evaluation (ProxyEvaluator::evaluate, search.cpp:107-112) ------
// Same partition + assignment as pass C, but instead of storing levels it
// accumulates sum (w - dequant(w))^2 per tile (fixed reduction order) and the
// per-tensor level histogram that estimate_compression needs.
__device__ __forceinline__ double block_sum_d(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    __syncthreads();
    return t;
}

template <bool EXPL>
__global__ void __launch_bounds__(kPB) eval_c_kernel(PassIn a, const LtParams* lp, const float* cb,
                                                     int cb_stride, const float* lb, int lb_stride,
                                                     const uint32_t* cb_len,
                                                     double* tile_diff,
                                                     unsigned long long* lvl_counts,
                                                     int lstride) {
    extern __shared__ float s_cb[];  // [cb_stride] codebook, then [kp] level bounds
    __shared__ double s_red[kPB / 32];
    __shared__ uint32_t s_cnt[66];
    const int ti = blockIdx.x;
    const Tile T = a.tiles[ti];
    const int lt = a.types[T.tensor];
    const uint32_t k = cb_len[lt], kp = pow2_ceil(k);
    float* s_lb = s_cb + cb_stride;
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) s_cb[j] = cb[lt * cb_stride + j];
    for (uint32_t j = threadIdx.x; j < kp; j += blockDim.x) s_lb[j] = lb[lt * lb_stride + j];
    for (int j = threadIdx.x; j < 66; j += blockDim.x) s_cnt[j] = 0;
    const LtParams P = lp[lt];
    __syncthreads();
    double acc = 0.0;
    for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 4) {
        const uint64_t idx = T.start + i;
        float4 wv = ld4(a.w + idx);
        float m[4], s[4];
        load_scores<EXPL>(a, idx, wv, m, s);
        const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i + j >= T.count) break;
            int part = classify(m[j], s[j], a.has_sens, a.metric, P);
            uint32_t lv;
            float deq;
            if (part == 0) {
                lv = level_of(s_lb, kp, wa[j]);
                deq = s_cb[lv];
            } else if (part == 1) {
                lv = k;
                deq = 0.0f;
            } else {
                lv = k + 1;
                deq = __uint_as_float((uint32_t)bf16_rne(wa[j]) << 16);
            }
            double d = __dsub_rn((double)wa[j], (double)deq);
            acc = __dadd_rn(acc, __dmul_rn(d, d));
            if (lv < 66) atomicAdd(&s_cnt[lv], 1u);
            else if ((int)lv < lstride)  // large alphabets: straight to the tensor's counts
                atomicAdd(lvl_counts + (size_t)T.tensor * lstride + lv, 1ull);
        }
    }
    double t = block_sum_d(acc, s_red);
    if (threadIdx.x == 0) tile_diff[ti] = t;
    __syncthreads();
    for (int j = threadIdx.x; j < (int)k + 2 && j < lstride; j += blockDim.x)
        if (s_cnt[j]) atomicAdd(lvl_counts + (size_t)T.tensor * lstride + j, (unsigned long long)s_cnt[j]);
}

// ---- batched candidate evaluation: several configs per read of w ------------------
// Candidates sharing a partition (alpha, prune_frac, protect_frac, metric) share
// pass B; their codebooks differ (bins, embed_bins, sigma, seed).  One CTA per tile
// classifies each element once and, for every candidate, finds its level, the
// dequantized value (quantize.cpp:427-462) and Σ(w - deq)² (search.cpp:35-46), and
// counts levels per tensor (search.cpp:66-81).
constexpr int kEvalM = 8;

struct EvalMulti {
    int m;
    const float* cb;        // [m][7][cbs]
    int cbs;
    const float* lb;        // [m][7][lbs]
    int lbs;
    const uint32_t* cb_len; // [m][7]
    double* tile_diff;      // [m][ntiles]
    unsigned long long* counts;  // [m][nt][lstride]
    int lstride;
    int ntiles;
    int nt;                 // tensors (counts stride)
};

template <bool EXPL>
__global__ void __launch_bounds__(kPB) eval_multi_kernel(PassIn a, const LtParams* lp, EvalMulti ev) {
    extern __shared__ float s_tab[];  // per candidate: codebook (cbs) + bounds (lbs)
    __shared__ double s_red[kPB / 32][kEvalM];
    __shared__ uint32_t s_cnt[kEvalM][66];
    __shared__ uint32_t s_k[kEvalM], s_kp[kEvalM];
    const int ti = blockIdx.x;
    const Tile T = a.tiles[ti];
    const int lt = a.types[T.tensor];
    const int m = ev.m, per = ev.cbs + ev.lbs;
    for (int c = threadIdx.x; c < m; c += blockDim.x) {
        s_k[c] = ev.cb_len[c * kLayerTypes + lt];
        s_kp[c] = pow2_ceil(s_k[c]);
    }
    for (int i = threadIdx.x; i < m * 66; i += blockDim.x) (&s_cnt[0][0])[i] = 0;
    __syncthreads();
    for (int c = 0; c < m; ++c) {
        for (int j = threadIdx.x; j < (int)s_k[c]; j += blockDim.x)
            s_tab[c * per + j] = ev.cb[((size_t)c * kLayerTypes + lt) * ev.cbs + j];
        for (int j = threadIdx.x; j < (int)s_kp[c]; j += blockDim.x)
            s_tab[c * per + ev.cbs + j] = ev.lb[((size_t)c * kLayerTypes + lt) * ev.lbs + j];
    }
    const LtParams P = lp[lt];
    __syncthreads();
    double acc[kEvalM];
#pragma unroll
    for (int c = 0; c < kEvalM; ++c) acc[c] = 0.0;
    for (uint32_t i = threadIdx.x * 4; i < T.count; i += kPB * 4) {
        const uint64_t idx = T.start + i;
        const float4 wv = ld4(a.w + idx);
        float mg[4], sn[4];
        load_scores<EXPL>(a, idx, wv, mg, sn);
        const float wa[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i + j >= T.count) break;
            const int part = classify(mg[j], sn[j], a.has_sens, a.metric, P);
            const float prot = __uint_as_float((uint32_t)bf16_rne(wa[j]) << 16);
#pragma unroll
            for (int c = 0; c < kEvalM; ++c) {
                if (c >= m) break;
                const uint32_t k = s_k[c];
                uint32_t lv;
                float deq;
                if (part == 0) {
                    lv = level_of(s_tab + c * per + ev.cbs, s_kp[c], wa[j]);
                    deq = s_tab[c * per + lv];
                } else if (part == 1) {
                    lv = k;
                    deq = 0.0f;
                } else {
                    lv = k + 1;
                    deq = prot;
                }
                const double d = __dsub_rn((double)wa[j], (double)deq);
                acc[c] = __dadd_rn(acc[c], __dmul_rn(d, d));
                if (lv < 66) atomicAdd(&s_cnt[c][lv], 1u);
                else if ((int)lv < ev.lstride)  // large alphabets: straight to global
                    atomicAdd(ev.counts + ((size_t)c * ev.nt + T.tensor) * ev.lstride + lv, 1ull);
            }
        }
    }
    // per candidate: warp sums, then the warps in a fixed order
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < kEvalM; ++c) {
        double v = acc[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) s_red[wid][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < m) {
        double t = 0.0;
        for (int w = 0; w < kPB / 32; ++w) t = __dadd_rn(t, s_red[w][threadIdx.x]);
        ev.tile_diff[(size_t)threadIdx.x * ev.ntiles + ti] = t;
    }
    for (int i = threadIdx.x; i < m * 66; i += blockDim.x) {
        const int c = i / 66, j = i % 66;
        if (j < (int)s_k[c] + 2 && j < ev.lstride && s_cnt[c][j])
            atomicAdd(ev.counts + ((size_t)c * ev.nt + T.tensor) * ev.lstride + j,
                      (unsigned long long)s_cnt[c][j]);
    }
}

// per-layer-type sums of several candidates' tile values (grid: one block each)
__global__ void __launch_bounds__(512) lt_sum_multi_kernel(const Tile* tiles, const uint8_t* types,
                                                           int ntiles, const double* tile_vals,
                                                           double* out /*[m][7]*/) {
    __shared__ double s_part[512][kLayerTypes];
    const double* tv = tile_vals + (size_t)blockIdx.x * ntiles;
    double loc[kLayerTypes] = {0, 0, 0, 0, 0, 0, 0};
    const int per = (ntiles + blockDim.x - 1) / blockDim.x;
    const int a0 = threadIdx.x * per, a1 = min(ntiles, a0 + per);
    for (int i = a0; i < a1; ++i) {
        const int lt = types[tiles[i].tensor];
        loc[lt] = __dadd_rn(loc[lt], tv[i]);
    }
    for (int lt = 0; lt < kLayerTypes; ++lt) s_part[threadIdx.x][lt] = loc[lt];
    __syncthreads();
    if (threadIdx.x < kLayerTypes) {
        double t = 0.0;
        for (int j = 0; j < (int)blockDim.x; ++j) t = __dadd_rn(t, s_part[j][threadIdx.x]);
        out[blockIdx.x * kLayerTypes + threadIdx.x] = t;
    }
}

// sum of squares (or squared differences) per tile, fixed order
__global__ void __launch_bounds__(kPB) tile_sq_kernel(const Tile* tiles, const float* x,
                                                      const float* y, double* tile_out) {
    __shared__ double s_red[kPB / 32];
    const Tile T = tiles[blockIdx.x];
    double acc = 0.0;
    for (uint32_t i = threadIdx.x; i < T.count; i += kPB) {
        double d = (double)x[T.start + i];
        if (y) d = __dsub_rn(d, (double)y[T.start + i]);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    double t = block_sum_d(acc, s_red);
    if (threadIdx.x == 0) tile_out[blockIdx.x] = t;
}

// per-layer-type totals over tiles, fixed order (contiguous chunks per thread)
__global__ void __launch_bounds__(512) lt_sum_kernel(const Tile* tiles, const uint8_t* types,
                                                      int ntiles, const double* tile_vals,
                                                      double* out /*[7]*/) {
    __shared__ double s_part[512][kLayerTypes];
    double loc[kLayerTypes] = {0, 0, 0, 0, 0, 0, 0};
    const int per = (ntiles + blockDim.x - 1) / blockDim.x;
    const int a0 = threadIdx.x * per, a1 = min(ntiles, a0 + per);
    for (int i = a0; i < a1; ++i) {
        const int lt = types[tiles[i].tensor];
        loc[lt] = __dadd_rn(loc[lt], tile_vals[i]);
    }
    for (int lt = 0; lt < kLayerTypes; ++lt) s_part[threadIdx.x][lt] = loc[lt];
    __syncthreads();
    if (threadIdx.x < kLayerTypes) {
        double t = 0.0;
        for (int j = 0; j < (int)blockDim.x; ++j) t = __dadd_rn(t, s_part[j][threadIdx.x]);
        out[threadIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) level_count_kernel(const Tile* tiles, const uint16_t* levels,
                                                          unsigned long long* counts, int lstride) {
    __shared__ uint32_t s_cnt[1024];
    const Tile T = tiles[blockIdx.x];
    for (int j = threadIdx.x; j < lstride && j < 1024; j += blockDim.x) s_cnt[j] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x) {
        uint32_t l = levels[T.start + i];
        if ((int)l < lstride && l < 1024) atomicAdd(&s_cnt[l], 1u);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < lstride && j < 1024; j += blockDim.x)
        if (s_cnt[j]) atomicAdd(counts + (size_t)T.tensor * lstride + j, (unsigned long long)s_cnt[j]);
}

// ---- host orchestration ---------------------------------------------------------
static PassIn pass_in(Engine& e, const DevCkpt& c, const AlphaTables& T, int metric) {
    DQTG_REQUIRE(c.w || c.L->N == 0, DQTG_ERROR, "checkpoint has no weights (released)");
    const Layout& L = *c.L;
    PassIn a{};
    a.tiles = L.d_tiles;
    a.ntiles = (int)L.tiles.size();
    a.types = L.d_types;
    a.tensor_off = L.d_off;
    a.w = c.w;
    a.ema = c.ema;
    a.mag = c.explicit_scores ? c.mag : nullptr;
    a.sens = c.explicit_scores ? c.sens : nullptr;
    a.has_sens = c.has_sens;
    a.metric = metric;
    a.tab = e.bucket_tab(T);
    a.HS = T.HS;
    a.err = e.d_err;
    a.tile_ctr = (unsigned int*)e.buf("q.tile_ctr", 64);
    return a;
}

static int stream_grid(Engine& e, int ntiles, int per_sm) {
    int g = e.num_sms * per_sm;
    return std::max(1, std::min(g, ntiles));
}

void quantize_plan(const Layout& L, const dqtg_config& cfg, bool has_sens, QuantPlan& plan) {
    // Validation in the reference's order (quantize.cpp:375, :35-38, :46-74).
    DQTG_REQUIRE(cfg.bins >= 1 && cfg.embed_bins >= 1, DQTG_ERROR, "bins must be >= 1");
    DQTG_REQUIRE(!(cfg.metric == 1 && !has_sens), DQTG_MISSING_SCORES,
                 "sensitivity prune metric requested without gradient history");
    plan = QuantPlan{};
    for (uint32_t i = 0; i < L.nt; ++i) {
        plan.present[L.types[i]] = true;
        plan.lt_n[L.types[i]] += L.numel[i];
    }
    const bool alpha_ok = cfg.alpha > 0.0 && cfg.alpha < 1.0;
    for (int lt = 0; lt < kLayerTypes; ++lt) {
        LtParams& p = plan.lp[lt];
        p.t_mag = p.t_sens = p.t_prune = FLT_MAX;
        p.flags = 0;
        if (!plan.present[lt]) continue;
        bool do_prune = cfg.prune_frac > 0.0 && lt != kEmbedding;
        if (do_prune) {
            DQTG_REQUIRE(alpha_ok, DQTG_ALPHA_OUT_OF_RANGE, "alpha must be in (0, 1)");
            DQTG_REQUIRE(cfg.prune_frac >= 0.0 && cfg.prune_frac <= 1.0, DQTG_ALPHA_OUT_OF_RANGE,
                         "quantile q must be in [0, 1]");
            DQTG_REQUIRE(plan.lt_n[lt] > 0, DQTG_EMPTY_SKETCH, "quantile of empty sketch");
            p.flags |= kDoPrune;
            plan.jobs.push_back(QJob{lt, 2, cfg.prune_frac, nullptr});
            if (cfg.metric == 1) plan.mask_sens |= 1u << lt;
            else plan.mask_mag |= 1u << lt;
        }
        bool do_protect = cfg.protect_frac > 0.0;
        double q_prot = 1.0 - cfg.protect_frac / 2.0;
        bool protect_all = do_protect && q_prot <= 0.0;
        if (do_protect) p.flags |= kDoProtect;
        if (protect_all) p.flags |= kProtectAll;
        if (do_protect && !protect_all) {
            DQTG_REQUIRE(alpha_ok, DQTG_ALPHA_OUT_OF_RANGE, "alpha must be in (0, 1)");
            DQTG_REQUIRE(plan.lt_n[lt] > 0, DQTG_EMPTY_SKETCH, "quantile of empty sketch");
            plan.jobs.push_back(QJob{lt, 0, q_prot, nullptr});
            plan.mask_mag |= 1u << lt;
            if (has_sens) {
                plan.jobs.push_back(QJob{lt, 1, q_prot, nullptr});
                plan.mask_sens |= 1u << lt;
            }
        }
    }
}

// Work area of one quantization (one config) on the engine.
struct Stage {
    std::string tag;
    QuantPlan plan;
    dqtg_config cfg{};
    uint64_t seed = 0;
    LtParams* d_lp = nullptr;
    unsigned long long *gh_val = nullptr, *tile_off = nullptr, *tensor_prot = nullptr;
    uint32_t* tile_prot = nullptr;
    double *pts = nullptr, *kw = nullptr;
    unsigned long long* kc = nullptr;
    int* n_keys = nullptr;
    int h_nkeys[kLayerTypes] = {0};
    std::vector<unsigned long long> h_tprot;
    float* d_cb = nullptr;  // [7][cb_stride]
    uint32_t cb_stride = 1;
    uint32_t* cb_len = nullptr;
    float* d_lb = nullptr;  // [7][lb_stride] level boundaries (level_bounds_kernel)
    uint32_t lb_stride = 1;
    uint8_t* parts = nullptr;  // pass B partition, 2 bits per element in element order (pass C)
};

static void stage_alloc(Engine& e, const Layout& L, int64_t HS, Stage& s, float* cb_dst) {
    const int ntiles = (int)L.tiles.size();
    const std::string& t = s.tag;
    s.d_lp = (LtParams*)e.buf(t + "lp", sizeof(LtParams) * kLayerTypes);
    s.gh_val = (unsigned long long*)e.buf(t + "gh_val", (size_t)kLayerTypes * HS * 8);
    s.tile_prot = (uint32_t*)e.buf(t + "tile_prot", (size_t)ntiles * 4 + 4);
    s.tile_off = (unsigned long long*)e.buf(t + "tile_off", (size_t)(ntiles + 1) * 8);
    s.tensor_prot = (unsigned long long*)e.buf(t + "tensor_prot", (size_t)(L.nt + 1) * 8);
    s.pts = (double*)e.buf(t + "pts", (size_t)kLayerTypes * HS * 8);
    s.kw = (double*)e.buf(t + "kw", (size_t)kLayerTypes * HS * 8);
    s.kc = (unsigned long long*)e.buf(t + "kc", (size_t)kLayerTypes * HS * 8);
    s.n_keys = (int*)e.buf(t + "nkeys", kLayerTypes * 4);
    s.cb_len = (uint32_t*)e.buf(t + "cblen", kLayerTypes * 4);
    s.cb_stride = std::max(1u, std::max(s.cfg.bins, s.cfg.embed_bins));
    s.d_cb = cb_dst ? cb_dst : (float*)e.buf(t + "cb", (size_t)kLayerTypes * s.cb_stride * 4);
    s.lb_stride = pow2_ceil(s.cb_stride);
    s.parts = (uint8_t*)e.buf(t + "parts", (size_t)L.Np / 4 + 16);
    s.d_lb = (float*)e.buf(t + "lb", (size_t)kLayerTypes * s.lb_stride * 4);
}

// level boundaries of every layer type's final codebook
static void stage_level_bounds(Engine& e, Stage& s) {
    { DQTG_SPAN(e, "level_bounds_kernel"); level_bounds_kernel<<<kLayerTypes, 64, s.cb_stride * 4 + 16, e.stream>>>(s.d_cb, (int)s.cb_stride, s.cb_len, s.d_lb, (int)s.lb_stride); }
    e.launched();
}

// pass A into gh_mag/gh_sens ([7][HS] each) for the given masks
// per_sm_cap: resident CTAs per SM at most (the sample pass: one -- a CTA's setup and
// histogram flush cost more than its handful of tiles)
static void stage_pass_a(Engine& e, const DevCkpt& c, const PassIn& a, uint32_t mask_mag,
                         uint32_t mask_sens, unsigned long long* gh_mag,
                         unsigned long long* gh_sens, int per_sm_cap = 8) {
    const int ntiles = a.ntiles;
    cudaStream_t st = e.stream;
    DQTG_CUDA(cudaMemsetAsync(a.tile_ctr, 0, 4, st));
    const size_t ct = a.tab.ctab ? ((size_t)a.tab.ctab_n + 1) * 4 : 0;  // + sentinel
    if (c.explicit_scores) {
        const size_t smem = (size_t)2 * kWinSlots * 4 + ct;
        const int grid = stream_grid(e, ntiles, std::min(3, per_sm_cap));
        ensure_dyn_smem((const void*)pass_a_kernel<true>, smem);
        { DQTG_SPAN(e, "pass_a_kernel"); pass_a_kernel<true><<<grid, kPB, smem, st>>>(a, gh_mag, gh_sens, mask_mag, mask_sens); }
    } else {
        const size_t smem = (size_t)2 * kPosSlots * 4 + ct;
        ensure_dyn_smem((const void*)pass_a_kernel<false>, smem);
        const int grid = stream_grid(e, ntiles, std::min(5, per_sm_cap));
        DQTG_CUDA(cudaFuncSetAttribute(pass_a_kernel<false>,
                                       cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        { DQTG_SPAN(e, "pass_a_kernel"); pass_a_kernel<false><<<grid, kPB, smem, st>>>(a, gh_mag, gh_sens, mask_mag, mask_sens); }
    }
    e.launched();
}

static void stage_thresholds(Engine& e, Stage& s, int64_t HS, const AlphaTables& T,
                             unsigned long long* gh_mag, unsigned long long* gh_sens,
                             LtParams* lp_out = nullptr, int* slot_out = nullptr) {
    cudaStream_t st = e.stream;
    if (!lp_out) lp_out = s.d_lp;
    DQTG_CUDA(cudaMemcpyAsync(lp_out, s.plan.lp, sizeof(s.plan.lp), cudaMemcpyHostToDevice, st));
    if (s.plan.jobs.empty()) return;
    for (auto& j : s.plan.jobs) {
        bool sens_hist = (j.which == 1) || (j.which == 2 && s.cfg.metric == 1);
        j.hist = (sens_hist ? gh_sens : gh_mag) + (size_t)j.lt * HS;
    }
    QJob* d_jobs = (QJob*)e.buf(s.tag + "jobs", sizeof(QJob) * s.plan.jobs.size());
    DQTG_CUDA(cudaMemcpyAsync(d_jobs, s.plan.jobs.data(), sizeof(QJob) * s.plan.jobs.size(),
                              cudaMemcpyHostToDevice, st));
    { DQTG_SPAN(e, "quantile_kernel"); quantile_kernel<<<(unsigned)s.plan.jobs.size(), 1024, 0, st>>>(d_jobs, HS, T.d_keyf, lp_out, slot_out); }
    e.launched();
}

static void stage_keys(Engine& e, const Layout& L, Stage& s, const AlphaTables& T) {
    const int64_t HS = T.HS;
    cudaStream_t st = e.stream;
    compact_keys(e, s.gh_val, HS, HS, T.d_key, s.cfg.sigma, kLayerTypes, s.pts, s.kc, s.kw, HS,
                 s.n_keys);
    s.h_tprot.resize(L.nt + 1);
    e.d2h(s.h_nkeys, s.n_keys, sizeof(s.h_nkeys));
    e.d2h(s.h_tprot.data(), s.tensor_prot, (L.nt + 1) * 8);
}

static void stage_pass_b(Engine& e, const DevCkpt& c, const PassIn& a, Stage& s,
                         const AlphaTables& T, bool keys = true) {
    const Layout& L = *c.L;
    const int ntiles = a.ntiles;
    const int64_t HS = T.HS;
    cudaStream_t st = e.stream;
    DQTG_CUDA(cudaMemsetAsync(s.gh_val, 0, (size_t)kLayerTypes * HS * 8, st));
    DQTG_CUDA(cudaMemsetAsync(s.tensor_prot, 0, (size_t)(L.nt + 1) * 8, st));
    DQTG_CUDA(cudaMemsetAsync(a.tile_ctr, 0, 4, st));
    const size_t smem = (size_t)kWinSlots * 4;
    int grid = stream_grid(e, ntiles, 6);
    DQTG_CUDA(cudaFuncSetAttribute(pass_b_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    DQTG_CUDA(cudaFuncSetAttribute(pass_b_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    if (ntiles) {
        if (c.explicit_scores)
            { DQTG_SPAN(e, "pass_b_kernel"); pass_b_kernel<true><<<grid, kPB, smem, st>>>(a, s.d_lp, s.gh_val, s.tile_prot, s.tensor_prot, s.parts); }
        else
            { DQTG_SPAN(e, "pass_b_kernel"); pass_b_kernel<false><<<grid, kPB, smem, st>>>(a, s.d_lp, s.gh_val, s.tile_prot, s.tensor_prot, s.parts); }
        e.launched();
    }
    { DQTG_SPAN(e, "scan_u32_kernel"); scan_u32_kernel<<<1, 1024, 0, st>>>(s.tile_prot, ntiles, s.tile_off); }
    e.launched();
    if (keys) stage_keys(e, L, s, T);
}

// Fused pass A+B (pass_ab_kernel) for derived scores without pruning.
// Opt-in (DQTG_FUSED_AB=1): it reads w + EMA once instead of twice, but at C2 the
// fused kernel runs at 0.97 ms against 0.39 + 0.36 ms for passes A and B (issue-
// and latency-bound at 3 resident CTAs per SM; pipelined chain 164 vs 188 GB/s).
static bool fusable(const DevCkpt& c, const Stage& s) {
    if (c.explicit_scores || c.L->sample_tiles.empty() || !getenv("DQTG_FUSED_AB")) return false;
    for (int lt = 0; lt < kLayerTypes; ++lt)
        if (s.plan.lp[lt].flags & (kDoPrune | kProtectAll)) return false;
    for (const QJob& j : s.plan.jobs)
        if (j.which == 2) return false;
    return true;
}

// Everything pass A, the thresholds and pass B produce, from one streaming pass over
// w + EMA; *flag_host (valid after the next sync) non-zero: a guessed threshold was
// too far off and pass B must run.
static void stage_fused_ab(Engine& e, const DevCkpt& c, const PassIn& a, Stage& s,
                           const AlphaTables& T, uint32_t* flag_host) {
    const Layout& L = *c.L;
    const int64_t HS = T.HS;
    cudaStream_t st = e.stream;
    const size_t hb = (size_t)kLayerTypes * HS * 8;
    // 1. threshold guess: the quantiles of a thinned tile sample
    auto* samp = (unsigned long long*)e.buf("q.samp", 2 * hb);
    DQTG_CUDA(cudaMemsetAsync(samp, 0, 2 * hb, st));
    PassIn as = a;
    as.tiles = L.d_sample;
    as.ntiles = (int)L.sample_tiles.size();
    stage_pass_a(e, c, as, s.plan.mask_mag, s.plan.mask_sens, samp, samp + (size_t)kLayerTypes * HS, 1);
    auto* d_lpg = (LtParams*)e.buf("q.lpg", sizeof(LtParams) * kLayerTypes);
    auto* slots = (int*)e.buf("q.slots", 2 * kLayerTypes * 3 * sizeof(int));
    DQTG_CUDA(cudaMemsetAsync(slots, 0xff, 2 * kLayerTypes * 3 * sizeof(int), st));
    stage_thresholds(e, s, HS, T, samp, samp + (size_t)kLayerTypes * HS, d_lpg, slots);
    auto* band = (float4*)e.buf("q.band", sizeof(float4) * kLayerTypes);
    auto* bslots = (int2*)e.buf("q.bslots", sizeof(int2) * kLayerTypes);
    const char* shift_env = getenv("DQTG_FUSED_GUESS_SHIFT");
    const int shift = shift_env ? atoi(shift_env) : 0;
    { DQTG_SPAN(e, "band_kernel"); band_kernel<<<1, 32, 0, st>>>(slots, T.d_keyf, T.NB, HS, band, bslots, d_lpg, shift); }
    // 2. the fused streaming pass
    auto* gh_w = (unsigned long long*)e.buf("q.gh_w", hb);
    auto* gh = (unsigned long long*)e.buf("q.gh_scores", 2 * hb);  // [magnitude][sensitivity]
    auto* prot = (unsigned long long*)e.buf("q.prot", hb);
    auto* small = (unsigned long long*)e.buf("q.fsmall", 32);
    const unsigned long long cap = L.N / 25 + 1024;  // 4 % of the elements
    auto* cand = (unsigned long long*)e.buf("q.cand", cap * 8);
    DQTG_CUDA(cudaMemsetAsync(gh_w, 0, hb, st));
    DQTG_CUDA(cudaMemsetAsync(gh, 0, 2 * hb, st));
    DQTG_CUDA(cudaMemsetAsync(prot, 0, hb, st));
    DQTG_CUDA(cudaMemsetAsync(s.tensor_prot, 0, (size_t)(L.nt + 1) * 8, st));
    DQTG_CUDA(cudaMemsetAsync(small, 0, 32, st));
    DQTG_CUDA(cudaMemsetAsync(a.tile_ctr, 0, 4, st));
    FuseArgs f{d_lpg, band, gh_w, gh + (size_t)kLayerTypes * HS, prot, s.parts, s.tile_prot,
               s.tensor_prot, cand, small, cap, (uint32_t*)(small + 1)};
    const size_t ct = a.tab.ctab ? ((size_t)a.tab.ctab_n + 1) * 4 : 0;
    const size_t smem = (size_t)(kWinSlots + kPosSlots) * 4 + ct;
    ensure_dyn_smem((const void*)pass_ab_kernel, smem);
    DQTG_CUDA(cudaFuncSetAttribute(pass_ab_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int per_sm = 0;
    DQTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pass_ab_kernel, kPB, smem));
    const int grid = stream_grid(e, a.ntiles, std::max(1, per_sm));
    { DQTG_SPAN(e, "pass_ab_kernel"); pass_ab_kernel<<<grid, kPB, smem, st>>>(a, f); }
    { DQTG_SPAN(e, "fold_abs_kernel"); fold_abs_kernel<<<dim3((unsigned)((HS + 255) / 256), kLayerTypes), 256, 0, st>>>(gh_w, gh, HS, T.NB); }
    // 3. exact thresholds, band check, corrections, value histogram
    stage_thresholds(e, s, HS, T, gh, gh + (size_t)kLayerTypes * HS, s.d_lp, slots + kLayerTypes * 3);
    { DQTG_SPAN(e, "band_check_kernel"); band_check_kernel<<<1, 32, 0, st>>>(slots + kLayerTypes * 3, bslots, T.NB, small, cap, f.flag); }
    { DQTG_SPAN(e, "fixup_kernel"); fixup_kernel<<<e.num_sms * 4, 256, 0, st>>>(a, f, s.d_lp); }
    { DQTG_SPAN(e, "value_hist_kernel"); value_hist_kernel<<<e.num_sms, 256, 0, st>>>(gh_w, prot, s.gh_val, (int64_t)kLayerTypes * HS); }
    e.launched(6);
    { DQTG_SPAN(e, "scan_u32_kernel"); scan_u32_kernel<<<1, 1024, 0, st>>>(s.tile_prot, a.ntiles, s.tile_off); }
    e.launched();
    stage_keys(e, L, s, T);
    e.d2h(flag_host, f.flag, 4);
}

// Pass A2 + candidate classification (see pass_a2_kernel) for the fused step: fills
// s.gh_val, s.tile_prot / tile_off / tensor_prot, s.d_lp and the protected bitmap.
// *flag_host (valid after the next sync) non-zero: fall back to pass B.
static bool a2_eligible(const DevCkpt& c, const Stage& s) {
    if (c.explicit_scores || c.L->sample_tiles.empty() || getenv("DQTG_NO_PASS_A2")) return false;
    for (int lt = 0; lt < kLayerTypes; ++lt)
        if (s.plan.lp[lt].flags & (kDoPrune | kProtectAll)) return false;
    for (const QJob& j : s.plan.jobs)
        if (j.which == 2) return false;
    return true;
}

static void stage_pass_a2(Engine& e, const DevCkpt& c, const PassIn& a, Stage& s,
                          const AlphaTables& T, uint32_t* pbits, uint32_t* flag_host) {
    const Layout& L = *c.L;
    const int64_t HS = T.HS;
    cudaStream_t st = e.stream;
    const size_t hb = (size_t)kLayerTypes * HS * 8;
    // 1. threshold guess: the quantiles of a thinned tile sample
    auto* samp = (unsigned long long*)e.buf("q.samp", 2 * hb);
    DQTG_CUDA(cudaMemsetAsync(samp, 0, 2 * hb, st));
    PassIn as = a;
    as.tiles = L.d_sample;
    as.ntiles = (int)L.sample_tiles.size();
    stage_pass_a(e, c, as, s.plan.mask_mag, s.plan.mask_sens, samp, samp + (size_t)kLayerTypes * HS, 1);
    auto* d_lpg = (LtParams*)e.buf("q.lpg", sizeof(LtParams) * kLayerTypes);
    auto* slots = (int*)e.buf("q.slots", 2 * kLayerTypes * 3 * sizeof(int));
    DQTG_CUDA(cudaMemsetAsync(slots, 0xff, 2 * kLayerTypes * 3 * sizeof(int), st));
    stage_thresholds(e, s, HS, T, samp, samp + (size_t)kLayerTypes * HS, d_lpg, slots);
    auto* lo = (float2*)e.buf("q.clo", sizeof(float2) * kLayerTypes);
    auto* lo_slot = (int2*)e.buf("q.closlot", sizeof(int2) * kLayerTypes);
    const char* sh_env = getenv("DQTG_A2_BOUND_SHIFT");
    { DQTG_SPAN(e, "cand_bounds_kernel"); cand_bounds_kernel<<<1, 32, 0, st>>>(slots, T.d_keyf, T.NB, HS, lo, lo_slot, sh_env ? atoi(sh_env) : 0); }
    // 2. the streaming pass
    auto* gh_w = (unsigned long long*)e.buf("q.gh_w", hb);
    auto* gh = (unsigned long long*)e.buf("q.gh_scores", 2 * hb);  // [magnitude][sensitivity]
    auto* prot = (unsigned long long*)e.buf("q.prot", hb);
    auto* small = (unsigned long long*)e.buf("q.a2small", 32);
    const unsigned long long cap = L.N / 16 + 4096;  // 6 % of the elements
    auto* cand = (uint4*)e.buf("q.cand2", cap * 16);
    DQTG_CUDA(cudaMemsetAsync(gh_w, 0, hb, st));
    DQTG_CUDA(cudaMemsetAsync(gh + (size_t)kLayerTypes * HS, 0, hb, st));
    DQTG_CUDA(cudaMemsetAsync(prot, 0, hb, st));
    DQTG_CUDA(cudaMemsetAsync(small, 0, 32, st));
    DQTG_CUDA(cudaMemsetAsync(a.tile_ctr, 0, 4, st));
    A2Args f{lo, lo_slot, gh_w, gh + (size_t)kLayerTypes * HS, cand, small, cap};
    const size_t ct = a.tab.ctab ? ((size_t)a.tab.ctab_n + 1) * 4 : 0;
    const size_t smem = (size_t)(kWinSlots + kPosSlots) * 4 + ct;
    if (getenv("DQTG_A2_REGS")) {  // the register-staged variant
        ensure_dyn_smem((const void*)pass_a2_kernel, smem);
        DQTG_CUDA(cudaFuncSetAttribute(pass_a2_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        DQTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pass_a2_kernel, kPB, smem));
        { DQTG_SPAN(e, "pass_a2_kernel"); pass_a2_kernel<<<stream_grid(e, a.ntiles, std::max(1, per_sm)), kPB, smem, st>>>(a, f); }
    } else {
        const size_t smem2 = 2 * sizeof(A2Stage) + smem;
        ensure_dyn_smem((const void*)pass_a2_tma_kernel, smem2);
        DQTG_CUDA(cudaFuncSetAttribute(pass_a2_tma_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        DQTG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pass_a2_tma_kernel, kPB, smem2));
        { DQTG_SPAN(e, "pass_a2_kernel"); pass_a2_tma_kernel<<<stream_grid(e, a.ntiles, std::max(1, per_sm)), kPB, smem2, st>>>(a, f); }
    }
    { DQTG_SPAN(e, "fold_abs_kernel"); fold_abs_kernel<<<dim3((unsigned)((HS + 255) / 256), kLayerTypes), 256, 0, st>>>(gh_w, gh, HS, T.NB); }
    if (c.has_sens) {  // the sensitivity histograms pass A2 left to the candidates
        LtCounts tot{};
        for (uint32_t i = 0; i < L.nt; ++i) tot.n[L.types[i]] += L.numel[i];
        { DQTG_SPAN(e, "sens_from_cand_kernel"); sens_from_cand_kernel<<<e.num_sms * 2, 256, 0, st>>>(a, cand, small, cap, lo_slot, gh + (size_t)kLayerTypes * HS); }
        { DQTG_SPAN(e, "sens_lump_kernel"); sens_lump_kernel<<<kLayerTypes, 256, 0, st>>>(lo_slot, gh + (size_t)kLayerTypes * HS, HS, tot); }
        e.launched(2);
    }
    // 3. exact thresholds, bound check, classification, value histogram
    stage_thresholds(e, s, HS, T, gh, gh + (size_t)kLayerTypes * HS, s.d_lp, slots + kLayerTypes * 3);
    auto* flag = (uint32_t*)(small + 1);
    { DQTG_SPAN(e, "cand_check_kernel"); cand_check_kernel<<<1, 32, 0, st>>>(slots + kLayerTypes * 3, lo_slot, small, cap, flag); }
    DQTG_CUDA(cudaMemsetAsync(pbits, 0, (L.Np + 31) / 32 * 4, st));
    DQTG_CUDA(cudaMemsetAsync(s.tile_prot, 0, (size_t)a.ntiles * 4 + 4, st));
    DQTG_CUDA(cudaMemsetAsync(s.tensor_prot, 0, (size_t)(L.nt + 1) * 8, st));
    { DQTG_SPAN(e, "cand_classify_kernel"); cand_classify_kernel<<<e.num_sms * 4, 256, 0, st>>>(a, cand, small, cap, s.d_lp, pbits, s.tile_prot, s.tensor_prot, prot); }
    if (L.nt) { DQTG_SPAN(e, "tensor_sum_kernel"); tensor_sum_kernel<<<L.nt, 256, 0, st>>>(s.tile_prot, L.d_tile0, s.tensor_prot); }
    { DQTG_SPAN(e, "value_hist_kernel"); value_hist_kernel<<<e.num_sms, 256, 0, st>>>(gh_w, prot, s.gh_val, (int64_t)kLayerTypes * HS); }
    { DQTG_SPAN(e, "scan_u32_kernel"); scan_u32_kernel<<<1, 1024, 0, st>>>(s.tile_prot, a.ntiles, s.tile_off); }
    e.launched(8);
    stage_keys(e, L, s, T);
    e.d2h(flag_host, flag, 4);
    if (getenv("DQTG_A2_TRACE")) {
        unsigned long long nc = 0;
        e.d2h(&nc, small, 8);
        e.sync();
        fprintf(stderr, "pass A2: %llu candidates (%.2f %% of %llu), flag %u\n", nc,
                100.0 * (double)nc / (double)std::max<uint64_t>(1, L.N), (unsigned long long)L.N, *flag_host);
    }
}

// After a sync: codebooks of every stage (all k-means problems in one launch).
static void stage_codebooks(Engine& e, std::vector<Stage*>& stages, const PassIn& a,
                            int64_t HS) {
    std::vector<KProblem> probs;
    std::vector<std::pair<Stage*, int>> slots;
    for (Stage* s : stages) {
        DQTG_CUDA(cudaMemsetAsync(s->cb_len, 0, kLayerTypes * 4, e.stream));
        for (int lt = 0; lt < kLayerTypes; ++lt) {
            if (s->h_nkeys[lt] == 0) continue;  // no QUANTIZE values: empty codebook
            DQTG_REQUIRE(s->cfg.sigma >= 0.0 && s->cfg.sigma <= 1.0, DQTG_ERROR,
                         "sigma must be in [0, 1]");
            const uint32_t k = lt == kEmbedding ? s->cfg.embed_bins : s->cfg.bins;
            const uint64_t seed = mix_seed(s->seed, (uint64_t)lt);  // quantize.cpp:393
            if ((uint32_t)s->h_nkeys[lt] < k) {
                PassIn aa = a;
                aa.metric = (int)s->cfg.metric;
                distinct_value_codebook(e, aa, s->d_lp, lt, k, s->cfg, seed, s->d_cb,
                                        (int)s->cb_stride, s->cb_len);
                continue;
            }
            KProblem p{};
            p.pts = s->pts + (size_t)lt * HS;
            p.w = s->kw + (size_t)lt * HS;
            p.n = s->h_nkeys[lt];
            p.k = (int)k;
            p.seed = seed;
            p.slot = (int)slots.size();
            probs.push_back(p);
            slots.push_back({s, lt});
        }
    }
    if (probs.empty()) return;
    // all problems write to a staging codebook array, then scatter to their stages
    int stride = 1;
    for (auto& p : probs) stride = std::max(stride, p.k);
    float* cb_all = (float*)e.buf("km.cb_all", probs.size() * stride * 4);
    uint32_t* len_all = (uint32_t*)e.buf("km.len_all", probs.size() * 4);
    run_kmeans(e, probs, cb_all, stride, len_all);
    for (size_t i = 0; i < slots.size(); ++i) {
        Stage* s = slots[i].first;
        int lt = slots[i].second;
        DQTG_CUDA(cudaMemcpyAsync(s->d_cb + (size_t)lt * s->cb_stride, cb_all + i * stride,
                                  (size_t)probs[i].k * 4, cudaMemcpyDeviceToDevice, e.stream));
        DQTG_CUDA(cudaMemcpyAsync(s->cb_len + lt, len_all + i, 4, cudaMemcpyDeviceToDevice,
                                  e.stream));
    }
}

static void stage_pass_c(Engine& e, const DevCkpt& c, const PassIn& a, Stage& s, QState& q) {
    const int ntiles = a.ntiles;
    cudaStream_t st = e.stream;
    stage_level_bounds(e, s);
    const size_t smem = (size_t)s.lb_stride * 4 + 16;
    // the partition comes from pass B's 2-bit codes: w is the only stream read here
    { DQTG_SPAN(e, "pass_c_kernel"); pass_c_kernel<false, true><<<ntiles, kPB, smem, st>>>(a, s.d_lp, s.d_lb, (int)s.lb_stride, s.cb_len, s.tile_off, q.d_levels, q.d_ppos, q.d_pval, s.parts); }
    e.launched();
    DQTG_CUDA(cudaGetLastError());
}

// Pass C of a deferred quantize (FuseC) as its own kernel, for a caller that could
// not fuse it after all.
void run_pass_c(Engine& e, const DevCkpt& c, const FuseC& f, QState& q) {
    const Layout& L = *c.L;
    DQTG_REQUIRE(f.parts, DQTG_ERROR, "deferred pass C without partition codes");
    PassIn a{};
    a.tiles = L.d_tiles;
    a.ntiles = (int)L.tiles.size();
    a.types = L.d_types;
    a.tensor_off = L.d_off;
    a.w = f.w;
    a.err = e.d_err;
    if (!a.ntiles) return;
    const size_t smem = (size_t)f.lb_stride * 4 + 16;
    { DQTG_SPAN(e, "pass_c_kernel"); pass_c_kernel<false, true><<<a.ntiles, kPB, smem, e.stream>>>(a, f.lp, f.lb, f.lb_stride, f.cb_len, f.tile_prot_off, q.d_levels, q.d_ppos, q.d_pval, f.parts); }
    e.launched();
    DQTG_CUDA(cudaGetLastError());
}

std::unique_ptr<QState> quantize(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                                 uint64_t seed, uint64_t step, FuseC* defer) {
    const Layout& L = *c.L;
    Stage s;
    s.tag = "q.";
    s.cfg = cfg;
    s.seed = seed;
    quantize_plan(L, cfg, c.has_sens, s.plan);
    auto q = std::make_unique<QState>();
    q->eng = &e;
    q->L = c.L;
    q->step = step;
    q->cfg = cfg;
    q->cb_stride = std::max(1u, std::max(cfg.bins, cfg.embed_bins));
    q->d_levels = (decltype(q->d_levels))e.dalloc(L.Np * 2);
    q->d_cb = (decltype(q->d_cb))e.dalloc((size_t)kLayerTypes * q->cb_stride * 4);
    q->prot_count.assign(L.nt, 0);
    q->prot_off.assign(L.nt + 1, 0);
    if (L.N == 0) {
        DQTG_CUDA(cudaMemsetAsync(q->d_levels, 0, L.Np * 2, e.stream));
        q->d_ppos = (decltype(q->d_ppos))e.dalloc(8);
        q->d_pval = (decltype(q->d_pval))e.dalloc(8);
        return q;
    }
    DQTG_REQUIRE(cfg.alpha > 0.0 && cfg.alpha < 1.0, DQTG_ALPHA_OUT_OF_RANGE,
                 "alpha must be in (0, 1)");
    AlphaTables& T = e.alpha_tables(cfg.alpha);
    const int64_t HS = T.HS;
    PassIn a = pass_in(e, c, T, (int)cfg.metric);
    stage_alloc(e, L, HS, s, q->d_cb);
    uint32_t* pbits = nullptr;
    if (defer && !s.plan.jobs.empty() && a2_eligible(c, s)) {
        // fused step: pass A2 + candidates instead of pass B (partition as a bitmap)
        uint32_t redo = 0;
        pbits = (uint32_t*)e.buf("q.pbits", (L.Np + 31) / 32 * 4 + 16);
        stage_pass_a2(e, c, a, s, T, pbits, &redo);
        e.check_err();  // syncs: n_keys + protected counts + the bound flag on the host
        if (redo) {  // an exact threshold below its candidate bound: passes A + B
            // (the sensitivity histograms of pass A2 were rebuilt above the bounds only,
            // so the exact thresholds come from a full pass A)
            pbits = nullptr;
            auto* gh = (unsigned long long*)e.buf("q.gh_scores", (size_t)2 * kLayerTypes * HS * 8);
            DQTG_CUDA(cudaMemsetAsync(gh, 0, (size_t)2 * kLayerTypes * HS * 8, e.stream));
            stage_pass_a(e, c, a, s.plan.mask_mag, s.plan.mask_sens, gh, gh + (size_t)kLayerTypes * HS);
            stage_thresholds(e, s, HS, T, gh, gh + (size_t)kLayerTypes * HS);
            stage_pass_b(e, c, a, s, T);
            e.check_err();
        }
    } else if (fusable(c, s) && !s.plan.jobs.empty()) {
        uint32_t redo = 0;
        stage_fused_ab(e, c, a, s, T, &redo);
        e.check_err();  // syncs: n_keys + protected counts + the band flag on the host
        if (redo) {     // a guessed threshold outside its band: pass B with the exact ones
            stage_pass_b(e, c, a, s, T);
            e.check_err();
        }
    } else {
        unsigned long long *gh_mag = nullptr, *gh_sens = nullptr;
        if (!s.plan.jobs.empty()) {
            auto* gh = (unsigned long long*)e.buf("q.gh_scores", (size_t)2 * kLayerTypes * HS * 8);
            DQTG_CUDA(cudaMemsetAsync(gh, 0, (size_t)2 * kLayerTypes * HS * 8, e.stream));
            gh_mag = gh;
            gh_sens = gh + (size_t)kLayerTypes * HS;
            stage_pass_a(e, c, a, s.plan.mask_mag, s.plan.mask_sens, gh_mag, gh_sens);
        }
        stage_thresholds(e, s, HS, T, gh_mag, gh_sens);
        stage_pass_b(e, c, a, s, T);
        e.check_err();  // syncs: n_keys + protected counts on the host
    }
    std::vector<Stage*> v{&s};
    stage_codebooks(e, v, a, HS);
    uint64_t acc = 0;
    for (uint32_t i = 0; i < L.nt; ++i) {
        q->prot_off[i] = acc;
        q->prot_count[i] = s.h_tprot[i];
        acc += s.h_tprot[i];
    }
    q->prot_off[L.nt] = acc;
    q->prot_total = acc;
    q->d_ppos = (decltype(q->d_ppos))e.dalloc((acc + 1) * 8);
    q->d_pval = (decltype(q->d_pval))e.dalloc((acc + 1) * 2);
    if (defer) {  // pass C runs inside the DELTA encoder (codec.cu, FuseC)
        stage_level_bounds(e, s);
        defer->w = c.w;
        defer->parts = pbits ? nullptr : s.parts;
        defer->pbits = pbits;
        defer->lb = s.d_lb;
        defer->lb_stride = (int)s.lb_stride;
        defer->cb_len = s.cb_len;
        defer->tile_prot_off = s.tile_off;
        defer->lp = s.d_lp;
    } else {
        stage_pass_c(e, c, a, s, *q);
    }
    std::vector<float> hcb((size_t)kLayerTypes * q->cb_stride);
    e.d2h(q->cb_len, s.cb_len, sizeof(q->cb_len));
    e.d2h(hcb.data(), q->d_cb, hcb.size() * 4);
    e.check_err();
    for (int lt = 0; lt < kLayerTypes; ++lt)
        q->cb[lt].assign(hcb.begin() + (size_t)lt * q->cb_stride,
                         hcb.begin() + (size_t)lt * q->cb_stride + q->cb_len[lt]);
    return q;
}

// ---- sharded quantization: the two histogram exchange points -----------------
// stage 1: score histograms [2][7][HS] (magnitude, sensitivity) of this shard
// stage 2: thresholds from the globally reduced score histograms, pass B ->
//          value histograms [7][HS] of this shard
// stage 3: codebooks from the globally reduced value histograms (identical on
//          every rank), pass C -> this shard's quantized state
uint64_t shard_hist_len(Engine& e, const dqtg_config& cfg, int which) {
    AlphaTables& T = e.alpha_tables(cfg.alpha);
    return (uint64_t)(which == 0 ? 2 : 1) * kLayerTypes * (uint64_t)T.HS;
}

void shard_stage1(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                  unsigned long long* score_hist) {
    QuantPlan plan;
    quantize_plan(*c.L, cfg, c.has_sens, plan);
    AlphaTables& T = e.alpha_tables(cfg.alpha);
    DQTG_CUDA(cudaMemsetAsync(score_hist, 0, (size_t)2 * kLayerTypes * T.HS * 8, e.stream));
    if (c.L->N == 0 || plan.jobs.empty()) return;
    PassIn a = pass_in(e, c, T, (int)cfg.metric);
    stage_pass_a(e, c, a, plan.mask_mag, plan.mask_sens, score_hist,
                 score_hist + (size_t)kLayerTypes * T.HS);
}

void shard_stage2(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                  const unsigned long long* score_hist, unsigned long long* value_hist) {
    const Layout& L = *c.L;
    auto s = std::make_unique<Stage>();
    char tag[40];
    snprintf(tag, sizeof(tag), "sh%p.", (const void*)&c);
    s->tag = tag;
    s->cfg = cfg;
    quantize_plan(L, cfg, c.has_sens, s->plan);
    AlphaTables& T = e.alpha_tables(cfg.alpha);
    stage_alloc(e, L, T.HS, *s, nullptr);
    s->gh_val = value_hist;
    stage_thresholds(e, *s, T.HS, T, const_cast<unsigned long long*>(score_hist),
                     const_cast<unsigned long long*>(score_hist) + (size_t)kLayerTypes * T.HS);
    PassIn a = pass_in(e, c, T, (int)cfg.metric);
    stage_pass_b(e, c, a, *s, T, false);
    e.pending[&c] = std::shared_ptr<void>(s.release(), [](void* p) { delete (Stage*)p; });
}

std::unique_ptr<QState> shard_stage3(Engine& e, const DevCkpt& c, const dqtg_config& cfg,
                                     uint64_t seed, uint64_t step,
                                     const unsigned long long* value_hist) {
    auto pit = e.pending.find(&c);
    DQTG_REQUIRE(pit != e.pending.end(), DQTG_ERROR, "quantize stage 3 without stage 2");
    std::shared_ptr<void> keep = pit->second;
    Stage& s = *(Stage*)keep.get();
    const Layout& L = *c.L;
    AlphaTables& T = e.alpha_tables(cfg.alpha);
    s.gh_val = const_cast<unsigned long long*>(value_hist);
    s.seed = seed;
    stage_keys(e, L, s, T);
    auto q = std::make_unique<QState>();
    q->eng = &e;
    q->L = c.L;
    q->step = step;
    q->cfg = cfg;
    q->cb_stride = s.cb_stride;
    q->d_levels = (uint16_t*)e.dalloc(L.Np * 2);
    q->d_cb = (float*)e.dalloc((size_t)kLayerTypes * q->cb_stride * 4);
    e.check_err();
    for (int lt = 0; lt < kLayerTypes; ++lt) {
        const uint32_t k = lt == kEmbedding ? cfg.embed_bins : cfg.bins;
        DQTG_REQUIRE(s.h_nkeys[lt] == 0 || (uint32_t)s.h_nkeys[lt] >= k, DQTG_ERROR,
                     "distinct-value codebook fallback needs all shards' values (unsupported "
                     "when sharded): layer type " + std::to_string(lt) + " has " +
                         std::to_string(s.h_nkeys[lt]) + " distinct keys for " + std::to_string(k) +
                         " bins");
    }
    std::vector<Stage*> v{&s};
    PassIn a = pass_in(e, c, T, (int)cfg.metric);
    s.d_cb = q->d_cb;
    stage_codebooks(e, v, a, T.HS);
    q->prot_count.assign(L.nt, 0);
    q->prot_off.assign(L.nt + 1, 0);
    uint64_t acc = 0;
    for (uint32_t i = 0; i < L.nt; ++i) {
        q->prot_off[i] = acc;
        q->prot_count[i] = s.h_tprot[i];
        acc += s.h_tprot[i];
    }
    q->prot_off[L.nt] = q->prot_total = acc;
    q->d_ppos = (uint64_t*)e.dalloc((acc + 1) * 8);
    q->d_pval = (uint16_t*)e.dalloc((acc + 1) * 2);
    if (L.N) stage_pass_c(e, c, a, s, *q);
    std::vector<float> hcb((size_t)kLayerTypes * q->cb_stride);
    e.d2h(q->cb_len, s.cb_len, sizeof(q->cb_len));
    e.d2h(hcb.data(), q->d_cb, hcb.size() * 4);
    e.check_err();
    for (int lt = 0; lt < kLayerTypes; ++lt)
        q->cb[lt].assign(hcb.begin() + (size_t)lt * q->cb_stride,
                         hcb.begin() + (size_t)lt * q->cb_stride + q->cb_len[lt]);
    e.pending.erase(&c);
    e.drop_scratch(s.tag);  // this shard's stage buffers (partition codes, histograms)
    return q;
}

void partition(Engine& e, const DevCkpt& c, const dqtg_config& cfg, uint8_t* const* masks) {
    const Layout& L = *c.L;
    Stage s;
    s.tag = "p.";
    s.cfg = cfg;
    quantize_plan(L, cfg, c.has_sens, s.plan);
    if (L.N == 0) return;
    AlphaTables* T = nullptr;
    if (!s.plan.jobs.empty()) T = &e.alpha_tables(cfg.alpha);
    else T = &e.alpha_tables(cfg.alpha > 0.0 && cfg.alpha < 1.0 ? cfg.alpha : 0.01);
    const int64_t HS = T->HS;
    PassIn a = pass_in(e, c, *T, (int)cfg.metric);
    s.d_lp = (LtParams*)e.buf("p.lp", sizeof(LtParams) * kLayerTypes);
    unsigned long long *gh_mag = nullptr, *gh_sens = nullptr;
    if (!s.plan.jobs.empty()) {
        auto* gh = (unsigned long long*)e.buf("q.gh_scores", (size_t)2 * kLayerTypes * HS * 8);
        DQTG_CUDA(cudaMemsetAsync(gh, 0, (size_t)2 * kLayerTypes * HS * 8, e.stream));
        gh_mag = gh;
        gh_sens = gh + (size_t)kLayerTypes * HS;
        stage_pass_a(e, c, a, s.plan.mask_mag, s.plan.mask_sens, gh_mag, gh_sens);
    }
    stage_thresholds(e, s, HS, *T, gh_mag, gh_sens);
    uint8_t* d_mask = (uint8_t*)e.buf("p.mask", L.Np + 16);
    if (c.explicit_scores)
        { DQTG_SPAN(e, "mask_kernel"); mask_kernel<true><<<a.ntiles, kPB, 0, e.stream>>>(a, s.d_lp, d_mask); }
    else
        { DQTG_SPAN(e, "mask_kernel"); mask_kernel<false><<<a.ntiles, kPB, 0, e.stream>>>(a, s.d_lp, d_mask); }
    e.launched();
    for (uint32_t i = 0; i < L.nt; ++i)
        if (L.numel[i]) e.from_device(masks[i], d_mask + L.off[i], L.numel[i]);
    e.check_err();
}

// proxy_quality_delta + estimate_compression from device partial sums (search.cpp:30-85)
static double quality_from(const Layout& L, const double* diff, const double* orig) {
    uint64_t count[kLayerTypes] = {0}, total = 0;
    for (uint32_t i = 0; i < L.nt; ++i) count[L.types[i]] += L.numel[i];
    for (int lt = 0; lt < kLayerTypes; ++lt) total += count[lt];
    if (total == 0) return 0.0;
    double q = 0.0;
    for (int lt = 0; lt < kLayerTypes; ++lt) {
        if (!count[lt]) continue;
        double rel = orig[lt] > 0.0 ? std::sqrt(diff[lt] / orig[lt]) : (diff[lt] > 0.0 ? 1.0 : 0.0);
        q += (double(count[lt]) / double(total)) * rel;
    }
    return q;
}

double estimate_from_counts(const Layout& L, const uint64_t* counts, int lstride,
                            const uint32_t* cb_len, const uint64_t* nprot) {
    double raw = 4.0 * double(L.N);
    double est = 64.0;
    for (uint32_t i = 0; i < L.nt; ++i) {
        const uint32_t levels = cb_len[L.types[i]] + 2;
        const double n = double(L.numel[i]);
        double bits = 0.0;
        for (uint32_t l = 0; l < levels && (int)l < lstride; ++l) {
            uint64_t c = counts[(size_t)i * lstride + l];
            if (!c) continue;
            double p = double(c) / n;
            bits -= double(c) * std::log2(p);
        }
        est += bits / 8.0;
        est += 10.0 * double(nprot[i]);
    }
    for (int lt = 0; lt < kLayerTypes; ++lt) est += 4.0 * double(cb_len[lt]);
    return raw / est;
}

// Partition key of a config: candidates with equal keys share pass B.
static bool same_partition(const dqtg_config& x, const dqtg_config& y) {
    return memcmp(&x.alpha, &y.alpha, 8) == 0 && memcmp(&x.prune_frac, &y.prune_frac, 8) == 0 &&
           memcmp(&x.protect_frac, &y.protect_frac, 8) == 0 && x.metric == y.metric;
}

void eval_batch(Engine& e, const DevCkpt& c, const dqtg_config* cfgs, const uint64_t* seeds,
                uint32_t m, double* quality, double* est) {
    const Layout& L = *c.L;
    if (!m) return;
    const int ntiles = (int)L.tiles.size();
    cudaStream_t st = e.stream;
    // sum of squares of the original weights per layer type (config independent)
    auto* tile_v = (double*)e.buf("ev.tile_v", (size_t)ntiles * 8 + 8);
    auto* d_lt = (double*)e.buf("ev.lt", 16 * 8);
    double orig[kLayerTypes] = {0};
    if (ntiles) {
        { DQTG_SPAN(e, "tile_sq_kernel"); tile_sq_kernel<<<ntiles, kPB, 0, st>>>(L.d_tiles, c.w, nullptr, tile_v); }
        { DQTG_SPAN(e, "lt_sum_kernel"); lt_sum_kernel<<<1, 512, 0, st>>>(L.d_tiles, L.d_types, ntiles, tile_v, d_lt); }
        e.launched(2);
        e.d2h(orig, d_lt, sizeof(orig));
    }
    std::vector<std::unique_ptr<Stage>> stages(m);
    std::map<uint64_t, std::pair<unsigned long long*, unsigned long long*>> scores_by_alpha;
    int lstride = 2;
    for (uint32_t i = 0; i < m; ++i) lstride = std::max<int>(lstride, std::max(cfgs[i].bins, cfgs[i].embed_bins) + 2);
    DQTG_REQUIRE(lstride <= 4098, DQTG_ERROR, "eval_batch supports up to 4096 bins");
    for (uint32_t i = 0; i < m; ++i) {
        auto s = std::make_unique<Stage>();
        s->tag = "ev" + std::to_string(i) + ".";
        s->cfg = cfgs[i];
        s->seed = seeds[i];
        quantize_plan(L, cfgs[i], c.has_sens, s->plan);
        stages[i] = std::move(s);
    }
    if (L.N == 0) {
        for (uint32_t i = 0; i < m; ++i) quality[i] = 0.0, est[i] = 0.0;
        return;
    }
    // partition groups: the first candidate of each key runs pass B for all of them
    std::vector<int> leader(m, -1);
    std::vector<std::vector<uint32_t>> groups;
    for (uint32_t i = 0; i < m; ++i) {
        for (size_t g = 0; g < groups.size() && leader[i] < 0; ++g)
            if (same_partition(cfgs[groups[g][0]], cfgs[i])) {
                leader[i] = (int)groups[g][0];
                groups[g].push_back(i);
            }
        if (leader[i] < 0) {
            leader[i] = (int)i;
            groups.push_back({i});
        }
    }
    for (uint32_t i = 0; i < m; ++i) {
        Stage& s = *stages[i];
        DQTG_REQUIRE(s.cfg.alpha > 0.0 && s.cfg.alpha < 1.0, DQTG_ALPHA_OUT_OF_RANGE,
                     "alpha must be in (0, 1)");
        AlphaTables& T = e.alpha_tables(s.cfg.alpha);
        stage_alloc(e, L, T.HS, s, nullptr);
        if (leader[i] != (int)i) {  // shares the leader's partition, value histogram, counts
            Stage& ld = *stages[leader[i]];
            s.d_lp = ld.d_lp;
            s.gh_val = ld.gh_val;
            s.tensor_prot = ld.tensor_prot;
            s.tile_prot = ld.tile_prot;
            s.tile_off = ld.tile_off;
            s.parts = ld.parts;
            stage_keys(e, L, s, T);  // keys + weights with this candidate's sigma
            continue;
        }
        // pass A once per alpha, all layer types, both score kinds
        uint64_t key;
        memcpy(&key, &s.cfg.alpha, 8);
        auto it = scores_by_alpha.find(key);
        if (it == scores_by_alpha.end()) {
            auto* gh = (unsigned long long*)e.buf("ev.gh_scores" + std::to_string(scores_by_alpha.size()),
                                                  (size_t)2 * kLayerTypes * T.HS * 8);
            DQTG_CUDA(cudaMemsetAsync(gh, 0, (size_t)2 * kLayerTypes * T.HS * 8, st));
            PassIn a = pass_in(e, c, T, 0);
            stage_pass_a(e, c, a, 0x7f, c.has_sens ? 0x7f : 0, gh, gh + (size_t)kLayerTypes * T.HS);
            it = scores_by_alpha.emplace(key, std::make_pair(gh, gh + (size_t)kLayerTypes * T.HS)).first;
        }
        stage_thresholds(e, s, T.HS, T, it->second.first, it->second.second);
        PassIn a = pass_in(e, c, T, (int)s.cfg.metric);
        stage_pass_b(e, c, a, s, T);
    }
    e.check_err();
    {
        // codebooks: problems of configs sharing an alpha go together
        std::map<uint64_t, std::vector<Stage*>> by_alpha;
        for (auto& sp : stages) {
            uint64_t key;
            memcpy(&key, &sp->cfg.alpha, 8);
            by_alpha[key].push_back(sp.get());
        }
        for (auto& kv : by_alpha) {
            AlphaTables& T = e.alpha_tables(kv.second[0]->cfg.alpha);
            PassIn aa = pass_in(e, c, T, 0);
            stage_codebooks(e, kv.second, aa, T.HS);
        }
    }
    // evaluation: kEvalM candidates of one partition group per read of w
    auto* counts = (unsigned long long*)e.buf("ev.counts", (size_t)kEvalM * L.nt * lstride * 8 + 8);
    auto* tdiff = (double*)e.buf("ev.tdiff", (size_t)kEvalM * ntiles * 8 + 8);
    auto* d_ltm = (double*)e.buf("ev.ltm", (size_t)kEvalM * kLayerTypes * 8);
    std::vector<uint64_t> hcounts((size_t)kEvalM * L.nt * lstride);
    for (const auto& grp : groups) {
        for (size_t g0 = 0; g0 < grp.size(); g0 += kEvalM) {
            const int mm = (int)std::min<size_t>(kEvalM, grp.size() - g0);
            uint32_t cbs = 1, lbs = 1;
            for (int j = 0; j < mm; ++j) {
                Stage& s = *stages[grp[g0 + j]];
                stage_level_bounds(e, s);
                cbs = std::max(cbs, s.cb_stride);
                lbs = std::max(lbs, s.lb_stride);
            }
            auto* mcb = (float*)e.buf("ev.mcb", (size_t)kEvalM * kLayerTypes * cbs * 4);
            auto* mlb = (float*)e.buf("ev.mlb", (size_t)kEvalM * kLayerTypes * lbs * 4);
            auto* mlen = (uint32_t*)e.buf("ev.mlen", (size_t)kEvalM * kLayerTypes * 4);
            for (int j = 0; j < mm; ++j) {
                Stage& s = *stages[grp[g0 + j]];
                DQTG_CUDA(cudaMemcpy2DAsync(mcb + (size_t)j * kLayerTypes * cbs, cbs * 4, s.d_cb,
                                            s.cb_stride * 4, s.cb_stride * 4, kLayerTypes,
                                            cudaMemcpyDeviceToDevice, st));
                DQTG_CUDA(cudaMemcpy2DAsync(mlb + (size_t)j * kLayerTypes * lbs, lbs * 4, s.d_lb,
                                            s.lb_stride * 4, s.lb_stride * 4, kLayerTypes,
                                            cudaMemcpyDeviceToDevice, st));
                DQTG_CUDA(cudaMemcpyAsync(mlen + j * kLayerTypes, s.cb_len, kLayerTypes * 4,
                                          cudaMemcpyDeviceToDevice, st));
            }
            DQTG_CUDA(cudaMemsetAsync(counts, 0, (size_t)mm * L.nt * lstride * 8, st));
            Stage& s0 = *stages[grp[g0]];
            AlphaTables& T = e.alpha_tables(s0.cfg.alpha);
            PassIn a = pass_in(e, c, T, (int)s0.cfg.metric);
            EvalMulti ev{mm, mcb, (int)cbs, mlb, (int)lbs, mlen, tdiff, counts, lstride, ntiles, (int)L.nt};
            const size_t smem = (size_t)mm * (cbs + lbs) * 4 + 16;
            if (c.explicit_scores)
                { DQTG_SPAN(e, "eval_multi_kernel"); eval_multi_kernel<true><<<ntiles, kPB, smem, st>>>(a, s0.d_lp, ev); }
            else
                { DQTG_SPAN(e, "eval_multi_kernel"); eval_multi_kernel<false><<<ntiles, kPB, smem, st>>>(a, s0.d_lp, ev); }
            { DQTG_SPAN(e, "lt_sum_multi_kernel"); lt_sum_multi_kernel<<<mm, 512, 0, st>>>(L.d_tiles, L.d_types, ntiles, tdiff, d_ltm); }
            e.launched(2);
            std::vector<double> diff((size_t)mm * kLayerTypes);
            std::vector<uint32_t> cbl((size_t)mm * kLayerTypes);
            e.d2h(diff.data(), d_ltm, diff.size() * 8);
            e.d2h(cbl.data(), mlen, cbl.size() * 4);
            e.d2h(hcounts.data(), counts, (size_t)mm * L.nt * lstride * 8);
            e.check_err();
            for (int j = 0; j < mm; ++j) {
                const uint32_t i = grp[g0 + j];
                Stage& s = *stages[i];
                quality[i] = quality_from(L, diff.data() + (size_t)j * kLayerTypes, orig);
                std::vector<uint64_t> np(L.nt);
                for (uint32_t t = 0; t < L.nt; ++t) np[t] = s.h_tprot[t];
                est[i] = estimate_from_counts(L, hcounts.data() + (size_t)j * L.nt * lstride, lstride,
                                              cbl.data() + (size_t)j * kLayerTypes, np.data());
            }
        }
    }
}

double proxy_quality(Engine& e, const DevCkpt& orig, const float* recon_dev) {
    const Layout& L = *orig.L;
    const int ntiles = (int)L.tiles.size();
    double o[kLayerTypes] = {0}, d[kLayerTypes] = {0};
    if (ntiles) {
        auto* tile_v = (double*)e.buf("pq.tile_v", (size_t)ntiles * 8 + 8);
        auto* d_lt = (double*)e.buf("pq.lt", 16 * 8);
        { DQTG_SPAN(e, "tile_sq_kernel"); tile_sq_kernel<<<ntiles, kPB, 0, e.stream>>>(L.d_tiles, orig.w, nullptr, tile_v); }
        { DQTG_SPAN(e, "lt_sum_kernel"); lt_sum_kernel<<<1, 512, 0, e.stream>>>(L.d_tiles, L.d_types, ntiles, tile_v, d_lt); }
        e.d2h(o, d_lt, sizeof(o));
        e.sync();
        { DQTG_SPAN(e, "tile_sq_kernel"); tile_sq_kernel<<<ntiles, kPB, 0, e.stream>>>(L.d_tiles, orig.w, recon_dev, tile_v); }
        { DQTG_SPAN(e, "lt_sum_kernel"); lt_sum_kernel<<<1, 512, 0, e.stream>>>(L.d_tiles, L.d_types, ntiles, tile_v, d_lt); }
        e.d2h(d, d_lt, sizeof(d));
        e.launched(4);
        e.sync();
    }
    return quality_from(L, d, o);
}

void level_counts(Engine& e, const QState& q, uint64_t* counts, int lstride) {
    const Layout& L = *q.L;
    auto* d = (unsigned long long*)e.buf("lc.counts", (size_t)L.nt * lstride * 8 + 8);
    DQTG_CUDA(cudaMemsetAsync(d, 0, (size_t)L.nt * lstride * 8, e.stream));
    if (!L.tiles.empty()) {
        DQTG_REQUIRE(lstride <= 1024, DQTG_ERROR, "too many levels for level_counts");
        { DQTG_SPAN(e, "level_count_kernel"); level_count_kernel<<<(unsigned)L.tiles.size(), 256, 0, e.stream>>>(L.d_tiles, q.d_levels, d, lstride); }
        e.launched();
    }
    e.from_device(counts, d, (size_t)L.nt * lstride * 8);
    e.sync();
}

// ---- state equality (round-trip checks without a host copy) ------------------------
__global__ void levels_diff_kernel(const Tile* tiles, const uint16_t* a, const uint16_t* b,
                                   unsigned int* diff) {
    const Tile T = tiles[blockIdx.x];
    bool d = false;
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x) d |= a[T.start + i] != b[T.start + i];
    if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(diff, 1u);
}
__global__ void words_diff_kernel(const uint8_t* a, const uint8_t* b, uint64_t n, unsigned int* diff) {
    bool d = false;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        d |= a[i] != b[i];
    if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(diff, 1u);
}

bool states_equal(Engine& e, const QState& a, const QState& b) {
    const Layout &LA = *a.L, &LB = *b.L;
    if (!LA.same_shape(LB) || a.step != b.step || a.prot_total != b.prot_total) return false;
    for (uint32_t i = 0; i < LA.nt; ++i)
        if (a.prot_count[i] != b.prot_count[i]) return false;
    for (int lt = 0; lt < kLayerTypes; ++lt)
        if (a.cb_len[lt] != b.cb_len[lt] || a.cb[lt] != b.cb[lt]) return false;
    auto* d = (unsigned int*)e.buf("eq.diff", 16);
    DQTG_CUDA(cudaMemsetAsync(d, 0, 4, e.stream));
    if (!LA.tiles.empty()) {
        { DQTG_SPAN(e, "levels_diff_kernel"); levels_diff_kernel<<<(unsigned)LA.tiles.size(), 256, 0, e.stream>>>(LA.d_tiles, a.d_levels, b.d_levels, d); }
        e.launched();
    }
    const uint64_t np = a.prot_total;
    if (np) {
        const unsigned g = (unsigned)std::min<uint64_t>((uint64_t)e.num_sms * 4, (np * 8 + 255) / 256);
        words_diff_kernel<<<g, 256, 0, e.stream>>>((const uint8_t*)a.d_ppos, (const uint8_t*)b.d_ppos, np * 8, d);
        words_diff_kernel<<<g, 256, 0, e.stream>>>((const uint8_t*)a.d_pval, (const uint8_t*)b.d_pval, np * 2, d);
        e.launched(2);
    }
    unsigned int h = 0;
    e.d2h(&h, d, 4);
    e.check_err();
    return h == 0;
}

// dequantize_checkpoint into device memory: outs[t] = tensor t's output (a device
// array of nt pointers).  No host synchronisation: errors surface at the next check.
void dequantize_to(Engine& e, const QState& q, float* const* outs_dev) {
    const Layout& L = *q.L;
    const int ntiles = (int)L.tiles.size();
    for (uint32_t t = 0; t < L.nt; ++t)  // a tensor without tiles references no entries
        DQTG_REQUIRE(L.numel[t] || !q.prot_count[t], DQTG_CORRUPT_INDEX, "unreferenced protected entries");
    if (!ntiles) return;
    auto* lo_hi = (unsigned long long*)e.buf("dq.lohi", (size_t)ntiles * 16 + 16);
    auto* poff = (unsigned long long*)e.buf("dq.poff", (size_t)(L.nt + 1) * 8);
    auto* cb_len_d = (uint32_t*)e.buf("dq.cblen", kLayerTypes * 4);
    std::vector<unsigned long long> po(q.prot_off.begin(), q.prot_off.end());
    po.resize(L.nt + 1, q.prot_total);
    e.to_device(poff, po.data(), po.size() * 8);
    e.to_device(cb_len_d, q.cb_len, sizeof(q.cb_len));
    { DQTG_SPAN(e, "prot_tile_range_kernel"); prot_tile_range_kernel<<<(ntiles + 255) / 256, 256, 0, e.stream>>>(
        L.d_tiles, ntiles, L.d_off, L.d_tile0, poff, q.d_ppos, lo_hi, e.d_err); }
    { DQTG_SPAN(e, "dequant_kernel"); dequant_kernel<<<ntiles, 256, 0, e.stream>>>(L.d_tiles, L.d_types, L.d_off, q.d_cb,
                                                 (int)q.cb_stride, cb_len_d, q.d_levels, lo_hi,
                                                 q.d_ppos, q.d_pval, outs_dev, e.d_err); }
    e.launched(2);
    DQTG_CUDA(cudaGetLastError());
}

void dequantize(Engine& e, const QState& q, float* out_dev) {  // padded contiguous output
    const Layout& L = *q.L;
    std::vector<float*> ptrs(L.nt);
    for (uint32_t t = 0; t < L.nt; ++t) ptrs[t] = out_dev + L.off[t];
    auto* d = (float**)e.buf("dq.outs", (size_t)L.nt * 8 + 8);
    e.to_device(d, ptrs.data(), (size_t)L.nt * 8);
    dequantize_to(e, q, d);
}

void scan_tiles(Engine& e, const uint32_t* in, int n, unsigned long long* out) {
    { DQTG_SPAN(e, "scan_u32_kernel"); scan_u32_kernel<<<1, 1024, 0, e.stream>>>(in, n, out); }
    e.launched();
}

}  // namespace dqtg
