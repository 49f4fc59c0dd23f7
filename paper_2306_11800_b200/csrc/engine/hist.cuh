// Exact log-bucket histogram device functions (sketch.cpp:21-31, 131-148).
#pragma once

#include "engine.h"

namespace dqtg {

// Smallest k with U(k) >= a (a = bits of |x|, a >= zbits, finite).  The float
// log2 estimate is within one bucket; integer compares against the boundary
// table make the result exact.
__device__ __forceinline__ int bucket_of(uint32_t a, const BucketTab& t) {
    if (t.cell) {  // one cell lookup (AlphaTables::d_cell)
        const uint2 c = __ldg(t.cell + (a >> t.cell_shift));
        return (int)c.x + (a > c.y ? 1 : 0);
    }
    const int kmin = (int)t.kmin, kmax = (int)t.kmax;
    float lg = __log2f(__uint_as_float(a));
    int k = (int)ceilf(lg * t.inv_log2_gamma);
    k = k < kmin ? kmin : (k > kmax ? kmax : k);
    // U(k) lives at U[k - kmin + 1]; both bounds are fetched together (independent
    // loads), the estimate is almost always exact or one off
    const uint32_t lo = __ldg(t.U + (k - kmin)), hi = __ldg(t.U + (k - kmin + 1));
    if (lo >= a && k > kmin) {
        --k;
        while (k > kmin && __ldg(t.U + (k - kmin)) >= a) --k;
    } else if (hi < a) {
        ++k;
        while (__ldg(t.U + (k - kmin + 1)) < a) ++k;
    }
    return k;
}

// Signed slot index of a finite float (ascending value order):
// neg k -> kmax-k, zero -> NB, pos k -> NB+1+k-kmin.
__device__ __forceinline__ int64_t slot_of(float v, const BucketTab& t) {
    uint32_t b = __float_as_uint(v), a = b & 0x7fffffffu;
    if (a < t.zbits) return t.NB;
    int k = bucket_of(a, t);
    return (b >> 31) ? (t.kmax - k) : (t.NB + 1 + k - t.kmin);
}

// Adds v to a shared-memory window histogram (sh[kWinSlots]) with spill to the
// global u64 histogram gh[HS] for buckets outside the window.
// Slow path of the slot-table adds: outside the window or non-finite.
__device__ __forceinline__ void hist_spill(unsigned long long* gh, float v, const BucketTab& t,
                                        uint32_t* err) {
    const uint32_t b = __float_as_uint(v), a = b & 0x7fffffffu;
    if (a >= 0x7f800000u) {
        atomicOr(err, kErrNonFinite);
        return;
    }
    const int k = bucket_of(a, t);
    atomicAdd(gh + ((b >> 31) ? (t.kmax - k) : (t.NB + 1 + k - t.kmin)), 1ull);
}

// Window slot p of |x| from the slot table (0 zero, 1..kWin window, else spill/bad).
__device__ __forceinline__ uint32_t slot_of_abs(uint32_t a, const BucketTab& t) {
    const uint2 c = __ldg(t.slot + (a >> t.cell_shift));
    return (a > c.y) ? (c.x >> 16) : (c.x & 0xffffu);
}

// Window slot of |x| from the compact table staged in shared memory (s_ctab), or
// kSlotSpill when |x| is outside [2^-32, 1) or the cell needs the exact path.
__device__ __forceinline__ uint32_t slot_shared(uint32_t a, const BucketTab& t, const uint32_t* s_ctab) {
    const uint32_t rel = (a >> t.cell_shift) - t.ctab_lo;
    if (rel >= t.ctab_n) return kSlotSpill;
    const uint32_t c = s_ctab[rel];
    const uint32_t off = a & ((1u << t.cell_shift) - 1u);
    const bool hi = off > ((c >> 13) & 0x1ffffu);
    const bool special = hi ? ((c >> 30) & 1u) : (c >> 31);
    return special ? kSlotSpill : (c & 0x1fffu) + (hi ? 1u : 0u);
}

__device__ __forceinline__ void hist_add(uint32_t* sh, unsigned long long* gh, float v,
                                         const BucketTab& t, uint32_t* err);

// hist_add / hist_add_pos with the shared compact table first
__device__ __forceinline__ void hist_add_s(uint32_t* sh, unsigned long long* gh, float v,
                                           const BucketTab& t, uint32_t* err, const uint32_t* s_ctab) {
    const uint32_t b = __float_as_uint(v);
    const uint32_t p = slot_shared(b & 0x7fffffffu, t, s_ctab);
    if (p <= (uint32_t)kWin) atomicAdd(sh + ((b >> 31) ? kWin - p : kWin + p), 1u);
    else hist_add(sh, gh, v, t, err);
}

__device__ __forceinline__ void hist_add(uint32_t* sh, unsigned long long* gh, float v,
                                         const BucketTab& t, uint32_t* err) {
    uint32_t b = __float_as_uint(v), a = b & 0x7fffffffu;
    if (t.slot) {  // one table load; signed window: neg kWin - p, zero kWin, pos kWin + p
        const uint32_t p = slot_of_abs(a, t);
        if (p <= (uint32_t)kWin) atomicAdd(sh + ((b >> 31) ? kWin - p : kWin + p), 1u);
        else hist_spill(gh, v, t, err);
        return;
    }
    if (a >= 0x7f800000u) {
        atomicOr(err, kErrNonFinite);
        return;
    }
    if (a < t.zbits) {  // |x| < 1e-12 (sketch.hpp:24), incl. -0.0
        atomicAdd(sh + kWin, 1u);
        return;
    }
    int k = bucket_of(a, t);
    int d = k - (int)t.kw_lo;
    bool neg = b >> 31;
    if ((unsigned)d < (unsigned)kWin)
        atomicAdd(sh + (neg ? kWin - 1 - d : kWin + 1 + d), 1u);
    else
        atomicAdd(gh + (neg ? (t.kmax - k) : (t.NB + 1 + k - t.kmin)), 1ull);
}

// Drains the window into gh and clears it.  Call between __syncthreads().
__device__ __forceinline__ void hist_flush(uint32_t* sh, unsigned long long* gh,
                                           const BucketTab& t) {
    for (int w = threadIdx.x; w < kWinSlots; w += blockDim.x) {
        uint32_t c = sh[w];
        if (!c) continue;
        sh[w] = 0;
        int64_t idx;
        if (w < kWin) {
            int64_t k = t.kw_lo + kWin - 1 - w;
            idx = t.kmax - k;
        } else if (w == kWin) {
            idx = t.NB;
        } else {
            int64_t k = t.kw_lo + (w - kWin - 1);
            idx = t.NB + 1 + k - t.kmin;
        }
        atomicAdd(gh + idx, (unsigned long long)c);
    }
}

// Non-negative inputs (derived scores |w|, |e*w|): a window of the zero bucket +
// kWin positive buckets (half the shared memory of the signed window).
constexpr int kPosSlots = kWin + 1;

__device__ __forceinline__ void hist_add_pos(uint32_t* sh, unsigned long long* gh, float v,
                                             const BucketTab& t, uint32_t* err) {
    const uint32_t a = __float_as_uint(v);  // v >= +0 (fabs of a finite float) or NaN/Inf
    if (t.slot) {
        const uint32_t p = slot_of_abs(a, t);
        if (p <= (uint32_t)kWin) atomicAdd(sh + p, 1u);
        else hist_spill(gh, v, t, err);
        return;
    }
    if (a >= 0x7f800000u) {
        atomicOr(err, kErrNonFinite);
        return;
    }
    if (a < t.zbits) {
        atomicAdd(sh, 1u);
        return;
    }
    const int k = bucket_of(a, t);
    const int d = k - (int)t.kw_lo;
    if ((unsigned)d < (unsigned)kWin) atomicAdd(sh + 1 + d, 1u);
    else atomicAdd(gh + (t.NB + 1 + k - t.kmin), 1ull);
}

__device__ __forceinline__ void hist_add_pos_s(uint32_t* sh, unsigned long long* gh, float v,
                                               const BucketTab& t, uint32_t* err,
                                               const uint32_t* s_ctab) {
    const uint32_t p = slot_shared(__float_as_uint(v), t, s_ctab);
    if (p <= (uint32_t)kWin) atomicAdd(sh + p, 1u);
    else hist_add_pos(sh, gh, v, t, err);
}

// Branch-free insertion of a non-negative value into a positive window histogram
// through the shared compact table (shared-window addresses precomputed): returns
// false when the value needs the exact path (outside the table, special cell, NaN,
// outside the window) -- the caller batches those.  The table has a sentinel entry
// at index ctab_n with both special bits set, so the range check is a min().
struct FastPos {
    uint32_t shift, lo, n, offmask, ctab_s;
};
__device__ __forceinline__ FastPos fast_pos(const BucketTab& t, const uint32_t* s_ctab) {
    return FastPos{t.cell_shift, t.ctab_lo, t.ctab_n, (1u << t.cell_shift) - 1u,
                   (uint32_t)__cvta_generic_to_shared(s_ctab)};
}
__device__ __forceinline__ bool hist_fast_pos(uint32_t win_s, uint32_t b, const FastPos& f) {
    const uint32_t rel = min((b >> f.shift) - f.lo, f.n);
    uint32_t c;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(c) : "r"(f.ctab_s + 4 * rel));
    const uint32_t hi = (b & f.offmask) > ((c >> 13) & 0x1ffffu) ? 1u : 0u;
    const uint32_t p = (c & 0x1fffu) + hi;
    const bool ok = !((c >> (31 - hi)) & 1u) && p <= (uint32_t)kWin;
    if (ok) asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(win_s + 4 * p) : "memory");
    return ok;
}

__device__ __forceinline__ void hist_flush_pos(uint32_t* sh, unsigned long long* gh,
                                               const BucketTab& t) {
    for (int w = threadIdx.x; w < kPosSlots; w += blockDim.x) {
        uint32_t c = sh[w];
        if (!c) continue;
        sh[w] = 0;
        const int64_t idx = w == 0 ? t.NB : t.NB + 1 + (t.kw_lo + (w - 1)) - t.kmin;
        atomicAdd(gh + idx, (unsigned long long)c);
    }
}

__device__ __forceinline__ void hist_clear(uint32_t* sh) {
    for (int w = threadIdx.x; w < kWinSlots; w += blockDim.x) sh[w] = 0;
}

}  // namespace dqtg
