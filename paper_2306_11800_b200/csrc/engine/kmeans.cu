// Histogram k-means on the device (quantize.cpp:94-325): key compaction + mix
// weights, k-means++ seeding, Lloyd, loss and restart selection.  One CTA per
// (problem, restart); see kmeans.cuh for the exactness strategy.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include "engine.h"
#include "kmeans.cuh"
#include "kmeans_api.h"

namespace dqtg {

constexpr int kKB = 512;  // threads per k-means CTA

// ---- key compaction + mix_weights (quantize.cpp:263-279) --------------------
// One CTA per problem: hist[HS] (u64, signed-slot order = ascending value) ->
// pts/cnt/w (ascending keys), n_keys.
__global__ void __launch_bounds__(1024) compact_keys_kernel(const unsigned long long* hist,
                                                            int64_t hs_stride, int64_t HS,
                                                            const double* key, double sigma,
                                                            double* pts, unsigned long long* cnt,
                                                            double* w, int64_t out_stride,
                                                            int* n_keys) {
    __shared__ unsigned long long s_scan[33];
    __shared__ unsigned long long s_maxc;
    __shared__ double s_maxk;
    const int p = blockIdx.x;
    const unsigned long long* h = hist + p * hs_stride;
    double* P = pts + p * out_stride;
    unsigned long long* Cn = cnt + p * out_stride;
    double* W = w + p * out_stride;
    if (threadIdx.x == 0) {
        s_maxc = 1;
        s_maxk = 0.0;
    }
    __syncthreads();
    unsigned long long base = 0;
    unsigned long long lmaxc = 1;
    double lmaxk = 0.0;
    for (int64_t c0 = 0; c0 < HS; c0 += blockDim.x) {
        int64_t i = c0 + threadIdx.x;
        unsigned long long c = i < HS ? h[i] : 0ull;
        unsigned long long flag = c ? 1ull : 0ull, tot;
        unsigned long long pos = block_exclusive_scan<unsigned long long>(flag, s_scan, &tot);
        if (c) {
            double k = key[i];
            P[base + pos] = k;
            Cn[base + pos] = c;
            lmaxc = c > lmaxc ? c : lmaxc;
            lmaxk = fmax(lmaxk, fabs(k));
        }
        base += tot;
    }
    atomicMax(&s_maxc, lmaxc);
    // fmax of non-negative doubles == max of their bit patterns
    atomicMax((unsigned long long*)&s_maxk, (unsigned long long)__double_as_longlong(lmaxk));
    __syncthreads();
    const double maxc = (double)s_maxc, maxk = s_maxk;
    for (unsigned long long i = threadIdx.x; i < base; i += blockDim.x) {
        double nc = __ddiv_rn((double)Cn[i], maxc);
        double nx = maxk > 0.0 ? __ddiv_rn(fabs(P[i]), maxk) : 0.0;
        W[i] = __dadd_rn(__dmul_rn(sigma, nc), __dmul_rn(__dsub_rn(1.0, sigma), nx));
    }
    if (threadIdx.x == 0) n_keys[p] = (int)base;
}

// ---- per-restart CTA -----------------------------------------------------
struct KShared {
    Mt64 rng;
    const double2* wx;  // (w, x) pairs in shared memory, or null (working set in global)
    int in_smem;        // pts/w/d2/prob/pref live in shared memory
    int pick;
    int done;
    int any_empty;
    double scale;
    double red[kKB / 32];
};

// Explicit shared-memory accesses for the serial chains (generic loads add latency).
__device__ __forceinline__ unsigned sh_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
// volatile + memory clobber: the loads must not move across __syncthreads() or the
// stores that produced the data (a plain asm is a pure function to the compiler)
__device__ __forceinline__ double ld_sh(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(sh_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ double2 ld_sh2(const double2* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(sh_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_sh(double* p, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(sh_addr(p)), "d"(v) : "memory");
}

// Sequential fp64 sum s += v[i] for i in [a, n) in index order (the reference's
// order), optional running values out[i] (SH: both arrays in shared memory).
template <bool SH>
__device__ __forceinline__ double seq_prefix(const double* v, int a, int n, double s, double* out) {
    int i = a;
    for (; i + 16 <= n; i += 16) {
        double cv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) cv[u] = SH ? ld_sh(v + i + u) : v[i + u];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            s = __dadd_rn(s, cv[u]);
            if (out) {
                if (SH) st_sh(out + i + u, s);
                else out[i + u] = s;
            }
        }
    }
    for (; i < n; ++i) {
        s = __dadd_rn(s, SH ? ld_sh(v + i) : v[i]);
        if (out) {
            if (SH) st_sh(out + i, s);
            else out[i] = s;
        }
    }
    return s;
}

// quantize.cpp:116-131: sequential prefix of prob (lane 0), binary search for the
// first positive entry whose running sum reaches r.  u >= 0: the uniform draw was
// already taken (by kpp_pick_par, whose certificate failed).
__device__ int kpp_pick(const double* prob, double* pref, int n, int from, KShared& sm,
                        double u = -1.0) {
    if (threadIdx.x == 0) {
        // pref[0..from) are unchanged from the previous pick (same terms, same order)
        double s = from > 0 ? pref[from - 1] : 0.0;
        s = sm.in_smem ? seq_prefix<true>(prob, from, n, s, pref) : seq_prefix<false>(prob, from, n, s, pref);
        if (n > 0) s = pref[n - 1];
        int res;
        if (!(s > 0.0)) {
            res = n;
        } else {
            double r = __dmul_rn(u >= 0.0 ? u : uniform01(sm.rng), s);
            int lo = 0, hi = n;
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (pref[mid] >= r) hi = mid;
                else lo = mid + 1;
            }
            while (lo < n && !(prob[lo] > 0.0)) ++lo;
            if (lo == n) {  // no crossing: last positive entry (last_pos)
                lo = n - 1;
                while (lo >= 0 && !(prob[lo] > 0.0)) --lo;
                res = lo < 0 ? n : lo;
            } else {
                res = lo;
            }
        }
        sm.pick = res;
    }
    __syncthreads();
    return sm.pick;
}

// Block-wide exclusive scan of one double per thread; *total = block sum.
__device__ double block_exscan_d(double v, double* slots /* kKB / 32 */, double* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = __dadd_rn(x, y);
    }
    if (lane == 31) slots[wid] = x;
    __syncthreads();
    double base = 0.0, tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        const double s = slots[w];
        if (w < wid) base = __dadd_rn(base, s);
        tot = __dadd_rn(tot, s);
    }
    *total = tot;
    __syncthreads();  // slots reusable
    return __dadd_rn(base, __dsub_rn(x, v)) ;
}

// The same pick from a parallel prefix with a rounding certificate.  Every thread
// sums a contiguous chunk of prob, the chunk sums are scanned, and the crossing of
// r is searched in the parallel prefix P.  The reference's sequential prefix s_i
// and P_i both lie within eps * P_i of the exact prefix (non-negative terms: any
// summation order of m terms errs by at most (m - 1) u times their sum), and its
// r = fl(u * s_n) lies in [r_lo, r_hi]; the crossing index i is accepted only when
// s_{i-1} < r <= s_i holds for every admissible value (P_{i-1} (1 + eps) < r_lo,
// P_i (1 - eps) >= r_hi) -- the reference's index then provably equals i.  Returns
// -1 when the certificate fails (the caller runs kpp_pick with the same draw,
// passed back in *u_out), n when the total is zero (no draw, as the reference).
__device__ int kpp_pick_par(const double* prob, int n, KShared& sm, double* u_out) {
    __shared__ double s_slots[kKB / 32];
    __shared__ double s_r[4];  // r_mid, r_lo, r_hi, u
    __shared__ int s_idx;
    __shared__ double s_pp[2];
    const int nt = blockDim.x, tid = threadIdx.x;
    const int C = (n + nt - 1) / nt;
    const int a = min(n, tid * C), b = min(n, a + C);
    double loc = 0.0;
    for (int i = a; i < b; ++i) loc = __dadd_rn(loc, prob[i]);
    double T;
    const double base = block_exscan_d(loc, s_slots, &T);
    const double eps = 4.0 * (double)(n + 64) * 0x1.0p-53;
    if (tid == 0) {
        s_idx = 0x7fffffff;
        if (T > 0.0) {
            const double u = uniform01(sm.rng);
            const double tlo = __dmul_rd(T, __dsub_rd(1.0, eps)), thi = __dmul_ru(T, __dadd_ru(1.0, eps));
            s_r[0] = __dmul_rn(u, T);
            s_r[1] = __dmul_rd(u, tlo);
            s_r[2] = __dmul_ru(u, thi);
            s_r[3] = u;
        }
    }
    __syncthreads();
    if (!(T > 0.0)) return n;  // uniform across the block: T is the same everywhere
    const double rm = s_r[0];
    double run = base;
    int hit = -1;
    double pp = 0.0, pc = 0.0;
    for (int i = a; i < b; ++i) {
        const double nx = __dadd_rn(run, prob[i]);
        if (nx >= rm) {
            hit = i, pp = run, pc = nx;
            break;
        }
        run = nx;
    }
    if (hit >= 0) atomicMin(&s_idx, hit);
    __syncthreads();
    if (hit >= 0 && hit == s_idx) s_pp[0] = pp, s_pp[1] = pc;
    __syncthreads();
    if (tid == 0) {
        int res = -1;
        if (s_idx != 0x7fffffff) {
            const bool below = __dmul_ru(s_pp[0], __dadd_ru(1.0, eps)) < s_r[1];
            const bool above = __dmul_rd(s_pp[1], __dsub_rd(1.0, eps)) >= s_r[2];
            if (below && above) res = s_idx;
        }
        sm.pick = res;
    }
    __syncthreads();
    const int res = sm.pick;
    if (res < 0) *u_out = s_r[3];
    __syncthreads();
    return res;
}

__device__ double block_max_d(double v, KShared& sm) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = sm.red[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = fmax(m, sm.red[i]);
        sm.red[0] = m;
    }
    __syncthreads();
    double r = sm.red[0];
    __syncthreads();
    return r;
}

__device__ void kpp_init_fast(const double* pts, const double* w, int n, int k, double* d2,
                              double* prob, double* pref, double* chosen, KShared& sm);

// weighted_kmeanspp_init (quantize.cpp:94-164).
__device__ void kpp_init(const double* pts, const double* w, int n, int k, double* d2,
                         double* prob, double* pref, double* chosen, KShared& sm,
                         bool certify = true) {
    if (certify && n >= 64) {
        kpp_init_fast(pts, w, n, k, d2, prob, pref, chosen, sm);
        return;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        d2[i] = __longlong_as_double(0x7ff0000000000000LL);
        prob[i] = w[i];
    }
    __syncthreads();
    int nc = 0;
    while (nc < k) {
        // parallel pick with a certificate; the sequential one when it fails (rare)
        double u = -1.0;
        int next = certify && n >= 64 ? kpp_pick_par(prob, n, sm, &u) : -1;
        if (next < 0) next = kpp_pick(prob, pref, n, 0, sm, u);
        if (threadIdx.x == 0) {
            bool taken = false;
            if (next != n)
                for (int j = 0; j < nc; ++j) taken |= (chosen[j] == pts[next]);
            if (next == n || taken) {  // first unchosen point
                for (int i = 0; i < n; ++i) {
                    bool c2 = false;
                    for (int j = 0; j < nc; ++j) c2 |= (chosen[j] == pts[i]);
                    if (!c2) {
                        next = i;
                        break;
                    }
                }
            }
            chosen[nc] = pts[next];
        }
        __syncthreads();
        const double v = chosen[nc];
        const bool first = nc == 0;
        ++nc;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double dd = __dsub_rn(pts[i], v);
            double sq = __dmul_rn(dd, dd);
            double cur = d2[i];
            if (sq < cur || first) {  // std::min(d2, d*d)
                cur = sq < cur ? sq : cur;
                d2[i] = cur;
                prob[i] = __dmul_rn(w[i], cur);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) IntroSort<double, LessD>{}.sort(chosen, k);
    __syncthreads();
}

// kpp_init with the certified parallel pick, two block barriers per pick.  Every
// thread owns a contiguous chunk of keys for the whole seeding: it sums its chunk's
// prob, searches its chunk for the crossing and updates its chunk's d2 / prob after
// the pick, so no barrier separates the update from the next pick's sums.  The draw
// is taken speculatively before the total is known (thread 0) and given back when
// the total is zero (the reference draws only for a positive total; mt64_next
// reads mt[mti++] after an optional regeneration, so mti-- undoes it exactly).
// Each candidate crossing carries its own certificate in the atomicMin key (index
// << 1 | failed), so the smallest crossing and its verdict arrive together.  A
// certified pick has prob > 0 (d2 > 0), so it is never an already-chosen centre;
// a failed certificate or a zero total takes kpp_pick / the first-unchosen scan.
__device__ void kpp_init_fast(const double* pts, const double* w, int n, int k, double* d2,
                              double* prob, double* pref, double* chosen, KShared& sm) {
    __shared__ double s_slots[2][kKB / 32];
    __shared__ double s_u[2];
    __shared__ unsigned long long s_key[2];
    const int nt = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int C = (n + nt - 1) / nt;
    const int a = min(n, tid * C), b = min(n, a + C);
    for (int i = a; i < b; ++i) {
        d2[i] = __longlong_as_double(0x7ff0000000000000LL);
        prob[i] = w[i];
    }
    if (tid == 0) s_key[0] = s_key[1] = ~0ull;
    const double eps = 4.0 * (double)(n + 64) * 0x1.0p-53;
    for (int nc = 0; nc < k; ++nc) {
        const int par = nc & 1;
        if (tid == 0) s_u[par] = uniform01(sm.rng);
        double loc = 0.0;
        for (int i = a; i < b; ++i) loc = __dadd_rn(loc, prob[i]);
        double x = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x = __dadd_rn(x, y);
        }
        double ex = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) ex = 0.0;
        if (lane == 31) s_slots[par][wid] = x;
        __syncthreads();  // B1
        if (tid == 0) s_key[par ^ 1] = ~0ull;  // the previous pick's key is read by now
        double T = 0.0, base = 0.0;
        for (int q = 0; q < nt / 32; ++q) {
            const double sv = s_slots[par][q];
            if (q < wid) base = __dadd_rn(base, sv);
            T = __dadd_rn(T, sv);
        }
        base = __dadd_rn(base, ex);
        int next = -1;
        double u = -1.0;
        if (T > 0.0) {
            u = s_u[par];
            const double tlo = __dmul_rd(T, __dsub_rd(1.0, eps)), thi = __dmul_ru(T, __dadd_ru(1.0, eps));
            const double rm = __dmul_rn(u, T), rlo = __dmul_rd(u, tlo), rhi = __dmul_ru(u, thi);
            double run = base;
            for (int i = a; i < b; ++i) {
                const double nx = __dadd_rn(run, prob[i]);
                if (nx >= rm) {
                    const bool below = __dmul_ru(run, __dadd_ru(1.0, eps)) < rlo;
                    const bool above = __dmul_rd(nx, __dsub_rd(1.0, eps)) >= rhi;
                    atomicMin(&s_key[par], ((unsigned long long)i << 1) | ((below && above) ? 0ull : 1ull));
                    break;
                }
                run = nx;
            }
        } else if (tid == 0) {
            --sm.rng.mti;  // no draw for a zero total
        }
        __syncthreads();  // B2
        if (T > 0.0) {
            const unsigned long long key = s_key[par];
            if (key != ~0ull && !(key & 1ull)) next = (int)(key >> 1);
        }
        if (next < 0) {  // uncertain (or zero total): the reference's sequential pick
            next = kpp_pick(prob, pref, n, 0, sm, u);
            if (tid == 0) {
                bool taken = false;
                if (next != n)
                    for (int j = 0; j < nc; ++j) taken |= (chosen[j] == pts[next]);
                if (next == n || taken) {  // first unchosen point
                    for (int i = 0; i < n; ++i) {
                        bool c2 = false;
                        for (int j = 0; j < nc; ++j) c2 |= (chosen[j] == pts[i]);
                        if (!c2) {
                            next = i;
                            break;
                        }
                    }
                }
                sm.pick = next;
            }
            __syncthreads();
            next = sm.pick;
        }
        const double v = pts[next];
        if (tid == 0) chosen[nc] = v;
        const bool first = nc == 0;
        for (int i = a; i < b; ++i) {
            const double dd = __dsub_rn(pts[i], v);
            const double sq = __dmul_rn(dd, dd);
            double cur = d2[i];
            if (sq < cur || first) {  // std::min(d2, d*d)
                cur = sq < cur ? sq : cur;
                d2[i] = cur;
                prob[i] = __dmul_rn(w[i], cur);
            }
        }
    }
    __syncthreads();
    if (tid == 0) IntroSort<double, LessD>{}.sort(chosen, k);
    __syncthreads();
}

// optional phase timing per CTA (DQTG_KM_TIMING=1): clocks of kpp / lloyd / loss,
// iterations, n, k, Lloyd chain steps (max over lanes, summed), Lloyd sum clocks
__device__ long long g_km_timing[1024][12];

// Sequential (w, w*x) sums over keys [a, b] from 0 in key order (the reference's
// accumulation order).  wx: (w, x) pairs in shared memory (one 16-byte load per
// key) or null.
__device__ __forceinline__ void chain_sums(const double2* wx, const double* w, const double* x,
                                           int a, int b, double& ws, double& wxs) {
    int i = a;
    const int e = b + 1;
    if (wx) {
        for (; i + 8 <= e; i += 8) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = ld_sh2(wx + i + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                ws = __dadd_rn(ws, v[u].x);
                wxs = __dadd_rn(wxs, __dmul_rn(v[u].x, v[u].y));
            }
        }
        for (; i < e; ++i) {
            const double2 v = ld_sh2(wx + i);
            ws = __dadd_rn(ws, v.x);
            wxs = __dadd_rn(wxs, __dmul_rn(v.x, v.y));
        }
        return;
    }
    for (; i + 8 <= e; i += 8) {
        double wv[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) wv[u] = w[i + u], xv[u] = x[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            ws = __dadd_rn(ws, wv[u]);
            wxs = __dadd_rn(wxs, __dmul_rn(wv[u], xv[u]));
        }
    }
    for (; i < e; ++i) {
        const double wi = w[i];
        ws = __dadd_rn(ws, wi);
        wxs = __dadd_rn(wxs, __dmul_rn(wi, x[i]));
    }
}

// ---- certified Lloyd steps ------------------------------------------------------
// The reference's cluster sums (quantize.cpp:200-205) are sequential fp64 chains, one
// per cluster -- at C2 the cluster of the many near-zero keys is ~1100 keys long,
// and ~40 iterations of that chain were the whole k-means time.  A certified step
// sums every cluster in parallel instead and carries each centre as an interval
// [lo, hi] that provably contains the reference's value (any summation order of m
// terms errs by at most (m - 1) u sum|t|, so the sequential and the parallel sums
// differ by at most 2 (m - 1) u sum|t|; the quotient is bounded with directed
// rounding).  The step's decisions are accepted only when they hold for every value
// in the intervals:
//   * well-separated ascending centres (the contiguous-cluster condition),
//   * every cluster boundary: the first key with |x - c[j+1]| < |x - c[j]| is
//     monotone in both centres, so equal boundaries at the lower and the upper
//     interval ends fix it,
//   * no empty cluster, and the movement test (max |next - c| <= tol * scale).
// The clusters of a certified step are then exactly the reference's, so the next
// step's sums are over the same keys -- the interval does not compound.  When a
// decision is not certain, the centres are made exact from the previous step's
// clusters with the reference's sequential chains and the step runs exactly; the
// final centres are always made exact the same way.
// The pointers are per-thread values derived from the kernel's shared-memory carve
// (not loaded from a shared struct), so the compiler emits shared loads for them.
struct LAux {
    double *lo, *hi, *nlo, *nhi, *sw, *swx, *sax;
    int *pf, *pl;  // clusters (first, last key) that produced the current intervals
    int* pe;       // boundaries of the previous certified step (search hint), -1: none
    int* exact;    // (shared) lo == hi == c are the reference's values
};

// exact centres from the sequential chains over clusters [f[j], l[j]] (warp 0)
__device__ void lloyd_exact_from(const double* pts, const double* w, const int* f, const int* l,
                                 int k, double* c, KShared& sm) {
    if ((threadIdx.x >> 5) == 0)
        for (int j = threadIdx.x & 31; j < k; j += 32) {
            double ws = 0.0, wxs = 0.0;
            chain_sums(sm.wx, w, pts, f[j], l[j], ws, wxs);
            c[j] = __ddiv_rn(wxs, ws);
        }
}

// first key (exclusive end of cluster j) with |x - b| < |x - a|
__device__ __forceinline__ int lloyd_boundary(const double* pts, int n, double a, double b) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const double x = pts[mid];
        if (fabs(__dsub_rn(x, b)) < fabs(__dsub_rn(x, a))) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// One certified step.  Returns 0: converged, 1: continue (centres <- next
// intervals), 2: not certain (nothing changed; run the exact step).
__device__ int lloyd_interval_step(const double* pts, const double* w, int n, LAux& X,
                                   int* first, int* last, int* cnt, int k, double gap, double thr,
                                   KShared& sm) {
    __shared__ int s_res;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long t0 = clock64();
    if (wid == 0) {
        bool ok = true;
        for (int j = lane; j + 1 < k; j += 32) ok &= __dsub_rn(X.lo[j + 1], X.hi[j]) > gap;
        ok = __all_sync(0xffffffffu, ok);
        if (ok) {
            for (int j = lane; j < k; j += 32) {
                int e = n;
                if (j + 1 < k) {
                    // the previous step's boundary first (it rarely moves): the predicate
                    // is monotone in the key, so e is the boundary iff P(e-1) fails and P(e) holds
                    const double a = X.lo[j], b = X.lo[j + 1];
                    auto P = [&](int i) { return fabs(__dsub_rn(pts[i], b)) < fabs(__dsub_rn(pts[i], a)); };
                    const int g = X.pe ? X.pe[j] : -1;
                    if (g < 0 || g > n) {
                        e = lloyd_boundary(pts, n, a, b);
                    } else {  // galloping search outward from the hint, then bisection
                        auto first_true = [&](int lo, int hi) {  // P(hi) holds or hi == n
                            while (lo < hi) {
                                const int mid = (lo + hi) >> 1;
                                if (P(mid)) hi = mid;
                                else lo = mid + 1;
                            }
                            return lo;
                        };
                        if (g == n || P(g)) {
                            int hi = g, lo = g - 1, d = 2;
                            while (lo >= 0 && P(lo)) hi = lo, lo = hi - d, d <<= 1;
                            e = first_true(max(lo + 1, 0), hi);
                        } else {
                            int lo = g + 1, hi = g + 1, d = 2;
                            while (hi < n && !P(hi)) lo = hi + 1, hi = lo + d - 1, d <<= 1;
                            e = first_true(lo, min(hi, n));
                        }
                    }
                    if (!*X.exact) {  // the same boundary at the upper interval ends
                        const double ah = X.hi[j], bh = X.hi[j + 1];
                        auto Q = [&](int i) { return fabs(__dsub_rn(pts[i], bh)) < fabs(__dsub_rn(pts[i], ah)); };
                        if (!((e == 0 || !Q(e - 1)) && (e == n || Q(e)))) ok = false;
                    }
                    if (X.pe) X.pe[j] = e;
                }
                last[j] = e;  // exclusive end
            }
            __syncwarp();
            for (int j = lane; j < k; j += 32) first[j] = j ? last[j - 1] : 0;
            __syncwarp();
            for (int j = lane; j < k; j += 32) {
                cnt[j] = last[j] - first[j];
                ok &= cnt[j] > 0;  // an empty cluster: the exact step reseeds it
            }
            ok = __all_sync(0xffffffffu, ok);
        }
        if (lane == 0) s_res = ok ? 1 : 2;
    }
    __syncthreads();
    const long long t1 = clock64();
    if (s_res == 2) {
        __syncthreads();
        return 2;
    }
    // parallel cluster sums: one warp per cluster, lanes stride over its keys, then a
    // shuffle reduction (any order: the bound above covers every order)
    for (int j = wid; j < k; j += (int)(blockDim.x >> 5)) {
        double ws = 0.0, wxs = 0.0, ax = 0.0;
        const int e = last[j];
        double ws2 = 0.0, wxs2 = 0.0, ax2 = 0.0;  // two chains per lane
        int i = first[j] + lane;
        for (; i + 32 < e; i += 64) {
            const double wi = w[i], xi = pts[i], wj = w[i + 32], xj = pts[i + 32];
            const double ti = __dmul_rn(wi, xi), tj = __dmul_rn(wj, xj);
            ws = __dadd_rn(ws, wi);
            wxs = __dadd_rn(wxs, ti);
            ax = __dadd_rn(ax, fabs(ti));
            ws2 = __dadd_rn(ws2, wj);
            wxs2 = __dadd_rn(wxs2, tj);
            ax2 = __dadd_rn(ax2, fabs(tj));
        }
        if (i < e) {
            const double wi = w[i], tt = __dmul_rn(wi, pts[i]);
            ws = __dadd_rn(ws, wi);
            wxs = __dadd_rn(wxs, tt);
            ax = __dadd_rn(ax, fabs(tt));
        }
        ws = __dadd_rn(ws, ws2);
        wxs = __dadd_rn(wxs, wxs2);
        ax = __dadd_rn(ax, ax2);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ws = __dadd_rn(ws, __shfl_xor_sync(0xffffffffu, ws, o));
            wxs = __dadd_rn(wxs, __shfl_xor_sync(0xffffffffu, wxs, o));
            ax = __dadd_rn(ax, __shfl_xor_sync(0xffffffffu, ax, o));
        }
        if (lane == 0) X.sw[j] = ws, X.swx[j] = wxs, X.sax[j] = ax;
    }
    __syncthreads();
    const long long t2 = clock64();
    if (wid == 0) {
        bool ok = true;
        double U = 0.0, L = 0.0;
        for (int j = lane; j < k; j += 32) {
            const double ws = X.sw[j];
            if (!(ws > 0.0)) {  // all weights zero: an empty cluster
                ok = false;
                continue;
            }
            const double e = 4.0 * (double)(cnt[j] + 16) * 0x1.0p-53;
            const double e2 = __dmul_ru(e, 1.0 + 0x1.0p-20);
            const double wsl = __dmul_rd(ws, __dsub_rd(1.0, e)), wsh = __dmul_ru(ws, __dadd_ru(1.0, e));
            const double d = __dmul_ru(e2, X.sax[j]);
            const double wxl = __dsub_rd(X.swx[j], d), wxh = __dadd_ru(X.swx[j], d);
            // quotient bounds: round-to-nearest divisions widened by one ulp (cheaper
            // than directed division; |rn(q) - q| <= ulp(q) / 2)
            double ql, qh;
            if (wxl >= 0.0) ql = __ddiv_rn(wxl, wsh), qh = __ddiv_rn(wxh, wsl);
            else if (wxh <= 0.0) ql = __ddiv_rn(wxl, wsl), qh = __ddiv_rn(wxh, wsh);
            else ql = __ddiv_rn(wxl, wsl), qh = __ddiv_rn(wxh, wsl);
            ql = __dsub_rd(ql, __dmul_ru(fabs(ql), 0x1.0p-52));
            qh = __dadd_ru(qh, __dmul_ru(fabs(qh), 0x1.0p-52));
            X.nlo[j] = ql;
            X.nhi[j] = qh;
            // movement bounds of |next - c|
            const double dh = __dsub_ru(qh, X.lo[j]), dl = __dsub_rd(ql, X.hi[j]);
            U = fmax(U, fmax(fabs(dh), fabs(dl)));
            if (dl > 0.0) L = fmax(L, dl);
            else if (dh < 0.0) L = fmax(L, -dh);
        }
        ok = __all_sync(0xffffffffu, ok);
        for (int o = 16; o > 0; o >>= 1) {
            U = fmax(U, __shfl_xor_sync(0xffffffffu, U, o));
            L = fmax(L, __shfl_xor_sync(0xffffffffu, L, o));
        }
        int res = 2;
        if (ok) {
            if (U <= thr) res = 0;
            else if (L > thr) res = 1;
        }
        if (res != 2) {
            for (int j = lane; j < k; j += 32) {
                X.lo[j] = X.nlo[j];
                X.hi[j] = X.nhi[j];
                X.pf[j] = first[j];
                X.pl[j] = last[j] - 1;
            }
        }
        if (lane == 0) {
            s_res = res;
            if (res != 2) *X.exact = 0;
        }
    }
    __syncthreads();
    const int r = s_res;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        long long* g = g_km_timing[blockIdx.x];
        g[8] += t1 - t0, g[9] += t2 - t1, g[10] += clock64() - t2;
    }
    return r;
}

// weighted_lloyd (quantize.cpp:180-254); c (k centres) is updated in place.
// With aux (LAux, 7k doubles + 3k ints), steps are certified interval steps
// whenever their decisions are certain (above); the others run exactly:
// iterations whose centres are strictly ascending and well separated (the fast
// path: clusters are contiguous key ranges) run on warp 0 alone with warp
// primitives, one lane per cluster chain.  The general assignment and the
// empty-cluster reseed use the whole block.
__device__ int lloyd_block(const double* pts, const double* w, int n, double* c, double* nx,
                           int* first, int* last, int* cnt, int k, double tol, int max_iter,
                           int* assign, double* score, ScoreVal* top, bool distinct,
                           KShared& sm, double* aux = nullptr) {
    __shared__ int s_fast, s_exact;
    LAux X;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double lm = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) lm = fmax(lm, fabs(pts[i]));
    double scale = block_max_d(lm, sm);
    if (scale == 0.0) scale = 1.0;
    const double gap = __dmul_rn(scale, 0x1.0p-40);
    const double thr = __dmul_rn(tol, scale);
    X.lo = aux, X.hi = aux + k, X.nlo = aux + 2 * k, X.nhi = aux + 3 * k;
    X.sw = aux + 4 * k, X.swx = aux + 5 * k, X.sax = aux + 6 * k;
    X.pf = (int*)(aux + 7 * k), X.pl = X.pf + k, X.pe = X.pl + k;
    X.exact = &s_exact;
    if (threadIdx.x == 0) s_exact = 1;
    __syncthreads();
    if (aux)
        for (int j = threadIdx.x; j < k; j += blockDim.x) X.lo[j] = X.hi[j] = c[j], X.pe[j] = -1;
    __syncthreads();
    int iters = 0;
    for (int it = 0; it < max_iter; ++it) {
        if (aux) {
            const int r = lloyd_interval_step(pts, w, n, X, first, last, cnt, k, gap, thr, sm);
            if (r != 2) {
                iters = it + 1;
                if (r == 0) break;
                continue;
            }
            if (!s_exact) {  // the exact step needs the reference's centres
                lloyd_exact_from(pts, w, X.pf, X.pl, k, c, sm);
                __syncthreads();
            }
        }
        if (wid == 0) {
            // Fast path: strictly ascending centres separated by far more than the
            // rounding of any |x - c| (gap > scale * 2^-40).  The distance sequence
            // over j is then strictly unimodal for every x, so the reference argmin
            // (strict <, lowest index on ties) is decided by neighbouring centres and
            // each cluster is the key range between two monotone boundaries.
            bool ok = true;
            for (int j = lane; j + 1 < k; j += 32) ok &= __dsub_rn(c[j + 1], c[j]) > gap;
            ok = __all_sync(0xffffffffu, ok);
            if (lane == 0) {
                s_fast = ok;
                sm.any_empty = 0;
                sm.done = 0;
            }
        }
        __syncthreads();
        const bool fast = s_fast;
        if (!fast) {
            for (int j = threadIdx.x; j < k; j += blockDim.x) {
                first[j] = 0x7fffffff;
                last[j] = -1;
                cnt[j] = 0;
            }
            __syncthreads();
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                double x = pts[i];
                int best = 0;
                double bd = fabs(__dsub_rn(x, c[0]));
                for (int j = 1; j < k; ++j) {
                    double d = fabs(__dsub_rn(x, c[j]));
                    if (d < bd) {
                        bd = d;
                        best = j;
                    }
                }
                assign[i] = best;
                atomicMin(&first[best], i);
                atomicMax(&last[best], i);
                atomicAdd(&cnt[best], 1);
            }
            __syncthreads();
        }
        if (wid == 0) {
            if (fast) {
                // start of cluster j+1 = first key whose distance to c[j+1] is < to c[j]
                for (int j = lane; j < k; j += 32) {
                    int lo = n, hi = n;  // last cluster ends at n
                    if (j + 1 < k) {
                        lo = 0;
                        const double a = c[j], b = c[j + 1];
                        while (lo < hi) {
                            int mid = (lo + hi) >> 1;
                            double x = pts[mid];
                            if (fabs(__dsub_rn(x, b)) < fabs(__dsub_rn(x, a))) hi = mid;
                            else lo = mid + 1;
                        }
                    }
                    last[j] = lo;  // exclusive end of cluster j (temporarily)
                }
                __syncwarp();
                for (int j = lane; j < k; j += 32) first[j] = j ? last[j - 1] : 0;
                __syncwarp();
                for (int j = lane; j < k; j += 32) {
                    cnt[j] = last[j] > first[j] ? last[j] - first[j] : 0;
                    last[j] = first[j] + cnt[j] - 1;
                }
                __syncwarp();
            }
            bool empty = false;
            long long t_sum = clock64();
            int steps_max = 0;
            for (int j = lane; j < k; j += 32) {
                double ws = 0.0, wxs = 0.0;
                if (cnt[j] > 0) {
                    if (last[j] - first[j] + 1 == cnt[j]) {
                        steps_max = max(steps_max, cnt[j]);
                        chain_sums(sm.wx, w, pts, first[j], last[j], ws, wxs);
                    } else {
                        for (int i = 0; i < n; ++i)
                            if (assign[i] == j) {
                                double wi = w[i];
                                ws = __dadd_rn(ws, wi);
                                wxs = __dadd_rn(wxs, __dmul_rn(wi, pts[i]));
                            }
                    }
                }
                if (ws > 0.0) {
                    nx[j] = __ddiv_rn(wxs, ws);
                    cnt[j] = 1;  // reuse as "non-empty" flag
                } else {
                    cnt[j] = 0;
                    empty = true;
                }
            }
            empty = __any_sync(0xffffffffu, empty);
            for (int o = 16; o > 0; o >>= 1) steps_max = max(steps_max, __shfl_xor_sync(0xffffffffu, steps_max, o));
            if (lane == 0 && blockIdx.x < 1024) {
                g_km_timing[blockIdx.x][6] += steps_max;
                g_km_timing[blockIdx.x][7] += clock64() - t_sum;
            }
            if (!empty) {  // convergence: max |nx - c| (exact, order-free), c <- nx
                double mv = 0.0;
                for (int j = lane; j < k; j += 32) mv = fmax(mv, fabs(__dsub_rn(nx[j], c[j])));
                for (int o = 16; o > 0; o >>= 1) mv = fmax(mv, __shfl_xor_sync(0xffffffffu, mv, o));
                __syncwarp();
                for (int j = lane; j < k; j += 32) c[j] = nx[j];
                if (lane == 0) sm.done = mv <= __dmul_rn(tol, scale);
            } else if (lane == 0) {
                sm.any_empty = 1;
            }
        }
        __syncthreads();
        if (sm.any_empty) {
            // re-seed empties to the points with the largest weighted squared
            // distance, libstdc++ sort order on ties (quantize.cpp:218-243)
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                double x = pts[i];
                double bd = __longlong_as_double(0x7ff0000000000000LL);
                for (int j = 0; j < k; ++j) {
                    double d = fabs(__dsub_rn(x, c[j]));
                    bd = d < bd ? d : bd;
                }
                score[i] = __dmul_rn(__dmul_rn(w[i], bd), bd);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                long nt = 0;
                for (int i = 0; i < n; ++i) {
                    double s = score[i];
                    if (s <= 0.0) continue;
                    double x = pts[i];
                    bool dup = false;
                    if (!distinct)
                        for (long t = 0; t < nt; ++t)
                            if (top[t].v == x) {
                                dup = true;
                                if (s > top[t].s) top[t].s = s;
                                break;
                            }
                    if (dup) continue;
                    top[nt].s = s;
                    top[nt].v = x;
                    ++nt;
                }
                IntroSort<ScoreVal, GreaterScore>{}.sort(top, nt);
                long used = 0;
                for (int j = 0; j < k; ++j)
                    if (!cnt[j] && used < nt) nx[j] = top[used++].v;
                double mv = 0.0;
                for (int j = 0; j < k; ++j) mv = fmax(mv, fabs(__dsub_rn(nx[j], c[j])));
                for (int j = 0; j < k; ++j) c[j] = nx[j];
                sm.done = mv <= __dmul_rn(tol, scale);
            }
            __syncthreads();
        }
        iters = it + 1;
        if (aux) {  // c is exact after an exact step
            __syncthreads();
            for (int j = threadIdx.x; j < k; j += blockDim.x) X.lo[j] = X.hi[j] = c[j];
            if (threadIdx.x == 0) s_exact = 1;
        }
        if (sm.done) break;
        __syncthreads();  // sm.done / s_fast are rewritten by the next iteration
    }
    if (aux) {
        __syncthreads();
        if (!s_exact) lloyd_exact_from(pts, w, X.pf, X.pl, k, c, sm);
        __syncthreads();
    }
    if (threadIdx.x == 0) IntroSort<double, LessD>{}.sort(c, k);
    __syncthreads();
    return iters;
}

// weighted_sq_loss (quantize.cpp:166-178): per-point minima in parallel, the sum
// sequentially in point order.
__device__ double sq_loss_block(const double* pts, const double* w, int n, const double* c, int k,
                                double* tmp, KShared& sm) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double best = __longlong_as_double(0x7ff0000000000000LL);
        for (int j = 0; j < k; ++j) {
            double d = __dsub_rn(pts[i], c[j]);
            double sq = __dmul_rn(d, d);
            best = sq < best ? sq : best;
        }
        tmp[i] = __dmul_rn(w[i], best);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double loss = sm.in_smem ? seq_prefix<true>(tmp, 0, n, 0.0, nullptr)
                                       : seq_prefix<false>(tmp, 0, n, 0.0, nullptr);
        sm.red[0] = loss;
    }
    __syncthreads();
    double r = sm.red[0];
    __syncthreads();
    return r;
}

// optional phase timing per CTA (DQTG_KM_TIMING=1): clocks of kpp / lloyd / loss, iterations, n

// SMEM: every problem's working set (n <= smem_n) lives in shared memory; the
// pointers are then derived from the shared carve in this instantiation, so every
// access to them compiles to a shared load (not a generic one).
template <bool SMEM>
__global__ void __launch_bounds__(kKB) kmeans_restarts_kernel(const KProblem* probs,
                                                              int restarts, int smem_n, int certify) {
    extern __shared__ double dsm[];
    __shared__ KShared sm;
    const KProblem& P = probs[blockIdx.x / restarts];
    const int t = blockIdx.x % restarts;
    const int n = P.n, k = P.k;
    if (n < k || k <= 0 || P.skip) return;
    double* c = dsm;
    double* nx = c + k;
    int* first = (int*)(nx + k);
    int* last = first + k;
    int* cnt = last + k;
    double* aux = dsm + 2 * k + (3 * k + 1) / 2 + 1;  // LAux: 7k doubles + 3k ints
    double* base = aux + 9 * k + 1;
    const double *pts, *w;
    double *d2, *prob, *pref;
    int* assign;
    if (SMEM) {  // working set in shared memory: the serial chains hit LDS, not L2
        double* sp = base;
        double* sw = sp + n;
        d2 = sw + n;
        prob = d2 + n;
        pref = prob + n;
        double2* wx = (double2*)(((uintptr_t)(pref + n) + 15) & ~(uintptr_t)15);
        assign = (int*)(wx + n);
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double pv = P.pts[i], wv = P.w[i];
            sp[i] = pv;
            sw[i] = wv;
            wx[i] = make_double2(wv, pv);
        }
        pts = sp;
        w = sw;
        if (threadIdx.x == 0) sm.wx = wx, sm.in_smem = 1;
    } else {
        if (threadIdx.x == 0) sm.wx = nullptr, sm.in_smem = 0;
        pts = P.pts;
        w = P.w;
        d2 = P.scratch + (size_t)t * P.scratch_stride;
        prob = d2 + n;
        pref = prob + n;
        assign = (int*)(pref + n);
    }
    ScoreVal* top = (ScoreVal*)d2;  // reseed scratch reuses d2/prob (2n doubles)
    if (threadIdx.x == 0 && blockIdx.x < 1024)
        for (int q = 6; q < 12; ++q) g_km_timing[blockIdx.x][q] = 0;
    if (threadIdx.x == 0) {
        const long long m0 = clock64();
        mt64_seed(sm.rng, P.seed + (uint64_t)t);
        if (blockIdx.x < 1024) g_km_timing[blockIdx.x][11] = clock64() - m0;
    }
    __syncthreads();
    mt64_regen_block(sm.rng);  // the first draw's regeneration, block-parallel
    const long long c0 = clock64();
    kpp_init(pts, w, n, k, d2, prob, pref, c, sm, certify);
    const long long c1 = clock64();
    const int its = lloyd_block(pts, w, n, c, nx, first, last, cnt, k, 1e-6, 100, assign, pref, top, true, sm,
                                certify ? aux : nullptr);
    const long long c2 = clock64();
    double loss = sq_loss_block(pts, w, n, c, k, prob, sm);
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        long long* g = g_km_timing[blockIdx.x];
        g[0] = c1 - c0, g[1] = c2 - c1, g[2] = clock64() - c2, g[3] = its, g[4] = n, g[5] = k;
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) P.centers[(size_t)t * k + j] = c[j];
    if (threadIdx.x == 0) P.loss[t] = loss;
}

// Restart selection + float cast + dedup (quantize.cpp:306-324).
__global__ void kmeans_select_kernel(const KProblem* probs, int restarts, float* cb_out,
                                     int cb_stride, uint32_t* cb_len) {
    const KProblem& P = probs[blockIdx.x];
    if (threadIdx.x != 0 || P.skip || P.n < P.k) return;
    double best = __longlong_as_double(0x7ff0000000000000LL);
    int bt = -1;
    for (int t = 0; t < restarts; ++t)
        if (P.loss[t] < best) {
            best = P.loss[t];
            bt = t;
        }
    float* cb = cb_out + (size_t)P.slot * cb_stride;
    uint32_t o = 0;
    if (bt >= 0)
        for (int j = 0; j < P.k; ++j) {
            float f = __double2float_rn(P.centers[(size_t)bt * P.k + j]);
            if (o == 0 || f != cb[o - 1]) cb[o++] = f;
        }
    cb_len[P.slot] = o;
}

// ---- host side -------------------------------------------------------------
void run_kmeans(Engine& e, std::vector<KProblem>& probs, float* cb_out, int cb_stride,
                uint32_t* cb_len_dev) {
    if (probs.empty()) return;
    const int restarts = 8;  // quantize.cpp:306
    size_t scratch_doubles = 0, centers = 0;
    int maxk = 1;
    for (auto& p : probs) {
        p.scratch_stride = (size_t)4 * p.n + 8;
        scratch_doubles += p.scratch_stride * restarts;
        centers += (size_t)p.k * restarts;
        maxk = p.k > maxk ? p.k : maxk;
    }
    double* scr = (double*)e.buf("km.scratch", scratch_doubles * 8);
    double* cen = (double*)e.buf("km.centers", (centers + 8) * 8);
    double* loss = (double*)e.buf("km.loss", probs.size() * restarts * 8);
    size_t so = 0, co = 0;
    for (size_t i = 0; i < probs.size(); ++i) {
        probs[i].scratch = scr + so;
        so += probs[i].scratch_stride * restarts;
        probs[i].centers = cen + co;
        co += (size_t)probs[i].k * restarts;
        probs[i].loss = loss + i * restarts;
    }
    KProblem* dp = (KProblem*)e.buf("km.probs", probs.size() * sizeof(KProblem));
    DQTG_CUDA(cudaMemcpyAsync(dp, probs.data(), probs.size() * sizeof(KProblem),
                              cudaMemcpyHostToDevice, e.stream));
    int maxn = 1;
    for (auto& p : probs) maxn = std::max(maxn, p.n);
    const size_t head = ((size_t)2 * maxk + (3 * maxk + 1) / 2 + 1 + 9 * maxk + 1) * 8;
    const size_t budget = 200 * 1024;
    int smem_n = (int)((budget - std::min(budget, head)) / 60);  // 5 doubles + pair + int per key
    size_t smem = head + (size_t)std::min(maxn, smem_n) * 60 + 96;
    // DQTG_KM_EXACT: every sum sequential (no certified parallel steps; tests compare)
    const int certify = getenv("DQTG_KM_EXACT") ? 0 : 1;
    // restarts on the engine's high-priority side stream (fork/join with events)
    void (*kfn)(const KProblem*, int, int, int) =
        maxn <= smem_n ? kmeans_restarts_kernel<true> : kmeans_restarts_kernel<false>;
    ensure_dyn_smem((const void*)kfn, smem);
    if (e.profiling || getenv("DQTG_NO_HI")) {
        DQTG_SPAN(e, "kmeans_restarts_kernel");
        kfn<<<(unsigned)(probs.size() * restarts), kKB, smem, e.stream>>>(dp, restarts, smem_n, certify);
    } else {
        cudaStream_t hs = e.hi();
        kfn<<<(unsigned)(probs.size() * restarts), kKB, smem, hs>>>(dp, restarts, smem_n, certify);
        e.hi_done();
    }
    { DQTG_SPAN(e, "kmeans_select_kernel"); kmeans_select_kernel<<<(unsigned)probs.size(), 32, 0, e.stream>>>(dp, restarts, cb_out,
                                                                       cb_stride, cb_len_dev); }
    e.launched(2);
    DQTG_CUDA(cudaGetLastError());
    if (getenv("DQTG_KM_TIMING")) {
        e.sync();
        static long long h[1024][12];
        DQTG_CUDA(cudaMemcpyFromSymbol(h, g_km_timing, sizeof(h)));
        for (size_t b = 0; b < probs.size() * restarts && b < 1024; ++b)
            fprintf(stderr, "km cta %zu: kpp %lld lloyd %lld loss %lld clk, iters %lld, n %lld k %lld, chain steps %lld in %lld clk, "
                    "interval bnd %lld sums %lld cert %lld, mt %lld\n", b,
                    h[b][0], h[b][1], h[b][2], h[b][3], h[b][4], h[b][5], h[b][6], h[b][7], h[b][8], h[b][9], h[b][10], h[b][11]);
    }
}

void compact_keys(Engine& e, const unsigned long long* hist, int64_t hs_stride, int64_t HS,
                  const double* key, double sigma, int nprob, double* pts,
                  unsigned long long* cnt, double* w, int64_t out_stride, int* n_keys) {
    { DQTG_SPAN(e, "compact_keys_kernel"); compact_keys_kernel<<<nprob, 1024, 0, e.stream>>>(hist, hs_stride, HS, key, sigma, pts, cnt,
                                                      w, out_stride, n_keys); }
    e.launched();
    DQTG_CUDA(cudaGetLastError());
}

}  // namespace dqtg

// ---- stand-alone clustering entry points (weighted_kmeanspp_init /
// weighted_lloyd / weighted_sq_loss, quantize.cpp:94-254) for arbitrary points ----
namespace dqtg {

__global__ void __launch_bounds__(kKB) kpp_api_kernel(const double* pts, const double* w, int n,
                                                      int k, uint64_t seed, double* scratch,
                                                      double* out, int* status) {
    extern __shared__ double dsm[];
    __shared__ KShared sm;
    if (threadIdx.x == 0) sm.wx = nullptr, sm.in_smem = 0;  // working set in global memory
    // validation (quantize.cpp:98-113): weights, total, distinct count
    if (threadIdx.x == 0) {
        int st = 0;
        bool pos = false;
        for (int i = 0; i < n; ++i) {
            if (!(w[i] >= 0.0)) st = 1;
            pos |= w[i] > 0.0;
        }
        if (!st && !pos) st = 2;
        if (!st) {
            double* d = scratch + (size_t)4 * n;
            for (int i = 0; i < n; ++i) d[i] = pts[i];
            IntroSort<double, LessD>{}.sort(d, n);
            int distinct = 0;
            for (int i = 0; i < n; ++i)
                if (i == 0 || !(d[i] == d[distinct - 1])) d[distinct++] = d[i];
            if (distinct < k) st = 3;
        }
        *status = st;
        mt64_seed(sm.rng, seed);
    }
    __syncthreads();
    if (*status) return;
    double* d2 = scratch;
    double* prob = d2 + n;
    double* pref = prob + n;
    kpp_init(pts, w, n, k, d2, prob, pref, dsm, sm);
    for (int j = threadIdx.x; j < k; j += blockDim.x) out[j] = dsm[j];
}

__global__ void __launch_bounds__(kKB) lloyd_api_kernel(const double* pts, const double* w, int n,
                                                        int k, double tol, int max_iter,
                                                        double* scratch, double* centers,
                                                        int* iters) {
    extern __shared__ double dsm[];
    __shared__ KShared sm;
    if (threadIdx.x == 0) sm.wx = nullptr, sm.in_smem = 0;  // working set in global memory
    double* c = dsm;
    double* nx = c + k;
    int* first = (int*)(nx + k);
    int* last = first + k;
    int* cnt = last + k;
    for (int j = threadIdx.x; j < k; j += blockDim.x) c[j] = centers[j];
    __syncthreads();
    int* assign = (int*)(scratch + (size_t)3 * n);
    ScoreVal* top = (ScoreVal*)scratch;
    double* score = scratch + (size_t)2 * n;
    int it = lloyd_block(pts, w, n, c, nx, first, last, cnt, k, tol, max_iter, assign, score, top,
                         false, sm);
    for (int j = threadIdx.x; j < k; j += blockDim.x) centers[j] = c[j];
    if (threadIdx.x == 0) *iters = it;
}

__global__ void __launch_bounds__(kKB) loss_api_kernel(const double* pts, const double* w, int n,
                                                       const double* c, int k, double* tmp,
                                                       double* out) {
    __shared__ KShared sm;
    if (threadIdx.x == 0) sm.wx = nullptr, sm.in_smem = 0;  // working set in global memory
    double l = sq_loss_block(pts, w, n, c, k, tmp, sm);
    if (threadIdx.x == 0) *out = l;
}

struct DevArrays {
    double *pts, *w, *scr, *c;
    int* st;
};

static DevArrays stage(Engine& e, const double* pts, const double* w, uint64_t n, uint32_t k,
                       const double* centers) {
    DevArrays d;
    d.pts = (double*)e.buf("kapi.pts", n * 8 + 8);
    d.w = (double*)e.buf("kapi.w", n * 8 + 8);
    d.scr = (double*)e.buf("kapi.scr", (5 * n + 8) * 8);
    d.c = (double*)e.buf("kapi.c", (size_t)k * 8 + 8);
    d.st = (int*)e.buf("kapi.st", 16);
    e.to_device(d.pts, pts, n * 8);
    e.to_device(d.w, w, n * 8);
    if (centers) e.to_device(d.c, centers, (size_t)k * 8);
    return d;
}

void kmeanspp_host_api(Engine& e, const double* pts, const double* w, uint64_t n, uint32_t k,
                       uint64_t seed, double* centers) {
    DQTG_REQUIRE(k >= 1, DQTG_ERROR, "k must be >= 1");
    DevArrays d = stage(e, pts, w, n, k, nullptr);
    { DQTG_SPAN(e, "kpp_api_kernel"); kpp_api_kernel<<<1, kKB, (size_t)k * 8 + 16, e.stream>>>(d.pts, d.w, (int)n, (int)k, seed,
                                                             d.scr, d.c, d.st); }
    e.launched();
    int st = 0;
    e.d2h(&st, d.st, 4);
    e.sync();
    DQTG_REQUIRE(st != 1, DQTG_ERROR, "weights must be non-negative");
    DQTG_REQUIRE(st != 2, DQTG_ERROR, "total weight must be positive");
    if (st == 3) {
        // count distinct again on the host side of the message only
        throw Fail(DQTG_TOO_FEW_DISTINCT, "need " + std::to_string(k) + " distinct points");
    }
    e.from_device(centers, d.c, (size_t)k * 8);
    e.sync();
}

void lloyd_host_api(Engine& e, const double* pts, const double* w, uint64_t n, double* centers,
                    uint32_t k, double tol, uint32_t max_iter, uint32_t* iters) {
    DQTG_REQUIRE(k >= 1, DQTG_ERROR, "no initial centers");
    DevArrays d = stage(e, pts, w, n, k, centers);
    int* it = d.st;
    { DQTG_SPAN(e, "lloyd_api_kernel"); lloyd_api_kernel<<<1, kKB, (size_t)k * (2 * 8 + 3 * 4) + 16, e.stream>>>(
        d.pts, d.w, (int)n, (int)k, tol, (int)max_iter, d.scr, d.c, it); }
    e.launched();
    int h = 0;
    e.d2h(&h, it, 4);
    e.from_device(centers, d.c, (size_t)k * 8);
    e.sync();
    if (iters) *iters = (uint32_t)h;
}

double sq_loss_host_api(Engine& e, const double* pts, const double* w, uint64_t n,
                        const double* centers, uint32_t k) {
    DevArrays d = stage(e, pts, w, n, k, centers);
    { DQTG_SPAN(e, "loss_api_kernel"); loss_api_kernel<<<1, kKB, 0, e.stream>>>(d.pts, d.w, (int)n, d.c, (int)k, d.scr, d.scr + n + 1); }
    e.launched();
    double h = 0;
    e.d2h(&h, d.scr + n + 1, 8);
    e.sync();
    return h;
}

}  // namespace dqtg
