// Device building blocks for the histogram k-means of quantize.cpp:94-325.
//
// Exactness strategy: every floating-point sum that the
// reference accumulates sequentially is accumulated sequentially here too, in
// the same order (one lane per sum); only order-independent work (distances,
// argmins, maxima, d2 updates) is spread across threads.  1-D nearest-centre
// cells are intervals of the sorted key array, so each cluster's weighted sums
// are contiguous-range sums that run in parallel across clusters.
#pragma once

#include "common.cuh"

namespace dqtg {

// ---- std::mt19937_64 (fully specified by the C++ standard) ----------------
struct Mt64 {
    uint64_t mt[312];
    int mti;
};

__device__ inline void mt64_seed(Mt64& r, uint64_t seed) {
    r.mt[0] = seed;
    for (int i = 1; i < 312; i++)
        r.mt[i] = 6364136223846793005ULL * (r.mt[i - 1] ^ (r.mt[i - 1] >> 62)) + (uint64_t)i;
    r.mti = 312;
}

__device__ inline uint64_t mt64_next(Mt64& r) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    if (r.mti >= 312) {
        int i;
        for (i = 0; i < 156; i++) {
            uint64_t x = (r.mt[i] & UM) | (r.mt[i + 1] & LM);
            r.mt[i] = r.mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        }
        for (; i < 311; i++) {
            uint64_t x = (r.mt[i] & UM) | (r.mt[i + 1] & LM);
            r.mt[i] = r.mt[i - 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        }
        uint64_t x = (r.mt[311] & UM) | (r.mt[0] & LM);
        r.mt[311] = r.mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        r.mti = 0;
    }
    uint64_t x = r.mt[r.mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

// The regeneration of mt64_next run by a whole block (blockDim >= 156): elements
// 0..155 read only old words, 156..310 the new word i - 156 and old words, 311 the
// new words 0 and 155, as in the sequential loop.  Same state, mti = 0.
__device__ inline void mt64_regen_block(Mt64& r) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    const int t = threadIdx.x;
    uint64_t v = 0;
    if (t < 156) {
        const uint64_t x = (r.mt[t] & UM) | (r.mt[t + 1] & LM);
        v = r.mt[t + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    __syncthreads();
    if (t < 156) r.mt[t] = v;
    __syncthreads();
    if (t >= 156 && t < 311) {
        const uint64_t x = (r.mt[t] & UM) | (r.mt[t + 1] & LM);
        v = r.mt[t - 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    __syncthreads();
    if (t >= 156 && t < 311) r.mt[t] = v;
    __syncthreads();
    if (t == 0) {
        const uint64_t x = (r.mt[311] & UM) | (r.mt[0] & LM);
        r.mt[311] = r.mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        r.mti = 0;
    }
    __syncthreads();
}

// quantize.cpp:23
__device__ inline double uniform01(Mt64& r) {
    return __dmul_rn((double)(mt64_next(r) >> 11), 0x1.0p-53);
}

// ---- libstdc++ std::sort, single thread (tie order of equal keys matters) --
template <typename T, typename Less>
struct IntroSort {
    Less less;
    __device__ void adjust_heap(T* f, long hole, long len, T val) {
        long top = hole, sc = hole;
        while (sc < (len - 1) / 2) {
            sc = 2 * (sc + 1);
            if (less(f[sc], f[sc - 1])) sc--;
            f[hole] = f[sc];
            hole = sc;
        }
        if ((len & 1) == 0 && sc == (len - 2) / 2) {
            sc = 2 * (sc + 1);
            f[hole] = f[sc - 1];
            hole = sc - 1;
        }
        long parent = (hole - 1) / 2;
        while (hole > top && less(f[parent], val)) {
            f[hole] = f[parent];
            hole = parent;
            parent = (hole - 1) / 2;
        }
        f[hole] = val;
    }
    __device__ void heapsort(T* f, T* l) {
        long len = l - f;
        if (len >= 2) {
            long parent = (len - 2) / 2;
            for (;;) {
                T v = f[parent];
                adjust_heap(f, parent, len, v);
                if (parent == 0) break;
                parent--;
            }
        }
        while (l - f > 1) {
            --l;
            T v = *l;
            *l = *f;
            adjust_heap(f, 0, l - f, v);
        }
    }
    __device__ static void swap(T* a, T* b) {
        T t = *a;
        *a = *b;
        *b = t;
    }
    __device__ void median_to_first(T* r, T* a, T* b, T* c) {
        if (less(*a, *b)) {
            if (less(*b, *c)) swap(r, b);
            else if (less(*a, *c)) swap(r, c);
            else swap(r, a);
        } else if (less(*a, *c)) swap(r, a);
        else if (less(*b, *c)) swap(r, c);
        else swap(r, b);
    }
    __device__ T* partition(T* f, T* l, T* p) {
        for (;;) {
            while (less(*f, *p)) ++f;
            --l;
            while (less(*p, *l)) --l;
            if (!(f < l)) return f;
            swap(f, l);
            ++f;
        }
    }
    __device__ void loop(T* f, T* l, long depth) {
        // explicit stack instead of recursion: (first,last,depth) of right parts
        T* sf[64];
        T* sl[64];
        long sd[64];
        int sp = 0;
        for (;;) {
            while (l - f > 16) {
                if (depth == 0) {
                    heapsort(f, l);
                    break;
                }
                --depth;
                T* mid = f + (l - f) / 2;
                median_to_first(f, f + 1, mid, l - 1);
                T* cut = partition(f + 1, l, f);
                // reference recurses into [cut, l) first, then loops on [f, cut)
                sf[sp] = f;
                sl[sp] = cut;
                sd[sp] = depth;
                sp++;
                f = cut;
            }
            if (!sp) return;
            --sp;
            f = sf[sp];
            l = sl[sp];
            depth = sd[sp];
        }
    }
    __device__ void linear_insert(T* l) {
        T val = *l;
        T* nx = l - 1;
        while (less(val, *nx)) {
            *l = *nx;
            l = nx;
            --nx;
        }
        *l = val;
    }
    __device__ void insertion(T* f, T* l) {
        if (f == l) return;
        for (T* i = f + 1; i != l; ++i) {
            if (less(*i, *f)) {
                T val = *i;
                for (T* m = i; m != f; --m) *m = *(m - 1);
                *f = val;
            } else
                linear_insert(i);
        }
    }
    __device__ void sort(T* f, long n) {
        if (n <= 0) return;
        T* l = f + n;
        long lg = 63 - __clzll((long long)n);
        loop(f, l, lg * 2);
        if (l - f > 16) {
            insertion(f, f + 16);
            for (T* i = f + 16; i != l; ++i) linear_insert(i);
        } else
            insertion(f, l);
    }
};

struct LessD {
    __device__ bool operator()(double a, double b) const { return a < b; }
};
struct LessF {
    __device__ bool operator()(float a, float b) const { return a < b; }
};
struct ScoreVal {
    double s, v;
};
struct GreaterScore {  // quantize.cpp:238-239
    __device__ bool operator()(const ScoreVal& a, const ScoreVal& b) const { return a.s > b.s; }
};

}  // namespace dqtg
