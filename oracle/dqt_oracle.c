/*
 * dqt_oracle.c — TEST INFRASTRUCTURE ONLY (see dqt_oracle.h).
 *
 * A plain-C restatement of the reference's checkpoint-compression path.  Every
 * function names the reference file:line it follows (paths relative to
 * /root/reference/proj).  Floating-point expressions are written in the same
 * order and precision as the reference and this file is compiled with
 * -ffp-contract=off, so results are bit-identical to the
 * reference built the same way; tests/test_oracle_pin.py proves it against
 * oracle/_ref.
 */
#define _GNU_SOURCE
#include "dqt_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ========================================================================= */
/* mt19937_64 (the reference uses std::mt19937_64, fully specified by C++11)  */
/* ========================================================================= */
typedef struct { uint64_t mt[312]; int mti; } mt64;

static void mt64_seed(mt64 *r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; i++)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

static uint64_t mt64_next(mt64 *r) {
    static const uint64_t mag01[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    if (r->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; i++) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        for (; i < 311; i++) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        }
        x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag01[(int)(x & 1ULL)];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* quantize.cpp:23 */
static double uniform01(mt64 *r) { return (double)(mt64_next(r) >> 11) * 0x1.0p-53; }

/* ========================================================================= */
/* libstdc++ std::sort (introsort, threshold 16, median-of-3, heapsort        */
/* fallback, final insertion sort).  Tie order of equal keys depends on this   */
/* exact algorithm (quantize.cpp:238-239 reseed order, :282-283 ±0 order).     */
/* ========================================================================= */
#define DEF_SORT(NAME, T, LESS, SWAP)                                                            \
    static void NAME##_adjust_heap(T *f, ptrdiff_t hole, ptrdiff_t len, T val) {                 \
        ptrdiff_t top = hole, sc = hole;                                                         \
        while (sc < (len - 1) / 2) {                                                             \
            sc = 2 * (sc + 1);                                                                   \
            if (LESS(f[sc], f[sc - 1])) sc--;                                                    \
            f[hole] = f[sc];                                                                     \
            hole = sc;                                                                           \
        }                                                                                        \
        if ((len & 1) == 0 && sc == (len - 2) / 2) {                                             \
            sc = 2 * (sc + 1);                                                                   \
            f[hole] = f[sc - 1];                                                                 \
            hole = sc - 1;                                                                       \
        }                                                                                        \
        ptrdiff_t parent = (hole - 1) / 2;                                                       \
        while (hole > top && LESS(f[parent], val)) {                                             \
            f[hole] = f[parent];                                                                 \
            hole = parent;                                                                       \
            parent = (hole - 1) / 2;                                                             \
        }                                                                                        \
        f[hole] = val;                                                                           \
    }                                                                                            \
    static void NAME##_heapsort(T *f, T *l) {                                                    \
        ptrdiff_t len = l - f;                                                                   \
        if (len >= 2) {                                                                          \
            ptrdiff_t parent = (len - 2) / 2;                                                    \
            for (;;) {                                                                           \
                T v = f[parent];                                                                 \
                NAME##_adjust_heap(f, parent, len, v);                                           \
                if (parent == 0) break;                                                          \
                parent--;                                                                        \
            }                                                                                    \
        }                                                                                        \
        while (l - f > 1) {                                                                      \
            --l;                                                                                 \
            T v = *l;                                                                            \
            *l = *f;                                                                             \
            NAME##_adjust_heap(f, 0, l - f, v);                                                  \
        }                                                                                        \
    }                                                                                            \
    static void NAME##_median_to_first(T *r, T *a, T *b, T *c) {                                 \
        if (LESS(*a, *b)) {                                                                      \
            if (LESS(*b, *c)) SWAP(r, b);                                                        \
            else if (LESS(*a, *c)) SWAP(r, c);                                                   \
            else SWAP(r, a);                                                                     \
        } else if (LESS(*a, *c)) SWAP(r, a);                                                     \
        else if (LESS(*b, *c)) SWAP(r, c);                                                       \
        else SWAP(r, b);                                                                         \
    }                                                                                            \
    static T *NAME##_partition(T *f, T *l, T *p) {                                               \
        for (;;) {                                                                               \
            while (LESS(*f, *p)) ++f;                                                            \
            --l;                                                                                 \
            while (LESS(*p, *l)) --l;                                                            \
            if (!(f < l)) return f;                                                              \
            SWAP(f, l);                                                                          \
            ++f;                                                                                 \
        }                                                                                        \
    }                                                                                            \
    static void NAME##_loop(T *f, T *l, ptrdiff_t depth) {                                       \
        while (l - f > 16) {                                                                     \
            if (depth == 0) {                                                                    \
                NAME##_heapsort(f, l);                                                           \
                return;                                                                          \
            }                                                                                    \
            --depth;                                                                             \
            T *mid = f + (l - f) / 2;                                                            \
            NAME##_median_to_first(f, f + 1, mid, l - 1);                                        \
            T *cut = NAME##_partition(f + 1, l, f);                                              \
            NAME##_loop(cut, l, depth);                                                          \
            l = cut;                                                                             \
        }                                                                                        \
    }                                                                                            \
    static void NAME##_linear_insert(T *l) {                                                     \
        T val = *l;                                                                              \
        T *nx = l - 1;                                                                           \
        while (LESS(val, *nx)) {                                                                 \
            *l = *nx;                                                                            \
            l = nx;                                                                              \
            --nx;                                                                                \
        }                                                                                        \
        *l = val;                                                                                \
    }                                                                                            \
    static void NAME##_insertion(T *f, T *l) {                                                   \
        if (f == l) return;                                                                      \
        for (T *i = f + 1; i != l; ++i) {                                                        \
            if (LESS(*i, *f)) {                                                                  \
                T val = *i;                                                                      \
                memmove(f + 1, f, (size_t)(i - f) * sizeof(T));                                  \
                *f = val;                                                                        \
            } else                                                                               \
                NAME##_linear_insert(i);                                                         \
        }                                                                                        \
    }                                                                                            \
    static void NAME(T *f, size_t n) {                                                           \
        if (n == 0) return;                                                                      \
        T *l = f + n;                                                                            \
        ptrdiff_t lg = 63 - __builtin_clzll((unsigned long long)n);                              \
        NAME##_loop(f, l, lg * 2);                                                               \
        if (l - f > 16) {                                                                        \
            NAME##_insertion(f, f + 16);                                                         \
            for (T *i = f + 16; i != l; ++i) NAME##_linear_insert(i);                            \
        } else                                                                                   \
            NAME##_insertion(f, l);                                                              \
    }

#define LT_PLAIN(a, b) ((a) < (b))
#define SWAP_F(x, y)            \
    do {                        \
        float t_ = *(x);        \
        *(x) = *(y);            \
        *(y) = t_;              \
    } while (0)
#define SWAP_D(x, y)            \
    do {                        \
        double t_ = *(x);       \
        *(x) = *(y);            \
        *(y) = t_;              \
    } while (0)
typedef struct { double s, v; } sv_pair;
#define LT_DESC(a, b) ((a).s > (b).s)
#define SWAP_P(x, y)            \
    do {                        \
        sv_pair t_ = *(x);      \
        *(x) = *(y);            \
        *(y) = t_;              \
    } while (0)

DEF_SORT(sort_f32, float, LT_PLAIN, SWAP_F)
DEF_SORT(sort_f64, double, LT_PLAIN, SWAP_D)
DEF_SORT(sort_pairs, sv_pair, LT_DESC, SWAP_P)

void dqo_sort_f32(float *v, size_t n) { sort_f32(v, n); }
void dqo_sort_f64(double *v, size_t n) { sort_f64(v, n); }
void dqo_sort_pairs_desc(double *score, double *value, size_t n) {
    sv_pair *p = malloc(n * sizeof *p + 1);
    for (size_t i = 0; i < n; i++) p[i].s = score[i], p[i].v = value[i];
    sort_pairs(p, n);
    for (size_t i = 0; i < n; i++) score[i] = p[i].s, value[i] = p[i].v;
    free(p);
}

/* ========================================================================= */
/* Sketch — sketch.cpp                                                        */
/* ========================================================================= */
typedef struct { double gamma, inv_ln_gamma, rep_scale; } sk_par;

static sk_par sk_params(double alpha) { /* sketch.cpp:14-19 */
    sk_par p;
    p.gamma = (1.0 + alpha) / (1.0 - alpha);
    p.inv_ln_gamma = 1.0 / log(p.gamma);
    p.rep_scale = 2.0 / (1.0 + p.gamma);
    return p;
}

static int64_t sk_bucket(const sk_par *p, double abs_x) { /* sketch.cpp:21-31 */
    double r = log(abs_x) * p->inv_ln_gamma;
    double nearest = nearbyint(r);
    if (fabs(r - nearest) > 1e-9 * fmax(1.0, fabs(r))) return (int64_t)ceil(r);
    int64_t k = (int64_t)nearest;
    while (pow(p->gamma, (double)(k - 1)) >= abs_x) --k;
    while (pow(p->gamma, (double)k) < abs_x) ++k;
    return k;
}

static double sk_rep(const sk_par *p, int64_t k) { /* sketch.cpp:33-37 */
    return p->rep_scale * pow(p->gamma, (double)k);
}

int64_t dqo_bucket_index(double alpha, double abs_x) {
    sk_par p = sk_params(alpha);
    return sk_bucket(&p, abs_x);
}
double dqo_representative(double alpha, int64_t k) {
    sk_par p = sk_params(alpha);
    return sk_rep(&p, k);
}

static const double kZeroMin = 1e-12; /* sketch.hpp:24 */

void dqo_sketch_range(double alpha, int64_t *kmin, int64_t *kmax) {
    sk_par p = sk_params(alpha);
    float zf = (float)kZeroMin;
    if ((double)zf < kZeroMin) zf = nextafterf(zf, INFINITY); /* smallest float >= 1e-12 */
    *kmin = sk_bucket(&p, (double)zf);
    *kmax = sk_bucket(&p, (double)FLT_MAX);
}

int dqo_sketch_init(dqo_sketch *s, double alpha) {
    if (!(alpha > 0.0) || !(alpha < 1.0)) return DQO_ERR_Q_RANGE; /* sketch.cpp:15 */
    sk_par p = sk_params(alpha);
    s->alpha = alpha;
    s->gamma = p.gamma;
    s->inv_ln_gamma = p.inv_ln_gamma;
    s->rep_scale = p.rep_scale;
    dqo_sketch_range(alpha, &s->kmin, &s->kmax);
    size_t nb = (size_t)(s->kmax - s->kmin + 1);
    s->pos = calloc(nb, sizeof(uint64_t));
    s->neg = calloc(nb, sizeof(uint64_t));
    s->zero = s->total = 0;
    return DQO_OK;
}

void dqo_sketch_free(dqo_sketch *s) {
    free(s->pos);
    free(s->neg);
    s->pos = s->neg = NULL;
}

/* sketch_build(const float*, n, alpha), sketch.cpp:131-148 */
void dqo_sketch_add_f32(dqo_sketch *s, const float *x, size_t n) {
    sk_par p = {s->gamma, s->inv_ln_gamma, s->rep_scale};
    for (size_t i = 0; i < n; ++i) {
        double v = x[i];
        double av = fabs(v);
        if (av < kZeroMin)
            ++s->zero;
        else if (v > 0)
            ++s->pos[sk_bucket(&p, av) - s->kmin];
        else
            ++s->neg[sk_bucket(&p, av) - s->kmin];
    }
    s->total += n;
}

/* Sketch::quantile, sketch.cpp:59-77 */
int dqo_sketch_quantile(const dqo_sketch *s, double q, double *out) {
    if (!(q >= 0.0 && q <= 1.0)) return DQO_ERR_Q_RANGE;
    if (s->total == 0) return DQO_ERR_EMPTY_SKETCH;
    sk_par p = {s->gamma, s->inv_ln_gamma, s->rep_scale};
    uint64_t rank = (uint64_t)ceil(q * (double)(s->total - 1)) + 1;
    if (rank > s->total) rank = s->total;
    uint64_t seen = 0;
    int64_t nb = s->kmax - s->kmin + 1;
    for (int64_t i = nb - 1; i >= 0; --i) {
        if (!s->neg[i]) continue;
        seen += s->neg[i];
        if (seen >= rank) { *out = -sk_rep(&p, i + s->kmin); return DQO_OK; }
    }
    seen += s->zero;
    if (seen >= rank) { *out = 0.0; return DQO_OK; }
    int64_t last = -1;
    for (int64_t i = 0; i < nb; ++i) {
        if (!s->pos[i]) continue;
        last = i;
        seen += s->pos[i];
        if (seen >= rank) { *out = sk_rep(&p, i + s->kmin); return DQO_OK; }
    }
    *out = last >= 0 ? sk_rep(&p, last + s->kmin) : 0.0;
    return DQO_OK;
}

size_t dqo_sketch_nbuckets(const dqo_sketch *s) {
    size_t n = s->zero ? 1 : 0;
    int64_t nb = s->kmax - s->kmin + 1;
    for (int64_t i = 0; i < nb; ++i) n += (s->pos[i] != 0) + (s->neg[i] != 0);
    return n;
}

/* Sketch::histogram, sketch.cpp:79-96 */
size_t dqo_sketch_histogram(const dqo_sketch *s, double *keys, uint64_t *counts) {
    sk_par p = {s->gamma, s->inv_ln_gamma, s->rep_scale};
    size_t o = 0;
    int64_t nb = s->kmax - s->kmin + 1;
    for (int64_t i = nb - 1; i >= 0; --i)
        if (s->neg[i]) keys[o] = -sk_rep(&p, i + s->kmin), counts[o++] = s->neg[i];
    if (s->zero) keys[o] = 0.0, counts[o++] = s->zero;
    for (int64_t i = 0; i < nb; ++i)
        if (s->pos[i]) keys[o] = sk_rep(&p, i + s->kmin), counts[o++] = s->pos[i];
    return o;
}

int dqo_sketch_dense(const float *x, size_t n, double alpha, int64_t *kmin, int64_t *kmax,
                     uint64_t *zero, uint64_t *pos_out, uint64_t *neg_out) {
    dqo_sketch s;
    int rc = dqo_sketch_init(&s, alpha);
    if (rc) return rc;
    dqo_sketch_add_f32(&s, x, n);
    *kmin = s.kmin;
    *kmax = s.kmax;
    *zero = s.zero;
    size_t nb = (size_t)(s.kmax - s.kmin + 1);
    if (pos_out) memcpy(pos_out, s.pos, nb * 8);
    if (neg_out) memcpy(neg_out, s.neg, nb * 8);
    dqo_sketch_free(&s);
    return DQO_OK;
}

/* ========================================================================= */
/* Ranker — ranker.cpp                                                        */
/* ========================================================================= */
/* ema_update, ranker.cpp:21-37 (float, no contraction) */
void dqo_ema_update(float *e, const float *g, size_t n, double beta) {
    const float b = (float)beta;
    for (size_t i = 0; i < n; ++i) e[i] = b * g[i] + (1.0f - b) * e[i];
}

/* compute_scores, ranker.cpp:79-101 */
void dqo_scores(const float *w, const float *ema, size_t n, float *mag, float *sens) {
    for (size_t i = 0; i < n; ++i) {
        mag[i] = fabsf(w[i]);
        if (ema && sens) sens[i] = fabsf(ema[i] * w[i]);
    }
}

/* ========================================================================= */
/* Clustering — quantize.cpp                                                  */
/* ========================================================================= */
uint64_t dqo_mix_seed(uint64_t seed, uint64_t salt) { /* quantize.cpp:13-18 */
    uint64_t z = seed + 0x9e3779b97f4a7c15ull * (salt + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* k-means++ pick, quantize.cpp:116-131; prob[] precomputed */
static size_t pick(mt64 *rng, const double *prob, size_t n) {
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) total += prob[i];
    if (!(total > 0.0)) return n;
    double r = uniform01(rng) * total;
    double cum = 0.0;
    size_t last_pos = n;
    for (size_t i = 0; i < n; ++i) {
        double p = prob[i];
        if (p <= 0.0) continue;
        last_pos = i;
        cum += p;
        if (cum >= r) return i;
    }
    return last_pos;
}

/* weighted_kmeanspp_init, quantize.cpp:94-164 */
int dqo_kmeanspp_init(const double *pts, const double *w, size_t n, uint32_t k, uint64_t seed,
                      double *out) {
    if (k == 0) return DQO_ERR;
    double total_w = 0.0;
    for (size_t i = 0; i < n; ++i) {
        if (!(w[i] >= 0.0)) return DQO_ERR;
        total_w += w[i];
    }
    if (!(total_w > 0.0)) return DQO_ERR;
    {
        double *d = malloc(n * sizeof(double) + 8);
        memcpy(d, pts, n * sizeof(double));
        sort_f64(d, n);
        size_t distinct = 0;
        for (size_t i = 0; i < n; ++i)
            if (i == 0 || !(d[i] == d[distinct - 1])) d[distinct++] = d[i];
        free(d);
        if (distinct < k) return DQO_ERR_TOO_FEW;
    }
    mt64 rng;
    mt64_seed(&rng, seed);
    double *d2 = malloc(n * sizeof(double) + 8), *prob = malloc(n * sizeof(double) + 8);
    for (size_t i = 0; i < n; ++i) d2[i] = INFINITY;
    uint32_t nc = 0;
#define ADD_CENTER(v)                                   \
    do {                                                \
        double v_ = (v);                                \
        out[nc++] = v_;                                 \
        for (size_t i_ = 0; i_ < n; ++i_) {             \
            double dd = pts[i_] - v_;                   \
            double sq = dd * dd;                        \
            d2[i_] = (sq < d2[i_]) ? sq : d2[i_];       \
        }                                               \
    } while (0)
    for (size_t i = 0; i < n; ++i) prob[i] = w[i];
    size_t first = pick(&rng, prob, n);
    ADD_CENTER(pts[first]);
    while (nc < k) {
        for (size_t i = 0; i < n; ++i) prob[i] = w[i] * d2[i];
        size_t next = pick(&rng, prob, n);
        int chosen = 0;
        if (next != n)
            for (uint32_t j = 0; j < nc; ++j)
                if (out[j] == pts[next]) chosen = 1;
        if (next == n || chosen) {
            for (size_t i = 0; i < n; ++i) {
                int c2 = 0;
                for (uint32_t j = 0; j < nc; ++j)
                    if (out[j] == pts[i]) c2 = 1;
                if (!c2) {
                    next = i;
                    break;
                }
            }
        }
        ADD_CENTER(pts[next]);
    }
#undef ADD_CENTER
    free(d2);
    free(prob);
    sort_f64(out, k);
    return DQO_OK;
}

/* weighted_sq_loss, quantize.cpp:166-178 */
double dqo_sq_loss(const double *pts, const double *w, size_t n, const double *c, uint32_t k) {
    double loss = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double best = INFINITY;
        for (uint32_t j = 0; j < k; ++j) {
            double d = pts[i] - c[j];
            double sq = d * d;
            best = (sq < best) ? sq : best; /* std::min(best, d*d) */
        }
        loss += w[i] * best;
    }
    return loss;
}

/* weighted_lloyd, quantize.cpp:180-254 (centers updated in place, sorted on return) */
int dqo_lloyd(const double *pts, const double *w, size_t n, double *centers, uint32_t k,
              double tol, uint32_t max_iter, uint32_t *iters_out) {
    if (k == 0) return DQO_ERR;
    double scale = 0.0;
    for (size_t i = 0; i < n; ++i) scale = fmax(scale, fabs(pts[i]));
    if (scale == 0.0) scale = 1.0;
    double *wsum = malloc(k * 8), *wxsum = malloc(k * 8), *next = malloc(k * 8);
    uint32_t *empties = malloc(k * 4);
    sv_pair *top = malloc((n + 1) * sizeof(sv_pair));
    uint32_t iters = 0;
    for (uint32_t it = 0; it < max_iter; ++it) {
        for (uint32_t j = 0; j < k; ++j) wsum[j] = wxsum[j] = 0.0;
        for (size_t i = 0; i < n; ++i) {
            double x = pts[i];
            uint32_t best = 0;
            double bd = fabs(x - centers[0]);
            for (uint32_t j = 1; j < k; ++j) {
                double d = fabs(x - centers[j]);
                if (d < bd) {
                    bd = d;
                    best = j;
                }
            }
            wsum[best] += w[i];
            wxsum[best] += w[i] * x;
        }
        uint32_t ne = 0;
        for (uint32_t j = 0; j < k; ++j) {
            if (wsum[j] > 0.0)
                next[j] = wxsum[j] / wsum[j];
            else
                empties[ne++] = j;
        }
        if (ne) {
            size_t nt = 0;
            for (size_t i = 0; i < n; ++i) {
                double x = pts[i];
                double bd = INFINITY;
                for (uint32_t j = 0; j < k; ++j) {
                    double d = fabs(x - centers[j]);
                    bd = (d < bd) ? d : bd; /* std::min(bd, d) */
                }
                double score = w[i] * bd * bd;
                if (score <= 0.0) continue;
                int dup = 0;
                for (size_t t = 0; t < nt; ++t)
                    if (top[t].v == x) {
                        dup = 1;
                        if (score > top[t].s) top[t].s = score;
                        break;
                    }
                if (dup) continue;
                top[nt].s = score;
                top[nt].v = x;
                nt++;
            }
            sort_pairs(top, nt);
            size_t c = 0;
            for (uint32_t e = 0; e < ne; ++e)
                if (c < nt) next[empties[e]] = top[c++].v;
        }
        double movement = 0.0;
        for (uint32_t j = 0; j < k; ++j) movement = fmax(movement, fabs(next[j] - centers[j]));
        memcpy(centers, next, k * 8);
        iters = it + 1;
        if (movement <= tol * scale) break;
    }
    sort_f64(centers, k);
    if (iters_out) *iters_out = iters;
    free(wsum);
    free(wxsum);
    free(next);
    free(empties);
    free(top);
    return DQO_OK;
}

/* approx_kmeans, quantize.cpp:256-325 */
int dqo_approx_kmeans(const float *values, size_t n, uint32_t k, double sigma, double alpha,
                      uint64_t seed, float *cb_out, uint32_t *len) {
    *len = 0;
    if (k == 0) return DQO_ERR;
    if (n == 0) return DQO_OK;
    if (!(sigma >= 0.0 && sigma <= 1.0)) return DQO_ERR;
    dqo_sketch s;
    int rc = dqo_sketch_init(&s, alpha);
    if (rc) return rc;
    dqo_sketch_add_f32(&s, values, n);
    size_t nb = dqo_sketch_nbuckets(&s);
    double *keys = malloc((nb + 1) * 8);
    uint64_t *counts = malloc((nb + 1) * 8);
    dqo_sketch_histogram(&s, keys, counts);
    dqo_sketch_free(&s);
    size_t np = nb;
    if (nb < k) {
        /* distinct-value fallback, quantize.cpp:280-300 */
        float *sorted = malloc(n * sizeof(float));
        memcpy(sorted, values, n * sizeof(float));
        sort_f32(sorted, n);
        free(keys);
        free(counts);
        keys = malloc(n * 8);
        counts = malloc(n * 8);
        np = 0;
        for (size_t i = 0; i < n; ++i) {
            float v = sorted[i];
            if (np == 0 || (double)v != keys[np - 1]) {
                keys[np] = v;
                counts[np++] = 1;
            } else
                ++counts[np - 1];
        }
        free(sorted);
        if (np <= k) {
            for (size_t i = 0; i < np; ++i) cb_out[i] = (float)keys[i];
            *len = (uint32_t)np;
            free(keys);
            free(counts);
            return DQO_OK;
        }
    }
    /* mix_weights, quantize.cpp:264-275 */
    double *w = malloc(np * 8);
    uint64_t maxc = 1;
    double maxk = 0.0;
    for (size_t i = 0; i < np; ++i) maxc = counts[i] > maxc ? counts[i] : maxc;
    for (size_t i = 0; i < np; ++i) maxk = fmax(maxk, fabs(keys[i]));
    for (size_t i = 0; i < np; ++i) {
        double nc = (double)counts[i] / (double)maxc;
        double nx = maxk > 0.0 ? fabs(keys[i]) / maxk : 0.0;
        w[i] = sigma * nc + (1.0 - sigma) * nx;
    }
    /* 8 restarts, quantize.cpp:306-317 */
    double *best_c = malloc(k * 8), *cand = malloc(k * 8);
    double best = INFINITY;
    int have = 0;
    for (uint32_t t = 0; t < 8; ++t) {
        rc = dqo_kmeanspp_init(keys, w, np, k, seed + t, cand);
        if (rc) break;
        dqo_lloyd(keys, w, np, cand, k, 1e-6, 100, NULL);
        double loss = dqo_sq_loss(keys, w, np, cand, k);
        if (loss < best) {
            best = loss;
            memcpy(best_c, cand, k * 8);
            have = 1;
        }
    }
    if (!rc && have) {
        uint32_t o = 0;
        for (uint32_t j = 0; j < k; ++j) {
            float f = (float)best_c[j];
            if (o == 0 || f != cb_out[o - 1]) cb_out[o++] = f;
        }
        *len = o;
    }
    free(best_c);
    free(cand);
    free(w);
    free(keys);
    free(counts);
    return rc;
}

/* nearest_center, quantize.cpp:327-335 */
uint32_t dqo_nearest_center(const float *c, uint32_t k, float v) {
    uint32_t lo = 0, hi = k; /* std::lower_bound: first c[i] >= v (i.e. !(c[i] < v)) */
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (c[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    if (lo == 0) return 0;
    if (lo == k) return k - 1;
    uint32_t h = lo, l = lo - 1;
    return (c[h] - v < v - c[l]) ? h : l;
}

uint16_t dqo_bf16_from_f32(float v) { /* quantize.cpp:337-342 */
    uint32_t bits;
    memcpy(&bits, &v, 4);
    bits += 0x7fffu + ((bits >> 16) & 1);
    return (uint16_t)(bits >> 16);
}
float dqo_bf16_to_f32(uint16_t v) {
    uint32_t bits = (uint32_t)v << 16;
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

/* ========================================================================= */
/* Partition + quantize — quantize.cpp:34-92, 373-425                         */
/* ========================================================================= */
static uint64_t *ckpt_numel(const dqo_ckpt *c) {
    uint64_t *n = malloc((c->nt + 1) * 8);
    size_t d = 0;
    for (uint32_t i = 0; i < c->nt; ++i) {
        uint64_t m = 1;
        for (uint8_t r = 0; r < c->ranks[i]; ++r) m *= c->dims[d++];
        n[i] = m;
    }
    return n;
}

int dqo_partition(const dqo_ckpt *c, const float *mag, const float *sens, const dqo_config *cfg,
                  uint8_t *part) {
    if (cfg->metric == 1 && !sens) return DQO_ERR_MISSING_SCORES;
    uint64_t *numel = ckpt_numel(c);
    uint64_t *off = malloc((c->nt + 1) * 8);
    off[0] = 0;
    for (uint32_t i = 0; i < c->nt; ++i) off[i + 1] = off[i] + numel[i];
    memset(part, 0, off[c->nt]);
    const float *ps = cfg->metric == 1 ? sens : mag;
    int rc = DQO_OK;
    for (int lt = 0; lt < 7 && !rc; ++lt) {
        int any = 0;
        for (uint32_t i = 0; i < c->nt; ++i) any |= (c->types[i] == lt);
        if (!any) continue;
        int do_prune = cfg->prune_frac > 0.0 && lt != 4;
        double t_prune = 0.0;
        if (do_prune) {
            dqo_sketch sk;
            if ((rc = dqo_sketch_init(&sk, cfg->alpha))) break;
            for (uint32_t i = 0; i < c->nt; ++i)
                if (c->types[i] == lt) dqo_sketch_add_f32(&sk, ps + off[i], numel[i]);
            rc = dqo_sketch_quantile(&sk, cfg->prune_frac, &t_prune);
            dqo_sketch_free(&sk);
            if (rc) break;
        }
        int do_protect = cfg->protect_frac > 0.0;
        double q_prot = 1.0 - cfg->protect_frac / 2.0;
        int protect_all = do_protect && q_prot <= 0.0;
        double t_mag = INFINITY, t_sens = INFINITY;
        if (do_protect && !protect_all) {
            dqo_sketch sk;
            if ((rc = dqo_sketch_init(&sk, cfg->alpha))) break;
            for (uint32_t i = 0; i < c->nt; ++i)
                if (c->types[i] == lt) dqo_sketch_add_f32(&sk, mag + off[i], numel[i]);
            rc = dqo_sketch_quantile(&sk, q_prot, &t_mag);
            dqo_sketch_free(&sk);
            if (rc) break;
            if (sens) {
                if ((rc = dqo_sketch_init(&sk, cfg->alpha))) break;
                for (uint32_t i = 0; i < c->nt; ++i)
                    if (c->types[i] == lt) dqo_sketch_add_f32(&sk, sens + off[i], numel[i]);
                rc = dqo_sketch_quantile(&sk, q_prot, &t_sens);
                dqo_sketch_free(&sk);
                if (rc) break;
            }
        }
        for (uint32_t i = 0; i < c->nt; ++i) {
            if (c->types[i] != lt) continue;
            for (uint64_t e = off[i]; e < off[i + 1]; ++e) {
                int prot = protect_all ||
                           (do_protect && ((double)mag[e] > t_mag || (sens && (double)sens[e] > t_sens)));
                if (prot)
                    part[e] = 2;
                else if (do_prune && (double)ps[e] <= t_prune)
                    part[e] = 1;
            }
        }
    }
    free(numel);
    free(off);
    return rc;
}

static char *xstrdup(const char *s) {
    size_t n = strlen(s);
    char *d = malloc(n + 1);
    memcpy(d, s, n + 1);
    return d;
}

static dqo_q *q_alloc_layout(const dqo_ckpt *c) {
    dqo_q *q = calloc(1, sizeof *q);
    q->nt = c->nt;
    q->t = calloc(c->nt + 1, sizeof(dqo_tensor));
    size_t d = 0;
    for (uint32_t i = 0; i < c->nt; ++i) {
        dqo_tensor *t = &q->t[i];
        t->name = xstrdup(c->names[i]);
        t->type = c->types[i];
        t->rank = c->ranks[i];
        t->dims = malloc((t->rank + 1) * 8);
        t->n = 1;
        for (uint8_t r = 0; r < t->rank; ++r) t->n *= (t->dims[r] = c->dims[d++]);
        t->levels = calloc(t->n + 1, 2);
    }
    return q;
}

int dqo_quantize(const dqo_ckpt *c, uint64_t step, const float *mag, const float *sens,
                 const dqo_config *cfg, uint64_t seed, dqo_q **out) {
    *out = NULL;
    if (cfg->bins < 1 || cfg->embed_bins < 1) return DQO_ERR;
    uint64_t *numel = ckpt_numel(c);
    uint64_t N = 0;
    for (uint32_t i = 0; i < c->nt; ++i) N += numel[i];
    uint8_t *part = malloc(N + 1);
    int rc = dqo_partition(c, mag, sens, cfg, part);
    if (rc) {
        free(part);
        free(numel);
        return rc;
    }
    dqo_q *q = q_alloc_layout(c);
    q->step = step;
    q->cfg = *cfg;
    float *vals = malloc(N * sizeof(float) + 4);
    for (int lt = 0; lt < 7 && !rc; ++lt) { /* quantize.cpp:382-394 */
        size_t nv = 0;
        uint64_t o = 0;
        for (uint32_t i = 0; i < c->nt; ++i) {
            if (c->types[i] == lt)
                for (uint64_t e = 0; e < numel[i]; ++e)
                    if (part[o + e] == 0) vals[nv++] = c->data[o + e];
            o += numel[i];
        }
        if (!nv) continue;
        uint32_t k = lt == 4 ? cfg->embed_bins : cfg->bins;
        q->cb[lt] = malloc(k * sizeof(float));
        rc = dqo_approx_kmeans(vals, nv, k, cfg->sigma, cfg->alpha, dqo_mix_seed(seed, (uint64_t)lt),
                               q->cb[lt], &q->cb_len[lt]);
    }
    free(vals);
    uint64_t o = 0;
    for (uint32_t i = 0; i < c->nt && !rc; ++i) { /* quantize.cpp:396-423 */
        dqo_tensor *t = &q->t[i];
        const float *cb = q->cb[t->type];
        uint32_t k = q->cb_len[t->type];
        uint16_t pruned = (uint16_t)k, prot = (uint16_t)(k + 1);
        uint64_t np = 0;
        for (uint64_t e = 0; e < t->n; ++e) np += part[o + e] == 2;
        t->nprot = np;
        t->ppos = malloc((np + 1) * 8);
        t->pval = malloc((np + 1) * 2);
        np = 0;
        for (uint64_t e = 0; e < t->n; ++e) {
            float v = c->data[o + e];
            switch (part[o + e]) {
                case 0: t->levels[e] = (uint16_t)dqo_nearest_center(cb, k, v); break;
                case 1: t->levels[e] = pruned; break;
                default:
                    t->levels[e] = prot;
                    t->ppos[np] = e;
                    t->pval[np++] = dqo_bf16_from_f32(v);
            }
        }
        o += t->n;
    }
    free(part);
    free(numel);
    if (rc) {
        dqo_q_free(q);
        return rc;
    }
    *out = q;
    return DQO_OK;
}

int dqo_dequantize(const dqo_q *q, float *out) { /* quantize.cpp:427-462 */
    uint64_t o = 0;
    for (uint32_t i = 0; i < q->nt; ++i) {
        const dqo_tensor *t = &q->t[i];
        const float *cb = q->cb[t->type];
        uint16_t pruned = (uint16_t)q->cb_len[t->type], prot = pruned + 1;
        uint64_t np = 0;
        for (uint64_t e = 0; e < t->n; ++e) {
            uint16_t l = t->levels[e];
            if (l < pruned)
                out[o + e] = cb[l];
            else if (l == pruned)
                out[o + e] = 0.0f;
            else if (l == prot) {
                if (np >= t->nprot || t->ppos[np] != e) return DQO_ERR_CORRUPT_INDEX;
                out[o + e] = dqo_bf16_to_f32(t->pval[np++]);
            } else
                return DQO_ERR_CORRUPT_INDEX;
        }
        if (np != t->nprot) return DQO_ERR_CORRUPT_INDEX;
        o += t->n;
    }
    return DQO_OK;
}

void dqo_q_free(dqo_q *q) {
    if (!q) return;
    for (uint32_t i = 0; i < q->nt; ++i) {
        free(q->t[i].name);
        free(q->t[i].dims);
        free(q->t[i].levels);
        free(q->t[i].ppos);
        free(q->t[i].pval);
    }
    free(q->t);
    for (int lt = 0; lt < 7; ++lt) free(q->cb[lt]);
    free(q);
}

uint64_t dqo_q_param_count(const dqo_q *q) {
    uint64_t n = 0;
    for (uint32_t i = 0; i < q->nt; ++i) n += q->t[i].n;
    return n;
}

uint32_t dqo_q_max_levels(const dqo_q *q) { /* quantize.cpp:357-365 */
    uint32_t m = 0;
    for (uint32_t i = 0; i < q->nt; ++i) {
        uint32_t l = q->cb_len[q->t[i].type] + 2;
        m = l > m ? l : m;
    }
    return m;
}

void dqo_q_levels(const dqo_q *q, uint16_t *out) {
    for (uint32_t i = 0; i < q->nt; ++i) {
        memcpy(out, q->t[i].levels, q->t[i].n * 2);
        out += q->t[i].n;
    }
}
void dqo_q_nprot(const dqo_q *q, uint64_t *out) {
    for (uint32_t i = 0; i < q->nt; ++i) out[i] = q->t[i].nprot;
}
void dqo_q_prot(const dqo_q *q, uint64_t *pos, uint16_t *val) {
    for (uint32_t i = 0; i < q->nt; ++i) {
        memcpy(pos, q->t[i].ppos, q->t[i].nprot * 8);
        memcpy(val, q->t[i].pval, q->t[i].nprot * 2);
        pos += q->t[i].nprot;
        val += q->t[i].nprot;
    }
}
uint32_t dqo_q_codebook(const dqo_q *q, int lt, float *out) {
    if (out && q->cb_len[lt]) memcpy(out, q->cb[lt], q->cb_len[lt] * 4);
    return q->cb_len[lt];
}

dqo_q *dqo_q_make(const dqo_ckpt *layout, uint64_t step, const dqo_config *cfg,
                  const uint32_t *cb_len, const float *cb_flat, const uint16_t *levels,
                  const uint64_t *nprot, const uint64_t *ppos, const uint16_t *pval) {
    dqo_q *q = q_alloc_layout(layout);
    q->step = step;
    q->cfg = *cfg;
    for (int lt = 0; lt < 7; ++lt) {
        q->cb_len[lt] = cb_len[lt];
        if (cb_len[lt]) {
            q->cb[lt] = malloc(cb_len[lt] * 4);
            memcpy(q->cb[lt], cb_flat, cb_len[lt] * 4);
            cb_flat += cb_len[lt];
        }
    }
    for (uint32_t i = 0; i < q->nt; ++i) {
        dqo_tensor *t = &q->t[i];
        memcpy(t->levels, levels, t->n * 2);
        levels += t->n;
        t->nprot = nprot[i];
        t->ppos = malloc((t->nprot + 1) * 8);
        t->pval = malloc((t->nprot + 1) * 2);
        memcpy(t->ppos, ppos, t->nprot * 8);
        memcpy(t->pval, pval, t->nprot * 2);
        ppos += t->nprot;
        pval += t->nprot;
    }
    return q;
}

/* ========================================================================= */
/* Codec — codec.cpp                                                          */
/* ========================================================================= */
int dqo_delta_compute(const uint16_t *prev, const uint16_t *cur, size_t n, uint32_t B,
                      uint16_t *out) { /* codec.cpp:12-24 */
    if (B == 0) return DQO_ERR;
    for (size_t i = 0; i < n; ++i) {
        if (prev[i] >= B || cur[i] >= B) return DQO_ERR_CORRUPT_INDEX;
        int32_t diff = (int32_t)prev[i] - (int32_t)cur[i];
        if (diff < 0) diff += (int32_t)B;
        out[i] = (uint16_t)diff;
    }
    return DQO_OK;
}

int dqo_delta_apply(const uint16_t *prev, const uint16_t *d, size_t n, uint32_t B,
                    uint16_t *out) { /* codec.cpp:26-37 */
    for (size_t i = 0; i < n; ++i) {
        if (prev[i] >= B || d[i] >= B) return DQO_ERR_CORRUPT_INDEX;
        int32_t v = (int32_t)prev[i] - (int32_t)d[i];
        if (v < 0) v += (int32_t)B;
        out[i] = (uint16_t)v;
    }
    return DQO_OK;
}

int dqo_rearrange(const uint16_t *d, const uint16_t *prev, size_t n, uint32_t B, uint16_t *out,
                  uint32_t *bucket_ids, uint64_t *sizes, uint32_t *ngroups) { /* codec.cpp:39-54 */
    uint64_t *cnt = calloc(B + 1, 8), *at = calloc(B + 1, 8);
    for (size_t i = 0; i < n; ++i) {
        if (prev[i] >= B) {
            free(cnt);
            free(at);
            return DQO_ERR_CORRUPT_INDEX;
        }
        cnt[prev[i]]++;
    }
    uint64_t o = 0;
    uint32_t g = 0;
    for (uint32_t b = 0; b < B; ++b) {
        at[b] = o;
        o += cnt[b];
        if (cnt[b]) {
            bucket_ids[g] = b;
            sizes[g++] = cnt[b];
        }
    }
    for (size_t i = 0; i < n; ++i) out[at[prev[i]]++] = d[i];
    *ngroups = g;
    free(cnt);
    free(at);
    return DQO_OK;
}

size_t dqo_rle_encode(const uint16_t *v, size_t n, int64_t *out) { /* codec.cpp:79-90 */
    size_t o = 0, i = 0;
    while (i < n) {
        size_t j = i;
        while (j < n && v[j] == v[i]) ++j;
        out[o++] = -(int64_t)v[i];
        if (j - i > 1) out[o++] = (int64_t)(j - i);
        i = j;
    }
    return o;
}

int dqo_rle_decode(const int64_t *s, size_t ns, uint64_t expected, uint16_t *out) {
    uint64_t o = 0; /* codec.cpp:92-107 */
    for (size_t i = 0; i < ns; ++i) {
        int64_t x = s[i];
        if (x > 0) return DQO_ERR_CORRUPT_BITSTREAM;
        if (-x > 0xffff) return DQO_ERR_CORRUPT_BITSTREAM;
        uint16_t v = (uint16_t)(-x);
        uint64_t run = 1;
        if (i + 1 < ns && s[i + 1] > 0) run = (uint64_t)s[++i];
        if (o + run > expected) return DQO_ERR_CORRUPT_BITSTREAM;
        for (uint64_t r = 0; r < run; ++r) out[o++] = v;
    }
    return o == expected ? DQO_OK : DQO_ERR_CORRUPT_BITSTREAM;
}

/* huffman_lengths, codec.cpp:137-189 */
typedef struct { uint64_t f; uint32_t order; int left, right; int64_t sym; } hnode;
static int hless(const hnode *a, int x, int y) { /* pq "top" = smallest (f, order) */
    if (a[x].f != a[y].f) return a[x].f < a[y].f;
    return a[x].order < a[y].order;
}
static void heap_push(int *h, size_t *n, const hnode *a, int v) {
    size_t i = (*n)++;
    h[i] = v;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (hless(a, h[i], h[p])) {
            int t = h[i];
            h[i] = h[p];
            h[p] = t;
            i = p;
        } else
            break;
    }
}
static int heap_pop(int *h, size_t *n, const hnode *a) {
    int top = h[0];
    h[0] = h[--(*n)];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && hless(a, h[l], h[m])) m = l;
        if (r < *n && hless(a, h[r], h[m])) m = r;
        if (m == i) break;
        int t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
    return top;
}
static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return x < y ? -1 : x > y;
}
typedef struct { int64_t sym; uint8_t len; } tentry;
static int cmp_tentry(const void *a, const void *b) {
    const tentry *x = a, *y = b;
    if (x->len != y->len) return x->len < y->len ? -1 : 1;
    return x->sym < y->sym ? -1 : x->sym > y->sym;
}

static int cmp_tentry_sym(const void *a, const void *b) {
    const tentry *x = a, *y = b;
    return x->sym < y->sym ? -1 : x->sym > y->sym;
}

static int huffman_lengths(const int64_t *s, size_t ns, tentry *table, size_t *tsize) {
    *tsize = 0;
    if (ns == 0) return DQO_OK;
    int64_t *sorted = malloc(ns * 8);
    memcpy(sorted, s, ns * 8);
    qsort(sorted, ns, 8, cmp_i64);
    size_t nd = 0;
    hnode *arena = malloc(2 * ns * sizeof(hnode) + sizeof(hnode));
    for (size_t i = 0; i < ns; ++i) { /* std::map<int64,uint64> freq, ascending key */
        if (i == 0 || sorted[i] != sorted[i - 1]) {
            arena[nd].f = 0;
            arena[nd].order = (uint32_t)nd;
            arena[nd].left = arena[nd].right = -1;
            arena[nd].sym = sorted[i];
            nd++;
        }
        arena[nd - 1].f++;
    }
    free(sorted);
    if (nd == 1) {
        table[0].sym = arena[0].sym;
        table[0].len = 1;
        *tsize = 1;
        free(arena);
        return DQO_OK;
    }
    int *heap = malloc(2 * nd * sizeof(int));
    size_t hn = 0, na = nd;
    for (size_t i = 0; i < nd; ++i) heap_push(heap, &hn, arena, (int)i);
    while (hn > 1) {
        int a = heap_pop(heap, &hn, arena);
        int b = heap_pop(heap, &hn, arena);
        arena[na].f = arena[a].f + arena[b].f;
        arena[na].order = (uint32_t)na;
        arena[na].left = a;
        arena[na].right = b;
        arena[na].sym = 0;
        heap_push(heap, &hn, arena, (int)na);
        na++;
    }
    /* depth-first walk, codec.cpp:172-184 */
    int *st = malloc(2 * na * sizeof(int));
    uint8_t *sd = malloc(2 * na);
    size_t sp = 0, o = 0;
    st[sp] = heap[0];
    sd[sp++] = 0;
    int rc = DQO_OK;
    while (sp) {
        --sp;
        int idx = st[sp];
        uint8_t depth = sd[sp];
        if (arena[idx].left < 0) {
            table[o].sym = arena[idx].sym;
            table[o++].len = depth;
        } else {
            if (depth >= 63) { rc = DQO_ERR; break; }
            st[sp] = arena[idx].left; sd[sp++] = depth + 1;
            st[sp] = arena[idx].right; sd[sp++] = depth + 1;
        }
    }
    qsort(table, o, sizeof(tentry), cmp_tentry);
    *tsize = o;
    free(st);
    free(sd);
    free(heap);
    free(arena);
    return rc;
}

/* assign_codes, codec.cpp:197-214 */
static int assign_codes(const tentry *t, size_t n, uint64_t *codes, uint8_t *max_len) {
    uint64_t code = 0, kraft = 0;
    uint8_t prev = n ? t[0].len : 0;
    *max_len = 0;
    for (size_t i = 0; i < n; ++i) {
        uint8_t len = t[i].len;
        if (len == 0 || len > 63 || len < prev) return DQO_ERR_CORRUPT_BITSTREAM;
        code <<= (len - prev);
        codes[i] = code++;
        prev = len;
        *max_len = len;
        kraft += 1ull << (63 - len);
        if (kraft > (1ull << 63)) return DQO_ERR_CORRUPT_BITSTREAM;
    }
    return DQO_OK;
}

typedef struct { uint8_t *b; size_t n, cap; } bytebuf;
static void bb_reserve(bytebuf *w, size_t extra) {
    if (w->n + extra > w->cap) {
        size_t c = w->cap ? w->cap : 256;
        while (c < w->n + extra) c *= 2;
        w->b = realloc(w->b, c);
        w->cap = c;
    }
}
static void bb_raw(bytebuf *w, const void *p, size_t n) {
    bb_reserve(w, n);
    memcpy(w->b + w->n, p, n);
    w->n += n;
}
static void bb_u8(bytebuf *w, uint8_t v) { bb_raw(w, &v, 1); }
static void bb_le(bytebuf *w, uint64_t v, int nb) {
    bb_reserve(w, nb);
    for (int i = 0; i < nb; ++i) w->b[w->n++] = (uint8_t)(v >> (8 * i));
}
static void bb_uvarint(bytebuf *w, uint64_t v) { /* bytes.hpp:36-42 */
    while (v >= 0x80) {
        bb_u8(w, (uint8_t)(v | 0x80));
        v >>= 7;
    }
    bb_u8(w, (uint8_t)v);
}
static void bb_svarint(bytebuf *w, int64_t v) { bb_uvarint(w, ((uint64_t)v << 1) ^ (uint64_t)(v >> 63)); }
static void bb_f64(bytebuf *w, double v) { uint64_t b; memcpy(&b, &v, 8); bb_le(w, b, 8); }
static void bb_f32(bytebuf *w, float v) { uint32_t b; memcpy(&b, &v, 4); bb_le(w, b, 4); }

/* huffman_encode, codec.cpp:218-232 with BitWriter :111-122 */
static int huff_encode(const int64_t *s, size_t ns, tentry *table, size_t *tsize, bytebuf *bits) {
    int rc = huffman_lengths(s, ns, table, tsize);
    if (rc) return rc;
    uint64_t *codes = malloc((*tsize + 1) * 8);
    uint8_t ml;
    if ((rc = assign_codes(table, *tsize, codes, &ml))) { free(codes); return rc; }
    /* std::map<sym,(code,len)> lookup, codec.cpp:222-224: sorted copy + bsearch */
    tentry *bysym = malloc((*tsize + 1) * sizeof(tentry));
    uint64_t *code_of = malloc((*tsize + 1) * 8);
    for (size_t j = 0; j < *tsize; ++j) bysym[j] = table[j];
    qsort(bysym, *tsize, sizeof(tentry), cmp_tentry_sym);
    for (size_t j = 0; j < *tsize; ++j) {
        size_t lo = 0, hi = *tsize;
        while (hi - lo > 1) { size_t m = (lo + hi) / 2; if (table[m].len < bysym[j].len || (table[m].len == bysym[j].len && table[m].sym <= bysym[j].sym)) lo = m; else hi = m; }
        code_of[j] = codes[lo];
    }
    int used = 0;
    for (size_t i = 0; i < ns; ++i) {
        size_t lo = 0, hi = *tsize;
        while (hi - lo > 1) { size_t m = (lo + hi) / 2; if (bysym[m].sym <= s[i]) lo = m; else hi = m; }
        uint64_t code = code_of[lo];
        int len = bysym[lo].len;
        for (int b = len - 1; b >= 0; --b) {
            if (used == 0) bb_u8(bits, 0);
            bits->b[bits->n - 1] |= (uint8_t)(((code >> b) & 1) << (7 - used));
            used = (used + 1) & 7;
        }
    }
    free(codes);
    free(bysym);
    free(code_of);
    return DQO_OK;
}

int dqo_huffman_encode(const int64_t *s, size_t ns, int64_t *tsym, uint8_t *tlen, size_t *tsize,
                       uint8_t **bytes, size_t *nbytes) {
    tentry *t = malloc((ns + 1) * sizeof(tentry));
    bytebuf bb = {0};
    int rc = huff_encode(s, ns, t, tsize, &bb);
    for (size_t i = 0; i < *tsize; ++i) tsym[i] = t[i].sym, tlen[i] = t[i].len;
    free(t);
    *bytes = bb.b;
    *nbytes = bb.n;
    return rc;
}

/* huffman_decode, codec.cpp:234-273 */
int dqo_huffman_decode(const int64_t *tsym, const uint8_t *tlen, size_t tsize,
                       const uint8_t *bytes, size_t nbytes, uint64_t count, int64_t *out) {
    if (count == 0) return DQO_OK;
    if (tsize == 0) return DQO_ERR_CORRUPT_BITSTREAM;
    for (size_t i = 1; i < tsize; ++i)
        if (tlen[i] < tlen[i - 1] || (tlen[i] == tlen[i - 1] && tsym[i] <= tsym[i - 1]))
            return DQO_ERR_CORRUPT_BITSTREAM;
    tentry *t = malloc(tsize * sizeof(tentry));
    uint64_t *codes = malloc(tsize * 8);
    if (!t || !codes) { free(t); free(codes); return DQO_ERR; }
    for (size_t i = 0; i < tsize; ++i) t[i].sym = tsym[i], t[i].len = tlen[i];
    uint8_t ml;
    int rc = assign_codes(t, tsize, codes, &ml);
    if (rc) { free(t); free(codes); return rc; }
    uint64_t first_code[64] = {0};
    size_t first_idx[64] = {0}, len_count[64] = {0};
    for (size_t i = 0; i < tsize; ++i) {
        uint8_t len = tlen[i];
        if (len_count[len] == 0) first_code[len] = codes[i], first_idx[len] = i;
        ++len_count[len];
    }
    size_t pos = 0, nbits = nbytes * 8;
    for (uint64_t n = 0; n < count && !rc; ++n) {
        uint64_t cur = 0;
        uint8_t len = 0;
        for (;;) {
            if (pos >= nbits) { rc = DQO_ERR_CORRUPT_BITSTREAM; break; }
            cur = (cur << 1) | (uint64_t)((bytes[pos >> 3] >> (7 - (pos & 7))) & 1);
            ++pos;
            ++len;
            if (len > ml) { rc = DQO_ERR_CORRUPT_BITSTREAM; break; }
            if (len_count[len] && cur >= first_code[len] && cur - first_code[len] < len_count[len]) {
                out[n] = tsym[first_idx[len] + (size_t)(cur - first_code[len])];
                break;
            }
        }
    }
    free(t);
    free(codes);
    return rc;
}

/* crc32, codec.cpp:275-288 */
uint32_t dqo_crc32(const uint8_t *data, size_t n) {
    static uint32_t table[256];
    static int init = 0;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xedb88320u ^ (c >> 1) : c >> 1;
            table[i] = c;
        }
        init = 1;
    }
    uint32_t c = 0xffffffffu;
    for (size_t i = 0; i < n; ++i) c = table[(c ^ data[i]) & 0xff] ^ (c >> 8);
    return c ^ 0xffffffffu;
}

/* encode_tensor_payload, codec.cpp:308-327 */
static int encode_payload(bytebuf *w, const uint16_t *prev, const uint16_t *cur, uint64_t n,
                          uint32_t B) {
    uint16_t *d = malloc(n * 2 + 2), *r = malloc(n * 2 + 2);
    uint32_t *ids = malloc((B + 1) * 4);
    uint64_t *sizes = malloc((B + 1) * 8);
    uint32_t ng = 0;
    int rc = dqo_delta_compute(prev, cur, n, B, d);
    if (!rc) rc = dqo_rearrange(d, prev, n, B, r, ids, sizes, &ng);
    int64_t *sym = malloc((2 * n + 1) * 8);
    tentry *t = malloc((2 * n + 1) * sizeof(tentry));
    if (!rc) {
        bb_uvarint(w, ng);
        uint64_t o = 0;
        for (uint32_t g = 0; g < ng && !rc; ++g) {
            size_t ns = dqo_rle_encode(r + o, sizes[g], sym);
            size_t tsize;
            bytebuf bits = {0};
            rc = huff_encode(sym, ns, t, &tsize, &bits);
            bb_uvarint(w, ids[g]);
            bb_uvarint(w, sizes[g]);
            bb_uvarint(w, ns);
            bb_uvarint(w, tsize);
            for (size_t i = 0; i < tsize; ++i) {
                bb_svarint(w, t[i].sym);
                bb_u8(w, t[i].len);
            }
            bb_uvarint(w, bits.n);
            bb_raw(w, bits.b, bits.n);
            free(bits.b);
            o += sizes[g];
        }
    }
    free(d); free(r); free(ids); free(sizes); free(sym); free(t);
    return rc;
}

static void write_config(bytebuf *w, const dqo_config *c) { /* codec.cpp:374-382 */
    bb_le(w, c->bins, 4);
    bb_le(w, c->embed_bins, 4);
    bb_f64(w, c->prune_frac);
    bb_f64(w, c->protect_frac);
    bb_u8(w, (uint8_t)c->metric);
    bb_f64(w, c->sigma);
    bb_f64(w, c->alpha);
}

static uint32_t level_stream_crc(const dqo_q *q) { /* codec.cpp:295-306 + crc32 */
    uint64_t total = dqo_q_param_count(q);
    uint8_t *bytes = malloc(total * 2 + 1);
    uint64_t o = 0;
    for (uint32_t i = 0; i < q->nt; ++i)
        for (uint64_t e = 0; e < q->t[i].n; ++e) {
            bytes[o++] = (uint8_t)q->t[i].levels[e];
            bytes[o++] = (uint8_t)(q->t[i].levels[e] >> 8);
        }
    uint32_t c = dqo_crc32(bytes, o);
    free(bytes);
    return c;
}

/* encode_delta_record, codec.cpp:398-460 */
int dqo_encode_record(const dqo_q *base, const dqo_q *target, double quality, uint8_t **out,
                      size_t *n) {
    *out = NULL;
    *n = 0;
    if (base) {
        if (base->nt != target->nt) return DQO_ERR_SHAPE;
        for (uint32_t i = 0; i < base->nt; ++i) {
            const dqo_tensor *a = &base->t[i], *b = &target->t[i];
            if (strcmp(a->name, b->name) || a->rank != b->rank || a->type != b->type ||
                memcmp(a->dims, b->dims, a->rank * 8))
                return DQO_ERR_SHAPE;
        }
    }
    uint32_t B = target->nt ? dqo_q_max_levels(target) : 0;
    if (base) {
        uint32_t bb = base->nt ? dqo_q_max_levels(base) : 0;
        B = bb > B ? bb : B;
    }
    if (B == 0) B = 2;
    bytebuf w = {0};
    bb_raw(&w, "DQDR", 4);
    bb_le(&w, 1, 4);
    bb_u8(&w, base ? 1 : 0);
    bb_le(&w, base ? base->step : 0, 8);
    bb_le(&w, target->step, 8);
    bb_le(&w, B, 4);
    write_config(&w, &target->cfg);
    bb_f64(&w, quality);
    uint8_t nlt = 0;
    for (int lt = 0; lt < 7; ++lt) nlt += target->cb_len[lt] != 0;
    bb_u8(&w, nlt);
    for (int lt = 0; lt < 7; ++lt) {
        if (!target->cb_len[lt]) continue;
        bb_u8(&w, (uint8_t)lt);
        bb_le(&w, target->cb_len[lt], 4);
        for (uint32_t j = 0; j < target->cb_len[lt]; ++j) bb_f32(&w, target->cb[lt][j]);
    }
    bb_le(&w, target->nt, 4);
    int rc = DQO_OK;
    for (uint32_t i = 0; i < target->nt && !rc; ++i) {
        const dqo_tensor *t = &target->t[i];
        size_t nl = strlen(t->name);
        bb_le(&w, nl, 2);
        bb_raw(&w, t->name, nl);
        bb_u8(&w, t->type);
        bb_u8(&w, t->rank);
        for (uint8_t r = 0; r < t->rank; ++r) bb_le(&w, t->dims[r], 8);
        bb_uvarint(&w, t->nprot);
        uint64_t pp = 0;
        for (uint64_t p = 0; p < t->nprot; ++p) {
            bb_uvarint(&w, p == 0 ? t->ppos[p] : t->ppos[p] - pp);
            bb_le(&w, t->pval[p], 2);
            pp = t->ppos[p];
        }
        uint16_t *zero = NULL;
        const uint16_t *prev = base ? base->t[i].levels : (zero = calloc(t->n + 1, 2));
        rc = encode_payload(&w, prev, t->levels, t->n, B);
        free(zero);
    }
    if (rc) { free(w.b); return rc; }
    bb_le(&w, level_stream_crc(target), 4);
    *out = w.b;
    *n = w.n;
    return DQO_OK;
}

/* ByteReader, bytes.hpp:56-132 */
typedef struct { const uint8_t *p; size_t n, pos; int err; } rd;
static int rd_need(rd *r, size_t k) {
    if (r->err) return 0;
    if (r->pos + k > r->n) { r->err = DQO_ERR_TRUNCATED; return 0; }
    return 1;
}
static uint64_t rd_le(rd *r, int nb) {
    if (!rd_need(r, nb)) return 0;
    uint64_t v = 0;
    for (int i = 0; i < nb; ++i) v |= (uint64_t)r->p[r->pos + i] << (8 * i);
    r->pos += nb;
    return v;
}
static uint64_t rd_uvarint(rd *r) {
    uint64_t v = 0;
    int shift = 0;
    for (;;) {
        uint8_t b = (uint8_t)rd_le(r, 1);
        if (r->err) return 0;
        v |= (uint64_t)(b & 0x7f) << shift;
        if (!(b & 0x80)) break;
        shift += 7;
        if (shift > 63) { r->err = DQO_ERR_TRUNCATED; return 0; }
    }
    return v;
}
static int64_t rd_svarint(rd *r) { uint64_t u = rd_uvarint(r); return (int64_t)(u >> 1) ^ -(int64_t)(u & 1); }
static double rd_f64(rd *r) { uint64_t b = rd_le(r, 8); double v; memcpy(&v, &b, 8); return v; }
static float rd_f32(rd *r) { uint32_t b = (uint32_t)rd_le(r, 4); float v; memcpy(&v, &b, 4); return v; }

/* decode_tensor_payload, codec.cpp:329-357 */
static int decode_payload(rd *r, const uint16_t *prev, uint64_t n, uint32_t B, uint16_t *out) {
    uint64_t ng = rd_uvarint(r);
    if (r->err) return r->err;
    uint16_t *deltas = malloc(n * 2 + 2);
    uint64_t *next = calloc(B + 1, 8), *start = calloc(B + 1, 8), *gsz = calloc(B + 1, 8);
    uint8_t *have = calloc(B + 1, 1);
    uint16_t *grouped = malloc(n * 2 + 2); /* concatenated group payloads */
    if (!deltas || !next || !start || !gsz || !have || !grouped) {
        free(deltas); free(next); free(start); free(gsz); free(have); free(grouped);
        return DQO_ERR; /* absurd element count from a corrupt shape */
    }
    uint64_t total = 0;
    int rc = DQO_OK;
    for (uint64_t g = 0; g < ng && !rc; ++g) {
        uint64_t bucket = rd_uvarint(r), elems = rd_uvarint(r), nsyms = rd_uvarint(r),
                 tsize = rd_uvarint(r);
        if (r->err) { rc = r->err; break; }
        /* absurd counts from corrupt varints: the reference's reserve() throws
           std::length_error / bad_alloc (no dqt type); every table entry takes >= 2
           bytes and every symbol >= 1 bit, so they are reported as truncation /
           corrupt bitstream here instead of crashing the checker */
        if (tsize > (r->n - r->pos) / 2) { rc = DQO_ERR_TRUNCATED; break; }
        int64_t *ts = malloc((tsize + 1) * 8);
        uint8_t *tl = malloc(tsize + 1);
        for (uint64_t i = 0; i < tsize; ++i) ts[i] = rd_svarint(r), tl[i] = (uint8_t)rd_le(r, 1);
        uint64_t nb = rd_uvarint(r);
        if (!r->err) rd_need(r, nb);
        if (r->err) { rc = r->err; free(ts); free(tl); break; }
        const uint8_t *bytes = r->p + r->pos;
        r->pos += nb;
        if (nsyms > nb * 8) { rc = DQO_ERR_CORRUPT_BITSTREAM; free(ts); free(tl); break; }
        int64_t *syms = malloc((nsyms + 1) * 8);
        rc = dqo_huffman_decode(ts, tl, tsize, bytes, nb, nsyms, syms);
        if (!rc && total + elems > n) rc = DQO_ERR_CORRUPT_INDEX;
        if (!rc) rc = dqo_rle_decode(syms, nsyms, elems, grouped + total);
        if (!rc) {
            if (bucket >= B) rc = DQO_ERR_CORRUPT_INDEX;
            else if (have[bucket]) rc = DQO_ERR_CORRUPT_INDEX;
            else { have[bucket] = 1; start[bucket] = total; gsz[bucket] = elems; }
        }
        total += elems;
        free(ts); free(tl); free(syms);
    }
    if (!rc && total != n) rc = DQO_ERR_CORRUPT_INDEX;
    for (uint64_t i = 0; i < n && !rc; ++i) { /* unrearrange, codec.cpp:56-77 */
        uint16_t src = prev[i];
        if (src >= B || !have[src] || next[src] >= gsz[src]) { rc = DQO_ERR_CORRUPT_INDEX; break; }
        deltas[i] = grouped[start[src] + next[src]++];
    }
    for (uint32_t b = 0; b < B && !rc; ++b)
        if (have[b] && next[b] != gsz[b]) rc = DQO_ERR_CORRUPT_INDEX;
    if (!rc) rc = dqo_delta_apply(prev, deltas, n, B, out);
    free(deltas); free(next); free(start); free(gsz); free(have); free(grouped);
    return rc;
}

/* decode_delta_record, codec.cpp:513-597 */
int dqo_decode_record(const uint8_t *rec, size_t n, const dqo_q *base, dqo_q **out) {
    *out = NULL;
    rd r = {rec, n, 0, 0};
    if (!rd_need(&r, 4)) return r.err;
    if (memcmp(rec, "DQDR", 4)) return DQO_ERR_BAD_MAGIC;
    r.pos = 4;
    if (rd_le(&r, 4) != 1) return r.err ? r.err : DQO_ERR_IO;
    int has_base = rd_le(&r, 1) != 0;
    uint64_t base_step = rd_le(&r, 8), target_step = rd_le(&r, 8);
    uint32_t B = (uint32_t)rd_le(&r, 4);
    if (r.err) return r.err;
    if (has_base && !base) return DQO_ERR_CHAIN;
    if (!has_base) base = NULL;
    if (base && base->step != base_step) return DQO_ERR_CHAIN;
    dqo_q *q = calloc(1, sizeof *q);
    q->step = target_step;
    q->cfg.bins = (uint32_t)rd_le(&r, 4);
    q->cfg.embed_bins = (uint32_t)rd_le(&r, 4);
    q->cfg.prune_frac = rd_f64(&r);
    q->cfg.protect_frac = rd_f64(&r);
    q->cfg.metric = (uint32_t)rd_le(&r, 1);
    q->cfg.sigma = rd_f64(&r);
    q->cfg.alpha = rd_f64(&r);
    rd_f64(&r);
    int rc = DQO_OK;
    uint8_t nlt = (uint8_t)rd_le(&r, 1);
    for (uint8_t i = 0; i < nlt && !r.err && !rc; ++i) {
        uint8_t lt = (uint8_t)rd_le(&r, 1);
        if (lt >= 7) { rc = DQO_ERR_CORRUPT_INDEX; break; }
        uint32_t len = (uint32_t)rd_le(&r, 4);
        if (r.err) break;
        if (!rd_need(&r, (size_t)len * 4)) break;
        free(q->cb[lt]);
        q->cb[lt] = malloc((size_t)len * 4 + 4);
        q->cb_len[lt] = len;
        for (uint32_t j = 0; j < len; ++j) q->cb[lt][j] = rd_f32(&r);
    }
    uint32_t nt = (uint32_t)rd_le(&r, 4);
    if (!rc && !r.err && base && base->nt != nt) rc = DQO_ERR_CHAIN;
    /* an absurd tensor count (corrupt input): reported as truncation, see decode_payload */
    if (!rc && !r.err && nt > (r.n - r.pos) / 4) rc = DQO_ERR_TRUNCATED;
    if (!rc && !r.err) {
        q->t = calloc(nt + 1, sizeof(dqo_tensor));
        q->nt = 0;
    }
    for (uint32_t i = 0; i < nt && !rc && !r.err; ++i) {
        dqo_tensor *t = &q->t[q->nt++];
        uint16_t nl = (uint16_t)rd_le(&r, 2);
        if (!rd_need(&r, nl)) break;
        t->name = malloc(nl + 1);
        memcpy(t->name, rec + r.pos, nl);
        t->name[nl] = 0;
        r.pos += nl;
        uint8_t lt = (uint8_t)rd_le(&r, 1);
        if (!r.err && lt >= 7) { rc = DQO_ERR_CORRUPT_INDEX; break; }
        t->type = lt;
        t->rank = (uint8_t)rd_le(&r, 1);
        t->dims = malloc((t->rank + 1) * 8);
        t->n = 1;
        for (uint8_t d = 0; d < t->rank; ++d) t->n *= (t->dims[d] = rd_le(&r, 8));
        if (r.err) break;
        /* checker limit: a corrupt shape must not make the test process allocate (and
           zero) terabytes; real test tensors are far below 2^30 elements */
        if (t->n > (1ull << 30)) { rc = DQO_ERR; break; }
        uint64_t np = rd_uvarint(&r);
        if (r.err) break;
        if (np > t->n) { rc = DQO_ERR_CORRUPT_INDEX; break; }
        t->nprot = np;
        if (np > (r.n - r.pos) / 3) { rc = DQO_ERR_TRUNCATED; break; } /* >= 3 bytes each (corrupt count) */
        t->ppos = malloc((np + 1) * 8);
        t->pval = malloc((np + 1) * 2);
        uint64_t pos = 0;
        for (uint64_t p = 0; p < np && !r.err; ++p) {
            uint64_t dd = rd_uvarint(&r);
            pos = p == 0 ? dd : pos + dd;
            if (pos >= t->n || (p > 0 && dd == 0)) { rc = DQO_ERR_CORRUPT_INDEX; break; }
            t->ppos[p] = pos;
            t->pval[p] = (uint16_t)rd_le(&r, 2);
        }
        if (rc || r.err) break;
        uint16_t *zero = NULL;
        const uint16_t *prev;
        if (base) {
            const dqo_tensor *bt = &base->t[i];
            if (strcmp(bt->name, t->name) || bt->rank != t->rank || bt->type != t->type ||
                memcmp(bt->dims, t->dims, t->rank * 8)) { rc = DQO_ERR_CHAIN; break; }
            prev = bt->levels;
        } else
            prev = zero = calloc(t->n + 1, 2);
        t->levels = malloc(t->n * 2 + 2);
        if (!prev || !t->levels) { free(zero); rc = DQO_ERR; break; }
        rc = decode_payload(&r, prev, t->n, B, t->levels);
        free(zero);
        if (rc) break;
        uint32_t maxl = q->cb_len[t->type] + 1;
        for (uint64_t e = 0; e < t->n; ++e)
            if (t->levels[e] > maxl) { rc = DQO_ERR_CORRUPT_INDEX; break; }
    }
    if (!rc && r.err) rc = r.err;
    if (!rc) {
        uint32_t stored = (uint32_t)rd_le(&r, 4);
        if (r.err) rc = r.err;
        else if (r.pos != r.n) rc = DQO_ERR_IO;
        else if (level_stream_crc(q) != stored) rc = DQO_ERR_CHECKSUM;
    }
    if (rc) { dqo_q_free(q); return rc; }
    *out = q;
    return DQO_OK;
}

/* payload_bytes_pe/rle/he, codec.cpp:601-646 */
uint64_t dqo_payload_bytes(const dqo_q *base, const dqo_q *target, int variant) {
    uint32_t B = dqo_q_max_levels(base), bt = dqo_q_max_levels(target);
    B = bt > B ? bt : B;
    uint64_t total = 0;
    for (uint32_t i = 0; i < target->nt; ++i) {
        uint64_t n = target->t[i].n;
        bytebuf w = {0};
        if (variant == 0) {
            encode_payload(&w, base->t[i].levels, target->t[i].levels, n, B);
            total += w.n;
        } else {
            uint16_t *d = malloc(n * 2 + 2);
            dqo_delta_compute(base->t[i].levels, target->t[i].levels, n, B, d);
            int64_t *sym = malloc((2 * n + 1) * 8);
            size_t ns;
            if (variant == 1)
                ns = dqo_rle_encode(d, n, sym);
            else {
                for (uint64_t e = 0; e < n; ++e) sym[e] = d[e];
                ns = n;
            }
            tentry *t = malloc((ns + 1) * sizeof(tentry));
            size_t tsize;
            bytebuf bits = {0};
            huff_encode(sym, ns, t, &tsize, &bits);
            bb_uvarint(&w, ns);
            bb_uvarint(&w, tsize);
            for (size_t j = 0; j < tsize; ++j) { bb_svarint(&w, t[j].sym); bb_u8(&w, t[j].len); }
            bb_uvarint(&w, bits.n);
            total += w.n + bits.n;
            free(bits.b); free(t); free(sym); free(d);
        }
        free(w.b);
    }
    return total;
}

void dqo_free(void *p) { free(p); }

/* ========================================================================= */
/* Evaluation — search.cpp:30-105                                             */
/* ========================================================================= */
double dqo_proxy_quality(const dqo_ckpt *orig, const float *recon) {
    double diff_sq[7] = {0}, orig_sq[7] = {0};
    uint64_t count[7] = {0};
    uint64_t *numel = ckpt_numel(orig);
    uint64_t o = 0;
    for (uint32_t i = 0; i < orig->nt; ++i) {
        int lt = orig->types[i];
        for (uint64_t e = 0; e < numel[i]; ++e) {
            double a = (double)orig->data[o + e], b = (double)recon[o + e];
            double d = a - b;
            diff_sq[lt] += d * d;
            orig_sq[lt] += a * a;
        }
        count[lt] += numel[i];
        o += numel[i];
    }
    free(numel);
    uint64_t total = 0;
    for (int lt = 0; lt < 7; ++lt) total += count[lt];
    if (total == 0) return 0.0;
    double quality = 0.0;
    for (int lt = 0; lt < 7; ++lt) {
        if (count[lt] == 0) continue;
        double rel;
        if (orig_sq[lt] > 0.0)
            rel = sqrt(diff_sq[lt] / orig_sq[lt]);
        else
            rel = diff_sq[lt] > 0.0 ? 1.0 : 0.0;
        quality += ((double)count[lt] / (double)total) * rel;
    }
    return quality;
}

double dqo_estimate_compression(const dqo_ckpt *c, const dqo_q *q) {
    uint64_t *numel = ckpt_numel(c);
    uint64_t pc = 0;
    for (uint32_t i = 0; i < c->nt; ++i) pc += numel[i];
    free(numel);
    double raw = 4.0 * (double)pc;
    double est = 64.0;
    for (uint32_t i = 0; i < q->nt; ++i) {
        const dqo_tensor *t = &q->t[i];
        uint32_t levels = q->cb_len[t->type] + 2;
        uint64_t *counts = calloc(levels + 40, 8);
        for (uint64_t e = 0; e < t->n; ++e) ++counts[t->levels[e]];
        double n = (double)t->n;
        double bits = 0.0;
        for (uint32_t l = 0; l < levels; ++l) {
            if (!counts[l]) continue;
            double p = (double)counts[l] / n;
            bits -= (double)counts[l] * log2(p);
        }
        free(counts);
        est += bits / 8.0;
        est += 10.0 * (double)t->nprot;
    }
    for (int lt = 0; lt < 7; ++lt) est += 4.0 * (double)q->cb_len[lt];
    return raw / est;
}

uint64_t dqo_config_hash(const dqo_config *cfg) { /* search.cpp:87-101 */
#define F2U(v) ({ double v_ = (v); uint64_t u_; memcpy(&u_, &v_, 8); u_; })
    uint64_t h = dqo_mix_seed(cfg->bins, 1);
    h = dqo_mix_seed(h ^ cfg->embed_bins, 2);
    h = dqo_mix_seed(h ^ F2U(cfg->prune_frac), 3);
    h = dqo_mix_seed(h ^ F2U(cfg->protect_frac), 4);
    h = dqo_mix_seed(h ^ (uint64_t)cfg->metric, 5);
    h = dqo_mix_seed(h ^ F2U(cfg->sigma), 6);
    h = dqo_mix_seed(h ^ F2U(cfg->alpha), 7);
#undef F2U
    return h;
}

uint64_t dqo_quantize_seed(uint64_t search_seed, const dqo_config *cfg) {
    return dqo_mix_seed(search_seed, dqo_config_hash(cfg));
}

/* ========================================================================= */
/* Synthetic trajectory — trajectory.cpp                                      */
/* ========================================================================= */
typedef struct { mt64 gen; double spare; int have; } nrng;
static double nrng_u(nrng *r) { return ((double)(mt64_next(&r->gen) >> 11) + 0.5) * 0x1.0p-53; }
static double nrng_next(nrng *r) { /* trajectory.cpp:22-33 */
    if (r->have) { r->have = 0; return r->spare; }
    double u = nrng_u(r), v = nrng_u(r);
    double rr = sqrt(-2.0 * log(u));
    r->spare = rr * sin(2.0 * M_PI * v);
    r->have = 1;
    return rr * cos(2.0 * M_PI * v);
}

int dqo_generate_trajectory(const uint64_t *numel, uint32_t nt, uint32_t steps, double lr0,
                            double decay, double noise, uint64_t seed, float *wout, float *gout) {
    if (steps < 2 || !(decay > 0.0 && decay <= 1.0) || !(lr0 > 0.0)) return DQO_ERR;
    const double kInit = 0.05; /* trajectory.cpp:10 */
    uint64_t N = 0;
    for (uint32_t i = 0; i < nt; ++i) N += numel[i];
    nrng r;
    mt64_seed(&r.gen, seed);
    r.have = 0;
    float *w = malloc(N * 4 + 4);
    for (uint64_t e = 0; e < N; ++e) w[e] = (float)(kInit * nrng_next(&r));
    double lr = lr0;
    for (uint32_t s = 0; s < steps; ++s) { /* trajectory.cpp:92-111 */
        float *ws = wout + (uint64_t)s * N, *gs = gout + (uint64_t)s * N;
        memcpy(ws, w, N * 4);
        for (uint64_t e = 0; e < N; ++e) gs[e] = w[e] + (float)(noise * kInit * nrng_next(&r));
        for (uint64_t e = 0; e < N; ++e) w[e] -= (float)lr * gs[e];
        lr *= decay;
    }
    free(w);
    return DQO_OK;
}

void dqo_default_layout(uint64_t params, uint64_t *numel, uint8_t *types, uint8_t *ranks,
                        uint64_t *dims) { /* trajectory.cpp:38-73 */
    static const double frac[9] = {0.15, 0.20, 0.10, 0.175, 0.165, 0.08, 0.005, 0.005, 0.12};
    static const uint8_t ty[9] = {4, 2, 2, 1, 1, 0, 3, 5, 6};
    static const int flat[9] = {0, 0, 0, 0, 0, 0, 1, 1, 0};
    for (int i = 0; i < 9; ++i) {
        long long r = llround(frac[i] * (double)params);
        uint64_t n = (uint64_t)r < 4 ? 4 : (uint64_t)r;
        types[i] = ty[i];
        if (flat[i]) {
            ranks[i] = 1;
            dims[2 * i] = n;
            dims[2 * i + 1] = 0;
            numel[i] = n;
        } else {
            uint64_t cols = 1;
            while (cols * cols < n) ++cols;
            uint64_t rows = (n + cols - 1) / cols;
            ranks[i] = 2;
            dims[2 * i] = rows;
            dims[2 * i + 1] = cols;
            numel[i] = rows * cols;
        }
    }
}
