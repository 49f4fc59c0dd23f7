/*
 * dqt_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference (DynaQuant `dqt`, /root/reference/proj)
 * checkpoint-compression hot path: sketch, scores, partition, histogram
 * k-means, level assignment, cyclic delta + rearrange + RLE + canonical
 * Huffman + CRC, DQDR record encode/decode, proxy evaluation.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker / CPU baseline.  The product
 * (paper_2306_11800_b200) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_pin.py checks every function here against
 * the reference compiled from its own sources (oracle/_ref, see Makefile) and
 * against the known-answer values of the reference's own unit tests
 * (tests/test_*.cpp in the reference); the C1 golden fingerprint (FULL record
 * CRC dcf04bba, DELTA aaaae4e6 — SURVEY.md §8c) is reproduced in
 * tests/test_oracle_pin.py.
 */
#ifndef DQT_ORACLE_H
#define DQT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { DQO_OK = 0, DQO_ERR = 1, DQO_ERR_EMPTY_SKETCH = 2, DQO_ERR_Q_RANGE = 3,
       DQO_ERR_TOO_FEW = 4, DQO_ERR_CORRUPT_INDEX = 5, DQO_ERR_CORRUPT_BITSTREAM = 6,
       DQO_ERR_CHECKSUM = 7, DQO_ERR_SHAPE = 8, DQO_ERR_CHAIN = 9, DQO_ERR_TRUNCATED = 10,
       DQO_ERR_BAD_MAGIC = 11, DQO_ERR_IO = 12, DQO_ERR_MISSING_SCORES = 13 };

typedef struct dqo_config {
    uint32_t bins, embed_bins;
    double prune_frac, protect_frac;
    uint32_t metric; /* 0 magnitude, 1 sensitivity */
    double sigma, alpha;
} dqo_config;

/* ---- sketch (sketch.cpp) ---------------------------------------------- */
int64_t dqo_bucket_index(double alpha, double abs_x);
double dqo_representative(double alpha, int64_t k);
/* Dense sketch over float inputs: counts for k in [kmin, kmax] per sign. */
typedef struct dqo_sketch {
    double alpha, gamma, inv_ln_gamma, rep_scale;
    int64_t kmin, kmax;
    uint64_t zero, total;
    uint64_t *pos, *neg;
} dqo_sketch;
int dqo_sketch_init(dqo_sketch *s, double alpha);
void dqo_sketch_free(dqo_sketch *s);
void dqo_sketch_add_f32(dqo_sketch *s, const float *x, size_t n);
int dqo_sketch_quantile(const dqo_sketch *s, double q, double *out);
/* keys/counts must hold at least dqo_sketch_nbuckets(s) entries */
size_t dqo_sketch_nbuckets(const dqo_sketch *s);
size_t dqo_sketch_histogram(const dqo_sketch *s, double *keys, uint64_t *counts);
/* convenience for ctypes: build over x and return the dense arrays */
int dqo_sketch_dense(const float *x, size_t n, double alpha, int64_t *kmin, int64_t *kmax,
                     uint64_t *zero, uint64_t *pos_out, uint64_t *neg_out);
void dqo_sketch_range(double alpha, int64_t *kmin, int64_t *kmax);

/* ---- ranker (ranker.cpp) ---------------------------------------------- */
void dqo_ema_update(float *ema, const float *g, size_t n, double beta);
void dqo_scores(const float *w, const float *ema, size_t n, float *mag, float *sens);

/* ---- std::sort (libstdc++ introsort) faithful port --------------------- */
void dqo_sort_f32(float *v, size_t n);
void dqo_sort_f64(double *v, size_t n);
/* pairs (score, value) sorted by score descending, as quantize.cpp:238-239 */
void dqo_sort_pairs_desc(double *score, double *value, size_t n);

/* ---- clustering (quantize.cpp) ---------------------------------------- */
uint64_t dqo_mix_seed(uint64_t seed, uint64_t salt);
int dqo_kmeanspp_init(const double *pts, const double *w, size_t n, uint32_t k, uint64_t seed,
                      double *centers_out);
int dqo_lloyd(const double *pts, const double *w, size_t n, double *centers, uint32_t k,
              double tol, uint32_t max_iter, uint32_t *iters_out);
double dqo_sq_loss(const double *pts, const double *w, size_t n, const double *c, uint32_t k);
/* codebook out must hold k floats; returns length in *len */
int dqo_approx_kmeans(const float *values, size_t n, uint32_t k, double sigma, double alpha,
                      uint64_t seed, float *cb_out, uint32_t *len);
uint32_t dqo_nearest_center(const float *c, uint32_t k, float v);
uint16_t dqo_bf16_from_f32(float v);
float dqo_bf16_to_f32(uint16_t v);

/* ---- quantized state ---------------------------------------------------- */
typedef struct dqo_tensor {
    char *name;
    uint8_t type, rank;
    uint64_t *dims;
    uint64_t n;
    uint16_t *levels;
    uint64_t nprot;
    uint64_t *ppos;
    uint16_t *pval;
} dqo_tensor;
typedef struct dqo_q {
    uint64_t step;
    dqo_config cfg;
    uint32_t cb_len[7];
    float *cb[7];
    uint32_t nt;
    dqo_tensor *t;
} dqo_q;

/* Checkpoint given flat: data[] holds all tensors concatenated in order. */
typedef struct dqo_ckpt {
    uint32_t nt;
    const char *const *names;
    const uint8_t *types;
    const uint8_t *ranks;
    const uint64_t *dims; /* concatenated */
    const float *data;
} dqo_ckpt;

/* partition (quantize.cpp:34-92): part[] per element, 0 quantize 1 prune 2 protect */
int dqo_partition(const dqo_ckpt *c, const float *mag, const float *sens, const dqo_config *cfg,
                  uint8_t *part);
int dqo_quantize(const dqo_ckpt *c, uint64_t step, const float *mag, const float *sens,
                 const dqo_config *cfg, uint64_t seed, dqo_q **out);
/* dequantize (quantize.cpp:427-462) into flat out[] */
int dqo_dequantize(const dqo_q *q, float *out);
void dqo_q_free(dqo_q *q);
uint64_t dqo_q_param_count(const dqo_q *q);
uint32_t dqo_q_max_levels(const dqo_q *q);
/* accessors for ctypes */
void dqo_q_levels(const dqo_q *q, uint16_t *out);
void dqo_q_nprot(const dqo_q *q, uint64_t *out);
void dqo_q_prot(const dqo_q *q, uint64_t *pos, uint16_t *val);
uint32_t dqo_q_codebook(const dqo_q *q, int lt, float *out);
/* build a state from arrays (levels flat, protected flat with per-tensor counts) */
dqo_q *dqo_q_make(const dqo_ckpt *layout, uint64_t step, const dqo_config *cfg,
                  const uint32_t *cb_len, const float *cb_flat, const uint16_t *levels,
                  const uint64_t *nprot, const uint64_t *ppos, const uint16_t *pval);

/* ---- codec (codec.cpp) -------------------------------------------------- */
int dqo_delta_compute(const uint16_t *prev, const uint16_t *cur, size_t n, uint32_t B,
                      uint16_t *out);
int dqo_delta_apply(const uint16_t *prev, const uint16_t *d, size_t n, uint32_t B, uint16_t *out);
/* stable group-by prev level: out_deltas in group order; bucket_ids/group_sizes (<=B) */
int dqo_rearrange(const uint16_t *d, const uint16_t *prev, size_t n, uint32_t B, uint16_t *out,
                  uint32_t *bucket_ids, uint64_t *sizes, uint32_t *ngroups);
/* returns symbol count; out must hold 2n */
size_t dqo_rle_encode(const uint16_t *v, size_t n, int64_t *out);
int dqo_rle_decode(const int64_t *s, size_t ns, uint64_t expected, uint16_t *out);
/* Huffman: table (sym,len) sorted by (len,sym); returns table size; bytes malloc'd */
int dqo_huffman_encode(const int64_t *s, size_t ns, int64_t *tsym, uint8_t *tlen, size_t *tsize,
                       uint8_t **bytes, size_t *nbytes);
int dqo_huffman_decode(const int64_t *tsym, const uint8_t *tlen, size_t tsize,
                       const uint8_t *bytes, size_t nbytes, uint64_t count, int64_t *out);
uint32_t dqo_crc32(const uint8_t *data, size_t n);
int dqo_encode_record(const dqo_q *base, const dqo_q *target, double quality, uint8_t **out,
                      size_t *n);
int dqo_decode_record(const uint8_t *rec, size_t n, const dqo_q *base, dqo_q **out);
uint64_t dqo_payload_bytes(const dqo_q *base, const dqo_q *target, int variant /*0 pe 1 rle 2 he*/);
void dqo_free(void *p);

/* ---- evaluation (search.cpp:30-85) -------------------------------------- */
double dqo_proxy_quality(const dqo_ckpt *orig, const float *recon);
double dqo_estimate_compression(const dqo_ckpt *c, const dqo_q *q);
uint64_t dqo_config_hash(const dqo_config *cfg);
uint64_t dqo_quantize_seed(uint64_t search_seed, const dqo_config *cfg);

/* ---- synthetic trajectory (trajectory.cpp) ------------------------------ */
/* Fills w[steps][N] and g[steps][N] for the given layout (numel per tensor). */
int dqo_generate_trajectory(const uint64_t *numel, uint32_t nt, uint32_t steps, double lr0,
                            double decay, double noise, uint64_t seed, float *w, float *g);
/* default_layout (trajectory.cpp:38-73): 9 tensors; writes numel[9], rows/cols */
void dqo_default_layout(uint64_t params, uint64_t *numel, uint8_t *types, uint8_t *ranks,
                        uint64_t *dims /* 2 per tensor */);

#ifdef __cplusplus
}
#endif
#endif
