/*
 * dqtg.h — C ABI of the B200 checkpoint-compression engine (libdqtg.so).
 *
 * Plain pointers and sizes only; no torch/CUDA types in the signatures
 * (streams are passed as an opaque void*).  Every entry point replaces one
 * function (or one loop) of the reference library `dqt`
 * (/root/reference/proj); the replaced interface is cited next to each
 * declaration.  The C++ drop-in library (include/dqt/ headers, libdqt.so) and the
 * Python module (dqt._dqt) are thin hosts over this ABI; INTEGRATION.md shows
 * the binding a maintainer adds to the reference to call it directly.
 *
 * Pointers named `*_any` may be host or device memory (detected with
 * cudaPointerGetAttributes); everything else is host memory unless the name
 * says `_dev`.  All calls are synchronous with respect to the host unless
 * stated otherwise and are serialised per engine (thread-safe).
 *
 * Errors: every call returns a dqtg_status; dqtg_last_error() returns the
 * message of the last failure on the calling thread.  Status codes map 1:1 to
 * the reference exception types (include/dqt/errors.hpp:8-39).
 */
#ifndef DQTG_H
#define DQTG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dqtg_status {
    DQTG_OK = 0,
    DQTG_ERROR = 1,                 /* dqt::Error */
    DQTG_BAD_MAGIC = 2,             /* dqt::BadMagic */
    DQTG_TRUNCATED = 3,             /* dqt::TruncatedFile */
    DQTG_SHAPE_MISMATCH = 4,        /* dqt::ShapeMismatch */
    DQTG_NON_FINITE = 5,            /* dqt::NonFiniteData */
    DQTG_IO = 6,                    /* dqt::IoError */
    DQTG_ALPHA_OUT_OF_RANGE = 7,    /* dqt::AlphaOutOfRange */
    DQTG_ALPHA_MISMATCH = 8,        /* dqt::AlphaMismatch */
    DQTG_EMPTY_SKETCH = 9,          /* dqt::EmptySketch */
    DQTG_MISSING_GRADIENTS = 10,    /* dqt::MissingGradients */
    DQTG_MISSING_SCORES = 11,       /* dqt::MissingScores */
    DQTG_TOO_FEW_DISTINCT = 12,     /* dqt::TooFewDistinctPoints */
    DQTG_CORRUPT_INDEX = 13,        /* dqt::CorruptIndex */
    DQTG_CORRUPT_BITSTREAM = 14,    /* dqt::CorruptBitstream */
    DQTG_CHECKSUM_MISMATCH = 15,    /* dqt::ChecksumMismatch */
    DQTG_CHAIN_CORRUPT = 16,        /* dqt::ChainCorrupt */
    DQTG_CUDA = 17                  /* CUDA runtime failure (surfaces as dqt::Error) */
} dqtg_status;

const char *dqtg_last_error(void);
const char *dqtg_version(void);

/* ---- engine ------------------------------------------------------------ */
typedef struct dqtg_engine dqtg_engine;
/* device: CUDA ordinal; stream: cudaStream_t to run on (NULL = an engine-owned
 * non-blocking stream; pass cudaStreamLegacy to run on the legacy default stream). */
dqtg_status dqtg_engine_create(int device, void *stream, dqtg_engine **out);
void dqtg_engine_destroy(dqtg_engine *e);
dqtg_status dqtg_engine_sync(dqtg_engine *e);
/* number of engine kernels launched so far (bench `gpu_launches`) */
uint64_t dqtg_engine_launches(const dqtg_engine *e);
/* per-kernel CUDA-event timing on the engine stream: enable, then read a JSON
 * object {"kernel": [launches, total_ms], ...} (resets the accumulated spans). */
dqtg_status dqtg_engine_profile(dqtg_engine *e, int enable);
dqtg_status dqtg_engine_profile_report(dqtg_engine *e, char *json, uint64_t cap);
/* host synchronisations of the engine stream so far and the host time blocked in them */
void dqtg_engine_sync_stats(const dqtg_engine *e, uint64_t *syncs, double *blocked_ms);

/* dqt::QuantConfig (quantize.hpp:13-26) */
typedef struct dqtg_config {
    uint32_t bins, embed_bins;
    double prune_frac, protect_frac;
    uint32_t metric; /* 0 = MAGNITUDE, 1 = SENSITIVITY (ranker.hpp:26) */
    double sigma, alpha;
} dqtg_config;

/* Checkpoint layout: tensors in checkpoint order (tensor.hpp:28-45). */
typedef struct dqtg_layout {
    uint32_t n_tensors;
    const char *const *names;   /* may be NULL when no record is produced */
    const uint8_t *types;       /* dqt::LayerType 0..6 */
    const uint8_t *ranks;
    const uint64_t *dims;       /* concatenated shapes */
} dqtg_layout;

/* ---- sketch: replaces sketch_build(const float*, n, alpha) (sketch.cpp:131-148)
 * Bucket counts over k in [kmin, kmax] (dqtg_sketch_range) for each sign plus the
 * zero bucket; pos/neg are host arrays of kmax-kmin+1 entries. */
dqtg_status dqtg_sketch_range(double alpha, int64_t *kmin, int64_t *kmax);
dqtg_status dqtg_sketch_build(dqtg_engine *e, const float *x_any, uint64_t n, double alpha,
                              uint64_t *zero, uint64_t *pos, uint64_t *neg);

/* ---- ranker: ema_update (ranker.cpp:21-37), compute_scores (ranker.cpp:79-101) */
dqtg_status dqtg_ema_update(dqtg_engine *e, float *ema_any, const float *g_any, uint64_t n,
                            double beta);
dqtg_status dqtg_compute_scores(dqtg_engine *e, const float *w_any, const float *ema_any,
                                uint64_t n, float *mag_any, float *sens_any);

/* ---- device checkpoint (weights + scores resident in HBM) ---------------- */
typedef struct dqtg_ckpt dqtg_ckpt;
dqtg_status dqtg_ckpt_create(dqtg_engine *e, const dqtg_layout *layout, dqtg_ckpt **out);
void dqtg_ckpt_destroy(dqtg_ckpt *c);
/* per-tensor weight pointers (tensor.hpp:30 NamedTensor::data) */
dqtg_status dqtg_ckpt_set_weights(dqtg_ckpt *c, const float *const *tensors_any);
/* frees the checkpoint's device buffers (weights, EMA, scores); the layout stays and the
 * next dqtg_ckpt_set_weights / set_ema allocates them again (a shard processed in
 * stages keeps only its current inputs resident; no reference counterpart) */
dqtg_status dqtg_ckpt_release(dqtg_ckpt *c);
/* explicit ScoreSet (ranker.hpp:34-42); sens may be NULL (has_sensitivity=false) */
dqtg_status dqtg_ckpt_set_scores(dqtg_ckpt *c, const float *const *mag_any,
                                 const float *const *sens_any);
/* scores derived on device from the EMA: magnitude |w|, sensitivity |e*w| fused into the
 * histogram / assign passes (compute_scores never materialised).  ema may be NULL. */
dqtg_status dqtg_ckpt_set_ema(dqtg_ckpt *c, const float *const *ema_any);
/* ema_update on the device-resident EMA (first call seeds it) */
dqtg_status dqtg_ckpt_update_ema(dqtg_ckpt *c, const float *const *grads_any, double beta);
uint64_t dqtg_ckpt_param_count(const dqtg_ckpt *c);
/* flat padded device buffers (for device-resident producers, e.g. the bench) */
float *dqtg_ckpt_weights_dev(dqtg_ckpt *c);
float *dqtg_ckpt_ema_dev(dqtg_ckpt *c);
/* element offset of tensor i inside the padded buffers */
uint64_t dqtg_ckpt_tensor_offset(const dqtg_ckpt *c, uint32_t i);
/* layout of tensor i (name NUL-terminated into cap bytes; dims holds `rank` entries) */
uint32_t dqtg_ckpt_tensor_count(const dqtg_ckpt *c);
dqtg_status dqtg_ckpt_tensor_info(const dqtg_ckpt *c, uint32_t i, char *name, uint64_t cap,
                                  uint8_t *type, uint8_t *rank, uint64_t *dims);
/* copy the weights back (tensor i -> out_any[i], numel floats; NULL entries skipped) */
dqtg_status dqtg_ckpt_download(dqtg_ckpt *c, float *const *out_any);
/* apply_layer_rules (src/tensor.cpp:225-227): replace the layer types (n_tensors entries) */
dqtg_status dqtg_ckpt_set_types(dqtg_ckpt *c, const uint8_t *types);

/* ---- DQT1 ingest: replaces read_checkpoint + validate (src/tensor.cpp:63-75,
 * 110-149) on the compress path.  Parses the tensor headers on the host (same
 * checks and status codes, in the same order), streams the data sections through
 * pinned staging chunks into a new device checkpoint (`threads` reader threads,
 * 0 = 8), and checks NaN/Inf on the device (DQTG_NON_FINITE names the first bad
 * tensor).  *step = Checkpoint::step; the meta section is returned raw
 * (u32 count | {u16 len, key | u32 len, value}) into meta[0..meta_cap), its
 * full length in *meta_len.  DQTG_INGEST_DIRECT reads with O_DIRECT (bypassing the
 * page cache) where the filesystem allows it. */
#define DQTG_INGEST_DIRECT 1
dqtg_status dqtg_ckpt_read_dqt1(dqtg_engine *e, const char *path, int flags, int threads,
                                dqtg_ckpt **out, uint64_t *step, uint8_t *meta,
                                uint64_t meta_cap, uint64_t *meta_len);

/* ---- quantized state (QuantizedCheckpoint, quantize.hpp:86-110) ----------- */
typedef struct dqtg_qstate dqtg_qstate;
typedef struct dqtg_qstate_info {
    uint64_t step;
    dqtg_config config;
    uint32_t codebook_len[7];
    uint32_t max_levels;
    uint64_t param_count;
    uint64_t protected_total;
} dqtg_qstate_info;

/* quantize_checkpoint(c, scores, cfg, seed) (quantize.cpp:373-425) */
dqtg_status dqtg_quantize(dqtg_engine *e, const dqtg_ckpt *c, const dqtg_config *cfg,
                          uint64_t seed, uint64_t step, dqtg_qstate **out);
dqtg_status dqtg_qstate_info_get(const dqtg_qstate *q, dqtg_qstate_info *info);
/* per-tensor protected counts (n_tensors entries) */
dqtg_status dqtg_qstate_protected_counts(const dqtg_qstate *q, uint64_t *counts);
/* copy out: levels[i] (numel_i u16), prot_pos[i]/prot_val[i] (count_i each), codebooks[lt]
 * (codebook_len[lt] floats).  Any pointer array may be NULL to skip that part. */
/* layout of a state (e.g. one made by dqtg_decode_record): tensor count; per tensor
 * its name (NUL-terminated, truncated to cap bytes), layer type, rank and dims[rank] */
uint32_t dqtg_qstate_tensor_count(const dqtg_qstate *s);
dqtg_status dqtg_qstate_tensor_info(const dqtg_qstate *s, uint32_t i, char *name, uint64_t cap,
                                    uint8_t *type, uint8_t *rank, uint64_t *dims);
dqtg_status dqtg_qstate_download(const dqtg_qstate *q, uint16_t *const *levels,
                                 uint64_t *const *prot_pos, uint16_t *const *prot_val,
                                 float *const *codebooks);
/* build a state from host arrays (encode_delta_record on caller-made states) */
dqtg_status dqtg_qstate_upload(dqtg_engine *e, const dqtg_layout *layout, uint64_t step,
                               const dqtg_config *cfg, const uint32_t *codebook_len,
                               const float *const *codebooks, const uint16_t *const *levels,
                               const uint64_t *prot_count, const uint64_t *const *prot_pos,
                               const uint16_t *const *prot_val, dqtg_qstate **out);
void dqtg_qstate_destroy(dqtg_qstate *q);
uint16_t *dqtg_qstate_levels_dev(dqtg_qstate *q);
/* dequantize_checkpoint (quantize.cpp:427-462) into per-tensor outputs */
dqtg_status dqtg_dequantize(dqtg_engine *e, const dqtg_qstate *q, float *const *out_any);

/* ---- DQDR records (codec.cpp:398-597) ---------------------------------- */
typedef struct dqtg_record dqtg_record;
/* encode_delta_record(base, target, quality_delta); base NULL = FULL record */
dqtg_status dqtg_encode_record(dqtg_engine *e, const dqtg_qstate *base,
                               const dqtg_qstate *target, double quality_delta,
                               dqtg_record **out);
/* payload_bytes_pe / _rle / _he (codec.cpp:615-646): encode_tensor_payload bytes of
 * the delta base -> target summed over tensors (variant 0), or the Huffman payload
 * size of the un-rearranged RLE stream (1) / of the raw deltas (2), computed by the
 * device encoder in its ablation modes; no record is written. */
dqtg_status dqtg_payload_bytes(dqtg_engine *e, const dqtg_qstate *base, const dqtg_qstate *target,
                               int variant, uint64_t *bytes);
uint64_t dqtg_record_size(const dqtg_record *r);
dqtg_status dqtg_record_copy(const dqtg_record *r, void *dst_host);
const uint8_t *dqtg_record_dev(const dqtg_record *r);
void dqtg_record_destroy(dqtg_record *r);
/* decode_delta_record(record, base) (codec.cpp:513-597) */
dqtg_status dqtg_decode_record(dqtg_engine *e, const uint8_t *rec, uint64_t n,
                               const dqtg_qstate *base, dqtg_qstate **out);
/* Chain::restore (chain.cpp:131-154): host records recs[0..n) decoded in order, each
 * against the previous one (recs[0] against base, or none for a FULL record); the host
 * walk of record k+1 overlaps the device decode of record k.  fn(user, k, state) sees
 * every decoded state (borrowed for the call); *last_out receives the last one. */
typedef void (*dqtg_state_fn)(void *user, uint64_t k, const dqtg_qstate *state);
dqtg_status dqtg_decode_chain(dqtg_engine *e, uint32_t n, const uint8_t *const *recs,
                              const uint64_t *sizes, const dqtg_qstate *base, dqtg_state_fn fn,
                              void *user, dqtg_qstate **last_out);

/* ---- tensor-sharded checkpoints (multi-GPU) ----------------
 * Thresholds and codebooks must come from the histograms of the WHOLE
 * checkpoint.  Each rank quantizes its shard in three stages; between them the
 * caller sums the u64 histogram buffers over all ranks (ncclAllReduce / any
 * collective, exact and order independent):
 *   stage1 -> score_hist [2*7*HS]      (all-reduce SUM)
 *   stage2 -> value_hist [7*HS]        (all-reduce SUM)
 *   stage3 -> quantized state of this shard (codebooks identical on every rank)
 * Buffers are device memory (dqtg_shard_hist_len entries of u64). */
uint64_t dqtg_shard_hist_len(dqtg_engine *e, const dqtg_config *cfg, int which /*0 score, 1 value*/);
dqtg_status dqtg_shard_stage1(dqtg_engine *e, const dqtg_ckpt *c, const dqtg_config *cfg,
                              uint64_t *score_hist_dev);
dqtg_status dqtg_shard_stage2(dqtg_engine *e, const dqtg_ckpt *c, const dqtg_config *cfg,
                              const uint64_t *score_hist_dev, uint64_t *value_hist_dev);
dqtg_status dqtg_shard_stage3(dqtg_engine *e, const dqtg_ckpt *c, const dqtg_config *cfg,
                              uint64_t seed, uint64_t step, const uint64_t *value_hist_dev,
                              dqtg_qstate **out);
/* encode this shard's tensor blocks with the GLOBAL alphabet B (max over ranks of
 * max_levels, codec.cpp:416-417) and the global tensor count; bytes
 * [*body_offset, size-4) are this rank's blocks, the last 4 bytes the CRC-32 of
 * its level stream (combine across ranks with the zlib crc32_combine rule). */
dqtg_status dqtg_encode_record_shard(dqtg_engine *e, const dqtg_qstate *base,
                                     const dqtg_qstate *target, double quality_delta,
                                     uint32_t global_B, uint32_t global_tensors,
                                     dqtg_record **out, uint64_t *body_offset);

/* ---- fused step: compute_scores + quantize_checkpoint + encode_delta_record
 * (the path Chain::append + cmd_compress run, chain.cpp:86-129 / dqt.cpp:208-210) */
dqtg_status dqtg_compress_step(dqtg_engine *e, const dqtg_ckpt *c, const dqtg_config *cfg,
                               uint64_t seed, uint64_t step, const dqtg_qstate *base,
                               double quality_delta, dqtg_qstate **state_out,
                               dqtg_record **record_out);

/* ---- NCCL communicator and the sharded step (multi-GPU) ------------
 * One process per GPU.  Rank 0 makes an id (dqtg_comm_unique_id), the caller passes
 * it to every rank out of band (e.g. torch.distributed.broadcast_object_list, MPI,
 * a file), and each rank calls dqtg_comm_init with its engine.  NCCL is loaded at
 * run time (libnccl.so.2).
 * dqtg_compress_sharded runs one Chain::append step (chain.cpp:86-129) of a
 * tensor-sharded checkpoint: `c` holds this rank's tensors (contiguous in the global
 * tensor order, rank order = tensor order), `base` this rank's previous state (null:
 * FULL record).  The score and value histograms are all-reduced on the engine
 * stream, every rank quantizes and encodes its own tensors, and rank 0 receives the
 * record of the whole checkpoint in *record_out (byte-identical to the single-GPU
 * dqtg_compress_step record; other ranks get null).  n_tensors_total = 0: the sum of
 * the ranks' tensor counts.  Replaces the reference's single-process
 * quantize_checkpoint + encode_delta_record (quantize.cpp:373-425, codec.cpp:398-460). */
#define DQTG_COMM_ID_BYTES 128
typedef struct dqtg_comm dqtg_comm;
dqtg_status dqtg_comm_unique_id(uint8_t *id_out /* DQTG_COMM_ID_BYTES */);
dqtg_status dqtg_comm_init(dqtg_engine *e, const uint8_t *id, int nranks, int rank,
                           dqtg_comm **out);
void dqtg_comm_destroy(dqtg_comm *c);
int dqtg_comm_rank(const dqtg_comm *c);
int dqtg_comm_size(const dqtg_comm *c);
/* in-place sum of a device u64 buffer over the ranks, on the engine stream */
dqtg_status dqtg_comm_allreduce_u64(dqtg_engine *e, dqtg_comm *c, uint64_t *buf_dev, uint64_t n);
dqtg_status dqtg_compress_sharded(dqtg_engine *e, dqtg_comm *c, const dqtg_ckpt *ckpt,
                                  const dqtg_config *cfg, uint64_t seed, uint64_t step,
                                  const dqtg_qstate *base, double quality_delta,
                                  uint32_t n_tensors_total, dqtg_qstate **state_out,
                                  dqtg_record **record_out);

/* ---- pipelined delta chain (Chain::append over a series, chain.cpp:86-129) ----
 * A pool of `workers` engines, each on its own CUDA stream and host thread.
 * Snapshot k runs on worker k mod W: quantized, then encoded as a delta against
 * snapshot k-1 (the stream waits on the event recorded after quantize(k-1));
 * states are released once both encodes that read them are done.  Records are
 * identical to dqtg_compress_step run in order.
 * weights[k * n_tensors + i] = tensor i of snapshot k (`_any`); ema[k * n_tensors
 * + i] = tensor i of snapshot k's gradient EMA (`_any`; the array null: magnitude
 * scores only).  A snapshot (or EMA) whose tensors form one device buffer in the
 * engine's padded layout (tensor i at base + off_i, as a dqtg_ckpt holds it) is
 * read in place; other snapshots are copied into a worker buffer first.  on_record(user, k, record) runs on a worker
 * thread (calls may arrive out of step order; the record is valid during the
 * call).  *last_out (optional) receives the state of the last snapshot. */
typedef struct dqtg_pipe dqtg_pipe;
typedef void (*dqtg_record_fn)(void *user, uint64_t k, const dqtg_record *record);
dqtg_status dqtg_pipe_create(int device, int workers, dqtg_pipe **out);
void dqtg_pipe_destroy(dqtg_pipe *p);
uint64_t dqtg_pipe_launches(const dqtg_pipe *p);
/* Orders every later dqtg_pipe_run's device work after the work queued on
 * `stream` (a cudaStream_t; null: none) before the run, and makes `stream` wait
 * for all workers at the end, so events recorded on it bracket the whole chain. */
void dqtg_pipe_set_stream(dqtg_pipe *p, void *stream);
/* Multi-GPU worker pool: one communicator per worker (n == workers; 0 clears).  Every
 * rank runs dqtg_pipe_run over its shard of each snapshot; snapshot k's sharded step
 * (dqtg_compress_sharded) runs on worker k mod W with comms[k mod W]; on_record is
 * called on rank 0 only, with the whole record. */
dqtg_status dqtg_pipe_set_comms(dqtg_pipe *p, dqtg_comm *const *comms, int n,
                                uint32_t n_tensors_total);
dqtg_status dqtg_pipe_run(dqtg_pipe *p, const dqtg_layout *layout,
                          const float *const *weights_any, uint64_t n_snapshots,
                          const uint64_t *steps, const float *const *ema_any,
                          const dqtg_config *cfg, uint64_t seed, const dqtg_qstate *base,
                          double quality_delta, dqtg_record_fn on_record, void *user,
                          dqtg_qstate **last_out);

/* partition_params (quantize.cpp:34-92): per-element part codes, 0 quantize,
 * 1 prune, 2 protect, written to masks[i] (numel_i bytes each) */
dqtg_status dqtg_partition(dqtg_engine *e, const dqtg_ckpt *c, const dqtg_config *cfg,
                           uint8_t *const *masks);
/* proxy_quality_delta(original, reconstructed) (search.cpp:30-61); per-layer-type
 * sums are reduced in a fixed parallel order (tolerance, not bit parity: §7 H9) */
dqtg_status dqtg_proxy_quality(dqtg_engine *e, const dqtg_layout *layout,
                               const float *const *orig_any, const float *const *recon_any,
                               double *quality);
/* releases the engine's scratch buffers, its pooled pinned decode staging and the
 * device's cached blocks (between workloads of very different sizes; no reference
 * counterpart) */
dqtg_status dqtg_engine_trim(dqtg_engine *e);
/* *equal = 1 when the two states have the same step, layout, codebooks, levels and
 * protected entries (compared on the device; round-trip checks of decode_delta_record,
 * codec.cpp:513-597, without a host copy of the levels) */
dqtg_status dqtg_qstate_equal(dqtg_engine *e, const dqtg_qstate *a, const dqtg_qstate *b,
                              int *equal);
/* per-tensor level histograms of a state, counts[i * stride + level] — the exact
 * integer input of estimate_compression (search.cpp:63-85) */
dqtg_status dqtg_level_counts(dqtg_engine *e, const dqtg_qstate *q, uint32_t stride,
                              uint64_t *counts);

/* ---- batched candidate evaluation: ProxyEvaluator::evaluate over m configs
 * (search.cpp:107-112) as EvalCache::prefetch batches them (search.cpp:174-204) */
dqtg_status dqtg_eval_batch(dqtg_engine *e, const dqtg_ckpt *c, const dqtg_config *cfgs,
                            const uint64_t *seeds, uint32_t m, double *quality_delta,
                            double *est_compression);

/* ---- clustering (quantize.cpp:94-325) ------------------------------------ */
dqtg_status dqtg_approx_kmeans(dqtg_engine *e, const float *values_any, uint64_t n, uint32_t k,
                               double sigma, double alpha, uint64_t seed, float *codebook,
                               uint32_t *len);
dqtg_status dqtg_kmeanspp_init(dqtg_engine *e, const double *points, const double *weights,
                               uint64_t n, uint32_t k, uint64_t seed, double *centers);
dqtg_status dqtg_lloyd(dqtg_engine *e, const double *points, const double *weights, uint64_t n,
                       double *centers, uint32_t k, double tol, uint32_t max_iter,
                       uint32_t *iterations);
dqtg_status dqtg_sq_loss(dqtg_engine *e, const double *points, const double *weights, uint64_t n,
                         const double *centers, uint32_t k, double *loss);

/* ---- codec primitives (codec.cpp:12-288) ---------------------------------- */
dqtg_status dqtg_delta_compute(dqtg_engine *e, const uint16_t *prev, const uint16_t *cur,
                               uint64_t n, uint32_t B, uint16_t *out);
dqtg_status dqtg_delta_apply(dqtg_engine *e, const uint16_t *prev, const uint16_t *deltas,
                             uint64_t n, uint32_t B, uint16_t *out);
dqtg_status dqtg_crc32(dqtg_engine *e, const uint8_t *data_any, uint64_t n, uint32_t *crc);

#ifdef __cplusplus
}
#endif
#endif /* DQTG_H */
