/* mfgpu.h — C-ABI of the B200 scoring engine (libmfgpu.so).
 *
 * Drop-in seam: this library replaces the reference's
 *   ScoringModel(container, compute_mode)        pkg/src/metricforge/encoder.py:94-118
 *   ScoringModel.score_records(encoded_records)  pkg/src/metricforge/encoder.py:214-226
 * i.e. everything from padded token ids to one float32 score per record
 * (forward, BOS pool, per-kind features, regression head). Its four-call
 * shape (create / score / last_error / destroy) mirrors the flat boundary the
 * reference exposes to other languages in pkg/frontend/src/boundary.ts:185-261
 * (create / evaluateBatch / lastError / destroy).
 *
 * Ownership: all host buffers are caller-owned and only read/written during
 * the call. The context owns device weights and workspaces. One caller thread
 * per context at a time (the Python wrapper serialises, like Evaluator's lock,
 * pkg/src/metricforge/evaluate.py:159,182).
 *
 * Return codes (mirroring the CLI's exit-code split, pkg/src/metricforge/cli.py:40-47):
 *   MFG_OK 0, MFG_ERR_RUNTIME 1 (CUDA / I/O), MFG_ERR_USAGE 2 (bad ids, lengths,
 *   arguments), MFG_ERR_CONTAINER 3 (format, missing or mis-shaped tensor).
 */
#ifndef MFGPU_H
#define MFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFG_OK 0
#define MFG_ERR_RUNTIME 1
#define MFG_ERR_USAGE 2
#define MFG_ERR_CONTAINER 3

/* Arithmetic of the encoder/head GEMMs. */
#define MFG_PREC_FP32 0   /* fp32-parity: fp16 hi/lo split operands, 3 tcgen05 MMAs per k-step
                             (~22 significant bits; |d| <= 1e-3 vs the fp32 reference) */
#define MFG_PREC_BF16 1   /* one bf16 MMA per k-step, fp32 accumulate (reported separately) */
#define MFG_PREC_BF16X3 2 /* bf16 hi/lo split, 3 MMAs: fp32 range, ~16 significant bits */
#define MFG_PREC_FP16 3   /* the reference's fp16 mode (`encoder.py:105, 120-130`): binary16
                             weights/activations, one fp16 MMA per k-step, fp32 accumulate,
                             binary16 rounding after every matmul, bias add, LN, GELU,
                             residual sum and head stage */

typedef struct mfg_ctx mfg_ctx;

typedef struct {
  const char* container_path; /* .mfrg file (pkg/src/metricforge/container.py layout) */
  int32_t device;             /* CUDA ordinal */
  int32_t precision;          /* MFG_PREC_* */
  int64_t max_tokens;         /* workspace capacity per device chunk (0 = default 262144) */
  int32_t max_records;        /* records per device chunk (0 = default 4096) */
  int32_t profile;            /* 1 = time every launch with CUDA events (see mfg_stats) */
} mfg_config;

/* Maps the container, checks the tensor-name/shape contract of
 * required_tensor_shapes (encoder.py:69-91), uploads and pre-splits weights. */
int mfg_create(const mfg_config* cfg, mfg_ctx** out);

/* Score n_records records of n_roles token sequences each.
 *   ids:        all sequences concatenated ROLE-MAJOR: role 0 of records 0..n-1,
 *               then role 1 of records 0..n-1, ...; values in [0, vocab_size)
 *   cu_seqlens: [n_roles * n_records + 1] offsets into ids (cu_seqlens[0] == 0)
 *   scores_out: [n_records] float32, same record order
 * Roles follow SEGMENT_ROLES (encoder.py:40-44): comet-qe (src, mt),
 * comet (src, mt, ref), bleurt (joint). */
int mfg_score_batch(mfg_ctx* ctx, int32_t n_records, int32_t n_roles, const int32_t* ids,
                    const int64_t* cu_seqlens, float* scores_out);

/* Same as mfg_score_batch with DEVICE-resident ids (role-major int32, on the
 * context's device) and a DEVICE scores_out buffer; cu_seqlens stays on the
 * host (chunk planning). Out-of-range ids are detected on the device. */
int mfg_score_device(mfg_ctx* ctx, int32_t n_records, int32_t n_roles, const int32_t* d_ids,
                     const int64_t* cu_seqlens, float* d_scores_out);

/* Launch every kernel / copy of this context on `stream` (a cudaStream_t of
 * the context's device; NULL restores the context's own stream). */
int mfg_set_stream(mfg_ctx* ctx, void* stream);

/* Error of the last failing call on ctx (ctx == NULL: last mfg_create / test
 * call on this thread). Copies a NUL-terminated message into buf. */
int mfg_last_error(const mfg_ctx* ctx, int32_t* code, char* buf, size_t cap);

void mfg_destroy(mfg_ctx* ctx);

/* Host-only check of a container (no device needed): mmap + header, tensor
 * index bounds (offsets / sizes inside the file, no overlaps, no duplicate
 * names), metric kind and the tensor-name/shape contract — what mfg_create
 * validates before touching the GPU (`container.py:293-322`,
 * `encoder.py:107-115`). The payload checksum is the Python
 * `open_container(validate=True)` step. Error text via mfg_last_error(NULL). */
int mfg_check_container(const char* path);

/* ---- introspection ------------------------------------------------------ */
typedef struct {
  int32_t kind; /* 0 comet-qe, 1 comet, 2 bleurt */
  int32_t vocab_size, d_model, n_heads, n_layers, d_ffn, max_position, pre_norm;
  int32_t n_roles, n_head_stages, precision, num_sms;
  int64_t device_bytes; /* weights + workspaces resident on the device */
  /* mfg_create phases (ms): CUDA context, container open (mmap, header, shape
   * contract), embeddings, layer weights (H2D + transpose/split), head, workspaces */
  double load_ms[6];
} mfg_model_info;
int mfg_get_model_info(const mfg_ctx* ctx, mfg_model_info* out);

#define MFG_NCLASS 8 /* qkv, o_proj, ffn1, ffn2, attention, layernorm, embed, head */
typedef struct {
  double device_ms;        /* sum over calls of first-H2D..last-D2H event time */
  int64_t calls, records, tokens, chunks;
  int64_t kernel_launches; /* kernels this library launched */
  /* per class (profile=1 only): event-timed ms, launches, algorithmic work */
  double class_ms[MFG_NCLASS];
  int64_t class_launches[MFG_NCLASS];
  double class_flops[MFG_NCLASS]; /* algorithmic FLOPs (real, unpadded dims) */
  double class_bytes[MFG_NCLASS]; /* algorithmic HBM bytes */
  /* fp32-parity path: chunks (and their records) re-scored with bf16 hi/lo pieces
   * because an activation left the fp16 range (|x| >= 65520) */
  int64_t fallback_chunks, fallback_records;
} mfg_stats;
int mfg_get_stats(const mfg_ctx* ctx, mfg_stats* out);
/* Switch per-launch CUDA-event timing (mfg_stats.class_ms) on or off between calls. */
int mfg_set_profile(mfg_ctx* ctx, int32_t enable);
int mfg_reset_stats(mfg_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MFGPU_H */
