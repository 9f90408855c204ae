/* mfhost.h — host-side packing C-ABI (libmfhost.so): bit-exact tokenizer,
 * batch planner and role-major packer feeding mfg_score_batch.
 *
 * Replaces, bit for bit:
 *   Vocabulary.encode                 pkg/src/metricforge/vocab.py:54-79
 *   encode_fields / _single / _joint  pkg/src/metricforge/vocab.py:104-143
 *   plan_batches                      pkg/src/metricforge/batching.py:61-73
 * and adds the role-major varlen packing that replaces pad_batch
 * (batching.py:76-91) on the device path.
 */
#ifndef MFHOST_H
#define MFHOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mfh_vocab mfh_vocab;

/* Build the matcher from n_tokens UTF-8 tokens joined by '\n' (id = position).
 * Specials (ids 0..4) never match text (vocab.py:43-46). Returns 0, or 2 on
 * invalid input. Duplicate / empty / special-prefix checks are the caller's
 * (the Python wrapper raises VocabularyError with the reference messages). */
int mfh_vocab_create(const char* blob, int64_t nbytes, int32_t n_tokens, mfh_vocab** out);
void mfh_vocab_destroy(mfh_vocab* v);
int32_t mfh_vocab_size(const mfh_vocab* v);
int32_t mfh_vocab_max_piece(const mfh_vocab* v); /* in code points */

/* Greedy longest-match ids of one UTF-8 text (no specials). Returns the id
 * count, or -(needed) when cap is too small. */
int64_t mfh_encode(const mfh_vocab* v, const char* text, int64_t nbytes, int32_t* out, int64_t cap);

/* encode_fields for n records. kind: 0 comet-qe (S,T), 1 comet (S,T,R),
 * 2 bleurt (T,R -> one joint sequence). blob holds all field texts; field_off
 * [n*n_fields+1] are byte offsets, record-major. Writes record-major sequences
 * (n_seqs = 2, 3, 1 per record) to ids_out with offsets seq_off[n*n_seqs+1].
 * Returns 0; 2 if max_len cannot hold the specials; -(needed) if ids_cap is
 * too small. n_threads <= 0 picks the hardware concurrency. */
int64_t mfh_encode_records(const mfh_vocab* v, int32_t kind, int32_t n, const char* blob,
                           const int64_t* field_off, int32_t max_len, int32_t n_threads,
                           int32_t* ids_out, int64_t ids_cap, int64_t* seq_off);

/* Native TSV intake + encode_fields (replaces the per-record
 * Python loop `records_from_tsv_lines` -> `EvalRecord.field_values` ->
 * `encode_fields`, pkg/src/metricforge/evaluate.py:112-123, 179-196 and
 * vocab.py:104-143). blob holds n_lines lines back to back, line i =
 * blob[line_off[i] .. line_off[i+1]); each is rstrip("\n")-ed and split on
 * '\t'. Output as mfh_encode_records. Returns 0; 3 when a line has the wrong
 * column count (*bad_line = its index within this call, *bad_cols = its count;
 * checked for all lines before any max_len error); 2 on bad arguments or a
 * max_len too small for the specials; -(needed) if ids_cap is too small. */
int64_t mfh_encode_tsv(const mfh_vocab* v, int32_t kind, const char* blob,
                       const int64_t* line_off, int64_t n_lines, int32_t max_len,
                       int32_t n_threads, int32_t* ids_out, int64_t ids_cap, int64_t* seq_off,
                       int64_t* bad_line, int32_t* bad_cols);

/* order[pos] = original index; windows of mini_batch*factor, stable sort by
 * (-length, index) inside a window when sort != 0. */
int mfh_plan(const int64_t* lengths, int64_t n, int32_t mini_batch, int32_t factor, int32_t sort,
             int64_t* order);

/* Gather records order[0..m) of a record-major encoding (n_seqs per record)
 * into the role-major layout of mfg_score_batch: ids_out, cu_out[n_seqs*m+1]. */
int mfh_pack_roles(const int32_t* ids, const int64_t* seq_off, int32_t n_seqs, const int64_t* order,
                   int64_t m, int32_t* ids_out, int64_t* cu_out);

#ifdef __cplusplus
}
#endif
#endif
