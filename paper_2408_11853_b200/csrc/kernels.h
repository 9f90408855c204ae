// Launch wrappers for the scoring-path kernels (see kernels.cu, gemm.cu).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <vector>

namespace mfg {

cudaError_t launch_embed(const int32_t* ids, const int32_t* cu, int nseq, int V, int d,
                         const float* tok, const float* pe, float* x32, int ld, uint16_t* xh,
                         uint16_t* xl, int fmt, int r16, int* flag, cudaStream_t st);
// y: fp32 rows, or binary16 rows when in16 (reference fp16 mode residual sums).
cudaError_t launch_layernorm(const void* y, int in16, int T, int d, int ld, const float* g,
                             const float* b, float* out32, uint16_t* oh, uint16_t* ol, int fmt,
                             int r16, int* ovf, cudaStream_t st);
// SIMT fp32 attention over (sequence, 64-query block) work items; Q|K|V read as
// hi(+lo) 16-bit pieces [T][ldq].
cudaError_t launch_attention(const uint16_t* qh, const uint16_t* ql, int ldq, int d, int heads,
                             const int32_t* cu,
                             const int2* work, int n_work, uint16_t* ch, uint16_t* cl,
                             int ldc, int fmt, int* ovf, cudaStream_t st);
// Persistent tcgen05 attention over (tile, head) items, d_head 64 or 80. A tile
// holds up to 4 whole sequences of <= 128 tokens at 32-aligned tile rows
// (att_plan_tiles). Maps: Q|K|V hi/lo [T][ldq] with box {64 cols, 32 rows}.
// mode: 3 = Q/K/V and P as hi/lo pairs (3 MMAs per product), 2 = single Q/K/V,
// P as hi/lo (reference fp16 mode), 1 = everything single (bf16 mode).
struct AttTile {
  int t0[4];   // first token of each sequence (packed stream index)
  int len[4];  // its length (0 = unused slot)
};
// th/tl: the same Q|K|V planes with box {16 cols, 32 rows}, 32B swizzle (head
// dims 64..79 of d_head 80; unused for d_head 64).
cudaError_t launch_attention_tc(const CUtensorMap* mh, const CUtensorMap* ml,
                                const CUtensorMap* th, const CUtensorMap* tl, int mode,
                                const AttTile* tiles, int n_tiles, int heads, int d, int fmt,
                                uint16_t* ch, uint16_t* cl, int ldc, int* ovf, int num_sms,
                                cudaStream_t st);
// tcgen05 attention for sequences of 129..512 tokens: one CTA per (work item,
// head), two passes over 128-key blocks (row stats, then P·V). Same maps/modes.
cudaError_t launch_attention_long(const CUtensorMap* mh, const CUtensorMap* ml,
                                  const CUtensorMap* th, const CUtensorMap* tl, int mode,
                                  const int2* work, int n_work, const int32_t* cu, int heads, int d,
                                  int fmt, uint16_t* ch, uint16_t* cl, int ldc, cudaStream_t st);
cudaError_t att_set_trace(long long* dev_buf);  // diagnostics: [4][64][8] clock64 or null
// Host: sequences of <= 128 tokens (when tc_ok) -> tiles; longer ones -> work
// items {seq, q0} for launch_attention_long (128-query blocks); without tc_ok
// every sequence -> SIMT work items (64-query blocks).
void att_plan_tiles(const int32_t* cu, int nseq, bool tc_ok, std::vector<AttTile>& tiles,
                    std::vector<int2>& work);
// Attention for the BOS query of every sequence only (last layer): q compact
// [nseq][ldqb], K|V from the packed Q|K|V rows [T][ldkv]; ctx -> compact [nseq][ldc].
// Sequences of <= 512 tokens, d_head <= 128.
cudaError_t launch_bos_attention(const uint16_t* qbh, const uint16_t* qbl, int ldqb,
                                 const uint16_t* kvh, const uint16_t* kvl, int ldkv, int d,
                                 int heads, const int32_t* cu, int nseq, uint16_t* ch, uint16_t* cl,
                                 int ldc, int fmt, cudaStream_t st);
cudaError_t launch_features(const float* x, int ld, int d, int kind, const int32_t* cu, int n,
                            uint16_t* fh, uint16_t* fl, int ldf, int fmt, int* ovf,
                            cudaStream_t st);
// Wᵀ rows row0.. = columns of w [K][N], split into 16-bit hi/lo pieces; with
// `alpha` (non-null) column n is multiplied by 1 / alpha[n] first (exact: powers of two).
cudaError_t launch_transpose_split(const float* w, int K, int N, uint16_t* hi, uint16_t* lo,
                                   int ldk, int row0, int fmt, int* ovf, cudaStream_t st,
                                   const float* alpha = nullptr);
// Per-column power-of-two prescale of w [K][N] for the fp16 hi/lo split:
// alpha[n] = 2^(e_n - 14) where 2^e_n <= max_k |w[k][n]| < 2^(e_n + 1), so the
// scaled column's largest element lies in [2^14, 2^15) (no fp16 overflow, the lo
// piece stays normal down to 2^-29 of the column max). Zero / non-finite columns
// get alpha = 1 (non-finite ones then flag the fp16 overflow as before).
cudaError_t launch_weight_scales(const float* w, int K, int N, float* alpha, cudaStream_t st);
// Copy the BOS row (cu[s]) of each sequence to compact row s (16-bit planes and/or fp32).
cudaError_t launch_gather_bos(const int32_t* cu, int nseq, int d, const uint16_t* sh,
                              const uint16_t* sl, int lds, const float* s32, int ld32, uint16_t* dh,
                              uint16_t* dl, int ldd, float* d32, int ldd32, cudaStream_t st);
cudaError_t launch_gather_col0(const float* out, int ld, int n, float* scores, cudaStream_t st);

// ---- tcgen05 GEMM (gemm.cu)
struct GemmArgs;
// Encode a 2-D 16-bit K-major tensor map (128B swizzle, box = 64 x box_rows).
bool make_tmap_u16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint64_t ld_elems, uint32_t box_rows, char* err, size_t errcap);
// General box: box_cols x box_rows, swizzle 128 / 64 / 32 bytes.
bool make_tmap_u16_box(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                       uint64_t ld_elems, uint32_t box_cols, uint32_t box_rows, int swizzle,
                       char* err, size_t errcap);
// Largest supported N tile dividing n_pad (n_pad % 64 == 0).
int gemm_pick_bn(int n_pad);
// Whether N tile `bn` runs on the CTA-pair kernel, and the weight tensor-map box
// rows that kernel expects (each CTA of a pair loads half of the N tile).
bool gemm_uses_pair(int bn);
int gemm_b_box_rows(int bn);
int gemm_kchunk_blocks(int K, bool fine = false);  // GemmArgs::kchunk for a GEMM of depth K
size_t gemm_partial_floats(int num_sms);  // GemmArgs::partial workspace size
// nsplit: 1 = one MMA per k-step (hi only), 2 = hi/lo pieces, 3 MMAs per k-step.
cudaError_t launch_gemm(const CUtensorMap* ah, const CUtensorMap* al, const CUtensorMap* bh,
                        const CUtensorMap* bl, int bn, int nsplit, int epi, const GemmArgs& a,
                        int num_sms, cudaStream_t st);

}  // namespace mfg
