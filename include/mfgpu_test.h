/* mfgpu_test.h — kernel-level entry points of libmfgpu.so used by the parity
 * tests (tests/test_gpu_kernels.py). Each call allocates its own device
 * buffers on the current device, runs ONE production kernel and copies the
 * result back; split (hi/lo) outputs are returned recombined as hi + lo.
 * Not part of the scoring API. Return codes as in mfgpu.h. */
#ifndef MFGPU_TEST_H
#define MFGPU_TEST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* out[M][N] = epilogue(A[M][K] · W[K][N] + bias[N] (+ residual[M][N])) through the
 * tcgen05 GEMM. epi: 0 f32, 1 f32+residual, 2 gelu (split out), 3 tanh (split out). */
int mfgt_gemm(int32_t precision, int32_t epi, int32_t M, int32_t N, int32_t K, const float* A,
              const float* W, const float* bias, const float* residual, float* out);

/* ctx[T][d] = attention of packed qkv[T][3d] (q | k | v per row), sequences given by
 * cu[n_seq + 1], heads = n_heads, scale 1/sqrt(d/heads). use_tc = 1 routes sequences
 * of <= 128 tokens with d_head 64 to the tcgen05 kernel, 0 forces the SIMT kernel. */
int mfgt_attention(int32_t precision, int32_t n_seq, const int32_t* cu, int32_t d,
                   int32_t n_heads, const float* qkv, float* ctx_out, int32_t use_tc);

/* Host-only (no device needed): the attention work planner. Sequences of <= 128
 * tokens go into tiles of <= 4 whole sequences at 32-aligned rows (tiles_out: per
 * tile t0[4] then len[4]); longer ones into {seq, q0} items of 128 queries
 * (64 when tc_ok == 0: every sequence goes to the SIMT kernel). */
int mfgt_plan_tiles(const int32_t* cu, int32_t nseq, int32_t tc_ok, int32_t* tiles_out,
                    int32_t* n_tiles, int32_t* work_out, int32_t* n_work, int32_t cap);

/* Diagnostics: enable = 1 starts recording a clock64 trace of the tcgen05
 * attention kernel (first 4 CTAs x 64 items x 8 events); enable = 0 stops and
 * copies it to host_out[2048]. */
int mfgt_att_trace(int32_t enable, long long* host_out);

/* out[T][d] = LayerNorm(y) with gain g and bias b (eps 1e-5). */
int mfgt_layernorm(int32_t T, int32_t d, const float* y, const float* g, const float* b,
                   float* out);

#ifdef __cplusplus
}
#endif
#endif
