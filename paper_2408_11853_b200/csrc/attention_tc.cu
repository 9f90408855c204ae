// tcgen05 attention for one (sequence, head) per CTA, sequences of <= 128
// tokens with d_head == 64 (XLM-R / InfoXLM / RemBERT shapes; the path of
// `pkg/src/metricforge/encoder.py:132-147` for every record of configs 2-4).
//
//   S = Q·Kᵀ      tcgen05.mma M=128 x N=round16(L) x K=64, fp32 in TMEM
//   P = exp(S·scale - rowmax)  (fp32, exact expf, keys >= L get exactly 0)
//   O = P·V       tcgen05.mma M=128 x N=64 x K=round16(L), V read MN-major
//   ctx = O / rowsum  -> 16-bit hi/lo pieces (the O-projection's A operand)
//
// Operands travel as 16-bit hi/lo pairs and each product is three MMAs
// (hi·hi + lo·hi + hi·lo), like the GEMMs, so S and O carry ~22 significant
// bits (fp16 pieces). Q, K, V tiles arrive by TMA (128B swizzle, 16-row boxes so
// only round16(L) rows are fetched) straight from
// the QKV GEMM output; P is written by the softmax threads into the (then dead)
// Q/K shared-memory region in the same swizzled K-major layout.
//
// 128 threads: thread r owns query row r (TMEM lane r). Thread 0 issues TMA and
// MMAs; warp 0 owns the TMEM allocation (256 columns: S 0..127, O 128..191).
// ~97 KB shared memory -> two CTAs per SM overlap softmax with MMA/TMA.
#include "kernels.h"
#include "ptx.cuh"

namespace mfg {

constexpr int ATC_THREADS = 128;
constexpr int ATC_TILE = 128 * 128;  // bytes of one 128-row x 64-col 16-bit tile
constexpr int ATC_SMEM = 1024 + 6 * ATC_TILE + 64;

__device__ __forceinline__ void tc_mma_f16kind(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t acc) {
  tc_mma_bf16(d, a, b, idesc, acc);
}

template <bool SPLIT>
__global__ void __launch_bounds__(ATC_THREADS, 2)
    attention_tc_kernel(const __grid_constant__ CUtensorMap mh,
                        const __grid_constant__ CUtensorMap ml, const int32_t* __restrict__ cu,
                        const int32_t* __restrict__ seqs, int d, float scale, int fmt,
                        uint16_t* __restrict__ ch, uint16_t* __restrict__ cl, int ldc, int* ovf) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  // tiles: 0 Qh, 1 Ql, 2 Kh, 3 Kl, 4 Vh, 5 Vl; after S: P_hi = tiles 0,1 (keys 0-63,
  // 64-127), P_lo = tiles 2,3.
  uint8_t* tile = sm;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 6 * ATC_TILE);  // load, s, o
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3);

  const int seq = seqs[blockIdx.x];
  const int h = blockIdx.y;
  const int start = cu[seq];
  const int L = cu[seq + 1] - start;
  const int n16 = (L + 15) & ~15;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tslot;

  if (tid == 0) {
    // 16-row boxes: fetch exactly round16(L) rows of Q, K and V (hi, lo)
    mbar_expect_tx(&bars[0], (uint32_t)n16 * 128 * (SPLIT ? 6 : 3));
    const int cq = h * 64, ck = d + h * 64, cv = 2 * d + h * 64;
    for (int r0 = 0; r0 < n16; r0 += 16) {
      const int so = r0 * 128;
      tma_load_2d(tile + 0 * ATC_TILE + so, &mh, &bars[0], cq, start + r0);
      tma_load_2d(tile + 2 * ATC_TILE + so, &mh, &bars[0], ck, start + r0);
      tma_load_2d(tile + 4 * ATC_TILE + so, &mh, &bars[0], cv, start + r0);
      if (SPLIT) {
        tma_load_2d(tile + 1 * ATC_TILE + so, &ml, &bars[0], cq, start + r0);
        tma_load_2d(tile + 3 * ATC_TILE + so, &ml, &bars[0], ck, start + r0);
        tma_load_2d(tile + 5 * ATC_TILE + so, &ml, &bars[0], cv, start + r0);
      }
    }
    mbar_wait(&bars[0], 0);
    tc_fence_after();
    // S[128 x n16] = Q Kᵀ
    const uint32_t idesc = idesc_f16kind(128, n16, fmt);
    const uint64_t qh = umma_desc_sw128(tile), kh = umma_desc_sw128(tile + 2 * ATC_TILE);
    const uint64_t ql = umma_desc_sw128(tile + ATC_TILE), kl = umma_desc_sw128(tile + 3 * ATC_TILE);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t adv = (uint64_t)(k * 32) >> 4;
      tc_mma_f16kind(tm, qh + adv, kh + adv, idesc, k != 0);
      if (SPLIT) {
        tc_mma_f16kind(tm, ql + adv, kh + adv, idesc, 1);
        tc_mma_f16kind(tm, qh + adv, kl + adv, idesc, 1);
      }
    }
    tc_commit(&bars[1]);
  }
  __syncwarp();

  // ---- softmax: thread tid owns query row tid
  mbar_wait(&bars[1], 0);
  tc_fence_after();
  const uint32_t trow = tm + ((uint32_t)(warp * 32) << 16);
  const int nchunk = (L + 31) >> 5;
  float mx = -INFINITY;
  for (int c = 0; c < nchunk; ++c) {
    float v[32];
    tmem_ld_32x32(trow + c * 32, v);
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (c * 32 + i < L) mx = fmaxf(mx, v[i] * scale);
  }
  float sum = 0.f;
  const int r = tid;
  for (int c = 0; c < nchunk; ++c) {
    float v[32];
    tmem_ld_32x32(trow + c * 32, v);
    uint32_t ph[16], pl[16];
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      float p0 = 0.f, p1 = 0.f;
      if (c * 32 + i < L) p0 = expf(v[i] * scale - mx);
      if (c * 32 + i + 1 < L) p1 = expf(v[i + 1] * scale - mx);
      sum += p0 + p1;
      uint16_t h0, l0, h1, l1;
      split16(p0, fmt, h0, l0);
      split16(p1, fmt, h1, l1);
      ph[i / 2] = h0 | ((uint32_t)h1 << 16);
      pl[i / 2] = l0 | ((uint32_t)l1 << 16);
    }
    // keys c*32..c*32+31 -> atom c/2, 16-byte units (c%2)*4 .. +3, swizzled by row
    uint8_t* hi_atom = tile + (c >> 1) * ATC_TILE;
    uint8_t* lo_atom = tile + (2 + (c >> 1)) * ATC_TILE;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int unit = (c & 1) * 4 + u;
      const uint32_t off = r * 128 + ((unit ^ (r & 7)) << 4);
      *reinterpret_cast<uint4*>(hi_atom + off) =
          make_uint4(ph[4 * u], ph[4 * u + 1], ph[4 * u + 2], ph[4 * u + 3]);
      if (SPLIT)
        *reinterpret_cast<uint4*>(lo_atom + off) =
            make_uint4(pl[4 * u], pl[4 * u + 1], pl[4 * u + 2], pl[4 * u + 3]);
    }
  }
  // P (generic-proxy smem writes) must be visible to the tensor core (async proxy)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (tid == 0) {
    // O[128 x 64] = P V, V is [keys][64] = MN-major B operand
    const uint32_t idesc = idesc_f16kind(128, 64, fmt) | (1u << 16);
    const uint32_t to = tm + 128;
    for (int k = 0; k < n16; k += 16) {
      const int atom = k >> 6;
      const uint64_t aoff = (uint64_t)((k & 63) * 2) >> 4;
      const uint64_t ph_ = umma_desc_sw128(tile + atom * ATC_TILE) + aoff;
      const uint64_t pl_ = umma_desc_sw128(tile + (2 + atom) * ATC_TILE) + aoff;
      const uint64_t vh = umma_desc_sw128(tile + 4 * ATC_TILE + k * 128);
      const uint64_t vl = umma_desc_sw128(tile + 5 * ATC_TILE + k * 128);
      tc_mma_f16kind(to, ph_, vh, idesc, k != 0);
      if (SPLIT) {
        tc_mma_f16kind(to, pl_, vh, idesc, 1);
        tc_mma_f16kind(to, ph_, vl, idesc, 1);
      }
    }
    tc_commit(&bars[2]);
  }
  __syncwarp();
  mbar_wait(&bars[2], 0);
  tc_fence_after();
  {
    // every lane runs the (warp-collective) TMEM loads; only rows < L store
    const float inv = 1.0f / sum;
    const size_t ob = (size_t)(start + r) * ldc + h * 64;
    bool ok = true;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v[32];
      tmem_ld_32x32(trow + 128 + c * 32, v);
      if (r < L) {
        uint32_t hh[16], ll[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          uint16_t h0, l0, h1, l1;
          ok &= split16(v[i] * inv, fmt, h0, l0);
          ok &= split16(v[i + 1] * inv, fmt, h1, l1);
          hh[i / 2] = h0 | ((uint32_t)h1 << 16);
          ll[i / 2] = l0 | ((uint32_t)l1 << 16);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          *reinterpret_cast<uint4*>(ch + ob + c * 32 + 8 * u) =
              make_uint4(hh[4 * u], hh[4 * u + 1], hh[4 * u + 2], hh[4 * u + 3]);
          if (SPLIT)
            *reinterpret_cast<uint4*>(cl + ob + c * 32 + 8 * u) =
                make_uint4(ll[4 * u], ll[4 * u + 1], ll[4 * u + 2], ll[4 * u + 3]);
        }
      }
    }
    if (!ok && ovf) atomicOr(ovf, 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tm);
  }
}

cudaError_t launch_attention_tc(const CUtensorMap* mh, const CUtensorMap* ml, bool split,
                                const int32_t* cu, const int32_t* seqs, int n_seqs, int heads,
                                int d, int fmt, uint16_t* ch, uint16_t* cl, int ldc, int* ovf,
                                cudaStream_t st) {
  if (n_seqs <= 0) return cudaSuccess;
  const float scale = 1.0f / sqrtf((float)d / (float)heads);
  dim3 grid(n_seqs, heads);
  if (split) {
    cudaFuncSetAttribute(attention_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         ATC_SMEM);
    attention_tc_kernel<true><<<grid, ATC_THREADS, ATC_SMEM, st>>>(*mh, *ml, cu, seqs, d, scale,
                                                                     fmt, ch, cl, ldc, ovf);
  } else {
    cudaFuncSetAttribute(attention_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         ATC_SMEM);
    attention_tc_kernel<false><<<grid, ATC_THREADS, ATC_SMEM, st>>>(*mh, *mh, cu, seqs, d, scale,
                                                                      fmt, ch, cl, ldc, ovf);
  }
  return cudaGetLastError();
}

}  // namespace mfg
