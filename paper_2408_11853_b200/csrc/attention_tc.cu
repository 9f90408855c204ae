// Persistent tcgen05 attention for sequences of <= 128 tokens with d_head 64
// (XLM-R / InfoXLM / RemBERT shapes: every record of configs 2-4). Replaces the
// per-head loop of `pkg/src/metricforge/encoder.py:132-147` (+ masked_softmax 60-66).
//
// Work item = (sequence, head). Per item:
//   S = Q·Kᵀ      tcgen05.mma M=128 x N=round16(L) x K=64 -> fp32 in TMEM
//   P = exp(S·scale - rowmax) = exp2f((S - rowmax)·scale·log2e) in fp32, keys >= L
//       get exactly 0
//   O = P·V       tcgen05.mma M=128 x N=64 x K=round16(L), V is an MN-major B
//   ctx = O / rowsum -> 16-bit hi/lo pieces (the O-projection's A operand)
// Operands are 16-bit hi/lo pairs and each product is three MMAs
// (hi·hi + lo·hi + hi·lo), like the GEMMs (~22 significant bits with fp16).
//
// One CTA per SM walks items round-robin. Items alternate between two lanes
// b = k & 1, each with its own smem buffer, TMEM region (S, then O in the same
// columns once S is dead) and softmax warp group, so one group's softmax runs
// while the other waits for its P·V MMAs and the TMA/MMA of later items:
//   warp 0 lane 0  TMA producer  (Q, K, V tiles, 16-row boxes, 128B swizzle)
//   warp 1 lane 0  MMA issuer    (event loop: S(k) when its tiles land, O(k) when
//                                 P(k) lands; neither queue blocks the other)
//   warps 2-5 / 6-9  softmax (row = TMEM lane, two TMEM passes: max, exp) and
//                  epilogue for the items of lane 0 / lane 1
// P is written, swizzled K-major, into the item's (dead) Q/K smem tiles.
#include "kernels.h"
#include "ptx.cuh"

namespace mfg {

constexpr int ATP_THREADS = 320;
constexpr int ATP_TILE = 128 * 128;            // one 128-row x 64-col 16-bit tile
constexpr int ATP_BUF = 6 * ATP_TILE;          // Qh Ql Kh Kl Vh Vl
constexpr int ATP_SMEM = 1024 + 2 * ATP_BUF + 256;

struct AttItem {
  int start, L, h;
};

__device__ __forceinline__ AttItem att_item(int it, const int32_t* cu, const int32_t* seqs,
                                            int heads) {
  const int s = seqs[it / heads];
  AttItem a;
  a.start = cu[s];
  a.L = cu[s + 1] - a.start;
  a.h = it % heads;
  return a;
}

template <bool SPLIT>
__global__ void __launch_bounds__(ATP_THREADS, 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap mh,
                        const __grid_constant__ CUtensorMap ml, const int32_t* __restrict__ cu,
                        const int32_t* __restrict__ seqs, int n_items, int heads, int d,
                        float scale, int fmt, uint16_t* __restrict__ ch,
                        uint16_t* __restrict__ cl, int ldc, int* ovf) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 2 * ATP_BUF);
  uint64_t* load_full = bars;       // [2]
  uint64_t* s_full = bars + 2;      // [2]
  uint64_t* p_full = bars + 4;      // [2]
  uint64_t* o_full = bars + 6;      // [2]  also: smem buffer free again
  uint64_t* t_empty = bars + 8;     // [2]  TMEM (S, O) buffer free again
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 10);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&load_full[b], 1);
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 4);
      mbar_init(&o_full[b], 1);
      mbar_init(&t_empty[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tslot;
  auto buf = [&](int b) { return sm + b * ATP_BUF; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int k = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++k) {
        const int b = k & 1;
        const uint32_t ph = (k >> 1) & 1;
        const AttItem a = att_item(it, cu, seqs, heads);
        const int n16 = (a.L + 15) & ~15;
        mbar_wait(&o_full[b], ph ^ 1);  // item k-2 finished reading this buffer
        mbar_expect_tx(&load_full[b], (uint32_t)n16 * 128 * (SPLIT ? 6 : 3));
        const int cq = a.h * 64, ck = d + a.h * 64, cv = 2 * d + a.h * 64;
        uint8_t* t = buf(b);
        for (int r0 = 0; r0 < n16; r0 += 16) {
          const int so = r0 * 128;
          tma_load_2d(t + 0 * ATP_TILE + so, &mh, &load_full[b], cq, a.start + r0);
          tma_load_2d(t + 2 * ATP_TILE + so, &mh, &load_full[b], ck, a.start + r0);
          tma_load_2d(t + 4 * ATP_TILE + so, &mh, &load_full[b], cv, a.start + r0);
          if (SPLIT) {
            tma_load_2d(t + 1 * ATP_TILE + so, &ml, &load_full[b], cq, a.start + r0);
            tma_load_2d(t + 3 * ATP_TILE + so, &ml, &load_full[b], ck, a.start + r0);
            tma_load_2d(t + 5 * ATP_TILE + so, &ml, &load_full[b], cv, a.start + r0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Event loop over two queues so neither blocks the other: S(ks) as soon as
    // its tiles landed and its TMEM region is free, O(ko) as soon as P(ko) landed.
    if (lane == 0) {
      const int mine = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
      int ks = 0, ko = 0;
      uint32_t idle = 0;
      while (ko < mine) {
        bool progress = false;
        if (ks < mine && ks < ko + 2) {
          const int b = ks & 1;
          const uint32_t ph = (ks >> 1) & 1;
          if (mbar_test(&t_empty[b], ph ^ 1) && mbar_test(&load_full[b], ph)) {
            tc_fence_after();
            const AttItem a = att_item(blockIdx.x + ks * gridDim.x, cu, seqs, heads);
            const int n16 = (a.L + 15) & ~15;
            const uint32_t idesc = idesc_f16kind(128, n16, fmt);
            uint8_t* t = buf(b);
            const uint64_t qh = umma_desc_sw128(t), kh = umma_desc_sw128(t + 2 * ATP_TILE);
            const uint64_t ql = umma_desc_sw128(t + ATP_TILE),
                           kl = umma_desc_sw128(t + 3 * ATP_TILE);
            const uint32_t ts = tm + b * 128;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t adv = (uint64_t)(kk * 32) >> 4;
              tc_mma_bf16(ts, qh + adv, kh + adv, idesc, kk != 0);
              if (SPLIT) {
                tc_mma_bf16(ts, ql + adv, kh + adv, idesc, 1);
                tc_mma_bf16(ts, qh + adv, kl + adv, idesc, 1);
              }
            }
            tc_commit(&s_full[b]);
            ++ks;
            progress = true;
          }
        }
        if (ko < ks) {
          const int b = ko & 1;
          const uint32_t ph = (ko >> 1) & 1;
          if (mbar_test(&p_full[b], ph)) {
            tc_fence_after();
            const AttItem a = att_item(blockIdx.x + ko * gridDim.x, cu, seqs, heads);
            const int n16 = (a.L + 15) & ~15;
            const uint32_t idesc = idesc_f16kind(128, 64, fmt) | (1u << 16);  // B MN-major
            uint8_t* t = buf(b);
            const uint32_t to = tm + b * 128;  // S is dead once P(ko) landed
            for (int kk = 0; kk < n16; kk += 16) {
              const int atom = kk >> 6;
              const uint64_t aoff = (uint64_t)((kk & 63) * 2) >> 4;
              const uint64_t ph_ = umma_desc_sw128(t + atom * ATP_TILE) + aoff;
              const uint64_t pl_ = umma_desc_sw128(t + (2 + atom) * ATP_TILE) + aoff;
              const uint64_t vh = umma_desc_sw128(t + 4 * ATP_TILE + kk * 128);
              const uint64_t vl = umma_desc_sw128(t + 5 * ATP_TILE + kk * 128);
              tc_mma_bf16(to, ph_, vh, idesc, kk != 0);
              if (SPLIT) {
                tc_mma_bf16(to, pl_, vh, idesc, 1);
                tc_mma_bf16(to, ph_, vl, idesc, 1);
              }
            }
            tc_commit(&o_full[b]);
            ++ko;
            progress = true;
          }
        }
        if (progress) {
          idle = 0;
        } else if (++idle > (1u << 27)) {
          __trap();  // protocol bug: never hang the GPU
        }
      }
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    const int g = (warp - 2) >> 2;   // lane (buffer) this group serves: items k = g, g+2, ...
    const int q = warp & 3;          // TMEM lane quarter
    const int r = q * 32 + lane;     // query row owned by this thread
    const float c2 = scale * 1.4426950408889634f;  // exp(x*scale) = 2^(x*c2)
    int j = 0;
    for (int it = blockIdx.x + g * gridDim.x; it < n_items; it += 2 * gridDim.x, ++j) {
      const int b = g;
      const uint32_t ph = j & 1;
      const AttItem a = att_item(it, cu, seqs, heads);
      const bool active = q * 32 < a.L;  // warp-uniform: warp owns >= 1 real row
      const uint32_t trow = tm + b * 128 + ((uint32_t)(q * 32) << 16);
      // ---- softmax: S row -> registers (single TMEM pass) -> P pieces in smem
      mbar_wait(&s_full[b], ph);
      tc_fence_after();
      float sum = 1.f;
      if (active) {
        // two TMEM passes (max, then exp) keep the row out of registers
        const int nchunk = (a.L + 31) >> 5;
        float mx = -INFINITY;
        for (int c = 0; c < nchunk; ++c) {
          float v[32];
          tmem_ld_32x32(trow + c * 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i < a.L) mx = fmaxf(mx, v[i]);
        }
        sum = 0.f;
        uint8_t* t = buf(b);
        for (int c = 0; c < nchunk; ++c) {
          float v[32];
          tmem_ld_32x32(trow + c * 32, v);
          uint32_t hh[16], ll[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float p0 = 0.f, p1 = 0.f;
            if (c * 32 + i < a.L) p0 = exp2f((v[i] - mx) * c2);
            if (c * 32 + i + 1 < a.L) p1 = exp2f((v[i + 1] - mx) * c2);
            sum += p0 + p1;
            uint16_t h0, l0, h1, l1;
            split16(p0, fmt, h0, l0);
            split16(p1, fmt, h1, l1);
            hh[i / 2] = h0 | ((uint32_t)h1 << 16);
            ll[i / 2] = l0 | ((uint32_t)l1 << 16);
          }
          uint8_t* hi_atom = t + (c >> 1) * ATP_TILE;
          uint8_t* lo_atom = t + (2 + (c >> 1)) * ATP_TILE;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int unit = (c & 1) * 4 + u;
            const uint32_t off = r * 128 + ((unit ^ (r & 7)) << 4);
            *reinterpret_cast<uint4*>(hi_atom + off) =
                make_uint4(hh[4 * u], hh[4 * u + 1], hh[4 * u + 2], hh[4 * u + 3]);
            if (SPLIT)
              *reinterpret_cast<uint4*>(lo_atom + off) =
                  make_uint4(ll[4 * u], ll[4 * u + 1], ll[4 * u + 2], ll[4 * u + 3]);
          }
        }
        // generic-proxy smem writes of P -> visible to the tensor core
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
      // ---- epilogue: O row / rowsum -> ctx pieces
      mbar_wait(&o_full[b], ph);
      tc_fence_after();
      if (active) {
        const float inv = 1.0f / sum;
        const size_t ob = (size_t)(a.start + r) * ldc + a.h * 64;
        bool ok = true;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          float v[32];
          tmem_ld_32x32(trow + c * 32, v);
          if (r < a.L) {
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&t_empty[b]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tm);
  }
}

cudaError_t launch_attention_tc(const CUtensorMap* mh, const CUtensorMap* ml, bool split,
                                const int32_t* cu, const int32_t* seqs, int n_seqs, int heads,
                                int d, int fmt, uint16_t* ch, uint16_t* cl, int ldc, int* ovf,
                                int num_sms, cudaStream_t st) {
  if (n_seqs <= 0) return cudaSuccess;
  const float scale = 1.0f / sqrtf((float)d / (float)heads);
  const int n_items = n_seqs * heads;
  const int grid = n_items < num_sms ? n_items : num_sms;
  if (split) {
    cudaFuncSetAttribute(attention_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         ATP_SMEM);
    attention_tc_kernel<true><<<grid, ATP_THREADS, ATP_SMEM, st>>>(
        *mh, *ml, cu, seqs, n_items, heads, d, scale, fmt, ch, cl, ldc, ovf);
  } else {
    cudaFuncSetAttribute(attention_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         ATP_SMEM);
    attention_tc_kernel<false><<<grid, ATP_THREADS, ATP_SMEM, st>>>(
        *mh, *mh, cu, seqs, n_items, heads, d, scale, fmt, ch, cl, ldc, ovf);
  }
  return cudaGetLastError();
}

}  // namespace mfg
