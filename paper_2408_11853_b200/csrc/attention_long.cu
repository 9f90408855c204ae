// tcgen05 attention for sequences longer than one 128-row tile (129..512 tokens:
// config 5's long tail), d_head 64 or 80. Same numerics as the tile kernel
// (`pkg/src/metricforge/encoder.py:132-147`, masked_softmax 60-66): operand
// pieces and MMA splits per MODE (3 = hi/lo pairs, 2 = binary16 Q/K/V with P
// as hi/lo, 1 = single), fp32 softmax.
//
// One CTA per (sequence, 128-query block, head); keys in blocks of 128, two
// passes so no accumulator is ever rescaled:
//   pass 1  S_j = Q·K_jᵀ  -> running row max m and row sum l (online, fp32)
//   pass 2  S_j again      -> P_j = exp(S_j - m) (final m) into TMEM as 16-bit
//                             pieces -> O += P_j·V_j (A from TMEM)
//   ctx = O / l
// Blocks are aligned to the sequence start, so a sequence's scores never
// depend on what else is in the batch. The work is a small share of tokens,
// so the schedule is synchronous (one issuing thread, four softmax warps).
#include <vector>

#include "kernels.h"
#include "ptx.cuh"

namespace mfg {

namespace {

constexpr int AL_THREADS = 192;        // warp 0 issue, warp 1 TMEM alloc, warps 2-5 softmax
constexpr int AL_TILE = 128 * 128;     // 128 rows x 64 cols, 128B swizzle
constexpr int AL_TTILE = 128 * 32;     // 128 rows x 16 cols, 32B swizzle (d_head 80 tail)

template <int MODE, int DH>
struct AlCfg {
  static constexpr bool SPLIT = MODE == 3;
  static constexpr bool TAIL = DH == 80;
  static constexpr int NPL = SPLIT ? 2 : 1;
  static constexpr int OP = NPL * (AL_TILE + (TAIL ? AL_TTILE : 0));  // Q or K
  // V for DH 80: per plane two 64-column 128B-swizzled atoms (dims 0..63, 64..127)
  // so P·V is one N=80 MN-major product per operand pair
  static constexpr int VPL = TAIL ? 2 * AL_TILE : AL_TILE;
  static constexpr int VOP = NPL * VPL;
  static constexpr int Q_OFF = 0, K_OFF = OP, V_OFF = 2 * OP;
  static constexpr int BAR_OFF = 2 * OP + VOP;
  static constexpr int SMEM = 1024 + BAR_OFF + 128;  // 6 barriers + TMEM slot
};

__device__ __forceinline__ void al_tmem_st_8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void al_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 128 rows of V (column block `col`) starting at token `tok0`, DH 80 as two
// 64-column atoms per plane (the second past the tensor's last column is zero-filled).
template <bool SPLIT, bool TAIL>
__device__ __forceinline__ void al_load_v(uint8_t* dst, const CUtensorMap* mh, const CUtensorMap* ml,
                                          uint64_t* bar, int col, int tok0) {
  constexpr int VPL = TAIL ? 2 * AL_TILE : AL_TILE;
  for (int r0 = 0; r0 < 128; r0 += 32) {
    tma_load_2d(dst + r0 * 128, mh, bar, col, tok0 + r0);
    if (SPLIT) tma_load_2d(dst + VPL + r0 * 128, ml, bar, col, tok0 + r0);
    if (TAIL) {
      tma_load_2d(dst + AL_TILE + r0 * 128, mh, bar, col + 64, tok0 + r0);
      if (SPLIT) tma_load_2d(dst + VPL + AL_TILE + r0 * 128, ml, bar, col + 64, tok0 + r0);
    }
  }
}

// 128 rows of one operand (Q, K or V column block `col`) starting at token `tok0`:
// four 32-row boxes per plane (+ the 16-column tail boxes for d_head 80).
template <bool SPLIT, bool TAIL>
__device__ __forceinline__ void al_load(uint8_t* dst, const CUtensorMap* mh, const CUtensorMap* ml,
                                        const CUtensorMap* th, const CUtensorMap* tl,
                                        uint64_t* bar, int col, int tok0) {
  constexpr int NPL = SPLIT ? 2 : 1;
  for (int r0 = 0; r0 < 128; r0 += 32) {
    tma_load_2d(dst + r0 * 128, mh, bar, col, tok0 + r0);
    if (SPLIT) tma_load_2d(dst + AL_TILE + r0 * 128, ml, bar, col, tok0 + r0);
    if (TAIL) {
      uint8_t* tt = dst + NPL * AL_TILE;
      tma_load_2d(tt + r0 * 32, th, bar, col + 64, tok0 + r0);
      if (SPLIT) tma_load_2d(tt + AL_TTILE + r0 * 32, tl, bar, col + 64, tok0 + r0);
    }
  }
}

template <int MODE, int DH>
__global__ void __launch_bounds__(AL_THREADS, 1)
    attention_long_kernel(const __grid_constant__ CUtensorMap mh,
                          const __grid_constant__ CUtensorMap ml,
                          const __grid_constant__ CUtensorMap th,
                          const __grid_constant__ CUtensorMap tl,
                          const int2* __restrict__ work, const int32_t* __restrict__ cu, int heads,
                          int d, float scale, int fmt, uint16_t* __restrict__ ch,
                          uint16_t* __restrict__ cl, int ldc) {
  using C = AlCfg<MODE, DH>;
  constexpr bool SPLIT = C::SPLIT, TAIL = C::TAIL, PSPLIT = MODE >= 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* b_lk = bars;        // TMA bytes: Q (first phase) and K blocks
  uint64_t* b_s = bars + 1;     // S MMAs done
  uint64_t* b_sm = bars + 2;    // softmax warps done with S (stats or P written), 128 arrivals
  uint64_t* b_o = bars + 3;     // P·V MMAs of a block done
  uint64_t* b_fin = bars + 4;   // last P·V done
  uint64_t* b_lv = bars + 5;    // TMA bytes: V blocks
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 6);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int2 w = work[blockIdx.x / heads];
  const int h = blockIdx.x % heads;
  const int seq = w.x, q0 = w.y;
  const int start = cu[seq], L = cu[seq + 1] - start;
  const int nkb = (L + 127) >> 7;
  const int cq = h * DH, ck = d + h * DH, cv = 2 * d + h * DH;

  if (tid == 0) {
    mbar_init(b_lk, 1);
    mbar_init(b_s, 1);
    mbar_init(b_sm, 128);
    mbar_init(b_o, 1);
    mbar_init(b_fin, 1);
    mbar_init(b_lv, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tslot;  // S / P in columns [0,128), O in [128, 128 + DH)

  if (warp == 0) {
    if (lane == 0) {
      // Each K block is loaded as soon as the previous S has read the K buffer,
      // each V block as soon as the previous P·V has read the V buffer, so the
      // loads run under the softmax instead of in front of every block.
      uint32_t ph_k = 0, ph_v = 0, ph_s = 0, ph_sm = 0, ph_o = 0;
      const uint32_t op_bytes = 128 * (128 + (TAIL ? 32 : 0)) * C::NPL;
      auto load_k = [&](int kb) {
        mbar_expect_tx(b_lk, op_bytes);
        al_load<SPLIT, TAIL>(sm + C::K_OFF, &mh, &ml, &th, &tl, b_lk, ck, start + kb * 128);
      };
      auto load_v = [&](int kb) {
        mbar_expect_tx(b_lv, 128 * (TAIL ? 256 : 128) * C::NPL);
        al_load_v<SPLIT, TAIL>(sm + C::V_OFF, &mh, &ml, b_lv, cv, start + kb * 128);
      };
      // Q rides on K(0)'s phase (one arrive.expect_tx per phase: the barrier counts 1)
      mbar_expect_tx(b_lk, 2 * op_bytes);
      al_load<SPLIT, TAIL>(sm + C::Q_OFF, &mh, &ml, &th, &tl, b_lk, cq, start + q0);
      al_load<SPLIT, TAIL>(sm + C::K_OFF, &mh, &ml, &th, &tl, b_lk, ck, start);
      const uint8_t* qt = sm + C::Q_OFF;
      const uint8_t* kt = sm + C::K_OFF;
      const uint8_t* vt = sm + C::V_OFF;
      for (int pass = 0; pass < 2; ++pass) {
        for (int kb = 0; kb < nkb; ++kb) {
          const int nk = min(128, L - kb * 128), n16 = (nk + 15) & ~15;
          mbar_wait(b_lk, ph_k);  // K(kb) landed
          ph_k ^= 1;
          if (pass) {
            mbar_wait(b_lv, ph_v);  // V(kb) landed
            ph_v ^= 1;
          }
          tc_fence_after();
          // ---- S = Q·K_blockᵀ
          const uint32_t idesc = idesc_f16kind(128, n16, fmt);
          const uint64_t qh = umma_desc_sw128(qt), kh = umma_desc_sw128(kt);
          const uint64_t ql = umma_desc_sw128(qt + AL_TILE), kl = umma_desc_sw128(kt + AL_TILE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32) >> 4;
            tc_mma_bf16(tm, qh + adv, kh + adv, idesc, kk != 0);
            if (SPLIT) {
              tc_mma_bf16(tm, ql + adv, kh + adv, idesc, 1);
              tc_mma_bf16(tm, qh + adv, kl + adv, idesc, 1);
            }
          }
          if (TAIL) {
            const uint8_t* qtt = qt + C::NPL * AL_TILE;
            const uint8_t* ktt = kt + C::NPL * AL_TILE;
            const uint64_t qht = umma_desc_sw32(qtt), kht = umma_desc_sw32(ktt);
            tc_mma_bf16(tm, qht, kht, idesc, 1);
            if (SPLIT) {
              tc_mma_bf16(tm, umma_desc_sw32(qtt + AL_TTILE), kht, idesc, 1);
              tc_mma_bf16(tm, qht, umma_desc_sw32(ktt + AL_TTILE), idesc, 1);
            }
          }
          tc_commit(b_s);
          mbar_wait(b_s, ph_s);  // S done: the K buffer is free
          ph_s ^= 1;
          if (kb + 1 < nkb) load_k(kb + 1);
          else if (pass == 0) {
            load_k(0);  // pass 2 starts over; the V buffer has not been used yet
            load_v(0);
          }
          mbar_wait(b_sm, ph_sm);  // softmax read S (pass 1) / wrote P (pass 2)
          ph_sm ^= 1;
          tc_fence_after();
          if (pass) {
            // ---- O += P·V_block (A = P from TMEM, B = V MN-major)
            // DH 80: one N=80 product (B spans the plane's two atoms, LBO = atom
            // stride) writing O columns 128..207 (dims 0..79)
            const uint32_t idescv = idesc_f16kind(128, DH, fmt) | (1u << 16);
            for (int kk = 0; kk < n16; kk += 16) {
              const uint32_t pa = tm + 32 * (kk >> 5) + 8 * ((kk >> 4) & 1);
              const uint32_t acc0 = (kb | kk) != 0;
              const uint64_t vh = TAIL ? umma_desc_sw128_mn(vt + kk * 128, AL_TILE)
                                       : umma_desc_sw128(vt + kk * 128);
              al_mma_ts(tm + 128, pa, vh, idescv, acc0);
              if (PSPLIT) al_mma_ts(tm + 128, pa + 16, vh, idescv, 1);
              if (SPLIT)
                al_mma_ts(tm + 128, pa,
                          TAIL ? umma_desc_sw128_mn(vt + C::VPL + kk * 128, AL_TILE)
                               : umma_desc_sw128(vt + AL_TILE + kk * 128),
                          idescv, 1);
            }
            tc_commit(kb + 1 == nkb ? b_fin : b_o);
            if (kb + 1 < nkb) {  // P (S columns) and V are overwritten by the next block
              mbar_wait(b_o, ph_o);
              ph_o ^= 1;
              load_v(kb + 1);
            }
          }
        }
      }
    }
  } else if (warp >= 2) {
    // ------------------------------------------------------------ softmax (row r)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float c2 = scale * 1.4426950408889634f;
    float m = -INFINITY, l = 0.f;
    uint32_t ph_s = 0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int nk = min(128, L - kb * 128), n16 = (nk + 15) & ~15;
        const int c_end = (n16 + 31) >> 5;
        mbar_wait(b_s, ph_s);
        ph_s ^= 1;
        tc_fence_after();
        if (pass == 0) {
          float mb = -INFINITY;
          for (int c = 0; c < c_end; ++c) {
            float v[32];
            tmem_ld_32x32(tm + lane_off + c * 32, v);
            const int e = nk - c * 32;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < e) mb = fmaxf(mb, v[i]);
          }
          const float mn = fmaxf(m, mb);
          float sb = 0.f;
          for (int c = 0; c < c_end; ++c) {
            float v[32];
            tmem_ld_32x32(tm + lane_off + c * 32, v);
            const int e = nk - c * 32;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < e) sb += fast_exp2((v[i] - mn) * c2);
          }
          l = l * fast_exp2((m - mn) * c2) + sb;  // m = -inf on the first block: exp2(-inf) = 0
          m = mn;
        } else {
          const float mc = m * c2;
          for (int c = 0; c < c_end; ++c) {
            float v[32];
            tmem_ld_32x32(tm + lane_off + c * 32, v);
            const int e = nk - c * 32;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t hh[8], ll[8];
#pragma unroll
              for (int i = 0; i < 16; i += 2) {
                const int j = half * 16 + i;
                const float p0 = j < e ? fast_exp2(fmaf(v[j], c2, -mc)) : 0.f;
                const float p1 = j + 1 < e ? fast_exp2(fmaf(v[j + 1], c2, -mc)) : 0.f;
                split2(p0, p1, fmt, hh[i / 2], ll[i / 2]);
              }
              al_tmem_st_8(tm + lane_off + c * 32 + half * 8, hh);
              if (PSPLIT) al_tmem_st_8(tm + lane_off + c * 32 + 16 + half * 8, ll);
            }
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        mbar_arrive(b_sm);
      }
    }
    // ---- ctx = O / l for the rows of this query block inside the sequence
    mbar_wait(b_fin, 0);
    tc_fence_after();
    const float inv = 1.0f / l;
    const bool valid = q0 + r < L;
    const size_t ob = (size_t)(start + q0 + r) * ldc + h * DH;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v[32];
      tmem_ld_32x32(tm + lane_off + 128 + c * 32, v);
      if (valid) {
        uint32_t hh[16], ll[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) split2(v[i] * inv, v[i + 1] * inv, fmt, hh[i / 2], ll[i / 2]);
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
    if (TAIL) {
      float v[32];
      tmem_ld_32x32(tm + lane_off + 192, v);  // columns 192..207 hold dims 64..79
      if (valid) {
        uint32_t hh[8], ll[8];
#pragma unroll
        for (int i = 0; i < 16; i += 2) split2(v[i] * inv, v[i + 1] * inv, fmt, hh[i / 2], ll[i / 2]);
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          *reinterpret_cast<uint4*>(ch + ob + 64 + 8 * u) =
              make_uint4(hh[4 * u], hh[4 * u + 1], hh[4 * u + 2], hh[4 * u + 3]);
          if (SPLIT)
            *reinterpret_cast<uint4*>(cl + ob + 64 + 8 * u) =
                make_uint4(ll[4 * u], ll[4 * u + 1], ll[4 * u + 2], ll[4 * u + 3]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(tm);
  }
}

template <int MODE, int DH>
static void al_launch(const CUtensorMap* mh, const CUtensorMap* ml, const CUtensorMap* th,
                      const CUtensorMap* tl, const int2* work, int n_work, const int32_t* cu,
                      int heads, int d, float scale, int fmt, uint16_t* ch, uint16_t* cl, int ldc,
                      cudaStream_t st) {
  constexpr int SM = AlCfg<MODE, DH>::SMEM;
  auto kern = attention_long_kernel<MODE, DH>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
  kern<<<n_work * heads, AL_THREADS, SM, st>>>(*mh, *ml, *th, *tl, work, cu, heads, d, scale, fmt,
                                               ch, cl, ldc);
}

}  // namespace

cudaError_t launch_attention_long(const CUtensorMap* mh, const CUtensorMap* ml,
                                  const CUtensorMap* th, const CUtensorMap* tl, int mode,
                                  const int2* work, int n_work, const int32_t* cu, int heads, int d,
                                  int fmt, uint16_t* ch, uint16_t* cl, int ldc, cudaStream_t st) {
  if (n_work <= 0) return cudaSuccess;
  const int dh = d / heads;
  if (dh != 64 && dh != 80) return cudaErrorInvalidValue;
  const float scale = 1.0f / sqrtf((float)d / (float)heads);
  const CUtensorMap* mlo = mode == 3 ? ml : mh;
  const CUtensorMap* tlo = mode == 3 ? tl : th;
#define AL_GO(M, D) al_launch<M, D>(mh, mlo, th, tlo, work, n_work, cu, heads, d, scale, fmt, ch, cl, ldc, st)
  if (dh == 64) {
    if (mode == 3) AL_GO(3, 64); else if (mode == 2) AL_GO(2, 64); else AL_GO(1, 64);
  } else {
    if (mode == 3) AL_GO(3, 80); else if (mode == 2) AL_GO(2, 80); else AL_GO(1, 80);
  }
#undef AL_GO
  return cudaGetLastError();
}

}  // namespace mfg
