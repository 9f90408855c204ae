// Persistent tcgen05 attention over packed 128-token tiles, d_head 64
// (XLM-R / InfoXLM / RemBERT shapes: every sequence of configs 2-4). Replaces the
// per-head loop of `pkg/src/metricforge/encoder.py:132-147` (+ masked_softmax 60-66).
//
// Tiles. The host packs whole sequences (each <= 128 tokens) greedily into tiles
// of 128 rows (`att_plan_tiles`, at most 4 sequences): sequence s of a tile sits
// at tile row o_s, a multiple of 32, loaded by TMA in 32-row boxes. A work item
// is (tile, head); its S = Q·Kᵀ is block-diagonal: a row attends only to the
// keys of its own sequence, every other key gets exactly 0 weight — which is the
// reference's per-sequence masked softmax, so sequences never mix. Because every
// sequence starts on a 32-row boundary, its keys fall into the same 16-key MMA
// k-steps and the same 32-key softmax chunks wherever it sits, and the other
// sequences only add exact zeros: scores are bitwise independent of which
// sequences share a tile (batch composition, chunking, GPU count).
//
// Per item:
//   S = Q·Kᵀ      tcgen05.mma M=128 x N=round16(n) x K=64, Q/K from smem (TMA)
//   P = exp(S·scale - rowmax) over the row's own keys, 0 elsewhere, fp32 math,
//       written back into S's TMEM columns as 16-bit pieces (P never touches smem)
//   O = P·V       tcgen05.mma M=128 x N=64 x K=round16(n), A = P from TMEM,
//                 B = V (MN-major) from smem
//   ctx = O / rowsum -> 16-bit hi/lo pieces (the O-projection's A operand)
// MODE 3 (fp32 parity): every product is three MMAs (hi·hi + lo·hi + hi·lo) of
// fp16 (or bf16) pieces, like the GEMMs (~22 significant bits with fp16).
// MODE 2 (reference fp16 mode): Q, K, V are the binary16 values the reference
// stores; S is one MMA (exact fp16 products, fp32 sums) and P = Ph + Pl keeps
// the fp32 softmax weights: O = Ph·V + Pl·V. MODE 1 (bf16): one MMA each.
//
// Roles (576 threads, one CTA per SM, items round-robin):
//   warp 0       TMA producer: Q|K ring (QK_ST stages) and V ring (V_ST stages)
//   warp 1       S issuer:     S(k) once its Q/K tiles landed and TMEM region k%2 is free
//   warp 18      O issuer:     P·V(k) once P(k) and V(k) are ready
//   (two issuer threads with blocking, hardware-suspended waits: neither queue
//   ever waits behind the other)
//   warps 2-9    group 0 (items k even, TMEM region 0): softmax, then epilogue
//   warps 10-17  group 1 (items k odd,  TMEM region 1)
// Inside a group two warps share each TMEM lane quarter (= 32 tile rows): warp
// hr takes rows 16hr..16hr+15 of it through the 16x32bx2 TMEM shape (lanes 0-15
// even key chunks / O columns 0..31, lanes 16-31 odd chunks / columns 32..63), so
// row max and row sum combine with one warp shuffle.
// TMEM columns: S/P of region b at 128b..128b+127; O of region b at 256+128b
// (MODE 3: Ph·Vh + Pl·Vh in the first 64 columns, Ph·Vl in the next 64).
// Measured (tools/mma_probe.cu): a 128xNx16 MMA costs >= ~72 cycles (SS) /
// ~107 cycles (A from TMEM) for N <= 128, so per item the tensor pipe needs
// ~1.1k cycles for S and ~2.5k for O.
// P layout in TMEM (A operand, K-major, two 16-bit values per 32-bit column):
// keys 32c..32c+31 -> hi pieces in columns 32c..32c+15, lo pieces in 32c+16..+31,
// i.e. exactly the columns of S chunk c that the same thread just consumed.
#include <vector>

#include "kernels.h"
#include "ptx.cuh"

namespace mfg {

constexpr int ATQ_THREADS = 608;
constexpr int ATQ_TILE = 128 * 128;  // 128 rows x 64 cols of 16-bit values (128B swizzle)

constexpr int ATQ_TTILE = 128 * 32;  // 128 rows x 16 cols (32B swizzle): head-dim tail 64..79

// DH = head dim, 64 or 80 (XLM-R XL). DH 80 keeps the first 64 columns of every
// Q/K/V tile in the 128B-swizzled layout and the last 16 in a 32B-swizzled
// "tail" tile: S = QKᵀ gets a 5th k-step from the tail tiles and P·V a second
// N=16 product.
template <int MODE, int DH>
struct AtqCfg {
  static constexpr bool SPLIT = MODE == 3;
  static constexpr bool TAIL = DH == 80;
  static constexpr int NPL_QK = SPLIT ? 4 : 2;  // Qh Kh (Ql Kl)
  static constexpr int NPL_V = SPLIT ? 2 : 1;   // Vh (Vl)
  static constexpr int QK_BYTES = NPL_QK * (ATQ_TILE + (TAIL ? ATQ_TTILE : 0));
  // V for DH 80: per plane two 128B-swizzled 64-column atoms (dims 0..63 and
  // 64..127 of the head's column block; only 64..79 are used), so P·V is ONE
  // N=80 MN-major product per plane instead of an N=64 + an N=16 one
  static constexpr int V_BYTES = NPL_V * (TAIL ? 2 * ATQ_TILE : ATQ_TILE);
  static constexpr int QK_ST = SPLIT ? 2 : 3;
  static constexpr int V_ST = SPLIT ? (TAIL ? 1 : 3) : (TAIL ? 3 : 5);
  static constexpr int BAR_OFF = QK_ST * QK_BYTES + V_ST * V_BYTES;
  static constexpr int SMEM = 1024 + BAR_OFF + 256;
  static_assert(SMEM <= 232448, "attention smem");
};

__device__ __forceinline__ void tmem_st_8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void st_global_256(void* p, const uint32_t (&r)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld_32x8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// 16 consecutive fp32 columns of this warp's lanes, without waiting (tc_wait_ld)
__device__ __forceinline__ void tmem_ld_raw16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 16x32bx2 shape: lanes 0-15 of the warp access TMEM lanes base+0..15 at columns
// [c, c+N), lanes 16-31 the same TMEM lanes at columns [c+N, c+2N) (split offset N).
__device__ __forceinline__ void tmem_ld_16x32bx2(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 32;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_16x32bx2_8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], 8;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// 8 columns per lane at c (lanes 0-15) and c+32 (lanes 16-31)
__device__ __forceinline__ void tmem_st_16x32bx2_8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x8.b32 [%0], 32, {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tmem_st_1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ float tmem_ld_1(uint32_t taddr) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return __uint_as_float(v);
}
__device__ __forceinline__ void tc_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// D[tmem] (+)= A[tmem] * B[smem], kind::f16.
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Optional per-item clock64 trace of the first 4 CTAs (diagnostics only,
// tools/att_trace.py): [cta][item][event], events S-issued, O-issued,
// S-seen, P-done, O-seen (epilogue), item-done (epilogue).
__device__ long long* g_att_trace = nullptr;
#define ATT_TRACE(k, ev)                                              \
  do {                                                                \
    if (g_att_trace && blockIdx.x < 4 && (k) < 64)                    \
      g_att_trace[(blockIdx.x * 64 + (k)) * 8 + (ev)] = clock64();    \
  } while (0)

// rows of a tile used by its sequences (last one unpadded)
__device__ __forceinline__ int att_tile_rows(const AttTile& t) {
  int o = 0, n = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (t.len[j] > 0) n = o + t.len[j];
    o += (t.len[j] + 31) & ~31;
  }
  return n;
}

template <int MODE, int DH>
__global__ void __launch_bounds__(ATQ_THREADS, 1)
    attention_tc_kernel(const __grid_constant__ CUtensorMap mh,
                        const __grid_constant__ CUtensorMap ml,
                        const __grid_constant__ CUtensorMap th,
                        const __grid_constant__ CUtensorMap tl_,
                        const AttTile* __restrict__ tiles, int n_items, int heads, int d,
                        float scale, int fmt, uint16_t* __restrict__ ch,
                        uint16_t* __restrict__ cl, int ldc) {
  using C = AtqCfg<MODE, DH>;
  constexpr bool TAIL = C::TAIL;
  constexpr bool SPLIT = MODE == 3;     // Q, K, V as hi/lo pairs
  constexpr bool PSPLIT = MODE >= 2;    // P as hi/lo pair
  constexpr bool DEFER = !SPLIT && DH == 64;  // deferred epilogue (4 O slots of 64 columns)
  auto oslot = [](int k) { return DEFER ? (k & 3) : (k & 1); };
  auto opar = [](int k) { return (uint32_t)((DEFER ? (k >> 2) : (k >> 1)) & 1); };
  auto ocol = [](int k) { return (uint32_t)(DEFER ? 256 + 64 * (k & 3) : 256 + 128 * (k & 1)); };
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::BAR_OFF);
  uint64_t* qk_full = bars;                 // [QK_ST]
  uint64_t* qk_empty = qk_full + C::QK_ST;  // [QK_ST]
  uint64_t* v_full = qk_empty + C::QK_ST;   // [V_ST]
  uint64_t* v_empty = v_full + C::V_ST;     // [V_ST]
  uint64_t* s_full = v_empty + C::V_ST;     // [2]  S(k) in region k&1
  uint64_t* p_full = s_full + 2;            // [2]  P(k) written (256 group threads)
  // O accumulators: MODE 3 / DH 80 one per region (128 columns, slot k & 1); the
  // single-plane DH 64 modes (DEFER) have four 64-column slots (k & 3), so a
  // group runs item k's epilogue after item k+2's softmax, off the S -> P·V chain.
  uint64_t* o_full = p_full + 2;            // [4]  O(k) done (also: P region free)
  uint64_t* o_empty = o_full + 4;           // [4]  DEFER: O slot read (256 group threads)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(o_empty + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < C::QK_ST; ++s) {
      mbar_init(&qk_full[s], 1);
      mbar_init(&qk_empty[s], 1);
    }
    for (int s = 0; s < C::V_ST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 256);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 256);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tslot;
  const int mine = blockIdx.x < n_items ? (n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto item_of = [&](int k) { return blockIdx.x + k * gridDim.x; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch(&mh);
      if (SPLIT) tma_prefetch(&ml);
      for (int k = 0; k < mine; ++k) {
        const int it = item_of(k);
        const AttTile tl = tiles[it / heads];
        const int h = it % heads;
        const int cq = h * DH, ck = d + h * DH, cv = 2 * d + h * DH;
        int rows32 = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) rows32 += (tl.len[j] + 31) & ~31;
        const int row_bytes = 128 + (TAIL ? 32 : 0);
        {
          const int s = k % C::QK_ST;
          mbar_wait(&qk_empty[s], ((k / C::QK_ST) & 1) ^ 1);
          mbar_expect_tx(&qk_full[s], rows32 * row_bytes * C::NPL_QK);
          uint8_t* t = sm + s * C::QK_BYTES;
          uint8_t* tt = t + C::NPL_QK * ATQ_TILE;  // tail tiles (DH 80)
          int o = 0;
          for (int j = 0; j < 4; ++j) {
            for (int r0 = 0; r0 < tl.len[j]; r0 += 32, o += 32) {
              const int tok = tl.t0[j] + r0;
              tma_load_2d(t + o * 128, &mh, &qk_full[s], cq, tok);
              tma_load_2d(t + ATQ_TILE + o * 128, &mh, &qk_full[s], ck, tok);
              if (SPLIT) {
                tma_load_2d(t + 2 * ATQ_TILE + o * 128, &ml, &qk_full[s], cq, tok);
                tma_load_2d(t + 3 * ATQ_TILE + o * 128, &ml, &qk_full[s], ck, tok);
              }
              if (TAIL) {
                tma_load_2d(tt + o * 32, &th, &qk_full[s], cq + 64, tok);
                tma_load_2d(tt + ATQ_TTILE + o * 32, &th, &qk_full[s], ck + 64, tok);
                if (SPLIT) {
                  tma_load_2d(tt + 2 * ATQ_TTILE + o * 32, &tl_, &qk_full[s], cq + 64, tok);
                  tma_load_2d(tt + 3 * ATQ_TTILE + o * 32, &tl_, &qk_full[s], ck + 64, tok);
                }
              }
            }
          }
        }
        {
          const int s = k % C::V_ST;
          mbar_wait(&v_empty[s], ((k / C::V_ST) & 1) ^ 1);
          mbar_expect_tx(&v_full[s], rows32 * (TAIL ? 256 : 128) * C::NPL_V);
          uint8_t* t = sm + C::QK_ST * C::QK_BYTES + s * C::V_BYTES;
          constexpr int VPL = TAIL ? 2 * ATQ_TILE : ATQ_TILE;  // bytes per V plane
          int o = 0;
          for (int j = 0; j < 4; ++j) {
            for (int r0 = 0; r0 < tl.len[j]; r0 += 32, o += 32) {
              const int tok = tl.t0[j] + r0;
              tma_load_2d(t + o * 128, &mh, &v_full[s], cv, tok);
              if (SPLIT) tma_load_2d(t + VPL + o * 128, &ml, &v_full[s], cv, tok);
              if (TAIL) {  // dims 64..127 (past the tensor's last column: zero-filled)
                tma_load_2d(t + ATQ_TILE + o * 128, &mh, &v_full[s], cv + 64, tok);
                if (SPLIT) tma_load_2d(t + VPL + ATQ_TILE + o * 128, &ml, &v_full[s], cv + 64, tok);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ S issuer
    if (lane == 0) {
      auto issue_s = [&](int k) {
        const int b = k & 1;
        const int n16 = (att_tile_rows(tiles[item_of(k) / heads]) + 15) & ~15;
        const int s = k % C::QK_ST;
        const uint32_t idesc = idesc_f16kind(128, n16, fmt);
        uint8_t* t = sm + s * C::QK_BYTES;
        const uint64_t qh = umma_desc_sw128(t), kh = umma_desc_sw128(t + ATQ_TILE);
        const uint64_t ql = umma_desc_sw128(t + 2 * ATQ_TILE),
                       kl = umma_desc_sw128(t + 3 * ATQ_TILE);
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
        if (TAIL) {  // head dims 64..79: one more k-step from the 32B-swizzled tail tiles
          uint8_t* tt = t + C::NPL_QK * ATQ_TILE;
          const uint64_t qht = umma_desc_sw32(tt), kht = umma_desc_sw32(tt + ATQ_TTILE);
          tc_mma_bf16(ts, qht, kht, idesc, 1);
          if (SPLIT) {
            const uint64_t qlt = umma_desc_sw32(tt + 2 * ATQ_TTILE),
                           klt = umma_desc_sw32(tt + 3 * ATQ_TTILE);
            tc_mma_bf16(ts, qlt, kht, idesc, 1);
            tc_mma_bf16(ts, qht, klt, idesc, 1);
          }
        }
        tc_commit(&s_full[b]);
        tc_commit(&qk_empty[s]);
      };
      for (int k = 0; k < mine; ++k) {
        if (k >= 2) mbar_wait(&o_full[oslot(k - 2)], opar(k - 2));  // region free
        mbar_wait(&qk_full[k % C::QK_ST], (k / C::QK_ST) & 1);
        tc_fence_after();
        ATT_TRACE(k, 0);
        issue_s(k);
      }
    }
  } else if (warp == 18) {
    // ------------------------------------------------------------ O issuer
    if (lane == 0) {
      auto issue_o = [&](int k) {
        const int b = k & 1;
        const int n16 = (att_tile_rows(tiles[item_of(k) / heads]) + 15) & ~15;
        const int s = k % C::V_ST;
        // B = V is MN-major (keys x head dims). MODE 3 issues Ph·[Vh | Vl] as one
        // N=128 MMA (Vh and Vl tiles 16 KB apart = the MN-direction atom stride)
        // into O columns [0,64) | [64,128), plus Pl·Vh into [0,64):
        // 2 A-from-TMEM MMAs per 16 keys instead of 3.
        const uint32_t idesc64 = idesc_f16kind(128, 64, fmt) | (1u << 16);
        const uint32_t idesc128 = idesc_f16kind(128, 128, fmt) | (1u << 16);
        uint8_t* t = sm + C::QK_ST * C::QK_BYTES + s * C::V_BYTES;
        const uint32_t tp = tm + b * 128, to = tm + ocol(k);
        const uint32_t idesc80 = idesc_f16kind(128, 80, fmt) | (1u << 16);
        for (int kk = 0; kk < n16; kk += 16) {
          const uint32_t ph_ = tp + 32 * (kk >> 5) + 8 * ((kk >> 4) & 1);
          const uint64_t vh = umma_desc_sw128(t + kk * 128);
          if (TAIL) {
            // DH 80: O[0,80) = P·V as one N=80 product per operand pair, B spanning
            // the plane's two 64-column atoms (LBO = atom stride); hi·hi + lo·hi + hi·lo
            const uint64_t v80h = umma_desc_sw128_mn(t + kk * 128, ATQ_TILE);
            tc_mma_ts(to, ph_, v80h, idesc80, kk != 0);
            if (PSPLIT) tc_mma_ts(to, ph_ + 16, v80h, idesc80, 1);
            if (SPLIT)
              tc_mma_ts(to, ph_, umma_desc_sw128_mn(t + 2 * ATQ_TILE + kk * 128, ATQ_TILE), idesc80, 1);
          } else {
            if (SPLIT)
              tc_mma_ts(to, ph_, umma_desc_sw128_mn(t + kk * 128, ATQ_TILE), idesc128, kk != 0);
            else
              tc_mma_ts(to, ph_, vh, idesc64, kk != 0);
            if (PSPLIT) tc_mma_ts(to, ph_ + 16, vh, idesc64, 1);
          }
        }
        tc_commit(&o_full[oslot(k)]);
        tc_commit(&v_empty[s]);
      };
      for (int k = 0; k < mine; ++k) {
        if (DEFER && k >= 4) mbar_wait(&o_empty[k & 3], ((k - 4) >> 2) & 1);  // slot read
        mbar_wait(&p_full[k & 1], (k >> 1) & 1);
        mbar_wait(&v_full[k % C::V_ST], (k / C::V_ST) & 1);
        tc_fence_after();
        ATT_TRACE(k, 1);
        issue_o(k);
      }
    }
  } else if (warp < 18) {
    // ------------------------------------------------------------ softmax + epilogue
    // Warp (q, hr) of a group owns tile rows 32q + 16hr .. +15 (TMEM lane quarter
    // q, lane half hr). With the 16x32bx2 TMEM shape, lanes 0-15 of the warp read
    // key chunk 2j and lanes 16-31 chunk 2j+1 of the same 16 rows, so the row max
    // and row sum combine with one shuffle (no cross-warp exchange).
    const int g = (warp - 2) >> 3;          // group = region = item parity
    const int hr = ((warp - 2) >> 2) & 1;   // which 16 rows of the quarter
    const int q = warp & 3;                 // TMEM lane quarter
    const int cp = lane >> 4;               // chunk parity this thread handles
    const int r = q * 32 + hr * 16 + (lane & 15);  // tile row owned by this thread
    const uint32_t lane_off = (uint32_t)(q * 32 + hr * 16) << 16;
    const float c2 = scale * 1.4426950408889634f;  // exp(x*scale) = 2^(x*c2)
    // This warp's rows lie in one 32-row granule = (part of) one sequence slot:
    // its keys are [ks, ke) of the tile (warp-uniform).
    struct Meta {
      int h, n16, ks, ke, t0;
      bool active;
    };
    auto meta = [&](int k) {
      const int it = item_of(k);
      const AttTile tl = tiles[it / heads];
      Meta m{it % heads, (att_tile_rows(tl) + 15) & ~15, 0, 0, 0, false};
      int o = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int L = tl.len[j], R = (L + 31) & ~31;
        if (q * 32 >= o && q * 32 < o + R) {
          m.ks = o;
          m.ke = o + L;
          m.t0 = tl.t0[j];
        }
        o += R;
      }
      m.active = m.ke > q * 32 + hr * 16;  // some row of this warp is real
      return m;
    };
    const bool tr = hr == 0 && q == 0 && lane == 0;
    // ---- epilogue of item k: lanes 0-15 O columns 0..31, lanes 16-31 columns 32..63
    auto epilogue = [&](int k, const Meta& m, float rsum) {
      mbar_wait(&o_full[oslot(k)], opar(k));
      if (tr) ATT_TRACE(k, 4);
      tc_fence_after();
      if (m.active) {
        const int h = m.h, ks = m.ks, ke = m.ke, t0 = m.t0;
        const uint32_t to = tm + lane_off + ocol(k);
        const float inv = 1.0f / rsum;
        const size_t ob = (size_t)(t0 + r - ks) * ldc + h * DH + cp * 32;
        float v[32];
        tmem_ld_16x32bx2(to, v);
        if (SPLIT && !TAIL) {  // O = Ph·Vh + Pl·Vh (columns 0..63) + Ph·Vl (64..127)
          float w[32];
          tmem_ld_16x32bx2(to + 64, w);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += w[i];
        }
        if (r < ke) {
          // ctx is a convex combination of range-checked V rows: no fp16 overflow;
          // 16 pieces = 32 bytes per plane -> one 256-bit store each
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t hh[8], ll[8];
#pragma unroll
            for (int i = 0; i < 16; i += 2)
              split2(v[half * 16 + i] * inv, v[half * 16 + i + 1] * inv, fmt, hh[i / 2], ll[i / 2]);
            st_global_256(ch + ob + half * 16, hh);
            if (SPLIT) st_global_256(cl + ob + half * 16, ll);
          }
        }
        if (TAIL) {  // head dims 64..79: lanes 0-15 dims 64..71, lanes 16-31 dims 72..79
          float t8[8];
          tmem_ld_16x32bx2_8(to + 64, t8);
          if (r < ke) {
            uint32_t hh[4], ll[4];
#pragma unroll
            for (int i = 0; i < 8; i += 2) split2(t8[i] * inv, t8[i + 1] * inv, fmt, hh[i / 2], ll[i / 2]);
            const size_t ot = (size_t)(t0 + r - ks) * ldc + h * DH + 64 + cp * 8;
            *reinterpret_cast<uint4*>(ch + ot) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
            if (SPLIT) *reinterpret_cast<uint4*>(cl + ot) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
          }
        }
      }
      tc_fence_before();
      if (DEFER) mbar_arrive(&o_empty[k & 3]);
      if (tr) ATT_TRACE(k, 5);
    };
    Meta prev{};
    float prev_rsum = 1.f;
    for (int k = g; k < mine; k += 2) {
      const int b = g;
      const Meta m = meta(k);
      const int n16 = m.n16, ks = m.ks, ke = m.ke;
      const bool active = m.active;
      mbar_wait(&s_full[b], (k >> 1) & 1);
      if (tr) ATT_TRACE(k, 2);
      tc_fence_after();
      float rsum = 1.f;
      if (active) {
        const uint32_t trow = tm + b * 128 + lane_off;
        const int c_lo = ks >> 5, c_hi = (ke - 1) >> 5, c_end = (n16 + 31) >> 5;
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (2 * j + 1 >= c_lo && 2 * j <= c_hi) {  // warp-uniform: the pair has keys
            float v[32];
            tmem_ld_16x32bx2(trow + j * 64, v);
            const int c = 2 * j + cp;
            if (c >= c_lo && c <= c_hi) {
              const int e = ke - c * 32;
              if (e >= 32) {
#pragma unroll
                for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (i < e) mx = fmaxf(mx, v[i]);
              }
            }
          }
        }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float mxc = mx * c2;
        float2 sum2 = make_float2(0.f, 0.f);  // even / odd keys, summed at the end
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (2 * j < c_end) {  // warp-uniform
            const int c = 2 * j + cp;
            const bool in = c >= c_lo && c <= c_hi;
            const int e = ke - c * 32;
            float v[32];
            tmem_ld_16x32bx2(trow + j * 64, v);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              uint32_t hh[8], ll[8];
              if (in && e >= 32) {
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                  const float2 t = ffma2(make_float2(v[half * 16 + i], v[half * 16 + i + 1]),
                                         make_float2(c2, c2), make_float2(-mxc, -mxc));
                  const float p0 = fast_exp2(t.x), p1 = fast_exp2(t.y);
                  sum2 = fadd2(sum2, make_float2(p0, p1));
                  split2(p0, p1, fmt, hh[i / 2], ll[i / 2]);
                }
              } else if (in) {
                const int eh = e - half * 16;
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                  const float2 t = ffma2(make_float2(v[half * 16 + i], v[half * 16 + i + 1]),
                                         make_float2(c2, c2), make_float2(-mxc, -mxc));
                  const float p0 = i < eh ? fast_exp2(t.x) : 0.f;
                  const float p1 = i + 1 < eh ? fast_exp2(t.y) : 0.f;
                  sum2 = fadd2(sum2, make_float2(p0, p1));
                  split2(p0, p1, fmt, hh[i / 2], ll[i / 2]);
                }
              } else {
#pragma unroll
                for (int i = 0; i < 8; ++i) hh[i] = ll[i] = 0u;
              }
              // lanes 0-15 -> chunk 2j, lanes 16-31 -> chunk 2j+1 (32 columns on)
              tmem_st_16x32bx2_8(trow + j * 64 + half * 8, hh);
              if (PSPLIT) tmem_st_16x32bx2_8(trow + j * 64 + 16 + half * 8, ll);
            }
          }
        }
        tc_wait_st();
        rsum = sum2.x + sum2.y;
        rsum += __shfl_xor_sync(0xffffffffu, rsum, 16);
      }
      tc_fence_before();
      mbar_arrive(&p_full[b]);
      if (tr) ATT_TRACE(k, 3);
      if (!DEFER) {
        epilogue(k, m, rsum);
      } else {
        if (k >= g + 2) epilogue(k - 2, prev, prev_rsum);  // O(k-2) finished during softmax(k)
        prev = m;
        prev_rsum = rsum;
      }
    }
    if (DEFER && mine > g) epilogue(g + 2 * ((mine - 1 - g) / 2), prev, prev_rsum);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tm);
  }
}

cudaError_t att_set_trace(long long* dev_buf) {
  return cudaMemcpyToSymbol(g_att_trace, &dev_buf, sizeof(dev_buf));
}

void att_plan_tiles(const int32_t* cu, int nseq, bool tc_ok, std::vector<AttTile>& tiles,
                    std::vector<int2>& work) {
  tiles.clear();
  work.clear();
  AttTile cur{};
  int used = 0, nslot = 0;  // 32-row granules used, sequences in `cur`
  for (int s = 0; s < nseq; ++s) {
    const int a = cu[s], L = cu[s + 1] - a;
    if (!tc_ok || L > 128) {  // SIMT: 64-query blocks; tcgen05 long kernel: 128-query blocks
      for (int q = 0; q < L; q += tc_ok ? 128 : 64) work.push_back(make_int2(s, q));
      continue;
    }
    const int R = (L + 31) & ~31;
    if (nslot == 4 || used + R > 128) {
      tiles.push_back(cur);
      cur = AttTile{};
      used = nslot = 0;
    }
    cur.t0[nslot] = a;
    cur.len[nslot] = L;
    ++nslot;
    used += R;
  }
  if (nslot) tiles.push_back(cur);
}

template <int MODE, int DH>
static void att_launch_tc(const CUtensorMap* mh, const CUtensorMap* ml, const CUtensorMap* th,
                          const CUtensorMap* tl, const AttTile* tiles, int n_items, int heads,
                          int d, float scale, int fmt, uint16_t* ch, uint16_t* cl, int ldc,
                          int grid, cudaStream_t st) {
  constexpr int SM = AtqCfg<MODE, DH>::SMEM;
  auto kern = attention_tc_kernel<MODE, DH>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SM);
  kern<<<grid, ATQ_THREADS, SM, st>>>(*mh, *ml, *th, *tl, tiles, n_items, heads, d, scale, fmt,
                                      ch, cl, ldc);
}

cudaError_t launch_attention_tc(const CUtensorMap* mh, const CUtensorMap* ml,
                                const CUtensorMap* th, const CUtensorMap* tl, int mode,
                                const AttTile* tiles, int n_tiles, int heads, int d, int fmt,
                                uint16_t* ch, uint16_t* cl, int ldc, int* ovf, int num_sms,
                                cudaStream_t st) {
  (void)ovf;  // ctx is a convex combination of range-checked V rows
  if (n_tiles <= 0) return cudaSuccess;
  const int dh = d / heads;
  if (dh != 64 && dh != 80) return cudaErrorInvalidValue;
  const float scale = 1.0f / sqrtf((float)d / (float)heads);
  const int n_items = n_tiles * heads;
  const int grid = n_items < num_sms ? n_items : num_sms;
  const CUtensorMap* mlo = mode == 3 ? ml : mh;
  const CUtensorMap* tlo = mode == 3 ? tl : th;
#define ATT_GO(M, D) \
  att_launch_tc<M, D>(mh, mlo, th, tlo, tiles, n_items, heads, d, scale, fmt, ch, cl, ldc, grid, st)
  if (dh == 64) {
    if (mode == 3) ATT_GO(3, 64); else if (mode == 2) ATT_GO(2, 64); else ATT_GO(1, 64);
  } else {
    if (mode == 3) ATT_GO(3, 80); else if (mode == 2) ATT_GO(2, 80); else ATT_GO(1, 80);
  }
#undef ATT_GO
  return cudaGetLastError();
}

}  // namespace mfg
