// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M, N] = A[M, K] · Bᵀ   with A row-major [M][K] and B stored [N][K]
//   (weights are transposed once at load so both operands are K-major).
//
// Replaces the reference's `_mm`/`_affine` (`pkg/src/metricforge/encoder.py:120-126`)
// and fuses the ops that follow each affine into the epilogue:
//   EPI_F32        out = acc + bias                         (QKV, head output)
//   EPI_F32_RES    out = acc + bias + residual              (O-proj, FFN2)
//   EPI_GELU_SPLIT out = gelu_tanh2(acc + bias) -> hi/lo pieces (FFN1, `encoder.py:149-151`)
//   EPI_TANH_SPLIT out = tanh(acc + bias)      -> hi/lo pieces (head hidden stages, `:190-196`)
//   EPI_SPLIT      out = acc + bias            -> hi/lo pieces (Q|K|V for attention)
//
// SPLIT=true: A = A_hi + A_lo and B = B_hi + B_lo are pairs of 16-bit pieces
// and every k-step issues  D += A_hi·B_hi + A_lo·B_hi + A_hi·B_lo  into one fp32
// TMEM accumulator. With fp16 pieces (the fp32-parity path) each operand keeps
// ~22 significant bits; with bf16 pieces ("bf16x3") ~16 bits over the fp32 range.
// SPLIT=false is the plain one-MMA-per-k-step path.
//
// Roles (384 threads): warp0 lane0 = TMA producer, warp1 lane0 = MMA issuer,
// warp2 = TMEM allocator, warps 4-11 = epilogue. Epilogue warp w reads TMEM
// lanes 32*(w%4)..+31 (= tile rows) and every other 32-column chunk; each chunk
// is transposed through shared memory so global traffic is float4 per lane,
// 4 full 128-byte row segments per warp instruction, with the residual chunk
// prefetched before the math. Two TMEM accumulators let the epilogue of tile i
// overlap the MMAs of tile i+1. Tiles are assigned round-robin to a persistent
// grid of <= #SM CTAs.
#pragma once
#include <type_traits>

#include "ptx.cuh"

namespace mfg {

enum EpiMode : int {
  EPI_F32 = 0, EPI_F32_RES = 1, EPI_GELU_SPLIT = 2, EPI_TANH_SPLIT = 3, EPI_SPLIT = 4
};

struct GemmArgs {
  int M, N, K;               // M real rows; N, K padded (N % BN == 0, K % 64 == 0)
  const float* bias;         // [N]
  const float* alpha;        // [N] or null: out = acc * alpha + bias. The fp32-parity path
                             // stores each weight column pre-scaled by a power of two
                             // (largest |w| in [2^14, 2^15)), so alpha = 2^-e is exact
  const float* residual;     // [M][ldr] (EPI_F32_RES), fp32 ...
  int ldr;
  const uint16_t* res_hi;    // ... or, when non-null, 16-bit hi (+ lo) pieces [M][ldr]
  const uint16_t* res_lo;    //     in `fmt` (residual stream kept as operand pieces)
  float* out_f32;            // [M][ldo] (EPI_F32*) ...
  int ldo;
  uint16_t* out16;           // ... or, when non-null, binary16 [M][ldo] (reference fp16 mode)
  uint16_t* out_hi;          // [M][ldh] (split epilogues), 16-bit pieces in `fmt`
  uint16_t* out_lo;          // may be null when the consumer GEMM is not split
  int ldh;
  int fmt;                   // FMT_F16 / FMT_BF16: operand format of A, B and out_hi/lo
  int* ovf;                  // set to 1 when an fp16 output overflows
  int group_m;               // tile raster: blocks of group_m M-tiles walk M fastest (0: N fastest)
  int r16;                   // reference binary16 mode (`encoder.py:120-126`): round the
                             // product to fp16, add the fp16 bias in fp16, round residual
                             // sums to fp16 (bias must hold fp16-representable values)
  int kchunk;                // CTA-pair kernel: k-blocks per fresh TMEM accumulator (0 = all K).
  int* tile_ctr;             // CTA-pair kernel: zeroed tile counter -> tiles handed out in index
                             // order as pairs free up (null: static round-robin)
  float* partial;            // [gridDim.x][256/4][128][4] fp32: running sum of the finished chunks
                             // (the tcgen05 accumulator rounds each MMA's add toward zero, so
                             // error grows with the adds per accumulator; chunk sums are
                             // added round-to-nearest on the CUDA cores)
};

__device__ __forceinline__ float round16(float v) { return __half2float(__float2half_rn(v)); }

// Tile index -> (m block, n block). group_m > 0: groups of group_m M-blocks
// walk M fastest, so the CTAs running at the same time share each weight
// (B) tile and re-read each activation (A) block while it is still in L2.
__device__ __forceinline__ void tile_mn(int tile, int num_m, int num_n, int group_m, int& m,
                                        int& n) {
  if (group_m <= 0) {
    m = tile / num_n;
    n = tile % num_n;
    return;
  }
  const int per = group_m * num_n;
  const int first = (tile / per) * group_m;
  const int gs = min(group_m, num_m - first);
  const int in = tile % per;
  m = first + in % gs;
  n = in / gs;
}

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 384;
constexpr int GEMM_EPI_WARPS = 8;
constexpr int GEMM_SMEM_LIMIT = 232448;  // 227 KB opt-in dynamic smem
// per-warp transpose buffer: 32 rows x 32 floats, 16-byte chunks XOR-swizzled by
// row (8 lanes writing or reading float4 hit 8 distinct bank quads)
constexpr int GEMM_EPI_STRIDE = 32;
constexpr int GEMM_EPI_BYTES = GEMM_EPI_WARPS * 32 * GEMM_EPI_STRIDE * 4;
constexpr int GEMM_BAR_BYTES = 320;
constexpr int TRING = 4;  // CTA-pair kernel: tile-id ring depth

template <int BN, bool SPLIT>
struct GemmCfg {
  static constexpr int NOPS = SPLIT ? 2 : 1;
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = NOPS * (A_BYTES + B_BYTES);
  static constexpr int STAGES_FIT =
      (GEMM_SMEM_LIMIT - 1024 - GEMM_EPI_BYTES - GEMM_BAR_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int SMEM_BYTES =
      1024 + STAGES * STAGE_BYTES + GEMM_EPI_BYTES + GEMM_BAR_BYTES;
  static constexpr uint32_t TMEM_COLS =
      2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  static_assert(STAGES >= 2, "pipeline needs at least two stages");
  static_assert(BN % 32 == 0 && BN >= 32 && BN <= 256, "BN");
};

__device__ __forceinline__ __half2 u2h2(uint32_t u) { return *reinterpret_cast<const __half2*>(&u); }
__device__ __forceinline__ uint32_t h22u(__half2 h) { return *reinterpret_cast<const uint32_t*>(&h); }

// One accumulator tile's epilogue for one warp: TMEM lanes = tile rows
// row0..row0+rows-1 (this warp's quarter), every other 32-column chunk starting
// at `half`*32; each chunk transposed through `buf` so global traffic is float4
// per lane, 4 full 128-byte row segments per warp instruction.
// FMT / R16 are the run-time `args.fmt` / `args.r16` hoisted to compile time.
// R16 (reference binary16 mode, `encoder.py:120-126`): the product is rounded to
// binary16 and the (binary16) bias added in binary16; both are exact IEEE binary16
// operations, done as packed __hadd2 (an fp32 sum of two binary16 values rounded
// once to binary16 is the correctly rounded binary16 sum, so this equals
// round16(round16(acc) + b)); with a binary16 residual and output the residual
// sum is one more __hadd2.
//
// CW (transpose width, 32 or 16 columns): each warp still owns the same 32-column
// chunks (the K-chunk partial sums are per warp), processed CW columns at a
// time; CW = 16 halves the transpose buffer (2 KB per warp), which buys the
// single-MMA kernels a sixth mainloop stage with all 16 epilogue warps.
template <int BN, int EPI, int NSUB, int FMT, bool R16, int CW = 32>
__device__ __forceinline__ void epi_tile_t(const GemmArgs& args, uint32_t tacc, int row0, int rows,
                                           int n0, int half, float* buf, int lane,
                                           const float* part_row = nullptr) {
  static_assert(CW == 32 || CW == 16, "transpose width");
  constexpr int NQ = CW / 4;        // float4 chunks per transposed row
  constexpr int RPI = 32 / NQ;      // rows per pass of the transposed phase (4 or 8)
  constexpr int NIT = 32 / RPI;     // passes (8 or 4)
  const int cg = lane % NQ;         // transposed phase: 4 columns 4*cg..4*cg+3
  const int rs = lane / NQ;         // row sub-index 0..RPI-1
  // 16-byte chunk swizzle of a transposed row (conflict-free writes and reads)
  auto swz = [](int r) { return CW == 32 ? (r & 7) : ((r >> 1) & 3); };
  const bool r16res = EPI == EPI_F32_RES && args.res_hi != nullptr;
  const bool h16 = R16 && r16res && args.res_lo == nullptr && args.out16 != nullptr;
  constexpr bool SPLIT_OUT = EPI == EPI_GELU_SPLIT || EPI == EPI_TANH_SPLIT || EPI == EPI_SPLIT;
  float amax = 0.f;  // largest |output| (fp16 overflow flag, split epilogues)
  uint32_t hinf = 0;  // R16 EPI_SPLIT: bit 15/31 set when a binary16 output is inf
#pragma unroll 1
  for (int c32 = half * 32; c32 < BN; c32 += 32 * NSUB)
#pragma unroll 1
  for (int c = c32; c < c32 + 32; c += CW) {
    const int col = n0 + c + 4 * cg;
    // prefetch this chunk's residual (8 x float4, or 8 x (hi, lo) 4 x 16-bit
    // pieces per lane) before touching TMEM; converted where it is consumed
    // float4 bits, or {hi pieces x2, lo pieces x2}; the reference binary16 mode
    // (R16) has no lo plane, so it keeps 8 bytes per row (register pressure of
    // the 16-warp single-MMA epilogue)
    using RawT = typename std::conditional<R16, uint2, uint4>::type;
    RawT rraw[NIT];
    if (EPI == EPI_F32_RES) {
#pragma unroll
      for (int it = 0; it < NIT; ++it) {
        const int r = it * RPI + rs;
        const size_t o = (size_t)(row0 + (r < rows ? r : 0)) * args.ldr + col;
        if constexpr (R16) {  // an fp32 residual (pre-norm x32) is read where it is used
          if (r16res) rraw[it] = *reinterpret_cast<const uint2*>(args.res_hi + o);
        } else if (r16res) {
          const uint2 h = *reinterpret_cast<const uint2*>(args.res_hi + o);
          const uint2 l = args.res_lo ? *reinterpret_cast<const uint2*>(args.res_lo + o)
                                      : make_uint2(0u, 0u);
          rraw[it] = make_uint4(h.x, h.y, l.x, l.y);
        } else {
          rraw[it] = *reinterpret_cast<const uint4*>(args.residual + o);
        }
      }
    }
    float v[CW];
    if constexpr (CW == 32) tmem_ld_32x32(tacc + c, v);
    else tmem_ld_32x16(tacc + c, v);
    if (part_row) {  // earlier K chunks of this tile (this thread's row, columns c..c+CW-1)
#pragma unroll
      for (int i = 0; i < CW; i += 4) {
        const float4 pp = *reinterpret_cast<const float4*>(part_row + (c + i) * GEMM_BM);
        v[i] += pp.x, v[i + 1] += pp.y, v[i + 2] += pp.z, v[i + 3] += pp.w;
      }
    }
#pragma unroll
    for (int i = 0; i < CW; i += 4)
      *reinterpret_cast<float4*>(buf + lane * CW + (((i >> 2) ^ swz(lane)) << 2)) =
          make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    __syncwarp();
    const float4 b = *reinterpret_cast<const float4*>(args.bias + col);
    // fma(acc, 1, b) == acc + b bitwise, so unscaled weights take the same path
    const float4 al = args.alpha ? *reinterpret_cast<const float4*>(args.alpha + col)
                                 : make_float4(1.f, 1.f, 1.f, 1.f);
    const __half2 bh01 = __floats2half2_rn(b.x, b.y), bh23 = __floats2half2_rn(b.z, b.w);
    auto row = [&](int it) {
      const int r = it * RPI + rs;
      const float4 s4 = *reinterpret_cast<const float4*>(buf + r * CW + ((cg ^ swz(r)) << 2));
      const size_t o = (size_t)(row0 + r);
      float2 x01, x23;
      if (R16) {
        __half2 h01 = __hadd2(__floats2half2_rn(s4.x, s4.y), bh01);
        __half2 h23 = __hadd2(__floats2half2_rn(s4.z, s4.w), bh23);
        if (EPI == EPI_F32_RES && h16) {
          h01 = __hadd2(h01, u2h2(rraw[it].x));
          h23 = __hadd2(h23, u2h2(rraw[it].y));
          *reinterpret_cast<uint2*>(args.out16 + o * args.ldo + col) =
              make_uint2(h22u(h01), h22u(h23));
          return;
        }
        if (EPI == EPI_SPLIT && args.out_lo == nullptr) {  // the sums are the output
          const uint32_t u01 = h22u(h01), u23 = h22u(h23);
          // |h| >= 0x7c00 (inf) sets bit 15 of its half after + 0x0400 (no carry out)
          hinf |= ((u01 & 0x7fff7fffu) + 0x04000400u) | ((u23 & 0x7fff7fffu) + 0x04000400u);
          *reinterpret_cast<uint2*>(args.out_hi + o * args.ldh + col) = make_uint2(u01, u23);
          return;
        }
        x01 = __half22float2(h01);
        x23 = __half22float2(h23);
      } else {
        x01 = ffma2(make_float2(s4.x, s4.y), make_float2(al.x, al.y), make_float2(b.x, b.y));
        x23 = ffma2(make_float2(s4.z, s4.w), make_float2(al.z, al.w), make_float2(b.z, b.w));
      }
      if (EPI == EPI_F32 || EPI == EPI_F32_RES) {
        if (EPI == EPI_F32_RES) {
          float2 r01, r23;
          if constexpr (R16) {
            if (r16res) {
              const uint16_t* h = reinterpret_cast<const uint16_t*>(&rraw[it].x);
              r01 = make_float2(load16(h, 0, FMT), load16(h, 1, FMT));
              r23 = make_float2(load16(h, 2, FMT), load16(h, 3, FMT));
            } else {
              const float4 rf = *reinterpret_cast<const float4*>(args.residual + o * args.ldr + col);
              r01 = make_float2(rf.x, rf.y);
              r23 = make_float2(rf.z, rf.w);
            }
          } else if (r16res) {
            const uint16_t* h = reinterpret_cast<const uint16_t*>(&rraw[it].x);
            const uint16_t* l = reinterpret_cast<const uint16_t*>(&rraw[it].z);
            r01 = make_float2(load16(h, 0, FMT) + load16(l, 0, FMT), load16(h, 1, FMT) + load16(l, 1, FMT));
            r23 = make_float2(load16(h, 2, FMT) + load16(l, 2, FMT), load16(h, 3, FMT) + load16(l, 3, FMT));
          } else {
            r01 = make_float2(__uint_as_float(rraw[it].x), __uint_as_float(rraw[it].y));
            r23 = make_float2(__uint_as_float(rraw[it].z), __uint_as_float(rraw[it].w));
          }
          x01 = fadd2(x01, r01);
          x23 = fadd2(x23, r23);
          if (R16) {
            x01 = make_float2(round16(x01.x), round16(x01.y));
            x23 = make_float2(round16(x23.x), round16(x23.y));
          }
        }
        if (args.out16) {
          *reinterpret_cast<uint2*>(args.out16 + o * args.ldo + col) =
              make_uint2(h22u(__floats2half2_rn(x01.x, x01.y)), h22u(__floats2half2_rn(x23.x, x23.y)));
        } else {
          *reinterpret_cast<float4*>(args.out_f32 + o * args.ldo + col) =
              make_float4(x01.x, x01.y, x23.x, x23.y);
        }
      } else {
        float2 y01 = x01, y23 = x23;
        if (EPI == EPI_GELU_SPLIT) {
          if (FMT == FMT_BF16 && args.out_lo == nullptr) {  // bf16 mode: one MUFU per value
            y01 = gelu_tanh2_bf16out(x01);
            y23 = gelu_tanh2_bf16out(x23);
          } else {
            y01 = gelu_tanh2(x01);
            y23 = gelu_tanh2(x23);
          }
        } else if (EPI == EPI_TANH_SPLIT) {
          y01 = make_float2(tanhf(x01.x), tanhf(x01.y));
          y23 = make_float2(tanhf(x23.x), tanhf(x23.y));
        }
        // fp16 range: |y| >= 65520 rounds to inf (binary16 overflow) -> flag below
        if (FMT == FMT_F16)
          amax = fmaxf(amax, fmaxf(fmaxf(fabsf(y01.x), fabsf(y01.y)), fmaxf(fabsf(y23.x), fabsf(y23.y))));
        uint32_t h01, h23, l01, l23;
        if (args.out_lo) {
          split2(y01.x, y01.y, FMT, h01, l01);
          split2(y23.x, y23.y, FMT, h23, l23);
          *reinterpret_cast<uint2*>(args.out_lo + o * args.ldh + col) = make_uint2(l01, l23);
        } else if (FMT == FMT_F16) {
          h01 = h22u(__floats2half2_rn(y01.x, y01.y));
          h23 = h22u(__floats2half2_rn(y23.x, y23.y));
        } else {
          const __nv_bfloat162 a = __floats2bfloat162_rn(y01.x, y01.y),
                               c2 = __floats2bfloat162_rn(y23.x, y23.y);
          h01 = *reinterpret_cast<const uint32_t*>(&a);
          h23 = *reinterpret_cast<const uint32_t*>(&c2);
        }
        *reinterpret_cast<uint2*>(args.out_hi + o * args.ldh + col) = make_uint2(h01, h23);
      }
    };
#pragma unroll
    for (int it = 0; it < NIT; ++it)
      if (it * RPI + rs < rows) row(it);
    __syncwarp();
  }
  if (SPLIT_OUT && FMT == FMT_F16 && args.ovf && (amax >= 65520.f || (hinf & 0x80008000u)))
    atomicOr(args.ovf, 1);
}

// Finished K chunk of a tile: this thread's TMEM lane (= row) and its columns,
// stored (first chunk) or added round-to-nearest into the fp32 running sum.
// Layout [column / 4][row][4]: a warp's float4 access covers 32 consecutive
// rows = 512 contiguous bytes (part_row points at this thread's row, column 0).
template <int BN, int NSUB>
__device__ __forceinline__ void drain_chunk(uint32_t tacc, float* part_row, bool first, int half) {
#pragma unroll 1
  for (int c = half * 32; c < BN; c += 32 * NSUB) {
    float v[32];
    tmem_ld_32x32(tacc + c, v);
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4* p = reinterpret_cast<float4*>(part_row + (c + i) * GEMM_BM);
      float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      if (!first) {
        const float4 q = *p;
        o.x += q.x, o.y += q.y, o.z += q.z, o.w += q.w;
      }
      *p = o;
    }
  }
}

// Calls f(integral_constant<FMT>, bool_constant<R16>) for the run-time format:
// the epilogue loop is instantiated once per combination (r16 implies fp16).
template <class F>
__device__ __forceinline__ void epi_dispatch(const GemmArgs& args, F&& f) {
  if (args.fmt == FMT_F16) {
    if (args.r16)
      f(std::integral_constant<int, FMT_F16>{}, std::true_type{});
    else
      f(std::integral_constant<int, FMT_F16>{}, std::false_type{});
  } else {
    f(std::integral_constant<int, FMT_BF16>{}, std::false_type{});
  }
}

// VAR pins the epilogue variant at compile time (1: binary16 reference mode,
// 2: bf16) so a kernel only carries the registers of the variant it runs; 0
// dispatches on the arguments.
template <int VAR, class F>
__device__ __forceinline__ void epi_dispatch_v(const GemmArgs& args, F&& f) {
  if constexpr (VAR == 1)
    f(std::integral_constant<int, FMT_F16>{}, std::true_type{});
  else if constexpr (VAR == 2)
    f(std::integral_constant<int, FMT_BF16>{}, std::false_type{});
  else
    epi_dispatch(args, f);
}

template <int BN, bool SPLIT, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapAh,
                   const __grid_constant__ CUtensorMap mapAl,
                   const __grid_constant__ CUtensorMap mapBh,
                   const __grid_constant__ CUtensorMap mapBl, const GemmArgs args) {
  using C = GemmCfg<BN, SPLIT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  float* epi_buf = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + GEMM_EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapAh);
    tma_prefetch(&mapBh);
    if (SPLIT) {
      tma_prefetch(&mapAl);
      tma_prefetch(&mapBl);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], GEMM_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_m = (args.M + GEMM_BM - 1) / GEMM_BM;
  const int num_n = args.N / BN;
  const int tiles = num_m * num_n;
  const int kblocks = args.K / GEMM_BK;

  auto stage_ptr = [&](int s, int which) -> uint8_t* {
    // which: 0 A_hi, 1 A_lo, 2 B_hi, 3 B_lo
    uint8_t* base = smem + s * C::STAGE_BYTES;
    if (which < 2) return base + which * C::A_BYTES;
    return base + C::NOPS * C::A_BYTES + (which - 2) * C::B_BYTES;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int mt, nt;
        tile_mn(tile, num_m, num_n, args.group_m, mt, nt);
        const int m0 = mt * GEMM_BM;
        const int n0 = nt * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          const int k0 = kb * GEMM_BK;
          tma_load_2d(stage_ptr(stage, 0), &mapAh, &full[stage], k0, m0);
          tma_load_2d(stage_ptr(stage, 2), &mapBh, &full[stage], k0, n0);
          if (SPLIT) {
            tma_load_2d(stage_ptr(stage, 1), &mapAl, &full[stage], k0, m0);
            tma_load_2d(stage_ptr(stage, 3), &mapBl, &full[stage], k0, n0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_f16kind(GEMM_BM, BN, (uint32_t)args.fmt);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ah = umma_desc_sw128(stage_ptr(stage, 0));
          const uint64_t bh = umma_desc_sw128(stage_ptr(stage, 2));
          const uint64_t al = SPLIT ? umma_desc_sw128(stage_ptr(stage, 1)) : 0;
          const uint64_t bl = SPLIT ? umma_desc_sw128(stage_ptr(stage, 3)) : 0;
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t adv = (uint64_t)(k * 32) >> 4;  // 16 bf16 along K
            tc_mma_bf16(d, ah + adv, bh + adv, idesc, (kb | k) != 0);
            if (SPLIT) {
              tc_mma_bf16(d, al + adv, bh + adv, idesc, 1);
              tc_mma_bf16(d, ah + adv, bl + adv, idesc, 1);
            }
          }
          tc_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;       // 0..7
    const int q = warp & 3;        // TMEM lane quarter == 32-row block of the tile
    const int half = ew >> 2;      // which alternate 32-column chunks this warp owns
    float* buf = epi_buf + ew * 32 * GEMM_EPI_STRIDE;
    epi_dispatch(args, [&](auto fmt_c, auto r16_c) {
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int mt, nt;
        tile_mn(tile, num_m, num_n, args.group_m, mt, nt);
        const int m0 = mt * GEMM_BM;
        const int n0 = nt * BN;
        const int row0 = m0 + q * 32;
        const int rows = min(32, args.M - row0);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (rows > 0)
          epi_tile_t<BN, EPI, 2, decltype(fmt_c)::value, decltype(r16_c)::value>(
              args, tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, row0, rows, n0, half, buf,
              lane);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    });
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------------
// CTA-pair variant (cluster of 2, tcgen05 cta_group::2), BN = 256: one tile is
// 256 rows x 256 columns; CTA rank r loads A rows m0+128r..+127 and B (weight)
// rows n0+128r..+127 into its own shared memory, the leader (rank 0) issues
// M=256 x N=256 x K=16 MMAs that read both CTAs' halves, and each CTA's
// accumulator (its 128 rows x 256 columns) lands in its own TMEM. Per CTA a
// k-block stage is A 16 KB + B 16 KB per piece instead of 16 + 32 KB, so three
// stages fit and each CTA pulls half the weight bytes per FLOP from L2.
// Barriers: full[s] lives in the leader (both CTAs' TMA bytes complete on it);
// empty[s] / tfull[a] are signalled in both CTAs by a multicast commit;
// tempty[a] lives in the leader and counts both CTAs' epilogue warps.
template <bool SPLIT, int EPI>
struct Gemm2Cfg {
  // Epilogue warps vs mainloop stages (they share the 227 KB of shared memory:
  // 4 KB of transpose buffer per epilogue warp). One-MMA (non-split) mainloops
  // need 3x the operand bytes per MMA-cycle and, with 5 stages, waited on TMA
  // data (ncu: their epilogue warps sat in the accumulator-full wait). Measured
  // per epilogue (same-box A/B, profiles/gemm_raster_r03.txt): 8 warps with the
  // 32-column transpose and 6 stages for the plain / residual / split epilogues;
  // 16 warps transposing 16 columns at a time (2 KB per warp, still 6 stages)
  // for GELU (FFN1), whose math needs the warps.
  static constexpr bool WIDE = !SPLIT && EPI == EPI_GELU_SPLIT;
  static constexpr int EPI_WARPS = WIDE ? 16 : 8;
  static constexpr int EPI_CW = WIDE ? 16 : 32;  // transpose width (epi_tile_t)
  static constexpr int THREADS = 128 + 32 * EPI_WARPS;
  static constexpr int EPI_BYTES = EPI_WARPS * 32 * EPI_CW * 4;
  static constexpr int NOPS = SPLIT ? 2 : 1;
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;  // this CTA's 128 rows
  static constexpr int B_BYTES = 128 * GEMM_BK * 2;      // this CTA's half of BN = 256
  static constexpr int STAGE_BYTES = NOPS * (A_BYTES + B_BYTES);
  static constexpr int STAGES_FIT =
      (GEMM_SMEM_LIMIT - 1024 - EPI_BYTES - GEMM_BAR_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + GEMM_BAR_BYTES;
  static_assert(STAGES >= 2, "pipeline needs at least two stages");
};

template <bool SPLIT, int EPI, int VAR = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Gemm2Cfg<SPLIT, EPI>::THREADS, 1)
    gemm2_tc_kernel(const __grid_constant__ CUtensorMap mapAh,
                    const __grid_constant__ CUtensorMap mapAl,
                    const __grid_constant__ CUtensorMap mapBh,
                    const __grid_constant__ CUtensorMap mapBl, const GemmArgs args) {
  using C = Gemm2Cfg<SPLIT, EPI>;
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  float* epi_buf = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* tr_full = tempty + 2;           // [TRING] tile id published (both CTAs)
  uint64_t* tr_empty = tr_full + TRING;     // [TRING] slot read by the MMA thread and rank 1's
                                            // producer (leader only; see ring_get)
  int* tring = reinterpret_cast<int*>(tr_empty + TRING);  // [TRING] tile ids, -1 = done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tring + TRING);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // Tile hand-out. The leader's producer thread takes the next tile (an atomic
  // counter: tiles start in index order as pairs free up, so the pairs that share
  // an A block or a weight slice stream it at the same time and hit in L2; the
  // static round-robin drifted apart over long K loops) and publishes it to a
  // TRING-deep ring in both CTAs; every other role reads the ids from its ring.
  // Slot release: only the leader's MMA thread and rank 1's producer arrive on
  // tr_empty (neither has generic global stores in flight, so the release-cluster
  // arrive is cheap). The epilogue warps need no release: they read slot i before
  // they drain any accumulator of tile i+1, and the producer can only publish
  // tile i+4 into that slot after the MMAs of tile i+3 started, which needed an
  // accumulator the epilogue drained from tile i+1 or later (with K-chunking,
  // every chunk alternates accumulators, which only tightens this).
  auto ring_get = [&](int i, int release) -> int {  // release: 0 none, 1 local, 2 remote
    const int slot = i % TRING;
    mbar_wait_cluster(&tr_full[slot], (uint32_t)(i / TRING) & 1);
    const int t = tring[slot];
    if (release == 1) mbar_arrive(&tr_empty[slot]);
    else if (release == 2) mbar_arrive_cluster(mapa_shared(&tr_empty[slot], 0));
    return t;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapAh);
    tma_prefetch(&mapBh);
    if (SPLIT) {
      tma_prefetch(&mapAl);
      tma_prefetch(&mapBl);
    }
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * C::EPI_WARPS);
    }
    for (int r = 0; r < TRING; ++r) {
      mbar_init(&tr_full[r], 1);
      mbar_init(&tr_empty[r], 2);  // leader's MMA thread + rank 1's producer
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_m = (args.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM);
  const int num_n = args.N / BN;
  const int tiles = num_m * num_n;
  const int kblocks = args.K / GEMM_BK;

  auto stage_ptr = [&](int s, int which) -> uint8_t* {
    // which: 0 A_hi, 1 A_lo, 2 B_hi, 3 B_lo
    uint8_t* base = smem + s * C::STAGE_BYTES;
    if (which < 2) return base + which * C::A_BYTES;
    return base + C::NOPS * C::A_BYTES + (which - 2) * C::B_BYTES;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t tring_peer = mapa_shared(tring, 1), trfull_peer = mapa_shared(tr_full, 1);
      for (int i = 0;; ++i) {
        int tile;
        if (rank == 0) {  // take the next tile and publish it to both CTAs' rings
          tile = args.tile_ctr ? atomicAdd(args.tile_ctr, 1) : pair + i * npairs;
          if (tile >= tiles) tile = -1;
          const int slot = i % TRING;
          mbar_wait_cluster(&tr_empty[slot], ((uint32_t)(i / TRING) & 1) ^ 1);
          tring[slot] = tile;
          st_shared_cluster_s32(tring_peer + 4 * slot, tile);
          mbar_arrive(&tr_full[slot]);
          mbar_arrive_cluster(trfull_peer + 8 * slot);
        } else {
          tile = ring_get(i, 2);
        }
        if (tile < 0) {
          // the last pair to finish re-arms the counter for the next launch (every
          // leader's final atomicAdd on tile_ctr[0] precedes its count here)
          if (rank == 0 && args.tile_ctr && atomicAdd(args.tile_ctr + 1, 1) == npairs - 1) {
            atomicExch(args.tile_ctr, 0);
            atomicExch(args.tile_ctr + 1, 0);
          }
          break;
        }
        int mt, nt;
        tile_mn(tile, num_m, num_n, args.group_m, mt, nt);
        const int m0 = mt * 2 * GEMM_BM + rank * GEMM_BM;
        const int n0 = nt * BN + rank * 128;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          const int k0 = kb * GEMM_BK;
          tma_load_2d_pair(stage_ptr(stage, 0), &mapAh, &full[stage], k0, m0);
          tma_load_2d_pair(stage_ptr(stage, 2), &mapBh, &full[stage], k0, n0);
          if (SPLIT) {
            tma_load_2d_pair(stage_ptr(stage, 1), &mapAl, &full[stage], k0, m0);
            tma_load_2d_pair(stage_ptr(stage, 3), &mapBl, &full[stage], k0, n0);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      // drain: the leader's last multicast commits must land before this CTA exits
      for (int i = 0; i < C::STAGES; ++i) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = idesc_f16kind(2 * GEMM_BM, BN, (uint32_t)args.fmt);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const int kc = args.kchunk > 0 ? args.kchunk : kblocks;
      for (int i = 0;; ++i) {
        if (ring_get(i, 1) < 0) break;
        for (int cb = 0; cb < kblocks; cb += kc) {  // one fresh accumulator per K chunk
          const int ce = min(kblocks, cb + kc);
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + acc * BN;
          for (int kb = cb; kb < ce; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint64_t ah = umma_desc_sw128(stage_ptr(stage, 0));
            const uint64_t bh = umma_desc_sw128(stage_ptr(stage, 2));
            const uint64_t al = SPLIT ? umma_desc_sw128(stage_ptr(stage, 1)) : 0;
            const uint64_t bl = SPLIT ? umma_desc_sw128(stage_ptr(stage, 3)) : 0;
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) {
              const uint64_t adv = (uint64_t)(k * 32) >> 4;  // 16 elements along K
              tc_mma_pair(d, ah + adv, bh + adv, idesc, (kb != cb) || k != 0);
              if (SPLIT) {
                tc_mma_pair(d, al + adv, bh + adv, idesc, 1);
                tc_mma_pair(d, ah + adv, bl + adv, idesc, 1);
              }
            }
            tc_commit_pair(&empty[stage], 3);
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          tc_commit_pair(&tfull[acc], 3);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;       // 0..EPI_WARPS-1
    const int q = warp & 3;        // TMEM lane quarter == 32-row block of this CTA's half tile
    const int half = ew >> 2;      // which 32-column chunks (every EPI_WARPS/4-th) it owns
    float* buf = epi_buf + ew * 32 * C::EPI_CW;
    const uint32_t tempty_leader = mapa_shared(&tempty[0], 0);
    const int kc = args.kchunk > 0 ? args.kchunk : kblocks;
    const int nch = (kblocks + kc - 1) / kc;
    float* part_row =
        nch > 1 ? args.partial + (size_t)blockIdx.x * GEMM_BM * BN + (q * 32 + lane) * 4 : nullptr;
    epi_dispatch_v<VAR>(args, [&](auto fmt_c, auto r16_c) {
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int i = 0;; ++i) {
        int tile = 0;
        if (lane == 0) tile = ring_get(i, 0);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile < 0) break;
        int mt, nt;
        tile_mn(tile, num_m, num_n, args.group_m, mt, nt);
        const int m0 = mt * 2 * GEMM_BM + rank * GEMM_BM;
        const int n0 = nt * BN;
        const int row0 = m0 + q * 32;
        const int rows = min(32, args.M - row0);
        for (int ch = 0; ch < nch; ++ch) {
          mbar_wait(&tfull[acc], acc_phase);
          tc_fence_after();
          const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
          if (ch + 1 < nch)
            drain_chunk<BN, C::EPI_WARPS / 4>(tacc, part_row, ch == 0, half);
          else if (rows > 0)
            epi_tile_t<BN, EPI, C::EPI_WARPS / 4, decltype(fmt_c)::value, decltype(r16_c)::value,
                       C::EPI_CW>(
                args, tacc, row0, rows, n0, half, buf, lane, part_row);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster_relaxed(tempty_leader + acc * 8);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      }
    });
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

}  // namespace mfg
