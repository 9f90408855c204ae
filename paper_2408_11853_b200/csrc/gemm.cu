// Host side of the tcgen05 GEMM: tensor-map encoding (driver entry point, no
// libcuda link dependency) and the template dispatch.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "gemm_tc.cuh"
#include "kernels.h"

namespace mfg {

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

bool make_tmap_u16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint64_t ld_elems, uint32_t box_rows, char* err, size_t errcap) {
  return make_tmap_u16_box(map, ptr, rows, cols, ld_elems, 64, box_rows, 128, err, errcap);
}

bool make_tmap_u16_box(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                       uint64_t ld_elems, uint32_t box_cols, uint32_t box_rows, int swizzle,
                       char* err, size_t errcap) {
  PFN_encodeTiled enc = get_encode_fn();
  if (!enc) {
    snprintf(err, errcap, "cuTensorMapEncodeTiled unavailable from the driver");
    return false;
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = swizzle == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(err, errcap, "cuTensorMapEncodeTiled failed (%d): rows=%llu cols=%llu ld=%llu box=%u",
             (int)r, (unsigned long long)rows, (unsigned long long)cols,
             (unsigned long long)ld_elems, box_rows);
    return false;
  }
  return true;
}

// BN = 256 weights run on the CTA-pair kernel (tcgen05 cta_group::2);
// MFG_GEMM_SINGLE=1 in the environment forces the single-CTA kernel (A/B runs).
bool gemm_uses_pair(int bn) {
  static const bool single = [] {
    const char* e = getenv("MFG_GEMM_SINGLE");
    return e && e[0] == '1';
  }();
  return bn == 256 && !single;
}

int gemm_b_box_rows(int bn) { return gemm_uses_pair(bn) ? 128 : bn; }

// K-chunked accumulation (CTA-pair kernel): the tcgen05 accumulator rounds each
// MMA's add toward zero, so GEMM error grows with the adds per accumulator
// (rms 6e-5 of the output std at K = 10240). GEMMs deeper than
// 4096 (XLM-R XL's FFN2, K = 10240) restart a fresh accumulator every 2048 K
// and sum the chunks round-to-nearest (rms 1.2e-5); XL's K = 2560 GEMMs run
// in two halves. At config 2's K = 1024 / 4096 the error is small enough for
// the parity gate and the chunk drains would cost ~1.5 % (measured). MFG_KCHUNK=E chunks every E elements whenever
// K > E; MFG_KCHUNK=0 disables. Returns k-blocks per chunk (0 = no chunking).
int gemm_kchunk_blocks(int K, bool fine) {
  static const int env = [] {
    const char* e = getenv("MFG_KCHUNK");
    return e ? atoi(e) : -1;
  }();
  int elems = env;
  // default: K > 4096 in 2048-K chunks; 2048 < K <= 4096 in two halves only when
  // K is not a power of two (XLM-R XL's 2560: measured at no cost, parity 2.5x).
  // `fine` (split-operand GEMMs of models narrower than 1024): 512-K chunks --
  // config 1's std-0.25 fixture model goes from 5.0e-4 to 2.75e-4 max |delta|
  // against the reference for -2.5 % device / -1 % e2e throughput (128-K chunks:
  // 2.1e-4 for -20 %)
  if (env < 0)
    elems = fine ? 512
                 : K > 4096 ? 2048 : (K > 2048 && (K & (K - 1)) != 0) ? (K / 2 + 63) / 64 * 64 : 0;
  if (elems <= 0 || K <= elems) return 0;
  return elems / GEMM_BK > 0 ? elems / GEMM_BK : 1;
}

size_t gemm_partial_floats(int num_sms) { return (size_t)num_sms * GEMM_BM * 256; }

int gemm_pick_bn(int n_pad) {
  if (n_pad % 256 == 0) return 256;
  if (n_pad % 128 == 0) return 128;
  return 64;
}

template <int BN, bool SPLIT, int EPI>
static cudaError_t run(const CUtensorMap* ah, const CUtensorMap* al, const CUtensorMap* bh,
                       const CUtensorMap* bl, const GemmArgs& a, int num_sms, cudaStream_t st) {
  using C = GemmCfg<BN, SPLIT>;
  auto kern = gemm_tc_kernel<BN, SPLIT, EPI>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles = ((a.M + GEMM_BM - 1) / GEMM_BM) * (a.N / BN);
  if (tiles <= 0) return cudaSuccess;
  const int grid = tiles < num_sms ? tiles : num_sms;
  kern<<<grid, GEMM_THREADS, C::SMEM_BYTES, st>>>(*ah, SPLIT ? *al : *ah, *bh, SPLIT ? *bl : *bh,
                                                   a);
  return cudaGetLastError();
}

template <bool SPLIT, int EPI>
static cudaError_t run2(const CUtensorMap* ah, const CUtensorMap* al, const CUtensorMap* bh,
                        const CUtensorMap* bl, const GemmArgs& a, int num_sms, cudaStream_t st) {
  using C = Gemm2Cfg<SPLIT, EPI>;
  // single-MMA kernels (16 epilogue warps, 96 registers) get their epilogue
  // variant fixed at compile time: the binary16 mode then needs no lo-plane
  // residual registers and does not spill in the epilogue loop
  auto kern = SPLIT ? gemm2_tc_kernel<SPLIT, EPI, 0>
              : a.fmt == FMT_F16 && a.r16 ? gemm2_tc_kernel<SPLIT, EPI, 1>
              : a.fmt == FMT_BF16 ? gemm2_tc_kernel<SPLIT, EPI, 2>
                                  : gemm2_tc_kernel<SPLIT, EPI, 0>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles = ((a.M + 2 * GEMM_BM - 1) / (2 * GEMM_BM)) * (a.N / 256);
  if (tiles <= 0) return cudaSuccess;
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  kern<<<2 * pairs, C::THREADS, C::SMEM_BYTES, st>>>(*ah, SPLIT ? *al : *ah, *bh,
                                                       SPLIT ? *bl : *bh, a);
  return cudaGetLastError();
}

template <bool SPLIT>
static cudaError_t run2_epi(int epi, const CUtensorMap* ah, const CUtensorMap* al,
                            const CUtensorMap* bh, const CUtensorMap* bl, const GemmArgs& a,
                            int num_sms, cudaStream_t st) {
  switch (epi) {
    case EPI_F32: return run2<SPLIT, EPI_F32>(ah, al, bh, bl, a, num_sms, st);
    case EPI_F32_RES: return run2<SPLIT, EPI_F32_RES>(ah, al, bh, bl, a, num_sms, st);
    case EPI_GELU_SPLIT: return run2<SPLIT, EPI_GELU_SPLIT>(ah, al, bh, bl, a, num_sms, st);
    case EPI_TANH_SPLIT: return run2<SPLIT, EPI_TANH_SPLIT>(ah, al, bh, bl, a, num_sms, st);
    case EPI_SPLIT: return run2<SPLIT, EPI_SPLIT>(ah, al, bh, bl, a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

template <int BN, bool SPLIT>
static cudaError_t run_epi(int epi, const CUtensorMap* ah, const CUtensorMap* al,
                           const CUtensorMap* bh, const CUtensorMap* bl, const GemmArgs& a,
                           int num_sms, cudaStream_t st) {
  switch (epi) {
    case EPI_F32: return run<BN, SPLIT, EPI_F32>(ah, al, bh, bl, a, num_sms, st);
    case EPI_F32_RES: return run<BN, SPLIT, EPI_F32_RES>(ah, al, bh, bl, a, num_sms, st);
    case EPI_GELU_SPLIT: return run<BN, SPLIT, EPI_GELU_SPLIT>(ah, al, bh, bl, a, num_sms, st);
    case EPI_TANH_SPLIT: return run<BN, SPLIT, EPI_TANH_SPLIT>(ah, al, bh, bl, a, num_sms, st);
    case EPI_SPLIT: return run<BN, SPLIT, EPI_SPLIT>(ah, al, bh, bl, a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_gemm(const CUtensorMap* ah, const CUtensorMap* al, const CUtensorMap* bh,
                        const CUtensorMap* bl, int bn, int nsplit, int epi, const GemmArgs& a_in,
                        int num_sms, cudaStream_t st) {
  if (a_in.K % GEMM_BK != 0 || a_in.N % bn != 0) return cudaErrorInvalidValue;
  // Tile raster (profiles/gemm_raster_r03.txt, measured per GEMM with ncu, with
  // the dynamic tile hand-out): N-fastest (an M-block's A is shared by its
  // concurrent N-tiles) except for wide GEMMs whose weight does not stay
  // L2-resident (> 48 MB of pieces, >= 16 N-tiles: XLM-R XL QKV 79 MB, FFN1
  // 105 MB), which walk groups of 8 M-blocks so a few N-tiles' weights are
  // shared by 8 concurrent M-blocks -- XL FFN1 DRAM read 98 -> 22 GB, -14 %.
  // (Config 2's FFN2 was grouped by 4 under the static schedule; with dynamic
  // tiles N-fastest reads less: 5.8 vs 6.3 GB.) MFG_GEMM_GROUP=G forces G.
  static const int group_env = [] {
    const char* e = getenv("MFG_GEMM_GROUP");
    return e ? atoi(e) : -1;
  }();
  GemmArgs a = a_in;
  const int num_n = a.N / bn;
  const double w_bytes = (double)a.N * a.K * (nsplit == 2 ? 4 : 2);
  const int group = gemm_uses_pair(bn) && num_n >= 16 && w_bytes > 48e6 ? 8 : 0;
  a.group_m = group_env >= 0 ? group_env : group;
  const bool split = nsplit == 2;
  if (!gemm_uses_pair(bn) || a.partial == nullptr) a.kchunk = 0;
  if (gemm_uses_pair(bn))
    return split ? run2_epi<true>(epi, ah, al, bh, bl, a, num_sms, st)
                 : run2_epi<false>(epi, ah, al, bh, bl, a, num_sms, st);
  if (split) {
    if (bn == 256) return run_epi<256, true>(epi, ah, al, bh, bl, a, num_sms, st);
    if (bn == 128) return run_epi<128, true>(epi, ah, al, bh, bl, a, num_sms, st);
    if (bn == 64) return run_epi<64, true>(epi, ah, al, bh, bl, a, num_sms, st);
  } else {
    if (bn == 256) return run_epi<256, false>(epi, ah, al, bh, bl, a, num_sms, st);
    if (bn == 128) return run_epi<128, false>(epi, ah, al, bh, bl, a, num_sms, st);
    if (bn == 64) return run_epi<64, false>(epi, ah, al, bh, bl, a, num_sms, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace mfg
