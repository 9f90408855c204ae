// Microbenchmark: tcgen05.mma issue->completion time for the attention shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2408_11853_b200/csrc tools/mma_probe.cu -o /tmp/mma_probe
// One CTA per SM; thread 0 issues batches of MMAs, commits, waits; cycles per batch.
#include <cstdio>
#include "ptx.cuh"
using namespace mfg;

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(long long* out, int mode, int N, int nmma, int reps) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  if (threadIdx.x == 0) {
    const uint32_t M = mode >= 2 ? 64 : 128;
    const uint32_t idesc = idesc_f16kind(M, N, 0) | ((mode & 1) ? (1u << 16) : 0u);
    const uint64_t a = umma_desc_sw128(sm), b = umma_desc_sw128(sm + 32768);
    long long tot = 0;
    for (int r = 0; r < reps; ++r) {
      const long long t0 = clock64();
      for (int i = 0; i < nmma; ++i) {
        if (mode == 0 || mode == 2) tc_mma_bf16(tm, a + 2 * (i & 3), b + 2 * (i & 3), idesc, i != 0);
        else mma_ts(tm + 256, tm + 8 * (i % 16), b + 128 * (i % 8), idesc, i != 0);
      }
      tc_commit(&bar);
      mbar_wait(&bar, r & 1);
      tot += clock64() - t0;
    }
    if (blockIdx.x == 0) out[0] = tot / reps;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tm); }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  struct { int mode, N, nmma; const char* what; } cases[] = {
    {0, 128, 1, "SS 128x128x16 x1"}, {0, 128, 12, "SS 128x128x16 x12"}, {0, 112, 12, "SS 128x112x16 x12"},
    {0, 64, 12, "SS 128x64x16 x12"}, {0, 256, 12, "SS 128x256x16 x12"}, {0, 256, 48, "SS 128x256x16 x48"},
    {0, 128, 48, "SS 128x128x16 x48"}, {1, 64, 1, "TS 128x64x16 x1"}, {1, 64, 21, "TS 128x64x16 x21"},
    {1, 64, 48, "TS 128x64x16 x48"}, {1, 128, 21, "TS 128x128x16 x21"}, {1, 256, 21, "TS 128x256x16 x21"},
    {2, 64, 12, "SS 64x64x16 x12"}, {2, 128, 12, "SS 64x128x16 x12"}, {2, 256, 12, "SS 64x256x16 x12"},
    {3, 64, 21, "TS 64x64x16 x21"}, {3, 128, 21, "TS 64x128x16 x21"}};
  for (auto& c : cases) {
    probe<<<148, 128, 100000>>>(d, c.mode, c.N, c.nmma, 64);
    cudaError_t e = cudaDeviceSynchronize();
    long long cyc = 0; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double ideal = (double)c.nmma * (c.mode >= 2 ? 64.0 : 128.0) * c.N * 16 * 2 / 8192.0;
    printf("%-22s %s  %6lld cycles/batch  (ideal %6.0f, %.2fx)\n", c.what, e ? cudaGetErrorString(e) : "ok", cyc, ideal, cyc / ideal);
  }
  return 0;
}
