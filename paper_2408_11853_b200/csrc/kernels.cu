// Non-GEMM kernels of the scoring path (sm_100a). Activations are token-packed
// ("varlen"): all sequences of all roles of a chunk are concatenated into one
// [T, d] stream; cu_seqlens[s]..cu_seqlens[s+1] are the rows of sequence s.
// Padded columns (d..ld) of every activation buffer are zero and stay zero.
#include "kernels.h"
#include "ptx.cuh"

namespace mfg {

// ------------------------------------------------------------------ embedding
// x_p = E_tok[id_p] + E_pos[p]   (`pkg/src/metricforge/encoder.py:166-168`)
// One CTA per sequence (positions restart at every cu_seqlens boundary), one
// warp per token. Ids outside [0, V) set bit 1 of `flag` (usage error) instead
// of reading out of bounds (`encoder.py:164-165`).
__global__ void embed_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ cu,
                             int V, int d, const float* __restrict__ tok,
                             const float* __restrict__ pe, float* __restrict__ x32, int ld,
                             uint16_t* __restrict__ xh, uint16_t* __restrict__ xl, int fmt,
                             int r16, int* flag) {
  const int start = cu[blockIdx.x], end = cu[blockIdx.x + 1];
  const int lane = threadIdx.x & 31;
  for (int t = start + (threadIdx.x >> 5); t < end; t += blockDim.x >> 5) {
    int id = ids[t];
    if (id < 0 || id >= V) {
      if (lane == 0) atomicOr(flag, 2);
      id = 0;
    }
    const float* a = tok + (size_t)id * d;
    const float* b = pe + (size_t)(t - start) * d;
    const size_t o = (size_t)t * ld;
    for (int c = lane; c < d; c += 32) {
      float v = a[c] + b[c];
      if (r16) v = __half2float(__float2half_rn(v));  // binary16 add (reference fp16 mode)
      if (x32) x32[o + c] = v;
      if (xh) store_split(xh, xl, o + c, v, fmt, flag);
    }
  }
}

// ------------------------------------------------------------------ layer norm
// out = (y - mean) / sqrt(var_pop + 1e-5) * g + b, one warp per row
// (`encoder.py:52-57, 128-130`). Writes any of: fp32 copy, 16-bit hi, lo pieces.
// V4 float4 per lane (d % 4 == 0), two-pass statistics from registers.
// IN16: the input row holds binary16 values (reference fp16 mode: the residual
// sum is already rounded to fp16), 2 instead of 4 bytes per element.
// One warp per row (a persistent row loop and a prefetched next row were both
// measured slower: fewer rows in flight per SM).
template <int V4, bool IN16>
__device__ __forceinline__ void ln_load_row(const void* __restrict__ yv, int t, int ld, int n4,
                                            int lane, float4 (&v)[V4]) {
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int c = i * 32 + lane;
    if (c >= n4) {
      v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (IN16) {
      const uint2 u = reinterpret_cast<const uint2*>(
          reinterpret_cast<const uint16_t*>(yv) + (size_t)t * ld)[c];
      const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
      const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
      v[i] = make_float4(a.x, a.y, b.x, b.y);
    } else {
      v[i] = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(yv) +
                                             (size_t)t * ld)[c];
    }
  }
}

// R16 (reference fp16 mode): the output is rounded to binary16, so the hi piece is
// that rounding and the lo piece is exactly 0.
template <int V4, bool IN16, bool R16>
__global__ void __launch_bounds__(256)
    layernorm_kernel(const void* __restrict__ yv, int T, int d, int ld,
                     const float* __restrict__ g, const float* __restrict__ bta,
                     float* __restrict__ out32, uint16_t* __restrict__ oh,
                     uint16_t* __restrict__ ol, int fmt, int* ovf) {
  const int lane = threadIdx.x & 31;
  const int n4 = d >> 2;
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T) return;
  float4 v[V4];
  ln_load_row<V4, IN16>(yv, t, ld, n4, lane, v);
  float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < V4; ++i)
    s2 = fadd2(s2, fadd2(make_float2(v[i].x, v[i].y), make_float2(v[i].z, v[i].w)));
  const float mean = warp_sum(s2.x + s2.y) / (float)d;
  const float2 nm = make_float2(-mean, -mean);
  float2 q2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    if (i * 32 + lane < n4) {
      const float2 a = fadd2(make_float2(v[i].x, v[i].y), nm);
      const float2 c = fadd2(make_float2(v[i].z, v[i].w), nm);
      q2 = ffma2(a, a, q2);
      q2 = ffma2(c, c, q2);
    }
  }
  const float rstd = 1.0f / sqrtf(warp_sum(q2.x + q2.y) / (float)d + 1e-5f);
  const float2 rs2 = make_float2(rstd, rstd);
  const size_t o = (size_t)t * ld;
  float amax = 0.f;
  uint32_t hinf = 0;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int c = i * 32 + lane;
    if (c < n4) {
      const float4 gg = reinterpret_cast<const float4*>(g)[c];
      const float4 bb = reinterpret_cast<const float4*>(bta)[c];
      const float2 r01 = ffma2(fmul2(fadd2(make_float2(v[i].x, v[i].y), nm), rs2),
                               make_float2(gg.x, gg.y), make_float2(bb.x, bb.y));
      const float2 r23 = ffma2(fmul2(fadd2(make_float2(v[i].z, v[i].w), nm), rs2),
                               make_float2(gg.z, gg.w), make_float2(bb.z, bb.w));
      if (R16) {
        const __half2 h01 = __floats2half2_rn(r01.x, r01.y), h23 = __floats2half2_rn(r23.x, r23.y);
        const uint32_t u01 = *reinterpret_cast<const uint32_t*>(&h01);
        const uint32_t u23 = *reinterpret_cast<const uint32_t*>(&h23);
        // |h| >= 0x7c00 (inf) sets bit 15 of its half after + 0x0400 (no carry out)
        hinf |= ((u01 & 0x7fff7fffu) + 0x04000400u) | ((u23 & 0x7fff7fffu) + 0x04000400u);
        if (out32) {
          const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
          reinterpret_cast<float4*>(out32 + o)[c] = make_float4(f01.x, f01.y, f23.x, f23.y);
        }
        if (oh) reinterpret_cast<uint2*>(oh + o)[c] = make_uint2(u01, u23);
        if (ol) reinterpret_cast<uint2*>(ol + o)[c] = make_uint2(0u, 0u);
      } else {
        if (out32) reinterpret_cast<float4*>(out32 + o)[c] = make_float4(r01.x, r01.y, r23.x, r23.y);
        if (oh) {
          // fp16 range: |r| >= 65520 rounds to inf -> flag
          amax = fmaxf(amax, fmaxf(fmaxf(fabsf(r01.x), fabsf(r01.y)), fmaxf(fabsf(r23.x), fabsf(r23.y))));
          uint32_t h01, h23, l01, l23;
          split2(r01.x, r01.y, fmt, h01, l01);
          split2(r23.x, r23.y, fmt, h23, l23);
          reinterpret_cast<uint2*>(oh + o)[c] = make_uint2(h01, h23);
          if (ol) reinterpret_cast<uint2*>(ol + o)[c] = make_uint2(l01, l23);
        }
      }
    }
  }
  const bool bad = R16 ? (hinf & 0x80008000u) != 0 : (fmt == FMT_F16 && amax >= 65520.f);
  if (bad && oh && ovf) atomicOr(ovf, 1);
}

// Scalar fallback for d % 4 != 0.
__device__ __forceinline__ float ln_in(const void* y, int in16, size_t i) {
  return in16 ? __half2float(__ushort_as_half(reinterpret_cast<const uint16_t*>(y)[i]))
              : reinterpret_cast<const float*>(y)[i];
}
__global__ void layernorm_scalar_kernel(const void* __restrict__ y, int in16, int T, int d,
                                        int ld, const float* __restrict__ g,
                                        const float* __restrict__ bta,
                                        float* __restrict__ out32, uint16_t* __restrict__ oh,
                                        uint16_t* __restrict__ ol, int fmt, int r16, int* ovf) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const size_t o = (size_t)t * ld;
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += ln_in(y, in16, o + c);
  const float mean = warp_sum(s) / (float)d;
  float q = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float a = ln_in(y, in16, o + c) - mean;
    q += a * a;
  }
  const float rstd = 1.0f / sqrtf(warp_sum(q) / (float)d + 1e-5f);
  for (int c = lane; c < d; c += 32) {
    float r = (ln_in(y, in16, o + c) - mean) * rstd * g[c] + bta[c];
    if (r16) r = __half2float(__float2half_rn(r));
    if (out32) out32[o + c] = r;
    if (oh) store_split(oh, ol, o + c, r, fmt, ovf);
  }
}

// ------------------------------------------------------------------ attention
// Exact fp32 masked-softmax attention per (sequence, head, 64-query block),
// flash-style over 64-key blocks (`encoder.py:132-147`, `masked_softmax` 60-66).
// PAD keys never exist in the packed layout; keys past the sequence end inside
// the last block get -inf and therefore exactly zero weight.
// CTA = 128 threads = 16 row groups (rg) x 8 column groups (cg). A thread owns
// 4 query rows; in S it owns keys cg + 8j (j < 8), in O the columns
// 32g + 4cg + {0..3}. Shared-memory operands are read as float4 (row strides
// are multiples of 4 floats; conflict-free across the 8 column groups).
constexpr int ATT_BQ = 64, ATT_BK = 64, ATT_THREADS = 128;
constexpr int ATT_PSTR = ATT_BK + 4;

template <int DHC>
struct AttCfg {
  static constexpr int DHMAX = DHC * 8;          // padded head dim
  static constexpr int STR = DHMAX + 4;          // Q/K/V row stride (floats)
  static constexpr int G = (DHMAX + 31) / 32;    // float4 column groups per thread in O
  static constexpr size_t SMEM = sizeof(float) * (3 * 64 * STR + 64 * ATT_PSTR);
};

// rows x dh fp32 tile = hi + lo of the QKV GEMM's 16-bit output pieces
__device__ __forceinline__ void att_load_tile(float* dst, int str, const uint16_t* hi,
                                              const uint16_t* lo, int ldq, int nrows, int dh,
                                              int dhmax, int tid, int fmt) {
  for (int i = tid; i < 64 * dhmax; i += ATT_THREADS) {
    const int r = i / dhmax, c = i % dhmax;
    float v = 0.f;
    if (r < nrows && c < dh) {
      const size_t o = (size_t)r * ldq + c;
      v = load16(hi, o, fmt);
      if (lo) v += load16(lo, o, fmt);
    }
    dst[r * str + c] = v;
  }
}

template <int DHC>
__global__ void __launch_bounds__(ATT_THREADS)
    attention_kernel(const uint16_t* __restrict__ qh, const uint16_t* __restrict__ ql, int ldq,
                     int d, int dh, float scale, const int32_t* __restrict__ cu,
                     const int2* __restrict__ work,
                     uint16_t* __restrict__ ch, uint16_t* __restrict__ cl, int ldc, int fmt,
                     int* ovf) {
  using C = AttCfg<DHC>;
  extern __shared__ float4 sm4[];
  float* Qs = reinterpret_cast<float*>(sm4);
  float* Ks = Qs + 64 * C::STR;
  float* Vs = Ks + 64 * C::STR;
  float* Ps = Vs + 64 * C::STR;

  const int2 w = work[blockIdx.x];
  const int seq = w.x, q0 = w.y;
  const int h = blockIdx.y;
  const int start = cu[seq];
  const int L = cu[seq + 1] - start;
  const int nq = min(ATT_BQ, L - q0);
  const int tid = threadIdx.x;
  const int rg = tid >> 3, cg = tid & 7;
  const int dh4 = (dh + 3) & ~3;
  const size_t qo = (size_t)(start + q0) * ldq + h * dh;
  att_load_tile(Qs, C::STR, qh + qo, ql ? ql + qo : nullptr, ldq, nq, dh, C::DHMAX, tid, fmt);

  float m[4], l[4], o[4][C::G * 4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    m[a] = -INFINITY;
    l[a] = 0.f;
#pragma unroll
    for (int i = 0; i < C::G * 4; ++i) o[a][i] = 0.f;
  }

  for (int k0 = 0; k0 < L; k0 += ATT_BK) {
    const int nk = min(ATT_BK, L - k0);
    __syncthreads();
    const size_t ko = (size_t)(start + k0) * ldq + d + h * dh;
    att_load_tile(Ks, C::STR, qh + ko, ql ? ql + ko : nullptr, ldq, nk, dh, C::DHMAX, tid, fmt);
    att_load_tile(Vs, C::STR, qh + ko + d, ql ? ql + ko + d : nullptr, ldq, nk, dh, C::DHMAX, tid,
                  fmt);
    __syncthreads();

    float s[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int j = 0; j < 8; ++j) s[a][j] = 0.f;
    for (int c = 0; c < dh4; c += 4) {
      float4 qv[4], kv[8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        qv[a] = *reinterpret_cast<const float4*>(Qs + (rg * 4 + a) * C::STR + c);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        kv[j] = *reinterpret_cast<const float4*>(Ks + (cg + 8 * j) * C::STR + c);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[a][j] = fmaf(qv[a].x, kv[j].x, s[a][j]);
          s[a][j] = fmaf(qv[a].y, kv[j].y, s[a][j]);
          s[a][j] = fmaf(qv[a].z, kv[j].z, s[a][j]);
          s[a][j] = fmaf(qv[a].w, kv[j].w, s[a][j]);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s[a][j] = (cg + 8 * j < nk) ? s[a][j] * scale : -INFINITY;
        mx = fmaxf(mx, s[a][j]);
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      const float mn = fmaxf(m[a], mx);
      const float corr = expf(m[a] - mn);  // exp(-inf) = 0 on the first block
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float p = expf(s[a][j] - mn);
        sum += p;
        Ps[(rg * 4 + a) * ATT_PSTR + cg + 8 * j] = p;
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      sum += __shfl_xor_sync(0xffffffffu, sum, 4);
      l[a] = l[a] * corr + sum;
      m[a] = mn;
#pragma unroll
      for (int i = 0; i < C::G * 4; ++i) o[a][i] *= corr;
    }
    __syncthreads();
    const int nk4 = (nk + 3) & ~3;  // P is exactly 0 for keys >= nk
    for (int j = 0; j < nk4; j += 4) {
      float4 pv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
        pv[a] = *reinterpret_cast<const float4*>(Ps + (rg * 4 + a) * ATT_PSTR + j);
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
#pragma unroll
        for (int g = 0; g < C::G; ++g) {
          const int c = 32 * g + 4 * cg;
          if (c < C::DHMAX) {
            const float4 vv = *reinterpret_cast<const float4*>(Vs + (j + jj) * C::STR + c);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const float p = jj == 0 ? pv[a].x : jj == 1 ? pv[a].y : jj == 2 ? pv[a].z : pv[a].w;
              o[a][4 * g + 0] = fmaf(p, vv.x, o[a][4 * g + 0]);
              o[a][4 * g + 1] = fmaf(p, vv.y, o[a][4 * g + 1]);
              o[a][4 * g + 2] = fmaf(p, vv.z, o[a][4 * g + 2]);
              o[a][4 * g + 3] = fmaf(p, vv.w, o[a][4 * g + 3]);
            }
          }
        }
      }
    }
  }

#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = rg * 4 + a;
    if (r >= nq) continue;
    const float inv = 1.0f / l[a];
    const size_t ob = (size_t)(start + q0 + r) * ldc + h * dh;
#pragma unroll
    for (int g = 0; g < C::G; ++g)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = 32 * g + 4 * cg + e;
        if (c < dh) store_split(ch, cl, ob + c, o[a][4 * g + e] * inv, fmt, ovf);
      }
  }
}

// ------------------------------------------------------------------ BOS-query attention
// Last layer: pooling reads only row 0 of each sequence (`encoder.py:181-185`), so
// only the BOS query of every (sequence, head) is needed. One warp per (s, h):
// scores over all keys of the sequence in fp32 from the hi(+lo) pieces, the
// reference's max / exp / sum (`masked_softmax`, `encoder.py:60-66`), ctx = Σ p v / sum.
// q: compact [S][ldqb] (this sequence's Q row), K|V: packed Q|K|V rows of qa.
// 16-bit pieces -> fp32 for 8 consecutive values (one 16-byte load per plane)
__device__ __forceinline__ void load8(const uint16_t* __restrict__ hi, const uint16_t* __restrict__ lo,
                                      size_t o, int fmt, float (&v)[8]) {
  const uint4 h = *reinterpret_cast<const uint4*>(hi + o);
  const uint16_t* hp = reinterpret_cast<const uint16_t*>(&h);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = load16(hp, i, fmt);
  if (lo) {
    const uint4 l = *reinterpret_cast<const uint4*>(lo + o);
    const uint16_t* lp = reinterpret_cast<const uint16_t*>(&l);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += load16(lp, i, fmt);
  }
}

// 4 warps per CTA, warp w -> head 4*blockIdx.y + w of sequence blockIdx.x.
// Requires dh % 8 == 0 and 16-byte aligned rows (true for the padded layouts).
__global__ void __launch_bounds__(128)
    bos_attention_kernel(const uint16_t* __restrict__ qbh, const uint16_t* __restrict__ qbl,
                         int ldqb, const uint16_t* __restrict__ kvh,
                         const uint16_t* __restrict__ kvl, int ldkv, int d, int dh, int heads,
                         float scale, const int32_t* __restrict__ cu, uint16_t* __restrict__ ch,
                         uint16_t* __restrict__ cl, int ldc, int fmt) {
  __shared__ float qs[4][128];
  __shared__ float ps[4][512];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x, h = blockIdx.y * 4 + w;
  if (h >= heads) return;
  const int start = cu[s], L = cu[s + 1] - start;
  for (int c = lane; c < dh; c += 32) {
    const size_t o = (size_t)s * ldqb + h * dh + c;
    qs[w][c] = load16(qbh, o, fmt) + (qbl ? load16(qbl, o, fmt) : 0.f);
  }
  __syncwarp();
  float mx = -INFINITY;
  for (int j = lane; j < L; j += 32) {
    const size_t ko = (size_t)(start + j) * ldkv + d + h * dh;
    float acc = 0.f;
    for (int c = 0; c < dh; c += 8) {
      float k[8];
      load8(kvh, kvl, ko + c, fmt, k);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fmaf(qs[w][c + i], k[i], acc);
    }
    ps[w][j] = acc * scale;
    mx = fmaxf(mx, acc * scale);
  }
  mx = warp_max(mx);
  __syncwarp();
  float sum = 0.f;
  for (int j = lane; j < L; j += 32) {
    const float p = expf(ps[w][j] - mx);
    ps[w][j] = p;
    sum += p;
  }
  sum = warp_sum(sum);
  __syncwarp();
  const float inv = 1.0f / sum;
  for (int c = lane; c < dh; c += 32) {
    // 4 keys per step with independent partial sums: the V loads of a step are
    // in flight together (one dependent chain per warp was latency-bound)
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const size_t vo = (size_t)start * ldkv + 2 * d + h * dh + c;
    int j = 0;
    for (; j + 4 <= L; j += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t o = vo + (size_t)(j + u) * ldkv;
        acc[u] = fmaf(ps[w][j + u], load16(kvh, o, fmt) + (kvl ? load16(kvl, o, fmt) : 0.f), acc[u]);
      }
    }
    for (; j < L; ++j) {
      const size_t o = vo + (size_t)j * ldkv;
      acc[0] = fmaf(ps[w][j], load16(kvh, o, fmt) + (kvl ? load16(kvl, o, fmt) : 0.f), acc[0]);
    }
    const float total = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    store_split(ch, cl, (size_t)s * ldc + h * dh + c, total * inv, fmt, nullptr);
  }
}

// ------------------------------------------------------------------ features
// BOS pooling (`encoder.py:181-185`) + per-kind feature vector (`:198-212`),
// written as the bf16 hi/lo A-operand of the first head GEMM.
// kind: 0 = comet-qe [t,s,t*s,|t-s|], 1 = comet [t,r,t*s,t*r,|t-s|,|t-r|], 2 = bleurt [j]
__global__ void features_kernel(const float* __restrict__ x, int ld, int d, int kind,
                                const int32_t* __restrict__ cu, int n,
                                uint16_t* __restrict__ fh, uint16_t* __restrict__ fl, int ldf,
                                int fmt, int* ovf) {
  const int r = blockIdx.x;
  const size_t ro = (size_t)r * ldf;
  // cu == nullptr: x holds one (BOS) row per sequence, sequence-indexed
  auto row = [&](int s) { return (size_t)(cu ? cu[s] : s) * ld; };
  const float* p0 = x + row(r);
  const float* p1 = kind != 2 ? x + row(n + r) : nullptr;
  const float* p2 = kind == 1 ? x + row(2 * n + r) : nullptr;
  auto put = [&](int c, float v) { store_split(fh, fl, ro + c, v, fmt, ovf); };
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    if (kind == 0) {
      const float s = p0[c], t = p1[c];
      put(c, t);
      put(d + c, s);
      put(2 * d + c, t * s);
      put(3 * d + c, fabsf(t - s));
    } else if (kind == 1) {
      const float s = p0[c], t = p1[c], rr = p2[c];
      put(c, t);
      put(d + c, rr);
      put(2 * d + c, t * s);
      put(3 * d + c, t * rr);
      put(4 * d + c, fabsf(t - s));
      put(5 * d + c, fabsf(t - rr));
    } else {
      put(c, p0[c]);
    }
  }
}

// ------------------------------------------------------------------ weight prep
// W[K][N] fp32 (row-vector x matrix, `pkg/README.md:137-140`) -> Wᵀ as bf16 hi
// (and lo) [Npad][Kpad], placed at row offset `row0` of the destination, zero
// padding untouched (destination is zero-initialised).
__global__ void transpose_split_kernel(const float* __restrict__ w, int K, int N,
                                       uint16_t* __restrict__ hi, uint16_t* __restrict__ lo,
                                       int ldk, int row0, int fmt, int* ovf,
                                       const float* __restrict__ alpha) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  const float s = alpha && n0 + threadIdx.x < N ? __frcp_rn(alpha[n0 + threadIdx.x]) : 1.f;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && n < N) ? w[(size_t)k * N + n] * s : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K)
      store_split(hi, lo, (size_t)(row0 + n) * ldk + k, tile[threadIdx.x][i], fmt, ovf);
  }
}

// Column maxima of |w| as float bits (non-negative floats order like their bits),
// accumulated with atomicMax into alpha_bits[N] (zeroed by the caller).
__global__ void colmax_kernel(const float* __restrict__ w, int K, int N,
                              unsigned* __restrict__ alpha_bits) {
  __shared__ unsigned part[8][32];
  const int n = blockIdx.x * 32 + threadIdx.x;
  unsigned m = 0;
  if (n < N)
    for (int k = blockIdx.y * 256 + threadIdx.y; k < min(K, (int)blockIdx.y * 256 + 256); k += 8)
      m = max(m, __float_as_uint(w[(size_t)k * N + n]) & 0x7fffffffu);
  part[threadIdx.y][threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    for (int i = 1; i < 8; ++i) m = max(m, part[i][threadIdx.x]);
    atomicMax(alpha_bits + n, m);
  }
}

// max bits -> alpha = 2^(e - 14) (see launch_weight_scales)
__global__ void colscale_kernel(float* __restrict__ alpha, int N) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const unsigned bits = __float_as_uint(alpha[n]);
  float a = 1.f;
  if (bits != 0 && bits < 0x7f800000u) {
    const int e = max(-100, (int)(bits >> 23) - 127);  // floor(log2 max); subnormals clamp
    a = __uint_as_float((unsigned)(e - 14 + 127) << 23);
  }
  alpha[n] = a;
}

// BOS rows -> compact sequence-indexed rows (the last layer only feeds pooling,
// `encoder.py:181-185`): dst row s = src row cu[s], for 16-bit planes and/or fp32.
__global__ void gather_bos_kernel(const int32_t* __restrict__ cu, int d,
                                  const uint16_t* __restrict__ sh, const uint16_t* __restrict__ sl,
                                  int lds, const float* __restrict__ s32, int ld32,
                                  uint16_t* __restrict__ dh, uint16_t* __restrict__ dl, int ldd,
                                  float* __restrict__ d32, int ldd32) {
  const int s = blockIdx.x;
  const size_t src = (size_t)cu[s];
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    if (sh) dh[(size_t)s * ldd + c] = sh[src * lds + c];
    if (sl) dl[(size_t)s * ldd + c] = sl[src * lds + c];
    if (s32) d32[(size_t)s * ldd32 + c] = s32[src * ld32 + c];
  }
}

// scores[i] = out[i * ld]  (column 0 of the final head stage, `encoder.py:196`)
__global__ void gather_col0_kernel(const float* __restrict__ out, int ld, int n,
                                   float* __restrict__ scores) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) scores[i] = out[(size_t)i * ld];
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_embed(const int32_t* ids, const int32_t* cu, int nseq, int V, int d,
                         const float* tok, const float* pe, float* x32, int ld, uint16_t* xh,
                         uint16_t* xl, int fmt, int r16, int* flag, cudaStream_t st) {
  if (nseq <= 0) return cudaSuccess;
  embed_kernel<<<nseq, 256, 0, st>>>(ids, cu, V, d, tok, pe, x32, ld, xh, xl, fmt, r16, flag);
  return cudaGetLastError();
}

template <int V4, bool IN16>
static cudaError_t ln_launch(const void* y, int T, int d, int ld, const float* g, const float* b,
                             float* out32, uint16_t* oh, uint16_t* ol, int fmt, int r16, int* ovf,
                             int rows_blocks, cudaStream_t st) {
  // 4 rows (warps) per CTA: small CTAs retire as soon as their rows are done
  if (r16)
    layernorm_kernel<V4, IN16, true><<<(T + 3) / 4, 128, 0, st>>>(y, T, d, ld, g, b, out32, oh, ol,
                                                                  fmt, ovf);
  else
    layernorm_kernel<V4, IN16, false><<<(T + 3) / 4, 128, 0, st>>>(y, T, d, ld, g, b, out32, oh,
                                                                   ol, fmt, ovf);
  return cudaGetLastError();
}

cudaError_t launch_layernorm(const void* y, int in16, int T, int d, int ld, const float* g,
                             const float* b, float* out32, uint16_t* oh, uint16_t* ol, int fmt,
                             int r16, int* ovf, cudaStream_t st) {
  if (T <= 0) return cudaSuccess;
  const int rows_blocks = (T + 7) / 8;
  dim3 block(256);
  const bool vec = d % 4 == 0 && ld % 4 == 0 && ((uintptr_t)y & 15) == 0 &&
                   ((uintptr_t)g & 15) == 0 && ((uintptr_t)b & 15) == 0;
  const int v4 = (d / 4 + 31) / 32;
  if (vec) {
#define LN_CASE(V)                                                                   \
    if (v4 <= V) {                                                                   \
      if (in16)                                                                      \
        return ln_launch<V, true>(y, T, d, ld, g, b, out32, oh, ol, fmt, r16, ovf,       \
                                  rows_blocks, st);                                  \
      return ln_launch<V, false>(y, T, d, ld, g, b, out32, oh, ol, fmt, r16, ovf,        \
                                 rows_blocks, st);                                   \
    }
    LN_CASE(1) LN_CASE(2) LN_CASE(4) LN_CASE(8) LN_CASE(9) LN_CASE(10) LN_CASE(12) LN_CASE(16)
    LN_CASE(20) LN_CASE(24) LN_CASE(32)
#undef LN_CASE
  }
  layernorm_scalar_kernel<<<rows_blocks, block, 0, st>>>(y, in16, T, d, ld, g, b, out32, oh, ol,
                                                         fmt, r16, ovf);
  return cudaGetLastError();
}

template <int DHC>
static cudaError_t att_launch(const uint16_t* qh, const uint16_t* ql, int ldq, int d, int dh,
                              float scale,
                              const int32_t* cu, const int2* work, int n_work, int heads,
                              uint16_t* ch, uint16_t* cl, int ldc, int fmt, int* ovf,
                              cudaStream_t st) {
  const size_t smem = AttCfg<DHC>::SMEM;
  cudaFuncSetAttribute(attention_kernel<DHC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  attention_kernel<DHC><<<dim3(n_work, heads), ATT_THREADS, smem, st>>>(qh, ql, ldq, d, dh, scale,
                                                                         cu, work, ch, cl, ldc,
                                                                         fmt, ovf);
  return cudaGetLastError();
}

cudaError_t launch_attention(const uint16_t* qh, const uint16_t* ql, int ldq, int d, int heads,
                             const int32_t* cu,
                             const int2* work, int n_work, uint16_t* ch, uint16_t* cl,
                             int ldc, int fmt, int* ovf, cudaStream_t st) {
  if (n_work <= 0) return cudaSuccess;
  const int dh = d / heads;
  const float scale = 1.0f / sqrtf((float)d / (float)heads);
  const int dhc = (dh + 7) / 8;
#define ATT_CASE(V) \
  if (dhc <= V) return att_launch<V>(qh, ql, ldq, d, dh, scale, cu, work, n_work, heads, ch, cl, ldc, fmt, ovf, st);
  ATT_CASE(1) ATT_CASE(2) ATT_CASE(4) ATT_CASE(8) ATT_CASE(10) ATT_CASE(12) ATT_CASE(16)
#undef ATT_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_bos_attention(const uint16_t* qbh, const uint16_t* qbl, int ldqb,
                                 const uint16_t* kvh, const uint16_t* kvl, int ldkv, int d,
                                 int heads, const int32_t* cu, int nseq, uint16_t* ch, uint16_t* cl,
                                 int ldc, int fmt, cudaStream_t st) {
  if (nseq <= 0) return cudaSuccess;
  const int dh = d / heads;
  if (dh > 128) return cudaErrorInvalidValue;
  const float scale = 1.0f / sqrtf((float)d / (float)heads);
  if (dh % 8) return cudaErrorInvalidValue;
  bos_attention_kernel<<<dim3(nseq, (heads + 3) / 4), 128, 0, st>>>(
      qbh, qbl, ldqb, kvh, kvl, ldkv, d, dh, heads, scale, cu, ch, cl, ldc, fmt);
  return cudaGetLastError();
}

cudaError_t launch_features(const float* x, int ld, int d, int kind, const int32_t* cu, int n,
                            uint16_t* fh, uint16_t* fl, int ldf, int fmt, int* ovf,
                            cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  features_kernel<<<n, 256, 0, st>>>(x, ld, d, kind, cu, n, fh, fl, ldf, fmt, ovf);
  return cudaGetLastError();
}

cudaError_t launch_transpose_split(const float* w, int K, int N, uint16_t* hi, uint16_t* lo,
                                   int ldk, int row0, int fmt, int* ovf, cudaStream_t st,
                                   const float* alpha) {
  dim3 grid((N + 31) / 32, (K + 31) / 32), block(32, 8);
  transpose_split_kernel<<<grid, block, 0, st>>>(w, K, N, hi, lo, ldk, row0, fmt, ovf, alpha);
  return cudaGetLastError();
}

cudaError_t launch_weight_scales(const float* w, int K, int N, float* alpha, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(alpha, 0, (size_t)N * sizeof(float), st);
  if (e != cudaSuccess) return e;
  dim3 grid((N + 31) / 32, (K + 255) / 256), block(32, 8);
  colmax_kernel<<<grid, block, 0, st>>>(w, K, N, reinterpret_cast<unsigned*>(alpha));
  colscale_kernel<<<(N + 255) / 256, 256, 0, st>>>(alpha, N);
  return cudaGetLastError();
}

cudaError_t launch_gather_bos(const int32_t* cu, int nseq, int d, const uint16_t* sh,
                              const uint16_t* sl, int lds, const float* s32, int ld32, uint16_t* dh,
                              uint16_t* dl, int ldd, float* d32, int ldd32, cudaStream_t st) {
  if (nseq <= 0) return cudaSuccess;
  gather_bos_kernel<<<nseq, 256, 0, st>>>(cu, d, sh, sl, lds, s32, ld32, dh, dl, ldd, d32, ldd32);
  return cudaGetLastError();
}

cudaError_t launch_gather_col0(const float* out, int ld, int n, float* scores, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  gather_col0_kernel<<<(n + 255) / 256, 256, 0, st>>>(out, ld, n, scores);
  return cudaGetLastError();
}

}  // namespace mfg
