// libmfgpu: scoring context and C-ABI (include/mfgpu.h).
//
// Replaces `ScoringModel` (`pkg/src/metricforge/encoder.py:94-226`): weights are
// uploaded once, matrices transposed to K-major and split into bf16 hi/lo pairs
// (fp32-parity) or rounded to bf16 (bf16 mode); a batch of records is scored as
// one token-packed stream per device chunk.
#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mfgpu.h"
#include "../../include/mfgpu_test.h"
#include "container.hpp"
#include "gemm_tc.cuh"
#include "kernels.h"

using namespace mfg;

namespace {

thread_local int g_code = 0;
thread_local std::string g_msg;

struct Fail {
  int code;
  std::string msg;
};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t _e = (x);                                                                  \
    if (_e != cudaSuccess)                                                                 \
      throw Fail{MFG_ERR_RUNTIME, std::string("CUDA error: ") + cudaGetErrorString(_e) +   \
                                      " at " #x};                                          \
  } while (0)

inline int pad64(int64_t x) { return (int)((x + 63) / 64 * 64); }
inline int64_t pad128(int64_t x) { return (x + 127) / 128 * 128; }
// Widths of 1024+ that are not multiples of 256 (RemBERT's d = 1152, 3d = 3456)
// are padded to 256 so their GEMMs run on the CTA-pair kernel (BN = 256, ~97-99 %
// tensor pipe) instead of the single-CTA BN = 128 one (~80 %); the padded weight
// rows and biases are zero, so the padded output columns are 0 and never read.
inline int padN(int64_t x) {
  const int p = pad64(x);
  return (p >= 1024 && p % 256) ? (int)((x + 255) / 256 * 256) : p;
}

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
};

// A GEMM weight: Wᵀ as bf16 hi (+lo) [Npad][Kpad], bias [Npad], tensor maps.
struct Weight {
  uint16_t *hi = nullptr, *lo = nullptr;
  float* bias = nullptr;
  float* alpha = nullptr;  // fp32-parity path: per-column 2^-e undoing the weight prescale
  int N = 0, K = 0, Npad = 0, Kpad = 0, bn = 64;
  CUtensorMap mh{}, ml{};
};

// A GEMM A-operand activation buffer [rows][ld] bf16 hi (+lo).
struct Act {
  uint16_t *hi = nullptr, *lo = nullptr;
  int64_t rows = 0;
  int ld = 0;
  CUtensorMap mh{}, ml{};
};

struct Layer {
  Weight qkv, o, w1, w2;
  Weight q_part, kv_part;  // views of qkv: rows [0,d) and [d,3d) (last layer only)
  float *g1 = nullptr, *b1 = nullptr, *g2 = nullptr, *b2 = nullptr;
};

enum Cls { C_QKV = 0, C_O, C_FFN1, C_FFN2, C_ATT, C_LN, C_EMB, C_HEAD };

// Host -> device weight upload (`container.py:363-412` mmap views -> HBM): the
// mmap'd (page-cache) bytes are copied by several host threads into one of two
// pinned chunks while the other chunk's async H2D copy (and the device-side
// transpose/split of earlier matrices) runs, instead of a pageable cudaMemcpy
// per tensor.
struct Uploader {
  static constexpr size_t CHUNK = 32u << 20;  // bytes per pinned chunk
  cudaStream_t st = nullptr;
  void* pinned[2] = {nullptr, nullptr};
  cudaEvent_t free_ev[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
  int cur = 0;
  unsigned nthreads = 4;

  void init(cudaStream_t s) {
    st = s;
    for (int i = 0; i < 2; ++i) {
      CK(cudaMallocHost(&pinned[i], CHUNK));
      CK(cudaEventCreateWithFlags(&free_ev[i], cudaEventDisableTiming));
    }
    const unsigned hc = std::thread::hardware_concurrency();
    nthreads = std::max(1u, std::min(8u, hc ? hc / 2 : 4u));
  }
  void release() {
    for (int i = 0; i < 2; ++i) {
      if (free_ev[i]) cudaEventSynchronize(free_ev[i]), cudaEventDestroy(free_ev[i]);
      if (pinned[i]) cudaFreeHost(pinned[i]);
      pinned[i] = nullptr;
      free_ev[i] = nullptr;
    }
  }
  ~Uploader() { release(); }
  void par_copy(void* dst, const void* src, size_t n) {
    if (n < (2u << 20) || nthreads <= 1) {
      memcpy(dst, src, n);
      return;
    }
    std::vector<std::thread> th;
    const size_t part = (n + nthreads - 1) / nthreads;
    for (unsigned i = 0; i < nthreads; ++i) {
      const size_t a = i * part, b = std::min(n, a + part);
      if (a >= b) break;
      th.emplace_back([=] { memcpy((char*)dst + a, (const char*)src + a, b - a); });
    }
    for (auto& t : th) t.join();
  }
  // async: dst (device) <- src (host) bytes; src may be reused as soon as this returns
  void upload(void* dst, const void* src, size_t n) {
    for (size_t off = 0; off < n; off += CHUNK) {
      const size_t k = std::min(CHUNK, n - off);
      if (used[cur]) CK(cudaEventSynchronize(free_ev[cur]));
      par_copy(pinned[cur], (const char*)src + off, k);
      CK(cudaMemcpyAsync((char*)dst + off, pinned[cur], k, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(free_ev[cur], st));
      used[cur] = true;
      cur ^= 1;
    }
  }
};

}  // namespace

// Kind and tensor-name/shape contract of an opened container (`encoder.py:107-115`).
static void check_contract(const Container& c) {
  const Manifest& man = c.manifest();
  if (man.like != "comet-qe" && man.like != "comet" && man.like != "bleurt")
    throw Fail{MFG_ERR_CONTAINER, "unknown metric kind '" + man.like + "'"};
  if (man.d_model <= 0 || man.n_heads <= 0 || man.d_model % man.n_heads != 0)
    throw Fail{MFG_ERR_CONTAINER, "d_model not divisible by n_heads"};
  for (auto& kv : required_shapes(man)) {
    const TensorView* t = c.find(kv.first);
    if (!t) throw Fail{MFG_ERR_CONTAINER, c.path() + ": missing tensor '" + kv.first + "'"};
    if (t->shape != kv.second)
      throw Fail{MFG_ERR_CONTAINER, c.path() + ": tensor '" + kv.first + "' has shape " +
                                        shape_repr(t->shape) + ", manifest implies " +
                                        shape_repr(kv.second)};
  }
}

struct mfg_ctx {
  int device = 0, precision = MFG_PREC_FP32, num_sms = 148;
  bool split = true, pre_norm = false, profile = false;
  bool res_bf16 = false;   // bf16 mode: residual stream as bf16 hi/lo pieces (post-norm)
  bool r16 = false;        // reference binary16 mode: every tensor and activation is fp16
  bool prescale = true;
  // load phases (ms): context, open (mmap + header + shape contract), embeddings,
  // layer weights (H2D + transpose/split), head weights, workspaces
  double load_ms[6] = {0, 0, 0, 0, 0, 0};    // fp32-parity path: power-of-two weight column prescale
                           // (MFG_WEIGHT_PRESCALE=0 disables it: accuracy A/B only)
  int fmt = FMT_F16;       // 16-bit operand format of every GEMM operand
  int* d_ovf = nullptr;    // fp16 range overflow flag (set by any producer)
  int* h_ovf = nullptr;
  Manifest man;
  int kind = 0, n_roles = 0;
  int d = 0, dp = 0, f = 0, fp = 0, H = 0, F = 0, Fp = 0, qkv_ld = 0;
  cudaStream_t st = nullptr;       // stream every launch goes to
  cudaStream_t own_st = nullptr;   // the one the context created
  std::vector<void*> allocs;
  int64_t device_bytes = 0;

  float *tok = nullptr, *pos = nullptr;
  std::vector<Layer> layers;
  std::vector<Weight> head;

  int64_t cap_tokens = 0;
  int cap_records = 0;
  float *x32 = nullptr, *y32 = nullptr;
  float* gemm_part = nullptr;  // K-chunk running sums of the CTA-pair GEMM (GemmArgs::partial)
  bool part_persist = false;   // gemm_part pinned in L2 (persisting window on the launch stream)
  int* tile_ctr = nullptr;     // CTA-pair GEMM tile counter + finished-pair count (self-resetting)
  bool dyn_tiles = !(getenv("MFG_TILE_DYN") && getenv("MFG_TILE_DYN")[0] == '0');  // A/B switch

  // split-operand (fp32-parity / bf16x3) GEMMs of models narrower than 1024 restart
  // the accumulator every 512 K (gemm_kchunk_blocks)
  bool fine_kchunk() const { return split && d < 1024; }

  void apply_l2_window(cudaStream_t s) {
    if (!part_persist || !s) return;
    int max_win = 0;
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, device);
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = gemm_part;
    v.accessPolicyWindow.num_bytes =
        std::min(gemm_partial_floats(num_sms) * sizeof(float), (size_t)std::max(0, max_win));
    v.accessPolicyWindow.hitRatio = 1.0f;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess)
      cudaGetLastError();  // best effort: only the DRAM traffic changes, never the results
  }
  Act xa, ca, ha, fa, qa;          // qa: Q|K|V pieces [T][qkv_ld]
  // last layer on BOS rows only (one row per sequence): ctx, residual/LN, FFN hidden, Q
  Act cb, xb, hb, qb;
  bool bos_qkv = false;  // last layer: K|V for all rows, Q + attention for BOS rows only
  float *x32b = nullptr, *y32b = nullptr;
  bool att_tc = false;              // tcgen05 attention usable (d_head == 64)
  AttTile *d_tiles = nullptr, *h_tiles = nullptr;  // attention tiles (att_plan_tiles)
  CUtensorMap qm32h{}, qm32l{};     // Q|K|V maps with 32-row boxes (attention tiles)
  CUtensorMap qt32h{}, qt32l{};     // ... 16-column tail boxes (d_head 80)
  std::vector<AttTile> v_tiles;
  std::vector<int2> v_work;
  std::vector<Act> ga;  // head hidden-stage outputs
  float* hout = nullptr;
  float* dscores = nullptr;
  int32_t *d_ids = nullptr, *d_cu = nullptr;
  int2* d_work = nullptr;
  int32_t *h_ids = nullptr, *h_cu = nullptr;
  int2* h_work = nullptr;
  float* h_scores = nullptr;
  int64_t work_cap = 0;

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  Uploader* up = nullptr;  // weight upload pipeline (build() only)
  size_t staging_half = 0;
  int stage_flip = 0;
  std::vector<cudaEvent_t> pev;  // profile event pool
  struct Rec {
    int cls;
    int e0, e1;
  };
  std::vector<Rec> recs;
  int pev_used = 0;
  mfg_stats stats{};

  int err_code = 0;
  std::string err_msg;

  template <class T>
  T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, count * sizeof(T)));
    allocs.push_back(p);
    device_bytes += (int64_t)(count * sizeof(T));
    CK(cudaMemsetAsync(p, 0, count * sizeof(T), st));
    return (T*)p;
  }

  // ---------------------------------------------------------------- profiling
  int ev_begin() {
    if (!profile) return -1;
    if (pev_used + 2 > (int)pev.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        pev.push_back(e);
      }
    }
    int i = pev_used;
    pev_used += 2;
    CK(cudaEventRecord(pev[i], st));
    return i;
  }
  void ev_end(int i, int cls, double flops, double bytes) {
    stats.kernel_launches += 1;
    stats.class_launches[cls] += 1;
    stats.class_flops[cls] += flops;
    stats.class_bytes[cls] += bytes;
    if (i < 0) return;
    CK(cudaEventRecord(pev[i + 1], st));
    recs.push_back({cls, i, i + 1});
  }
  void collect_profile() {
    for (auto& r : recs) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, pev[r.e0], pev[r.e1]));
      stats.class_ms[r.cls] += ms;
    }
    recs.clear();
    pev_used = 0;
  }

  // ---------------------------------------------------------------- setup
  void make_act(Act& a, int64_t rows, int cols_pad, bool with_lo) {
    char err[256];
    a.rows = pad128(rows);
    a.ld = cols_pad;
    a.hi = dalloc<uint16_t>((size_t)a.rows * a.ld);
    if (!make_tmap_u16(&a.mh, a.hi, a.rows, a.ld, a.ld, GEMM_BM, err, sizeof err))
      throw Fail{MFG_ERR_RUNTIME, err};
    if (with_lo) {
      a.lo = dalloc<uint16_t>((size_t)a.rows * a.ld);
      if (!make_tmap_u16(&a.ml, a.lo, a.rows, a.ld, a.ld, GEMM_BM, err, sizeof err))
        throw Fail{MFG_ERR_RUNTIME, err};
    }
  }

  // Upload one or more fp32 [K][N_i] matrices side by side along N as a single Wᵀ.
  void make_weight(Weight& w, const std::vector<const TensorView*>& mats,
                   const std::vector<const TensorView*>& biases, float* staging_dev,
                   std::vector<float>& host_tmp) {
    char err[256];
    w.K = (int)mats[0]->shape[0];
    w.N = 0;
    for (auto* m : mats) w.N += (int)m->shape[1];
    w.Kpad = pad64(w.K);
    w.Npad = padN(w.N);
    w.bn = gemm_pick_bn(w.Npad);
    w.hi = dalloc<uint16_t>((size_t)w.Npad * w.Kpad);
    if (split) w.lo = dalloc<uint16_t>((size_t)w.Npad * w.Kpad);
    // fp16 hi/lo pieces: every weight column is pre-scaled by a power of two so its
    // largest element sits in [2^14, 2^15): any finite weight fits the fp16 range and
    // the lo piece keeps 11 bits for elements down to 2^-15 of the column max (the
    // epilogue multiplies the accumulator back by alpha, exactly)
    if (split && fmt == FMT_F16 && prescale) w.alpha = dalloc<float>(w.Npad);
    int row0 = 0;
    for (auto* m : mats) {
      const float* src = host_f32(*m, host_tmp);
      // two device staging halves alternate so the next matrix's H2D overlaps this transpose
      float* stg = staging_dev + (stage_flip ^= 1) * staging_half;
      up->upload(stg, src, m->numel() * 4);
      if (w.alpha)
        CK(launch_weight_scales(stg, (int)m->shape[0], (int)m->shape[1], w.alpha + row0, st));
      CK(launch_transpose_split(stg, (int)m->shape[0], (int)m->shape[1], w.hi, w.lo,
                                w.Kpad, row0, fmt, d_ovf, st, w.alpha ? w.alpha + row0 : nullptr));
      row0 += (int)m->shape[1];
    }
    w.bias = dalloc<float>(w.Npad);
    int off = 0;
    for (auto* b : biases) {
      const float* src = host_vec(*b, host_tmp);
      up->upload(w.bias + off, src, b->numel() * 4);
      off += (int)b->numel();
    }
    if (!make_tmap_u16(&w.mh, w.hi, w.Npad, w.Kpad, w.Kpad, gemm_b_box_rows(w.bn), err, sizeof err))
      throw Fail{MFG_ERR_RUNTIME, err};
    if (split && !make_tmap_u16(&w.ml, w.lo, w.Npad, w.Kpad, w.Kpad, gemm_b_box_rows(w.bn), err,
                                sizeof err))
      throw Fail{MFG_ERR_RUNTIME, err};
  }

  static const float* host_f32(const TensorView& t, std::vector<float>& tmp) {
    if (t.dtype == "f32") return reinterpret_cast<const float*>(t.data);
    // binary16 -> fp32 (exact), as `tensor.astype(float32)` in the reference
    tmp.resize(t.numel());
    const uint16_t* h = reinterpret_cast<const uint16_t*>(t.data);
    for (int64_t i = 0; i < t.numel(); ++i) {
      uint32_t s = (h[i] & 0x8000u) << 16, e = (h[i] >> 10) & 0x1F, m = h[i] & 0x3FF, bits;
      if (e == 0) {
        if (m == 0) bits = s;
        else {
          e = 127 - 15 + 1;
          while (!(m & 0x400)) { m <<= 1; --e; }
          bits = s | (e << 23) | ((m & 0x3FF) << 13);
        }
      } else if (e == 31) bits = s | 0x7F800000u | (m << 13);
      else bits = s | ((e + 127 - 15) << 23) | (m << 13);
      memcpy(&tmp[i], &bits, 4);
    }
    return tmp.data();
  }

  // fp32 view of a vector/table; in binary16 mode rounded like `tensor.astype(float16)`
  // (`encoder.py:102-118`) — GEMM weights get the same rounding from transpose_split.
  const float* host_vec(const TensorView& t, std::vector<float>& tmp) const {
    const float* src = host_f32(t, tmp);
    if (!r16) return src;
    if (src != tmp.data()) tmp.assign(src, src + t.numel());
    for (auto& v : tmp) v = __half2float(__float2half_rn(v));
    return tmp.data();
  }
  float* upload_vec(const TensorView& t, size_t pad_to = 0) {
    std::vector<float> tmp;
    const float* src = host_vec(t, tmp);
    float* p = dalloc<float>(std::max<size_t>(pad_to, (size_t)t.numel()));
    up->upload(p, src, t.numel() * 4);
    return p;
  }

  void build(const mfg_config& cfg) {
    // MFG_LOAD_TRACE=1: phase timings of the weight upload on stderr
    // (always recorded per phase in load_ms, mfg_model_info)
    const bool trace = getenv("MFG_LOAD_TRACE") != nullptr;
    auto clk = [] { return std::chrono::steady_clock::now(); };
    auto t_start = clk();
    auto t_prev = t_start;
    auto lap = [&](const char* what, int phase = -1) {
      cudaStreamSynchronize(st);
      auto now = clk();
      if (phase >= 0) load_ms[phase] += std::chrono::duration<double, std::milli>(now - t_prev).count();
      t_prev = now;
      if (trace)
        fprintf(stderr, "mfg load: %-12s %8.1f ms\n", what,
                std::chrono::duration<double, std::milli>(now - t_start).count());
    };
    Container c(cfg.container_path);
    lap("open", 1);
    if (const char* e = getenv("MFG_WEIGHT_PRESCALE")) prescale = e[0] != '0';
    man = c.manifest();
    check_contract(c);
    kind = man.like == "comet-qe" ? 0 : man.like == "comet" ? 1 : 2;
    n_roles = kind == 0 ? 2 : kind == 1 ? 3 : 1;
    pre_norm = man.norm_style == "pre";
    d = (int)man.d_model;
    dp = padN(d);
    f = (int)man.d_ffn;
    fp = padN(f);
    H = (int)man.n_heads;
    F = feature_multiplier(man.like) * d;
    Fp = pad64(F);
    if (d / H > 128) throw Fail{MFG_ERR_CONTAINER, "head dimension > 128 is not supported"};

    // staging buffer for the largest matrix upload
    int64_t big = 0;
    for (auto& kv : required_shapes(man))
      if (kv.second.size() == 2 && kv.first.rfind("emb.", 0) != 0) {
        int64_t n = kv.second[0] * kv.second[1];
        big = std::max(big, n);
      }
    float* staging = nullptr;
    staging_half = (size_t)std::max<int64_t>(big, 1);
    CK(cudaMalloc(&staging, staging_half * 2 * 4));
    Uploader uploader;
    uploader.init(st);
    up = &uploader;
    std::vector<float> tmp;
    d_ovf = dalloc<int>(1);
    CK(cudaMallocHost(&h_ovf, sizeof(int)));
    try {
      lap("setup", 1);
      tok = upload_vec(*c.find("emb.tok"));
      lap("emb.tok", 2);
      pos = upload_vec(*c.find("emb.pos"));
      layers.resize(man.n_layers);
      for (int i = 0; i < man.n_layers; ++i) {
        std::string p = "layer." + std::to_string(i);
        Layer& L = layers[i];
        auto T = [&](const std::string& n) { return c.find(p + n); };
        make_weight(L.qkv, {T(".att.q.w"), T(".att.k.w"), T(".att.v.w")},
                    {T(".att.q.b"), T(".att.k.b"), T(".att.v.b")}, staging, tmp);
        make_weight(L.o, {T(".att.o.w")}, {T(".att.o.b")}, staging, tmp);
        make_weight(L.w1, {T(".ffn.w1")}, {T(".ffn.b1")}, staging, tmp);
        make_weight(L.w2, {T(".ffn.w2")}, {T(".ffn.b2")}, staging, tmp);
        L.g1 = upload_vec(*T(".norm1.g"));
        L.b1 = upload_vec(*T(".norm1.b"));
        L.g2 = upload_vec(*T(".norm2.g"));
        L.b2 = upload_vec(*T(".norm2.b"));
      }
      lap("layers", 3);
      // last layer's Q / K|V views of the fused QKV weight (needs d % 64 == 0 so the
      // split falls on a padded-row boundary, and tile-aligned N for both parts)
      if (!layers.empty() && d % 64 == 0) {
        Weight& w = layers.back().qkv;
        const int bq = gemm_pick_bn(d), bkv = gemm_pick_bn(2 * d);
        bos_qkv = w.N == 3 * d && (d / H) % 8 == 0;
        auto view = [&](Weight& v, int row0, int n, int bn) {
          char err[256];
          v = Weight{};
          v.hi = w.hi + (size_t)row0 * w.Kpad;
          v.lo = w.lo ? w.lo + (size_t)row0 * w.Kpad : nullptr;
          v.bias = w.bias + row0;
          v.alpha = w.alpha ? w.alpha + row0 : nullptr;
          v.N = n;
          v.K = w.K;
          v.Npad = n;
          v.Kpad = w.Kpad;
          v.bn = bn;
          if (!make_tmap_u16(&v.mh, v.hi, n, v.Kpad, v.Kpad, gemm_b_box_rows(bn), err, sizeof err))
            throw Fail{MFG_ERR_RUNTIME, err};
          if (v.lo && !make_tmap_u16(&v.ml, v.lo, n, v.Kpad, v.Kpad, gemm_b_box_rows(bn), err,
                                     sizeof err))
            throw Fail{MFG_ERR_RUNTIME, err};
        };
        if (bos_qkv) {
          view(layers.back().q_part, 0, d, bq);
          view(layers.back().kv_part, d, 2 * d, bkv);
        }
      }
      const size_t stages = man.head_hidden.size() + 1;
      head.resize(stages);
      for (size_t j = 0; j < stages; ++j) {
        std::string p = "head." + std::to_string(j);
        make_weight(head[j], {c.find(p + ".w")}, {c.find(p + ".b")}, staging, tmp);
      }
    } catch (...) {
      cudaStreamSynchronize(st);
      up = nullptr;
      cudaFree(staging);
      throw;
    }
    CK(cudaStreamSynchronize(st));
    up = nullptr;
    CK(cudaFree(staging));
    CK(cudaMemcpy(h_ovf, d_ovf, sizeof(int), cudaMemcpyDeviceToHost));
    if (*h_ovf)
      throw Fail{MFG_ERR_USAGE, "a weight is not finite (inf or nan)"};
    qkv_ld = layers.empty() ? pad64(3 * d) : layers[0].qkv.Npad;

    lap("weights", 4);
    // workspaces
    cap_tokens = pad128(cfg.max_tokens > 0 ? cfg.max_tokens : 262144);
    cap_records = cfg.max_records > 0 ? cfg.max_records : 4096;
    x32 = dalloc<float>((size_t)cap_tokens * dp);
    gemm_part = dalloc<float>(gemm_partial_floats(num_sms));
    tile_ctr = dalloc<int>(2);
    // K-chunked GEMMs (K > 4096, or XL's 2560) round-trip their fp32 chunk sums
    // through gemm_part once per chunk and tile; under the activation and weight
    // streams those lines were evicted to DRAM between the drain and the next
    // read (ncu, config 5: ~60 GB of extra DRAM traffic per layer). Pin the
    // buffer in L2 as a persisting access-policy window on the launch stream.
    part_persist = (gemm_kchunk_blocks(dp, fine_kchunk()) > 0 ||
                    gemm_kchunk_blocks(fp, fine_kchunk()) > 0) &&
                   !(getenv("MFG_L2_PERSIST") && getenv("MFG_L2_PERSIST")[0] == '0');
    if (part_persist) {
      int max_persist = 0;
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
      const size_t want = gemm_partial_floats(num_sms) * sizeof(float);
      if (max_persist <= 0 ||
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min(want, (size_t)max_persist)) !=
              cudaSuccess) {
        part_persist = false;
        cudaGetLastError();
      } else {
        apply_l2_window(st);
      }
    }
    y32 = dalloc<float>((size_t)cap_tokens * dp);
    make_act(qa, cap_tokens, qkv_ld, split);
    {
      char err[256];
      if (!make_tmap_u16(&qm32h, qa.hi, qa.rows, qa.ld, qa.ld, 32, err, sizeof err))
        throw Fail{MFG_ERR_RUNTIME, err};
      if (split && !make_tmap_u16(&qm32l, qa.lo, qa.rows, qa.ld, qa.ld, 32, err, sizeof err))
        throw Fail{MFG_ERR_RUNTIME, err};
      if (!make_tmap_u16_box(&qt32h, qa.hi, qa.rows, qa.ld, qa.ld, 16, 32, 32, err, sizeof err))
        throw Fail{MFG_ERR_RUNTIME, err};
      if (split &&
          !make_tmap_u16_box(&qt32l, qa.lo, qa.rows, qa.ld, qa.ld, 16, 32, 32, err, sizeof err))
        throw Fail{MFG_ERR_RUNTIME, err};
    }
    att_tc = (d / H == 64 || d / H == 80) && (d % 64 == 0);
    // post-norm bf16 mode: the residual stream travels as bf16 hi/lo pieces of
    // the layer input (~16 significant bits instead of a separate fp32 copy)
    // (MFG_BF16_RES32=1 keeps the fp32 residual copy: accuracy A/B runs)
    const char* res32 = getenv("MFG_BF16_RES32");
    res_bf16 = !split && !r16 && !pre_norm && !(res32 && res32[0] == '1');
    make_act(xa, cap_tokens, dp, split || res_bf16);
    make_act(ca, cap_tokens, dp, split);
    make_act(ha, cap_tokens, fp, split);
    make_act(fa, cap_records, Fp, split);
    {
      const int64_t ns = (int64_t)cap_records * n_roles;
      make_act(cb, ns, dp, split);
      make_act(xb, ns, dp, split || res_bf16);
      make_act(hb, ns, fp, split);
      make_act(qb, ns, dp, split);
      x32b = dalloc<float>((size_t)pad128(ns) * dp);
      y32b = dalloc<float>((size_t)pad128(ns) * dp);
    }
    ga.resize(head.size() - 1);
    for (size_t j = 0; j + 1 < head.size(); ++j) make_act(ga[j], cap_records, head[j].Npad, split);
    hout = dalloc<float>((size_t)pad128(cap_records) * head.back().Npad);
    dscores = dalloc<float>(cap_records);
    d_ids = dalloc<int32_t>(cap_tokens);
    d_cu = dalloc<int32_t>((size_t)cap_records * n_roles + 1);
    d_tiles = dalloc<AttTile>((size_t)cap_records * n_roles);
    CK(cudaMallocHost(&h_tiles, (size_t)cap_records * n_roles * sizeof(AttTile)));
    work_cap = cap_tokens / 1 + (int64_t)cap_records * n_roles;
    d_work = dalloc<int2>(work_cap);
    CK(cudaMallocHost(&h_ids, cap_tokens * 4));
    CK(cudaMallocHost(&h_cu, ((size_t)cap_records * n_roles + 1) * 4));
    CK(cudaMallocHost(&h_work, work_cap * sizeof(int2)));
    CK(cudaMallocHost(&h_scores, cap_records * 4));
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
    lap("workspaces", 5);
  }

  // ---------------------------------------------------------------- forward
  void gemm(const Act& a, const Weight& w, int M, int epi, int cls, const float* res, int ldr,
            float* out32, int ldo, Act* outa, const Act* res16 = nullptr, int out_col = 0,
            bool as16 = false) {
    GemmArgs g{};
    g.M = M;
    g.N = w.Npad;
    g.K = w.Kpad;
    g.bias = w.bias;
    g.alpha = w.alpha;
    g.kchunk = gemm_kchunk_blocks(w.Kpad, fine_kchunk());
    g.partial = gemm_part;
    g.tile_ctr = dyn_tiles ? tile_ctr : nullptr;
    g.residual = res;
    g.ldr = ldr;
    if (res16) {
      g.res_hi = res16->hi;
      g.res_lo = res16->lo;
      g.ldr = res16->ld;
    }
    g.out_f32 = as16 ? nullptr : out32;
    g.out16 = as16 ? reinterpret_cast<uint16_t*>(out32) : nullptr;
    g.ldo = ldo;
    g.fmt = fmt;
    g.ovf = d_ovf;
    g.r16 = r16;
    if (outa) {
      g.out_hi = outa->hi + out_col;
      g.out_lo = outa->lo ? outa->lo + out_col : nullptr;
      g.ldh = outa->ld;
    }
    int e = ev_begin();
    CK(launch_gemm(&a.mh, split ? &a.ml : &a.mh, &w.mh, split ? &w.ml : &w.mh, w.bn,
                   split ? 2 : 1, epi, g, num_sms, st));
    const double flops = 2.0 * M * (double)w.N * w.K;
    double bytes = (double)M * w.K * (split ? 4 : 2) + (double)w.N * w.K * (split ? 4 : 2);
    bytes += (double)M * w.N * (epi == EPI_F32 ? 4 : epi == EPI_F32_RES ? 8 : (split ? 4 : 2));
    ev_end(e, cls, flops, bytes);
  }

  void layernorm(const float* y, int T, const float* g, const float* b, float* out32, Act* a,
                 bool in16 = false) {
    int e = ev_begin();
    CK(launch_layernorm(y, in16, T, d, dp, g, b, out32, a ? a->hi : nullptr,
                        a ? a->lo : nullptr, fmt, r16, d_ovf, st));
    ev_end(e, C_LN, 0,
           (double)T * d * ((in16 ? 2 : 4) + (out32 ? 4 : 0) + (a ? (split ? 4 : 2) : 0)));
  }

  // One device chunk: m records, T tokens, role-major packing in h_* staging.
  // One device chunk: m records, T tokens; ids already in d_ids (role-major),
  // cu / work items in the pinned h_* staging. Scores land in dscores[0..m).
  void forward_chunk(int m, int64_t T, int64_t n_work, int n_tiles, double sum_l2, int max_l) {
    const bool bos_q = bos_qkv && max_l <= 512;  // BOS attention kernel keeps <= 512 scores
    const int nseq = m * n_roles;
    CK(cudaMemcpyAsync(d_cu, h_cu, (nseq + 1) * 4, cudaMemcpyHostToDevice, st));
    if (n_tiles > 0)
      CK(cudaMemcpyAsync(d_tiles, h_tiles, n_tiles * sizeof(AttTile), cudaMemcpyHostToDevice, st));
    if (n_work > 0)
      CK(cudaMemcpyAsync(d_work, h_work, n_work * sizeof(int2), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(d_ovf, 0, sizeof(int), st));
    const int Ti = (int)T;
    {
      int e = ev_begin();
      // post-norm: the residual stream lives only in the operand pieces xa (fp16
      // hi + lo ~ 22 bits; exact binary16 in fp16 mode; bf16 hi + lo ~ 16 bits in
      // bf16 mode), so LayerNorm
      // writes 8 instead of 12 bytes per element; x32 is written once, by the
      // last LayerNorm, for pooling
      const bool res16 = !pre_norm && (split || r16 || res_bf16) && !layers.empty();
      CK(launch_embed(d_ids, d_cu, nseq, (int)man.vocab_size, d, tok, pos, res16 ? nullptr : x32,
                      dp, pre_norm ? nullptr : xa.hi, pre_norm ? nullptr : xa.lo, fmt, r16, d_ovf,
                      st));
      ev_end(e, C_EMB, 0, (double)T * d * (8 + (res16 ? 0 : 4) + (pre_norm ? 0 : (split ? 4 : 2))));
    }
    const bool res16 = !pre_norm && (split || r16 || res_bf16) && !layers.empty();
    const bool y16 = res16 && r16;  // O-proj / FFN2 outputs as binary16 (reference fp16 mode)
    const int S = nseq;
    // BOS rows of xa (the layer input pieces) and, when the residual is fp32, of x32
    auto gather_inputs = [&]() {
      int e = ev_begin();
      CK(launch_gather_bos(d_cu, S, d, xa.hi, xa.lo, xa.ld, res16 ? nullptr : x32, dp, xb.hi,
                           xb.lo, xb.ld, x32b, dp, st));
      ev_end(e, C_HEAD, 0, (double)S * d * 12);
    };
    for (size_t li = 0; li < layers.size(); ++li) {
      Layer& L = layers[li];
      const bool last = li + 1 == layers.size();
      if (pre_norm) layernorm(x32, Ti, L.g1, L.b1, nullptr, &xa);
      if (last && bos_q) {
        // Last layer: only BOS queries are pooled, so Q (and attention) run on one
        // row per sequence; K and V still cover every token.
        gather_inputs();
        gemm(xa, L.kv_part, Ti, EPI_SPLIT, C_QKV, nullptr, 0, nullptr, 0, &qa, nullptr, d);
        gemm(xb, L.q_part, S, EPI_SPLIT, C_QKV, nullptr, 0, nullptr, 0, &qb);
        int e = ev_begin();
        CK(launch_bos_attention(qb.hi, qb.lo, qb.ld, qa.hi, qa.lo, qa.ld, d, H, d_cu, S, cb.hi,
                                cb.lo, cb.ld, fmt, st));
        ev_end(e, C_ATT, 4.0 * (double)T * d, (double)T * 2 * d * (split ? 4 : 2));
        break;
      }
      gemm(xa, L.qkv, Ti, EPI_SPLIT, C_QKV, nullptr, 0, nullptr, 0, &qa);
      {
        const double bytes = (double)T * d * 4 * (split ? 4 : 2);
        int e = ev_begin();
        if (n_tiles > 0)
          CK(launch_attention_tc(&qm32h, split ? &qm32l : &qm32h, &qt32h, split ? &qt32l : &qt32h,
                                 split ? 3 : r16 ? 2 : 1, d_tiles, n_tiles, H, d, fmt, ca.hi,
                                 ca.lo, ca.ld, d_ovf, num_sms, st));
        if (n_work > 0 && att_tc)
          CK(launch_attention_long(&qm32h, split ? &qm32l : &qm32h, &qt32h,
                                   split ? &qt32l : &qt32h, split ? 3 : r16 ? 2 : 1, d_work,
                                   (int)n_work, d_cu, H, d, fmt, ca.hi, ca.lo, ca.ld, st));
        else if (n_work > 0)
          CK(launch_attention(qa.hi, qa.lo, qa.ld, d, H, d_cu, d_work, (int)n_work, ca.hi, ca.lo,
                              ca.ld, fmt, d_ovf, st));
        ev_end(e, C_ATT, 4.0 * sum_l2 * d, bytes);
        if (n_tiles > 0 && n_work > 0) stats.kernel_launches += 1;
      }
      if (last) break;  // the last layer's O-proj / FFN run on the BOS rows only (below)
      if (!pre_norm) {
        // reference fp16 mode: the rounded residual sums travel as binary16
        gemm(ca, L.o, Ti, EPI_F32_RES, C_O, x32, dp, y32, dp, nullptr, res16 ? &xa : nullptr, 0,
             y16);
        layernorm(y32, Ti, L.g1, L.b1, res16 ? nullptr : x32, &xa, y16);
        gemm(xa, L.w1, Ti, EPI_GELU_SPLIT, C_FFN1, nullptr, 0, nullptr, 0, &ha);
        gemm(ha, L.w2, Ti, EPI_F32_RES, C_FFN2, x32, dp, y32, dp, nullptr, res16 ? &xa : nullptr, 0,
             y16);
        layernorm(y32, Ti, L.g2, L.b2, res16 ? nullptr : x32, &xa, y16);
      } else {
        gemm(ca, L.o, Ti, EPI_F32_RES, C_O, x32, dp, y32, dp, nullptr);
        layernorm(y32, Ti, L.g2, L.b2, nullptr, &xa);
        gemm(xa, L.w1, Ti, EPI_GELU_SPLIT, C_FFN1, nullptr, 0, nullptr, 0, &ha);
        gemm(ha, L.w2, Ti, EPI_F32_RES, C_FFN2, y32, dp, x32, dp, nullptr);
      }
    }
    // Last layer: pooling reads only the BOS row of every sequence (`encoder.py:181-185`)
    // and rows are independent after attention, so the O-projection, both
    // LayerNorms and the FFN run on one row per sequence (bitwise the same values).
    if (!layers.empty()) {
      Layer& L = layers.back();
      if (!bos_q) {  // full last-layer attention: gather its BOS rows
        int e = ev_begin();
        CK(launch_gather_bos(d_cu, S, d, ca.hi, ca.lo, ca.ld, nullptr, 0, cb.hi, cb.lo, cb.ld,
                             nullptr, 0, st));
        ev_end(e, C_HEAD, 0, (double)S * d * 8);
        gather_inputs();
      }
      if (!pre_norm) {
        gemm(cb, L.o, S, EPI_F32_RES, C_O, x32b, dp, y32b, dp, nullptr, res16 ? &xb : nullptr, 0,
             y16);
        layernorm(y32b, S, L.g1, L.b1, res16 ? nullptr : x32b, &xb, y16);
        gemm(xb, L.w1, S, EPI_GELU_SPLIT, C_FFN1, nullptr, 0, nullptr, 0, &hb);
        gemm(hb, L.w2, S, EPI_F32_RES, C_FFN2, x32b, dp, y32b, dp, nullptr, res16 ? &xb : nullptr, 0,
             y16);
        layernorm(y32b, S, L.g2, L.b2, x32b, &xb, y16);
      } else {
        gemm(cb, L.o, S, EPI_F32_RES, C_O, x32b, dp, y32b, dp, nullptr);
        layernorm(y32b, S, L.g2, L.b2, nullptr, &xb);
        gemm(xb, L.w1, S, EPI_GELU_SPLIT, C_FFN1, nullptr, 0, nullptr, 0, &hb);
        gemm(hb, L.w2, S, EPI_F32_RES, C_FFN2, y32b, dp, x32b, dp, nullptr);
      }
    }
    {
      int e = ev_begin();
      CK(launch_features(layers.empty() ? x32 : x32b, dp, d, kind, layers.empty() ? d_cu : nullptr,
                         m, fa.hi, fa.lo, fa.ld, fmt, d_ovf, st));
      ev_end(e, C_HEAD, 0, (double)m * (n_roles * d * 4 + F * (split ? 4 : 2)));
    }
    const Act* in = &fa;
    for (size_t j = 0; j < head.size(); ++j) {
      const bool last = j + 1 == head.size();
      if (last) {
        gemm(*in, head[j], m, EPI_F32, C_HEAD, nullptr, 0, hout, head[j].Npad, nullptr);
      } else {
        gemm(*in, head[j], m, EPI_TANH_SPLIT, C_HEAD, nullptr, 0, nullptr, 0, &ga[j]);
        in = &ga[j];
      }
    }
    {
      int e = ev_begin();
      CK(launch_gather_col0(hout, head.back().Npad, m, dscores, st));
      ev_end(e, C_HEAD, 0, (double)m * 8);
    }
  }

  // Returns true when an fp16 operand piece overflowed (|x| >= 65520) in the chunk.
  bool check_flag() {
    CK(cudaMemcpyAsync(h_ovf, d_ovf, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*h_ovf & 2)
      throw Fail{MFG_ERR_USAGE,
                 "token id out of range for vocab_size " + std::to_string(man.vocab_size)};
    return (*h_ovf & 1) != 0;
  }

  // ---------------------------------------------------------------- range fallback
  // The fp32-parity path keeps activations as fp16 hi/lo pieces; an activation
  // beyond the fp16 range (the reference computes in fp32 and has no such limit,
  // `encoder.py:120-130`) re-scores that chunk on a twin context with bf16 hi/lo
  // pieces (fp32 range, ~16 significant bits, 3 MMAs per k-step), built on first
  // use from the same container. Counted in mfg_stats.fallback_*.
  mfg_config cfg_copy{};
  std::string cfg_path;
  mfg_ctx* twin = nullptr;

  void rescore_chunk_bf16x3(int m, int64_t T, const int32_t* chunk_ids, float* out, bool device_io) {
    if (!twin) {
      mfg_config tc = cfg_copy;
      tc.container_path = cfg_path.c_str();
      tc.precision = MFG_PREC_BF16X3;
      tc.profile = 0;
      twin = new mfg_ctx();
      try {
        twin->init(tc);
      } catch (...) {
        delete twin;
        twin = nullptr;
        throw;
      }
    }
    twin->st = st;
    std::vector<int64_t> cu64((size_t)m * n_roles + 1);
    for (size_t i = 0; i < cu64.size(); ++i) cu64[i] = h_cu[i];
    if (cu64.back() != T) throw Fail{MFG_ERR_RUNTIME, "fallback chunk bookkeeping"};
    const int64_t launches0 = twin->stats.kernel_launches;
    twin->score(m, n_roles, chunk_ids, cu64.data(), out, device_io);
    stats.kernel_launches += twin->stats.kernel_launches - launches0;
    stats.fallback_chunks += 1;
    stats.fallback_records += m;
  }

  void init(const mfg_config& cfg) {
    if (cfg.precision < MFG_PREC_FP32 || cfg.precision > MFG_PREC_FP16)
      throw Fail{MFG_ERR_USAGE, "unknown precision " + std::to_string(cfg.precision)};
    cfg_copy = cfg;
    cfg_path = cfg.container_path;
    device = cfg.device;
    precision = cfg.precision;
    split = cfg.precision == MFG_PREC_FP32 || cfg.precision == MFG_PREC_BF16X3;
    r16 = cfg.precision == MFG_PREC_FP16;
    fmt = (cfg.precision == MFG_PREC_FP32 || r16) ? FMT_F16 : FMT_BF16;
    profile = cfg.profile != 0;
    const auto t0 = std::chrono::steady_clock::now();
    CK(cudaSetDevice(device));
    CK(cudaFree(nullptr));  // create the primary context here (timed as its own phase)
    int major = 0, minor = 0;
    CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    CK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device));
    if (major != 10 || minor != 0)
      throw Fail{MFG_ERR_RUNTIME, "libmfgpu is built for sm_100a (B200); device is sm_" +
                                      std::to_string(major) + std::to_string(minor)};
    CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&own_st, cudaStreamNonBlocking));
    st = own_st;
    load_ms[0] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    build(cfg);
  }

  // ids / out are host pointers (device_io == false) or device pointers (true);
  // cu_seqlens is always a host array.
  void score(int32_t n, int32_t n_roles_in, const int32_t* ids, const int64_t* cu, float* out,
             bool device_io) {
    if (n < 0) throw Fail{MFG_ERR_USAGE, "n_records must be >= 0"};
    if (n_roles_in != n_roles)
      throw Fail{MFG_ERR_USAGE, "model kind '" + man.like + "' scores " + std::to_string(n_roles) +
                                    " sequences per record, got " + std::to_string(n_roles_in)};
    if (n == 0) return;
    const int64_t nseq = (int64_t)n * n_roles;
    if (cu[0] != 0) throw Fail{MFG_ERR_USAGE, "cu_seqlens[0] must be 0"};
    for (int64_t s = 0; s < nseq; ++s) {
      const int64_t L = cu[s + 1] - cu[s];
      if (L > man.max_position)
        throw Fail{MFG_ERR_USAGE, "sequence length " + std::to_string(L) +
                                      " exceeds limit " + std::to_string(man.max_position)};
      if (L <= 0) throw Fail{MFG_ERR_USAGE, "cannot pool a row with no tokens"};
    }
    if (!device_io) {
      const int64_t total = cu[nseq];
      for (int64_t t = 0; t < total; ++t)
        if (ids[t] < 0 || ids[t] >= man.vocab_size)
          throw Fail{MFG_ERR_USAGE,
                     "token id out of range for vocab_size " + std::to_string(man.vocab_size)};
    }

    CK(cudaEventRecord(ev0, st));
    int r0 = 0;
    while (r0 < n) {
      // greedy chunk by records within token / record / work capacity
      int r1 = r0;
      int64_t T = 0, W = 0;
      while (r1 < n && r1 - r0 < cap_records) {
        int64_t t = 0, w = 0;
        for (int k = 0; k < n_roles; ++k) {
          const int64_t L = cu[(int64_t)k * n + r1 + 1] - cu[(int64_t)k * n + r1];
          t += L;
          w += (L + 63) / 64;
        }
        if (T + t > cap_tokens || W + w > work_cap) break;
        T += t;
        W += w;
        ++r1;
      }
      if (r1 == r0) throw Fail{MFG_ERR_USAGE, "record exceeds device chunk capacity"};
      const int m = r1 - r0;
      // role-major chunk: cu / work items on the host, ids staged per role
      int64_t at = 0;
      double sum_l2 = 0;
      int64_t max_l = 0;
      h_cu[0] = 0;
      for (int k = 0; k < n_roles; ++k) {
        const int64_t s0 = (int64_t)k * n + r0, s1 = (int64_t)k * n + r1;
        const int64_t len = cu[s1] - cu[s0];
        if (device_io)
          CK(cudaMemcpyAsync(d_ids + at, ids + cu[s0], len * 4, cudaMemcpyDeviceToDevice, st));
        else
          memcpy(h_ids + at, ids + cu[s0], len * 4);
        for (int64_t s = s0; s < s1; ++s) {
          const int64_t L = cu[s + 1] - cu[s];
          const int ls = (int)(k * m + (s - s0));
          h_cu[ls + 1] = (int32_t)(at + (cu[s + 1] - cu[s0]));
          sum_l2 += (double)L * L;
          max_l = std::max<int64_t>(max_l, L);
        }
        at += len;
      }
      att_plan_tiles(h_cu, m * n_roles, att_tc, v_tiles, v_work);
      std::copy(v_tiles.begin(), v_tiles.end(), h_tiles);
      std::copy(v_work.begin(), v_work.end(), h_work);
      if (!device_io) CK(cudaMemcpyAsync(d_ids, h_ids, T * 4, cudaMemcpyHostToDevice, st));
      forward_chunk(m, T, (int64_t)v_work.size(), (int)v_tiles.size(), sum_l2, (int)max_l);
      if (device_io) {
        CK(cudaMemcpyAsync(out + r0, dscores, m * 4, cudaMemcpyDeviceToDevice, st));
        if (check_flag()) rescore_chunk_bf16x3(m, T, d_ids, out + r0, true);
      } else {
        CK(cudaMemcpyAsync(h_scores, dscores, m * 4, cudaMemcpyDeviceToHost, st));
        if (check_flag()) rescore_chunk_bf16x3(m, T, h_ids, out + r0, false);
        else memcpy(out + r0, h_scores, m * 4);
      }
      stats.tokens += T;
      stats.chunks += 1;
      r0 = r1;
    }
    CK(cudaEventRecord(ev1, st));
    CK(cudaEventSynchronize(ev1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    stats.device_ms += ms;
    stats.calls += 1;
    stats.records += n;
    if (profile) collect_profile();
  }

  ~mfg_ctx() {
    if (st) cudaStreamSynchronize(st);
    if (part_persist) cudaCtxResetPersistingL2Cache();  // release the pinned lines
    delete twin;
    for (void* p : allocs) cudaFree(p);
    if (h_ids) cudaFreeHost(h_ids);
    if (h_cu) cudaFreeHost(h_cu);
    if (h_work) cudaFreeHost(h_work);
    if (h_scores) cudaFreeHost(h_scores);
    if (h_tiles) cudaFreeHost(h_tiles);
    if (h_ovf) cudaFreeHost(h_ovf);
    for (auto e : pev) cudaEventDestroy(e);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (own_st) cudaStreamDestroy(own_st);
  }
};

// ======================================================================= C-ABI
static int set_global(int code, const std::string& msg) {
  g_code = code;
  g_msg = msg;
  return code;
}

extern "C" int mfg_create(const mfg_config* cfg, mfg_ctx** out) {
  if (!cfg || !out || !cfg->container_path) return set_global(MFG_ERR_USAGE, "null argument");
  *out = nullptr;
  mfg_ctx* c = new mfg_ctx();
  try {
    c->init(*cfg);
  } catch (const Fail& f) {
    delete c;
    return set_global(f.code, f.msg);
  } catch (const ContainerError& e) {
    delete c;
    return set_global(MFG_ERR_CONTAINER, e.what());
  } catch (const std::exception& e) {
    delete c;
    return set_global(MFG_ERR_RUNTIME, e.what());
  }
  *out = c;
  return set_global(MFG_OK, "");
}

extern "C" int mfg_check_container(const char* path) {
  if (!path) return set_global(MFG_ERR_USAGE, "null argument");
  try {
    Container c(path);
    check_contract(c);
  } catch (const Fail& f) {
    return set_global(f.code, f.msg);
  } catch (const ContainerError& e) {
    return set_global(MFG_ERR_CONTAINER, e.what());
  } catch (const std::exception& e) {
    return set_global(MFG_ERR_RUNTIME, e.what());
  }
  return set_global(MFG_OK, "");
}

extern "C" int mfg_score_batch(mfg_ctx* c, int32_t n, int32_t n_roles, const int32_t* ids,
                               const int64_t* cu, float* scores) {
  if (!c) return set_global(MFG_ERR_USAGE, "null context");
  try {
    CK(cudaSetDevice(c->device));
    c->score(n, n_roles, ids, cu, scores, false);
  } catch (const Fail& f) {
    c->err_code = f.code;
    c->err_msg = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    c->err_code = MFG_ERR_RUNTIME;
    c->err_msg = e.what();
    return MFG_ERR_RUNTIME;
  }
  c->err_code = 0;
  c->err_msg.clear();
  return MFG_OK;
}

extern "C" int mfg_score_device(mfg_ctx* c, int32_t n, int32_t n_roles, const int32_t* d_ids,
                                const int64_t* cu, float* d_scores) {
  if (!c) return set_global(MFG_ERR_USAGE, "null context");
  try {
    CK(cudaSetDevice(c->device));
    c->score(n, n_roles, d_ids, cu, d_scores, true);
  } catch (const Fail& f) {
    c->err_code = f.code;
    c->err_msg = f.msg;
    return f.code;
  } catch (const std::exception& e) {
    c->err_code = MFG_ERR_RUNTIME;
    c->err_msg = e.what();
    return MFG_ERR_RUNTIME;
  }
  c->err_code = 0;
  c->err_msg.clear();
  return MFG_OK;
}

extern "C" int mfg_set_stream(mfg_ctx* c, void* stream) {
  if (!c) return set_global(MFG_ERR_USAGE, "null context");
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  c->st = stream ? (cudaStream_t)stream : c->own_st;
  c->apply_l2_window(c->st);
  return MFG_OK;
}

extern "C" int mfg_last_error(const mfg_ctx* c, int32_t* code, char* buf, size_t cap) {
  const int cd = c ? c->err_code : g_code;
  const std::string& m = c ? c->err_msg : g_msg;
  if (code) *code = cd;
  if (buf && cap) {
    size_t k = std::min(cap - 1, m.size());
    memcpy(buf, m.data(), k);
    buf[k] = 0;
  }
  return MFG_OK;
}

extern "C" void mfg_destroy(mfg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  delete c;
}

extern "C" int mfg_get_model_info(const mfg_ctx* c, mfg_model_info* o) {
  if (!c || !o) return MFG_ERR_USAGE;
  o->kind = c->kind;
  o->vocab_size = (int32_t)c->man.vocab_size;
  o->d_model = c->d;
  o->n_heads = c->H;
  o->n_layers = (int32_t)c->man.n_layers;
  o->d_ffn = c->f;
  o->max_position = (int32_t)c->man.max_position;
  o->pre_norm = c->pre_norm;
  o->n_roles = c->n_roles;
  o->n_head_stages = (int32_t)c->head.size();
  o->precision = c->precision;
  o->num_sms = c->num_sms;
  o->device_bytes = c->device_bytes;
  for (int i = 0; i < 6; ++i) o->load_ms[i] = c->load_ms[i];
  return MFG_OK;
}

extern "C" int mfg_get_stats(const mfg_ctx* c, mfg_stats* o) {
  if (!c || !o) return MFG_ERR_USAGE;
  *o = c->stats;
  return MFG_OK;
}

extern "C" int mfg_set_profile(mfg_ctx* c, int32_t enable) {
  if (!c) return set_global(MFG_ERR_USAGE, "null context");
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  if (c->profile && !enable) c->collect_profile();
  c->profile = enable != 0;
  return MFG_OK;
}

extern "C" int mfg_reset_stats(mfg_ctx* c) {
  if (!c) return MFG_ERR_USAGE;
  c->stats = mfg_stats{};
  return MFG_OK;
}

// ================================================================= test entry points
namespace {
struct Scratch {
  std::vector<void*> ps;
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    ps.push_back(p);
    CK(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    return (T*)p;
  }
  ~Scratch() {
    for (void* p : ps) cudaFree(p);
  }
};

__global__ void split_rows_kernel(const float* src, int rows, int cols, uint16_t* hi,
                                  uint16_t* lo, int ld, int fmt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)rows * cols) return;
  const int r = (int)(i / cols), c = (int)(i % cols);
  store_split(hi, lo, (size_t)r * ld + c, src[i], fmt, nullptr);
}
__global__ void join_rows_kernel(const uint16_t* hi, const uint16_t* lo, int ld,
                                 int rows, int cols, float* dst, int fmt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)rows * cols) return;
  const int r = (int)(i / cols), c = (int)(i % cols);
  float v = load16(hi, (size_t)r * ld + c, fmt);
  if (lo) v += load16(lo, (size_t)r * ld + c, fmt);
  dst[i] = v;
}

template <class F>
int guarded(F&& fn) {
  try {
    fn();
  } catch (const Fail& f) {
    return set_global(f.code, f.msg);
  } catch (const std::exception& e) {
    return set_global(MFG_ERR_RUNTIME, e.what());
  }
  return set_global(MFG_OK, "");
}
}  // namespace

extern "C" int mfgt_gemm(int32_t precision, int32_t epi, int32_t M, int32_t N, int32_t K,
                         const float* A, const float* W, const float* bias,
                         const float* residual, float* out) {
  return guarded([&] {
    const bool split = precision == MFG_PREC_FP32 || precision == MFG_PREC_BF16X3;
    const bool r16 = precision == MFG_PREC_FP16;
    const int fmt = (precision == MFG_PREC_FP32 || r16) ? FMT_F16 : FMT_BF16;
    int dev = 0, sms = 148;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    Scratch s;
    char err[256];
    const int Kp = pad64(K), Np = pad64(N);
    const int64_t Mp = pad128(M);
    const int bn = gemm_pick_bn(Np);
    float* dA = s.alloc<float>((size_t)M * K);
    float* dW = s.alloc<float>((size_t)K * N);
    CK(cudaMemcpy(dA, A, (size_t)M * K * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dW, W, (size_t)K * N * 4, cudaMemcpyHostToDevice));
    auto* ah = s.alloc<uint16_t>(Mp * Kp);
    auto* al = split ? s.alloc<uint16_t>(Mp * Kp) : nullptr;
    auto* wh = s.alloc<uint16_t>((size_t)Np * Kp);
    auto* wl = split ? s.alloc<uint16_t>((size_t)Np * Kp) : nullptr;
    const int64_t tot = (int64_t)M * K;
    split_rows_kernel<<<(unsigned)((tot + 255) / 256), 256>>>(dA, M, K, ah, al, Kp, fmt);
    CK(cudaGetLastError());
    float* dal = nullptr;
    if (split && fmt == FMT_F16) {  // the engine's per-column weight prescale
      dal = s.alloc<float>(Np);
      CK(launch_weight_scales(dW, K, N, dal, 0));
    }
    CK(launch_transpose_split(dW, K, N, wh, wl, Kp, 0, fmt, nullptr, 0, dal));
    float* db = s.alloc<float>(Np);
    if (bias) {
      std::vector<float> b(bias, bias + N);
      if (r16)
        for (auto& v : b) v = __half2float(__float2half_rn(v));
      CK(cudaMemcpy(db, b.data(), N * 4, cudaMemcpyHostToDevice));
    }
    float* dr = s.alloc<float>((size_t)M * Np);
    if (residual)
      CK(cudaMemcpy2D(dr, Np * 4, residual, N * 4, N * 4, M, cudaMemcpyHostToDevice));
    float* d32 = s.alloc<float>((size_t)M * Np);
    auto* oh = s.alloc<uint16_t>((size_t)M * Np);
    auto* ol = split ? s.alloc<uint16_t>((size_t)M * Np) : nullptr;
    CUtensorMap mah, mal, mwh, mwl;
    if (!make_tmap_u16(&mah, ah, Mp, Kp, Kp, GEMM_BM, err, sizeof err) ||
        !make_tmap_u16(&mwh, wh, Np, Kp, Kp, gemm_b_box_rows(bn), err, sizeof err))
      throw Fail{MFG_ERR_RUNTIME, err};
    if (split && (!make_tmap_u16(&mal, al, Mp, Kp, Kp, GEMM_BM, err, sizeof err) ||
                  !make_tmap_u16(&mwl, wl, Np, Kp, Kp, gemm_b_box_rows(bn), err, sizeof err)))
      throw Fail{MFG_ERR_RUNTIME, err};
    GemmArgs g{};
    g.M = M;
    g.N = Np;
    g.K = Kp;
    g.bias = db;
    g.alpha = dal;
    g.residual = dr;
    g.ldr = Np;
    g.out_f32 = d32;
    g.ldo = Np;
    g.out_hi = oh;
    g.out_lo = ol;
    g.ldh = Np;
    g.fmt = fmt;
    g.ovf = nullptr;
    g.r16 = r16;
    g.kchunk = gemm_kchunk_blocks(Kp);
    g.partial = s.alloc<float>(gemm_partial_floats(sms));
    g.tile_ctr = s.alloc<int>(2);
    CK(launch_gemm(&mah, split ? &mal : &mah, &mwh, split ? &mwl : &mwh, bn, split ? 2 : 1, epi,
                   g, sms, 0));
    CK(cudaDeviceSynchronize());
    if (epi == EPI_F32 || epi == EPI_F32_RES) {
      CK(cudaMemcpy2D(out, N * 4, d32, Np * 4, N * 4, M, cudaMemcpyDeviceToHost));
    } else {
      float* tmpd = s.alloc<float>((size_t)M * N);
      join_rows_kernel<<<(unsigned)(((int64_t)M * N + 255) / 256), 256>>>(oh, ol, Np, M, N, tmpd, fmt);
      CK(cudaGetLastError());
      CK(cudaMemcpy(out, tmpd, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
    }
  });
}

extern "C" int mfgt_attention(int32_t precision, int32_t n_seq, const int32_t* cu, int32_t d,
                              int32_t n_heads, const float* qkv, float* ctx_out, int32_t use_tc) {
  return guarded([&] {
    const bool split = precision == MFG_PREC_FP32 || precision == MFG_PREC_BF16X3;
    const bool r16 = precision == MFG_PREC_FP16;
    const int fmt = (precision == MFG_PREC_FP32 || r16) ? FMT_F16 : FMT_BF16;
    Scratch s;
    char err[256];
    const int T = cu[n_seq];
    const int64_t Tp = pad128(T) + 128;
    const int ldq = pad64(3 * d), ldc = pad64(d);
    float* dq = s.alloc<float>((size_t)T * 3 * d);
    CK(cudaMemcpy(dq, qkv, (size_t)T * 3 * d * 4, cudaMemcpyHostToDevice));
    auto* qh = s.alloc<uint16_t>((size_t)Tp * ldq);
    auto* ql = split ? s.alloc<uint16_t>((size_t)Tp * ldq) : nullptr;
    const int64_t tot = (int64_t)T * 3 * d;
    split_rows_kernel<<<(unsigned)((tot + 255) / 256), 256>>>(dq, T, 3 * d, qh, ql, ldq, fmt);
    CK(cudaGetLastError());
    int32_t* dcu = s.alloc<int32_t>(n_seq + 1);
    CK(cudaMemcpy(dcu, cu, (n_seq + 1) * 4, cudaMemcpyHostToDevice));
    const bool tc_ok = use_tc && (d / n_heads == 64 || d / n_heads == 80) && (d % 64 == 0);
    std::vector<int2> work;
    std::vector<AttTile> tiles;
    att_plan_tiles(cu, n_seq, tc_ok, tiles, work);
    int2* dw = s.alloc<int2>(work.size());
    if (!work.empty())
      CK(cudaMemcpy(dw, work.data(), work.size() * sizeof(int2), cudaMemcpyHostToDevice));
    AttTile* dt = s.alloc<AttTile>(tiles.size());
    if (!tiles.empty())
      CK(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(AttTile), cudaMemcpyHostToDevice));
    auto* ch = s.alloc<uint16_t>((size_t)T * ldc);
    auto* cl = split ? s.alloc<uint16_t>((size_t)T * ldc) : nullptr;
    CUtensorMap mh, ml, th, tl;
    if (tc_ok) {
      if (!make_tmap_u16(&mh, qh, Tp, ldq, ldq, 32, err, sizeof err) ||
          !make_tmap_u16_box(&th, qh, Tp, ldq, ldq, 16, 32, 32, err, sizeof err))
        throw Fail{MFG_ERR_RUNTIME, err};
      if (split && (!make_tmap_u16(&ml, ql, Tp, ldq, ldq, 32, err, sizeof err) ||
                    !make_tmap_u16_box(&tl, ql, Tp, ldq, ldq, 16, 32, 32, err, sizeof err)))
        throw Fail{MFG_ERR_RUNTIME, err};
    }
    const int mode = split ? 3 : r16 ? 2 : 1;
    if (!tiles.empty()) {
      int sms = 148, dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      CK(launch_attention_tc(&mh, split ? &ml : &mh, &th, split ? &tl : &th, mode, dt,
                             (int)tiles.size(), n_heads, d, fmt, ch, cl, ldc, nullptr, sms, 0));
    }
    if (!work.empty() && tc_ok)
      CK(launch_attention_long(&mh, split ? &ml : &mh, &th, split ? &tl : &th, mode, dw,
                               (int)work.size(), dcu, n_heads, d, fmt, ch, cl, ldc, 0));
    else if (!work.empty())
      CK(launch_attention(qh, ql, ldq, d, n_heads, dcu, dw, (int)work.size(), ch, cl, ldc, fmt,
                          nullptr, 0));
    float* o = s.alloc<float>((size_t)T * d);
    join_rows_kernel<<<(unsigned)(((int64_t)T * d + 255) / 256), 256>>>(ch, cl, ldc, T, d, o, fmt);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(ctx_out, o, (size_t)T * d * 4, cudaMemcpyDeviceToHost));
  });
}

// Host-only: the attention work planner (att_plan_tiles) for CPU tests.
// tiles_out: n_tiles x {t0[4], len[4]}; work_out: n_work x {seq, q0}.
extern "C" int mfgt_plan_tiles(const int32_t* cu, int32_t nseq, int32_t tc_ok, int32_t* tiles_out,
                               int32_t* n_tiles, int32_t* work_out, int32_t* n_work,
                               int32_t cap) {
  std::vector<AttTile> tiles;
  std::vector<int2> work;
  att_plan_tiles(cu, nseq, tc_ok != 0, tiles, work);
  if ((int64_t)tiles.size() > cap || (int64_t)work.size() > cap) return MFG_ERR_USAGE;
  for (size_t i = 0; i < tiles.size(); ++i)
    for (int j = 0; j < 4; ++j) {
      tiles_out[i * 8 + j] = tiles[i].t0[j];
      tiles_out[i * 8 + 4 + j] = tiles[i].len[j];
    }
  for (size_t i = 0; i < work.size(); ++i) {
    work_out[2 * i] = work[i].x;
    work_out[2 * i + 1] = work[i].y;
  }
  *n_tiles = (int32_t)tiles.size();
  *n_work = (int32_t)work.size();
  return MFG_OK;
}

// Diagnostics: route the next attention launches' per-item clock64 trace to a
// device buffer (enable = 1), or copy it to host_out[4*64*8] and stop (enable = 0).
extern "C" int mfgt_att_trace(int32_t enable, long long* host_out) {
  static long long* buf = nullptr;
  return guarded([&] {
    const size_t n = 4 * 64 * 8;
    if (enable) {
      if (!buf) CK(cudaMalloc(&buf, n * sizeof(long long)));
      CK(cudaMemset(buf, 0, n * sizeof(long long)));
      CK(att_set_trace(buf));
    } else {
      CK(cudaDeviceSynchronize());
      CK(att_set_trace(nullptr));
      if (buf && host_out) CK(cudaMemcpy(host_out, buf, n * sizeof(long long), cudaMemcpyDeviceToHost));
    }
  });
}

extern "C" int mfgt_layernorm(int32_t T, int32_t d, const float* y, const float* g,
                              const float* b, float* out) {
  return guarded([&] {
    Scratch s;
    float* dy = s.alloc<float>((size_t)T * d);
    float* dg = s.alloc<float>(d);
    float* db = s.alloc<float>(d);
    float* dout = s.alloc<float>((size_t)T * d);
    CK(cudaMemcpy(dy, y, (size_t)T * d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dg, g, d * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, b, d * 4, cudaMemcpyHostToDevice));
    CK(launch_layernorm(dy, 0, T, d, d, dg, db, dout, nullptr, nullptr, FMT_BF16, 0, nullptr, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, dout, (size_t)T * d * 4, cudaMemcpyDeviceToHost));
  });
}
