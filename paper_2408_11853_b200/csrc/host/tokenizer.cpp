// Host packing library (include/mfhost.h): code-point trie tokenizer, per-kind
// sequence assembly, batch planner, role-major packer. All integer work; the
// output must equal the reference's bit for bit (tests/test_host_packing.py).
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/mfhost.h"

namespace {

constexpr uint32_t MARKER = 0x2581;  // '▁'
constexpr int32_t UNK = 1, BOS = 2, EOS = 3, SEP = 4, N_SPECIAL = 5;

// Python's str.isspace() set (what str.split() splits on), Python 3.12 UCD.
inline bool py_isspace(uint32_t c) {
  if (c <= 0x20) return c == 0x20 || (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x1F);
  if (c < 0x85) return false;
  return c == 0x85 || c == 0xA0 || c == 0x1680 || (c >= 0x2000 && c <= 0x200A) || c == 0x2028 ||
         c == 0x2029 || c == 0x202F || c == 0x205F || c == 0x3000;
}

// Lenient UTF-8 decoder (input comes from Python str.encode(surrogatepass)).
inline uint32_t next_cp(const unsigned char*& p, const unsigned char* e) {
  uint32_t c = *p++;
  if (c < 0x80) return c;
  int n = c >= 0xF0 ? 3 : c >= 0xE0 ? 2 : c >= 0xC0 ? 1 : 0;
  c &= n == 3 ? 0x07 : n == 2 ? 0x0F : 0x1F;
  while (n-- > 0 && p < e) c = (c << 6) | (*p++ & 0x3F);
  return c;
}

inline uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace

struct mfh_vocab {
  int32_t size = 0, max_piece = 0;
  // trie: edge table keyed by (node << 21 | code point), open addressing
  std::vector<uint64_t> keys;
  std::vector<int32_t> vals;
  uint64_t mask = 0;
  std::vector<int32_t> term;  // token id ending at node, -1 if none

  int32_t child(int32_t node, uint32_t cp) const {
    const uint64_t k = ((uint64_t)node << 21) | cp;
    for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
      if (keys[h] == k) return vals[h];
      if (keys[h] == ~0ull) return -1;
    }
  }
  void insert_edge(uint64_t k, int32_t v) {
    for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
      if (keys[h] == ~0ull) {
        keys[h] = k;
        vals[h] = v;
        return;
      }
    }
  }

  // Vocabulary.encode: whitespace split, "▁"-join, greedy longest match.
  void encode(const char* text, int64_t nbytes, std::vector<uint32_t>& s,
              std::vector<int32_t>& out) const {
    s.clear();
    const unsigned char* p = (const unsigned char*)text;
    const unsigned char* e = p + nbytes;
    bool in_word = false;
    while (p < e) {
      const uint32_t c = next_cp(p, e);
      if (py_isspace(c)) {
        in_word = false;
      } else {
        if (!in_word) s.push_back(MARKER);
        in_word = true;
        s.push_back(c);
      }
    }
    const size_t n = s.size();
    size_t pos = 0;
    while (pos < n) {
      int32_t node = 0, best = -1;
      size_t best_len = 0;
      for (size_t j = pos; j < n; ++j) {
        node = child(node, s[j]);
        if (node < 0) break;
        if (term[node] >= 0) {
          best = term[node];
          best_len = j - pos + 1;
        }
      }
      if (best < 0) {
        out.push_back(UNK);
        pos += 1;
      } else {
        out.push_back(best);
        pos += best_len;
      }
    }
  }
};

extern "C" int mfh_vocab_create(const char* blob, int64_t nbytes, int32_t n_tokens,
                                mfh_vocab** out) {
  if (!out || n_tokens < 0) return 2;
  auto* v = new mfh_vocab();
  v->size = n_tokens;
  // split blob on '\n'
  std::vector<std::pair<int64_t, int64_t>> toks;
  toks.reserve(n_tokens);
  int64_t st = 0;
  for (int64_t i = 0; i <= nbytes; ++i)
    if (i == nbytes || blob[i] == '\n') {
      toks.push_back({st, i});
      st = i + 1;
    }
  if ((int32_t)toks.size() != n_tokens) {
    delete v;
    return 2;
  }
  int64_t cps = 0;
  for (int32_t i = N_SPECIAL; i < n_tokens; ++i) cps += toks[i].second - toks[i].first;
  uint64_t cap = 16;
  while (cap < (uint64_t)(2 * cps + 16)) cap <<= 1;
  v->keys.assign(cap, ~0ull);
  v->vals.assign(cap, -1);
  v->mask = cap - 1;
  v->term.assign(1, -1);
  for (int32_t i = N_SPECIAL; i < n_tokens; ++i) {
    const unsigned char* p = (const unsigned char*)blob + toks[i].first;
    const unsigned char* e = (const unsigned char*)blob + toks[i].second;
    int32_t node = 0, len = 0;
    while (p < e) {
      const uint32_t c = next_cp(p, e);
      int32_t ch = v->child(node, c);
      if (ch < 0) {
        ch = (int32_t)v->term.size();
        v->term.push_back(-1);
        v->insert_edge(((uint64_t)node << 21) | c, ch);
      }
      node = ch;
      ++len;
    }
    if (node != 0 && v->term[node] < 0) v->term[node] = i;  // first occurrence wins
    v->max_piece = std::max(v->max_piece, len);
  }
  *out = v;
  return 0;
}

extern "C" void mfh_vocab_destroy(mfh_vocab* v) { delete v; }
extern "C" int32_t mfh_vocab_size(const mfh_vocab* v) { return v ? v->size : 0; }
extern "C" int32_t mfh_vocab_max_piece(const mfh_vocab* v) { return v ? v->max_piece : 0; }

extern "C" int64_t mfh_encode(const mfh_vocab* v, const char* text, int64_t nbytes, int32_t* out,
                              int64_t cap) {
  std::vector<uint32_t> s;
  std::vector<int32_t> ids;
  v->encode(text, nbytes, s, ids);
  if ((int64_t)ids.size() > cap) return -(int64_t)ids.size();
  std::copy(ids.begin(), ids.end(), out);
  return (int64_t)ids.size();
}

namespace {

struct Part {
  std::vector<int32_t> ids;
  std::vector<int64_t> lens;
  int err = 0;
};

// encode_fields for records [r0, r1) (vocab.py:104-143)
void encode_range(const mfh_vocab* v, int kind, int r0, int r1, const char* blob,
                  const int64_t* off, int max_len, Part& out) {
  const int nf = kind == 1 ? 3 : 2;
  std::vector<uint32_t> s;
  std::vector<int32_t> a, b;
  for (int r = r0; r < r1; ++r) {
    const int64_t* fo = off + (int64_t)r * nf;
    if (kind == 2) {
      if (max_len < 3) {
        out.err = 2;
        return;
      }
      a.clear();
      b.clear();
      v->encode(blob + fo[0], fo[1] - fo[0], s, a);
      v->encode(blob + fo[1], fo[2] - fo[1], s, b);
      // pop from the longer side, ties pop the second (closed form)
      const int64_t budget = max_len - 3;
      int64_t na = (int64_t)a.size(), nb = (int64_t)b.size();
      if (na + nb > budget) {
        const int64_t keep_a = std::min(na, std::max((budget + 1) / 2, budget - nb));
        na = keep_a;
        nb = budget - keep_a;
      }
      out.ids.push_back(BOS);
      out.ids.insert(out.ids.end(), a.begin(), a.begin() + na);
      out.ids.push_back(SEP);
      out.ids.insert(out.ids.end(), b.begin(), b.begin() + nb);
      out.ids.push_back(EOS);
      out.lens.push_back(na + nb + 3);
    } else {
      for (int k = 0; k < nf; ++k) {
        a.clear();
        v->encode(blob + fo[k], fo[k + 1] - fo[k], s, a);
        int64_t n = (int64_t)a.size() + 2;
        if (n > max_len) {
          if (max_len < 2) {
            out.err = 2;
            return;
          }
          // ids[:max_len-1] + [EOS]: keep BOS + max_len-2 content ids
          out.ids.push_back(BOS);
          out.ids.insert(out.ids.end(), a.begin(), a.begin() + (max_len - 2));
          out.ids.push_back(EOS);
          out.lens.push_back(max_len);
        } else {
          out.ids.push_back(BOS);
          out.ids.insert(out.ids.end(), a.begin(), a.end());
          out.ids.push_back(EOS);
          out.lens.push_back(n);
        }
      }
    }
  }
}

}  // namespace

extern "C" int64_t mfh_encode_records(const mfh_vocab* v, int32_t kind, int32_t n,
                                      const char* blob, const int64_t* field_off,
                                      int32_t max_len, int32_t n_threads, int32_t* ids_out,
                                      int64_t ids_cap, int64_t* seq_off) {
  if (!v || kind < 0 || kind > 2 || n < 0) return 2;
  if (n == 0) {
    seq_off[0] = 0;
    return 0;
  }
  int th = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  th = std::max(1, std::min(th, (n + 63) / 64));
  std::vector<Part> parts(th);
  std::vector<std::thread> pool;
  for (int t = 0; t < th; ++t) {
    const int r0 = (int)((int64_t)n * t / th), r1 = (int)((int64_t)n * (t + 1) / th);
    if (th == 1)
      encode_range(v, kind, r0, r1, blob, field_off, max_len, parts[t]);
    else
      pool.emplace_back(encode_range, v, kind, r0, r1, blob, field_off, max_len,
                        std::ref(parts[t]));
  }
  for (auto& t : pool) t.join();
  int64_t total = 0;
  for (auto& p : parts) {
    if (p.err) return p.err;
    total += (int64_t)p.ids.size();
  }
  if (total > ids_cap) return -total;
  int64_t at = 0, si = 0;
  seq_off[0] = 0;
  for (auto& p : parts) {
    std::memcpy(ids_out + at, p.ids.data(), p.ids.size() * 4);
    at += (int64_t)p.ids.size();
    for (int64_t L : p.lens) {
      seq_off[si + 1] = seq_off[si] + L;
      ++si;
    }
  }
  return 0;
}

extern "C" int mfh_plan(const int64_t* lengths, int64_t n, int32_t mini_batch, int32_t factor,
                        int32_t sort, int64_t* order) {
  if (mini_batch < 1 || factor < 1) return 2;
  const int64_t win = (int64_t)mini_batch * factor;
  std::iota(order, order + n, (int64_t)0);
  if (sort)
    for (int64_t s = 0; s < n; s += win) {
      const int64_t e = std::min(n, s + win);
      std::stable_sort(order + s, order + e, [&](int64_t a, int64_t b) {
        return lengths[a] > lengths[b];  // ties keep index order (stable)
      });
    }
  return 0;
}

extern "C" int mfh_pack_roles(const int32_t* ids, const int64_t* seq_off, int32_t n_seqs,
                              const int64_t* order, int64_t m, int32_t* ids_out,
                              int64_t* cu_out) {
  int64_t at = 0;
  cu_out[0] = 0;
  for (int32_t k = 0; k < n_seqs; ++k)
    for (int64_t i = 0; i < m; ++i) {
      const int64_t s = order[i] * n_seqs + k;
      const int64_t L = seq_off[s + 1] - seq_off[s];
      std::memcpy(ids_out + at, ids + seq_off[s], L * 4);
      at += L;
      cu_out[k * m + i + 1] = at;
    }
  return 0;
}
