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
  // Trie: edge table keyed by (node << 21 | code point), open addressing. One
  // 16-byte slot holds the key, the child node and the token id ending at the
  // child, so each step of a walk touches one cache line.
  struct Edge {
    uint64_t key;
    int32_t child, term;
  };
  std::vector<Edge> edges;
  uint64_t mask = 0;
  int32_t n_nodes = 1;
  int32_t child(int32_t node, uint32_t cp, int32_t& term) const {
    const uint64_t k = ((uint64_t)node << 21) | cp;
    for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask) {
      const Edge& e = edges[h];
      if (e.key == k) {
        term = e.term;
        return e.child;
      }
      if (e.key == ~0ull) return -1;
    }
  }
  Edge& edge_slot(uint64_t k) {
    for (uint64_t h = mix(k) & mask;; h = (h + 1) & mask)
      if (edges[h].key == k || edges[h].key == ~0ull) return edges[h];
  }

  // Whole-piece table keyed by the piece's UTF-8 bytes (text and vocabulary both
  // come from Python's canonical encoder, so byte equality is code-point
  // equality). When no piece holds the word marker after its first code point,
  // no match can run past the end of a word, so the piece equal to the rest of
  // the word (if any) is the longest match there: one lookup instead of a walk
  // per code point. Pieces of <= 16 bytes compare inside their 32-byte slot.
  struct Piece {
    uint64_t h;
    int32_t id, len;
    unsigned char b[16];
  };
  std::vector<Piece> pieces;
  std::vector<std::string> long_pieces;  // > 16 bytes, indexed by slot
  std::vector<int32_t> long_of;          // slot -> index into long_pieces (-1)
  uint64_t pmask = 0;
  int32_t max_piece_bytes = 0;
  bool words_closed = true;  // no piece has the marker at index > 0

  static uint64_t hash_bytes(const unsigned char* p, size_t n) {
    uint64_t h = 0x243F6A8885A308D3ull ^ n;
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w;
      std::memcpy(&w, p + i, 8);
      h = mix(h ^ w);
    }
    uint64_t w = 0;
    std::memcpy(&w, p + i, n - i);
    return mix(h ^ w);
  }

  // id of the piece whose bytes are p[0..n), -1 if none
  int32_t whole(const unsigned char* p, size_t n) const {
    if (n == 0 || (int64_t)n > max_piece_bytes) return -1;
    return whole_h(p, n, hash_bytes(p, n));
  }
  int32_t whole_h(const unsigned char* p, size_t n, uint64_t hv) const {
    for (uint64_t h = hv & pmask;; h = (h + 1) & pmask) {
      const Piece& q = pieces[h];
      if (q.id < 0) return -1;
      if (q.h == hv && q.len == (int32_t)n) {
        const unsigned char* r = n <= 16 ? q.b : (const unsigned char*)long_pieces[long_of[h]].data();
        if (std::memcmp(r, p, n) == 0) return q.id;
      }
    }
  }
  void add_piece(const unsigned char* p, size_t n, int32_t id) {
    const uint64_t hv = hash_bytes(p, n);
    for (uint64_t h = hv & pmask;; h = (h + 1) & pmask) {
      Piece& q = pieces[h];
      if (q.id < 0) {
        q.h = hv;
        q.id = id;
        q.len = (int32_t)n;
        if (n <= 16) {
          std::memcpy(q.b, p, n);
        } else {
          long_of[h] = (int32_t)long_pieces.size();
          long_pieces.emplace_back((const char*)p, n);
        }
        max_piece_bytes = std::max(max_piece_bytes, (int32_t)n);
        return;
      }
      if (whole(p, n) >= 0) return;  // first occurrence wins
    }
  }

  // greedy longest match of s[pos..end) from the trie; returns the match length
  // (0: no piece matches) and its id
  size_t walk(const uint32_t* s, size_t pos, size_t end, int32_t& id) const {
    int32_t node = 0;
    size_t best_len = 0;
    id = -1;
    for (size_t j = pos; j < end; ++j) {
      int32_t term;
      node = child(node, s[j], term);
      if (node < 0) break;
      if (term >= 0) {
        id = term;
        best_len = j - pos + 1;
      }
    }
    return best_len;
  }

  // Vocabulary.encode: whitespace split, "▁"-join, greedy longest match.
  void encode(const char* text, int64_t nbytes, std::vector<uint32_t>& s,
              std::vector<int32_t>& out) const {
    const unsigned char* p0 = (const unsigned char*)text;
    const unsigned char* e = p0 + nbytes;
    if (!words_closed) {  // pieces may span words: walk the whole "▁"-joined sequence
      s.clear();
      bool in_word = false;
      for (const unsigned char* p = p0; p < e;) {
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
        int32_t id;
        const size_t len = walk(s.data(), pos, n, id);
        out.push_back(len ? id : UNK);
        pos += len ? len : 1;
      }
      return;
    }
    // Words are cut, hashed and their table slots prefetched in batches of 32,
    // then resolved in order: the independent lookups overlap their cache misses.
    constexpr int BATCH = 32;
    struct Word {
      const unsigned char* w0;
      uint32_t wb;
      uint64_t h;  // hash of "▁" + word
      bool fits;   // short enough to be one piece
    };
    Word batch[BATCH];
    unsigned char key[3 + 64];
    key[0] = 0xE2, key[1] = 0x96, key[2] = 0x81;  // "▁" in UTF-8
    std::vector<uint32_t> boff;                      // byte offset of each code point
    const unsigned char* p = p0;
    bool more = true;
    while (more) {
      int nb = 0;
      while (nb < BATCH) {
        // next word: [w0, w1) bytes of non-space code points
        const unsigned char* w0 = nullptr;
        while (p < e) {
          const unsigned char* q = p;
          const uint32_t c = *p < 0x80 ? *p++ : next_cp(p, e);
          if (!py_isspace(c)) {
            w0 = q;
            break;
          }
        }
        if (!w0) {
          more = false;
          break;
        }
        while (p < e) {
          const unsigned char* q = p;
          const uint32_t c = *p < 0x80 ? *p++ : next_cp(p, e);
          if (py_isspace(c)) {
            p = q;
            break;
          }
        }
        Word& w = batch[nb++];
        w.w0 = w0;
        w.wb = (uint32_t)(p - w0);
        w.fits = w.wb + 3 <= (uint32_t)max_piece_bytes && w.wb <= 64;
        if (w.fits) {
          std::memcpy(key + 3, w0, w.wb);
          w.h = hash_bytes(key, w.wb + 3);
          __builtin_prefetch(&pieces[w.h & pmask]);
        }
      }
      for (int i = 0; i < nb; ++i) {
        const Word& w = batch[i];
        if (w.fits) {  // whole word, marker included
          std::memcpy(key + 3, w.w0, w.wb);
          const int32_t id = whole_h(key, w.wb + 3, w.h);
          if (id >= 0) {
            out.push_back(id);
            continue;
          }
        }
        // the word is not one piece: greedy walk over its code points
        const unsigned char* w0 = w.w0;
        const unsigned char* w1 = w0 + w.wb;
        s.clear();
        boff.clear();
        s.push_back(MARKER);
        boff.push_back(0);
        for (const unsigned char* q = w0; q < w1;) {
          boff.push_back((uint32_t)(q - w0));
          s.push_back(next_cp(q, w1));
        }
        const size_t n = s.size();
        size_t pos = 0;
        while (pos < n) {
          if (pos > 0) {  // the rest of the word as one piece?
            const int32_t id = whole(w0 + boff[pos], w.wb - boff[pos]);
            if (id >= 0) {
              out.push_back(id);
              break;
            }
          }
          int32_t wid;
          const size_t len = walk(s.data(), pos, n, wid);
          out.push_back(len ? wid : UNK);
          pos += len ? len : 1;
        }
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
  v->edges.assign(cap, mfh_vocab::Edge{~0ull, -1, -1});
  v->mask = cap - 1;
  uint64_t pcap = 16;
  while (pcap < (uint64_t)(2 * n_tokens + 16)) pcap <<= 1;
  v->pieces.assign(pcap, mfh_vocab::Piece{0, -1, 0, {}});
  v->long_of.assign(pcap, -1);
  v->pmask = pcap - 1;
  std::vector<uint32_t> cp;
  for (int32_t i = N_SPECIAL; i < n_tokens; ++i) {
    const unsigned char* p = (const unsigned char*)blob + toks[i].first;
    const unsigned char* e = (const unsigned char*)blob + toks[i].second;
    cp.clear();
    int32_t node = 0;
    mfh_vocab::Edge* last = nullptr;
    while (p < e) {
      const uint32_t c = next_cp(p, e);
      if (c == MARKER && !cp.empty()) v->words_closed = false;
      cp.push_back(c);
      mfh_vocab::Edge& ed = v->edge_slot(((uint64_t)node << 21) | c);
      if (ed.key == ~0ull) {
        ed.key = ((uint64_t)node << 21) | c;
        ed.child = v->n_nodes++;
      }
      node = ed.child;
      last = &ed;
    }
    if (last && last->term < 0) last->term = i;  // first occurrence wins
    if (!cp.empty())
      v->add_piece((const unsigned char*)blob + toks[i].first,
                   (size_t)(toks[i].second - toks[i].first), i);
    v->max_piece = std::max(v->max_piece, (int32_t)cp.size());
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
// Field k of record r is blob[span[2(r nf + k)] .. span[2(r nf + k) + 1]).
void encode_range(const mfh_vocab* v, int kind, int64_t r0, int64_t r1, const char* blob,
                  const int64_t* span, int max_len, Part& out) {
  const int nf = kind == 1 ? 3 : 2;
  std::vector<uint32_t> s;
  std::vector<int32_t> a, b;
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t* fs = span + 2 * r * nf;
    if (kind == 2) {
      if (max_len < 3) {
        out.err = 2;
        return;
      }
      a.clear();
      b.clear();
      v->encode(blob + fs[0], fs[1] - fs[0], s, a);
      v->encode(blob + fs[2], fs[3] - fs[2], s, b);
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
        v->encode(blob + fs[2 * k], fs[2 * k + 1] - fs[2 * k], s, a);
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

// Runs encode_range over n records on th threads and concatenates the parts.
int64_t encode_spans(const mfh_vocab* v, int kind, int64_t n, const char* blob,
                     const int64_t* span, int max_len, int n_threads, int32_t* ids_out,
                     int64_t ids_cap, int64_t* seq_off) {
  int th = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  th = (int)std::max<int64_t>(1, std::min<int64_t>(th, (n + 63) / 64));
  if (n_threads <= 0 && n > 0) {
    // auto: at least 256 KB of text per thread -- a reference window of short
    // records (1024 x ~100 B) encodes fastest on one thread (measured 860k vs
    // 570k records/s with 8), long ones still split (config 2: 1.3 MB per window)
    const int nf = kind == 1 ? 3 : 2;
    const int64_t bytes = span[2 * n * nf - 1] - span[0];
    th = (int)std::max<int64_t>(1, std::min<int64_t>(th, bytes >> 18));
  }
  std::vector<Part> parts(th);
  std::vector<std::thread> pool;
  for (int t = 0; t < th; ++t) {
    const int64_t r0 = n * t / th, r1 = n * (t + 1) / th;
    if (th == 1)
      encode_range(v, kind, r0, r1, blob, span, max_len, parts[t]);
    else
      pool.emplace_back(encode_range, v, kind, r0, r1, blob, span, max_len, std::ref(parts[t]));
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
  const int nf = kind == 1 ? 3 : 2;
  std::vector<int64_t> span(2 * (size_t)n * nf);
  for (int64_t j = 0; j < (int64_t)n * nf; ++j) {
    span[2 * j] = field_off[j];
    span[2 * j + 1] = field_off[j + 1];
  }
  return encode_spans(v, kind, n, blob, span.data(), max_len, n_threads, ids_out, ids_cap,
                      seq_off);
}

// Native TSV intake (`evaluate.py:117-123`: line.rstrip("\n").split("\t"), exact
// column count else ColumnCountError(line index)): column check over all lines
// first (a bad line wins over a max_len error, as in the reference's order),
// then encode_fields on the field spans.
extern "C" int64_t mfh_encode_tsv(const mfh_vocab* v, int32_t kind, const char* blob,
                                  const int64_t* line_off, int64_t n_lines, int32_t max_len,
                                  int32_t n_threads, int32_t* ids_out, int64_t ids_cap,
                                  int64_t* seq_off, int64_t* bad_line, int32_t* bad_cols) {
  if (!v || kind < 0 || kind > 2 || n_lines < 0 || !bad_line || !bad_cols) return 2;
  *bad_line = -1;
  *bad_cols = 0;
  if (n_lines == 0) {
    seq_off[0] = 0;
    return 0;
  }
  const int nf = kind == 1 ? 3 : 2;
  std::vector<int64_t> span(2 * (size_t)n_lines * nf);
  int th = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  th = (int)std::max<int64_t>(1, std::min<int64_t>(th, (n_lines + 1023) / 1024));
  std::vector<int64_t> first_bad(th, -1);
  std::vector<int32_t> first_cols(th, 0);
  auto split = [&](int t, int64_t l0, int64_t l1) {
    for (int64_t l = l0; l < l1; ++l) {
      const int64_t b0 = line_off[l];
      int64_t b1 = line_off[l + 1];
      while (b1 > b0 && blob[b1 - 1] == '\n') --b1;  // rstrip("\n")
      int cols = 0;
      int64_t st = b0;
      int64_t* fs = span.data() + 2 * l * nf;
      for (int64_t i = b0;; ++i) {
        if (i == b1 || blob[i] == '\t') {
          if (cols < nf) {
            fs[2 * cols] = st;
            fs[2 * cols + 1] = i;
          }
          ++cols;
          st = i + 1;
          if (i == b1) break;
        }
      }
      if (cols != nf) {
        first_bad[t] = l;
        first_cols[t] = cols;
        return;  // later lines of this chunk cannot be reported first
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < th; ++t) {
    const int64_t l0 = n_lines * t / th, l1 = n_lines * (t + 1) / th;
    if (th == 1)
      split(t, l0, l1);
    else
      pool.emplace_back(split, t, l0, l1);
  }
  for (auto& t : pool) t.join();
  for (int t = 0; t < th; ++t)
    if (first_bad[t] >= 0) {
      *bad_line = first_bad[t];
      *bad_cols = first_cols[t];
      return 3;
    }
  return encode_spans(v, kind, n_lines, blob, span.data(), max_len, n_threads, ids_out, ids_cap,
                      seq_off);
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
