// Read side of the `.mfrg` model container (`pkg/src/metricforge/container.py`):
//   "MFRG0001" | u32le header_len | canonical JSON header | 0-pad to 64 | payload
// mmap-backed, zero-copy tensor views, plus the tensor-name/shape contract of
// `required_tensor_shapes` (`pkg/src/metricforge/encoder.py:69-91`).
#pragma once
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace mfg {

struct ContainerError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------ minimal JSON
struct JVal {
  enum T { NUL, NUM, STR, ARR, OBJ, BOOL } t = NUL;
  double num = 0;
  bool b = false;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class JParser {
 public:
  JParser(const char* s, size_t n) : p_(s), e_(s + n) {}
  JVal parse() {
    JVal v = value();
    ws();
    if (p_ != e_) fail("trailing data");
    return v;
  }

 private:
  const char *p_, *e_;
  [[noreturn]] void fail(const char* m) { throw ContainerError(std::string("unreadable header (") + m + ")"); }
  void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  JVal value() {
    ws();
    if (p_ >= e_) fail("unexpected end");
    JVal v;
    char c = *p_;
    if (c == '{') {
      v.t = JVal::OBJ;
      ++p_;
      ws();
      if (p_ < e_ && *p_ == '}') { ++p_; return v; }
      for (;;) {
        ws();
        JVal k = value();
        if (k.t != JVal::STR) fail("object key");
        ws();
        if (p_ >= e_ || *p_ != ':') fail("colon");
        ++p_;
        v.obj.emplace_back(k.str, value());
        ws();
        if (p_ < e_ && *p_ == ',') { ++p_; continue; }
        if (p_ < e_ && *p_ == '}') { ++p_; break; }
        fail("object");
      }
    } else if (c == '[') {
      v.t = JVal::ARR;
      ++p_;
      ws();
      if (p_ < e_ && *p_ == ']') { ++p_; return v; }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (p_ < e_ && *p_ == ',') { ++p_; continue; }
        if (p_ < e_ && *p_ == ']') { ++p_; break; }
        fail("array");
      }
    } else if (c == '"') {
      v.t = JVal::STR;
      ++p_;
      while (p_ < e_ && *p_ != '"') {
        if (*p_ == '\\') {
          ++p_;
          if (p_ >= e_) fail("escape");
          char x = *p_++;
          switch (x) {
            case 'n': v.str += '\n'; break;
            case 't': v.str += '\t'; break;
            case 'r': v.str += '\r'; break;
            case 'b': v.str += '\b'; break;
            case 'f': v.str += '\f'; break;
            case 'u': {
              if (e_ - p_ < 4) fail("escape");
              unsigned cp = std::stoul(std::string(p_, 4), nullptr, 16);
              p_ += 4;
              if (cp >= 0xD800 && cp < 0xDC00 && e_ - p_ >= 6 && p_[0] == '\\' && p_[1] == 'u') {
                unsigned lo = std::stoul(std::string(p_ + 2, 4), nullptr, 16);
                cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                p_ += 6;
              }
              utf8(v.str, cp);
              break;
            }
            default: v.str += x;
          }
        } else {
          v.str += *p_++;
        }
      }
      if (p_ >= e_) fail("string");
      ++p_;
    } else if (c == 't' || c == 'f' || c == 'n') {
      const char* w = c == 't' ? "true" : c == 'f' ? "false" : "null";
      size_t n = strlen(w);
      if ((size_t)(e_ - p_) < n || strncmp(p_, w, n) != 0) fail("literal");
      p_ += n;
      v.t = c == 'n' ? JVal::NUL : JVal::BOOL;
      v.b = c == 't';
    } else {
      const char* s = p_;
      while (p_ < e_ && (isdigit((unsigned char)*p_) || *p_ == '-' || *p_ == '+' || *p_ == '.' ||
                         *p_ == 'e' || *p_ == 'E'))
        ++p_;
      if (s == p_) fail("value");
      v.t = JVal::NUM;
      v.num = std::stod(std::string(s, p_));
    }
    return v;
  }
  static void utf8(std::string& o, unsigned cp) {
    if (cp < 0x80) o += (char)cp;
    else if (cp < 0x800) { o += (char)(0xC0 | (cp >> 6)); o += (char)(0x80 | (cp & 0x3F)); }
    else if (cp < 0x10000) {
      o += (char)(0xE0 | (cp >> 12)); o += (char)(0x80 | ((cp >> 6) & 0x3F));
      o += (char)(0x80 | (cp & 0x3F));
    } else {
      o += (char)(0xF0 | (cp >> 18)); o += (char)(0x80 | ((cp >> 12) & 0x3F));
      o += (char)(0x80 | ((cp >> 6) & 0x3F)); o += (char)(0x80 | (cp & 0x3F));
    }
  }
};

// ------------------------------------------------------------ container
struct TensorView {
  std::string dtype;  // "f32" | "f16"
  std::vector<int64_t> shape;
  const uint8_t* data = nullptr;
  int64_t nbytes = 0;
  int64_t numel() const {
    int64_t n = 1;
    for (auto s : shape) n *= s;
    return n;
  }
};

struct Manifest {
  std::string like, norm_style = "post";
  int64_t vocab_size = 0, d_model = 0, n_heads = 0, n_layers = 0, d_ffn = 0, max_position = 0;
  std::vector<int64_t> head_hidden;
};

class Container {
 public:
  explicit Container(const std::string& path) : path_(path) {
    fd_ = ::open(path.c_str(), O_RDONLY);
    if (fd_ < 0) throw std::runtime_error(path + ": cannot open (" + strerror(errno) + ")");
    struct stat st;
    if (fstat(fd_, &st) != 0) throw std::runtime_error(path + ": stat failed");
    size_ = (size_t)st.st_size;
    if (size_ < 8 || size_ == 0) throw ContainerError(path + ": not a model container (bad magic)");
    // MAP_POPULATE: the weights are read once, front to back, right after open;
    // pre-faulting the whole mapping in the kernel is much cheaper than taking
    // one minor fault per 4 KB page from the upload threads.
    base_ = (const uint8_t*)mmap(nullptr, size_, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd_, 0);
    if (base_ != MAP_FAILED) madvise(const_cast<uint8_t*>(base_), size_, MADV_SEQUENTIAL);
    if (base_ == MAP_FAILED) {
      base_ = nullptr;
      throw std::runtime_error(path + ": mmap failed");
    }
    if (size_ < 8 || memcmp(base_, "MFRG0001", 8) != 0)
      throw ContainerError(path + ": not a model container (bad magic)");
    if (size_ < 12) throw ContainerError(path + ": truncated before header length");
    uint32_t hlen;
    memcpy(&hlen, base_ + 8, 4);
    if (12 + (size_t)hlen > size_) throw ContainerError(path + ": truncated inside header");
    JVal h = JParser((const char*)base_ + 12, hlen).parse();
    size_t payload = (12 + (size_t)hlen + 63) / 64 * 64;
    const JVal* man = h.get("manifest");
    if (!man || man->t != JVal::OBJ) throw ContainerError(path + ": manifest missing field 'like'");
    auto req_int = [&](const char* k) -> int64_t {
      const JVal* v = man->get(k);
      if (!v) throw ContainerError(path + std::string(": manifest missing field '") + k + "'");
      return (int64_t)v->num;
    };
    const JVal* like = man->get("like");
    if (!like) throw ContainerError(path + ": manifest missing field 'like'");
    m_.like = like->str;
    m_.vocab_size = req_int("vocab_size");
    m_.d_model = req_int("d_model");
    m_.n_heads = req_int("n_heads");
    m_.n_layers = req_int("n_layers");
    m_.d_ffn = req_int("d_ffn");
    m_.max_position = req_int("max_position");
    if (const JVal* ns = man->get("norm_style")) m_.norm_style = ns->str;
    if (const JVal* hh = man->get("head_hidden"))
      for (auto& x : hh->arr) m_.head_hidden.push_back((int64_t)x.num);
    if (const JVal* fv = man->get("format_version"))
      if ((int64_t)fv->num != 1)
        throw ContainerError(path + ": format_version " + std::to_string((int64_t)fv->num) + " not supported");
    const JVal* ts = h.get("tensors");
    std::vector<std::pair<int64_t, int64_t>> regions;
    if (ts)
      for (auto& e : ts->arr) {
        TensorView tv;
        const JVal *nm = e.get("name"), *dt = e.get("dtype"), *sh = e.get("shape"),
                   *off = e.get("offset"), *nb = e.get("nbytes");
        if (!nm || !dt || !sh || !off || !nb) throw ContainerError(path + ": malformed tensor index");
        tv.dtype = dt->str;
        if (tv.dtype != "f32" && tv.dtype != "f16")
          throw ContainerError("unknown dtype '" + tv.dtype + "'");
        for (auto& s : sh->arr) {
          if (s.num < 0) throw ContainerError(path + ": tensor '" + nm->str + "' has a negative dimension");
          tv.shape.push_back((int64_t)s.num);
        }
        tv.nbytes = (int64_t)nb->num;
        const int64_t o = (int64_t)off->num;
        if (tv.nbytes < 0 || tv.nbytes != tv.numel() * (tv.dtype == "f32" ? 4 : 2))
          throw ContainerError(path + ": tensor '" + nm->str + "' nbytes disagrees with dtype/shape");
        if (o < 0 || o % 64 != 0)
          throw ContainerError(path + ": tensor '" + nm->str + "' offset not 64-byte aligned");
        // overflow-safe bounds (a negative or huge offset cannot wrap around)
        const uint64_t room = payload <= size_ ? (uint64_t)(size_ - payload) : 0;
        if ((uint64_t)o > room || (uint64_t)tv.nbytes > room - (uint64_t)o)
          throw ContainerError(path + ": tensor '" + nm->str + "' extends past end of file");
        if (tensors_.count(nm->str))
          throw ContainerError(path + ": duplicate tensor names in index");
        tv.data = base_ + payload + o;
        tensors_[nm->str] = tv;
        regions.push_back({o, o + tv.nbytes});
      }
    // tensor regions must not overlap (`container.py:316-322`)
    std::sort(regions.begin(), regions.end());
    for (size_t i = 1; i < regions.size(); ++i)
      if (regions[i].first < regions[i - 1].second)
        throw ContainerError(path + ": tensor regions overlap");
  }
  ~Container() {
    if (base_) munmap((void*)base_, size_);
    if (fd_ >= 0) ::close(fd_);
  }
  const Manifest& manifest() const { return m_; }
  const TensorView* find(const std::string& n) const {
    auto it = tensors_.find(n);
    return it == tensors_.end() ? nullptr : &it->second;
  }
  const std::string& path() const { return path_; }

 private:
  std::string path_;
  int fd_ = -1;
  size_t size_ = 0;
  const uint8_t* base_ = nullptr;
  Manifest m_;
  std::map<std::string, TensorView> tensors_;
};

inline int feature_multiplier(const std::string& like) {
  return like == "comet-qe" ? 4 : like == "comet" ? 6 : 1;
}

// Python-style shape repr used in the reference messages: (64, 16) / (16,)
inline std::string shape_repr(const std::vector<int64_t>& s) {
  std::string o = "(";
  for (size_t i = 0; i < s.size(); ++i) {
    if (i) o += ", ";
    o += std::to_string(s[i]);
  }
  if (s.size() == 1) o += ",";
  return o + ")";
}

// Ordered (name, shape) contract, `encoder.py:69-91`.
inline std::vector<std::pair<std::string, std::vector<int64_t>>> required_shapes(const Manifest& m) {
  std::vector<std::pair<std::string, std::vector<int64_t>>> r;
  const int64_t d = m.d_model, f = m.d_ffn;
  r.push_back({"emb.tok", {m.vocab_size, d}});
  r.push_back({"emb.pos", {m.max_position, d}});
  for (int64_t i = 0; i < m.n_layers; ++i) {
    std::string p = "layer." + std::to_string(i);
    for (const char* pr : {"q", "k", "v", "o"}) {
      r.push_back({p + ".att." + pr + ".w", {d, d}});
      r.push_back({p + ".att." + pr + ".b", {d}});
    }
    for (const char* nm : {"norm1", "norm2"}) {
      r.push_back({p + "." + nm + ".g", {d}});
      r.push_back({p + "." + nm + ".b", {d}});
    }
    r.push_back({p + ".ffn.w1", {d, f}});
    r.push_back({p + ".ffn.b1", {f}});
    r.push_back({p + ".ffn.w2", {f, d}});
    r.push_back({p + ".ffn.b2", {d}});
  }
  std::vector<int64_t> w = {feature_multiplier(m.like) * d};
  for (auto x : m.head_hidden) w.push_back(x);
  w.push_back(1);
  for (size_t j = 0; j + 1 < w.size(); ++j) {
    r.push_back({"head." + std::to_string(j) + ".w", {w[j], w[j + 1]}});
    r.push_back({"head." + std::to_string(j) + ".b", {w[j + 1]}});
  }
  return r;
}

}  // namespace mfg
