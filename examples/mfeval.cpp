// mfeval — the scoring path driven from C++ only, through the two C-ABIs a
// non-Python host binds (include/mfhost.h, include/mfgpu.h). It is what the
// reference's `metricforge-eval --stdin --stdin-file FILE` does
// (pkg/src/metricforge/cli.py:145-184 -> Evaluator.evaluate_lines,
// evaluate.py:179-206): per window of mini_batch * maxi_batch_factor lines,
//   mfh_encode_tsv  (column split + checks + encode_fields)
//   mfh_plan        (length-sorted mini-batch plan)
//   mfh_pack_roles  (role-major varlen packing)
//   mfg_score_batch (device forward + head)
// then the inverse permutation, and one "%.Nf" line per record. Its output is
// byte-identical to the Python CLI's (tests/test_gpu_examples.py).
//
//   mfeval MODEL.mfrg VOCAB.txt INPUT.tsv [--precision N] [--gpu-precision fp32|bf16|bf16x3|fp16]
//          [--max-len N] [--mini-batch N] [--maxi-batch N] [--device N]
//
// Exit codes as the CLI (cli.py:40-47): 0 ok, 1 runtime, 2 usage / input.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string_view>
#include <unordered_set>
#include <vector>

#include "mfgpu.h"
#include "mfhost.h"

namespace {

const char* PROG = "mfeval";

int fail(int code, const std::string& msg) {
  std::fprintf(stderr, "%s: error: %s\n", PROG, msg.c_str());
  return code;
}

bool read_file(const char* path, std::string& out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  char buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) out.append(buf, n);
  std::fclose(f);
  return true;
}

// Python text mode (universal newlines): "\r\n" and "\r" read as "\n".
std::string universal_newlines(const std::string& s) {
  std::string o;
  o.reserve(s.size());
  for (size_t i = 0; i < s.size(); ++i) {
    if (s[i] == '\r') {
      o.push_back('\n');
      if (i + 1 < s.size() && s[i + 1] == '\n') ++i;
    } else {
      o.push_back(s[i]);
    }
  }
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr,
                 "usage: %s MODEL.mfrg VOCAB.txt INPUT.tsv [--precision N] "
                 "[--gpu-precision fp32|bf16|bf16x3|fp16] [--max-len N] [--mini-batch N] "
                 "[--maxi-batch N] [--device N]\n",
                 PROG);
    return 2;
  }
  int digits = 4, max_len = 512, mini_batch = 128, maxi_batch = 8, device = 0;
  int32_t prec = MFG_PREC_FP32;
  for (int i = 4; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> const char* {
      if (i + 1 >= argc) std::exit(fail(2, "missing value for " + a));
      return argv[++i];
    };
    if (a == "--precision") digits = std::atoi(val());
    else if (a == "--max-len") max_len = std::atoi(val());
    else if (a == "--mini-batch") mini_batch = std::atoi(val());
    else if (a == "--maxi-batch") maxi_batch = std::atoi(val());
    else if (a == "--device") device = std::atoi(val());
    else if (a == "--gpu-precision") {
      const std::string p = val();
      if (p == "fp32") prec = MFG_PREC_FP32;
      else if (p == "bf16") prec = MFG_PREC_BF16;
      else if (p == "bf16x3") prec = MFG_PREC_BF16X3;
      else if (p == "fp16") prec = MFG_PREC_FP16;
      else return fail(2, "unknown --gpu-precision " + p);
    } else {
      return fail(2, "unknown argument " + a);
    }
  }
  if (mini_batch < 1 || maxi_batch < 1) return fail(2, "batch sizes must be >= 1");

  // ---- vocabulary (load_vocab: universal newlines, split on "\n", drop one trailing "")
  std::string vtext;
  if (!read_file(argv[2], vtext)) return fail(1, std::string("cannot read ") + argv[2]);
  vtext = universal_newlines(vtext);
  std::vector<std::string_view> toks;
  for (size_t st = 0;;) {
    const size_t nl = vtext.find('\n', st);
    toks.emplace_back(vtext.data() + st, (nl == std::string::npos ? vtext.size() : nl) - st);
    if (nl == std::string::npos) break;
    st = nl + 1;
  }
  if (!toks.empty() && toks.back().empty()) toks.pop_back();
  if (toks.empty()) return fail(1, std::string(argv[2]) + ": empty vocabulary file");
  const char* specials[5] = {"<pad>", "<unk>", "<s>", "</s>", "<sep>"};
  std::unordered_set<std::string_view> seen;
  for (size_t i = 0; i < toks.size(); ++i) {
    if (toks[i].empty()) return fail(1, "empty token at line " + std::to_string(i + 1));
    if (!seen.insert(toks[i]).second)
      return fail(1, "duplicate token at line " + std::to_string(i + 1));
    if (i < 5 && toks[i] != specials[i]) return fail(1, "first five tokens must be the specials");
  }
  if (toks.size() < 5) return fail(1, "first five tokens must be the specials");
  std::string vblob;
  for (size_t i = 0; i < toks.size(); ++i) {
    if (i) vblob.push_back('\n');
    vblob.append(toks[i]);
  }
  mfh_vocab* vocab = nullptr;
  if (mfh_vocab_create(vblob.data(), (int64_t)vblob.size(), (int32_t)toks.size(), &vocab) != 0)
    return fail(1, "vocabulary construction failed");

  // ---- model
  mfg_config cfg{};
  cfg.container_path = argv[1];
  cfg.device = device;
  cfg.precision = prec;
  mfg_ctx* ctx = nullptr;
  if (mfg_create(&cfg, &ctx) != MFG_OK) {
    int32_t code = 1;
    char msg[1024];
    mfg_last_error(nullptr, &code, msg, sizeof msg);
    return fail(code == MFG_ERR_USAGE ? 2 : 1, msg);
  }
  mfg_model_info info{};
  mfg_get_model_info(ctx, &info);
  const int n_roles = info.n_roles;
  const int eff_len = max_len < info.max_position ? max_len : info.max_position;
  const int n_cols = info.kind == 1 ? 3 : 2;

  // ---- input lines (text mode; each line keeps its "\n", stripped by mfh_encode_tsv)
  std::string text;
  if (!read_file(argv[3], text)) return fail(1, std::string("cannot read ") + argv[3]);
  text = universal_newlines(text);
  std::vector<int64_t> line_off{0};
  for (size_t i = 0; i < text.size(); ++i)
    if (text[i] == '\n') line_off.push_back((int64_t)i + 1);
  if (line_off.back() != (int64_t)text.size()) line_off.push_back((int64_t)text.size());
  const int64_t n_lines = (int64_t)line_off.size() - 1;

  // ---- windows
  const int64_t window = (int64_t)mini_batch * maxi_batch;
  std::vector<float> scores(n_lines);
  std::vector<int32_t> ids, packed;
  std::vector<int64_t> seq_off, lengths, order, cu;
  std::vector<float> win_scores;
  for (int64_t w0 = 0; w0 < n_lines; w0 += window) {
    const int64_t n = (n_lines - w0 < window) ? n_lines - w0 : window;
    const int64_t* lo = line_off.data() + w0;
    std::vector<int64_t> rel(n + 1);
    for (int64_t i = 0; i <= n; ++i) rel[i] = lo[i] - lo[0];
    const int64_t cap = 2 * (rel[n]) + 4 * (int64_t)n_roles * n + 8;
    ids.resize(cap);
    seq_off.assign(n * n_roles + 1, 0);
    int64_t bad_line = -1;
    int32_t bad_cols = 0;
    const int64_t rc = mfh_encode_tsv(vocab, info.kind, text.data() + lo[0], rel.data(), n, eff_len,
                                      0, ids.data(), cap, seq_off.data(), &bad_line, &bad_cols);
    if (rc == 3)
      return fail(2, "line " + std::to_string(w0 + bad_line) + ": expected " +
                         std::to_string(n_cols) + " tab-separated columns, got " +
                         std::to_string(bad_cols));
    if (rc != 0) return fail(1, "tokenizer failed (" + std::to_string(rc) + ")");
    lengths.assign(n, 0);
    for (int64_t r = 0; r < n; ++r)
      lengths[r] = seq_off[(r + 1) * n_roles] - seq_off[r * n_roles];
    order.resize(n);
    mfh_plan(lengths.data(), n, mini_batch, maxi_batch, 1, order.data());
    packed.resize(seq_off[n * n_roles]);
    cu.resize(n * n_roles + 1);
    mfh_pack_roles(ids.data(), seq_off.data(), n_roles, order.data(), n, packed.data(), cu.data());
    win_scores.resize(n);
    if (mfg_score_batch(ctx, (int32_t)n, n_roles, packed.data(), cu.data(), win_scores.data()) !=
        MFG_OK) {
      int32_t code = 1;
      char msg[1024];
      mfg_last_error(ctx, &code, msg, sizeof msg);
      return fail(1, msg);
    }
    for (int64_t i = 0; i < n; ++i) scores[w0 + order[i]] = win_scores[i];  // restore_order
  }

  // f"{v:.{precision}f}" per record (cli.py:178-184): both are correctly rounded
  std::string out;
  char buf[64];
  for (float s : scores) {
    std::snprintf(buf, sizeof buf, "%.*f\n", digits, (double)s);
    out += buf;
  }
  std::fwrite(out.data(), 1, out.size(), stdout);
  mfg_destroy(ctx);
  mfh_vocab_destroy(vocab);
  return 0;
}
