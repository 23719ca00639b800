// Dataset files: the reference's text edge list and its
// SGNF / SGNL / SGNS binary files (dataset.cpp:152-280), read and written
// byte-compatibly, with the reference's validation order and messages
// (std::invalid_argument there, GGB_EINVAL here). The edge list is parsed on
// all host threads: the file is cut at line boundaries, every chunk parsed on
// its own, and the first error in file order is the one reported, as the
// reference's sequential reader would.
#include <algorithm>
#include <cctype>
#include <cstring>
#include <fstream>
#include <limits>
#include <thread>

#include "dsio.hpp"

namespace ggb {
namespace {

[[noreturn]] void input_error(const std::string& msg) { fail(GGB_EINVAL, msg); }

void read_exact(std::ifstream& f, void* p, size_t len, const std::string& path, const char* what) {
  f.read(static_cast<char*>(p), static_cast<std::streamsize>(len));
  if (static_cast<size_t>(f.gcount()) != len)
    input_error(path + ": truncated while reading " + what + " at offset " +
                std::to_string(static_cast<long long>(f.tellg())));
}

void check_magic(std::ifstream& f, const char expect[4], const std::string& path) {
  char magic[4];
  read_exact(f, magic, 4, path, "magic");
  if (std::memcmp(magic, expect, 4) != 0)
    input_error(path + ": magic mismatch at offset 0, expected " + std::string(expect, 4));
}

uint64_t read_u64(std::ifstream& f, const std::string& path, const char* what) {
  uint64_t v;
  read_exact(f, &v, sizeof v, path, what);
  return v;
}

void write_exact(std::ofstream& f, const void* p, size_t len) {
  f.write(static_cast<const char*>(p), static_cast<std::streamsize>(len));
}

// operator>>(int64_t) on [p, e): whitespace, optional sign, decimal digits;
// false (stream failure) on no digits or overflow
bool parse_i64(const char*& p, const char* e, int64_t& out) {
  while (p < e && std::isspace(static_cast<unsigned char>(*p))) ++p;
  const char* q = p;
  bool neg = false;
  if (q < e && (*q == '+' || *q == '-')) neg = *q++ == '-';
  if (q >= e || !std::isdigit(static_cast<unsigned char>(*q))) return false;
  uint64_t v = 0;
  const uint64_t lim = neg ? uint64_t{1} << 63 : static_cast<uint64_t>(std::numeric_limits<int64_t>::max());
  bool over = false;
  while (q < e && std::isdigit(static_cast<unsigned char>(*q))) {
    const uint64_t d = static_cast<uint64_t>(*q++ - '0');
    if (v > (lim - d) / 10) over = true;
    if (!over) v = v * 10 + d;
  }
  p = q;
  if (over) return false;
  out = neg ? static_cast<int64_t>(0 - v) : static_cast<int64_t>(v);
  return true;
}

struct ChunkResult {
  std::vector<int64_t> uv;
  int64_t max_id = -1;
  int64_t lines = 0;
  int64_t err_line = -1;  // local line number of the first error
  std::string err;
};

void parse_chunk(const char* b, const char* e, ChunkResult& r) {
  const char* p = b;
  while (p < e) {
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
    const char* le = nl ? nl : e;
    ++r.lines;
    const char* hash = static_cast<const char*>(std::memchr(p, '#', static_cast<size_t>(le - p)));
    const char* ce = hash ? hash : le;
    const char* q = p;
    int64_t u, v;
    if (parse_i64(q, ce, u)) {  // else: blank or comment-only line
      if (!parse_i64(q, ce, v)) {
        r.err_line = r.lines;
        r.err = "expected 'u v'";
        return;
      }
      if (u < 0 || v < 0) {
        r.err_line = r.lines;
        r.err = "negative vertex id";
        return;
      }
      r.uv.push_back(u);
      r.uv.push_back(v);
      r.max_id = std::max({r.max_id, u, v});
    }
    p = nl ? nl + 1 : e;
  }
}

}  // namespace

// load_edge_list (dataset.cpp:152-176)
std::vector<int64_t> read_edge_list(const std::string& path, int64_t* n_out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) input_error(path + ": cannot open");
  f.seekg(0, std::ios::end);
  const std::streamoff size = f.tellg();
  f.seekg(0, std::ios::beg);
  std::string buf(static_cast<size_t>(std::max<std::streamoff>(size, 0)), '\0');
  if (size > 0) f.read(buf.data(), size);
  const char* base = buf.data();
  const char* end = base + buf.size();
  const int T = static_cast<int>(std::max(1u, std::min(std::thread::hardware_concurrency(), 32u)));
  const int chunks = buf.size() < (size_t{1} << 22) ? 1 : T;
  std::vector<const char*> cut(static_cast<size_t>(chunks) + 1, end);
  cut[0] = base;
  for (int c = 1; c < chunks; ++c) {
    const char* p = std::max(cut[c - 1], base + buf.size() * c / chunks);
    const char* nl = p < end ? static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p))) : nullptr;
    cut[c] = nl ? nl + 1 : end;
  }
  std::vector<ChunkResult> res(static_cast<size_t>(chunks));
  {
    std::vector<std::thread> th;
    for (int c = 0; c < chunks; ++c) th.emplace_back([&, c] { parse_chunk(cut[c], cut[c + 1], res[c]); });
    for (auto& t : th) t.join();
  }
  int64_t line0 = 0, total = 0, max_id = -1;
  for (auto& r : res) {
    if (r.err_line >= 0) input_error(path + ": line " + std::to_string(line0 + r.err_line) + ": " + r.err);
    line0 += r.lines;
    total += static_cast<int64_t>(r.uv.size());
    max_id = std::max(max_id, r.max_id);
  }
  std::vector<int64_t> uv;
  uv.reserve(static_cast<size_t>(total));
  for (auto& r : res) uv.insert(uv.end(), r.uv.begin(), r.uv.end());
  if (n_out) *n_out = max_id + 1;
  return uv;
}

// load_dataset (dataset.cpp:178-239): features, labels, split, then the edges
HostDataset load_dataset(const std::string& graph_path, const std::string& feature_path,
                         const std::string& label_path, const std::string& split_path, std::vector<int64_t>* uv_out) {
  HostDataset ds;
  {
    std::ifstream f(feature_path, std::ios::binary);
    if (!f) input_error(feature_path + ": cannot open");
    check_magic(f, "SGNF", feature_path);
    ds.n = static_cast<int64_t>(read_u64(f, feature_path, "n"));
    ds.d_in = static_cast<int64_t>(read_u64(f, feature_path, "d_in"));
    ds.features.resize(static_cast<size_t>(ds.n) * static_cast<size_t>(ds.d_in));
    read_exact(f, ds.features.data(), ds.features.size() * sizeof(float), feature_path, "feature rows");
  }
  {
    std::ifstream f(label_path, std::ios::binary);
    if (!f) input_error(label_path + ": cannot open");
    check_magic(f, "SGNL", label_path);
    const auto n = static_cast<int64_t>(read_u64(f, label_path, "n"));
    if (n != ds.n)
      input_error(label_path + ": length mismatch, n=" + std::to_string(n) + " vs features n=" + std::to_string(ds.n));
    ds.n_classes = static_cast<int64_t>(read_u64(f, label_path, "n_classes"));
    ds.labels.resize(static_cast<size_t>(n));
    read_exact(f, ds.labels.data(), ds.labels.size() * sizeof(int32_t), label_path, "class ids");
    for (int64_t v = 0; v < n; ++v) {
      const auto c = ds.labels[static_cast<size_t>(v)];
      if (c < 0 || c >= ds.n_classes)
        input_error(label_path + ": class id out of range at offset " + std::to_string(20 + v * 4));
    }
  }
  {
    std::ifstream f(split_path, std::ios::binary);
    if (!f) input_error(split_path + ": cannot open");
    check_magic(f, "SGNS", split_path);
    const auto n = static_cast<int64_t>(read_u64(f, split_path, "n"));
    if (n != ds.n) input_error(split_path + ": length mismatch, n=" + std::to_string(n));
    ds.split.resize(static_cast<size_t>(n));
    read_exact(f, ds.split.data(), ds.split.size(), split_path, "split tags");
    for (int64_t v = 0; v < n; ++v)
      if (ds.split[static_cast<size_t>(v)] > 3)
        input_error(split_path + ": invalid split tag at offset " + std::to_string(12 + v));
  }
  std::vector<int64_t> uv = read_edge_list(graph_path, nullptr);
  for (size_t k = 0; k < uv.size(); ++k)
    if (uv[k] >= ds.n) input_error(graph_path + ": vertex id >= n=" + std::to_string(ds.n));
  ds.adj = normalize_adjacency(uv.data(), static_cast<int64_t>(uv.size() / 2), ds.n);
  if (uv_out) *uv_out = std::move(uv);
  return ds;
}

// save_edge_list / save_features / save_labels / save_split (dataset.cpp:241-280)
void save_edge_list(const std::string& path, const int64_t* uv, int64_t m) {
  std::ofstream f(path, std::ios::binary);
  if (!f) input_error(path + ": cannot open for writing");
  std::string out;
  out.reserve(static_cast<size_t>(std::min<int64_t>(m, int64_t{1} << 24)) * 16);
  char tmp[48];
  for (int64_t e = 0; e < m; ++e) {
    const int len = std::snprintf(tmp, sizeof tmp, "%lld %lld\n", static_cast<long long>(uv[2 * e]),
                                  static_cast<long long>(uv[2 * e + 1]));
    out.append(tmp, static_cast<size_t>(len));
    if (out.size() > (size_t{1} << 26)) {
      write_exact(f, out.data(), out.size());
      out.clear();
    }
  }
  write_exact(f, out.data(), out.size());
}

void save_features(const std::string& path, int64_t n, int64_t d_in, const float* features) {
  std::ofstream f(path, std::ios::binary);
  if (!f) input_error(path + ": cannot open for writing");
  write_exact(f, "SGNF", 4);
  const auto un = static_cast<uint64_t>(n), ud = static_cast<uint64_t>(d_in);
  write_exact(f, &un, 8);
  write_exact(f, &ud, 8);
  write_exact(f, features, static_cast<size_t>(n) * static_cast<size_t>(d_in) * sizeof(float));
}

void save_labels(const std::string& path, int64_t n, int64_t n_classes, const int32_t* labels) {
  std::ofstream f(path, std::ios::binary);
  if (!f) input_error(path + ": cannot open for writing");
  write_exact(f, "SGNL", 4);
  const auto un = static_cast<uint64_t>(n), uc = static_cast<uint64_t>(n_classes);
  write_exact(f, &un, 8);
  write_exact(f, &uc, 8);
  write_exact(f, labels, static_cast<size_t>(n) * sizeof(int32_t));
}

void save_split(const std::string& path, int64_t n, const uint8_t* split) {
  std::ofstream f(path, std::ios::binary);
  if (!f) input_error(path + ": cannot open for writing");
  write_exact(f, "SGNS", 4);
  const auto un = static_cast<uint64_t>(n);
  write_exact(f, &un, 8);
  write_exact(f, split, static_cast<size_t>(n));
}

}  // namespace ggb
