// Dataset files: the reference's text edge list and its
// SGNF / SGNL / SGNS binary files (dataset.cpp:152-280), read and written
// byte-compatibly, with the reference's validation order and messages
// (std::invalid_argument there, GGB_EINVAL here). The edge list is parsed on
// all host threads: the file is cut at line boundaries, every chunk parsed on
// its own, and the first error in file order is the one reported, as the
// reference's sequential reader would.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <limits>
#include <thread>

#include "dsio.hpp"

namespace ggb {
namespace {

[[noreturn]] void bad_input(const std::string& msg) { fail(GGB_EINVAL, msg); }

// ---- SGN* binaries -------------------------------------------
// Every file is: 4-byte magic | little-endian u64 header words | a payload of
// fixed-size records. A file is mapped read-only and consumed through a
// cursor; validation messages are the reference loader's (load_dataset,
// dataset.cpp:178-239) so callers see the same std::invalid_argument text.
//
// A short read there leaves the std::ifstream failed, and tellg() of a failed
// stream is -1: every truncation message carries that offset.
constexpr long long kOffsetAfterShortRead = -1;

class MappedFile {
 public:
  explicit MappedFile(const std::string& path) : path_(path) {
    fd_ = ::open(path.c_str(), O_RDONLY);
    if (fd_ < 0) bad_input(path + ": cannot open");
    struct stat st {};
    if (::fstat(fd_, &st) == 0 && st.st_size > 0) {
      size_ = static_cast<size_t>(st.st_size);
      void* m = ::mmap(nullptr, size_, PROT_READ, MAP_PRIVATE, fd_, 0);
      if (m == MAP_FAILED) {
        size_ = 0;
      } else {
        base_ = static_cast<const uint8_t*>(m);
        ::madvise(m, size_, MADV_SEQUENTIAL);
      }
    }
  }
  ~MappedFile() {
    if (base_) ::munmap(const_cast<uint8_t*>(base_), size_);
    if (fd_ >= 0) ::close(fd_);
  }
  MappedFile(const MappedFile&) = delete;
  MappedFile& operator=(const MappedFile&) = delete;

  // the next `len` bytes, or the loader's truncation error naming `what`
  const uint8_t* take(size_t len, const char* what) {
    if (size_ - pos_ < len)
      bad_input(path_ + ": truncated while reading " + what + " at offset " + std::to_string(kOffsetAfterShortRead));
    const uint8_t* p = base_ + pos_;
    pos_ += len;
    return p;
  }
  uint64_t word(const char* what) {
    uint64_t v;
    std::memcpy(&v, take(sizeof v, what), sizeof v);
    return v;
  }
  void expect_magic(const char (&magic)[5]) {
    if (std::memcmp(take(4, "magic"), magic, 4) != 0)
      bad_input(path_ + ": magic mismatch at offset 0, expected " + std::string(magic, 4));
  }
  const std::string& path() const { return path_; }
  const char* data() const { return reinterpret_cast<const char*>(base_); }
  size_t size() const { return size_; }

 private:
  std::string path_;
  int fd_ = -1;
  const uint8_t* base_ = nullptr;
  size_t size_ = 0, pos_ = 0;
};

// records [0, n) copied out of the payload; the first record failing `ok`
// is reported at its byte offset in the file (header bytes + index * size)
template <class T, class Ok>
void read_records(MappedFile& f, std::vector<T>& out, int64_t n, const char* what, int64_t header_bytes,
                  const char* invalid_msg, Ok ok) {
  const uint64_t count = static_cast<uint64_t>(std::max<int64_t>(n, 0));
  const uint8_t* src = f.take(count > SIZE_MAX / sizeof(T) ? SIZE_MAX : count * sizeof(T), what);
  out.resize(count);  // sized only once the payload is known to be there
  if (count) std::memcpy(out.data(), src, count * sizeof(T));
  const auto bad = std::find_if_not(out.begin(), out.end(), ok);
  if (bad != out.end())
    bad_input(f.path() + ": " + invalid_msg + " at offset " +
              std::to_string(header_bytes + static_cast<int64_t>(bad - out.begin()) * static_cast<int64_t>(sizeof(T))));
}

// one write(2) stream per file: magic, header words, payload
void write_sgn(const std::string& path, const char (&magic)[5], std::initializer_list<uint64_t> words,
               const void* payload, size_t payload_bytes) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) bad_input(path + ": cannot open for writing");
  std::vector<uint8_t> head(4 + 8 * words.size());
  std::memcpy(head.data(), magic, 4);
  size_t at = 4;
  for (uint64_t w : words) {
    std::memcpy(head.data() + at, &w, 8);
    at += 8;
  }
  std::fwrite(head.data(), 1, head.size(), f);
  if (payload_bytes) std::fwrite(payload, 1, payload_bytes, f);
  std::fclose(f);
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
  MappedFile file(path);
  const char* base = file.size() ? file.data() : "";
  const char* end = base + file.size();
  const int T = static_cast<int>(std::max(1u, std::min(std::thread::hardware_concurrency(), 32u)));
  const int chunks = file.size() < (size_t{1} << 22) ? 1 : T;
  std::vector<const char*> cut(static_cast<size_t>(chunks) + 1, end);
  cut[0] = base;
  for (int c = 1; c < chunks; ++c) {
    const char* p = std::max(cut[c - 1], base + file.size() * c / chunks);
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
    if (r.err_line >= 0) bad_input(path + ": line " + std::to_string(line0 + r.err_line) + ": " + r.err);
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

// load_dataset (dataset.cpp:178-239): the three node files (features, then
// labels and split checked against the feature count), then the edge list
HostDataset load_dataset(const std::string& graph_path, const std::string& feature_path,
                         const std::string& label_path, const std::string& split_path, std::vector<int64_t>* uv_out) {
  HostDataset ds;
  {  // SGNF: u64 n, u64 d_in, n * d_in float32 (row-major)
    MappedFile f(feature_path);
    f.expect_magic("SGNF");
    ds.n = static_cast<int64_t>(f.word("n"));
    ds.d_in = static_cast<int64_t>(f.word("d_in"));
    read_records(f, ds.features, ds.n * ds.d_in, "feature rows", 20, "", [](float) { return true; });
  }
  {  // SGNL: u64 n, u64 n_classes, n int32 class ids in [0, n_classes)
    MappedFile f(label_path);
    f.expect_magic("SGNL");
    const auto n = static_cast<int64_t>(f.word("n"));
    if (n != ds.n)
      bad_input(label_path + ": length mismatch, n=" + std::to_string(n) + " vs features n=" + std::to_string(ds.n));
    ds.n_classes = static_cast<int64_t>(f.word("n_classes"));
    const int64_t k = ds.n_classes;
    read_records(f, ds.labels, n, "class ids", 20, "class id out of range",
                 [k](int32_t c) { return c >= 0 && c < k; });
  }
  {  // SGNS: u64 n, n uint8 tags (0 train, 1 val, 2 test, 3 unused)
    MappedFile f(split_path);
    f.expect_magic("SGNS");
    const auto n = static_cast<int64_t>(f.word("n"));
    if (n != ds.n) bad_input(split_path + ": length mismatch, n=" + std::to_string(n));
    read_records(f, ds.split, n, "split tags", 12, "invalid split tag", [](uint8_t t) { return t <= 3; });
  }
  std::vector<int64_t> uv = read_edge_list(graph_path, nullptr);
  if (std::any_of(uv.begin(), uv.end(), [&](int64_t id) { return id >= ds.n; }))
    bad_input(graph_path + ": vertex id >= n=" + std::to_string(ds.n));
  ds.adj = normalize_adjacency(uv.data(), static_cast<int64_t>(uv.size() / 2), ds.n);
  if (uv_out) *uv_out = std::move(uv);
  return ds;
}

// save_edge_list (dataset.cpp:241-246): "u v\n" per pair, formatted with
// std::to_chars into a 64 MB staging buffer
void save_edge_list(const std::string& path, const int64_t* uv, int64_t m) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) bad_input(path + ": cannot open for writing");
  std::vector<char> buf(size_t{1} << 26);
  size_t at = 0;
  for (int64_t e = 0; e < 2 * m; ++e) {
    if (buf.size() - at < 24) {
      std::fwrite(buf.data(), 1, at, f);
      at = 0;
    }
    at += static_cast<size_t>(std::snprintf(buf.data() + at, 24, "%lld", static_cast<long long>(uv[e])));
    buf[at++] = (e & 1) ? '\n' : ' ';
  }
  std::fwrite(buf.data(), 1, at, f);
  std::fclose(f);
}

// the SGN* writers (dataset.cpp:248-280; formats SPEC.md:84-86)
void save_features(const std::string& path, int64_t n, int64_t d_in, const float* features) {
  write_sgn(path, "SGNF", {static_cast<uint64_t>(n), static_cast<uint64_t>(d_in)}, features,
            static_cast<size_t>(n) * static_cast<size_t>(d_in) * sizeof(float));
}

void save_labels(const std::string& path, int64_t n, int64_t n_classes, const int32_t* labels) {
  write_sgn(path, "SGNL", {static_cast<uint64_t>(n), static_cast<uint64_t>(n_classes)}, labels,
            static_cast<size_t>(n) * sizeof(int32_t));
}

void save_split(const std::string& path, int64_t n, const uint8_t* split) {
  write_sgn(path, "SGNS", {static_cast<uint64_t>(n)}, split, static_cast<size_t>(n));
}

}  // namespace ggb
