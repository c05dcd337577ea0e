#include "soa_io.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>

namespace ffb {

namespace {

constexpr char kMagic[8] = {'F', 'F', 'S', 'O', 'A', '0', '1', '\0'};
constexpr std::uint64_t kAlign = 4096;
constexpr std::size_t kChunk = 16u << 20;  // staging chunk (bytes)

std::uint64_t round_up(std::uint64_t x, std::uint64_t a) { return (x + a - 1) / a * a; }

[[noreturn]] void io_error(const std::string& path, const std::string& what) {
  data_error(path + ": " + what + (errno ? std::string(" (") + std::strerror(errno) + ")" : ""));
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

void write_all(int fd, const void* p, std::size_t n, const std::string& path) {
  const char* c = static_cast<const char*>(p);
  while (n > 0) {
    const ssize_t w = ::write(fd, c, n);
    if (w < 0) {
      if (errno == EINTR) continue;
      io_error(path, "write failed");
    }
    c += w;
    n -= static_cast<std::size_t>(w);
  }
}

void pread_all(int fd, void* p, std::size_t n, std::uint64_t off, const std::string& path) {
  char* c = static_cast<char*>(p);
  while (n > 0) {
    const ssize_t r = ::pread(fd, c, n, static_cast<off_t>(off));
    if (r < 0) {
      if (errno == EINTR) continue;
      io_error(path, "read failed");
    }
    if (r == 0) {
      errno = 0;
      io_error(path, "truncated file");
    }
    c += r;
    off += static_cast<std::uint64_t>(r);
    n -= static_cast<std::size_t>(r);
  }
}

template <class T>
T get(const std::vector<char>& b, std::size_t at) {
  T v;
  std::memcpy(&v, b.data() + at, sizeof(T));
  return v;
}

std::uint64_t add_words(std::uint64_t acc, const char* p, std::size_t bytes) {
  for (std::size_t i = 0; i + 8 <= bytes; i += 8) {
    std::uint64_t w;
    std::memcpy(&w, p + i, 8);
    acc += w;
  }
  return acc;
}

// Pinned staging buffers are pinned once per process and reused by every load
// (pinning is far slower than the copies it enables: ~0.3 s per 512 MiB).
struct StagingPool {
  std::mutex mu;
  std::vector<char*> free;
  char* take() {
    {
      std::lock_guard<std::mutex> lk(mu);
      if (!free.empty()) {
        char* b = free.back();
        free.pop_back();
        return b;
      }
    }
    char* b = nullptr;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&b), kChunk, cudaHostAllocPortable), "cudaHostAlloc(staging)");
    return b;
  }
  void give(char* b) {
    std::lock_guard<std::mutex> lk(mu);
    free.push_back(b);
  }
};
StagingPool& staging_pool() {
  static StagingPool* p = new StagingPool();  // process lifetime (pinned memory stays registered)
  return *p;
}

}  // namespace

std::uint64_t soa_checksum(const double* col, long long n) {
  return add_words(0, reinterpret_cast<const char*>(col), static_cast<std::size_t>(n) * 8u);
}

void soa_write(const std::string& path, const std::vector<std::string>& names,
               const std::vector<const double*>& cols, long long n) {
  if (names.size() != cols.size() || names.empty()) usage_error("soa_write: names / columns mismatch");
  if (n < 0) usage_error("soa_write: negative row count");
  std::size_t hdr = 24;
  for (const std::string& s : names) hdr += 4 + s.size() + 8;
  const std::uint64_t H = round_up(hdr, kAlign);
  std::vector<char> h(H, 0);
  std::memcpy(h.data(), kMagic, 8);
  const std::uint32_t nc = static_cast<std::uint32_t>(names.size());
  const std::uint32_t hb = static_cast<std::uint32_t>(H);
  const std::uint64_t nr = static_cast<std::uint64_t>(n);
  std::memcpy(h.data() + 8, &nc, 4);
  std::memcpy(h.data() + 12, &hb, 4);
  std::memcpy(h.data() + 16, &nr, 8);
  std::size_t at = 24;
  for (std::size_t i = 0; i < names.size(); ++i) {
    const std::uint32_t L = static_cast<std::uint32_t>(names[i].size());
    std::memcpy(h.data() + at, &L, 4);
    std::memcpy(h.data() + at + 4, names[i].data(), L);
    const std::uint64_t sum = n > 0 ? soa_checksum(cols[i], n) : 0;
    std::memcpy(h.data() + at + 4 + L, &sum, 8);
    at += 4 + L + 8;
  }
  errno = 0;
  Fd f;
  f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (f.fd < 0) io_error(path, "cannot create");
  write_all(f.fd, h.data(), h.size(), path);
  const std::uint64_t bytes = nr * 8u;
  const std::vector<char> pad(round_up(bytes, kAlign) - bytes, 0);
  for (std::size_t i = 0; i < cols.size(); ++i) {
    if (bytes) write_all(f.fd, cols[i], bytes, path);
    if (!pad.empty()) write_all(f.fd, pad.data(), pad.size(), path);
  }
  if (::close(f.fd) != 0) {
    f.fd = -1;
    io_error(path, "close failed");
  }
  f.fd = -1;
}

SoaHeader soa_read_header(const std::string& path) {
  errno = 0;
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  if (f.fd < 0) io_error(path, "cannot open");
  struct stat st {};
  if (::fstat(f.fd, &st) != 0) io_error(path, "stat failed");
  const std::uint64_t size = static_cast<std::uint64_t>(st.st_size);
  errno = 0;
  if (size < 24) data_error(path + ": not an ffsoa file (too short)");
  std::vector<char> b(24);
  pread_all(f.fd, b.data(), 24, 0, path);
  if (std::memcmp(b.data(), kMagic, 8) != 0) data_error(path + ": not an ffsoa file (bad magic)");
  SoaHeader h;
  const std::uint32_t nc = get<std::uint32_t>(b, 8);
  h.header_bytes = get<std::uint32_t>(b, 12);
  h.nrows = static_cast<long long>(get<std::uint64_t>(b, 16));
  if (nc == 0 || h.header_bytes < 24 || h.header_bytes % kAlign != 0 || h.nrows < 0 || h.header_bytes > size) {
    data_error(path + ": corrupt ffsoa header");
  }
  b.resize(h.header_bytes);
  pread_all(f.fd, b.data(), h.header_bytes, 0, path);
  std::size_t at = 24;
  for (std::uint32_t i = 0; i < nc; ++i) {
    if (at + 4 > b.size()) data_error(path + ": corrupt ffsoa header");
    const std::uint32_t L = get<std::uint32_t>(b, at);
    if (at + 4 + L + 8 > b.size()) data_error(path + ": corrupt ffsoa header");
    h.names.emplace_back(b.data() + at + 4, L);
    h.checksums.push_back(get<std::uint64_t>(b, at + 4 + L));
    at += 4 + L + 8;
  }
  h.column_stride = round_up(static_cast<std::uint64_t>(h.nrows) * 8u, kAlign);
  if (size < h.header_bytes + nc * h.column_stride) data_error(path + ": truncated ffsoa file");
  return h;
}

std::vector<std::vector<double>> soa_read_host(const std::string& path, SoaHeader* header) {
  const SoaHeader h = soa_read_header(path);
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  if (f.fd < 0) io_error(path, "cannot open");
  std::vector<std::vector<double>> cols(h.names.size(), std::vector<double>(static_cast<std::size_t>(h.nrows)));
  for (std::size_t c = 0; c < cols.size(); ++c) {
    if (h.nrows > 0) {
      pread_all(f.fd, cols[c].data(), static_cast<std::size_t>(h.nrows) * 8u, h.header_bytes + c * h.column_stride,
                path);
    }
    if (soa_checksum(cols[c].data(), h.nrows) != h.checksums[c]) {
      data_error(path + ": checksum mismatch in column '" + h.names[c] + "'");
    }
  }
  if (header) *header = h;
  return cols;
}

std::shared_ptr<DeviceDataset> soa_load_device(const std::string& path, SoaLoadStats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  const SoaHeader h = soa_read_header(path);
  auto ds = DeviceDataset::allocate(h.names, h.nrows);
  const std::uint64_t bytes = static_cast<std::uint64_t>(h.nrows) * 8u;
  const std::size_t chunk = static_cast<std::size_t>(std::min<std::uint64_t>(kChunk, round_up(bytes, kAlign)));
  const std::uint64_t per_col = bytes ? (bytes + chunk - 1) / chunk : 0;
  const std::uint64_t nchunks = per_col * h.names.size();
  // kReaders threads, each with two pinned staging buffers and its own stream: chunk j
  // goes to reader j % kReaders, whose copy of one buffer overlaps its read (and
  // checksum) of the other; page-cache reads and checksums run in parallel across readers
  constexpr int kReaders = 4;
  const int readers = static_cast<int>(std::min<std::uint64_t>(kReaders, std::max<std::uint64_t>(nchunks, 1)));
  std::vector<std::vector<std::uint64_t>> sums(readers, std::vector<std::uint64_t>(h.names.size(), 0));
  std::vector<std::string> errors(readers);
  int device = 0;
  cuda_check(cudaGetDevice(&device), "cudaGetDevice");
  auto work = [&](int r) {
    char* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    cudaStream_t s = nullptr;
    Fd f;
    try {
      cuda_check(cudaSetDevice(device), "cudaSetDevice");
      f.fd = ::open(path.c_str(), O_RDONLY);
      if (f.fd < 0) io_error(path, "cannot open");
      cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
      for (int k = 0; k < 2; ++k) {
        stage[k] = staging_pool().take();
        cuda_check(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming), "cudaEventCreate");
      }
      int k = 0;
      for (std::uint64_t j = static_cast<std::uint64_t>(r); j < nchunks; j += static_cast<std::uint64_t>(readers), ++k) {
        const std::size_t c = static_cast<std::size_t>(j / per_col);
        const std::uint64_t off = (j % per_col) * chunk;
        const std::size_t len = static_cast<std::size_t>(std::min<std::uint64_t>(chunk, bytes - off));
        char* buf = stage[k & 1];
        // the copy that last used this buffer must have finished reading it
        cuda_check(cudaEventSynchronize(done[k & 1]), "cudaEventSynchronize");
        pread_all(f.fd, buf, len, h.header_bytes + c * h.column_stride + off, path);
        cuda_check(cudaMemcpyAsync(reinterpret_cast<char*>(ds->cols[c]) + off, buf, len, cudaMemcpyHostToDevice, s),
                   "cudaMemcpyAsync(H2D chunk)");
        cuda_check(cudaEventRecord(done[k & 1], s), "cudaEventRecord");
        sums[r][c] = add_words(sums[r][c], buf, len);  // overlaps the copy just issued
      }
      cuda_check(cudaStreamSynchronize(s), "H2D upload");
    } catch (const std::exception& e) {
      errors[r] = e.what();
    }
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
    for (int k = 0; k < 2; ++k) {
      if (stage[k]) staging_pool().give(stage[k]);
      if (done[k]) cudaEventDestroy(done[k]);
    }
  };
  if (nchunks > 0) {
    std::vector<std::thread> pool;
    for (int r = 1; r < readers; ++r) pool.emplace_back(work, r);
    work(0);
    for (auto& t : pool) t.join();
  }
  for (const std::string& e : errors) {
    if (!e.empty()) data_error(e);
  }
  for (std::size_t c = 0; c < h.names.size(); ++c) {
    std::uint64_t sum = 0;  // wrapping addition: the chunk sums combine in any order
    for (int r = 0; r < readers; ++r) sum += sums[r][c];
    if (sum != h.checksums[c]) data_error(path + ": checksum mismatch in column '" + h.names[c] + "'");
  }
  if (stats) {
    stats->bytes = bytes * h.names.size();
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return ds;
}

}  // namespace ffb
