// Storage / PCIe design probe (not product code): measures the host-side options for
// moving checkpoint bytes between HBM and a tmpfs/NVMe directory.
//   A) D2H into pinned slots, then pwrite() by T threads       (classic staging)
//   B) ftruncate+mmap the file, cudaHostRegister it, D2H straight into the page cache
//   C) pread() into pinned slots then H2D                       (restore, classic)
//   D) mmap + cudaHostRegister the file, H2D straight from the page cache
// Usage: io_probe <dir> <total_GB> <threads> <file_MB> <slot_MB>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

static void memcpy_probe(int T, size_t bytes) {
  std::vector<char*> a(T), b(T);
  for (int t = 0; t < T; ++t) { a[t] = (char*)aligned_alloc(4096, bytes); b[t] = (char*)aligned_alloc(4096, bytes); memset(a[t], 1, bytes); memset(b[t], 2, bytes); }
  double t0 = now();
  std::vector<std::thread> th;
  for (int t = 0; t < T; ++t) th.emplace_back([&, t] { for (int r = 0; r < 4; ++r) memcpy(b[t], a[t], bytes); });
  for (auto& x : th) x.join();
  printf("memcpy T=%d: %.2f GB/s (copied bytes)\n", T, 4.0 * T * bytes / (now() - t0) / 1e9);
  for (int t = 0; t < T; ++t) { free(a[t]); free(b[t]); }
}

int main(int argc, char** argv) {
  if (argc == 2) { for (int T : {1, 4, 8, 16}) memcpy_probe(T, 256 << 20); return 0; }
  std::string dir = argv[1];
  double total_gb = atof(argv[2]);
  int T = atoi(argv[3]);
  size_t file_bytes = (size_t)atoll(argv[4]) << 20;
  size_t slot = (size_t)atoll(argv[5]) << 20;
  size_t nfiles = (size_t)(total_gb * 1e9 / file_bytes);
  size_t total = nfiles * file_bytes;
  char* dev;
  CK(cudaMalloc(&dev, file_bytes));
  CK(cudaMemset(dev, 7, file_bytes));
  std::vector<cudaStream_t> streams(T);
  for (auto& s : streams) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<char*> slots(T);
  for (auto& p : slots) CK(cudaHostAlloc(&p, slot, cudaHostAllocDefault));
  auto path = [&](size_t i) { return dir + "/probe_" + std::to_string(i) + ".bin"; };

  // A) staged write
  {
    std::atomic<size_t> next{0};
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        size_t i;
        while ((i = next.fetch_add(1)) < nfiles) {
          int fd = open((path(i) + ".partial").c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
          for (size_t o = 0; o < file_bytes; o += slot) {
            size_t n = std::min(slot, file_bytes - o);
            CK(cudaMemcpyAsync(slots[t], dev + o, n, cudaMemcpyDeviceToHost, streams[t]));
            CK(cudaStreamSynchronize(streams[t]));
            size_t w = 0;
            while (w < n) w += pwrite(fd, slots[t] + w, n - w, o + w);
          }
          close(fd);
          rename((path(i) + ".partial").c_str(), path(i).c_str());
        }
      });
    for (auto& x : th) x.join();
    double dt = now() - t0;
    printf("A staged-write   T=%d file=%zuMB slot=%zuMB: %.2f GB/s\n", T, file_bytes >> 20,
           slot >> 20, total / dt / 1e9);
  }
  // C) staged read
  {
    std::atomic<size_t> next{0};
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        size_t i;
        while ((i = next.fetch_add(1)) < nfiles) {
          int fd = open(path(i).c_str(), O_RDONLY);
          for (size_t o = 0; o < file_bytes; o += slot) {
            size_t n = std::min(slot, file_bytes - o);
            size_t r = 0;
            while (r < n) r += pread(fd, slots[t] + r, n - r, o + r);
            CK(cudaMemcpyAsync(dev + o, slots[t], n, cudaMemcpyHostToDevice, streams[t]));
            CK(cudaStreamSynchronize(streams[t]));
          }
          close(fd);
        }
      });
    for (auto& x : th) x.join();
    double dt = now() - t0;
    printf("C staged-read    T=%d: %.2f GB/s\n", T, total / dt / 1e9);
  }
  for (size_t i = 0; i < nfiles; ++i) unlink(path(i).c_str());
  // E) plain pwrite from pinned memory (storage only, no GPU)
  {
    std::atomic<size_t> next{0};
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        size_t i;
        while ((i = next.fetch_add(1)) < nfiles) {
          int fd = open(path(i).c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
          if (getenv("FALLOC")) posix_fallocate(fd, 0, file_bytes);
          for (size_t o = 0; o < file_bytes; o += slot) {
            size_t n = std::min(slot, file_bytes - o);
            size_t w = 0;
            while (w < n) w += pwrite(fd, slots[t] + w, n - w, o + w);
          }
          close(fd);
        }
      });
    for (auto& x : th) x.join();
    double dt = now() - t0;
    printf("E pwrite-only    T=%d: %.2f GB/s\n", T, total / dt / 1e9);
  }
  {
    std::atomic<size_t> next{0};
    double t0 = now();
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        size_t i;
        while ((i = next.fetch_add(1)) < nfiles) {
          int fd = open(path(i).c_str(), O_RDONLY);
          for (size_t o = 0; o < file_bytes; o += slot) {
            size_t n = std::min(slot, file_bytes - o);
            size_t r = 0;
            while (r < n) r += pread(fd, slots[t] + r, n - r, o + r);
          }
          close(fd);
        }
      });
    for (auto& x : th) x.join();
    double dt = now() - t0;
    printf("F pread-only     T=%d: %.2f GB/s\n", T, total / dt / 1e9);
  }
  for (size_t i = 0; i < nfiles; ++i) unlink(path(i).c_str());
  return 0;
}
