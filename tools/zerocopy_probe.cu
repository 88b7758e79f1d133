// Design probe: DMA directly between HBM and tmpfs page-cache pages (mmap +
// cudaHostRegister), no CPU copy.  Measures registration cost and end-to-end GB/s.
//   R) restore: existing file -> mmap(MAP_SHARED|MAP_POPULATE) -> register -> H2D
//   W) save:    new file -> fallocate -> mmap(MAP_POPULATE) -> register -> D2H -> unregister
// Usage: zerocopy_probe <dir> <threads> <file_MB> <files>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      printf("CUDA %s at line %d\n", cudaGetErrorString(e), __LINE__);                     \
      exit(1);                                                                              \
    }                                                                                       \
  } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  std::string dir = argv[1];
  int T = atoi(argv[2]);
  size_t fb = (size_t)atoll(argv[3]) << 20;
  int nf = atoi(argv[4]);
  char* dev;
  CK(cudaMalloc(&dev, fb * T));
  CK(cudaMemset(dev, 3, fb * T));
  std::vector<cudaStream_t> st(T);
  for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  auto path = [&](int i) { return dir + "/zc_" + std::to_string(i); };
  for (int mode = 0; mode < 2; ++mode) {  // 0 = W (save), 1 = R (restore)
    for (int rep = 0; rep < 2; ++rep) {
      std::atomic<int> next{0};
      std::atomic<long> reg_ns{0}, unreg_ns{0}, map_ns{0};
      double t0 = now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          int i;
          while ((i = next.fetch_add(1)) < nf) {
            double a = now();
            int fd = open(path(i).c_str(), mode == 0 ? (O_RDWR | O_CREAT | O_TRUNC) : O_RDWR, 0644);
            if (mode == 0 && fallocate(fd, 0, 0, fb) != 0) { perror("fallocate"); exit(2); }
            char* m = (char*)mmap(nullptr, fb, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, 0);
            if (m == MAP_FAILED) { perror("mmap"); exit(2); }
            double b = now();
            CK(cudaHostRegister(m, fb, cudaHostRegisterDefault));
            double c = now();
            if (mode == 0) CK(cudaMemcpyAsync(m, dev + t * fb, fb, cudaMemcpyDeviceToHost, st[t]));
            else CK(cudaMemcpyAsync(dev + t * fb, m, fb, cudaMemcpyHostToDevice, st[t]));
            CK(cudaStreamSynchronize(st[t]));
            double d = now();
            CK(cudaHostUnregister(m));
            double e = now();
            munmap(m, fb);
            close(fd);
            map_ns += (long)((b - a) * 1e9);
            reg_ns += (long)((c - b) * 1e9);
            unreg_ns += (long)((e - d) * 1e9);
          }
        });
      for (auto& x : th) x.join();
      double dt = now() - t0;
      double gb = (double)fb * nf / 1e9;
      printf("%s T=%d file=%zuMB files=%d: %.2f GB/s  (per-thread sums: map+alloc %.2fs register %.2fs unregister %.2fs)\n",
             mode == 0 ? "W zero-copy save   " : "R zero-copy restore", T, fb >> 20, nf, gb / dt,
             map_ns * 1e-9, reg_ns * 1e-9, unreg_ns * 1e-9);
    }
  }
  for (int i = 0; i < nf; ++i) unlink(path(i).c_str());
  return 0;
}
