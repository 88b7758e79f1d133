// Design probe for the registered recycle pool: DMA straight between HBM and tmpfs
// page-cache pages that stay registered with CUDA across saves (mmap MAP_SHARED +
// cudaHostRegister once), against DMA into cudaHostAlloc memory.  Registration is timed
// separately (it is paid once per file, when the file first enters the pool).
//
//   mapped_dma_probe <dir> <files> <file_MiB> [reps]
//
// Prints one JSON line: register GB/s, steady D2H/H2D GB/s into the mappings and into
// pinned memory, and whether pread sees the DMA'd bytes.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e = (x);                                                         \
    if (e != cudaSuccess) {                                                      \
      printf("{\"error\": \"%s at line %d\"}\n", cudaGetErrorString(e), __LINE__); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  std::string dir = argv[1];
  const int nf = atoi(argv[2]);
  const size_t fb = (size_t)atoll(argv[3]) << 20;
  const int reps = argc > 4 ? atoi(argv[4]) : 3;
  char* dev;
  CK(cudaMalloc(&dev, fb));
  CK(cudaMemset(dev, 0x3c, fb));
  std::vector<char*> maps(nf);
  std::vector<int> fds(nf);
  std::vector<char> zeros(8 << 20, 0);
  double t0 = now();
  for (int i = 0; i < nf; ++i) {  // fresh files (pages allocated here, as a first save would)
    std::string p = dir + "/m" + std::to_string(i);
    fds[i] = open(p.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    for (size_t o = 0; o < fb; o += zeros.size()) pwrite(fds[i], zeros.data(), zeros.size(), o);
  }
  double t_create = now() - t0;
  t0 = now();
  for (int i = 0; i < nf; ++i) {
    maps[i] = (char*)mmap(nullptr, fb, PROT_READ | PROT_WRITE, MAP_SHARED, fds[i], 0);
    if (maps[i] == MAP_FAILED) {
      printf("{\"error\": \"mmap\"}\n");
      return 1;
    }
  }
  double t_map = now() - t0;
  t0 = now();
  for (int i = 0; i < nf; ++i) CK(cudaHostRegister(maps[i], fb, cudaHostRegisterPortable));
  double t_reg = now() - t0;
  char* pinned;
  CK(cudaHostAlloc(&pinned, fb, cudaHostAllocDefault));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto timed = [&](bool d2h, bool mapped) {
    double best = 0;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(a, s));
      for (int i = 0; i < nf; ++i) {
        char* h = mapped ? maps[i] : pinned;
        if (d2h) CK(cudaMemcpyAsync(h, dev, fb, cudaMemcpyDeviceToHost, s));
        else CK(cudaMemcpyAsync(dev, h, fb, cudaMemcpyHostToDevice, s));
      }
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      best = std::max(best, (double)fb * nf / (ms * 1e-3) / 1e9);
    }
    return best;
  };
  double d2h_map = timed(true, true), h2d_map = timed(false, true);
  double d2h_pin = timed(true, false), h2d_pin = timed(false, false);
  // the DMA'd bytes are the file's bytes (page cache)
  CK(cudaMemcpy(maps[0], dev, fb, cudaMemcpyDeviceToHost));
  std::vector<char> chk(4096);
  pread(fds[nf - 1], chk.data(), chk.size(), fb - 4096);
  bool ok_last = chk[0] == 0x3c && chk[4095] == 0x3c;
  pread(fds[0], chk.data(), chk.size(), 0);
  bool ok = ok_last && chk[0] == 0x3c;
  t0 = now();
  for (int i = 0; i < nf; ++i) CK(cudaHostUnregister(maps[i]));
  double t_unreg = now() - t0;
  for (int i = 0; i < nf; ++i) {
    munmap(maps[i], fb);
    close(fds[i]);
    unlink((dir + "/m" + std::to_string(i)).c_str());
  }
  const double gb = (double)fb * nf / 1e9;
  printf("{\"files\": %d, \"file_MiB\": %zu, \"create_GBps\": %.2f, \"mmap_s\": %.4f, \"register_GBps\": %.2f, "
         "\"unregister_GBps\": %.2f, \"d2h_mapped_GBps\": %.2f, \"h2d_mapped_GBps\": %.2f, "
         "\"d2h_pinned_GBps\": %.2f, \"h2d_pinned_GBps\": %.2f, \"pread_sees_dma\": %s}\n",
         nf, fb >> 20, gb / t_create, t_map, gb / t_reg, gb / t_unreg, d2h_map, h2d_map, d2h_pin, h2d_pin,
         ok ? "true" : "false");
  return 0;
}
