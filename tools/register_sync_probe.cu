// Does cudaHostRegister wait for work running on the GPU?  A long kernel runs in the
// primary context while another thread registers 64 MiB of a tmpfs file mapping:
//   (a) from the primary context (runtime API),
//   (b) from a secondary driver-API context (cuCtxCreate) with CU_MEMHOSTREGISTER_PORTABLE,
// and the registration is then used for a D2H in the primary context.
//
//   register_sync_probe <dir>
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

__global__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : "/dev/shm";
  const size_t sz = 64 << 20;
  std::vector<char*> maps;
  std::vector<char> buf(sz, 1);
  for (int i = 0; i < 4; ++i) {
    std::string p = dir + "/rs" + std::to_string(i);
    int fd = open(p.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0644);
    if (write(fd, buf.data(), sz) != (ssize_t)sz) return 1;
    maps.push_back((char*)mmap(nullptr, sz, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
    close(fd);
  }
  cudaSetDevice(0);
  cudaFree(0);
  char* dev;
  cudaMalloc(&dev, sz);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  // idle GPU: baseline registration time
  double t0 = now();
  cudaHostRegister(maps[0], sz, cudaHostRegisterPortable);
  double idle_ms = (now() - t0) * 1e3;
  // busy GPU: a ~2 s kernel on another stream
  spin<<<1, 1, 0, s>>>(4000000000LL);
  std::this_thread::sleep_for(std::chrono::milliseconds(100));
  t0 = now();
  cudaError_t e1 = cudaHostRegister(maps[1], sz, cudaHostRegisterPortable);
  double busy_primary_ms = (now() - t0) * 1e3;
  cudaStreamSynchronize(s);
  // secondary context, busy GPU
  cuInit(0);
  CUdevice cudev;
  cuDeviceGet(&cudev, 0);
  CUcontext second = nullptr, primary = nullptr;
  cuCtxGetCurrent(&primary);
  double busy_secondary_ms = -1;
  CUresult r2 = CUDA_ERROR_UNKNOWN;
  spin<<<1, 1, 0, s>>>(4000000000LL);
  std::this_thread::sleep_for(std::chrono::milliseconds(100));
  std::thread th([&] {
    if (cuCtxCreate(&second, 0, cudev) != CUDA_SUCCESS) return;
    double a = now();
    r2 = cuMemHostRegister(maps[2], sz, CU_MEMHOSTREGISTER_PORTABLE);
    busy_secondary_ms = (now() - a) * 1e3;
    cuCtxPopCurrent(nullptr);
  });
  th.join();
  // the secondary-context registration used by a D2H in the primary context
  cudaStreamSynchronize(s);
  cudaMemset(dev, 7, sz);
  cudaError_t e3 = cudaMemcpy(maps[2], dev, sz, cudaMemcpyDeviceToHost);
  bool ok = maps[2][0] == 7 && maps[2][sz - 1] == 7;
  cudaPointerAttributes at;
  cudaError_t e4 = cudaPointerGetAttributes(&at, maps[2]);
  printf("{\"idle_register_ms\": %.2f, \"busy_primary_register_ms\": %.2f, \"busy_secondary_register_ms\": %.2f, "
         "\"primary_err\": \"%s\", \"secondary_rc\": %d, \"d2h_into_secondary_registration\": \"%s\", \"bytes_ok\": %s, "
         "\"attr\": \"%s type=%d\"}\n",
         idle_ms, busy_primary_ms, busy_secondary_ms, cudaGetErrorString(e1), (int)r2, cudaGetErrorString(e3),
         ok ? "true" : "false", cudaGetErrorString(e4), (int)at.type);
  for (int i = 0; i < 4; ++i) unlink((dir + "/rs" + std::to_string(i)).c_str());
  return 0;
}
