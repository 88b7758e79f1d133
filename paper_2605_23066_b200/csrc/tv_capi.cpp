// extern "C" surface of libtvgpu.so (declared in include/tvgpu.h), plus the peer/IPC
// helpers and the roofline probes that bench.py runs in the same job as the numbers.

#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tv_internal.h"

namespace tv {

thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
const std::string& get_error() { return g_last_error; }

int engine_create(int, int64_t, int64_t, int, tv_engine**);
int engine_destroy(tv_engine*);
int engine_save(tv_engine*, const tv_write_item*, int, const tv_output*, int, const char*, int,
                tv_stats*);
int engine_load(tv_engine*, const tv_read_item*, int, const tv_input*, int, const tv_copy*, int,
                tv_stats*);
int copy_boxes(int, const tv_copy*, int, cudaStream_t);
int kernel_timing(int);
int kernel_timing_collect(double*, double*, int64_t*, int64_t*);

}  // namespace tv

extern "C" {

int tv_abi_version(void) { return TV_ABI_VERSION; }

int tv_last_error(char* buf, size_t len) {
  const std::string& e = tv::get_error();
  if (buf && len) {
    size_t n = std::min(len - 1, e.size());
    std::memcpy(buf, e.data(), n);
    buf[n] = 0;
  }
  return (int)e.size();
}

int tv_copy_boxes(int device, const tv_copy* copies, int n, void* stream) {
  tv::DeviceGuard guard;
  if (n < 0 || (n > 0 && !copies)) {
    tv::set_error("tv_copy_boxes: bad arguments");
    return TV_ERR_ARG;
  }
  return tv::copy_boxes(device, copies, n, reinterpret_cast<cudaStream_t>(stream));
}

int tv_kernel_timing(int enable) { return tv::kernel_timing(enable); }

int tv_kernel_timing_collect(double* ms_total, double* ms_max, int64_t* bytes,
                             int64_t* launches) {
  tv::DeviceGuard guard;
  return tv::kernel_timing_collect(ms_total, ms_max, bytes, launches);
}

int64_t tv_copy_bytes(const tv_copy* copies, int n) {
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    int64_t b = copies[i].itemsize;
    for (int d = 0; d < copies[i].rank; ++d) b *= copies[i].ext[d];
    total += b;
  }
  return total;
}

int tv_engine_create(int n_slots, int64_t slot_bytes, int64_t staging_bytes, int n_threads,
                     tv_engine** out) {
  tv::DeviceGuard guard;
  if (!out) {
    tv::set_error("tv_engine_create: out is NULL");
    return TV_ERR_ARG;
  }
  return tv::engine_create(n_slots, slot_bytes, staging_bytes, n_threads, out);
}

int tv_engine_destroy(tv_engine* e) {
  tv::DeviceGuard guard; return tv::engine_destroy(e); }

int tv_engine_save(tv_engine* e, const tv_write_item* items, int n_items,
                   const tv_output* outputs, int n_outputs, tv_stats* stats) {
  tv::DeviceGuard guard;
  if (!e || n_items < 0 || n_outputs < 0) {
    tv::set_error("tv_engine_save: bad arguments");
    return TV_ERR_ARG;
  }
  return tv::engine_save(e, items, n_items, outputs, n_outputs, nullptr, 0, stats);
}

int tv_engine_save_pooled(tv_engine* e, const tv_write_item* items, int n_items,
                          const tv_output* outputs, int n_outputs, const char* pool_dir,
                          int pool_flags, tv_stats* stats) {
  tv::DeviceGuard guard;
  if (!e || n_items < 0 || n_outputs < 0) {
    tv::set_error("tv_engine_save_pooled: bad arguments");
    return TV_ERR_ARG;
  }
  return tv::engine_save(e, items, n_items, outputs, n_outputs,
                         (pool_dir && pool_dir[0]) ? pool_dir : nullptr, pool_flags, stats);
}

int tv_engine_load(tv_engine* e, const tv_read_item* items, int n_items, const tv_input* inputs,
                   int n_inputs, const tv_copy* copies, int n_copies, tv_stats* stats) {
  tv::DeviceGuard guard;
  if (!e || n_items < 0 || n_inputs < 0 || n_copies < 0) {
    tv::set_error("tv_engine_load: bad arguments");
    return TV_ERR_ARG;
  }
  return tv::engine_load(e, items, n_items, inputs, n_inputs, copies, n_copies, stats);
}

int tv_recycle_many(const char* const* paths, int n, const char* pool_dir, int n_threads,
                    uint8_t* ok) {
  if (n < 0 || (n > 0 && (!paths || !ok)) || !pool_dir || !pool_dir[0]) {
    tv::set_error("tv_recycle_many: bad arguments");
    return TV_ERR_ARG;
  }
  ::mkdir(pool_dir, 0777);
  const int t = std::max(1, std::min(n_threads, std::max(1, n)));
  static std::atomic<uint64_t> seq{0};
  const uint64_t stamp = (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
  std::atomic<int> next{0};
  std::atomic<int> failed{-1};
  std::atomic<int> err_no{0};
  auto work = [&] {
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
      struct stat st;
      if (::stat(paths[i], &st) != 0) {
        ok[i] = 0;
        if (errno != ENOENT && errno != ENOTDIR) {
          int expect = -1;
          if (failed.compare_exchange_strong(expect, i)) err_no.store(errno);
        }
        continue;
      }
      bool moved = false;
      if (S_ISREG(st.st_mode) && st.st_size > 0) {
        const std::string dir = std::string(pool_dir) + "/" + std::to_string((long long)st.st_size);
        ::mkdir(dir.c_str(), 0777);  // EEXIST is fine
        const std::string dst = dir + "/" + std::to_string((long long)::getpid()) + "-" +
                                std::to_string(stamp) + "-" + std::to_string(seq.fetch_add(1));
        moved = ::rename(paths[i], dst.c_str()) == 0;
      }
      if (!moved) tv::mapping_release_path(paths[i]);
      if (moved || ::unlink(paths[i]) == 0) {
        ok[i] = 1;
      } else {
        ok[i] = 0;
        if (errno != ENOENT && errno != ENOTDIR) {
          int expect = -1;
          if (failed.compare_exchange_strong(expect, i)) err_no.store(errno);
        }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (failed.load() >= 0) {
    tv::set_error(std::string("recycle ") + paths[failed.load()] + ": " + std::strerror(err_no.load()));
    return TV_ERR_IO;
  }
  return TV_OK;
}

int tv_unlink_many(const char* const* paths, int n, int n_threads, uint8_t* ok) {
  if (n < 0 || (n > 0 && (!paths || !ok))) {
    tv::set_error("tv_unlink_many: bad arguments");
    return TV_ERR_ARG;
  }
  const int t = std::max(1, std::min(n_threads, std::max(1, n)));
  std::atomic<int> next{0};
  std::atomic<int> failed{-1};
  std::atomic<int> err_no{0};
  auto work = [&] {
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
      tv::mapping_release_path(paths[i]);  // a registered file: drop its mapping first
      if (::unlink(paths[i]) == 0) {
        ok[i] = 1;
      } else {
        ok[i] = 0;
        if (errno != ENOENT && errno != ENOTDIR) {
          int expect = -1;
          if (failed.compare_exchange_strong(expect, i)) err_no.store(errno);
        }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (failed.load() >= 0) {
    tv::set_error(std::string("unlink ") + paths[failed.load()] + ": " + std::strerror(err_no.load()));
    return TV_ERR_IO;
  }
  return TV_OK;
}

int tv_enable_peer_access(const int* devices, int n) {
  tv::DeviceGuard guard;
  for (int i = 0; i < n; ++i) {
    TV_CUDA_CHECK(cudaSetDevice(devices[i]));
    for (int j = 0; j < n; ++j) {
      if (i == j || devices[i] == devices[j]) continue;
      int can = 0;
      TV_CUDA_CHECK(cudaDeviceCanAccessPeer(&can, devices[i], devices[j]));
      if (!can) {
        tv::set_error("GPU " + std::to_string(devices[i]) + " cannot access GPU " +
                      std::to_string(devices[j]) + " (no P2P path)");
        return TV_ERR_CUDA;
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        tv::set_error(std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        return TV_ERR_CUDA;
      }
    }
  }
  return TV_OK;
}

// cuMemGetAddressRange through the runtime's driver entry point (no -lcuda needed).
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

int tv_ipc_export(int device, uint64_t ptr, uint8_t handle_out[64], uint64_t* base_offset_out) {
  tv::DeviceGuard guard;
  TV_CUDA_CHECK(cudaSetDevice(device));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  TV_CUDA_CHECK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
  if (!fn) {
    tv::set_error("cuMemGetAddressRange unavailable");
    return TV_ERR_CUDA;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (reinterpret_cast<AddrRangeFn>(fn)(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) {
    tv::set_error("cuMemGetAddressRange failed");
    return TV_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  TV_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle_out, &h, 64);
  *base_offset_out = ptr - (uint64_t)base;
  return TV_OK;
}

int tv_ipc_import(int device, const uint8_t handle[64], uint64_t* ptr_out) {
  tv::DeviceGuard guard;
  TV_CUDA_CHECK(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void* p = nullptr;
  TV_CUDA_CHECK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr_out = reinterpret_cast<uint64_t>(p);
  return TV_OK;
}

int tv_ipc_close(int device, uint64_t ptr) {
  tv::DeviceGuard guard;
  TV_CUDA_CHECK(cudaSetDevice(device));
  TV_CUDA_CHECK(cudaIpcCloseMemHandle(reinterpret_cast<void*>(ptr)));
  return TV_OK;
}

static double wall() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

namespace {

// fio-style probe: n_threads files of file_bytes, block_bytes pwrite then pread from
// pinned memory.  With device >= 0 a DMA thread keeps that GPU's copy engine busy for
// the whole window (D2H during the writes, H2D during the reads) and its rate is
// returned too: the contended rates of a copy-through-pinned pipeline.
int probe_storage_impl(const char* dir, int n_threads, int64_t file_bytes, int64_t block_bytes,
                       int device, double* write_gbps, double* read_gbps, double* d2h_gbps,
                       double* h2d_gbps, double* rewrite_gbps = nullptr) {
  if (!dir || n_threads < 1 || file_bytes < 1 || block_bytes < 1) {
    tv::set_error("tv_probe_storage: bad arguments");
    return TV_ERR_ARG;
  }
  std::vector<char*> bufs(n_threads, nullptr);
  for (auto& b : bufs) {
    cudaError_t e = cudaHostAlloc(&b, block_bytes, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      for (auto q : bufs)
        if (q) cudaFreeHost(q);
      tv::set_error(std::string("probe cudaHostAlloc: ") + cudaGetErrorString(e));
      return TV_ERR_NOMEM;
    }
    std::memset(b, 0x5a, block_bytes);
  }
  const int64_t dma_bytes = 64ll << 20;
  char *dbuf = nullptr, *hbuf = nullptr;
  cudaStream_t st = nullptr;
  if (device >= 0) {
    cudaSetDevice(device);
    if (cudaMalloc(&dbuf, dma_bytes) != cudaSuccess || cudaHostAlloc(&hbuf, dma_bytes, cudaHostAllocDefault) != cudaSuccess ||
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
      tv::set_error("probe: DMA buffers");
      return TV_ERR_NOMEM;
    }
  }
  auto path = [&](int t) { return std::string(dir) + "/.tvgpu_probe_" + std::to_string(t); };
  std::atomic<int> failed{0};
  bool truncate = true;  // false: overwrite the files the write pass left (recycled pages)
  auto run = [&](bool write, double* dma_gbps) {
    std::atomic<bool> stop{false};
    std::atomic<int64_t> moved{0};
    double d0 = 0, d1 = 0;
    std::thread dma;
    if (device >= 0) {
      dma = std::thread([&] {
        cudaSetDevice(device);
        d0 = wall();
        while (!stop.load()) {
          if (write) cudaMemcpyAsync(hbuf, dbuf, dma_bytes, cudaMemcpyDeviceToHost, st);
          else cudaMemcpyAsync(dbuf, hbuf, dma_bytes, cudaMemcpyHostToDevice, st);
          cudaStreamSynchronize(st);
          moved += dma_bytes;
        }
        d1 = wall();
      });
    }
    std::vector<std::thread> th;
    double t0 = wall();
    for (int t = 0; t < n_threads; ++t)
      th.emplace_back([&, t] {
        int fd = write ? ::open(path(t).c_str(), O_WRONLY | O_CREAT | (truncate ? O_TRUNC : 0) | O_CLOEXEC, 0644)
                       : ::open(path(t).c_str(), O_RDONLY | O_CLOEXEC);
        if (fd < 0) {
          failed = 1;
          return;
        }
        for (int64_t o = 0; o < file_bytes; o += block_bytes) {
          int64_t n = std::min(block_bytes, file_bytes - o), done = 0;
          while (done < n) {
            ssize_t r = write ? ::pwrite(fd, bufs[t] + done, n - done, o + done)
                              : ::pread(fd, bufs[t] + done, n - done, o + done);
            if (r <= 0) {
              if (r < 0 && errno == EINTR) continue;
              failed = 1;
              break;
            }
            done += r;
          }
        }
        ::close(fd);
      });
    for (auto& x : th) x.join();
    const double gbps = (double)file_bytes * n_threads / (wall() - t0) / 1e9;
    if (device >= 0) {
      stop = true;
      dma.join();
      if (dma_gbps) *dma_gbps = (double)moved.load() / std::max(1e-9, d1 - d0) / 1e9;
    }
    return gbps;
  };
  *write_gbps = run(true, d2h_gbps);
  if (rewrite_gbps) {
    truncate = false;
    *rewrite_gbps = run(true, nullptr);
    truncate = true;
  }
  *read_gbps = run(false, h2d_gbps);
  for (int t = 0; t < n_threads; ++t) ::unlink(path(t).c_str());
  for (auto b : bufs) cudaFreeHost(b);
  if (device >= 0) {
    cudaStreamDestroy(st);
    cudaFree(dbuf);
    cudaFreeHost(hbuf);
  }
  if (failed) {
    tv::set_error(std::string("probe I/O failed in ") + dir);
    return TV_ERR_IO;
  }
  return TV_OK;
}

}  // namespace

int tv_probe_storage(const char* dir, int n_threads, int64_t file_bytes, int64_t block_bytes,
                     double* write_gbps, double* read_gbps) {
  return probe_storage_impl(dir, n_threads, file_bytes, block_bytes, -1, write_gbps, read_gbps,
                            nullptr, nullptr);
}

int tv_probe_storage_rewrite(const char* dir, int n_threads, int64_t file_bytes,
                             int64_t block_bytes, double* write_gbps, double* rewrite_gbps,
                             double* read_gbps) {
  if (!rewrite_gbps) {
    tv::set_error("tv_probe_storage_rewrite: bad arguments");
    return TV_ERR_ARG;
  }
  return probe_storage_impl(dir, n_threads, file_bytes, block_bytes, -1, write_gbps, read_gbps,
                            nullptr, nullptr, rewrite_gbps);
}

int tv_probe_storage_dma(const char* dir, int n_threads, int64_t file_bytes, int64_t block_bytes,
                         int device, double* write_gbps, double* read_gbps, double* d2h_gbps,
                         double* h2d_gbps) {
  tv::DeviceGuard guard;
  if (device < 0) {
    tv::set_error("tv_probe_storage_dma: needs a device");
    return TV_ERR_ARG;
  }
  return probe_storage_impl(dir, n_threads, file_bytes, block_bytes, device, write_gbps, read_gbps,
                            d2h_gbps, h2d_gbps);
}

int tv_probe_pcie(int device, int64_t bytes, int reps, double* d2h_gbps, double* h2d_gbps) {
  tv::DeviceGuard guard;
  TV_CUDA_CHECK(cudaSetDevice(device));
  char *d = nullptr, *h = nullptr;
  TV_CUDA_CHECK(cudaMalloc(&d, bytes));
  cudaError_t e = cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  if (e != cudaSuccess) {
    cudaFree(d);
    tv::set_error(std::string("probe cudaHostAlloc: ") + cudaGetErrorString(e));
    return TV_ERR_NOMEM;
  }
  cudaStream_t s;
  cudaEvent_t a, b;
  TV_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  TV_CUDA_CHECK(cudaEventCreate(&a));
  TV_CUDA_CHECK(cudaEventCreate(&b));
  double best[2] = {0, 0};
  for (int dir = 0; dir < 2; ++dir) {
    for (int r = 0; r < reps + 1; ++r) {
      TV_CUDA_CHECK(cudaEventRecord(a, s));
      if (dir == 0)
        TV_CUDA_CHECK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
      else
        TV_CUDA_CHECK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
      TV_CUDA_CHECK(cudaEventRecord(b, s));
      TV_CUDA_CHECK(cudaEventSynchronize(b));
      float ms = 0;
      TV_CUDA_CHECK(cudaEventElapsedTime(&ms, a, b));
      if (r > 0) best[dir] = std::max(best[dir], bytes / (ms * 1e-3) / 1e9);
    }
  }
  *d2h_gbps = best[0];
  *h2d_gbps = best[1];
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  cudaFreeHost(h);
  cudaFree(d);
  return TV_OK;
}

}  // extern "C"
