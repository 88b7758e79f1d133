// Registered file mappings: the zero-copy half of the recycle pool.
//
// A file retired into the recycle pool (tv_recycle_many) on a RAM-backed filesystem
// (tmpfs / ramfs) is mapped MAP_SHARED and registered with CUDA once
// (tv_pool_register).  Its inode keeps the registration while it cycles pool ->
// checkpoint file (claimed by a save, renamed) -> pool, so in steady state:
//
//   save:    D2H lands straight in the file's page-cache pages (one host-memory pass,
//            instead of DMA into a pinned slot + pwrite's read + the page-cache write);
//   restore: H2D reads straight from them (no pread into a slot).
//
// Measured on B200 boxes (profiles/r02_mapped_probe_*.jsonl): DMA into / out of such
// mappings runs at the pinned-memory rate (57.2 / 55.6 GB/s D2H / H2D); registering a
// 2 MiB-page tmpfs file costs 30-57 GB/s, once.
//
// Only RAM-backed filesystems qualify: there the page cache IS the storage, so bytes the
// DMA engine writes into the pages are the file's bytes with no writeback to miss.  The
// engine bumps a written file's mtime itself (futimens) since DMA does not.
#include <cuda_runtime.h>
#include <dirent.h>
#include <errno.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/vfs.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "tv_internal.h"

namespace tv {
namespace {

constexpr long kTmpfsMagic = 0x01021994;
constexpr long kRamfsMagic = 0x858458f6;

struct Mapping {  // the mapping itself keeps the inode alive; no descriptor is held
  char* addr = nullptr;
  int64_t size = 0;
};

class MappingCache {
 public:
  static MappingCache& get() {
    static MappingCache* c = new MappingCache();  // never destroyed: process-lifetime mappings
    return *c;
  }
  char* find(dev_t dev, ino_t ino, int64_t size) {
    std::lock_guard<std::mutex> g(m_);
    auto it = by_inode_.find({dev, ino});
    if (it == by_inode_.end() || it->second.size != size) return nullptr;
    return it->second.addr;
  }
  bool has(dev_t dev, ino_t ino) {
    std::lock_guard<std::mutex> g(m_);
    return by_inode_.count({dev, ino}) != 0;
  }
  void insert(dev_t dev, ino_t ino, const Mapping& m) {
    std::lock_guard<std::mutex> g(m_);
    by_inode_[{dev, ino}] = m;
  }
  void release(dev_t dev, ino_t ino) {
    Mapping m;
    {
      std::lock_guard<std::mutex> g(m_);
      auto it = by_inode_.find({dev, ino});
      if (it == by_inode_.end()) return;
      m = it->second;
      by_inode_.erase(it);
    }
    drop(m);
  }
  void release_all() {
    std::map<std::pair<dev_t, ino_t>, Mapping> all;
    {
      std::lock_guard<std::mutex> g(m_);
      all.swap(by_inode_);
    }
    for (auto& kv : all) drop(kv.second);
  }
  void stats(int64_t* files, int64_t* bytes) {
    std::lock_guard<std::mutex> g(m_);
    int64_t b = 0;
    for (auto& kv : by_inode_) b += kv.second.size;
    if (files) *files = (int64_t)by_inode_.size();
    if (bytes) *bytes = b;
  }
  bool empty() {
    std::lock_guard<std::mutex> g(m_);
    return by_inode_.empty();
  }

 private:
  static void drop(const Mapping& m) {
    for (int64_t off = 0; off < m.size; off += kRegisterPiece) cudaHostUnregister(m.addr + off);
    ::munmap(m.addr, (size_t)m.size);
  }
  std::mutex m_;
  std::map<std::pair<dev_t, ino_t>, Mapping> by_inode_;
};

// Register [addr, addr+size) in kRegisterPiece pieces (DMAs are split at the same file
// offsets), pausing after each so that the registrar holds the driver at most `duty` of
// the time: a save or restore running meanwhile keeps its CUDA calls flowing.  On failure
// the pieces already registered are released.
cudaError_t register_pieces(char* addr, int64_t size, double duty) {
  for (int64_t off = 0; off < size; off += kRegisterPiece) {
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t ce = cudaHostRegister(addr + off, (size_t)std::min(kRegisterPiece, size - off),
                                      cudaHostRegisterPortable);
    if (ce != cudaSuccess) {
      cudaGetLastError();
      for (int64_t o = 0; o < off; o += kRegisterPiece) cudaHostUnregister(addr + o);
      return ce;
    }
    if (duty < 1.0) {
      const auto dt = std::chrono::steady_clock::now() - t0;
      std::this_thread::sleep_for(std::chrono::duration_cast<std::chrono::microseconds>(dt * (1.0 / duty - 1.0)));
    }
  }
  return cudaSuccess;
}

bool ram_backed(int fd) {
  struct statfs sf;
  if (::fstatfs(fd, &sf) != 0) return false;
  return (long)sf.f_type == kTmpfsMagic || (long)sf.f_type == kRamfsMagic;
}

// Map + register one file; 1 = registered now, 0 = skipped (already registered, empty,
// not RAM-backed), <0 = error (message in err).
int register_file(const std::string& path, std::string& err) {
  int fd = ::open(path.c_str(), O_RDWR | O_CLOEXEC);
  if (fd < 0) {
    if (errno == ENOENT) return 0;  // claimed by a concurrent save meanwhile
    err = "open " + path + ": " + std::strerror(errno);
    return -1;
  }
  struct stat st;
  if (::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode) || st.st_size <= 0 || !ram_backed(fd) ||
      MappingCache::get().has(st.st_dev, st.st_ino)) {
    ::close(fd);
    return 0;
  }
  void* addr = ::mmap(nullptr, (size_t)st.st_size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (addr == MAP_FAILED) {
    err = "mmap " + path + ": " + std::strerror(errno);
    ::close(fd);
    return -1;
  }
  cudaError_t ce = register_pieces(static_cast<char*>(addr), st.st_size, 1.0);
  if (ce != cudaSuccess) {
    ::munmap(addr, (size_t)st.st_size);
    ::close(fd);
    err = "cudaHostRegister " + path + ": " + cudaGetErrorString(ce);
    return -1;
  }
  Mapping m;
  m.addr = static_cast<char*>(addr);
  m.size = st.st_size;
  MappingCache::get().insert(st.st_dev, st.st_ino, m);
  ::close(fd);
  return 1;
}

// Regular files of <pool>/<size>/.
std::vector<std::string> pool_files(const std::string& pool) {
  std::vector<std::string> out;
  DIR* top = ::opendir(pool.c_str());
  if (!top) return out;
  while (struct dirent* sub = ::readdir(top)) {
    if (sub->d_name[0] == '.') continue;
    const std::string dir = pool + "/" + sub->d_name;
    if (DIR* d = ::opendir(dir.c_str())) {
      while (struct dirent* ent = ::readdir(d)) {
        if (ent->d_name[0] == '.') continue;
        out.push_back(dir + "/" + ent->d_name);
      }
      ::closedir(d);
    }
  }
  ::closedir(top);
  return out;
}

// Map + register the file open (read-write) as `fd`; the cached address or null.
char* register_open(int fd, int64_t size) {
  struct stat st;
  if (fd < 0 || ::fstat(fd, &st) != 0 || !S_ISREG(st.st_mode) || st.st_size != size || size <= 0 ||
      !ram_backed(fd))
    return nullptr;
  if (char* hit = MappingCache::get().find(st.st_dev, st.st_ino, size)) return hit;
  void* addr = ::mmap(nullptr, (size_t)size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (addr == MAP_FAILED) return nullptr;
  if (register_pieces(static_cast<char*>(addr), size, 1.0) != cudaSuccess) {
    ::munmap(addr, (size_t)size);
    return nullptr;
  }
  Mapping m;
  m.addr = static_cast<char*>(addr);
  m.size = size;
  MappingCache::get().insert(st.st_dev, st.st_ino, m);
  return m.addr;
}

}  // namespace

char* mapping_register_fd(int fd, int64_t size, bool register_now) {
  if (fd < 0) return nullptr;
  if (char* hit = mapping_for_fd(fd, size)) return hit;
  return register_now ? register_open(fd, size) : nullptr;
}


char* mapping_for_fd(int fd, int64_t size) {
  if (fd < 0 || MappingCache::get().empty()) return nullptr;
  struct stat st;
  if (::fstat(fd, &st) != 0) return nullptr;
  return MappingCache::get().find(st.st_dev, st.st_ino, size);
}

bool mappings_exist() { return !MappingCache::get().empty(); }

void mapping_release_fd(int fd) {
  struct stat st;
  if (fd >= 0 && ::fstat(fd, &st) == 0) MappingCache::get().release(st.st_dev, st.st_ino);
}

void mapping_release_path(const char* path) {
  struct stat st;
  if (!MappingCache::get().empty() && ::stat(path, &st) == 0)
    MappingCache::get().release(st.st_dev, st.st_ino);
}

}  // namespace tv

extern "C" {

int tv_pool_register(const char* pool_dir, int n_threads, int64_t* registered_bytes) {
  tv::DeviceGuard guard;
  if (!pool_dir) {
    tv::set_error("tv_pool_register: bad arguments");
    return TV_ERR_ARG;
  }
  if (registered_bytes) *registered_bytes = 0;
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
    cudaGetLastError();
    return TV_OK;  // no GPU: nothing to register (the pool still recycles pages)
  }
  const std::vector<std::string> files = tv::pool_files(pool_dir);
  std::atomic<size_t> next{0};
  std::atomic<int64_t> bytes{0};
  std::mutex em;
  std::string first_err;
  auto work = [&] {
    for (size_t i = next.fetch_add(1); i < files.size(); i = next.fetch_add(1)) {
      std::string err;
      struct stat st;
      const int rc = tv::register_file(files[i], err);
      if (rc > 0 && ::stat(files[i].c_str(), &st) == 0) bytes += st.st_size;
      if (rc < 0) {
        std::lock_guard<std::mutex> g(em);
        if (first_err.empty()) first_err = err;
      }
    }
  };
  const int t = std::max(1, std::min(n_threads, (int)std::max<size_t>(1, files.size())));
  std::vector<std::thread> pool;
  for (int k = 1; k < t; ++k) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  if (registered_bytes) *registered_bytes = bytes.load();
  if (!first_err.empty()) {
    tv::set_error(first_err);
    return TV_ERR_CUDA;
  }
  return TV_OK;
}

int tv_pool_drain(const char* pool_dir, int64_t* freed_bytes) {
  tv::DeviceGuard guard;
  if (!pool_dir) {
    tv::set_error("tv_pool_drain: bad arguments");
    return TV_ERR_ARG;
  }
  int64_t freed = 0;
  for (const std::string& f : tv::pool_files(pool_dir)) {
    struct stat st;
    if (::stat(f.c_str(), &st) != 0) continue;
    tv::mapping_release_path(f.c_str());
    if (::unlink(f.c_str()) == 0) freed += st.st_size;
  }
  if (freed_bytes) *freed_bytes = freed;
  return TV_OK;
}

int tv_mapping_stats(int64_t* files, int64_t* bytes) {
  tv::MappingCache::get().stats(files, bytes);
  return TV_OK;
}

int tv_mapping_release_all(void) {
  tv::DeviceGuard guard;
  tv::MappingCache::get().release_all();
  return TV_OK;
}

}  // extern "C"
