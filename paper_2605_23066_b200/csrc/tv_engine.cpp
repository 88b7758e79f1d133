// libtvgpu I/O engine: the save and restore pipelines between HBM and storage.
//
// Save (tv_engine_save) — replaces SaveSession.write_phase → ProcessArrayWriter
// (chunkstore.py:352-454) → FilesystemBackend._put (backend.py:398-403):
//   producer (caller thread) walks the chunk payloads in file order and fills a ring of
//   pinned host slots: a payload that is one contiguous byte range of its device array
//   is DMA'd straight from HBM (no kernel), a strided box is first packed by the
//   box-copy kernel into device staging and then DMA'd; every slot gets a CUDA event.
//   Storage threads take filled slots, wait for their event, pwrite the bytes at their
//   file offsets, and commit a file (<path>.partial → rename) when its last byte lands.
//   D2H of slot k+1.. overlaps the writes of slot k; n_threads files are written at once.
//
// Restore (tv_engine_load) — replaces ChunkReader.read_range (chunkstore.py:507-593) and
// _execute_reads/_assemble (load_pipeline.py:406-493):
//   reader threads pread byte ranges into pinned slots and issue the H2D themselves,
//   either straight into the destination shard (contiguous destination) or into device
//   staging; when the last piece of an item has landed, the same thread launches the
//   item's box copies (unpack / reshard scatter), whose destinations may be other GPUs
//   (NVLink P2P or IPC-mapped) — the read-once fan-out.
//
// Knobs (measured defaults): one DMA stream per device
// (TVGPU_DMA_STREAMS > 1 was 15-20 % slower), cudaHostAlloc slots (TVGPU_HUGE_RING=1: one
// THP-backed pinned region, measured neutral).

#include <cuda_runtime.h>
#include <errno.h>
#include <dirent.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/types.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "tv_internal.h"

namespace tv {

namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Accumulates seconds from many threads.
struct Clock {
  std::atomic<int64_t> ns{0};
  void add(double seconds) { ns += (int64_t)(seconds * 1e9); }
  double seconds() const { return ns.load() * 1e-9; }
};

std::string errno_msg(const std::string& what, const std::string& path) {
  return what + " " + path + ": " + std::strerror(errno);
}

// ---- small concurrency helpers -----------------------------------------------------

template <typename T>
class Queue {
 public:
  void push(T v) {
    {
      std::lock_guard<std::mutex> g(m_);
      q_.push_back(std::move(v));
    }
    cv_.notify_one();
  }
  bool pop(T& out) {  // false when closed and drained
    std::unique_lock<std::mutex> g(m_);
    cv_.wait(g, [&] { return closed_ || !q_.empty(); });
    if (q_.empty()) return false;
    out = std::move(q_.front());
    q_.pop_front();
    return true;
  }
  void close() {
    {
      std::lock_guard<std::mutex> g(m_);
      closed_ = true;
    }
    cv_.notify_all();
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  std::deque<T> q_;
  bool closed_ = false;
};

struct ErrorSlot {
  std::mutex m;
  std::atomic<bool> failed{false};
  int code = TV_OK;
  std::string msg;
  void set(int c, const std::string& s) {
    std::lock_guard<std::mutex> g(m);
    if (!failed.load()) {
      code = c;
      msg = s;
      failed.store(true);
    }
  }
};

// mkdir -p with a cache of directories known to exist.
class DirMaker {
 public:
  bool ensure(const std::string& dir, std::string& err) {
    if (dir.empty()) return true;
    {
      std::lock_guard<std::mutex> g(m_);
      if (done_.count(dir)) return true;
    }
    std::string cur;
    size_t pos = 0;
    while (pos != std::string::npos) {
      pos = dir.find('/', pos + 1);
      cur = dir.substr(0, pos);
      if (cur.empty()) continue;
      if (mkdir(cur.c_str(), 0777) != 0 && errno != EEXIST) {
        err = errno_msg("mkdir", cur);
        return false;
      }
    }
    std::lock_guard<std::mutex> g(m_);
    done_.insert(dir);
    return true;
  }

 private:
  std::mutex m_;
  std::unordered_set<std::string> done_;
};

std::string parent_of(const std::string& path) {
  size_t p = path.rfind('/');
  return p == std::string::npos ? std::string() : path.substr(0, p);
}

// ---- kernel timing (tv_kernel_timing) ---------------------------------------------------

// Algorithmic HBM bytes of one launch: every byte copied is read once and written once;
// a converting copy reads source elements and writes destination elements.
int64_t job_traffic(const std::vector<CopyJob>& jobs) {
  int64_t b = 0;
  for (const auto& j : jobs) b += 2 * j.run * j.nruns;
  return b;
}
int64_t job_traffic(const std::vector<CastJob>& jobs) {
  int64_t b = 0;
  for (const auto& j : jobs) b += j.run * j.nruns * (dtype_size(j.sdt) + dtype_size(j.ddt));
  return b;
}

// While enabled, every box-copy / cast launch is bracketed by two timing events on its
// stream: the first is recorded after the job-table upload, so the window is the kernel
// (plus launch latency), not the host's enqueue work.  Collected (and reset) on demand.
class KernelTimer {
 public:
  std::atomic<bool> on{false};
  struct Rec {
    int device;
    cudaEvent_t a, b;
    int64_t bytes;
  };
  cudaError_t begin(int device, cudaStream_t stream, cudaEvent_t* a) {
    cudaError_t e = cudaEventCreate(a);
    if (e == cudaSuccess) e = cudaEventRecord(*a, stream);
    (void)device;
    return e;
  }
  cudaError_t end(int device, cudaStream_t stream, cudaEvent_t a, int64_t bytes) {
    cudaEvent_t b;
    cudaError_t e = cudaEventCreate(&b);
    if (e == cudaSuccess) e = cudaEventRecord(b, stream);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(m_);
    recs_.push_back({device, a, b, bytes});
    return cudaSuccess;
  }
  int collect(double* ms_total, double* ms_max, int64_t* bytes, int64_t* launches) {
    std::vector<Rec> recs;
    {
      std::lock_guard<std::mutex> g(m_);
      recs.swap(recs_);
    }
    double tot = 0, mx = 0;
    int64_t by = 0;
    int rc = TV_OK;
    for (auto& r : recs) {
      float ms = 0;
      cudaSetDevice(r.device);
      if (rc == TV_OK) {
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess) {
          set_error(std::string("tv_kernel_timing_collect: ") + cudaGetErrorString(e));
          rc = TV_ERR_CUDA;
        }
      }
      tot += ms;
      mx = std::max(mx, (double)ms);
      by += r.bytes;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    if (ms_total) *ms_total = tot;
    if (ms_max) *ms_max = mx;
    if (bytes) *bytes = by;
    if (launches) *launches = (int64_t)recs.size();
    return rc;
  }

 private:
  std::mutex m_;
  std::vector<Rec> recs_;
};

KernelTimer g_timer;

// ---- per-device resources -------------------------------------------------------------

// Uploads CopyJob tables to the device through a pinned ring; a region is reused only
// after the kernel that read it has completed (event).
class JobUploader {
 public:
  explicit JobUploader(int device) : device_(device) {}
  ~JobUploader() {
    cudaSetDevice(device_);
    for (auto& r : inflight_) cudaEventDestroy(r.ev);
    for (auto ev : free_events_) cudaEventDestroy(ev);
    if (host_) cudaFreeHost(host_);
    if (dev_) cudaFree(dev_);
  }
  // Copies `jobs`, launches the kernel, retires the region with an event.
  int run(std::vector<CopyJob>& jobs, cudaStream_t stream, int64_t* launches) {
    return run_generic(jobs, stream, launches, plan_units, launch_copy_jobs);
  }
  int run_cast(std::vector<CastJob>& jobs, cudaStream_t stream, int64_t* launches) {
    return run_generic(jobs, stream, launches, plan_cast_units, launch_cast_jobs);
  }

 private:
  template <typename Job, typename Plan, typename Launch>
  int run_generic(std::vector<Job>& jobs, cudaStream_t stream, int64_t* launches, Plan plan,
                  Launch launch) {
    if (jobs.empty()) return TV_OK;
    const int64_t total_units = plan(jobs);
    const size_t bytes = jobs.size() * sizeof(Job);
    std::lock_guard<std::mutex> g(m_);
    if (bytes > cap_) {
      // Grow (rare): drain everything, reallocate.
      for (auto& r : inflight_) {
        cudaEventSynchronize(r.ev);
        free_events_.push_back(r.ev);
      }
      inflight_.clear();
      if (host_) cudaFreeHost(host_);
      if (dev_) cudaFree(dev_);
      cap_ = std::max<size_t>(bytes * 2, 1 << 20);
      TV_CUDA_CHECK(cudaHostAlloc(&host_, cap_, cudaHostAllocDefault));
      TV_CUDA_CHECK(cudaMalloc(&dev_, cap_));
      head_ = 0;
    }
    if (head_ + bytes > cap_) head_ = 0;
    // Wait for in-flight regions overlapping [head_, head_+bytes).
    for (auto it = inflight_.begin(); it != inflight_.end();) {
      bool overlap = it->off < head_ + bytes && head_ < it->off + it->len;
      if (overlap || cudaEventQuery(it->ev) == cudaSuccess) {
        TV_CUDA_CHECK(cudaEventSynchronize(it->ev));
        free_events_.push_back(it->ev);
        it = inflight_.erase(it);
      } else {
        ++it;
      }
    }
    std::memcpy(host_ + head_, jobs.data(), bytes);
    TV_CUDA_CHECK(cudaMemcpyAsync(dev_ + head_, host_ + head_, bytes, cudaMemcpyHostToDevice,
                                  stream));
    const bool timed = g_timer.on.load(std::memory_order_relaxed);
    cudaEvent_t t0 = nullptr;
    if (timed) TV_CUDA_CHECK(g_timer.begin(device_, stream, &t0));
    TV_CUDA_CHECK(launch(reinterpret_cast<const Job*>(dev_ + head_), jobs.data(), (int)jobs.size(),
                         total_units, stream));
    if (timed) TV_CUDA_CHECK(g_timer.end(device_, stream, t0, job_traffic(jobs)));
    cudaEvent_t ev;
    if (free_events_.empty()) {
      TV_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    } else {
      ev = free_events_.back();
      free_events_.pop_back();
    }
    TV_CUDA_CHECK(cudaEventRecord(ev, stream));
    inflight_.push_back({head_, bytes, ev});
    head_ += (bytes + 255) & ~size_t(255);
    if (launches) ++*launches;
    return TV_OK;
  }

  struct Region {
    size_t off, len;
    cudaEvent_t ev;
  };
  int device_;
  std::mutex m_;
  char* host_ = nullptr;
  char* dev_ = nullptr;
  size_t cap_ = 0, head_ = 0;
  std::deque<Region> inflight_;
  std::vector<cudaEvent_t> free_events_;
};

// First-fit allocator over one device staging buffer; frees are deferred to events.
class StagingPool {
 public:
  StagingPool(int device, int64_t bytes) : device_(device), cap_(bytes) {}
  ~StagingPool() {
    cudaSetDevice(device_);
    for (auto& p : pending_) cudaEventDestroy(p.ev);
    if (base_) cudaFree(base_);
  }
  int init() {
    if (base_ || cap_ == 0) return TV_OK;
    TV_CUDA_CHECK(cudaMalloc(&base_, cap_));
    free_[0] = cap_;
    return TV_OK;
  }
  int64_t capacity() const { return cap_; }
  // Blocks until `bytes` (≤ capacity) are free; returns offset.
  int alloc(int64_t bytes, int64_t* off, ErrorSlot& err) {
    bytes = (bytes + 255) & ~int64_t(255);
    if (bytes > cap_) {
      set_error("staging request " + std::to_string(bytes) + " > capacity " +
                std::to_string(cap_));
      return TV_ERR_NOMEM;
    }
    std::unique_lock<std::mutex> g(m_);
    for (;;) {
      reap(false);
      for (auto it = free_.begin(); it != free_.end(); ++it) {
        if (it->second >= bytes) {
          *off = it->first;
          int64_t rest = it->second - bytes, at = it->first + bytes;
          free_.erase(it);
          if (rest) free_[at] = rest;
          return TV_OK;
        }
      }
      if (err.failed.load()) return TV_ERR_STATE;
      if (pending_.empty()) {
        g.unlock();
        std::this_thread::sleep_for(std::chrono::microseconds(50));
        g.lock();
        continue;
      }
      reap(true);  // wait for the oldest pending free
    }
  }
  // Free [off, off+bytes) once `ev` (recorded after the last reader) completes.
  void free_after(int64_t off, int64_t bytes, cudaEvent_t ev) {
    bytes = (bytes + 255) & ~int64_t(255);
    std::lock_guard<std::mutex> g(m_);
    pending_.push_back({off, bytes, ev});
  }
  char* base() const { return base_; }

 private:
  struct Pending {
    int64_t off, len;
    cudaEvent_t ev;
  };
  void release(int64_t off, int64_t len) {
    auto it = free_.emplace(off, len).first;
    auto next = std::next(it);
    if (next != free_.end() && it->first + it->second == next->first) {
      it->second += next->second;
      free_.erase(next);
    }
    if (it != free_.begin()) {
      auto prev = std::prev(it);
      if (prev->first + prev->second == it->first) {
        prev->second += it->second;
        free_.erase(it);
      }
    }
  }
  void reap(bool block) {
    while (!pending_.empty()) {
      auto& p = pending_.front();
      if (block) {
        cudaEventSynchronize(p.ev);
        block = false;
      } else if (cudaEventQuery(p.ev) != cudaSuccess) {
        break;
      }
      cudaEventDestroy(p.ev);
      release(p.off, p.len);
      pending_.pop_front();
    }
  }
  int device_;
  int64_t cap_;
  char* base_ = nullptr;
  std::mutex m_;
  std::map<int64_t, int64_t> free_;
  std::deque<Pending> pending_;
};

// DMA/kernel streams per device.  Work that must stay ordered (a slot's pack kernel and
// its D2H; an item's H2D pieces and its unpack) always goes to one stream, chosen by the
// slot / item index, so several copy engines can move independent slots at once.
int dma_streams() {
  const char* v = std::getenv("TVGPU_DMA_STREAMS");
  const int n = v ? std::atoi(v) : 1;
  return std::max(1, std::min(n, 16));
}

struct DeviceCtx {
  int device = -1;
  std::vector<cudaStream_t> streams;
  cudaStream_t zero_copy = nullptr;  // DMA straight into / out of registered file pages
  // packed zero-copy: strided boxes are packed here, then DMA'd into the registered file
  // (a small ring of its own: the save path's staging is indexed by pinned slot)
  char* zc_ring = nullptr;
  std::vector<cudaEvent_t> zc_ev;
  std::vector<char> zc_used;
  int zc_next = 0;
  std::unique_ptr<JobUploader> uploader;
  std::unique_ptr<StagingPool> staging;
  cudaStream_t stream_for(int64_t k) const { return streams[(size_t)(k % (int64_t)streams.size())]; }
};

}  // namespace
}  // namespace tv

struct tv_engine {
  int n_slots;
  int64_t slot_bytes;
  int64_t staging_bytes;
  int n_threads;
  std::vector<char*> slots;  // pinned
  char* ring = nullptr;       // one huge-page region holding every slot (TVGPU_HUGE_RING=1)
  size_t ring_bytes = 0;
  std::mutex dev_m;
  std::map<int, std::unique_ptr<tv::DeviceCtx>> devices;
  std::mutex call_m;  // one save/load at a time per engine
};

namespace tv {
namespace {

int device_ctx(tv_engine* e, int device, DeviceCtx** out) {
  std::lock_guard<std::mutex> g(e->dev_m);
  auto it = e->devices.find(device);
  if (it == e->devices.end()) {
    auto ctx = std::make_unique<DeviceCtx>();
    ctx->device = device;
    TV_CUDA_CHECK(cudaSetDevice(device));
    ctx->streams.resize(dma_streams());
    for (auto& st : ctx->streams) TV_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    TV_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->zero_copy, cudaStreamNonBlocking));
    ctx->uploader = std::make_unique<JobUploader>(device);
    ctx->staging = std::make_unique<StagingPool>(device, e->staging_bytes);
    int rc = ctx->staging->init();
    if (rc != TV_OK) return rc;
    it = e->devices.emplace(device, std::move(ctx)).first;
  }
  *out = it->second.get();
  return TV_OK;
}

int64_t box_bytes(const int64_t* ext, int rank, int isz) {
  int64_t n = isz;
  for (int i = 0; i < rank; ++i) n *= ext[i];
  return n;
}

// Split the box (origin `off`, extent `ext` inside an array) into consecutive sub-boxes
// of at most max_bytes each, in row-major payload order.
struct SubBox {
  int64_t off[TV_MAX_RANK];
  int64_t ext[TV_MAX_RANK];
  int64_t nbytes;
};
void split_box(const int64_t* off, const int64_t* ext, int rank, int isz, int64_t max_bytes,
               std::vector<SubBox>& out) {
  SubBox b;
  std::memcpy(b.off, off, sizeof(int64_t) * rank);
  std::memcpy(b.ext, ext, sizeof(int64_t) * rank);
  b.nbytes = box_bytes(ext, rank, isz);
  if (b.nbytes <= max_bytes || rank == 0) {
    out.push_back(b);
    return;
  }
  int d = 0;
  while (d < rank && ext[d] == 1) ++d;
  const int64_t row = b.nbytes / ext[d];
  if (row <= max_bytes) {
    const int64_t per = std::max<int64_t>(1, max_bytes / row);
    for (int64_t i = 0; i < ext[d]; i += per) {
      SubBox s = b;
      s.off[d] = off[d] + i;
      s.ext[d] = std::min(per, ext[d] - i);
      s.nbytes = row * s.ext[d];
      out.push_back(s);
    }
    return;
  }
  for (int64_t i = 0; i < ext[d]; ++i) {
    int64_t o2[TV_MAX_RANK], e2[TV_MAX_RANK];
    std::memcpy(o2, off, sizeof(int64_t) * rank);
    std::memcpy(e2, ext, sizeof(int64_t) * rank);
    o2[d] = off[d] + i;
    e2[d] = 1;
    split_box(o2, e2, rank, isz, max_bytes, out);
  }
}

// ---- save ------------------------------------------------------------------------------

struct WriteSeg {     // bytes of one output inside one slot
  int out;
  int64_t slot_off;
  int64_t file_off;
  int64_t n;
};
struct D2HSeg {       // contiguous device range → slot
  const char* src;
  int64_t slot_off;
  int64_t n;
};
struct SaveSlot {
  int index = -1;
  int lane = 0;
  int device = -1;
  int64_t fill = 0;
  std::vector<WriteSeg> writes;
  std::vector<D2HSeg> d2h;
  std::vector<tv_copy> packs;        // dst = staging
  std::vector<int64_t> pack_offs;    // slot offset of each pack
  cudaEvent_t ev = nullptr;
};

struct OutputState {
  std::string path;   // empty → host buffer
  char* host = nullptr;
  char* mapped = nullptr;  // registered page-cache mapping of a claimed recycled file
  int64_t direct = 0;      // bytes DMA'd straight into `mapped`
  int64_t size = 0;
  std::atomic<int64_t> left{0};
  std::once_flag opened;
  int fd = -1;
  std::atomic<bool> committed{false};
};

// Recycled files (FilesystemBackend page recycling): `<pool>/<size>/<name>` are whole
// files of exactly <size> bytes retired from older checkpoints.  An output of that size
// claims one by renaming it to its `.partial` name and overwrites every byte in place:
// the page cache already holds its pages, so the write skips page allocation and zeroing
// (and, in a VM, the host's re-fault of pages returned by free-page reporting).
class FilePool {
 public:
  explicit FilePool(std::string dir) : dir_(std::move(dir)) {}
  bool empty() const { return dir_.empty(); }
  // Move one pooled file of exactly `size` bytes to `dst`; false when none is left.
  bool claim(int64_t size, const std::string& dst) {
    Bucket* b = bucket(size);
    for (;;) {
      const size_t i = b->next.fetch_add(1);
      if (i >= b->names.size()) return false;
      if (::rename((b->dir + "/" + b->names[i]).c_str(), dst.c_str()) == 0) return true;
    }
  }

 private:
  struct Bucket {
    std::string dir;
    std::vector<std::string> names;
    std::atomic<size_t> next{0};
  };
  Bucket* bucket(int64_t size) {
    std::lock_guard<std::mutex> g(m_);
    auto it = buckets_.find(size);
    if (it != buckets_.end()) return it->second.get();
    auto b = std::make_unique<Bucket>();
    b->dir = dir_ + "/" + std::to_string(size);
    if (DIR* d = ::opendir(b->dir.c_str())) {
      while (struct dirent* ent = ::readdir(d)) {
        if (ent->d_name[0] == '.') continue;
        b->names.emplace_back(ent->d_name);
      }
      ::closedir(d);
    }
    Bucket* raw = b.get();
    buckets_.emplace(size, std::move(b));
    return raw;
  }
  std::string dir_;
  std::mutex m_;
  std::map<int64_t, std::unique_ptr<Bucket>> buckets_;
};

class SaveRun {
 public:
  SaveRun(tv_engine* e, const tv_write_item* items, int n_items, const tv_output* outs,
          int n_outs, tv_stats* st, const char* pool_dir = nullptr, int pool_flags = 0)
      : e_(e), items_(items), n_items_(n_items), n_outs_(n_outs), stats_(st),
        pool_(pool_dir ? pool_dir : ""), pool_flags_(pool_flags) {
    outs_.reset(new OutputState[n_outs]);
    for (int i = 0; i < n_outs; ++i) {
      outs_[i].path = outs[i].path ? outs[i].path : "";
      outs_[i].host = reinterpret_cast<char*>(outs[i].host);
      outs_[i].size = outs[i].size;
      outs_[i].left.store(outs[i].size);
    }
    claimed_.assign(n_outs > 0 ? n_outs : 1, 0);
  }

  int run() {
    const double t0 = now_s();
    // Validate coverage: every output byte must be produced exactly by the items.
    std::vector<int64_t> produced(n_outs_, 0);
    for (int i = 0; i < n_items_; ++i) {
      const auto& it = items_[i];
      if (it.file < 0 || it.file >= n_outs_ || it.rank < 0 || it.rank > TV_MAX_RANK ||
          it.itemsize <= 0) {
        set_error("malformed write item " + std::to_string(i));
        return TV_ERR_ARG;
      }
      int64_t n = box_bytes(it.ext, it.rank, it.itemsize);
      if (it.file_off < 0 || it.file_off + n > outs_[it.file].size) {
        set_error("write item " + std::to_string(i) + " outside its output");
        return TV_ERR_ARG;
      }
      produced[it.file] += n;
    }
    for (int o = 0; o < n_outs_; ++o) {
      if (produced[o] != outs_[o].size) {
        set_error("output " + std::to_string(o) + " covered by " + std::to_string(produced[o]) +
                  " of " + std::to_string(outs_[o].size) + " bytes");
        return TV_ERR_ARG;
      }
    }
    for (int s = 0; s < e_->n_slots; ++s) free_slots_.push(s);
    direct_.assign(n_items_, 0);
    if (!pool_.empty()) claim_outputs();
    assign_lanes();
    std::vector<std::thread> writers;
    for (int t = 0; t < (int)lanes_.size(); ++t) writers.emplace_back([this, t] { writer_loop(t); });
    // Zero-byte outputs are committed up front.
    for (int o = 0; o < n_outs_; ++o)
      if (outs_[o].size == 0) finish_output(o);
    std::thread zero_copy;
    if (!zq_.empty()) zero_copy = std::thread([this] { zero_copy_loop(); });
    produce();
    if (steal_) {
      // the slot path takes zero-copy items from the back of the queue while the DMA
      // path takes them from the front: the two paths split the work at their own rates
      while (!err_.failed.load()) {
        std::vector<int> batch;
        for (int k = 0; k < std::max(1, e_->n_threads); ++k) {
          int i;
          if (!take_back(&i)) break;
          batch.push_back(i);
        }
        if (batch.empty()) break;
        for (int i : batch) cursors_[lane_of_[items_[i].file]].items.push_back(i);
        produce();
      }
    }
    for (auto& q : lanes_) q->close();
    for (auto& w : writers) w.join();
    if (zero_copy.joinable()) zero_copy.join();
    for (auto& ev : events_) cudaEventDestroy(ev);
    if (err_.failed.load()) {
      abort_outputs();
      set_error(err_.msg);
      return err_.code;
    }
    stats_->seconds_total += now_s() - t0;
    return TV_OK;
  }

 private:
  // Files are distributed over writer lanes (one per storage thread), largest first onto
  // the least-loaded lane: a file is only ever written by its lane's thread, because
  // tmpfs (and most local filesystems) serialise concurrent writes to one inode.  The
  // producer fills slots round-robin across lanes so every lane streams concurrently.
  struct LaneCursor {
    std::vector<int> items;  // item indices of this lane's files, in item order
    size_t pos = 0;
    int64_t done = 0;        // payload bytes of items[pos] already placed
    std::vector<SubBox> subs;
    size_t sub_pos = 0;
    bool split = false;
    bool finished() const { return pos >= items.size(); }
  };

  // Zero-copy path (registered recycle pool, tv_mapped.cpp).  Outputs are opened up
  // front: each claims a recycled file of its size; when that file's pages are
  // registered, every contiguous item of the output is DMA'd straight into them and
  // never touches a pinned slot or a writer thread.
  void claim_outputs() {
    {
      int64_t total = 0;
      for (int o = 0; o < n_outs_; ++o) total += outs_[o].size;
      const char* v = std::getenv("TVGPU_REGISTER_BUDGET");
      const double frac = v ? std::atof(v) : 1.0;
      register_budget_.store((int64_t)(frac * (double)total));
    }
    // outputs are claimed by a few threads (rename + open + inode lookup)
    std::atomic<int> next{0};
    auto work = [&] {
      for (int o = next.fetch_add(1); o < n_outs_ && !err_.failed.load(); o = next.fetch_add(1))
        claim_output(o);
    };
    const int t = std::max(1, std::min({8, e_->n_threads, n_outs_}));
    std::vector<std::thread> pool;
    for (int k = 1; k < t; ++k) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    if (pool_flags_ & TV_POOL_REGISTER) {
      // Files this process claims for the first time are registered now, one after the
      // other (concurrent cudaHostRegister calls serialise in the driver and slow each
      // other down; a background registrar slowed the concurrent saves): once per file
      // lifetime, within TVGPU_REGISTER_BUDGET (default 1.0) of this save's bytes.
      for (int o = 0; o < n_outs_ && !err_.failed.load(); ++o) {
        OutputState& out = outs_[o];
        if (out.fd < 0 || !claimed_[o] || out.mapped) continue;
        if (register_budget_.fetch_sub(out.size) < out.size) continue;
        out.mapped = mapping_register_fd(out.fd, out.size, true);
        registered_now_ += 1;
      }
    }
    // registered outputs take the zero-copy path only when this save chose it
    if (!(pool_flags_ & TV_POOL_ZERO_COPY))
      for (int o = 0; o < n_outs_; ++o) outs_[o].mapped = nullptr;
    build_zero_copy_queue();
  }

  void claim_output(int o) {
    OutputState& out = outs_[o];
    if (out.path.empty() || out.size == 0) return;
    std::call_once(out.opened, [&] { open_output(out); });
    if (out.fd < 0 || !claimed_[o]) return;
    // a recycled file keeps its registration from earlier generations (cached by inode)
    if (pool_flags_ & (TV_POOL_REGISTER | TV_POOL_ZERO_COPY)) out.mapped = mapping_for_fd(out.fd, out.size);
  }

  void build_zero_copy_queue() {
    for (int i = 0; i < n_items_; ++i) {
      const auto& it = items_[i];
      const int64_t n = box_bytes(it.ext, it.rank, it.itemsize);
      if (n > 0 && outs_[it.file].mapped) {  // contiguous: one DMA; strided: pack + DMA
        direct_[i] = 1;
        zq_.push_back(i);
      }
    }
    zhi_ = zq_.size();
    const char* v = std::getenv("TVGPU_SAVE_STEAL");
    steal_ = v ? std::atoi(v) != 0 : false;
  }

  bool take_front(int* i) {
    std::lock_guard<std::mutex> g(zq_m_);
    if (zlo_ >= zhi_) return false;
    *i = zq_[zlo_++];
    return true;
  }
  bool take_back(int* i) {
    std::lock_guard<std::mutex> g(zq_m_);
    if (zlo_ >= zhi_) return false;
    *i = zq_[--zhi_];
    return true;
  }

  // D2H of `n` contiguous device bytes into a registered file mapping at `file_off`,
  // never across a registration piece.
  bool dma_into_file(const char* src, char* mapped, int64_t file_off, int64_t n, cudaStream_t st) {
    for (int64_t a = 0; a < n;) {
      const int64_t at = file_off + a;
      const int64_t k = std::min(n - a, (at / kRegisterPiece + 1) * kRegisterPiece - at);
      if (cudaMemcpyAsync(mapped + at, src + a, k, cudaMemcpyDefault, st) != cudaSuccess) return false;
      a += k;
    }
    return true;
  }

  // A strided box (e.g. a replica-parallel column segment): packed by the box-copy kernel
  // into a staging chunk of the device's zero-copy ring, then DMA'd into the file, chunk by
  // chunk in payload order (split_box keeps the file contiguous), all on the zero-copy
  // stream; a ring chunk is reused after its DMA's event.
  bool pack_into_file(const tv_write_item& it, DeviceCtx* ctx) {
    constexpr int kChunks = 4;
    const int64_t chunk = kRegisterPiece;
    if (!ctx->zc_ring) {
      if (cudaMalloc(&ctx->zc_ring, kChunks * chunk) != cudaSuccess) {
        err_.set(TV_ERR_NOMEM, "zero-copy pack ring");
        return false;
      }
      ctx->zc_ev.assign(kChunks, nullptr);
      ctx->zc_used.assign(kChunks, 0);
      for (auto& ev : ctx->zc_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    }
    std::vector<SubBox> subs;
    split_box(it.src.off, it.ext, it.rank, it.itemsize, chunk, subs);
    int64_t pos = it.file_off;
    for (const SubBox& sb : subs) {
      const int slot = ctx->zc_next;
      ctx->zc_next = (slot + 1) % kChunks;
      if (ctx->zc_used[slot]) cudaEventSynchronize(ctx->zc_ev[slot]);
      char* stage = ctx->zc_ring + (int64_t)slot * chunk;
      tv_copy cp{};
      cp.src = it.src;
      std::memcpy(cp.src.off, sb.off, sizeof(int64_t) * it.rank);
      std::memcpy(cp.ext, sb.ext, sizeof(int64_t) * it.rank);
      cp.rank = it.rank;
      cp.itemsize = it.itemsize;
      cp.dst.base = reinterpret_cast<uint64_t>(stage);
      for (int d = 0; d < it.rank; ++d) {
        cp.dst.shape[d] = sb.ext[d];
        cp.dst.off[d] = 0;
      }
      std::vector<CopyJob> jobs;
      std::string why;
      if (!normalize(cp, jobs, why)) {
        err_.set(TV_ERR_ARG, "pack: " + why);
        return false;
      }
      int64_t launches = 0;
      int rc = ctx->uploader->run(jobs, ctx->zero_copy, &launches);
      if (rc != TV_OK) {
        err_.set(rc, get_error());
        return false;
      }
      stats_launches_ += launches;
      stats_bytes_packed_ += sb.nbytes;
      if (!dma_into_file(stage, outs_[it.file].mapped, pos, sb.nbytes, ctx->zero_copy) ||
          cudaEventRecord(ctx->zc_ev[slot], ctx->zero_copy) != cudaSuccess)
        return false;
      ctx->zc_used[slot] = 1;
      pos += sb.nbytes;
    }
    return true;
  }

  // The DMA path: zero-copy items from the front of the queue, D2H straight into the
  // registered pages of their output on the device's zero-copy stream, at most `window`
  // bytes in flight; an item's bytes count toward its output once its event completed.
  void zero_copy_loop() {
    const char* w = std::getenv("TVGPU_ZC_WINDOW");
    const int64_t window = w ? std::atoll(w) : (int64_t)1 << 30;
    struct Flight {
      int item;
      int device;
      int64_t n;
      cudaEvent_t ev;
    };
    std::deque<Flight> flight;
    int64_t in_flight = 0;
    auto retire = [&](const Flight& f) {
      cudaSetDevice(f.device);
      const double t0 = now_s();
      cudaError_t ce = cudaEventSynchronize(f.ev);
      wait_dma_.add(now_s() - t0);
      cudaEventDestroy(f.ev);
      if (ce != cudaSuccess) {
        err_.set(TV_ERR_CUDA, std::string("zero-copy D2H: ") + cudaGetErrorString(ce));
        return false;
      }
      stats_bytes_storage_ += f.n;
      zero_copy_bytes_ += f.n;
      OutputState& o = outs_[items_[f.item].file];
      if (o.left.fetch_sub(f.n) == f.n) return finish_output(items_[f.item].file);
      return true;
    };
    int i;
    while (!err_.failed.load() && take_front(&i)) {
      const auto& it = items_[i];
      DeviceCtx* ctx = nullptr;
      int rc = device_ctx(e_, it.device, &ctx);
      if (rc != TV_OK) {
        err_.set(rc, get_error());
        break;
      }
      cudaSetDevice(it.device);
      int64_t boff = 0, bn = 0;
      cudaEvent_t ev;
      bool ok = true;
      if (box_contiguous(it.src, it.ext, it.rank, it.itemsize, &boff, &bn)) {
        ok = dma_into_file(reinterpret_cast<const char*>(it.src.base) + boff, outs_[it.file].mapped,
                           it.file_off, bn, ctx->zero_copy);
      } else {
        bn = box_bytes(it.ext, it.rank, it.itemsize);
        ok = pack_into_file(it, ctx);
      }
      if (!ok || cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventRecord(ev, ctx->zero_copy) != cudaSuccess) {
        err_.set(TV_ERR_CUDA, std::string("zero-copy D2H: ") + cudaGetErrorString(cudaGetLastError()));
        break;
      }
      stats_dma_ += 1;
      stats_bytes_device_ += bn;
      flight.push_back({i, it.device, bn, ev});
      in_flight += bn;
      while (in_flight > window && !flight.empty()) {
        Flight f = flight.front();
        flight.pop_front();
        in_flight -= f.n;
        if (!retire(f)) break;
      }
    }
    while (!flight.empty()) {  // drain (also after an error: no event is left behind)
      Flight f = flight.front();
      flight.pop_front();
      if (err_.failed.load()) {
        cudaSetDevice(f.device);
        cudaEventSynchronize(f.ev);
        cudaEventDestroy(f.ev);
        continue;
      }
      retire(f);
    }
  }

  void assign_lanes() {
    const int L = std::max(1, e_->n_threads);
    lanes_.clear();
    for (int k = 0; k < L; ++k) lanes_.emplace_back(new Queue<SaveSlot>());
    inflight_.reset(new std::atomic<int>[L]);
    for (int k = 0; k < L; ++k) inflight_[k] = 0;
    cursors_.assign(L, LaneCursor());
    std::vector<int> order(n_outs_);
    for (int o = 0; o < n_outs_; ++o) order[o] = o;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return outs_[a].size > outs_[b].size; });
    std::vector<int64_t> load(L, 0);
    lane_of_.assign(n_outs_, 0);
    for (int o : order) {
      int best = 0;
      for (int k = 1; k < L; ++k)
        if (load[k] < load[best]) best = k;
      lane_of_[o] = best;
      load[best] += std::max<int64_t>(outs_[o].size, 1);
    }
    for (int i = 0; i < n_items_; ++i)
      if (!direct_[i]) cursors_[lane_of_[items_[i].file]].items.push_back(i);
  }

  // Fill slot `cur` from lane `k`; returns false on error.
  bool fill_slot(LaneCursor& c, SaveSlot& cur) {
    const int64_t cap = e_->slot_bytes;
    const size_t max_packs = 512;
    while (!c.finished()) {
      const auto& it = items_[c.items[c.pos]];
      const int64_t n = box_bytes(it.ext, it.rank, it.itemsize);
      if (n == 0) {
        ++c.pos;
        continue;
      }
      if (cur.device >= 0 && cur.device != it.device) return true;
      int64_t boff = 0, bn = 0;
      if (box_contiguous(it.src, it.ext, it.rank, it.itemsize, &boff, &bn)) {
        const int64_t take = std::min(n - c.done, cap - cur.fill);
        if (take <= 0) return true;
        const char* src = reinterpret_cast<const char*>(it.src.base) + boff + c.done;
        cur.device = it.device;
        cur.d2h.push_back({src, cur.fill, take});
        cur.writes.push_back({it.file, cur.fill, it.file_off + c.done, take});
        cur.fill += take;
        c.done += take;
        if (c.done == n) {
          ++c.pos;
          c.done = 0;
        }
        continue;
      }
      if (!c.split) {
        c.subs.clear();
        split_box(it.src.off, it.ext, it.rank, it.itemsize, cap, c.subs);
        c.sub_pos = 0;
        c.split = true;
      }
      const SubBox& sb = c.subs[c.sub_pos];
      if (cur.fill + sb.nbytes > cap || cur.packs.size() >= max_packs) return true;
      tv_copy cp{};
      cp.src = it.src;
      std::memcpy(cp.src.off, sb.off, sizeof(int64_t) * it.rank);
      std::memcpy(cp.ext, sb.ext, sizeof(int64_t) * it.rank);
      cp.rank = it.rank;
      cp.itemsize = it.itemsize;
      for (int d = 0; d < it.rank; ++d) {
        cp.dst.shape[d] = sb.ext[d];  // dst base set in submit() (staging address)
        cp.dst.off[d] = 0;
      }
      cur.device = it.device;
      cur.packs.push_back(cp);
      cur.pack_offs.push_back(cur.fill);
      cur.writes.push_back({it.file, cur.fill, it.file_off + c.done, sb.nbytes});
      cur.fill += sb.nbytes;
      c.done += sb.nbytes;
      if (++c.sub_pos == c.subs.size()) {
        ++c.pos;
        c.done = 0;
        c.split = false;
      }
    }
    return true;
  }

  void produce() {
    std::vector<int> active;
    for (size_t k = 0; k < cursors_.size(); ++k)
      if (!cursors_[k].finished()) active.push_back((int)k);
    // A lane never holds more than its share of the ring, so a slow writer cannot starve
    // the others of slots.
    const int cap = std::max(2, (int)(2 * e_->n_slots / std::max<size_t>(1, active.size())));
    while (!active.empty() && !err_.failed.load()) {
      std::vector<int> still;
      bool progressed = false;
      for (int k : active) {
        if (err_.failed.load()) return;
        if (inflight_[k].load() >= cap) {
          still.push_back(k);
          continue;
        }
        progressed = true;
        int s;
        const double t0 = now_s();
        if (!free_slots_.pop(s)) return;
        wait_slot_.add(now_s() - t0);
        inflight_[k]++;
        SaveSlot cur;
        cur.index = s;
        cur.lane = k;
        if (!fill_slot(cursors_[k], cur)) return;
        if (cur.fill == 0 && cur.writes.empty()) {
          inflight_[k]--;
          free_slots_.push(s);
        } else if (!submit(cur)) {
          return;
        }
        if (!cursors_[k].finished()) still.push_back(k);
      }
      active.swap(still);
      if (!progressed) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }

  bool submit(SaveSlot& s) {
    DeviceCtx* ctx = nullptr;
    int rc = device_ctx(e_, s.device, &ctx);
    if (rc != TV_OK) {
      err_.set(rc, get_error());
      return false;
    }
    if (cudaSetDevice(s.device) != cudaSuccess) {
      err_.set(TV_ERR_CUDA, "cudaSetDevice failed");
      return false;
    }
    char* host = e_->slots[s.index];
    cudaStream_t stream = ctx->stream_for(s.index);
    if (!s.packs.empty()) {
      if (ctx->staging->capacity() < (int64_t)e_->n_slots * e_->slot_bytes) {
        err_.set(TV_ERR_NOMEM, "device staging smaller than n_slots*slot_bytes");
        return false;
      }
      char* stage = ctx->staging->base() + (int64_t)s.index * e_->slot_bytes;
      std::vector<CopyJob> jobs;
      std::string why;
      for (size_t k = 0; k < s.packs.size(); ++k) {
        s.packs[k].dst.base = reinterpret_cast<uint64_t>(stage + s.pack_offs[k]);
        if (!normalize(s.packs[k], jobs, why)) {
          err_.set(TV_ERR_ARG, "pack: " + why);
          return false;
        }
        stats_bytes_packed_ += box_bytes(s.packs[k].ext, s.packs[k].rank, s.packs[k].itemsize);
      }
      int64_t launches = 0;
      rc = ctx->uploader->run(jobs, stream, &launches);
      if (rc != TV_OK) {
        err_.set(rc, get_error());
        return false;
      }
      stats_launches_ += launches;
      // D2H the packed bytes (adjacent packs coalesced).
      for (size_t k = 0; k < s.packs.size();) {
        int64_t start = s.pack_offs[k];
        int64_t end = start + box_bytes(s.packs[k].ext, s.packs[k].rank, s.packs[k].itemsize);
        size_t j = k + 1;
        while (j < s.packs.size() && s.pack_offs[j] == end) {
          end += box_bytes(s.packs[j].ext, s.packs[j].rank, s.packs[j].itemsize);
          ++j;
        }
        s.d2h.push_back({stage + start, start, end - start});
        k = j;
      }
    }
    for (auto& d : s.d2h) {
      // cudaMemcpyDefault: the source is HBM, or pinned host memory when the async
      // snapshot fell back to a host arena (save_pipeline._snapshot_arena); UVA resolves it.
      if (cudaMemcpyAsync(host + d.slot_off, d.src, d.n, cudaMemcpyDefault, stream) !=
          cudaSuccess) {
        err_.set(TV_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(cudaGetLastError()));
        return false;
      }
      stats_dma_ += 1;
      stats_bytes_device_ += d.n;
    }
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, stream) != cudaSuccess) {
      err_.set(TV_ERR_CUDA, "event record failed");
      return false;
    }
    {
      std::lock_guard<std::mutex> g(ev_m_);
      events_.push_back(ev);
    }
    s.ev = ev;
    lanes_[s.lane]->push(std::move(s));
    return true;
  }

  void writer_loop(int lane) {
    SaveSlot s;
    while (lanes_[lane]->pop(s)) {
      if (!err_.failed.load()) {
        const double t0 = now_s();
        cudaError_t ce = cudaEventSynchronize(s.ev);
        wait_dma_.add(now_s() - t0);
        if (ce != cudaSuccess) err_.set(TV_ERR_CUDA, std::string("D2H/pack: ") + cudaGetErrorString(ce));
      }
      if (!err_.failed.load()) {
        const char* host = e_->slots[s.index];
        const double t0 = now_s();
        for (auto& w : s.writes) {
          if (!write_seg(w, host)) break;
        }
        io_.add(now_s() - t0);
      }
      inflight_[lane]--;
      free_slots_.push(s.index);
    }
  }

  bool write_seg(const WriteSeg& w, const char* host) {
    OutputState& o = outs_[w.out];
    if (o.path.empty()) {
      std::memcpy(o.host + w.file_off, host + w.slot_off, w.n);
    } else {
      std::call_once(o.opened, [&] { open_output(o); });
      if (o.fd < 0) return false;
      int64_t done = 0;
      while (done < w.n) {
        ssize_t r = ::pwrite(o.fd, host + w.slot_off + done, w.n - done, w.file_off + done);
        if (r < 0) {
          if (errno == EINTR) continue;
          err_.set(TV_ERR_IO, errno_msg("pwrite", o.path));
          return false;
        }
        done += r;
      }
    }
    stats_bytes_storage_ += w.n;
    if (o.left.fetch_sub(w.n) == w.n) return finish_output(w.out);
    return true;
  }

  // `<path>.partial`, write-only: a recycled file of the output's exact size when the
  // pool has one (overwritten in full: run() checked every byte is produced), else new.
  void open_output(OutputState& o) {
    std::string err;
    if (!dirs_.ensure(parent_of(o.path), err)) {
      err_.set(TV_ERR_IO, err);
      return;
    }
    std::string tmp = o.path + ".partial";
    if (!pool_.empty() && o.size > 0 && pool_.claim(o.size, tmp)) {
      o.fd = ::open(tmp.c_str(), O_RDWR | O_CLOEXEC);  // read-write: mmap-able
      if (o.fd >= 0) {
        recycled_ += 1;
        claimed_[&o - outs_.get()] = 1;
        return;
      }
    }
    o.fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0666);
    if (o.fd < 0) err_.set(TV_ERR_IO, errno_msg("open", tmp));
  }

  bool finish_output(int idx) {
    OutputState& o = outs_[idx];
    if (o.path.empty()) {
      o.committed.store(true);
      return true;
    }
    if (o.size == 0) {
      std::call_once(o.opened, [&] { open_output(o); });
      if (o.fd < 0) return false;
    }
    if (o.mapped) ::futimens(o.fd, nullptr);  // DMA'd bytes do not touch the mtime
    if (::close(o.fd) != 0) {
      err_.set(TV_ERR_IO, errno_msg("close", o.path));
      return false;
    }
    o.fd = -1;
    std::string tmp = o.path + ".partial";
    if (::rename(tmp.c_str(), o.path.c_str()) != 0) {
      err_.set(TV_ERR_IO, errno_msg("rename", tmp));
      return false;
    }
    o.committed.store(true);
    files_ += 1;
    return true;
  }

  void abort_outputs() {
    for (int i = 0; i < n_outs_; ++i) {
      OutputState& o = outs_[i];
      if (o.path.empty() || o.committed.load()) continue;
      if (o.fd >= 0) {
        if (o.mapped) mapping_release_fd(o.fd);  // its pages go with the file
        ::close(o.fd);
        o.fd = -1;
        ::unlink((o.path + ".partial").c_str());
      }
    }
  }

 public:
  void publish_stats() {
    stats_->bytes_device += stats_bytes_device_.load();
    stats_->bytes_storage += stats_bytes_storage_.load();
    stats_->bytes_packed += stats_bytes_packed_.load();
    stats_->kernel_launches += stats_launches_.load();
    stats_->dma_copies += stats_dma_.load();
    stats_->files += files_.load();
    stats_->recycled_files += recycled_.load();
    stats_->zero_copy_bytes += zero_copy_bytes_.load();
    stats_->seconds_io += io_.seconds();
    stats_->seconds_wait_dma += wait_dma_.seconds();
    stats_->seconds_wait_slot += wait_slot_.seconds();
  }

 private:
  tv_engine* e_;
  const tv_write_item* items_;
  int n_items_;
  int n_outs_;
  tv_stats* stats_;
  FilePool pool_;
  const int pool_flags_;
  std::atomic<int64_t> recycled_{0}, zero_copy_bytes_{0}, register_budget_{0}, registered_now_{0};
  std::vector<char> claimed_;                      // output claimed a recycled file
  std::vector<char> direct_;                       // item eligible for the zero-copy path
  std::vector<int> zq_;                            // zero-copy queue (item order)
  std::mutex zq_m_;
  size_t zlo_ = 0, zhi_ = 0;                       // front (DMA path) / back (slot path)
  bool steal_ = false;                             // TVGPU_SAVE_STEAL: slot path steals from the back
  std::unique_ptr<OutputState[]> outs_;
  Queue<int> free_slots_;
  std::vector<std::unique_ptr<Queue<SaveSlot>>> lanes_;
  std::unique_ptr<std::atomic<int>[]> inflight_;
  std::vector<LaneCursor> cursors_;
  Clock io_, wait_dma_, wait_slot_;
  std::vector<int> lane_of_;
  ErrorSlot err_;
  DirMaker dirs_;
  std::mutex ev_m_;
  std::vector<cudaEvent_t> events_;
  std::atomic<int64_t> stats_bytes_device_{0}, stats_bytes_storage_{0}, stats_bytes_packed_{0},
      stats_launches_{0}, stats_dma_{0}, files_{0};
};

// ---- restore -----------------------------------------------------------------------------

struct InputState {
  std::string path;
  const char* host = nullptr;
  int64_t size = 0;
  std::once_flag opened;
  int fd = -1;
  const char* mapped = nullptr;  // registered page-cache mapping (zero-copy H2D source)
};

struct ItemState {
  std::atomic<int> left{0};
  char* base = nullptr;      // landing address on the reader device
  int64_t staged_off = -1;   // staging offset when not direct
};

struct ReadTask {
  int item;
  int slot;
  int64_t off;   // within the item
  int64_t n;
};

class LoadRun {
 public:
  LoadRun(tv_engine* e, const tv_read_item* items, int n_items, const tv_input* ins, int n_ins,
          const tv_copy* copies, int n_copies, tv_stats* st)
      : e_(e), items_(items), n_items_(n_items), n_ins_(n_ins), copies_(copies),
        n_copies_(n_copies), stats_(st) {
    ins_.reset(new InputState[n_ins]);
    for (int i = 0; i < n_ins; ++i) {
      ins_[i].path = ins[i].path ? ins[i].path : "";
      ins_[i].host = reinterpret_cast<const char*>(ins[i].host);
      ins_[i].size = ins[i].size;
    }
    states_.reset(new ItemState[n_items > 0 ? n_items : 1]);
    slot_events_.assign(e->n_slots, nullptr);
    slot_event_dev_.assign(e->n_slots, -1);
  }

  int run() {
    const double t0 = now_s();
    for (int i = 0; i < n_items_; ++i) {
      const auto& it = items_[i];
      if (it.input < 0 || it.input >= n_ins_ || it.nbytes < 0 || it.first_copy < 0 ||
          it.n_copies < 0 || it.first_copy + it.n_copies > n_copies_) {
        set_error("malformed read item " + std::to_string(i));
        return TV_ERR_ARG;
      }
      if (ins_[it.input].size >= 0 && it.in_off + it.nbytes > ins_[it.input].size) {
        set_error("read item " + std::to_string(i) + " beyond the end of its input");
        return TV_ERR_ARG;
      }
      if (it.direct_dst == 0 && it.n_copies == 0) {
        set_error("read item " + std::to_string(i) + " has no destination");
        return TV_ERR_ARG;
      }
    }
    for (int s = 0; s < e_->n_slots; ++s) free_slots_.push(s);
    std::vector<std::thread> readers;
    for (int t = 0; t < e_->n_threads; ++t) readers.emplace_back([this] { reader_loop(); });
    produce();
    tasks_.close();
    for (auto& r : readers) r.join();
    // Drain all devices used.
    for (auto& kv : used_devices_) {
      cudaSetDevice(kv.first);
      for (cudaStream_t st : kv.second->streams) {
        cudaError_t ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) err_.set(TV_ERR_CUDA, std::string("restore stream: ") + cudaGetErrorString(ce));
      }
    }
    for (int s = 0; s < e_->n_slots; ++s)
      if (slot_events_[s]) cudaEventDestroy(slot_events_[s]);
    for (int i = 0; i < n_ins_; ++i)
      if (ins_[i].fd >= 0) ::close(ins_[i].fd);
    if (err_.failed.load()) {
      set_error(err_.msg);
      return err_.code;
    }
    stats_->seconds_total += now_s() - t0;
    return TV_OK;
  }

  void publish_stats() {
    stats_->bytes_device += bytes_device_.load();
    stats_->bytes_storage += bytes_storage_.load();
    stats_->bytes_packed += bytes_packed_.load();
    stats_->kernel_launches += launches_.load();
    stats_->dma_copies += dma_.load();
    stats_->files += files_.load();
    stats_->zero_copy_bytes += zero_copy_bytes_.load();
    stats_->seconds_io += io_.seconds();
    stats_->seconds_wait_dma += wait_dma_.seconds();
    stats_->seconds_wait_slot += wait_slot_.seconds();
  }

 private:
  DeviceCtx* ctx_for(int device) {
    std::lock_guard<std::mutex> g(used_m_);
    auto it = used_devices_.find(device);
    if (it != used_devices_.end()) return it->second;
    DeviceCtx* ctx = nullptr;
    int rc = device_ctx(e_, device, &ctx);
    if (rc != TV_OK) {
      err_.set(rc, get_error());
      return nullptr;
    }
    used_devices_[device] = ctx;
    return ctx;
  }

  int acquire_slot() {
    int s;
    const double t0 = now_s();
    if (!free_slots_.pop(s)) return -1;
    const double t1 = now_s();
    wait_slot_.add(t1 - t0);
    if (slot_events_[s]) {
      cudaSetDevice(slot_event_dev_[s]);
      cudaEventSynchronize(slot_events_[s]);  // previous H2D out of this slot done
    }
    wait_dma_.add(now_s() - t1);
    return s;
  }

  void produce() {
    const int64_t cap = e_->slot_bytes;
    for (int i = 0; i < n_items_ && !err_.failed.load(); ++i) {
      const auto& it = items_[i];
      if (it.nbytes == 0) continue;  // nothing to land, nothing to scatter
      DeviceCtx* ctx = ctx_for(it.device);
      if (!ctx) return;
      ItemState& st = states_[i];
      if (it.direct_dst) {
        st.base = reinterpret_cast<char*>(it.direct_dst);
      } else {
        int64_t off = 0;
        int rc = ctx->staging->alloc(it.nbytes, &off, err_);
        if (rc != TV_OK) {
          err_.set(rc, get_error());
          return;
        }
        st.staged_off = off;
        st.base = ctx->staging->base() + off;
      }
      if (maps_ && ins_[it.input].host == nullptr) {
        InputState& in = ins_[it.input];
        std::call_once(in.opened, [&] { open_input(in); });
        if (err_.failed.load()) return;
        if (in.mapped) {
          if (!run_mapped(i, in.mapped)) return;
          continue;
        }
      }
      const int pieces = (int)((it.nbytes + cap - 1) / cap);
      st.left.store(pieces);
      for (int p = 0; p < pieces; ++p) {
        int s = acquire_slot();
        if (s < 0 || err_.failed.load()) return;
        const int64_t off = (int64_t)p * cap;
        tasks_.push({i, s, off, std::min(cap, it.nbytes - off)});
      }
    }
  }

  void reader_loop() {
    ReadTask t;
    while (tasks_.pop(t)) {
      bool released = false;
      if (!err_.failed.load()) released = run_task(t);
      if (!released) free_slots_.push(t.slot);
    }
  }

  bool fetch(InputState& in, char* dst, int64_t off, int64_t n) {
    if (in.path.empty()) {
      std::memcpy(dst, in.host + off, n);
      return true;
    }
    std::call_once(in.opened, [&] { open_input(in); });
    if (in.fd < 0) return false;
    int64_t done = 0;
    while (done < n) {
      ssize_t r = ::pread(in.fd, dst + done, n - done, off + done);
      if (r < 0) {
        if (errno == EINTR) continue;
        err_.set(TV_ERR_IO, errno_msg("pread", in.path));
        return false;
      }
      if (r == 0) {
        err_.set(TV_ERR_IO, "short read from " + in.path);
        return false;
      }
      done += r;
    }
    return true;
  }

  void open_input(InputState& in) {
    in.fd = ::open(in.path.c_str(), O_RDONLY | O_CLOEXEC);
    if (in.fd < 0) {
      err_.set(TV_ERR_IO, errno_msg("open", in.path));
      return;
    }
    files_ += 1;
    if (maps_) in.mapped = mapping_for_fd(in.fd, in.size);
  }

  // Zero-copy restore of an item whose file is a registered mapping: H2D straight from
  // the page-cache pages (no pread, no slot), then its copies, on the item's stream.
  bool run_mapped(int i, const char* src) {
    const auto& it = items_[i];
    ItemState& st = states_[i];
    DeviceCtx* ctx = ctx_for(it.device);
    if (!ctx) return false;
    cudaSetDevice(it.device);
    cudaStream_t stream = ctx->stream_for(i);
    for (int64_t a = 0; a < it.nbytes;) {  // never across a registration piece
      const int64_t at = it.in_off + a;
      const int64_t n = std::min(it.nbytes - a, (at / kRegisterPiece + 1) * kRegisterPiece - at);
      if (cudaMemcpyAsync(st.base + a, src + at, n, cudaMemcpyDefault, stream) != cudaSuccess) {
        err_.set(TV_ERR_CUDA, std::string("zero-copy H2D: ") + cudaGetErrorString(cudaGetLastError()));
        return false;
      }
      a += n;
    }
    dma_ += 1;
    bytes_device_ += it.nbytes;
    bytes_storage_ += it.nbytes;
    zero_copy_bytes_ += it.nbytes;
    launch_copies(i);
    return !err_.failed.load();
  }

  // Returns true when the slot has been handed back to the free list.
  bool run_task(const ReadTask& t) {
    const auto& it = items_[t.item];
    ItemState& st = states_[t.item];
    char* host = e_->slots[t.slot];
    const double t0 = now_s();
    if (!fetch(ins_[it.input], host, it.in_off + t.off, t.n)) return false;
    io_.add(now_s() - t0);
    bytes_storage_ += t.n;
    DeviceCtx* ctx = ctx_for(it.device);
    if (!ctx) return false;
    cudaSetDevice(it.device);
    cudaStream_t stream = ctx->stream_for(t.item);  // every piece of an item: one stream
    if (cudaMemcpyAsync(st.base + t.off, host, t.n, cudaMemcpyHostToDevice, stream) !=
        cudaSuccess) {
      err_.set(TV_ERR_CUDA, std::string("H2D: ") + cudaGetErrorString(cudaGetLastError()));
      return false;
    }
    dma_ += 1;
    bytes_device_ += t.n;
    cudaEvent_t& ev = slot_events_[t.slot];
    if (ev && slot_event_dev_[t.slot] != it.device) {
      cudaEventDestroy(ev);
      ev = nullptr;
    }
    if (!ev) {
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      slot_event_dev_[t.slot] = it.device;
    }
    cudaEventRecord(ev, stream);
    free_slots_.push(t.slot);
    if (st.left.fetch_sub(1) == 1) launch_copies(t.item);
    return true;
  }

  void launch_copies(int item) {
    const auto& it = items_[item];
    ItemState& st = states_[item];
    DeviceCtx* ctx = ctx_for(it.device);
    if (!ctx) return;
    cudaSetDevice(it.device);
    cudaStream_t stream = ctx->stream_for(item);  // after this item's H2D pieces
    if (it.n_copies > 0) {
      std::vector<CopyJob> jobs;
      std::vector<CastJob> casts;
      std::string why;
      for (int c = 0; c < it.n_copies; ++c) {
        tv_copy cp = copies_[it.first_copy + c];
        cp.src.base = reinterpret_cast<uint64_t>(st.base) + cp.src.base;
        const bool ok = is_cast(cp) ? normalize_cast(cp, casts, why) : normalize(cp, jobs, why);
        if (!ok) {
          err_.set(TV_ERR_ARG, "unpack: " + why);
          return;
        }
        bytes_packed_ += box_bytes(cp.ext, cp.rank, cp.itemsize);
      }
      int64_t launches = 0;
      int rc = ctx->uploader->run(jobs, stream, &launches);
      if (rc == TV_OK) rc = ctx->uploader->run_cast(casts, stream, &launches);
      if (rc != TV_OK) {
        err_.set(rc, get_error());
        return;
      }
      launches_ += launches;
    }
    if (st.staged_off >= 0) {
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      cudaEventRecord(ev, stream);
      ctx->staging->free_after(st.staged_off, it.nbytes, ev);
    }
  }

  tv_engine* e_;
  const tv_read_item* items_;
  int n_items_;
  int n_ins_;
  const tv_copy* copies_;
  int n_copies_;
  tv_stats* stats_;
  std::unique_ptr<InputState[]> ins_;
  std::unique_ptr<ItemState[]> states_;
  std::vector<cudaEvent_t> slot_events_;
  std::vector<int> slot_event_dev_;
  Queue<int> free_slots_;
  Queue<ReadTask> tasks_;
  ErrorSlot err_;
  std::mutex used_m_;
  std::map<int, DeviceCtx*> used_devices_;
  std::atomic<int64_t> bytes_device_{0}, bytes_storage_{0}, bytes_packed_{0}, launches_{0},
      dma_{0}, files_{0}, zero_copy_bytes_{0};
  Clock io_, wait_dma_, wait_slot_;
  const bool maps_ = mappings_exist();  // any registered file mapping in this process
};

}  // namespace

int engine_create(int n_slots, int64_t slot_bytes, int64_t staging_bytes, int n_threads,
                  tv_engine** out) {
  if (n_slots < 1 || slot_bytes < 4096 || n_threads < 1 || staging_bytes < 0) {
    set_error("bad engine parameters");
    return TV_ERR_ARG;
  }
  auto e = std::make_unique<tv_engine>();
  e->n_slots = n_slots;
  e->slot_bytes = slot_bytes;
  e->staging_bytes = std::max<int64_t>(staging_bytes, (int64_t)n_slots * slot_bytes);
  e->n_threads = n_threads;
  const char* huge = std::getenv("TVGPU_HUGE_RING");
  if (huge && std::atoi(huge) != 0) {
    // One 2 MiB-page region (THP via madvise), faulted in, then pinned: fewer TLB entries
    // for both the writers' reads and the copy engine's accesses.
    const size_t hp = 2u << 20;
    e->ring_bytes = (((size_t)n_slots * (size_t)slot_bytes) + hp - 1) / hp * hp;
    void* m = mmap(nullptr, e->ring_bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (m == MAP_FAILED) {
      set_error("mmap of the huge-page slot ring failed");
      return TV_ERR_NOMEM;
    }
    madvise(m, e->ring_bytes, MADV_HUGEPAGE);
    std::memset(m, 0, e->ring_bytes);
    cudaError_t ce = cudaHostRegister(m, e->ring_bytes, cudaHostRegisterPortable);
    if (ce != cudaSuccess) {
      munmap(m, e->ring_bytes);
      set_error(std::string("cudaHostRegister(slot ring): ") + cudaGetErrorString(ce));
      return TV_ERR_NOMEM;
    }
    e->ring = static_cast<char*>(m);
    for (int i = 0; i < n_slots; ++i) e->slots.push_back(e->ring + (size_t)i * slot_bytes);
    *out = e.release();
    return TV_OK;
  }
  for (int i = 0; i < n_slots; ++i) {
    char* p = nullptr;
    cudaError_t ce = cudaHostAlloc(&p, slot_bytes, cudaHostAllocPortable);
    if (ce != cudaSuccess) {
      for (auto q : e->slots) cudaFreeHost(q);
      set_error(std::string("cudaHostAlloc: ") + cudaGetErrorString(ce));
      return TV_ERR_NOMEM;
    }
    e->slots.push_back(p);
  }
  *out = e.release();
  return TV_OK;
}

int engine_destroy(tv_engine* e) {
  if (!e) return TV_OK;
  {
    std::lock_guard<std::mutex> g(e->dev_m);
    for (auto& kv : e->devices) {
      cudaSetDevice(kv.first);
      for (cudaStream_t st : kv.second->streams) cudaStreamSynchronize(st);
      if (kv.second->zero_copy) cudaStreamSynchronize(kv.second->zero_copy);
      for (auto ev : kv.second->zc_ev) cudaEventDestroy(ev);
      if (kv.second->zc_ring) cudaFree(kv.second->zc_ring);
      kv.second->uploader.reset();
      kv.second->staging.reset();
      for (cudaStream_t st : kv.second->streams) cudaStreamDestroy(st);
      if (kv.second->zero_copy) cudaStreamDestroy(kv.second->zero_copy);
    }
    e->devices.clear();
  }
  if (e->ring) {
    cudaHostUnregister(e->ring);
    munmap(e->ring, e->ring_bytes);
  } else {
    for (auto p : e->slots) cudaFreeHost(p);
  }
  delete e;
  return TV_OK;
}

int engine_save(tv_engine* e, const tv_write_item* items, int n_items, const tv_output* outputs,
                int n_outputs, const char* pool_dir, int pool_flags, tv_stats* stats) {
  std::lock_guard<std::mutex> g(e->call_m);
  tv_stats local{};
  SaveRun run(e, items, n_items, outputs, n_outputs, stats ? stats : &local, pool_dir, pool_flags);
  int rc = run.run();
  run.publish_stats();
  return rc;
}

int engine_load(tv_engine* e, const tv_read_item* items, int n_items, const tv_input* inputs,
                int n_inputs, const tv_copy* copies, int n_copies, tv_stats* stats) {
  std::lock_guard<std::mutex> g(e->call_m);
  tv_stats local{};
  LoadRun run(e, items, n_items, inputs, n_inputs, copies, n_copies, stats ? stats : &local);
  int rc = run.run();
  run.publish_stats();
  return rc;
}

int kernel_timing(int enable) {
  g_timer.on.store(enable != 0);
  return TV_OK;
}

int kernel_timing_collect(double* ms_total, double* ms_max, int64_t* bytes, int64_t* launches) {
  return g_timer.collect(ms_total, ms_max, bytes, launches);
}

// Standalone batched copy (tv_copy_boxes): one launch on the caller's stream.
int copy_boxes(int device, const tv_copy* copies, int n, cudaStream_t stream) {
  std::vector<CopyJob> jobs;
  std::vector<CastJob> casts;
  std::string why;
  for (int i = 0; i < n; ++i) {
    const bool ok = is_cast(copies[i]) ? normalize_cast(copies[i], casts, why)
                                       : normalize(copies[i], jobs, why);
    if (!ok) {
      set_error("tv_copy_boxes: copy " + std::to_string(i) + ": " + why);
      return TV_ERR_ARG;
    }
  }
  if (jobs.empty() && casts.empty()) return TV_OK;
  static std::mutex m;
  static std::map<int, std::unique_ptr<JobUploader>> uploaders;
  JobUploader* up;
  {
    std::lock_guard<std::mutex> g(m);
    auto& slot = uploaders[device];
    if (!slot) slot = std::make_unique<JobUploader>(device);
    up = slot.get();
  }
  TV_CUDA_CHECK(cudaSetDevice(device));
  int rc = up->run(jobs, stream, nullptr);
  if (rc == TV_OK) rc = up->run_cast(casts, stream, nullptr);
  return rc;
}

}  // namespace tv
