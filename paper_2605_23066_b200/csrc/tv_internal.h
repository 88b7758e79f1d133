// Internal declarations shared by the libtvgpu translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "tvgpu.h"

namespace tv {

// Restores the calling thread's current CUDA device on scope exit: no entry point of the
// library may leave the caller (e.g. torch) on another device.
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Thread-local last error (tv_last_error).
void set_error(const std::string& msg);
const std::string& get_error();

#define TV_CUDA_CHECK(expr)                                                              \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ::tv::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " (" +        \
                      __FILE__ + ":" + std::to_string(__LINE__) + ")");                  \
      return TV_ERR_CUDA;                                                                \
    }                                                                                    \
  } while (0)

// Canonical form of one box copy: `nruns` contiguous runs of `run` bytes, the run
// index decomposed over up to three outer dimensions (n[0] fastest) with byte strides
// ss/ds on the source/destination side.  Produced on the host by normalize().
struct CopyJob {
  const char* src;
  char* dst;
  int64_t run;        // bytes per contiguous run (identical on both sides)
  int64_t n[3];       // outer extents (n[0] varies fastest); unused dims are 1
  int64_t ss[3];      // source byte strides of the outer dims
  int64_t ds[3];      // destination byte strides
  int64_t nruns;      // n[0]*n[1]*n[2]
  int64_t units;      // work units of this job (see kernel)
  int64_t unit_begin; // prefix sum of units over the batch
  int32_t vec;        // vector width in bytes (1,2,4,8,16)
  int32_t mode;       // 0 = warp per run segment, 1 = flat (short runs), 2 = warp per run group
  int32_t group;      // mode 2: consecutive runs of dim 0 per warp unit
  int32_t pad_;
};

// Split a tv_copy into canonical jobs (appends; returns false on malformed input).
bool normalize(const tv_copy& c, std::vector<CopyJob>& out, std::string& err);

// Assign units/unit_begin and launch the batched copy kernel on `stream`.
// `dev_jobs` must point to device-visible memory holding `jobs` (the caller stages it).
int64_t plan_units(std::vector<CopyJob>& jobs);
cudaError_t launch_copy_jobs(const CopyJob* dev_jobs, const CopyJob* host_jobs, int n_jobs,
                             int64_t total_units, cudaStream_t stream);

// Converting copy (load-time cast fused into the unpack): like CopyJob but in elements,
// with different element sizes on both sides.
struct CastJob {
  const char* src;
  char* dst;
  int64_t run;        // elements per contiguous run
  int64_t n[3];
  int64_t ss[3];      // source byte strides of the outer dims
  int64_t ds[3];      // destination byte strides
  int64_t nruns;
  int64_t units;
  int64_t unit_begin;
  uint32_t* flags;    // check word (TV_CAST_* bits)
  int32_t sdt;        // TV_DT_* source / destination element types
  int32_t ddt;
  int32_t mode;       // 0 = warp per run segment, 1 = flat (short runs)
  int32_t pad;
};

bool is_cast(const tv_copy& c);
int dtype_size(int dt);
bool normalize_cast(const tv_copy& c, std::vector<CastJob>& out, std::string& err);
int64_t plan_cast_units(std::vector<CastJob>& jobs);
// Jobs are grouped by dtype pair by plan_cast_units (unit_begin restarts per group);
// one launch per group of the pair's specialised kernel.
cudaError_t launch_cast_jobs(const CastJob* dev_jobs, const CastJob* host_jobs, int n_jobs,
                             int64_t total_units, cudaStream_t stream);

// Is the box a single contiguous byte range of its array?  Sets byte offset/length.
bool box_contiguous(const tv_array_box& b, const int64_t* ext, int rank, int itemsize,
                    int64_t* byte_off, int64_t* nbytes);

// Registered file mappings are registered in pieces of this many bytes (at file offsets
// that are multiples of it); a DMA into / out of a mapping never crosses a piece boundary.
constexpr int64_t kRegisterPiece = (int64_t)64 << 20;

// Registered file mappings (tv_mapped.cpp): the registered, MAP_SHARED mapping of the
// file open as `fd` when its inode is in the cache with exactly `size` bytes, else null.
char* mapping_for_fd(int fd, int64_t size);
// The cached registered mapping of the file open (read-write) as `fd`; when there is none,
// `register_now` and the file lives on a RAM-backed filesystem, map + register it now.
char* mapping_register_fd(int fd, int64_t size, bool register_now);
bool mappings_exist();
void mapping_release_fd(int fd);
void mapping_release_path(const char* path);

}  // namespace tv
