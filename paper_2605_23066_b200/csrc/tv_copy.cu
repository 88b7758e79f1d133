// Batched N-d box copy for sm_100a: the pack (save), unpack/scatter (restore) and
// snapshot kernel of the checkpoint data path.
//
// Every copy between two row-major arrays is reduced on the host to "nruns contiguous
// runs of `run` bytes" with up to three outer dimensions (CopyJob).  One launch covers a
// whole batch of jobs (e.g. all 873 leaves of a Llama-3-8B tree): block b finds its job
// by binary search over the jobs' block prefix sums, so there is one launch per batch,
// not per chunk.  The copy itself moves 16-byte vectors whenever run length, strides and
// both base addresses allow it (coalesced LDG.128/STG.128), with every lane keeping up
// to 8 independent loads in flight before it stores (ILP hides HBM/NVLink latency).
//
// Reference seams replaced (treevault, /root/reference/pkg/src/treevault):
//   save_pipeline.py:323-324  leaf.data[sel].copy()                  (snapshot)
//   chunkstore.py:387-392     np.ascontiguousarray(values[sel])      (pack)
//   chunkstore.py:579-592     out[dst] = data[src]                   (unpack)
//   load_pipeline.py:467-471  out[sel] = data                        (assemble/scatter)

#include <algorithm>
#include <cstring>

#include "tv_internal.h"

namespace tv {

namespace {

constexpr int kThreads = 256;          // 8 warps per CTA
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 8;             // vectors in flight per lane (mode 0)
constexpr int kSegVecs = 32 * kUnroll; // vectors per warp work unit (mode 0)
constexpr int kFlatPerThread = 4;      // vectors per thread (mode 1)
constexpr int kFlatVecs = kThreads * kFlatPerThread;

template <int V>
struct VecT;
template <>
struct VecT<16> {
  using T = uint4;
};
template <>
struct VecT<8> {
  using T = uint2;
};
template <>
struct VecT<4> {
  using T = uint32_t;
};
template <>
struct VecT<2> {
  using T = uint16_t;
};
template <>
struct VecT<1> {
  using T = uint8_t;
};

template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
  return __ldcs(p);
}
template <>
__device__ __forceinline__ uint4 ld_stream<uint4>(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
template <>
__device__ __forceinline__ uint16_t ld_stream<uint16_t>(const uint16_t* p) {
  return *p;
}
template <>
__device__ __forceinline__ uint8_t ld_stream<uint8_t>(const uint8_t* p) {
  return *p;
}

__device__ __forceinline__ int find_job(const CopyJob* jobs, int n_jobs, int64_t block) {
  int lo = 0, hi = n_jobs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].unit_begin <= block)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void run_origin(const CopyJob& j, int64_t r, int64_t& so,
                                           int64_t& dof) {
  int64_t i0 = r % j.n[0];
  int64_t t = r / j.n[0];
  int64_t i1 = t % j.n[1];
  int64_t i2 = t / j.n[1];
  so = i0 * j.ss[0] + i1 * j.ss[1] + i2 * j.ss[2];
  dof = i0 * j.ds[0] + i1 * j.ds[1] + i2 * j.ds[2];
}

// Mode 0: one warp copies one segment (≤ kSegVecs vectors) of one run.
template <int V>
__device__ __forceinline__ void copy_segment(const CopyJob& j, int64_t local_block) {
  using T = typename VecT<V>::T;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t vpr = j.run / V;
  const int64_t segs = (vpr + kSegVecs - 1) / kSegVecs;
  const int64_t unit = local_block * kWarps + warp;
  if (unit >= j.nruns * segs) return;
  const int64_t r = unit / segs;
  const int64_t s = unit - r * segs;
  int64_t so, dof;
  run_origin(j, r, so, dof);
  const T* src = reinterpret_cast<const T*>(j.src + so) + s * kSegVecs;
  T* dst = reinterpret_cast<T*>(j.dst + dof) + s * kSegVecs;
  const int64_t left = vpr - s * kSegVecs;
  const int nv = (int)(left < kSegVecs ? left : kSegVecs);
  T buf[kUnroll];
#pragma unroll
  for (int k = 0; k < kUnroll; ++k) {
    int idx = lane + 32 * k;
    if (idx < nv) buf[k] = ld_stream(src + idx);
  }
#pragma unroll
  for (int k = 0; k < kUnroll; ++k) {
    int idx = lane + 32 * k;
    if (idx < nv) dst[idx] = buf[k];
  }
}

// Mode 2: mid-length runs (< kSegVecs / 2 vectors).  One warp copies a group of
// consecutive runs along dim 0 (≤ kSegVecs vectors in all), so every lane still keeps up
// to kUnroll loads in flight — a warp per run left one per lane on 512-byte runs (0.51 of
// a 2-D tensor-map TMA pack, profiles/r02_tma2d_pack_probe.jsonl; with groups 0.92, and
// above TMA on 128-byte runs: r02_box_copy_group_mode_ab.jsonl).  The group origin is
// decomposed once; runs inside it are ss[0] / ds[0] apart.
template <int V>
__device__ __forceinline__ void copy_group(const CopyJob& j, int64_t local_block) {
  using T = typename VecT<V>::T;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int vpr = (int)(j.run / V);
  const int64_t per_row = (j.n[0] + j.group - 1) / j.group;
  const int64_t unit = local_block * kWarps + warp;
  const int64_t outer = unit / per_row;
  if (outer >= j.n[1] * j.n[2]) return;
  const int64_t first = (unit - outer * per_row) * j.group;
  const int64_t left = j.n[0] - first;
  const int nv = (int)(left < j.group ? left : j.group) * vpr;
  const int64_t i1 = outer % j.n[1], i2 = outer / j.n[1];
  const char* src = j.src + first * j.ss[0] + i1 * j.ss[1] + i2 * j.ss[2];
  char* dst = j.dst + first * j.ds[0] + i1 * j.ds[1] + i2 * j.ds[2];
  T buf[kUnroll];
#pragma unroll
  for (int k = 0; k < kUnroll; ++k) {
    const int idx = lane + 32 * k, q = idx / vpr;
    if (idx < nv) buf[k] = ld_stream(reinterpret_cast<const T*>(src + q * j.ss[0]) + (idx - q * vpr));
  }
#pragma unroll
  for (int k = 0; k < kUnroll; ++k) {
    const int idx = lane + 32 * k, q = idx / vpr;
    if (idx < nv) reinterpret_cast<T*>(dst + q * j.ds[0])[idx - q * vpr] = buf[k];
  }
}

// Mode 1: short runs; each thread decomposes its own vector indices.
template <int V>
__device__ __forceinline__ void copy_flat(const CopyJob& j, int64_t local_block) {
  using T = typename VecT<V>::T;
  const int64_t vpr = j.run / V;
  const int64_t total = j.nruns * vpr;
  const int64_t base = local_block * kFlatVecs;
  T buf[kFlatPerThread];
  T* dsts[kFlatPerThread];
#pragma unroll
  for (int k = 0; k < kFlatPerThread; ++k) {
    int64_t v = base + k * kThreads + threadIdx.x;
    dsts[k] = nullptr;
    if (v < total) {
      int64_t r = v / vpr;
      int64_t w = v - r * vpr;
      int64_t so, dof;
      run_origin(j, r, so, dof);
      buf[k] = ld_stream(reinterpret_cast<const T*>(j.src + so) + w);
      dsts[k] = reinterpret_cast<T*>(j.dst + dof) + w;
    }
  }
#pragma unroll
  for (int k = 0; k < kFlatPerThread; ++k)
    if (dsts[k] != nullptr) *dsts[k] = buf[k];
}

template <int V>
__device__ __forceinline__ void dispatch_mode(const CopyJob& j, int64_t local_block) {
  if (j.mode == 0)
    copy_segment<V>(j, local_block);
  else if (j.mode == 2)
    copy_group<V>(j, local_block);
  else
    copy_flat<V>(j, local_block);
}

__global__ void __launch_bounds__(kThreads) box_copy_kernel(const CopyJob* __restrict__ jobs,
                                                            int n_jobs, int64_t block0) {
  const int64_t block = block0 + blockIdx.x;
  const int ji = find_job(jobs, n_jobs, block);
  const CopyJob j = jobs[ji];
  const int64_t local = block - j.unit_begin;
  if (local >= j.units) return;
  switch (j.vec) {
    case 16:
      dispatch_mode<16>(j, local);
      break;
    case 8:
      dispatch_mode<8>(j, local);
      break;
    case 4:
      dispatch_mode<4>(j, local);
      break;
    case 2:
      dispatch_mode<2>(j, local);
      break;
    default:
      dispatch_mode<1>(j, local);
      break;
  }
}

struct Dim {
  int64_t n, ss, ds;  // extent, source / destination element strides
};

int vec_width(uint64_t g) {
  if (g == 0) return 16;
  uint64_t low = g & (~g + 1);
  return (int)std::min<uint64_t>(low, 16);
}

}  // namespace

bool normalize(const tv_copy& c, std::vector<CopyJob>& out, std::string& err) {
  const int rank = c.rank;
  const int64_t isz = c.itemsize;
  if (rank < 0 || rank > TV_MAX_RANK || isz <= 0) {
    err = "bad rank/itemsize";
    return false;
  }
  for (int i = 0; i < rank; ++i) {
    if (c.ext[i] < 0 || c.src.off[i] < 0 || c.dst.off[i] < 0 ||
        c.src.off[i] + c.ext[i] > c.src.shape[i] || c.dst.off[i] + c.ext[i] > c.dst.shape[i]) {
      err = "box outside its array in dim " + std::to_string(i);
      return false;
    }
    if (c.ext[i] == 0) return true;  // empty box: nothing to move
  }
  // Row-major element strides and base offsets.
  int64_t sst[TV_MAX_RANK], dst_[TV_MAX_RANK];
  int64_t s_acc = 1, d_acc = 1;
  for (int i = rank - 1; i >= 0; --i) {
    sst[i] = s_acc;
    dst_[i] = d_acc;
    s_acc *= c.src.shape[i];
    d_acc *= c.dst.shape[i];
  }
  int64_t sbase = 0, dbase = 0;
  for (int i = 0; i < rank; ++i) {
    sbase += c.src.off[i] * sst[i];
    dbase += c.dst.off[i] * dst_[i];
  }
  // Dims with extent > 1, merged inner-first where both sides are contiguous.
  std::vector<Dim> m;  // m[0] innermost
  for (int i = rank - 1; i >= 0; --i) {
    if (c.ext[i] == 1) continue;
    Dim d{c.ext[i], sst[i], dst_[i]};
    if (!m.empty() && d.ss == m.back().n * m.back().ss && d.ds == m.back().n * m.back().ds)
      m.back().n *= d.n;
    else
      m.push_back(d);
  }
  int64_t run = isz;
  if (!m.empty() && m[0].ss == 1 && m[0].ds == 1) {
    run = m[0].n * isz;
    m.erase(m.begin());
  }
  // Up to three outer dims per job; extra (outermost) dims are enumerated on the host.
  std::vector<Dim> inner(m.begin(), m.begin() + std::min<size_t>(3, m.size()));
  std::vector<Dim> extra(m.begin() + inner.size(), m.end());
  int64_t combos = 1;
  for (auto& d : extra) combos *= d.n;
  for (int64_t k = 0; k < combos; ++k) {
    int64_t t = k, soff = sbase, doff = dbase;
    for (auto& d : extra) {
      int64_t i = t % d.n;
      t /= d.n;
      soff += i * d.ss;
      doff += i * d.ds;
    }
    CopyJob j{};
    j.src = reinterpret_cast<const char*>(c.src.base) + soff * isz;
    j.dst = reinterpret_cast<char*>(c.dst.base) + doff * isz;
    j.run = run;
    uint64_t g = (uint64_t)run | (uint64_t)reinterpret_cast<uintptr_t>(j.src) |
                 (uint64_t)reinterpret_cast<uintptr_t>(j.dst);
    for (int q = 0; q < 3; ++q) {
      if (q < (int)inner.size()) {
        j.n[q] = inner[q].n;
        j.ss[q] = inner[q].ss * isz;
        j.ds[q] = inner[q].ds * isz;
        g |= (uint64_t)j.ss[q] | (uint64_t)j.ds[q];
      } else {
        j.n[q] = 1;
        j.ss[q] = 0;
        j.ds[q] = 0;
      }
    }
    j.nruns = j.n[0] * j.n[1] * j.n[2];
    j.vec = vec_width(g);
    // ≥ 2 KiB-class runs: a warp per run segment; shorter ones: a warp per group of runs
    // when a group fills at least two vectors per lane; else flat (or a warp per run)
    const int64_t vpr = run / j.vec;
    const int64_t group = std::min<int64_t>(j.n[0], kSegVecs / std::max<int64_t>(vpr, 1));
    j.group = 1;
    if (vpr >= kSegVecs / 2) {
      j.mode = 0;
    } else if (group * vpr >= 64) {
      j.mode = 2;
      j.group = (int32_t)group;
    } else {
      j.mode = vpr >= 32 ? 0 : 1;
    }
    out.push_back(j);
  }
  return true;
}

int64_t plan_units(std::vector<CopyJob>& jobs) {
  int64_t total = 0;
  for (auto& j : jobs) {
    const int64_t vpr = j.run / j.vec;
    if (j.mode == 0) {
      const int64_t segs = (vpr + kSegVecs - 1) / kSegVecs;
      j.units = (j.nruns * segs + kWarps - 1) / kWarps;
    } else if (j.mode == 2) {
      const int64_t groups = j.n[1] * j.n[2] * ((j.n[0] + j.group - 1) / j.group);
      j.units = (groups + kWarps - 1) / kWarps;
    } else {
      j.units = (j.nruns * vpr + kFlatVecs - 1) / kFlatVecs;
    }
    j.unit_begin = total;
    total += j.units;
  }
  return total;
}

cudaError_t launch_copy_jobs(const CopyJob* dev_jobs, const CopyJob*, int n_jobs,
                             int64_t total_units, cudaStream_t stream) {
  const int64_t max_grid = 0x7fffffffLL;
  for (int64_t b0 = 0; b0 < total_units; b0 += max_grid) {
    const unsigned grid = (unsigned)std::min<int64_t>(max_grid, total_units - b0);
    box_copy_kernel<<<grid, kThreads, 0, stream>>>(dev_jobs, n_jobs, b0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

bool box_contiguous(const tv_array_box& b, const int64_t* ext, int rank, int itemsize,
                    int64_t* byte_off, int64_t* nbytes) {
  // Contiguous iff, after the first dim with extent > 1, every dim is full.
  int64_t stride = 1, off = 0, n = 1;
  int64_t strides[TV_MAX_RANK];
  for (int i = rank - 1; i >= 0; --i) {
    strides[i] = stride;
    stride *= b.shape[i];
  }
  int first = -1;
  for (int i = 0; i < rank; ++i) {
    off += b.off[i] * strides[i];
    n *= ext[i];
    if (first < 0 && ext[i] > 1) first = i;
  }
  if (first >= 0) {
    for (int i = first + 1; i < rank; ++i)
      if (ext[i] != b.shape[i]) return false;
  }
  *byte_off = off * itemsize;
  *nbytes = n * itemsize;
  return true;
}

}  // namespace tv
