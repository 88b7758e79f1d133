// Converting box copy: the load-time cast of the reference (treemodel.py:417-484,
// cast_leaf / _convert_values) fused into the restore's unpack/scatter, so a checkpoint
// stored in one dtype lands in the target dtype in one pass over HBM (no second buffer,
// no second kernel).  Semantics:
//   float narrowing  round-to-nearest-even (f64->f32 cvt.rn; f32->bf16 RNE on the bits;
//                    f64->bf16 and int->bf16 go through f32 exactly like the host path)
//   int  -> int      checked: any out-of-range value sets TV_CAST_OVERFLOW
//   float-> int      checked: non-finite -> NONFINITE, non-integral -> NONINTEGRAL,
//                    out of range -> OVERFLOW (the caller raises CastError by priority)
//   widening         exact
// bool never converts (rejected by the planner, like the reference).

#include <algorithm>
#include <cmath>
#include <cstring>

#include "tv_internal.h"

namespace tv {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPerLane = 8;
constexpr int kSeg = 32 * kPerLane;     // elements per warp unit (mode 0)
constexpr int kFlatPer = 4;
constexpr int kFlat = kThreads * kFlatPer;

__device__ __forceinline__ bool is_float(int dt) {
  return dt == TV_DT_F32 || dt == TV_DT_F64 || dt == TV_DT_BF16;
}

__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}

__device__ __forceinline__ uint16_t f32_to_bf16(float f) {
  uint32_t bits = __float_as_uint(f);
  if ((bits & 0x7f800000u) == 0x7f800000u && (bits & 0x007fffffu))  // NaN: keep it quiet
    return (uint16_t)((bits >> 16) | 0x40);
  uint64_t r = ((uint64_t)bits + 0x7fffu + ((bits >> 16) & 1u)) >> 16;
  return (uint16_t)r;
}

struct Value {
  double f;    // float sources
  long long i; // integer sources
};

__device__ __forceinline__ Value load_value(const char* p, int dt) {
  Value v{0.0, 0};
  switch (dt) {
    case TV_DT_F32: v.f = (double)*reinterpret_cast<const float*>(p); break;
    case TV_DT_F64: v.f = *reinterpret_cast<const double*>(p); break;
    case TV_DT_BF16: v.f = (double)bf16_to_f32(*reinterpret_cast<const uint16_t*>(p)); break;
    case TV_DT_I32: v.i = *reinterpret_cast<const int32_t*>(p); break;
    case TV_DT_I64: v.i = *reinterpret_cast<const long long*>(p); break;
    case TV_DT_U8: v.i = *reinterpret_cast<const uint8_t*>(p); break;
    default: v.i = *reinterpret_cast<const uint8_t*>(p); break;
  }
  return v;
}

__device__ __forceinline__ void int_range(int dt, long long& lo, long long& hi) {
  switch (dt) {
    case TV_DT_I32: lo = INT32_MIN; hi = INT32_MAX; break;
    case TV_DT_U8: lo = 0; hi = 255; break;
    default: lo = LLONG_MIN; hi = LLONG_MAX; break;
  }
}

// Convert one element; returns TV_CAST_* bits of a violated check.
__device__ __forceinline__ uint32_t convert(const char* sp, char* dp, int sdt, int ddt) {
  const Value v = load_value(sp, sdt);
  uint32_t bad = 0;
  if (is_float(sdt)) {
    const double x = v.f;
    switch (ddt) {
      case TV_DT_F32: *reinterpret_cast<float*>(dp) = __double2float_rn(x); break;
      case TV_DT_F64: *reinterpret_cast<double*>(dp) = x; break;
      case TV_DT_BF16:
        *reinterpret_cast<uint16_t*>(dp) = f32_to_bf16(sdt == TV_DT_F64 ? __double2float_rn(x) : (float)x);
        break;
      default: {  // float -> int, checked
        long long lo, hi;
        int_range(ddt, lo, hi);
        long long q = 0;
        if (!isfinite(x)) {
          bad |= TV_CAST_NONFINITE;
        } else if (x != floor(x)) {
          bad |= TV_CAST_NONINTEGRAL;
        } else if (ddt == TV_DT_I64 ? (x >= 9223372036854775808.0 || x < -9223372036854775808.0)
                                    : (x < (double)lo || x > (double)hi)) {
          bad |= TV_CAST_OVERFLOW;
        } else {
          q = (long long)x;
        }
        if (ddt == TV_DT_I32) *reinterpret_cast<int32_t*>(dp) = (int32_t)q;
        else if (ddt == TV_DT_I64) *reinterpret_cast<long long*>(dp) = q;
        else *reinterpret_cast<uint8_t*>(dp) = (uint8_t)q;
      }
    }
  } else {
    const long long x = v.i;
    switch (ddt) {
      case TV_DT_F32: *reinterpret_cast<float*>(dp) = __ll2float_rn(x); break;
      case TV_DT_F64: *reinterpret_cast<double*>(dp) = __ll2double_rn(x); break;
      case TV_DT_BF16: *reinterpret_cast<uint16_t*>(dp) = f32_to_bf16(__ll2float_rn(x)); break;
      default: {  // int -> int, checked
        long long lo, hi;
        int_range(ddt, lo, hi);
        if (x < lo || x > hi) bad |= TV_CAST_OVERFLOW;
        if (ddt == TV_DT_I32) *reinterpret_cast<int32_t*>(dp) = (int32_t)x;
        else if (ddt == TV_DT_I64) *reinterpret_cast<long long*>(dp) = x;
        else *reinterpret_cast<uint8_t*>(dp) = (uint8_t)x;
      }
    }
  }
  return bad;
}

__device__ __forceinline__ int find_cast_job(const CastJob* jobs, int n, int64_t block) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (jobs[mid].unit_begin <= block) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void origin(const CastJob& j, int64_t r, int64_t& so, int64_t& dof) {
  int64_t i0 = r % j.n[0], t = r / j.n[0];
  int64_t i1 = t % j.n[1], i2 = t / j.n[1];
  so = i0 * j.ss[0] + i1 * j.ss[1] + i2 * j.ss[2];
  dof = i0 * j.ds[0] + i1 * j.ds[1] + i2 * j.ds[2];
}

__global__ void __launch_bounds__(kThreads) box_cast_kernel(const CastJob* __restrict__ jobs,
                                                            int n_jobs, int64_t block0) {
  const int64_t block = block0 + blockIdx.x;
  const CastJob j = jobs[find_cast_job(jobs, n_jobs, block)];
  const int64_t local = block - j.unit_begin;
  const int ssz = j.sdt == TV_DT_F64 || j.sdt == TV_DT_I64 ? 8 : j.sdt == TV_DT_F32 || j.sdt == TV_DT_I32 ? 4
                  : j.sdt == TV_DT_BF16 ? 2 : 1;
  const int dsz = j.ddt == TV_DT_F64 || j.ddt == TV_DT_I64 ? 8 : j.ddt == TV_DT_F32 || j.ddt == TV_DT_I32 ? 4
                  : j.ddt == TV_DT_BF16 ? 2 : 1;
  uint32_t bad = 0;
  if (local < j.units) {
    if (j.mode == 0) {
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      const int64_t segs = (j.run + kSeg - 1) / kSeg;
      const int64_t unit = local * kWarps + warp;
      if (unit < j.nruns * segs) {
        const int64_t r = unit / segs, s = unit - r * segs;
        int64_t so, dof;
        origin(j, r, so, dof);
        const int64_t e0 = s * kSeg;
        const int64_t left = j.run - e0;
        const int nv = (int)(left < kSeg ? left : kSeg);
#pragma unroll
        for (int k = 0; k < kPerLane; ++k) {
          const int idx = lane + 32 * k;
          if (idx < nv)
            bad |= convert(j.src + so + (e0 + idx) * ssz, j.dst + dof + (e0 + idx) * dsz, j.sdt, j.ddt);
        }
      }
    } else {
      const int64_t total = j.nruns * j.run;
#pragma unroll
      for (int k = 0; k < kFlatPer; ++k) {
        const int64_t v = local * kFlat + k * kThreads + threadIdx.x;
        if (v < total) {
          const int64_t r = v / j.run, w = v - r * j.run;
          int64_t so, dof;
          origin(j, r, so, dof);
          bad |= convert(j.src + so + w * ssz, j.dst + dof + w * dsz, j.sdt, j.ddt);
        }
      }
    }
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicOr(j.flags, bad);
}

}  // namespace

bool is_cast(const tv_copy& c) { return c.src_dtype != TV_DT_RAW; }

int dtype_size(int dt) {
  switch (dt) {
    case TV_DT_F64: case TV_DT_I64: return 8;
    case TV_DT_F32: case TV_DT_I32: return 4;
    case TV_DT_BF16: return 2;
    case TV_DT_U8: case TV_DT_BOOL: return 1;
    default: return 0;
  }
}

bool normalize_cast(const tv_copy& c, std::vector<CastJob>& out, std::string& err) {
  const int rank = c.rank;
  const int ssz = dtype_size(c.src_dtype), dsz = dtype_size(c.dst_dtype);
  if (rank < 0 || rank > TV_MAX_RANK || ssz == 0 || dsz == 0 || c.itemsize != ssz) {
    err = "bad converting copy (rank/dtype/itemsize)";
    return false;
  }
  if (c.src_dtype == TV_DT_BOOL || c.dst_dtype == TV_DT_BOOL || !c.flags) {
    err = "bool never converts; converting copies need a flags word";
    return false;
  }
  for (int i = 0; i < rank; ++i) {
    if (c.ext[i] < 0 || c.src.off[i] < 0 || c.dst.off[i] < 0 ||
        c.src.off[i] + c.ext[i] > c.src.shape[i] || c.dst.off[i] + c.ext[i] > c.dst.shape[i]) {
      err = "box outside its array in dim " + std::to_string(i);
      return false;
    }
    if (c.ext[i] == 0) return true;
  }
  int64_t sst[TV_MAX_RANK], dst_[TV_MAX_RANK];
  int64_t sa = 1, da = 1, sbase = 0, dbase = 0;
  for (int i = rank - 1; i >= 0; --i) {
    sst[i] = sa;
    dst_[i] = da;
    sa *= c.src.shape[i];
    da *= c.dst.shape[i];
  }
  for (int i = 0; i < rank; ++i) {
    sbase += c.src.off[i] * sst[i];
    dbase += c.dst.off[i] * dst_[i];
  }
  struct D { int64_t n, s, d; };
  std::vector<D> m;  // inner-first, element strides
  for (int i = rank - 1; i >= 0; --i) {
    if (c.ext[i] == 1) continue;
    D x{c.ext[i], sst[i], dst_[i]};
    if (!m.empty() && x.s == m.back().n * m.back().s && x.d == m.back().n * m.back().d)
      m.back().n *= x.n;
    else
      m.push_back(x);
  }
  int64_t run = 1;
  if (!m.empty() && m[0].s == 1 && m[0].d == 1) {
    run = m[0].n;
    m.erase(m.begin());
  }
  std::vector<D> inner(m.begin(), m.begin() + std::min<size_t>(3, m.size()));
  std::vector<D> extra(m.begin() + inner.size(), m.end());
  int64_t combos = 1;
  for (auto& d : extra) combos *= d.n;
  for (int64_t k = 0; k < combos; ++k) {
    int64_t t = k, so = sbase, dof = dbase;
    for (auto& d : extra) {
      int64_t i = t % d.n;
      t /= d.n;
      so += i * d.s;
      dof += i * d.d;
    }
    CastJob j{};
    j.src = reinterpret_cast<const char*>(c.src.base) + so * ssz;
    j.dst = reinterpret_cast<char*>(c.dst.base) + dof * dsz;
    j.run = run;
    for (int q = 0; q < 3; ++q) {
      bool have = q < (int)inner.size();
      j.n[q] = have ? inner[q].n : 1;
      j.ss[q] = have ? inner[q].s * ssz : 0;
      j.ds[q] = have ? inner[q].d * dsz : 0;
    }
    j.nruns = j.n[0] * j.n[1] * j.n[2];
    j.flags = reinterpret_cast<uint32_t*>(c.flags);
    j.sdt = c.src_dtype;
    j.ddt = c.dst_dtype;
    j.mode = run >= 32 ? 0 : 1;
    out.push_back(j);
  }
  return true;
}

int64_t plan_cast_units(std::vector<CastJob>& jobs) {
  int64_t total = 0;
  for (auto& j : jobs) {
    if (j.mode == 0) {
      const int64_t segs = (j.run + kSeg - 1) / kSeg;
      j.units = (j.nruns * segs + kWarps - 1) / kWarps;
    } else {
      j.units = (j.nruns * j.run + kFlat - 1) / kFlat;
    }
    j.unit_begin = total;
    total += j.units;
  }
  return total;
}

cudaError_t launch_cast_jobs(const CastJob* dev_jobs, int n_jobs, int64_t total_units,
                             cudaStream_t stream) {
  const int64_t max_grid = 0x7fffffffLL;
  for (int64_t b0 = 0; b0 < total_units; b0 += max_grid) {
    const unsigned grid = (unsigned)std::min<int64_t>(max_grid, total_units - b0);
    box_cast_kernel<<<grid, kThreads, 0, stream>>>(dev_jobs, n_jobs, b0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace tv
