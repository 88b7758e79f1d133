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

#include <cuda_bf16.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "tv_internal.h"

#ifndef TV_CAST_STREAM
#define TV_CAST_STREAM 0
#endif

namespace tv {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kFlatPer = 4;
constexpr int kFlat = kThreads * kFlatPer;

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

// ---- typed conversion (the hot loop is specialised per dtype pair) ------------------------

struct BF16 {
  uint16_t bits;
};

template <typename T> struct Kind;  // 0 = float, 1 = integer
template <> struct Kind<float> { static constexpr int v = 0; };
template <> struct Kind<double> { static constexpr int v = 0; };
template <> struct Kind<BF16> { static constexpr int v = 0; };
template <> struct Kind<int32_t> { static constexpr int v = 1; };
template <> struct Kind<long long> { static constexpr int v = 1; };
template <> struct Kind<uint8_t> { static constexpr int v = 1; };

__device__ __forceinline__ double as_double(float x) { return (double)x; }
__device__ __forceinline__ double as_double(double x) { return x; }
__device__ __forceinline__ double as_double(BF16 x) { return (double)bf16_to_f32(x.bits); }
__device__ __forceinline__ long long as_ll(int32_t x) { return x; }
__device__ __forceinline__ long long as_ll(long long x) { return x; }
__device__ __forceinline__ long long as_ll(uint8_t x) { return x; }

template <typename D> struct Narrow;
template <> struct Narrow<int32_t> {
  static constexpr long long lo = INT32_MIN, hi = INT32_MAX;
};
template <> struct Narrow<long long> {
  static constexpr long long lo = LLONG_MIN, hi = LLONG_MAX;
};
template <> struct Narrow<uint8_t> {
  static constexpr long long lo = 0, hi = 255;
};

// float source -> float destination
__device__ __forceinline__ float f2f(double x, float*) { return __double2float_rn(x); }
__device__ __forceinline__ double f2f(double x, double*) { return x; }

template <typename S, typename D>
__device__ __forceinline__ D cvt(S x, uint32_t& bad) {
  if constexpr (Kind<S>::v == 0 && Kind<D>::v == 0) {
    if constexpr (std::is_same<D, BF16>::value) {
      float f;
      if constexpr (std::is_same<S, double>::value) f = __double2float_rn(x);
      else if constexpr (std::is_same<S, float>::value) f = x;
      else f = bf16_to_f32(x.bits);
      return BF16{f32_to_bf16(f)};
    } else if constexpr (std::is_same<S, float>::value && std::is_same<D, float>::value) {
      return x;
    } else {
      return f2f(as_double(x), (D*)nullptr);
    }
  } else if constexpr (Kind<S>::v == 0) {  // float -> int (checked)
    const double v = as_double(x);
    if (!isfinite(v)) {
      bad |= TV_CAST_NONFINITE;
      return D(0);
    }
    if (v != floor(v)) {
      bad |= TV_CAST_NONINTEGRAL;
      return D(0);
    }
    const bool over = std::is_same<D, long long>::value
                          ? (v >= 9223372036854775808.0 || v < -9223372036854775808.0)
                          : (v < (double)Narrow<D>::lo || v > (double)Narrow<D>::hi);
    if (over) {
      bad |= TV_CAST_OVERFLOW;
      return D(0);
    }
    return (D)(long long)v;
  } else if constexpr (Kind<D>::v == 0) {  // int -> float
    const long long v = as_ll(x);
    if constexpr (std::is_same<D, BF16>::value) return BF16{f32_to_bf16(__ll2float_rn(v))};
    else if constexpr (std::is_same<D, float>::value) return __ll2float_rn(v);
    else return __ll2double_rn(v);
  } else {  // int -> int (checked)
    const long long v = as_ll(x);
    if (v < Narrow<D>::lo || v > Narrow<D>::hi) bad |= TV_CAST_OVERFLOW;
    return (D)v;
  }
}

// f32 -> bf16 for two elements with one cvt.rn.bf16x2.f32 (round-to-nearest-even, exact
// for every non-NaN input incl. denormals and overflow to inf — the same result as the
// integer RNE of f32_to_bf16); NaNs take the host path's payload-keeping quiet NaN.
__device__ __forceinline__ void cvt_pair_f32_bf16(float a, float b, BF16& ra, BF16& rb) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  ra.bits = __bfloat16_as_ushort(h.x);
  rb.bits = __bfloat16_as_ushort(h.y);
  if (a != a) ra.bits = f32_to_bf16(a);
  if (b != b) rb.bits = f32_to_bf16(b);
}

template <typename T, int N>
struct alignas(sizeof(T) * N) Pack {
  T v[N];
};

// Mode 0: a warp converts one segment of a run.  Full, aligned segments take the fast
// path: every lane first issues kU 4-element vector loads (ILP: kU*16 B in flight per lane
// for f32), then converts and stores them; tails / misaligned runs go element by element
// (still coalesced across the warp).
#ifndef TV_CAST_SEGV
#define TV_CAST_SEGV 2048  // measured: 1024 -> 0.71, 2048 -> 0.78 of the copy peak (f32->bf16)
#endif
constexpr int kSegV = TV_CAST_SEGV;  // elements per warp unit

// Read-only streaming load of one vector pack (each byte is read exactly once: no L1
// allocation), 16 bytes per instruction.
template <typename P>
__device__ __forceinline__ P ld_pack(const P* p) {
#if TV_CAST_STREAM
  if constexpr (sizeof(P) % 16 == 0) {
    P r;
    const uint4* s = reinterpret_cast<const uint4*>(p);
    uint4* d = reinterpret_cast<uint4*>(&r);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(P) / 16); ++i)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(d[i].x), "=r"(d[i].y), "=r"(d[i].z), "=r"(d[i].w)
                   : "l"(s + i));
    return r;
  } else {
    return *p;
  }
#else
  return *p;
#endif
}

template <typename S, typename D>
__device__ __forceinline__ void cast_segment(const CastJob& j, int64_t local, uint32_t& bad) {
  // Vector width: the narrower side moves 16 bytes per access (f32->bf16: 8 elements =
  // 32 B loaded, 16 B stored per lane-step).
  constexpr int kVec = 16 / (sizeof(S) < sizeof(D) ? sizeof(S) : sizeof(D)) > 8
                           ? 8 : 16 / (sizeof(S) < sizeof(D) ? sizeof(S) : sizeof(D));
  constexpr int kU = kSegV / (32 * kVec);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t segs = (j.run + kSegV - 1) / kSegV;
  const int64_t unit = local * kWarps + warp;
  if (unit >= j.nruns * segs) return;
  const int64_t r = unit / segs, sg = unit - r * segs;
  int64_t so, dof;
  origin(j, r, so, dof);
  const S* src = reinterpret_cast<const S*>(j.src + so) + sg * kSegV;
  D* dst = reinterpret_cast<D*>(j.dst + dof) + sg * kSegV;
  const int64_t left = j.run - sg * kSegV;
  const int nv = (int)(left < kSegV ? left : kSegV);
  const bool vec = nv == kSegV &&
                   ((reinterpret_cast<uintptr_t>(src) % sizeof(Pack<S, kVec>)) == 0) &&
                   ((reinterpret_cast<uintptr_t>(dst) % sizeof(Pack<D, kVec>)) == 0);
  if (vec) {
    Pack<S, kVec> in[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      in[u] = ld_pack(reinterpret_cast<const Pack<S, kVec>*>(src + (lane + 32 * u) * kVec));
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      Pack<D, kVec> out;
#pragma unroll
      for (int k = 0; k < kVec; ++k) {
        if constexpr (std::is_same<S, float>::value && std::is_same<D, BF16>::value) {
          if (k % 2 == 0) cvt_pair_f32_bf16(in[u].v[k], in[u].v[k + 1], out.v[k], out.v[k + 1]);
        } else {
          out.v[k] = cvt<S, D>(in[u].v[k], bad);
        }
      }
      *reinterpret_cast<Pack<D, kVec>*>(dst + (lane + 32 * u) * kVec) = out;
    }
    return;
  }
  for (int e = lane; e < nv; e += 32) dst[e] = cvt<S, D>(src[e], bad);
}

template <typename S, typename D>
__device__ __forceinline__ void cast_flat(const CastJob& j, int64_t local, uint32_t& bad) {
  const int64_t total = j.nruns * j.run;
#pragma unroll
  for (int k = 0; k < kFlatPer; ++k) {
    const int64_t v = local * kFlat + k * kThreads + threadIdx.x;
    if (v < total) {
      const int64_t r = v / j.run, w = v - r * j.run;
      int64_t so, dof;
      origin(j, r, so, dof);
      reinterpret_cast<D*>(j.dst + dof)[w] = cvt<S, D>(reinterpret_cast<const S*>(j.src + so)[w], bad);
    }
  }
}

template <typename S, typename D>
__device__ __forceinline__ void cast_job(const CastJob& j, int64_t local, uint32_t& bad) {
  if (j.mode == 0) cast_segment<S, D>(j, local, bad);
  else cast_flat<S, D>(j, local, bad);
}

// One kernel per (source, destination) dtype pair: each instantiation holds only its own
// conversion path, so its register allocation (and occupancy) is that path's, not the
// worst case over every pair.  A batch is grouped by pair on the host.
template <typename S, typename D>
__global__ void __launch_bounds__(kThreads) box_cast_kernel(const CastJob* __restrict__ jobs,
                                                            int n_jobs, int64_t block0) {
  const int64_t block = block0 + blockIdx.x;
  const CastJob j = jobs[find_cast_job(jobs, n_jobs, block)];
  const int64_t local = block - j.unit_begin;
  uint32_t bad = 0;
  if (local < j.units) cast_job<S, D>(j, local, bad);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if (bad && (threadIdx.x & 31) == 0) atomicOr(j.flags, bad);
}

using CastKernel = void (*)(const CastJob*, int, int64_t);

template <typename S>
CastKernel pick_dst(int ddt) {
  switch (ddt) {
    case TV_DT_F32: return box_cast_kernel<S, float>;
    case TV_DT_F64: return box_cast_kernel<S, double>;
    case TV_DT_BF16: return box_cast_kernel<S, BF16>;
    case TV_DT_I32: return box_cast_kernel<S, int32_t>;
    case TV_DT_I64: return box_cast_kernel<S, long long>;
    case TV_DT_U8: return box_cast_kernel<S, uint8_t>;
    default: return nullptr;
  }
}

CastKernel pick_kernel(int sdt, int ddt) {
  switch (sdt) {
    case TV_DT_F32: return pick_dst<float>(ddt);
    case TV_DT_F64: return pick_dst<double>(ddt);
    case TV_DT_BF16: return pick_dst<BF16>(ddt);
    case TV_DT_I32: return pick_dst<int32_t>(ddt);
    case TV_DT_I64: return pick_dst<long long>(ddt);
    case TV_DT_U8: return pick_dst<uint8_t>(ddt);
    default: return nullptr;
  }
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
  // Group by dtype pair (one kernel each); units are numbered within each group.
  std::stable_sort(jobs.begin(), jobs.end(), [](const CastJob& a, const CastJob& b) {
    return a.sdt != b.sdt ? a.sdt < b.sdt : a.ddt < b.ddt;
  });
  int64_t total = 0, group = 0;
  for (size_t i = 0; i < jobs.size(); ++i) {
    auto& j = jobs[i];
    if (i > 0 && (j.sdt != jobs[i - 1].sdt || j.ddt != jobs[i - 1].ddt)) group = 0;
    if (j.mode == 0) {
      const int64_t segs = (j.run + kSegV - 1) / kSegV;
      j.units = (j.nruns * segs + kWarps - 1) / kWarps;
    } else {
      j.units = (j.nruns * j.run + kFlat - 1) / kFlat;
    }
    j.unit_begin = group;
    group += j.units;
    total += j.units;
  }
  return total;
}

cudaError_t launch_cast_jobs(const CastJob* dev_jobs, const CastJob* host_jobs, int n_jobs,
                             int64_t, cudaStream_t stream) {
  const int64_t max_grid = 0x7fffffffLL;
  for (int g0 = 0; g0 < n_jobs;) {
    int g1 = g0 + 1;
    while (g1 < n_jobs && host_jobs[g1].sdt == host_jobs[g0].sdt &&
           host_jobs[g1].ddt == host_jobs[g0].ddt)
      ++g1;
    const CastKernel k = pick_kernel(host_jobs[g0].sdt, host_jobs[g0].ddt);
    if (!k) return cudaErrorInvalidValue;
    const int64_t units = host_jobs[g1 - 1].unit_begin + host_jobs[g1 - 1].units;
    for (int64_t b0 = 0; b0 < units; b0 += max_grid) {
      const unsigned grid = (unsigned)std::min<int64_t>(max_grid, units - b0);
      k<<<grid, kThreads, 0, stream>>>(dev_jobs + g0, g1 - g0, b0);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    g0 = g1;
  }
  return cudaSuccess;
}

}  // namespace tv
