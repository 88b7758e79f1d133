// Design probe (round 2): would a 2-D tensor-map TMA pack beat the box-copy kernel on the
// strided packs of the save path?  The replica-parallel save packs column boxes out of
// row-major shards (q/o (1024,2048) out of (1024,4096), down
// (1024,7168) out of (1024,14336)); a tensor-parallel reshard cuts narrower ones.  Each
// case packs every row's first W bf16 columns of an (R, C) array into a dense (R, W)
// array three ways and prints GB/s (read + write bytes, the MEASURED_PEAKS convention):
//   box_copy — the product kernel, through the library's C ABI (tv_copy_boxes)
//   tma2d    — persistent CTAs; one elected thread streams (BH x BW) tiles through a
//              STAGES-deep shared-memory ring: cp.async.bulk.tensor.2d load (source
//              tensor map, completion on an mbarrier) then cp.async.bulk.tensor.2d store
//              (destination tensor map, bulk_group); a stage is refilled once its store
//              has read it (wait_group.read 1: one store in flight behind each load)
//   ce2d     — cudaMemcpy2DAsync device-to-device (copy engines)
// Every output is compared with box_copy's on the device.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Iinclude \
//        -o tools/tma2d_pack_probe tools/tma2d_pack_probe.cu \
//        -Lpaper_2605_23066_b200 -ltvgpu -Xlinker -rpath,'$ORIGIN/../paper_2605_23066_b200' \
//        -L/usr/local/cuda/lib64/stubs -lcuda
//   tools/tma2d_pack_probe            (LD_LIBRARY_PATH=<dir> times another libtvgpu.so build)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tvgpu.h"

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void load_tile(const CUtensorMap* map, uint32_t dst, uint32_t bar, int x, int y,
                                          uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

template <int kStages>
__global__ void __launch_bounds__(32) tma2d_pack(const __grid_constant__ CUtensorMap src_map,
                                                 const __grid_constant__ CUtensorMap dst_map, int bw, int bh,
                                                 int tiles_x, int64_t n_tiles) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t full[kStages];
  if (threadIdx.x != 0) return;  // one elected thread drives the pipeline
  const uint32_t tile_bytes = (uint32_t)bw * bh * 2;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[kStages] = {0};
  const int64_t step = gridDim.x;
  int64_t issued = blockIdx.x;
  for (int s = 0; s < kStages && issued < n_tiles; ++s, issued += step)
    load_tile(&src_map, smem_u32(smem + (size_t)s * tile_bytes), smem_u32(&full[s]),
              (int)(issued % tiles_x) * bw, (int)(issued / tiles_x) * bh, tile_bytes);
  int s = 0, prev = -1;
  for (int64_t t = blockIdx.x; t < n_tiles; t += step) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&full[s])),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(&dst_map)),
                 "r"((int)(t % tiles_x) * bw), "r"((int)(t / tiles_x) * bh),
                 "r"(smem_u32(smem + (size_t)s * tile_bytes))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (prev >= 0 && issued < n_tiles) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // prev stage's store has read it
      load_tile(&src_map, smem_u32(smem + (size_t)prev * tile_bytes), smem_u32(&full[prev]),
                (int)(issued % tiles_x) * bw, (int)(issued / tiles_x) * bh, tile_bytes);
      issued += step;
    }
    prev = s;
    s = (s + 1) % kStages;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void count_diff(const uint4* a, const uint4* b, int64_t n, unsigned long long* bad) {
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 x = a[i], y = b[i];
    local += (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
  if (local) atomicAdd(bad, local);
}

__global__ void fill(uint32_t* p, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (uint32_t)(i * 2654435761u) ^ (uint32_t)(i >> 17);
}

static CUtensorMap make_map(void* base, uint64_t cols, uint64_t rows, uint64_t row_bytes, uint32_t bw,
                            uint32_t bh) {
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {bw, bh};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, base, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::fprintf(stderr, "cuTensorMapEncodeTiled failed: %d\n", (int)r);
    std::exit(1);
  }
  return m;
}

struct Case {
  const char* name;
  int64_t rows, cols, w;  // pack cols [0, w) of an (rows, cols) bf16 array
};

int main() {
  const Case cases[] = {
      {"contiguous_4096_of_4096", 131072, 4096, 4096},  // one run (the snapshot), 1 GiB out
      {"q_o_2048_of_4096", 65536, 4096, 2048},      // 4 KiB runs, 256 MiB out
      {"down_7168_of_14336", 16384, 14336, 7168},   // 14 KiB runs, 224 MiB out
      {"tp_1024_of_4096", 65536, 4096, 1024},       // 2 KiB runs, 128 MiB out
      {"tp_512_of_4096", 131072, 4096, 512},        // 1 KiB runs, 128 MiB out
      {"tp_256_of_4096", 262144, 4096, 256},        // 512 B runs, 128 MiB out
      {"tp_64_of_4096", 1048576, 4096, 64},         // 128 B runs, 128 MiB out
  };
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  unsigned long long* bad;
  CK(cudaMalloc(&bad, sizeof(*bad)));
  for (const Case& c : cases) {
    const int64_t src_bytes = c.rows * c.cols * 2, out_bytes = c.rows * c.w * 2;
    char *src, *ref, *out;
    CK(cudaMalloc(&src, src_bytes));
    CK(cudaMalloc(&ref, out_bytes));
    CK(cudaMalloc(&out, out_bytes));
    fill<<<sms * 8, 256>>>((uint32_t*)src, src_bytes / 4);
    auto time_it = [&](const char* how, const char* variant, auto fn) {
      for (int w = 0; w < 3; ++w) fn();
      CK(cudaDeviceSynchronize());
      float best = 1e30f, sum = 0;
      const int reps = 10;
      for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0));
        fn();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
        sum += ms;
      }
      CK(cudaGetLastError());
      unsigned long long nbad = 0;
      if (std::strcmp(how, "box_copy") != 0) {
        CK(cudaMemset(bad, 0, sizeof(*bad)));
        count_diff<<<sms * 4, 256>>>((const uint4*)ref, (const uint4*)out, out_bytes / 16, bad);
        CK(cudaMemcpy(&nbad, bad, sizeof(nbad), cudaMemcpyDeviceToHost));
        CK(cudaMemset(out, 0, out_bytes));
      }
      std::printf(
          "{\"case\": \"%s\", \"how\": \"%s\", \"variant\": \"%s\", \"run_bytes\": %lld, \"out_bytes\": %lld, "
          "\"best_ms\": %.4f, \"mean_ms\": %.4f, \"GBps_rw_best\": %.1f, \"GBps_rw_mean\": %.1f, "
          "\"mismatched_vectors\": %llu}\n",
          c.name, how, variant, (long long)(c.w * 2), (long long)out_bytes, best, sum / reps,
          2.0 * out_bytes / (best / 1e3) / 1e9, 2.0 * out_bytes / (sum / reps / 1e3) / 1e9, nbad);
      std::fflush(stdout);
    };
    tv_copy cp;
    std::memset(&cp, 0, sizeof(cp));
    cp.src.base = (uint64_t)src;
    cp.src.shape[0] = c.rows;
    cp.src.shape[1] = c.cols;
    cp.dst.base = (uint64_t)ref;
    cp.dst.shape[0] = c.rows;
    cp.dst.shape[1] = c.w;
    cp.ext[0] = c.rows;
    cp.ext[1] = c.w;
    cp.rank = 2;
    cp.itemsize = 2;
    time_it("box_copy", "tv_copy_boxes", [&] {
      if (tv_copy_boxes(0, &cp, 1, nullptr) != 0) {
        char msg[512];
        tv_last_error(msg, sizeof msg);
        std::fprintf(stderr, "tv_copy_boxes: %s\n", msg);
        std::exit(1);
      }
    });
    time_it("ce2d", "cudaMemcpy2DAsync", [&] {
      CK(cudaMemcpy2DAsync(out, c.w * 2, src, c.cols * 2, c.w * 2, c.rows, cudaMemcpyDeviceToDevice, 0));
    });
    // tiles: 512 B x 64 rows (32 KiB) when the box is at least 256 columns wide, else
    // W columns x (32 KiB / row bytes) rows
    const int bw = c.w >= 256 ? 256 : (int)c.w;
    const int bh = (int)(32768 / (bw * 2)) > 256 ? 256 : (int)(32768 / (bw * 2));
    const uint32_t tile = (uint32_t)bw * bh * 2;
    CUtensorMap smap = make_map(src, c.cols, c.rows, c.cols * 2, bw, bh);
    CUtensorMap dmap = make_map(out, c.w, c.rows, c.w * 2, bw, bh);
    const int tiles_x = (int)(c.w / bw);
    const int64_t n_tiles = (int64_t)tiles_x * (c.rows / bh);
    auto run_tma = [&](auto stages_c, int per_sm) {
      constexpr int S = decltype(stages_c)::value;
      const int smem = S * tile;
      CK(cudaFuncSetAttribute(tma2d_pack<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      char variant[96];
      std::snprintf(variant, sizeof variant, "tile %dx%d B, %d stages, %d CTA/SM", bh, bw * 2, S, per_sm);
      time_it("tma2d", variant, [&] {
        tma2d_pack<S><<<sms * per_sm, 32, smem>>>(smap, dmap, bw, bh, tiles_x, n_tiles);
      });
    };
    run_tma(std::integral_constant<int, 6>{}, 1);
    run_tma(std::integral_constant<int, 3>{}, 2);
    run_tma(std::integral_constant<int, 4>{}, 1);
    run_tma(std::integral_constant<int, 2>{}, 3);
    CK(cudaFree(src));
    CK(cudaFree(ref));
    CK(cudaFree(out));
  }
  return 0;
}
