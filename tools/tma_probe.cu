// Design probe: is TMA (cp.async.bulk, global -> shared -> global through an mbarrier
// pipeline) a faster way than the box-copy kernel's LDG.128/STG.128 to move the large
// contiguous runs of a device snapshot?  Copies N bytes device-to-device three ways and
// prints GB/s (read + write bytes, the MEASURED_PEAKS convention):
//   ldst  — grid-stride 16-byte vector copy, 8 vectors in flight per lane (box_copy's
//           contiguous path)
//   tma   — persistent CTAs (one per SM x k), each streaming 32 KiB blocks through a
//           STAGES-deep shared-memory ring: one elected thread issues
//           cp.async.bulk.shared::cluster.global (completion on an mbarrier) and
//           cp.async.bulk.global.shared::cta (bulk_group) per block
//   ce    — cudaMemcpyAsync device-to-device (copy engines)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
//   tools/tma_probe [GiB]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

constexpr int kBlock = 16 * 1024;  // granularity of the copied size (lcm of variants' blocks)

__global__ void __launch_bounds__(256) ldst_copy(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                 int64_t n_vec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  for (int64_t base = ((int64_t)blockIdx.x * blockDim.x) * 8 + threadIdx.x; base < n_vec; base += stride) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int64_t i = base + (int64_t)k * blockDim.x;
      if (i < n_vec)
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                     : "l"(src + i));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int64_t i = base + (int64_t)k * blockDim.x;
      if (i < n_vec) dst[i] = v[k];
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kStages, int kBlock>
__global__ void __launch_bounds__(32) tma_copy(const char* __restrict__ src, char* __restrict__ dst,
                                               int64_t n_blocks) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[kStages];
  if (threadIdx.x != 0) return;  // one elected thread drives the whole pipeline
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[kStages] = {0};
  const int64_t first = blockIdx.x, step = gridDim.x;
  // prologue: fill the ring
  int64_t issued = first;
  for (int s = 0; s < kStages && issued < n_blocks; ++s, issued += step) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"(kBlock));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + s * kBlock)),
        "l"(src + issued * kBlock), "r"(kBlock), "r"(smem_u32(&full[s]))
        : "memory");
  }
  int s = 0;
  for (int64_t b = first; b < n_blocks; b += step) {
    // wait for block b to land in stage s
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&full[s])),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + b * kBlock),
                 "r"(smem_u32(smem + s * kBlock)), "r"(kBlock)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (issued < n_blocks) {
      // the stage is refilled only after its store has finished reading shared memory
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                   "r"(kBlock));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + s * kBlock)),
          "l"(src + issued * kBlock), "r"(kBlock), "r"(smem_u32(&full[s]))
          : "memory");
      issued += step;
    }
    s = (s + 1) % kStages;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// Same ring, but a stage is refilled one iteration after its store was issued, so one
// bulk store stays in flight while the next load is issued (wait_group.read 1).
template <int kStages, int kBlock>
__global__ void __launch_bounds__(32) tma_copy2(const char* __restrict__ src, char* __restrict__ dst,
                                                int64_t n_blocks) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t phase[kStages] = {0};
  const int64_t first = blockIdx.x, step = gridDim.x;
  int64_t issued = first;
  for (int s = 0; s < kStages && issued < n_blocks; ++s, issued += step) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"(kBlock));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + s * kBlock)),
        "l"(src + issued * kBlock), "r"(kBlock), "r"(smem_u32(&full[s]))
        : "memory");
  }
  int s = 0, prev = -1;
  for (int64_t b = first; b < n_blocks; b += step) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&full[s])),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + b * kBlock),
                 "r"(smem_u32(smem + s * kBlock)), "r"(kBlock)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (prev >= 0 && issued < n_blocks) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // prev stage's store read
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[prev])),
                   "r"(kBlock));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem + prev * kBlock)),
          "l"(src + issued * kBlock), "r"(kBlock), "r"(smem_u32(&full[prev]))
          : "memory");
      issued += step;
    }
    prev = s;
    s = (s + 1) % kStages;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? std::atof(argv[1]) : 8.0;
  int64_t bytes = (int64_t)(gib * (1 << 30));
  bytes -= bytes % kBlock;
  char *a, *b;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 1, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto time_it = [&](const char* name, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(e0));
      fn();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    std::printf("{\"case\": \"%s\", \"bytes\": %lld, \"ms\": %.3f, \"GBps_rw\": %.1f}\n", name,
                (long long)bytes, best, 2.0 * bytes / (best / 1e3) / 1e9);
  };
  const int64_t n_vec = bytes / 16;
  time_it("ldst_grid_1184x256", [&] { ldst_copy<<<sms * 8, 256>>>((const uint4*)a, (uint4*)b, n_vec); });
  time_it("ldst_grid_full", [&] {
    ldst_copy<<<(unsigned)((n_vec + 2047) / 2048), 256>>>((const uint4*)a, (uint4*)b, n_vec);
  });
  auto tma = [&](auto stages_c, auto block_c, int per_sm) {
    constexpr int S = decltype(stages_c)::value, B = decltype(block_c)::value;
    const int smem = S * B;
    CK(cudaFuncSetAttribute(tma_copy<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    char name[96];
    std::snprintf(name, sizeof name, "tma_%dx%d_stages%d_%dKiB", sms, per_sm, S, B / 1024);
    time_it(name, [&] { tma_copy<S, B><<<sms * per_sm, 32, smem>>>(a, b, bytes / B); });
  };
  auto tma2 = [&](auto stages_c, auto block_c, int per_sm) {
    constexpr int S = decltype(stages_c)::value, B = decltype(block_c)::value;
    const int smem = S * B;
    CK(cudaFuncSetAttribute(tma_copy2<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    char name[96];
    std::snprintf(name, sizeof name, "tma2_%dx%d_stages%d_%dKiB", sms, per_sm, S, B / 1024);
    time_it(name, [&] { tma_copy2<S, B><<<sms * per_sm, 32, smem>>>(a, b, bytes / B); });
  };
  using std::integral_constant;
  tma2(integral_constant<int, 6>{}, integral_constant<int, 32768>{}, 1);
  tma2(integral_constant<int, 12>{}, integral_constant<int, 16384>{}, 1);
  tma2(integral_constant<int, 6>{}, integral_constant<int, 16384>{}, 2);
  tma2(integral_constant<int, 3>{}, integral_constant<int, 65536>{}, 1);
  tma(integral_constant<int, 6>{}, integral_constant<int, 32768>{}, 1);
  tma(integral_constant<int, 3>{}, integral_constant<int, 32768>{}, 2);
  tma(integral_constant<int, 6>{}, integral_constant<int, 16384>{}, 2);
  tma(integral_constant<int, 3>{}, integral_constant<int, 65536>{}, 1);
  tma(integral_constant<int, 4>{}, integral_constant<int, 16384>{}, 3);
  tma(integral_constant<int, 12>{}, integral_constant<int, 16384>{}, 1);
  time_it("ce_memcpy_d2d", [&] { CK(cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice)); });
  // correctness of the TMA path
  CK(cudaMemset(b, 0, bytes));
  CK(cudaMemset(a, 0x5a, bytes));
  tma_copy<6, 32768><<<sms, 32, 6 * 32768>>>(a, b, bytes / 32768);
  CK(cudaDeviceSynchronize());
  unsigned char probe[4] = {0};
  CK(cudaMemcpy(probe, b + bytes - 4, 4, cudaMemcpyDeviceToHost));
  std::printf("{\"tma_tail_ok\": %s}\n", probe[0] == 0x5a && probe[3] == 0x5a ? "true" : "false");
  CK(cudaMemset(b, 0, bytes));
  CK(cudaFuncSetAttribute(tma_copy2<6, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768));
  tma_copy2<6, 32768><<<sms, 32, 6 * 32768>>>(a, b, bytes / 32768);
  CK(cudaDeviceSynchronize());
  unsigned char* hb = (unsigned char*)std::malloc(bytes);
  CK(cudaMemcpy(hb, b, bytes, cudaMemcpyDeviceToHost));
  int64_t bad = 0;
  for (int64_t i = 0; i < bytes; ++i) bad += hb[i] != 0x5a;
  std::printf("{\"tma2_all_bytes_ok\": %s}\n", bad == 0 ? "true" : "false");
  return 0;
}
