// Weight-streaming microbenchmark for the decode-tick design: how fast can
// G CTAs pull a bf16 matrix into shared memory through an S-stage ring?
//   mode 0: 2-D TMA boxes [64 cols x BR rows] (128B swizzle) of a row-major
//           [R][K] matrix, k-blocks innermost (the tick kernel's pattern)
//   mode 1: 1-D bulk copies of BR*128-byte contiguous blocks (weights stored
//           pre-tiled, each ring stage one contiguous run)
//   mode 2: mode 1 plus a second 2 KB bulk copy per stage from a small
//           L2-resident buffer (the tick's activation block)
// One producer thread issues, one consumer thread waits and frees the slot
// (no MMA).  Reports aggregate and per-SM GB/s; a second pass over a buffer
// that fits L2 shows the L2 -> SM rate.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/tma_bw tools/tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const char* base,
                                                       int mode, int BR, int S, int kb_per_row, long boxes) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int stage_bytes = BR * 128;
  uint64_t* full = (uint64_t*)(smem + (size_t)S * stage_bytes);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // CTA c takes boxes c, c + G, ... in tile-major order (contiguous runs of k-blocks per CTA)
  const long per = (boxes + gridDim.x - 1) / gridDim.x;
  const long b0 = blockIdx.x * per, b1 = b0 + per < boxes ? b0 + per : boxes;
  if (threadIdx.x == 0) {
    int it = 0;
    for (long b = b0; b < b1; b++, it++) {
      const int s = it % S;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&empty[s])), "r"(((it / S) & 1) ^ 1) : "memory");
      const int xb = mode == 2 ? 2048 : 0;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes + xb) : "memory");
      if (mode == 2)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(smem + (size_t)S * stage_bytes + 2 * S * 8 + 1024 + (size_t)s * 2048)),
                     "l"(base + (b % 64) * 2048), "r"(2048), "r"(su32(&full[s])) : "memory");
      if (mode == 0) {
        const int kb = (int)(b % kb_per_row), tile = (int)(b / kb_per_row);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(su32(smem + (size_t)s * stage_bytes)), "l"(&map), "r"(kb * 64), "r"(tile * BR), "r"(su32(&full[s]))
            : "memory");
      } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(smem + (size_t)s * stage_bytes)), "l"(base + b * stage_bytes), "r"(stage_bytes),
                     "r"(su32(&full[s])) : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    int it = 0;
    for (long b = b0; b < b1; b++, it++) {
      const int s = it % S;
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&full[s])), "r"((it / S) & 1) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int G = argc > 2 ? atoi(argv[2]) : 148;
  const int BR = argc > 3 ? atoi(argv[3]) : 128;
  const int S = argc > 4 ? atoi(argv[4]) : 11;
  const long mb = argc > 5 ? atol(argv[5]) : 1024;  // matrix size in MB
  const int K = 4096;
  const long R = mb * 1024 * 1024 / (K * 2);
  char* w;
  CK(cudaMalloc(&w, (size_t)R * K * 2));
  CK(cudaMemset(w, 1, (size_t)R * K * 2));
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)R};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)BR};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int stage_bytes = BR * 128;
  const size_t smem = (size_t)S * stage_bytes + 2 * S * 8 + 1024 + (mode == 2 ? (size_t)S * 2048 : 0);
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int kb_per_row = K / 64;
  const long boxes = (R / BR) * kb_per_row;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 6; rep++) {
    cudaEventRecord(e0);
    stream_kernel<<<G, 64, smem>>>(map, w, mode, BR, S, kb_per_row, boxes);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  CK(cudaGetLastError());
  const double bytes = (double)boxes * stage_bytes;
  printf("mode %d G %3d BR %3d S %2d %5ld MB: %7.1f us  %7.0f GB/s  %6.1f GB/s/SM\n", mode, G, BR, S, mb, best * 1e3,
         bytes / best / 1e6, bytes / best / 1e6 / G);
  return 0;
}
