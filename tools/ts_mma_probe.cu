// Probe: weights staged smem -> TMEM with tcgen05.cp (128x256b, SW128 K-major
// descriptor), then tcgen05.mma with A read from TMEM ("TS" form), against the
// usual A-from-shared ("SS") MMA on the same 128 x 64 tile and 16 x 64 batch
// tile.  Used to validate the O-weights-in-TMEM staging of the decode tick.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/ts_mma_probe.cu -o tools/ts_mma_probe
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_2506_07639_b200/csrc/tc_util.cuh"

using namespace fe::tc;
constexpr int MT = 128, XR = 16, KBK = 64;

__device__ void store_sw128(unsigned char* tile, const __nv_bfloat16* src, int rows) {
  // row r, 16-byte chunk c -> r * 128 + ((c ^ (r & 7)) * 16)
  for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) {
    const int r = i / 8, c = i % 8;
    const uint4 v = *reinterpret_cast<const uint4*>(src + r * KBK + c * 8);
    *reinterpret_cast<uint4*>(tile + r * 128 + ((c ^ (r & 7)) * 16)) = v;
  }
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* out_ss, float* out_ts) {
  __shared__ __align__(1024) unsigned char sa[MT * 128];
  __shared__ __align__(1024) unsigned char sb[XR * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  store_sw128(sa, A, MT);
  store_sw128(sb, B, XR);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t idesc = idesc_bf16(MT, XR);
  // columns: [0,16) SS accumulator, [16,32) TS accumulator, [64,96) A copy
  if (threadIdx.x == 0) {
    const uint64_t da = smem_desc(sa), db = smem_desc(sb);
    for (int k = 0; k < KBK / 16; k++) {
      const uint64_t off = (uint64_t)((k * 32) >> 4);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 64 + k * 8), "l"(da + off));
    }
    for (int k = 0; k < KBK / 16; k++) {
      const uint64_t off = (uint64_t)((k * 32) >> 4);
      const uint32_t acc = k > 0;
      asm volatile(
          "{ .reg .pred p; setp.ne.b32 p, %4, 0;"
          " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
          ::"r"(tmem), "l"(da + off), "l"(db + off), "r"(idesc), "r"(acc));
      asm volatile(
          "{ .reg .pred p; setp.ne.b32 p, %4, 0;"
          " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
          ::"r"(tmem + 16), "r"(tmem + 64 + k * 8), "l"(db + off), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int which = 0; which < 2; which++) {
    uint32_t raw[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(raw[0]), "=r"(raw[1]), "=r"(raw[2]), "=r"(raw[3]), "=r"(raw[4]), "=r"(raw[5]), "=r"(raw[6]),
          "=r"(raw[7]), "=r"(raw[8]), "=r"(raw[9]), "=r"(raw[10]), "=r"(raw[11]), "=r"(raw[12]), "=r"(raw[13]),
          "=r"(raw[14]), "=r"(raw[15])
        : "r"(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(which * 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float* o = which ? out_ts : out_ss;
    for (int j = 0; j < 16; j++) o[(32 * warp + lane) * XR + j] = __uint_as_float(raw[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(128));
}

int main() {
  __nv_bfloat16 hA[MT * KBK], hB[XR * KBK];
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 9) & 0xFFFF) / 32768.0f - 1.0f; };
  for (auto& v : hA) v = __float2bfloat16(rnd());
  for (auto& v : hB) v = __float2bfloat16(rnd());
  __nv_bfloat16 *dA, *dB;
  float *dss, *dts;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dss, MT * XR * 4); cudaMalloc(&dts, MT * XR * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  probe<<<1, 128>>>(dA, dB, dss, dts);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("ts_mma_probe: CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  static float ss[MT * XR], ts[MT * XR];
  cudaMemcpy(ss, dss, sizeof ss, cudaMemcpyDeviceToHost);
  cudaMemcpy(ts, dts, sizeof ts, cudaMemcpyDeviceToHost);
  double max_ref = 0, max_ss = 0, max_ts = 0;
  for (int r = 0; r < MT; r++)
    for (int c = 0; c < XR; c++) {
      double ref = 0;
      for (int k = 0; k < KBK; k++) ref += (double)__bfloat162float(hA[r * KBK + k]) * __bfloat162float(hB[c * KBK + k]);
      max_ref = fmax(max_ref, fabs(ref));
      max_ss = fmax(max_ss, fabs(ref - ss[r * XR + c]));
      max_ts = fmax(max_ts, fabs(ref - ts[r * XR + c]));
    }
  int same = 0;
  for (int i = 0; i < MT * XR; i++) same += ss[i] == ts[i];
  printf("ts_mma_probe: max|ref| %.3f  SS err %.2e  TS err %.2e  TS==SS bitwise %d/%d\n", max_ref, max_ss, max_ts, same,
         MT * XR);
  return (max_ts < 1e-3 && same == MT * XR) ? 0 : 2;
}
