// tcgen05 tensor-core GEMM for the dense contractions of the bf16 path
// (trunk prefill and wide row batches): D[m, n] = sum_k A[m, k] * B[n, k]
// with A = staged activations [rows, K] and B = weights [N, K], both
// K-major bf16, fp32 accumulation in TMEM.
//
// Per CTA one 128 x 128 output tile:
//   warp 0      TMA producer: 128B-swizzled [128 x 64] boxes of A and B into a
//               kStages-deep shared-memory ring (mbarrier full/empty pipeline)
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue
//               (M=128, N=128, K=16 per instruction, 4 per 64-wide k-block),
//               tcgen05.commit releases ring slots and signals the epilogue
//   warps 2-5   epilogue: tcgen05.ld 32x32b rows of the accumulator, fused
//               RoPE + paged-KV append (QKV), residual add (O / down),
//               SiLU(gate)*up (gate/up, B tile = 64 gate rows ++ 64 up rows),
//               or a plain fp32 store.
// bf16 mode only: the tensor-core reduction order is not the canonical one,
// so the fp32 (bit-exact) mode keeps using the CUDA-core GEMV.
#include "common.cuh"
#include "engine_internal.h"
#include "gemm_tc.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <stdexcept>
#include <string>

namespace fe {

namespace {

constexpr int BM = 128, BN = 128, BK = 64, kStages = 6;
constexpr int kTileBytes = BM * BK * 2;                   // 16 KB per operand per stage
constexpr int kSmem = kStages * 2 * kTileBytes + 1024 + 256;
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(su32(dst)), "l"(map), "r"(x), "r"(y), "r"(su32(bar)) : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  const uint64_t addr = su32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= (uint64_t)1 << 16;                // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;      // SBO
  d |= (uint64_t)1 << 46;                // version (sm100)
  d |= (uint64_t)2 << 61;                // SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B bf16, K-major both, N = 128, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; i++) v[i] = __uint_as_float(r[i]);
}

struct TcArgs {
  int M, N, K;          // rows of A (tokens), output features, reduction
  int epi;              // TcEpi
  float* y;             // STORE: [M][ldy]; RESID: residual stream [M][N]
  int ldy;
  __nv_bfloat16* act;   // SWIGLU: [M][F]
  int F;
  // QKV
  float* q;
  __nv_bfloat16* kv_pool;
  size_t page_elems, layer_off;
  const float* rope;
  const RowMeta* rows;
  int H, hd, d;
};

__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = smem;                               // [kStages][128 x 64] bf16
  unsigned char* sb = smem + kStages * kTileBytes;        // [kStages][128 x 64] bf16
  uint64_t* full = (uint64_t*)(smem + 2 * kStages * kTileBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = (uint32_t*)(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int kblocks = (a.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 128 fp32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (int kb = 0; kb < kblocks; kb++) {
        const int s = kb % kStages;
        const uint32_t round = kb / kStages;
        mbar_wait(&empty[s], (round & 1) ^ 1);
        mbar_expect_tx(&full[s], 2 * kTileBytes);
        tma_load_2d(sa + s * kTileBytes, &map_a, &full[s], kb * BK, m0);
        if (a.epi == TC_SWIGLU) {  // 64 gate rows ++ 64 up rows of the same features
          const int f0 = blockIdx.x * (BN / 2);
          tma_load_2d(sb + s * kTileBytes, &map_b, &full[s], kb * BK, f0);
          tma_load_2d(sb + s * kTileBytes + kTileBytes / 2, &map_b, &full[s], kb * BK, a.F + f0);
        } else {
          tma_load_2d(sb + s * kTileBytes, &map_b, &full[s], kb * BK, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      for (int kb = 0; kb < kblocks; kb++) {
        const int s = kb % kStages;
        mbar_wait(&full[s], (kb / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = smem_desc(sa + s * kTileBytes);
        const uint64_t db = smem_desc(sb + s * kTileBytes);
#pragma unroll
        for (int k = 0; k < BK / 16; k++) {
          // advance 16 bf16 = 32 bytes along K inside the swizzle atom
          const uint64_t off = (uint64_t)((k * 32) >> 4);
          const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
          asm volatile(
              "{ .reg .pred p; setp.ne.b32 p, %4, 0;"
              " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
              ::"r"(tmem), "l"(da + off), "l"(db + off), "r"(kIdesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(su32(&empty[s])) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(su32(tmem_full)) : "memory");
    }
  } else {
    // ---- epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31
    const int lane_base = 32 * (warp & 3);
    const int row = m0 + lane_base + lane;
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = tmem + ((uint32_t)lane_base << 16);
    const bool live = row < a.M;
    if (a.epi == TC_STORE || a.epi == TC_RESID) {
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(tbase + c, v);
        if (!live) continue;
        float* dst = a.y + (size_t)row * a.ldy + n0 + c;
        if (a.epi == TC_STORE) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        } else {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 o = *reinterpret_cast<float4*>(dst + i);
            o.x += v[i]; o.y += v[i + 1]; o.z += v[i + 2]; o.w += v[i + 3];
            *reinterpret_cast<float4*>(dst + i) = o;
          }
        }
      }
    } else if (a.epi == TC_SWIGLU) {
      const int f0 = blockIdx.x * (BN / 2);
      for (int c = 0; c < BN / 2; c += 32) {
        float g[32], u[32];
        tmem_ld32(tbase + c, g);
        tmem_ld32(tbase + BN / 2 + c, u);
        if (!live) continue;
        __nv_bfloat16* dst = a.act + (size_t)row * a.F + f0 + c;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          __nv_bfloat162 p;
          p.x = __float2bfloat16_rn(silu_mul(g[i], u[i]));
          p.y = __float2bfloat16_rn(silu_mul(g[i + 1], u[i + 1]));
          *reinterpret_cast<__nv_bfloat162*>(dst + i) = p;
        }
      }
    } else {  // TC_QKV: tile = one head of the q, k or v section (BN == head_dim == 128)
      const int sec = n0 / a.d, h = (n0 % a.d) / a.hd, half = a.hd >> 1;
      RowMeta m{};
      if (live) m = a.rows[row];
      for (int c = 0; c < half; c += 32) {
        float x1[32], x2[32];
        tmem_ld32(tbase + c, x1);
        tmem_ld32(tbase + half + c, x2);
        if (!live) continue;
        if (sec < 2) {
          const float* cs = a.rope + (size_t)m.pos * a.hd;
#pragma unroll
          for (int i = 0; i < 32; i++) {
            const float co = cs[c + i], sn = cs[half + c + i];
            const float r1 = __fmaf_rn(x1[i], co, -__fmul_rn(x2[i], sn));
            const float r2 = __fmaf_rn(x2[i], co, __fmul_rn(x1[i], sn));
            x1[i] = r1;
            x2[i] = r2;
          }
        }
        if (sec == 0) {
          float* qr = a.q + (size_t)row * a.d + h * a.hd;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            *reinterpret_cast<float4*>(qr + c + i) = make_float4(x1[i], x1[i + 1], x1[i + 2], x1[i + 3]);
            *reinterpret_cast<float4*>(qr + half + c + i) = make_float4(x2[i], x2[i + 1], x2[i + 2], x2[i + 3]);
          }
        } else {
          __nv_bfloat16* kv = a.kv_pool + (size_t)m.kv_page * a.page_elems + a.layer_off +
                              ((size_t)((sec - 1) * a.H + h) * FE_PAGE + m.kv_slot) * a.hd;
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            __nv_bfloat162 p1, p2;
            p1.x = __float2bfloat16_rn(x1[i]); p1.y = __float2bfloat16_rn(x1[i + 1]);
            p2.x = __float2bfloat16_rn(x2[i]); p2.y = __float2bfloat16_rn(x2[i + 1]);
            *reinterpret_cast<__nv_bfloat162*>(kv + c + i) = p1;
            *reinterpret_cast<__nv_bfloat162*>(kv + half + c + i) = p2;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

}  // namespace

TmaMap make_kmajor_map(const void* base, int rows, int K, int ld_elems, int box_rows) {
  TmaMap t{};
  CUtensorMap* map = reinterpret_cast<CUtensorMap*>(t.bytes);
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 2};
  const cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return t;
}

int tc_box_rows(int epi) { return epi == TC_SWIGLU ? BN / 2 : BN; }

void launch_gemm_tc(const TmaMap& a_map, const TmaMap& b_map, const TcLaunch& l, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  TcArgs a{};
  a.M = l.M; a.N = l.N; a.K = l.K; a.epi = l.epi;
  a.y = l.y; a.ldy = l.ldy; a.act = l.act; a.F = l.F;
  a.q = l.q; a.kv_pool = l.kv_pool; a.page_elems = l.page_elems; a.layer_off = l.layer_off;
  a.rope = l.rope; a.rows = l.rows; a.H = l.H; a.hd = l.hd; a.d = l.d;
  const int n_tiles = l.epi == TC_SWIGLU ? (l.F / (BN / 2)) : (l.N / BN);
  dim3 grid(n_tiles, (l.M + BM - 1) / BM);
  gemm_tc_kernel<<<grid, kThreads, kSmem, s>>>(*reinterpret_cast<const CUtensorMap*>(a_map.bytes),
                                               *reinterpret_cast<const CUtensorMap*>(b_map.bytes), a);
}

}  // namespace fe
