#include <cstdio>
#include <cstdlib>
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
#include "tc_util.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdexcept>
#include <string>

namespace fe {

int g_sk_stages = 10;

namespace {

constexpr int BM = 128, BN = 128, BK = 64, kStages = 6;
constexpr int kTileBytes = BM * BK * 2;                   // 16 KB per operand per stage
constexpr int kSmem = kStages * 2 * kTileBytes + 1024 + 256;
constexpr int kThreads = 192;

using namespace tc;

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
  // M tiles fastest: the CTAs sharing a weight tile run together, so wide
  // batches read each weight tile from DRAM once (L2 serves the others)
  const int m_tile = blockIdx.x, n_tile = blockIdx.y;
  const int n0 = n_tile * BN, m0 = m_tile * BM;
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
          const int f0 = n_tile * (BN / 2);
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
      const int f0 = n_tile * (BN / 2);
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

// ----------------------------------------------------------------------------
// Skinny decode GEMM (swap-AB): D[n, b] = sum_k W[n, k] * X[b, k] for up to 16
// batch rows.  A = weights (M = 128 weight rows per tile), B = staged rows
// (N = 16), so every weight byte is streamed from HBM exactly once per
// iteration and consumed by the tensor core (7 rows of FFMA per weight element
// would make a CUDA-core GEMV issue-bound).
//
// Persistent: one CTA per SM walks a static list of units (row tile, K split).
// The TMA ring and the MMA issue run ahead across unit boundaries while two
// TMEM accumulators ping-pong between the MMA warp and the epilogue warps, so
// the weight stream never drains between units.  Split partials are reduced
// in a fixed order by the last CTA of each tile (deterministic), which then
// applies the fused epilogue.
constexpr int SN = 16;                        // batch columns per MMA
constexpr int kSkStagesMax = 10;
constexpr int kSkAcc = 4;                     // TMEM accumulator ring (units in flight)
constexpr int kSkA = BM * BK * 2;             // 16 KB weights per stage
constexpr int kSkB = SN * BK * 2;             // 2 KB activations per stage
template <int STAGES>
constexpr int sk_smem() { return STAGES * (kSkA + kSkB) + BM * (SN + 1) * 4 + 1024 + 2048; }
constexpr uint32_t kSkIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(SN >> 3) << 17) |
                              ((uint32_t)(BM >> 4) << 24);

struct SkArgs {
  int N, K, B;            // weight rows, reduction, live batch rows
  int tiles, splits, kb_per_split, units;
  int epi;
  float* partial;         // [splits][N][B]
  int* counters;          // [tiles]
  // epilogue operands (see TcArgs)
  float* y;               // RESID: x [rows][ldy]
  int ldy;
  __nv_bfloat16* act;
  int F;
  float* q;
  __nv_bfloat16* kv_pool;
  size_t page_elems, layer_off;
  const float* rope;
  const RowMeta* rows;    // batch rows (QKV) / all rows (ARGMAX via head_rows)
  const int32_t* head_rows;
  int H, hd, d;
  unsigned long long* part_keys;  // ARGMAX: [B][tiles]
  float* logits;
  int V, n_text;
};

__device__ __forceinline__ void unit_of(const SkArgs& a, int u, int kb_total, int* tile, int* split, int* kb0,
                                        int* kb1) {
  *tile = u / a.splits;
  *split = u % a.splits;
  *kb0 = *split * a.kb_per_split;
  *kb1 = min(kb_total, *kb0 + a.kb_per_split);
}

template <int kSkStages>
__global__ void __launch_bounds__(kThreads, 1)
skinny_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                 const SkArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = smem;
  unsigned char* sb = smem + kSkStages * kSkA;
  float* tile = (float*)(sb + kSkStages * kSkB);           // [128][SN + 1]
  uint64_t* full = (uint64_t*)(tile + BM * (SN + 1));
  uint64_t* empty = full + kSkStages;
  uint64_t* acc_full = empty + kSkStages;                  // [kSkAcc]
  uint64_t* acc_empty = acc_full + kSkAcc;                 // [kSkAcc]
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + kSkAcc);
  int* last_flag = (int*)(tmem_slot + 1);
  unsigned long long* red = (unsigned long long*)(tmem_slot + 4);  // [SN][4], 8-byte aligned

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb_total = (a.K + BK - 1) / BK;
  const bool swiglu = a.epi == TC_SWIGLU;
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
    for (int s = 0; s < kSkStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < kSkAcc; i++) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // kSkAcc 16-column fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "n"(kSkAcc * SN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer, runs ahead across units
      // Weights do not depend on the previous kernel: the first ring's worth of
      // weight tiles is requested before griddepcontrol.wait (PDL), the
      // activation tiles after it.
      auto load_w = [&](int s, int tl, int kb) {
        if (swiglu) {
          const int f0 = tl * (BM / 2);
          tma_load_2d(sa + s * kSkA, &map_w, &full[s], kb * BK, f0);
          tma_load_2d(sa + s * kSkA + kSkA / 2, &map_w, &full[s], kb * BK, a.F + f0);
        } else {
          tma_load_2d(sa + s * kSkA, &map_w, &full[s], kb * BK, tl * BM);
        }
      };
      int pre = 0;  // stages prefetched before the dependency wait
      {
        int u = blockIdx.x, tl, sp, kb0, kb1;
        if (u < a.units) unit_of(a, u, kb_total, &tl, &sp, &kb0, &kb1);
        int kb = u < a.units ? kb0 : 0;
        while (u < a.units && pre < kSkStages) {
          mbar_expect_tx(&full[pre], kSkA + kSkB);
          load_w(pre, tl, kb);
          pre++;
          if (++kb == kb1) {
            u += gridDim.x;
            if (u < a.units) { unit_of(a, u, kb_total, &tl, &sp, &kb0, &kb1); kb = kb0; }
          }
        }
      }
      pdl_wait();
      int it = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x) {
        int tl, sp, kb0, kb1;
        unit_of(a, u, kb_total, &tl, &sp, &kb0, &kb1);
        for (int kb = kb0; kb < kb1; kb++, it++) {
          const int s = it % kSkStages;
          if (it >= pre) {
            mbar_wait(&empty[s], ((it / kSkStages) & 1) ^ 1);
            mbar_expect_tx(&full[s], kSkA + kSkB);
            load_w(s, tl, kb);
          }
          tma_load_2d(sb + s * kSkB, &map_x, &full[s], kb * BK, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: accumulator (local unit index & 1)
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < a.units; u += gridDim.x, lu++) {
        int tl, sp, kb0, kb1;
        unit_of(a, u, kb_total, &tl, &sp, &kb0, &kb1);
        const int acc = lu % kSkAcc;
        mbar_wait(&acc_empty[acc], ((lu / kSkAcc) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dst = tmem + (uint32_t)(acc * SN);
        for (int kb = kb0; kb < kb1; kb++, it++) {
          const int s = it % kSkStages;
          mbar_wait(&full[s], (it / kSkStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = smem_desc(sa + s * kSkA);
          const uint64_t db = smem_desc(sb + s * kSkB);
#pragma unroll
          for (int k = 0; k < BK / 16; k++) {
            const uint64_t off = (uint64_t)((k * 32) >> 4);
            const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0;"
                " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                ::"r"(dst), "l"(da + off), "l"(db + off), "r"(kSkIdesc), "r"(accum));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(su32(&empty[s])) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(su32(&acc_full[acc])) : "memory");
      }
    }
  } else {
    // ---- epilogue warps: thread <-> weight row r of the tile
    const int r = 32 * (warp & 3) + lane;
    const int et = threadIdx.x - 64;  // 0..127
    pdl_wait();  // epilogue writes / reads outputs of earlier kernels
    int lu = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, lu++) {
      int tl, sp, kb0, kb1;
      unit_of(a, u, kb_total, &tl, &sp, &kb0, &kb1);
      const int acc = lu % kSkAcc;
      mbar_wait(&acc_full[acc], (lu / kSkAcc) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t raw[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(raw[0]), "=r"(raw[1]), "=r"(raw[2]), "=r"(raw[3]), "=r"(raw[4]), "=r"(raw[5]), "=r"(raw[6]),
            "=r"(raw[7]), "=r"(raw[8]), "=r"(raw[9]), "=r"(raw[10]), "=r"(raw[11]), "=r"(raw[12]), "=r"(raw[13]),
            "=r"(raw[14]), "=r"(raw[15])
          : "r"(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(acc * SN)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // accumulator drained: hand it back to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acc_empty[acc])) : "memory");

      const int n0 = tl * BM;
      const int nrow = swiglu ? (r < 64 ? tl * 64 + r : a.F + tl * 64 + r - 64) : n0 + r;
      const bool row_ok = nrow < a.N;
      if (a.splits == 1) {
#pragma unroll
        for (int b = 0; b < SN; b++) tile[r * (SN + 1) + b] = __uint_as_float(raw[b]);
      } else {
        // partial of this unit: [unit][128 rows][16 columns] fp32, 4 x 16-byte stores per thread
        float4* dst = reinterpret_cast<float4*>(a.partial + ((size_t)u * BM + r) * SN);
#pragma unroll
        for (int i = 0; i < SN / 4; i++)
          __stcg(dst + i, make_float4(__uint_as_float(raw[4 * i]), __uint_as_float(raw[4 * i + 1]),
                                      __uint_as_float(raw[4 * i + 2]), __uint_as_float(raw[4 * i + 3])));
        // one gpu-scope fence per CTA after the CTA barrier publishes all 128
        // threads' partials before the arrival count (split-K serial pattern)
        __threadfence();  // each thread publishes its rows of the partial
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          const int prev = atomicAdd(&a.counters[tl], 1);
          const bool last = prev == a.splits - 1;
          if (last) {
            a.counters[tl] = 0;  // reset for the next launch
            __threadfence();
          }
          *last_flag = last;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (!*last_flag) continue;
        // fixed-order reduction over the tile's splits (units tl*splits .. +splits-1)
        float4 acc4[SN / 4];
#pragma unroll
        for (int i = 0; i < SN / 4; i++) acc4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < a.splits; q++) {
          const float4* src = reinterpret_cast<const float4*>(a.partial + ((size_t)(tl * a.splits + q) * BM + r) * SN);
          float4 v[SN / 4];
#pragma unroll
          for (int i = 0; i < SN / 4; i++) v[i] = __ldcg(src + i);
#pragma unroll
          for (int i = 0; i < SN / 4; i++) {
            acc4[i].x += v[i].x; acc4[i].y += v[i].y; acc4[i].z += v[i].z; acc4[i].w += v[i].w;
          }
        }
#pragma unroll
        for (int i = 0; i < SN / 4; i++) {
          tile[r * (SN + 1) + 4 * i] = acc4[i].x;
          tile[r * (SN + 1) + 4 * i + 1] = acc4[i].y;
          tile[r * (SN + 1) + 4 * i + 2] = acc4[i].z;
          tile[r * (SN + 1) + 4 * i + 3] = acc4[i].w;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      // ---- fused epilogues on the reduced [128 x B] tile
      if (a.epi == TC_RESID) {
        if (row_ok)
          for (int b = 0; b < a.B; b++) a.y[(size_t)b * a.ldy + nrow] += tile[r * (SN + 1) + b];
      } else if (a.epi == TC_SWIGLU) {
        if (et < 64 && tl * 64 + et < a.F)
          for (int b = 0; b < a.B; b++)
            a.act[(size_t)b * a.F + tl * 64 + et] =
                __float2bfloat16_rn(silu_mul(tile[et * (SN + 1) + b], tile[(et + 64) * (SN + 1) + b]));
      } else if (a.epi == TC_QKV) {
        if (et < 64) {
          const int sec = n0 / a.d, h = (n0 % a.d) / a.hd, half = a.hd >> 1;
          for (int b = 0; b < a.B; b++) {
            const RowMeta m = a.rows[b];
            float x1 = tile[et * (SN + 1) + b], x2 = tile[(et + half) * (SN + 1) + b];
            if (sec < 2) {
              const float* cs = a.rope + (size_t)m.pos * a.hd;
              const float co = cs[et], sn = cs[half + et];
              const float r1 = __fmaf_rn(x1, co, -__fmul_rn(x2, sn));
              const float r2 = __fmaf_rn(x2, co, __fmul_rn(x1, sn));
              x1 = r1;
              x2 = r2;
            }
            if (sec == 0) {
              float* qr = a.q + (size_t)b * a.d + h * a.hd;
              qr[et] = x1;
              qr[et + half] = x2;
            } else {
              __nv_bfloat16* kv = a.kv_pool + (size_t)m.kv_page * a.page_elems + a.layer_off +
                                  ((size_t)((sec - 1) * a.H + h) * FE_PAGE + m.kv_slot) * a.hd;
              kv[et] = __float2bfloat16_rn(x1);
              kv[et + half] = __float2bfloat16_rn(x2);
            }
          }
        }
      } else if (a.epi == TC_ARGMAX) {
        for (int b = 0; b < a.B; b++) {
          const float v = tile[r * (SN + 1) + b];
          unsigned long long k = (row_ok && nrow < a.n_text) ? argmax_key(v, nrow) : 0ull;
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, off));
          if (lane == 0) red[b * 4 + (warp & 3)] = k;
          if (row_ok && a.logits) {
            const RowMeta m = a.rows[a.head_rows[b]];
            if (m.logit_row >= 0) a.logits[(size_t)m.logit_row * a.V + nrow] = v;
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et < a.B) {
          unsigned long long k = 0ull;
          for (int w = 0; w < 4; w++) k = max(k, red[et * 4 + w]);
          a.part_keys[(size_t)et * a.tiles + tl] = k;
        }
      } else {  // TC_STORE: y[b][n]
        if (row_ok)
          for (int b = 0; b < a.B; b++) a.y[(size_t)b * a.ldy + nrow] = tile[r * (SN + 1) + b];
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // tile / red reused by the next unit
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kSkAcc * SN));
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

int skinny_max_rows() { return SN; }

int skinny_tiles(int epi, int N, int F) { return epi == TC_SWIGLU ? F / (BM / 2) : (N + BM - 1) / BM; }

void launch_skinny_tc(const TmaMap& w_map, const TmaMap& x_map, const SkLaunch& l, cudaStream_t s) {
  static bool configured = false;
  static int n_sm = 148;
  if (!configured) {
    cudaFuncSetAttribute(skinny_tc_kernel<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, sk_smem<10>());
    cudaFuncSetAttribute(skinny_tc_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, sk_smem<5>());
    // maximum shared-memory carveout, so two 5-stage CTAs (of consecutive
    // PDL-chained launches) can be resident on one SM
    cudaFuncSetAttribute(skinny_tc_kernel<5>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(skinny_tc_kernel<10>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (getenv("FE_DEBUG_OCC")) {
      int o5 = 0, o10 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o5, skinny_tc_kernel<5>, kThreads, sk_smem<5>());
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o10, skinny_tc_kernel<10>, kThreads, sk_smem<10>());
      fprintf(stderr, "skinny occupancy: 5 stages %d CTAs/SM (%d B), 10 stages %d CTAs/SM (%d B)\n", o5, sk_smem<5>(), o10,
              sk_smem<10>());
      size_t avail1 = 0, avail2 = 0;
      cudaOccupancyAvailableDynamicSMemPerBlock(&avail1, skinny_tc_kernel<5>, 1, kThreads);
      cudaOccupancyAvailableDynamicSMemPerBlock(&avail2, skinny_tc_kernel<5>, 2, kThreads);
      int smpm = 0, smpb = 0;
      cudaDeviceGetAttribute(&smpm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
      cudaDeviceGetAttribute(&smpb, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
      fprintf(stderr, "avail dyn smem: 1 CTA %zu, 2 CTAs %zu; per SM %d, per block optin %d\n", avail1, avail2, smpm, smpb);
      cudaFuncAttributes fa{};
      cudaError_t er = cudaFuncGetAttributes(&fa, skinny_tc_kernel<5>);
      fprintf(stderr, "attrs(%d): regs %d static %zu maxdyn %d carveout %d maxthreads %d\n", (int)er, fa.numRegs,
              fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.preferredShmemCarveout, fa.maxThreadsPerBlock);
      int rps = 0, maxb = 0;
      cudaDeviceGetAttribute(&rps, cudaDevAttrMaxRegistersPerMultiprocessor, 0);
      cudaDeviceGetAttribute(&maxb, cudaDevAttrMaxBlocksPerMultiprocessor, 0);
      fprintf(stderr, "regs/SM %d max blocks/SM %d\n", rps, maxb);
    }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    configured = true;
  }
  const int tiles = skinny_tiles(l.epi, l.N, l.F);
  const int kb_total = (l.K + BK - 1) / BK;
  // Pick the K split that balances units over the persistent CTAs, keeping the
  // split partial traffic (splits * N * B * 8 bytes) under ~8% of the weights.
  const double weight_bytes = (double)l.N * l.K * 2.0;
  int best_kb = kb_total;
  double best_eff = -1.0;
  for (int kb_per = kb_total; kb_per >= 4; kb_per--) {
    const int splits = (kb_total + kb_per - 1) / kb_per;
    const int units = tiles * splits;
    if (splits > 1 && (units * (double)BM * SN * 8.0 > 0.06 * weight_bytes || splits > 8)) break;
    const int rounds = (units + n_sm - 1) / n_sm;
    // balance, with a small per-unit epilogue cost
    const double eff = (double)tiles * kb_total / ((double)n_sm * rounds * (kb_per + 1.0));
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best_kb = kb_per;
    }
  }
  SkArgs a{};
  a.N = l.N; a.K = l.K; a.B = l.B; a.epi = l.epi;
  a.kb_per_split = best_kb;
  a.splits = (kb_total + best_kb - 1) / best_kb;
  a.tiles = tiles;
  a.units = tiles * a.splits;
  a.partial = l.partial; a.counters = l.counters;
  a.y = l.y; a.ldy = l.ldy; a.act = l.act; a.F = l.F; a.q = l.q; a.kv_pool = l.kv_pool;
  a.page_elems = l.page_elems; a.layer_off = l.layer_off; a.rope = l.rope; a.rows = l.rows;
  a.head_rows = l.head_rows; a.H = l.H; a.hd = l.hd; a.d = l.d; a.part_keys = l.part_keys;
  a.logits = l.logits; a.V = l.V; a.n_text = l.n_text;
  const int grid = std::min(a.units, n_sm);
  const CUtensorMap& wm = *reinterpret_cast<const CUtensorMap*>(w_map.bytes);
  const CUtensorMap& xm = *reinterpret_cast<const CUtensorMap*>(x_map.bytes);
  if (g_sk_stages <= 5) launch_k(skinny_tc_kernel<5>, dim3(grid), dim3(kThreads), (size_t)sk_smem<5>(), s, wm, xm, a);
  else launch_k(skinny_tc_kernel<10>, dim3(grid), dim3(kThreads), (size_t)sk_smem<10>(), s, wm, xm, a);
}

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
  dim3 grid((l.M + BM - 1) / BM, n_tiles);
  gemm_tc_kernel<<<grid, kThreads, kSmem, s>>>(*reinterpret_cast<const CUtensorMap*>(a_map.bytes),
                                               *reinterpret_cast<const CUtensorMap*>(b_map.bytes), a);
}

}  // namespace fe
