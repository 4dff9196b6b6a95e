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
int g_sk_splits = 0;  // engine option "sk_splits": force the skinny K split (0: cost model)

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
// CTA-pair persistent GEMM (the dense-contraction path: trunk prefill and
// wide decode batches).  A cluster of two CTAs on one TPC computes a
// 256 x BN output tile with tcgen05.mma.cta_group::2 (M = 256): CTA rank r
// stages A rows [m0 + 128 r, +128) and B rows [n0 + BN/2 r, +BN/2) of every
// 64-wide k-block, so each SM streams half the operand bytes of a 1-CTA
// 128 x BN tile of the same MMA rate (L2 -> SM traffic per flop: 128x128
// 1-CTA tiles 1, this kernel 1/2 at BN = 256).  The leader CTA (rank 0)
// issues every MMA; both CTAs' TMA loads complete on the leader's `full`
// barrier, the MMA commit multicasts to both CTAs' `empty` / `tfull`
// barriers, and each CTA's epilogue drains its own 128 TMEM lanes (= its 128
// tile rows x BN columns).  Two TMEM accumulators (2 x BN columns) let the
// epilogue of tile i overlap the mainloop of tile i + 1; tiles are walked
// persistently (m fastest, so concurrently running pairs share weight tiles
// in L2).
//
// B tile columns: rank 0's BN/2 rows then rank 1's; for SwiGLU rank 0 loads
// gate rows [f0, f0 + BN/2) and rank 1 the up rows [F + f0, ...), so columns
// [0, BN/2) are gate and [BN/2, BN) up of the same BN/2 features.  B tensor
// maps use 64-row boxes (BN/2 = 64 or 128 -> 1 or 2 boxes per stage).
// ----------------------------------------------------------------------------
constexpr int kPairThreads = 192;
constexpr int kPairMaxPairs = 74;  // 148 SMs

template <int BN>
__host__ __device__ constexpr int pair_stages() { return BN == 256 ? 6 : 8; }
template <int BN>
__host__ __device__ constexpr int pair_stage_bytes() { return BM * BK * 2 + (BN / 2) * BK * 2; }
template <int BN>
constexpr int pair_smem() { return pair_stages<BN>() * pair_stage_bytes<BN>() + 1024 + 256; }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(saddr), "r"(rank));
  return out;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(su32(b)), "r"(parity) : "memory");
}
// TMA 2-D load into this CTA's shared memory, completing on the pair
// leader's mbarrier (`bar_cluster`: a shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int x, int y,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(su32(dst)), "l"(map), "r"(x), "r"(y), "r"(bar_cluster), "l"(policy) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

struct PairArgs {
  TcArgs t;
  int m_tiles, n_tiles;
  int kblocks;
  // stream-K schedule (DP + one stream-K wave): tiles [0, dp) are walked
  // data-parallel (pair p: p, p + P, ...); the k-iterations of tiles
  // [dp, tiles) are split evenly over the P pairs, pair p taking
  // [p W / P, (p + 1) W / P) of the W = (tiles - dp) * kblocks iterations.
  int dp;
  long long W;
  float* scratch;   // [P][2 slots][2 ranks][BN / 4][128] float4: partial segments
  int* counters;    // [tiles - dp][2 ranks]: arrivals of a tile's partial segments
  // split-K (one m tile, few n tiles: the decode-width regime): data-parallel
  // units (tile, split) over k-ranges of kbs blocks; each unit stores its raw
  // fp32 tile to split_out[split][M][N] and launch_splitk_reduce sums the
  // splits in order and runs the fused epilogue
  int splits, kbs, tiles;
  float* split_out;
};

struct Seg {
  int tile, k0, k1;
  int split;
  bool sk;   // from the stream-K range
};

// The segments of one pair in order (identical walk in every role).
struct SegIter {
  int t_dp, dp, P, KB, tiles, kbs;
  long long i, i1;
  __device__ SegIter(const PairArgs& p, int pair, int n_pairs) {
    P = n_pairs;
    dp = p.dp;
    KB = p.kblocks;
    tiles = p.tiles;
    kbs = p.kbs;
    t_dp = pair;
    i = (long long)pair * p.W / n_pairs;
    i1 = (long long)(pair + 1) * p.W / n_pairs;
  }
  __device__ bool next(Seg& s) {
    if (t_dp < dp) {  // unit t_dp = (tile, split)
      s.tile = t_dp % tiles;
      s.split = t_dp / tiles;
      s.k0 = s.split * kbs;
      s.k1 = min(KB, s.k0 + kbs);
      s.sk = false;
      t_dp += P;
      return true;
    }
    if (i >= i1) return false;
    const int t = (int)(i / KB), k0 = (int)(i % KB);
    const int k1 = (int)min((long long)KB, (long long)k0 + (i1 - i));
    s.tile = dp + t; s.k0 = k0; s.k1 = k1; s.split = 0; s.sk = true;
    i += k1 - k0;
    return true;
  }
};

__device__ __forceinline__ long long sk_start(const PairArgs& p, int q, int P) { return (long long)q * p.W / P; }
// the pair whose stream-K range holds iteration x (the largest q with start(q) <= x)
__device__ __forceinline__ int sk_owner(const PairArgs& p, long long x, int P) {
  int q = (int)(x * P / p.W);
  while (q + 1 < P && sk_start(p, q + 1, P) <= x) q++;
  while (q > 0 && sk_start(p, q, P) > x) q--;
  return q;
}

// Fused epilogue of one tile row (`row`; TMEM lane / scratch row r) over BN
// columns, the accumulator values coming from `ld(c, v)` (32 columns at c).
template <int BN, typename LD>
__device__ __forceinline__ void pair_epilogue_row(const TcArgs& a, int row, int n_tile, LD&& ld) {
  const int n0 = n_tile * BN;
  if (a.epi == TC_STORE || a.epi == TC_RESID) {
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      ld(c, v);
      if (row >= a.M) continue;
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
#pragma unroll 1
    for (int c = 0; c < BN / 2; c += 32) {
      float g[32], u[32];
      ld(c, g);
      ld(BN / 2 + c, u);
      if (row >= a.M) continue;
      __nv_bfloat16* dst = a.act + (size_t)row * a.F + f0 + c;
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          __nv_bfloat162 p;
          p.x = __float2bfloat16_rn(silu_mul(g[i + 2 * j], u[i + 2 * j]));
          p.y = __float2bfloat16_rn(silu_mul(g[i + 2 * j + 1], u[i + 2 * j + 1]));
          w[j] = *reinterpret_cast<uint32_t*>(&p);
        }
        *reinterpret_cast<uint4*>(dst + i) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  } else {  // TC_QKV: BN / 128 heads of the q, k or v section (head_dim 128)
    RowMeta m{};
    if (row < a.M) m = a.rows[row];
#pragma unroll 1
    for (int hh = 0; hh < BN / 128; hh++) {
      const int nh = n0 + hh * 128;
      const int sec = nh / a.d, h = (nh % a.d) / 128;
#pragma unroll 1
      for (int c = 0; c < 64; c += 32) {
        float x1[32], x2[32];
        ld(hh * 128 + c, x1);
        ld(hh * 128 + 64 + c, x2);
        if (row >= a.M) continue;
        if (sec < 2) {
          const float* cs = a.rope + (size_t)m.pos * 128;
#pragma unroll
          for (int i = 0; i < 32; i++) {
            const float co = cs[c + i], sn = cs[64 + c + i];
            const float r1 = __fmaf_rn(x1[i], co, -__fmul_rn(x2[i], sn));
            const float r2 = __fmaf_rn(x2[i], co, __fmul_rn(x1[i], sn));
            x1[i] = r1;
            x2[i] = r2;
          }
        }
        if (sec == 0) {
          float* qr = a.q + (size_t)row * a.d + h * 128;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            *reinterpret_cast<float4*>(qr + c + i) = make_float4(x1[i], x1[i + 1], x1[i + 2], x1[i + 3]);
            *reinterpret_cast<float4*>(qr + 64 + c + i) = make_float4(x2[i], x2[i + 1], x2[i + 2], x2[i + 3]);
          }
        } else {
          __nv_bfloat16* kv = a.kv_pool + (size_t)m.kv_page * a.page_elems + a.layer_off +
                              ((size_t)((sec - 1) * a.H + h) * FE_PAGE + m.kv_slot) * 128;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint32_t w1[4], w2[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
              __nv_bfloat162 p1, p2;
              p1.x = __float2bfloat16_rn(x1[i + 2 * j]); p1.y = __float2bfloat16_rn(x1[i + 2 * j + 1]);
              p2.x = __float2bfloat16_rn(x2[i + 2 * j]); p2.y = __float2bfloat16_rn(x2[i + 2 * j + 1]);
              w1[j] = *reinterpret_cast<uint32_t*>(&p1);
              w2[j] = *reinterpret_cast<uint32_t*>(&p2);
            }
            *reinterpret_cast<uint4*>(kv + c + i) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
            *reinterpret_cast<uint4*>(kv + 64 + c + i) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
          }
        }
      }
    }
  }
}

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
gemm_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const PairArgs p) {
  constexpr int ST = pair_stages<BN>();
  constexpr int kA = BM * BK * 2;               // 16 KB: this CTA's 128 A rows
  constexpr int kB = (BN / 2) * BK * 2;          // this CTA's BN/2 B rows
  constexpr int kBoxB = 64 * BK * 2;             // one 64-row B box
  constexpr uint32_t kIdesc2 = idesc_bf16(256, BN);
  constexpr int kCols = 2 * BN;                  // two accumulators
  constexpr size_t kPart = (size_t)BM * BN;      // floats of one partial (one rank's 128 rows)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = smem;
  unsigned char* sb = smem + ST * kA;
  uint64_t* full = (uint64_t*)(sb + ST * kB);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;   // [2]
  uint64_t* tempty = tfull + 2;   // [2] (leader's: arrivals from both CTAs' epilogues)
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  int* last_flag = (int*)(tmem_slot + 1);

  const TcArgs& a = p.t;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_b) : "memory");
    for (int s = 0; s < ST; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; i++) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // same warp in both CTAs: the pair's accumulator columns
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrival
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel's tail; nothing global is touched before it has completed
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer (both CTAs)
      const uint64_t pol = policy_evict_last();   // weight tiles are re-read by the other m tiles
      const uint32_t full0 = map_to_rank(su32(full), 0);
      int it = 0;
      SegIter si(p, pair, n_pairs);
      Seg sg;
      while (si.next(sg)) {
        const int m_tile = sg.tile % p.m_tiles, n_tile = sg.tile / p.m_tiles;
        const int arow = m_tile * 256 + (int)rank * 128;
        int brow;
        if (a.epi == TC_SWIGLU) brow = (rank == 0 ? 0 : a.F) + n_tile * (BN / 2);
        else brow = n_tile * BN + (int)rank * (BN / 2);
        for (int kb = sg.k0; kb < sg.k1; kb++, it++) {
          const int s = it % ST;
          mbar_wait(&empty[s], ((it / ST) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * (kA + kB));
          const uint32_t fb = full0 + (uint32_t)s * 8u;
          tma_load_2d_pair(sa + s * kA, &map_a, fb, kb * BK, arow, pol);
#pragma unroll
          for (int j = 0; j < BN / 128; j++)
            tma_load_2d_pair(sb + s * kB + j * kBoxB, &map_b, fb, kb * BK, brow + 64 * j, pol);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---- MMA issuer (leader only)
      int it = 0, lt = 0;
      SegIter si(p, pair, n_pairs);
      Seg sg;
      for (; si.next(sg); lt++) {
        const int acc = lt & 1;
        mbar_wait_cluster(&tempty[acc], ((lt >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dst = tmem + (uint32_t)(acc * BN);
        for (int kb = sg.k0; kb < sg.k1; kb++, it++) {
          const int s = it % ST;
          mbar_wait(&full[s], (it / ST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = smem_desc(sa + s * kA);
          const uint64_t db = smem_desc(sb + s * kB);
#pragma unroll
          for (int k = 0; k < BK / 16; k++) {
            const uint64_t off = (uint64_t)((k * 32) >> 4);
            const uint32_t accum = (kb > sg.k0 || k > 0) ? 1u : 0u;
            asm volatile(
                "{ .reg .pred p; setp.ne.b32 p, %4, 0;"
                " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p; }"
                ::"r"(dst), "l"(da + off), "l"(db + off), "r"(kIdesc2), "r"(accum));
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
              ::"r"(su32(&empty[s])), "h"((uint16_t)3) : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
            ::"r"(su32(&tfull[acc])), "h"((uint16_t)3) : "memory");
      }
    }
  } else {
    // ---- epilogue warps 2..5 (both CTAs): TMEM lanes 32*(warp%4) .. +31 = tile rows
    const int lane_base = 32 * (warp & 3);
    const int r = lane_base + lane;            // this thread's row of the CTA's 128
    const uint32_t tempty0 = map_to_rank(su32(tempty), 0);
    int lt = 0;
    SegIter si(p, pair, n_pairs);
    Seg sg;
    for (; si.next(sg); lt++) {
      const int m_tile = sg.tile % p.m_tiles, n_tile = sg.tile / p.m_tiles;
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int row = m_tile * 256 + (int)rank * 128 + r;
      const uint32_t tacc = tmem + ((uint32_t)lane_base << 16) + (uint32_t)(acc * BN);
      auto release_acc = [&]() {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 2 && lane == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];"
                       ::"r"(tempty0 + (uint32_t)acc * 8u) : "memory");
      };
      if (p.split_out) {  // split-K unit: raw fp32 tile -> split_out[split] (logical columns)
        float* dst = p.split_out + ((size_t)sg.split * a.M + row) * a.N;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          float v[32];
          tmem_ld32(tacc + c, v);  // warp-collective: every lane, rows past M discard
          if (row >= a.M) continue;
          const int col = a.epi == TC_SWIGLU ? (c < BN / 2 ? n_tile * (BN / 2) + c : a.F + n_tile * (BN / 2) + c - BN / 2)
                                             : n_tile * BN + c;
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            __stcg(reinterpret_cast<float4*>(dst + col + i), make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        }
        release_acc();
        continue;
      }
      if (sg.k0 == 0 && sg.k1 == p.kblocks) {  // whole tile: fused epilogue straight from TMEM
        pair_epilogue_row<BN>(a, row, n_tile, [&](int c, float(&v)[32]) { tmem_ld32(tacc + c, v); });
        release_acc();
        continue;
      }
      // partial segment: accumulator -> this pair's scratch slot (coalesced float4
      // columns); slot 0 = the pair's first stream-K segment, 1 = its last
      const int slot = (sk_start(p, pair, n_pairs) / p.kblocks == sg.tile - p.dp) ? 0 : 1;
      float4* dst = reinterpret_cast<float4*>(p.scratch + ((size_t)(pair * 2 + slot) * 2 + rank) * kPart);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        float v[32];
        tmem_ld32(tacc + c, v);
#pragma unroll
        for (int j = 0; j < 8; j++)
          __stcg(dst + (size_t)(c / 4 + j) * BM + r, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
      }
      __threadfence();
      release_acc();
      // the tile's segments: pairs q_first .. q_last of the stream-K range
      const long long x0 = (long long)(sg.tile - p.dp) * p.kblocks;
      const int q_first = sk_owner(p, x0, n_pairs), q_last = sk_owner(p, x0 + p.kblocks - 1, n_pairs);
      const int nseg = q_last - q_first + 1;
      int* cnt = p.counters + (size_t)(sg.tile - p.dp) * 2 + rank;
      if (warp == 2 && lane == 0) {
        const int prev = atomicAdd(cnt, 1);
        const bool last = prev == nseg - 1;
        if (last) *cnt = 0;  // ready for the next launch
        *last_flag = last;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (!*last_flag) continue;
      __threadfence();
      // last arrival: sum the segments in k order (deterministic) and run the epilogue
      pair_epilogue_row<BN>(a, row, n_tile, [&](int c, float(&v)[32]) {
#pragma unroll
        for (int j = 0; j < 32; j++) v[j] = 0.0f;
        for (int q = q_first; q <= q_last; q++) {
          const long long qs = sk_start(p, q, n_pairs);
          const int qslot = (qs / p.kblocks == sg.tile - p.dp) ? 0 : 1;  // q's first segment, or its last
          const float4* src = reinterpret_cast<const float4*>(p.scratch + ((size_t)(q * 2 + qslot) * 2 + rank) * kPart);
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const float4 w = __ldcg(src + (size_t)(c / 4 + j) * BM + r);
            v[4 * j] += w.x; v[4 * j + 1] += w.y; v[4 * j + 2] += w.z; v[4 * j + 3] += w.w;
          }
        }
      });
      asm volatile("bar.sync 1, 128;" ::: "memory");  // last_flag reused by the next segment
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // the peer's TMEM / shared memory is in use until the pair is done
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
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
// SN = batch columns per MMA (16 / 32 / 64 / 128 / 256: the row count rounded
// up); the 16-row activation boxes of the lane's tensor maps are loaded SN / 16
// at a time into one K-major [SN x 64] operand tile.  The epilogue drains the
// accumulator 16 columns at a time through a [128 x 16] shared tile, so the
// shared memory left for the TMA ring does not shrink with SN.
constexpr int kSkA = BM * BK * 2;             // 16 KB weights per stage
constexpr int kSkBox = 16;                    // rows per activation TMA box
constexpr int kSkChunk = 16;                  // accumulator columns per epilogue chunk
template <int SN>
__host__ __device__ constexpr int sk_b_bytes() { return SN * BK * 2; }
template <int SN>
__host__ __device__ constexpr int sk_acc() { return SN <= 128 ? 4 : 2; }   // TMEM ring depth (<= 512 columns)
template <int SN, int STAGES>
constexpr int sk_smem() {
  return STAGES * (kSkA + sk_b_bytes<SN>()) + BM * (kSkChunk + 1) * 4 + 1024 /* align */ + 1024 /* barriers, red */;
}
template <int SN>
constexpr int sk_stages() { return SN <= 32 ? 10 : SN == 64 ? 8 : SN == 128 ? 6 : 4; }  // ~200 KB ring

struct SkArgs {
  int N, K, B, b0;        // weight rows, reduction, batch rows of this launch, first batch row
  int tiles, splits, kb_per_split, units;
  int epi;
  float* partial;         // [units][128][SN]
  int* counters;          // [tiles]
  // epilogue operands (see TcArgs); batch row b of this launch is row b0 + b
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
  unsigned long long* part_keys;  // ARGMAX: [rows][tiles]
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&raw)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(raw[0]), "=r"(raw[1]), "=r"(raw[2]), "=r"(raw[3]), "=r"(raw[4]), "=r"(raw[5]), "=r"(raw[6]),
        "=r"(raw[7]), "=r"(raw[8]), "=r"(raw[9]), "=r"(raw[10]), "=r"(raw[11]), "=r"(raw[12]), "=r"(raw[13]),
        "=r"(raw[14]), "=r"(raw[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Fused epilogue of one 16-column chunk (batch rows c0 .. c0 + nb - 1 of the
// launch) of a reduced [128 x 16] tile `ct` (row stride 17).  Called by the
// 128 epilogue threads; r = this thread's weight row of the tile.
__device__ __forceinline__ void sk_epilogue_chunk(const SkArgs& a, const float* ct, unsigned long long* red,
                                                  int tl, int c0, int nb, int r, int warp, int lane) {
  const int et = r;
  const int n0 = tl * BM;
  const bool swiglu = a.epi == TC_SWIGLU;
  const int nrow = swiglu ? (r < 64 ? tl * 64 + r : a.F + tl * 64 + r - 64) : n0 + r;
  const bool row_ok = nrow < a.N;
  const int g0 = a.b0 + c0;  // global batch row of column 0 of the chunk
  if (a.epi == TC_RESID) {
    if (row_ok)
      for (int j = 0; j < nb; j++) a.y[(size_t)(g0 + j) * a.ldy + nrow] += ct[r * (kSkChunk + 1) + j];
  } else if (a.epi == TC_SWIGLU) {
    if (et < 64 && tl * 64 + et < a.F)
      for (int j = 0; j < nb; j++)
        a.act[(size_t)(g0 + j) * a.F + tl * 64 + et] =
            __float2bfloat16_rn(silu_mul(ct[et * (kSkChunk + 1) + j], ct[(et + 64) * (kSkChunk + 1) + j]));
  } else if (a.epi == TC_QKV) {
    if (et < 64) {
      const int sec = n0 / a.d, h = (n0 % a.d) / a.hd, half = a.hd >> 1;
      for (int j = 0; j < nb; j++) {
        const int b = g0 + j;
        const RowMeta m = a.rows[b];
        float x1 = ct[et * (kSkChunk + 1) + j], x2 = ct[(et + half) * (kSkChunk + 1) + j];
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
    for (int j = 0; j < nb; j++) {
      const float v = ct[r * (kSkChunk + 1) + j];
      unsigned long long k = (row_ok && nrow < a.n_text) ? argmax_key(v, nrow) : 0ull;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, off));
      if (lane == 0) red[j * 4 + (warp & 3)] = k;
      if (row_ok && a.logits) {
        const RowMeta m = a.rows[a.head_rows[g0 + j]];
        if (m.logit_row >= 0) a.logits[(size_t)m.logit_row * a.V + nrow] = v;
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (et < nb) {
      unsigned long long k = 0ull;
      for (int w = 0; w < 4; w++) k = max(k, red[et * 4 + w]);
      a.part_keys[(size_t)(g0 + et) * a.tiles + tl] = k;
    }
  } else {  // TC_STORE: y[b][n]
    if (row_ok)
      for (int j = 0; j < nb; j++) a.y[(size_t)(g0 + j) * a.ldy + nrow] = ct[r * (kSkChunk + 1) + j];
  }
}

template <int SN, int kSkStages>
__global__ void __launch_bounds__(kThreads, 1)
skinny_tc_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                 const SkArgs a) {
  constexpr int kSkB = sk_b_bytes<SN>();
  constexpr int kSkAcc = sk_acc<SN>();
  constexpr uint32_t kSkIdesc = idesc_bf16(BM, SN);
  constexpr int kTmemCols = kSkAcc * SN;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = smem;
  unsigned char* sb = smem + kSkStages * kSkA;
  float* ct = (float*)(sb + kSkStages * kSkB);             // [128][16 + 1] chunk tile
  uint64_t* full = (uint64_t*)(ct + BM * (kSkChunk + 1));
  uint64_t* empty = full + kSkStages;
  uint64_t* acc_full = empty + kSkStages;                  // [kSkAcc]
  uint64_t* acc_empty = acc_full + kSkAcc;                 // [kSkAcc]
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + kSkAcc);
  int* last_flag = (int*)(tmem_slot + 1);
  unsigned long long* red = (unsigned long long*)(tmem_slot + 4);  // [16][4], 8-byte aligned

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
  if (warp == 1) {  // kSkAcc SN-column fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "n"(kTmemCols));
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
#pragma unroll
          for (int j = 0; j < SN / kSkBox; j++)
            tma_load_2d(sb + s * kSkB + j * kSkBox * BK * 2, &map_x, &full[s], kb * BK, a.b0 + j * kSkBox);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer: accumulator (local unit index) % kSkAcc
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
    const int n_chunks = (a.B + kSkChunk - 1) / kSkChunk;   // live 16-column chunks
    pdl_wait();  // epilogue writes / reads outputs of earlier kernels
    int lu = 0;
    for (int u = blockIdx.x; u < a.units; u += gridDim.x, lu++) {
      int tl, sp, kb0, kb1;
      unit_of(a, u, kb_total, &tl, &sp, &kb0, &kb1);
      const int acc = lu % kSkAcc;
      mbar_wait(&acc_full[acc], (lu / kSkAcc) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tacc = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(acc * SN);
      if (a.splits == 1) {
        // chunk by chunk: TMEM -> shared chunk tile -> fused epilogue
        for (int c = 0; c < n_chunks; c++) {
          uint32_t raw[16];
          tmem_ld16(tacc + c * kSkChunk, raw);
#pragma unroll
          for (int j = 0; j < 16; j++) ct[r * (kSkChunk + 1) + j] = __uint_as_float(raw[j]);
          asm volatile("bar.sync 1, 128;" ::: "memory");
          sk_epilogue_chunk(a, ct, red, tl, c * kSkChunk, min(kSkChunk, a.B - c * kSkChunk), r, warp, lane);
          asm volatile("bar.sync 1, 128;" ::: "memory");  // ct / red reused by the next chunk
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acc_empty[acc])) : "memory");
        continue;
      }
      // split-K: drain into this unit's partial [unit][128 rows][SN] fp32
      for (int c = 0; c < n_chunks; c++) {
        uint32_t raw[16];
        tmem_ld16(tacc + c * kSkChunk, raw);
        float4* dst = reinterpret_cast<float4*>(a.partial + ((size_t)u * BM + r) * SN + c * kSkChunk);
#pragma unroll
        for (int i = 0; i < 4; i++)
          __stcg(dst + i, make_float4(__uint_as_float(raw[4 * i]), __uint_as_float(raw[4 * i + 1]),
                                      __uint_as_float(raw[4 * i + 2]), __uint_as_float(raw[4 * i + 3])));
      }
      // accumulator drained: hand it back to the MMA warp
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      // one gpu-scope fence per thread publishes its partial rows before the
      // CTA's arrival on the tile counter (split-K serial pattern)
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acc_empty[acc])) : "memory");
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
      // fixed-order reduction over the tile's splits (units tl*splits .. +splits-1), chunk by chunk
      for (int c = 0; c < n_chunks; c++) {
        float4 acc4[4];
#pragma unroll
        for (int i = 0; i < 4; i++) acc4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < a.splits; q++) {
          const float4* src = reinterpret_cast<const float4*>(
              a.partial + ((size_t)(tl * a.splits + q) * BM + r) * SN + c * kSkChunk);
          float4 v[4];
#pragma unroll
          for (int i = 0; i < 4; i++) v[i] = __ldcg(src + i);
#pragma unroll
          for (int i = 0; i < 4; i++) {
            acc4[i].x += v[i].x; acc4[i].y += v[i].y; acc4[i].z += v[i].z; acc4[i].w += v[i].w;
          }
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
          ct[r * (kSkChunk + 1) + 4 * i] = acc4[i].x;
          ct[r * (kSkChunk + 1) + 4 * i + 1] = acc4[i].y;
          ct[r * (kSkChunk + 1) + 4 * i + 2] = acc4[i].z;
          ct[r * (kSkChunk + 1) + 4 * i + 3] = acc4[i].w;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        sk_epilogue_chunk(a, ct, red, tl, c * kSkChunk, min(kSkChunk, a.B - c * kSkChunk), r, warp, lane);
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

// Split-K reduction with the fused epilogue (the pair GEMM's split mode):
// RESID split-K reduce fused with the RMSNorm that follows it: one block per
// row; x += sum of the splits (split order, as splitk_reduce_kernel), then
// out = bf16(x * rsqrt(mean x^2 + eps) * w) with rmsnorm_bf16_kernel's thread
// mapping and summation order, so the result is bit-identical to the two
// kernels run back to back.
__global__ void __launch_bounds__(256) splitk_resid_norm_kernel(const float* __restrict__ part, int S, TcArgs a,
                                                                const float* __restrict__ w,
                                                                __nv_bfloat16* __restrict__ out, float eps) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8];
  const int row = blockIdx.x, d = a.N;
  const size_t plane = (size_t)a.M * a.N;
  float* xr = a.y + (size_t)row * a.ldy;
  const float* pr = part + (size_t)row * a.N;
  float ss = 0.0f;
  // this thread's 16-byte groups: chunk c (k = 8 tid + 2048 c), halves h;
  // every load of a split is issued before any add (latency, not bandwidth,
  // bounds a 448-row reduce)
  constexpr int kMaxChunks = 2;  // d <= 4096 in registers; longer rows loop
  for (int kc = 8 * threadIdx.x; kc < d; kc += 8 * blockDim.x * kMaxChunks) {
    float4 v[2 * kMaxChunks];
    bool on[kMaxChunks];
#pragma unroll
    for (int c = 0; c < kMaxChunks; c++) on[c] = kc + c * 8 * blockDim.x < d;
#pragma unroll
    for (int c = 0; c < kMaxChunks; c++)
#pragma unroll
      for (int h = 0; h < 2; h++)
        if (on[c]) v[2 * c + h] = __ldcg(reinterpret_cast<const float4*>(pr + kc + c * 8 * blockDim.x + 4 * h));
    for (int sp = 1; sp < S; sp++) {
      float4 u[2 * kMaxChunks];
#pragma unroll
      for (int c = 0; c < kMaxChunks; c++)
#pragma unroll
        for (int h = 0; h < 2; h++)
          if (on[c]) u[2 * c + h] = __ldcg(reinterpret_cast<const float4*>(pr + sp * plane + kc + c * 8 * blockDim.x + 4 * h));
#pragma unroll
      for (int i = 0; i < 2 * kMaxChunks; i++)
        if (on[i / 2]) { v[i].x += u[i].x; v[i].y += u[i].y; v[i].z += u[i].z; v[i].w += u[i].w; }
    }
#pragma unroll
    for (int c = 0; c < kMaxChunks; c++) {
      if (!on[c]) continue;
      float* xk = xr + kc + c * 8 * blockDim.x;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const float4 o = *reinterpret_cast<const float4*>(xk + 4 * h);
        float4& acc = v[2 * c + h];
        acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
        *reinterpret_cast<float4*>(xk + 4 * h) = acc;
      }
      ss = fmaf(v[2 * c].x, v[2 * c].x, fmaf(v[2 * c].y, v[2 * c].y, fmaf(v[2 * c].z, v[2 * c].z,
               fmaf(v[2 * c].w, v[2 * c].w, ss))));
      ss = fmaf(v[2 * c + 1].x, v[2 * c + 1].x, fmaf(v[2 * c + 1].y, v[2 * c + 1].y,
               fmaf(v[2 * c + 1].z, v[2 * c + 1].z, fmaf(v[2 * c + 1].w, v[2 * c + 1].w, ss))));
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; i++) tot += red[i];
  const float r = rsqrtf(tot / (float)d + eps);
  __nv_bfloat16* o = out + (size_t)row * d;
  for (int k = 8 * threadIdx.x; k < d; k += 8 * blockDim.x) {  // this thread's own x writes
    const float4 x0 = *reinterpret_cast<const float4*>(xr + k);
    const float4 x1 = *reinterpret_cast<const float4*>(xr + k + 4);
    const float4 wa = *reinterpret_cast<const float4*>(w + k);
    const float4 wb = *reinterpret_cast<const float4*>(w + k + 4);
    __nv_bfloat162 y[4];
    y[0] = __floats2bfloat162_rn(x0.x * r * wa.x, x0.y * r * wa.y);
    y[1] = __floats2bfloat162_rn(x0.z * r * wa.z, x0.w * r * wa.w);
    y[2] = __floats2bfloat162_rn(x1.x * r * wb.x, x1.y * r * wb.y);
    y[3] = __floats2bfloat162_rn(x1.z * r * wb.z, x1.w * r * wb.w);
    *reinterpret_cast<uint4*>(o + k) = *reinterpret_cast<const uint4*>(y);
  }
}

// sums split_out[0 .. S-1][row][col] in split order (deterministic) and
// applies the GEMM's epilogue -- STORE / RESID (float4 per thread), SwiGLU
// (gate col j, up col F + j), QKV (RoPE pairs c, c + 64 of a head; q rows or
// the paged K/V append).
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ part, int S, TcArgs a) {
  pdl_trigger();
  pdl_wait();
  const size_t plane = (size_t)a.M * a.N;
  if (a.epi == TC_STORE || a.epi == TC_RESID) {
    const size_t n4 = plane / 4;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      float4 acc = __ldcg(reinterpret_cast<const float4*>(part) + i);
      for (int sp = 1; sp < S; sp++) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(part + sp * plane) + i);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      const size_t row = i * 4 / a.N, col = i * 4 % a.N;
      float4* dst = reinterpret_cast<float4*>(a.y + row * a.ldy + col);
      if (a.epi == TC_RESID) {
        const float4 o = *dst;
        acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
      }
      *dst = acc;
    }
  } else if (a.epi == TC_SWIGLU) {
    const size_t n4 = (size_t)a.M * a.F / 4;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
      const size_t row = i * 4 / a.F, j = i * 4 % a.F;
      const float* g0 = part + row * a.N + j;
      float4 g = __ldcg(reinterpret_cast<const float4*>(g0)), u = __ldcg(reinterpret_cast<const float4*>(g0 + a.F));
      for (int sp = 1; sp < S; sp++) {
        const float4 vg = __ldcg(reinterpret_cast<const float4*>(g0 + sp * plane));
        const float4 vu = __ldcg(reinterpret_cast<const float4*>(g0 + sp * plane + a.F));
        g.x += vg.x; g.y += vg.y; g.z += vg.z; g.w += vg.w;
        u.x += vu.x; u.y += vu.y; u.z += vu.z; u.w += vu.w;
      }
      __nv_bfloat162 p0, p1;
      p0.x = __float2bfloat16_rn(silu_mul(g.x, u.x)); p0.y = __float2bfloat16_rn(silu_mul(g.y, u.y));
      p1.x = __float2bfloat16_rn(silu_mul(g.z, u.z)); p1.y = __float2bfloat16_rn(silu_mul(g.w, u.w));
      __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(a.act + row * a.F + j);
      dst[0] = p0;
      dst[1] = p1;
    }
  } else {  // TC_QKV: thread = (row, head section, 4 rotary pairs)
    const int heads = a.N / 128;
    const size_t n = (size_t)a.M * heads * 16;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const int c = (int)(i % 16) * 4;
      const size_t rh = i / 16;
      const int hs = (int)(rh % heads);
      const size_t row = rh / heads;
      const int nh = hs * 128, sec = nh / a.d, h = (nh % a.d) / 128;
      const float* p1 = part + row * a.N + nh + c;
      float4 x1 = __ldcg(reinterpret_cast<const float4*>(p1)), x2 = __ldcg(reinterpret_cast<const float4*>(p1 + 64));
      for (int sp = 1; sp < S; sp++) {
        const float4 v1 = __ldcg(reinterpret_cast<const float4*>(p1 + sp * plane));
        const float4 v2 = __ldcg(reinterpret_cast<const float4*>(p1 + sp * plane + 64));
        x1.x += v1.x; x1.y += v1.y; x1.z += v1.z; x1.w += v1.w;
        x2.x += v2.x; x2.y += v2.y; x2.z += v2.z; x2.w += v2.w;
      }
      float a1[4] = {x1.x, x1.y, x1.z, x1.w}, a2[4] = {x2.x, x2.y, x2.z, x2.w};
      const RowMeta m = a.rows[row];
      if (sec < 2) {
        const float* cs = a.rope + (size_t)m.pos * 128;
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const float co = cs[c + e], sn = cs[64 + c + e];
          const float r1 = __fmaf_rn(a1[e], co, -__fmul_rn(a2[e], sn));
          const float r2 = __fmaf_rn(a2[e], co, __fmul_rn(a1[e], sn));
          a1[e] = r1;
          a2[e] = r2;
        }
      }
      if (sec == 0) {
        float* qr = a.q + row * a.d + h * 128;
        *reinterpret_cast<float4*>(qr + c) = make_float4(a1[0], a1[1], a1[2], a1[3]);
        *reinterpret_cast<float4*>(qr + 64 + c) = make_float4(a2[0], a2[1], a2[2], a2[3]);
      } else {
        __nv_bfloat16* kv = a.kv_pool + (size_t)m.kv_page * a.page_elems + a.layer_off +
                            ((size_t)((sec - 1) * a.H + h) * FE_PAGE + m.kv_slot) * 128;
        __nv_bfloat162 q0, q1, q2, q3;
        q0.x = __float2bfloat16_rn(a1[0]); q0.y = __float2bfloat16_rn(a1[1]);
        q1.x = __float2bfloat16_rn(a1[2]); q1.y = __float2bfloat16_rn(a1[3]);
        q2.x = __float2bfloat16_rn(a2[0]); q2.y = __float2bfloat16_rn(a2[1]);
        q3.x = __float2bfloat16_rn(a2[2]); q3.y = __float2bfloat16_rn(a2[3]);
        reinterpret_cast<__nv_bfloat162*>(kv + c)[0] = q0;
        reinterpret_cast<__nv_bfloat162*>(kv + c)[1] = q1;
        reinterpret_cast<__nv_bfloat162*>(kv + 64 + c)[0] = q2;
        reinterpret_cast<__nv_bfloat162*>(kv + 64 + c)[1] = q3;
      }
    }
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

int skinny_max_rows() { return 1 << 20; }  // wider batches run in 256-row slices
int skinny_cols(int rows) {
  return rows <= 16 ? 16 : rows <= 32 ? 32 : rows <= 64 ? 64 : rows <= 128 ? 128 : 256;
}

int skinny_tiles(int epi, int N, int F) { return epi == TC_SWIGLU ? F / (BM / 2) : (N + BM - 1) / BM; }

namespace {
int g_n_sm = 0;

template <int SN, int ST>
void sk_configure() {
  cudaFuncSetAttribute(skinny_tc_kernel<SN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, sk_smem<SN, ST>());
  cudaFuncSetAttribute(skinny_tc_kernel<SN, ST>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

template <int SN, int ST>
void sk_launch(const CUtensorMap& wm, const CUtensorMap& xm, const SkArgs& a, cudaStream_t s) {
  const int grid = std::min(a.units, g_n_sm);
  launch_k(skinny_tc_kernel<SN, ST>, dim3(grid), dim3(kThreads), (size_t)sk_smem<SN, ST>(), s, wm, xm, a);
}

// K split balancing the units over the persistent CTAs, keeping the split
// partial traffic (units * 128 * sn * 8 bytes) under ~6 % of the weights: a
// split unit costs a partial store, a gpu-scope fence, a tile-counter atomic
// and its share of the owner's ordered reduction (measured ~3 us per unit,
// tools/bench_skinny.py), so only weight-light splits pay off.
int pick_kb_per_split(int tiles, int kb_total, int sn, double weight_bytes) {
  int best_kb = kb_total;
  double best_eff = -1.0;
  for (int kb_per = kb_total; kb_per >= 4; kb_per--) {
    const int splits = (kb_total + kb_per - 1) / kb_per;
    const int units = tiles * splits;
    if (splits > 1 && (units * (double)BM * sn * 8.0 > 0.06 * weight_bytes || splits > 8)) break;
    const int rounds = (units + g_n_sm - 1) / g_n_sm;
    // balance, with a small per-unit epilogue cost
    const double eff = (double)tiles * kb_total / ((double)g_n_sm * rounds * (kb_per + 1.0));
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best_kb = kb_per;
    }
  }
  return best_kb;
}
}  // namespace

size_t skinny_partial_floats(int N, int K) {
  // the largest plan pick_kb_per_split can return (any row count), or a
  // forced split of up to 16 (option sk_splits) at 16 columns
  const size_t tiles = (size_t)(N + BM - 1) / BM;
  return std::max((size_t)(0.06 * (double)N * K * 2.0 / 8.0) + (size_t)BM * 256 * 8, tiles * 16 * BM * 16);
}

void launch_skinny_tc(const TmaMap& w_map, const TmaMap& x_map, const SkLaunch& l, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    // 16 columns: 10 stages, or 5 so two CTAs of consecutive PDL-chained
    // launches fit on one SM (maximum shared-memory carveout)
    sk_configure<16, 10>();
    sk_configure<16, 5>();
    sk_configure<32, sk_stages<32>()>();
    sk_configure<64, sk_stages<64>()>();
    sk_configure<128, sk_stages<128>()>();
    sk_configure<256, sk_stages<256>()>();
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_n_sm, cudaDevAttrMultiProcessorCount, dev);
    configured = true;
  }
  const CUtensorMap& wm = *reinterpret_cast<const CUtensorMap*>(w_map.bytes);
  const CUtensorMap& xm = *reinterpret_cast<const CUtensorMap*>(x_map.bytes);
  const int tiles = skinny_tiles(l.epi, l.N, l.F);
  const int kb_total = (l.K + BK - 1) / BK;
  // > 256 rows: 256-row slices, each streaming the weights once more
  for (int b0 = 0; b0 < l.B; b0 += 256) {
    const int rows = std::min(256, l.B - b0);
    const int sn = skinny_cols(rows);
    const int forced = sn == 16 ? g_sk_splits : std::min(g_sk_splits, 2);   // within the scratch bound
    const int kb_per = forced > 0 ? (kb_total + forced - 1) / forced
                                       : pick_kb_per_split(tiles, kb_total, sn, (double)l.N * l.K * 2.0);
    SkArgs a{};
    a.N = l.N; a.K = l.K; a.B = rows; a.b0 = b0; a.epi = l.epi;
    a.kb_per_split = kb_per;
    a.splits = (kb_total + kb_per - 1) / kb_per;
    a.tiles = tiles;
    a.units = tiles * a.splits;
    a.partial = l.partial; a.counters = l.counters;
    a.y = l.y; a.ldy = l.ldy; a.act = l.act; a.F = l.F; a.q = l.q; a.kv_pool = l.kv_pool;
    a.page_elems = l.page_elems; a.layer_off = l.layer_off; a.rope = l.rope; a.rows = l.rows;
    a.head_rows = l.head_rows; a.H = l.H; a.hd = l.hd; a.d = l.d; a.part_keys = l.part_keys;
    a.logits = l.logits; a.V = l.V; a.n_text = l.n_text;
    switch (sn) {
      case 16:
        if (g_sk_stages <= 5) sk_launch<16, 5>(wm, xm, a, s);
        else sk_launch<16, 10>(wm, xm, a, s);
        break;
      case 32: sk_launch<32, sk_stages<32>()>(wm, xm, a, s); break;
      case 64: sk_launch<64, sk_stages<64>()>(wm, xm, a, s); break;
      case 128: sk_launch<128, sk_stages<128>()>(wm, xm, a, s); break;
      default: sk_launch<256, sk_stages<256>()>(wm, xm, a, s); break;
    }
  }
}

namespace {
TcArgs tc_args(const TcLaunch& l) {
  TcArgs a{};
  a.M = l.M; a.N = l.N; a.K = l.K; a.epi = l.epi;
  a.y = l.y; a.ldy = l.ldy; a.act = l.act; a.F = l.F;
  a.q = l.q; a.kv_pool = l.kv_pool; a.page_elems = l.page_elems; a.layer_off = l.layer_off;
  a.rope = l.rope; a.rows = l.rows; a.H = l.H; a.hd = l.hd; a.d = l.d;
  return a;
}
}  // namespace

void launch_gemm_tc_v1(const TmaMap& a_map, const TmaMap& b_map, const TcLaunch& l, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  const TcArgs a = tc_args(l);
  const int n_tiles = l.epi == TC_SWIGLU ? (l.F / (BN / 2)) : (l.N / BN);
  dim3 grid((l.M + BM - 1) / BM, n_tiles);
  gemm_tc_kernel<<<grid, kThreads, kSmem, s>>>(*reinterpret_cast<const CUtensorMap*>(a_map.bytes),
                                               *reinterpret_cast<const CUtensorMap*>(b_map.bytes), a);
}

int g_pair_bn = 0;  // engine option "tc_bn": force the pair tile width (0: 256 where it divides)
int g_pair_split = 1;  // engine option "tc_split": split-K for decode-width batches
int g_pair_maxp = 0;  // engine option "tc_maxp": cap on the pairs of a launch (measurement only)
int g_pair_sk = 0;  // engine option "tc_sk": stream-K the last waves (measured slower: the 256 x 256 fp32
                    // partials cost more than the wave tail they remove, profiles/r2_gemm_pair_sk.txt)

size_t pair_sk_scratch_floats() { return (size_t)kPairMaxPairs * 2 * 2 * BM * 256; }
int pair_sk_counters() { return 4 * kPairMaxPairs; }

int pair_tile_n(int M, int N, int epi, int F) {
  (void)M;
  if (g_pair_bn == 128 || g_pair_bn == 256) return g_pair_bn;
  // 256 wherever it divides: measured faster than 128 at every 7B shape and
  // row count (tools/bench_gemm.py, profiles/r2_gemm_pair.json), including
  // those where 128 needs fewer waves -- a 128-wide pair tile streams 1.5x
  // the operand bytes per flop and is L2-bandwidth bound
  const int cols = epi == TC_SWIGLU ? 2 * F : N;
  return cols % 256 == 0 ? 256 : 128;
}

bool launch_gemm_tc(const TmaMap& a_map, const TmaMap& b_map64, const TcLaunch& l, cudaStream_t s) {
  static bool configured = false;
  static int n_sm = 0;
  if (!configured) {
    cudaFuncSetAttribute(gemm_pair_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem<128>());
    cudaFuncSetAttribute(gemm_pair_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem<256>());
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    configured = true;
  }
  if (l.epi == TC_QKV && l.hd != 128) throw std::runtime_error("gemm_tc: QKV epilogue needs head_dim 128");
  PairArgs p{};
  p.t = tc_args(l);
  const int bn = pair_tile_n(l.M, l.N, l.epi, l.F);
  const int cols = l.epi == TC_SWIGLU ? 2 * l.F : l.N;
  if (cols % bn || l.K % BK) throw std::runtime_error("gemm_tc: N % tile and K % 64 must be 0");
  p.m_tiles = (l.M + 255) / 256;
  p.n_tiles = cols / bn;
  p.kblocks = l.K / BK;
  const int tiles = p.m_tiles * p.n_tiles;
  const int P = std::min(tiles * p.kblocks, std::min(g_pair_maxp > 0 ? g_pair_maxp : n_sm / 2, kPairMaxPairs));
  // DP for all but the last one-to-two waves, which are stream-K'd (no wave tail)
  // split-K when the tiles do not fill the pairs (decode-width batches, O and
  // down projections): the split count minimising waves x k-blocks per unit
  // + a per-split cost for the partial traffic (~4 k-block wave-times per
  // 168 x 4096 fp32 plane; measured, profiles/r2_gemm_pair_split.txt)
  int S = 1;
  if (g_pair_split > 1 && l.split_scratch && (size_t)g_pair_split * l.M * cols <= l.split_floats &&
      p.kblocks / g_pair_split >= 4) {
    S = g_pair_split;  // forced (option tc_split = S > 1; measurement only)
  } else if (g_pair_split && l.split_scratch && tiles < P) {
    double best = 1e30;
    const double plane = (double)l.M * cols / (168.0 * 4096.0);
    for (int sp = 1; sp <= 8; sp++) {
      if ((size_t)sp * l.M * cols > l.split_floats || (sp > 1 && p.kblocks / sp < 4)) break;
      const int units = tiles * sp;
      const double t = (double)((units + P - 1) / P) * ((p.kblocks + sp - 1) / sp) + (sp > 1 ? 4.0 * sp * plane : 0.0);
      if (t < best - 1e-9) { best = t; S = sp; }
    }
  }
  p.tiles = tiles;
  p.splits = S;
  p.kbs = (p.kblocks + S - 1) / S;
  p.split_out = S > 1 ? l.split_scratch : nullptr;
  const int units = tiles * S;
  p.dp = (S > 1 || !g_pair_sk || !l.sk_scratch) ? units : (tiles >= 2 * P ? (tiles / P - 1) * P : 0);
  p.W = (long long)(tiles - std::min(p.dp, tiles)) * p.kblocks;
  p.scratch = l.sk_scratch;
  p.counters = l.sk_counters;
  const int grid = 2 * (p.dp == units ? std::min(units, P) : P);
  const CUtensorMap& am = *reinterpret_cast<const CUtensorMap*>(a_map.bytes);
  const CUtensorMap& bm = *reinterpret_cast<const CUtensorMap*>(b_map64.bytes);
  if (bn == 256) launch_k(gemm_pair_kernel<256>, dim3(grid), dim3(kPairThreads), (size_t)pair_smem<256>(), s, am, bm, p);
  else launch_k(gemm_pair_kernel<128>, dim3(grid), dim3(kPairThreads), (size_t)pair_smem<128>(), s, am, bm, p);
  if (S > 1 && l.epi == TC_RESID && l.norm_w && l.norm_out && l.N % 8 == 0 && l.ldy % 4 == 0) {
    launch_k(splitk_resid_norm_kernel, dim3(l.M), dim3(256), 0, s, (const float*)l.split_scratch, S, p.t, l.norm_w,
             l.norm_out, l.norm_eps);
    return true;
  }
  if (S > 1) {
    const size_t work = l.epi == TC_SWIGLU ? (size_t)l.M * l.F / 4 : l.epi == TC_QKV ? (size_t)l.M * (l.N / 128) * 16
                                                                                   : (size_t)l.M * l.N / 4;
    const int blocks = (int)std::min<size_t>((work + 255) / 256, (size_t)n_sm * 8);
    launch_k(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, s, (const float*)l.split_scratch, S, p.t);
  }
  return false;
}

}  // namespace fe
