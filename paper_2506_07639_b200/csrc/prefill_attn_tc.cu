// Causal prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA),
// bf16 path, head_dim 128 -- K10 of SURVEY §2.3.  Same work split as the
// mma.sync kernel (prefill_attn.cu: query tiles of one sequence's consecutive
// positions, paged K/V), with 128-row query tiles:
//
//   * Q tile [128 rows x 128 dims] staged once in shared memory (bf16, scaled
//     to the exp2 domain, 128-byte-swizzled K-major: the UMMA A layout).
//   * per KV page (64 keys): K and V [64 keys x 128 dims] land by TMA (two
//     64 x 64 swizzled boxes each) in a 4-stage ring over a 2-D tensor map of
//     the pool.
//   * S = Q K^T: tcgen05.mma M=128 N=64 (8 x K=16), fp32 into TMEM
//     (double-buffered: S of page j+1 is issued before the softmax of page j).
//   * softmax: thread = query row = TMEM lane; tcgen05.ld its 64 scores, causal
//     mask, online max / sum; P (bf16) -> shared memory in the UMMA K-major
//     layout (double-buffered).
//   * O += P V: tcgen05.mma M=128 N=128 (4 x K=16) with V as an MN-major B
//     operand straight from the TMA tile, accumulating in TMEM across pages.
//     The running max is only raised (and O rescaled through tcgen05.ld/st)
//     when a row's new scores exceed it by more than 2^8, so the usual page
//     needs no O traffic at all; exp2 of scores against the stale max stays
//     <= 256 and the final O / l is exact.
//   * one elected thread issues TMA and MMA; tcgen05.commit -> mbarriers.
#include "common.cuh"
#include "engine_internal.h"
#include "gemm_tc.h"
#include "tc_util.cuh"

#include <cuda.h>
#include <cuda_bf16.h>

namespace fe {
namespace {

using namespace tc;

constexpr int HD = 128;
constexpr int QR = 128;                       // query rows per CTA (UMMA M)
constexpr int kBox = 64 * 64 * 2;             // 8 KB: 64 rows x 64 dims
constexpr int kKV = 4 * kBox;                 // K lo, K hi, V lo, V hi of one page
constexpr int kQ = QR * HD * 2;               // 32 KB: Q tile (two 128 x 64 boxes)
constexpr int kP = QR * 64 * 2;               // 16 KB: P tile [128 x 64 keys]
constexpr int NKV = 4;                        // K/V pages in flight
constexpr int kSmem = NKV * kKV + kQ + 2 * kP + 1024 + 256;
constexpr float kRescale = 8.0f;              // log2 headroom before the running max is raised
constexpr int kTmemCols = 256;                // S0 [0,64) S1 [64,128) O [128,256)

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

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

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// MN-major (N contiguous) 128B-swizzled UMMA descriptor: 64-element rows of
// 128 B, K rows 128 B apart; the next 8 K rows at SBO, the next 64 N at LBO
__device__ __forceinline__ uint64_t smem_desc_mn(const void* p, uint32_t lbo_bytes) {
  const uint64_t addr = su32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;  // leading byte offset: next 64-wide N block
  d |= (uint64_t)(1024 >> 4) << 32;                  // stride byte offset: next 8 K rows
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                            // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0;"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
      ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

constexpr uint32_t kIdS = idesc_bf16(QR, 64);                       // S = Q K^T
constexpr uint32_t kIdPV = idesc_bf16(QR, HD) | (1u << 16);         // O += P V, V MN-major

__global__ void __launch_bounds__(128, 1)
prefill_attn_tc_kernel(const __grid_constant__ CUtensorMap pool_map, const PrefillTile* __restrict__ tiles,
                       const int32_t* __restrict__ ptab, const float* __restrict__ q, int L, int layer, int H, int d,
                       float scale_log2, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* skv = smem;                       // [NKV][K lo, K hi, V lo, V hi]
  unsigned char* sq = smem + NKV * kKV;            // Q: [dims 0-63 | dims 64-127] x 128 rows
  unsigned char* sp = sq + kQ;                     // P: [2][128 x 64]
  uint64_t* full = (uint64_t*)(sp + 2 * kP);       // [NKV] K/V landed
  uint64_t* s_done = full + NKV;                   // [2] S MMAs of a page complete
  uint64_t* pv_done = s_done + 2;                  // [2] P V MMAs complete (P buffer + K/V stage free)
  uint32_t* tmem_slot = (uint32_t*)(pv_done + 2);

  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int h = blockIdx.y;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&pool_map) : "memory");
    for (int i = 0; i < NKV; i++) mbar_init(&full[i], 1);
    for (int i = 0; i < 2; i++) {
      mbar_init(&s_done[i], 1);
      mbar_init(&pv_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_wait();  // q and the K/V of this forward's rows come from the QKV GEMM
  // heaviest tiles first: a tile's pages grow with its position, so the CTAs
  // that spill into a second wave are the short ones
  const PrefillTile tile = tiles[gridDim.x - 1 - blockIdx.x];
  const int32_t* pages = ptab + tile.pages;
  const int pos0 = tile.pos0, n_rows = tile.n;
  const int n_pages = (pos0 + n_rows - 1) / FE_PAGE + 1;

  auto issue_kv = [&](int j) {  // page j -> stage j % NKV (thread 0)
    const int st = j % NKV;
    const int rk = (((pages[j] * L + layer) * 2 + 0) * H + h) * 64;
    const int rv = rk + H * 64;
    unsigned char* b = skv + st * kKV;
    mbar_expect_tx(&full[st], kKV);
    tma_load_2d(b, &pool_map, &full[st], 0, rk);
    tma_load_2d(b + kBox, &pool_map, &full[st], 64, rk);
    tma_load_2d(b + 2 * kBox, &pool_map, &full[st], 0, rv);
    tma_load_2d(b + 3 * kBox, &pool_map, &full[st], 64, rv);
  };
  if (tid == 0)
    for (int j = 0; j < min(NKV, n_pages); j++) issue_kv(j);

  // Q row `tid` -> bf16 (exp2 domain), 128B-swizzled K-major
  const int r = tid;                       // query row of the tile = TMEM lane
  const int pos = pos0 + r;
  const bool live = r < n_rows;
  {
    const float* qr = q + (size_t)(tile.row0 + (live ? r : 0)) * d + h * HD;
#pragma unroll
    for (int c = 0; c < 16; c++) {  // 16-byte chunk c = dims 8c .. 8c + 7
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
      if (live) {
        a = *reinterpret_cast<const float4*>(qr + 8 * c);
        b = *reinterpret_cast<const float4*>(qr + 8 * c + 4);
      }
      const float s = scale_log2;
      const uint4 v = make_uint4(pack2(a.x * s, a.y * s), pack2(a.z * s, a.w * s), pack2(b.x * s, b.y * s),
                                 pack2(b.z * s, b.w * s));
      *reinterpret_cast<uint4*>(sq + (c >> 3) * (QR * 128) + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_lane = tmem + ((uint32_t)(32 * warp) << 16);
  const uint32_t t_o = 128;  // O accumulator columns

  auto issue_s = [&](int j) {  // S_j = Q K_j^T -> TMEM cols (j & 1) * 64 (thread 0)
    const int st = j & 1, kst = j % NKV;
    mbar_wait(&full[kst], (j / NKV) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned char* kb = skv + kst * kKV;
#pragma unroll
    for (int ks = 0; ks < 8; ks++) {
      const uint64_t off = (uint64_t)(((ks & 3) * 32) >> 4);
      mma_f16(tmem + (uint32_t)(st * 64), smem_desc(sq + (ks >> 2) * (QR * 128)) + off,
              smem_desc(kb + (ks >> 2) * kBox) + off, kIdS, ks > 0 ? 1u : 0u);
    }
    mma_commit(&s_done[st]);
  };
  if (tid == 0) issue_s(0);

  float m_used = -INFINITY, l = 0.0f;  // running (stale) max, sum -- this thread's row
  for (int j = 0; j < n_pages; j++) {
    const int st = j & 1;
    // S of the next page while this page's softmax runs (its K stage and S
    // buffer are free once the P V of page j - 1 completed)
    // (S buffer (j + 1) & 1 was read by every thread before the last
    // iteration's barrier; page j + 1's K/V stage was issued NKV - 1 pages ago)
    if (tid == 0 && j + 1 < n_pages) issue_s(j + 1);
    mbar_wait(&s_done[st], (j >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float s[64];
    {
      float a[32], b[32];
      tmem_ld32(t_lane + (uint32_t)(st * 64), a);
      tmem_ld32(t_lane + (uint32_t)(st * 64 + 32), b);
#pragma unroll
      for (int i = 0; i < 32; i++) { s[i] = a[i]; s[32 + i] = b[i]; }
    }
    const int kbase = j * FE_PAGE;
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < 64; i++) {
      s[i] = (live && kbase + i <= pos) ? s[i] : -INFINITY;
      mx = fmaxf(mx, s[i]);
    }
    // raise the running max only when the new scores would overflow the headroom
    const bool raise = mx > m_used + kRescale;
    if (__any_sync(0xffffffffu, raise && j > 0)) {
      // the P V of page j - 1 must have landed in O before O is rescaled
      mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float f = raise ? exp2f(m_used - mx) : 1.0f;  // m_used = -inf -> 0 (O is still 0)
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        float o[32];
        tmem_ld32(t_lane + t_o + c, o);
#pragma unroll
        for (int i = 0; i < 32; i++) o[i] *= f;
        tmem_st32(t_lane + t_o + c, o);
      }
      if (raise) l *= f;
    }
    if (raise) m_used = mx;
    const float mu = m_used == -INFINITY ? 0.0f : m_used;
    float sum = 0.0f;
    unsigned char* pb = sp + st * kP;
    // P buffer st is free once the P V that read it (page j - 2) completed
    if (j >= 2) mbar_wait(&pv_done[st], ((j - 2) >> 1) & 1);
#pragma unroll
    for (int c = 0; c < 8; c++) {
      float p[8];
#pragma unroll
      for (int e = 0; e < 8; e++) {
        p[e] = exp2f(s[8 * c + e] - mu);
        sum += p[e];
      }
      const uint4 v = make_uint4(pack2(p[0], p[1]), pack2(p[2], p[3]), pack2(p[4], p[5]), pack2(p[6], p[7]));
      *reinterpret_cast<uint4*>(pb + r * 128 + ((c ^ (r & 7)) << 4)) = v;
    }
    l += sum;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // every row's P and O rescale are in place
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const unsigned char* vb = skv + (j % NKV) * kKV + 2 * kBox;
#pragma unroll
      for (int kk = 0; kk < 4; kk++)  // 16 keys per MMA
        mma_f16(tmem + t_o, smem_desc(pb) + (uint64_t)((kk * 32) >> 4), smem_desc_mn(vb + kk * 2048, kBox), kIdPV,
                (j > 0 || kk > 0) ? 1u : 0u);
      mma_commit(&pv_done[st]);
      if (j >= 1 && j - 1 + NKV < n_pages) {  // refill page j - 1's stage (its P V is done by now)
        mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
        issue_kv(j - 1 + NKV);
      }
    }
  }
  // O / l -> bf16 attention output
  const int jl = n_pages - 1;
  mbar_wait(&pv_done[jl & 1], (jl >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const float inv = l > 0.0f ? 1.0f / l : 0.0f;
#pragma unroll 1
  for (int c = 0; c < HD; c += 32) {
    float o[32];
    tmem_ld32(t_lane + t_o + c, o);
    if (live) {
      __nv_bfloat16* dst = out + (size_t)(tile.row0 + r) * d + h * HD + c;
#pragma unroll
      for (int i = 0; i < 32; i += 8)
        *reinterpret_cast<uint4*>(dst + i) = make_uint4(pack2(o[i] * inv, o[i + 1] * inv),
                                                         pack2(o[i + 2] * inv, o[i + 3] * inv),
                                                         pack2(o[i + 4] * inv, o[i + 5] * inv),
                                                         pack2(o[i + 6] * inv, o[i + 7] * inv));
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

}  // namespace

void launch_prefill_attention_tc(const Fwd& f, const ModelDims& m, const TmaMap& pool_map, const float* q, int layer,
                                 void* out, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(prefill_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  launch_k(prefill_attn_tc_kernel, dim3(f.n_ptiles, m.H), dim3(128), (size_t)kSmem, s,
           *reinterpret_cast<const CUtensorMap*>(pool_map.bytes), f.ptiles, f.ptab, q, m.L, layer, m.H, m.d,
           m.attn_scale * 1.4426950408889634f, (__nv_bfloat16*)out);
}

}  // namespace fe
