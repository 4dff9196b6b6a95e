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
//   * a dedicated issuer warp (one lane) drives TMA and MMA two pages ahead of
//     the softmax warps; tcgen05.commit and warp arrivals -> mbarriers.
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
constexpr int kHalf = 2 * kBox;               // 16 KB: K (or V) of one page, dims 0-63 | 64-127
constexpr int kQ = QR * HD * 2;               // 32 KB: Q tile (two 128 x 64 boxes)
constexpr int kP = QR * 64 * 2;               // 16 KB: P tile [128 x 64 keys]
constexpr int NK = 4, NV = 4;                 // K and V pages in flight (separate rings)
constexpr int NS = 3;                         // S (TMEM) and P (smem) buffers
constexpr int kSmem = (NK + NV) * kHalf + kQ + NS * kP + 3072 + 1024 + 256;
constexpr float kRescale = 8.0f;              // log2 headroom before the running max is raised
constexpr int kTmemCols = 512;                // S0-2 [0,192), O [256,384)

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// 2^x on the SFU, flush-to-zero (x <= kRescale here: scores minus the stale running max)
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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
constexpr int kSoftWarps = 8;                                       // 2 per 32-row TMEM lane group
constexpr int kIssuer = kSoftWarps;                                 // warp index of the TMA/MMA issuer
constexpr int kThreads = 32 * (kSoftWarps + 1);
// diagnostics (option "pattn_trace"): clock64 stamps of head 0's CTAs, 512 per tile
#define PT_STAMP(slot) \
  do {                                                                                   \
    if (trace && h == 0 && (slot) < 512) trace[tix * 512 + (slot)] = clock64(); \
  } while (0)

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void pair_sync(int id) {  // the two softmax warps of one lane group
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{ .reg .pred P; elect.sync _|P, 0xffffffff; selp.b32 %0, 1, 0, P; }" : "=r"(p));
  return p != 0;
}

// Warps 0-7: softmax.  Warp w owns query rows 32 (w & 3) .. + 31 (its TMEM
// lane group) and key half w >> 2 (32 of a page's 64 keys); the two warps of
// a lane group swap their row maxima through shared memory once per page.
// Warp 8: TMA + MMA issue (the whole warp runs the schedule, one elected lane
// issues), three pages of S ahead of the softmax so the issue latency of the
// next S never sits on the softmax's critical path.  K and V have separate
// rings: a K stage frees when its S completes, a V stage when its P V does.
// Handshakes, all mbarriers:
//   full_k/full_v[st]  TMA -> issuer        K (V) of a page landed
//   s_full[b]          issuer -> softmax    S_j complete in TMEM buffer j % 3
//   p_full[b]          softmax -> issuer    P_j written (and any O rescale stored)
//   pv_done[b]         issuer -> both       P_j V_j complete: O stable, P buffer free
__global__ void __launch_bounds__(kThreads, 1)
prefill_attn_tc_kernel(const __grid_constant__ CUtensorMap pool_map, const PrefillTile* __restrict__ tiles,
                       const int32_t* __restrict__ ptab, const float* __restrict__ q, int L, int layer, int H, int d,
                       float scale_log2, __nv_bfloat16* __restrict__ out, unsigned long long* trace) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sk = smem;                        // [NK][K lo, K hi]
  unsigned char* sv = sk + NK * kHalf;             // [NV][V lo, V hi]
  unsigned char* sq = sv + NV * kHalf;             // Q: [dims 0-63 | dims 64-127] x 128 rows
  unsigned char* sp = sq + kQ;                     // P: [NS][128 x 64]
  float* red = (float*)(sp + NS * kP);             // [2 pages][2 halves][128 rows] maxima, then [2][128] sums
  uint64_t* full_k = (uint64_t*)(red + 768);       // [NK]
  uint64_t* full_v = full_k + NK;                  // [NV]
  uint64_t* s_full = full_v + NV;                  // [NS]
  uint64_t* p_full = s_full + NS;                  // [NS]
  uint64_t* pv_done = p_full + NS;                 // [NS]
  uint32_t* tmem_slot = (uint32_t*)(pv_done + NS);

  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // 1-D grid in block-launch order heaviest tile first across all heads:
  // block b -> tile n_tiles - 1 - b / H, head b % H (a tile's pages grow with
  // its position, so the blocks left for a second wave are the short ones)
  const int n_tiles = gridDim.x / H;
  const int h = blockIdx.x % H, tix = blockIdx.x / H;
  if (warp == kIssuer) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&pool_map) : "memory");
      for (int i = 0; i < NK; i++) mbar_init(&full_k[i], 1);
      for (int i = 0; i < NV; i++) mbar_init(&full_v[i], 1);
      for (int i = 0; i < NS; i++) {
        mbar_init(&s_full[i], 1);
        mbar_init(&p_full[i], kSoftWarps);
        mbar_init(&pv_done[i], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) PT_STAMP(0);
  pdl_wait();  // q and the K/V of this forward's rows come from the QKV GEMM
  const PrefillTile tile = tiles[n_tiles - 1 - tix];
  const int32_t* pages = ptab + tile.pages;
  const int pos0 = tile.pos0, n_rows = tile.n;
  const int n_pages = (pos0 + n_rows - 1) / FE_PAGE + 1;

  // K (kv = 0) or V (kv = 1) of page j -> its ring stage (elected issuer lane)
  auto issue_load = [&](int j, int kv) {
    const int st = j % (kv ? NV : NK);
    const int row = ((((pages[j] * L + layer) * 2 + kv) * H + h) * 64);
    unsigned char* b = (kv ? sv : sk) + st * kHalf;
    uint64_t* bar = kv ? &full_v[st] : &full_k[st];
    mbar_expect_tx(bar, kHalf);
    tma_load_2d(b, &pool_map, bar, 0, row);
    tma_load_2d(b + kBox, &pool_map, bar, 64, row);
  };
  if (warp == kIssuer && lane == 0) {  // barriers were initialised by this thread
    for (int j = 0; j < min(NK, n_pages); j++) issue_load(j, 0);
    for (int j = 0; j < min(NV, n_pages); j++) issue_load(j, 1);
  }

  // Q -> bf16 (exp2 domain), 128B-swizzled K-major: softmax warp w stages rows
  // 16 w .. 16 w + 15, one coalesced 512-byte row per load (lane = 4 dims)
  if (warp < kSoftWarps) {
    const int c = lane >> 1;               // 16-byte chunk = dims 8c .. 8c + 7
#pragma unroll 8
    for (int i = 0; i < 16; i++) {
      const int row = 16 * warp + i;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < n_rows) a = *reinterpret_cast<const float4*>(q + (size_t)(tile.row0 + row) * d + h * HD + 4 * lane);
      const float sc = scale_log2;
      *reinterpret_cast<uint2*>(sq + (c >> 3) * (QR * 128) + row * 128 + (((c & 7) ^ (row & 7)) << 4) +
                                ((lane & 1) << 3)) = make_uint2(pack2(a.x * sc, a.y * sc), pack2(a.z * sc, a.w * sc));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_o = 256;  // O accumulator columns
  if (tid == 0) PT_STAMP(1);

  if (warp == kIssuer) {
    // descriptors as base + (byte offset >> 4): the start-address field is the
    // low 14 bits and every operand lies below 256 KB, so plain adds are exact
    const uint64_t dq = smem_desc(sq), dk = smem_desc(sk), dp = smem_desc(sp), dv = smem_desc_mn(sv, kBox);
    auto mma_s = [&](int j) {  // S_j = Q K_j^T -> TMEM cols (j % NS) * 64
      const int kst = j % NK;
      mbar_wait(&full_k[kst], (j / NK) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (elect_one()) {
        const uint32_t dst = tmem + (uint32_t)((j % NS) * 64);
        const uint64_t kb = dk + (uint64_t)((kst * kHalf) >> 4);
#pragma unroll
        for (int ks = 0; ks < 8; ks++) {
          const uint64_t off = (uint64_t)((ks & 3) * 2 + (ks >> 2) * ((QR * 128) >> 4));
          const uint64_t koff = (uint64_t)((ks & 3) * 2 + (ks >> 2) * (kBox >> 4));
          mma_f16(dst, dq + off, kb + koff, kIdS, ks > 0 ? 1u : 0u);
        }
        mma_commit(&s_full[j % NS]);
      }
      __syncwarp();
    };
    for (int j = 0; j < min(NS, n_pages); j++) mma_s(j);
    for (int m = 0; m < 2 && m + NK < n_pages; m++) {  // K stages of pages 0, 1 free once their S completed
      mbar_wait(&s_full[m % NS], (m / NS) & 1);
      if (elect_one()) issue_load(m + NK, 0);
      __syncwarp();
    }
    for (int j = 0; j < n_pages; j++) {
      const int b = j % NS, vst = j % NV;
      mbar_wait(&p_full[b], (j / NS) & 1);
      if (lane == 0) PT_STAMP(16 + 16 * j + 12);
      mbar_wait(&full_v[vst], (j / NV) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (elect_one()) {
        const uint64_t pb = dp + (uint64_t)((b * kP) >> 4);
        const uint64_t vb = dv + (uint64_t)((vst * kHalf) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; kk++)  // 16 keys per MMA
          mma_f16(tmem + t_o, pb + (uint64_t)(kk * 2), vb + (uint64_t)(kk * (2048 >> 4)), kIdPV,
                  (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit(&pv_done[b]);
      }
      __syncwarp();
      if (lane == 0) PT_STAMP(16 + 16 * j + 13);
      // S buffer b was read by the softmax before p_full[b]
      if (j + NS < n_pages) mma_s(j + NS);
      if (lane == 0) PT_STAMP(16 + 16 * j + 14);
      // refills: page j + 2's K stage (its S was issued an iteration ago) and
      // page j - 1's V stage (its P V likewise) -- both all but certainly done
      if (j + 2 + NK < n_pages) {
        mbar_wait(&s_full[(j + 2) % NS], ((j + 2) / NS) & 1);
        if (elect_one()) issue_load(j + 2 + NK, 0);
        __syncwarp();
      }
      if (j >= 1 && j - 1 + NV < n_pages) {
        mbar_wait(&pv_done[(j - 1) % NS], ((j - 1) / NS) & 1);
        if (elect_one()) issue_load(j - 1 + NV, 1);
        __syncwarp();
      }
    }
  } else {
    const int grp = warp & 3, hf = warp >> 2;     // lane group, key half
    const int r = 32 * grp + lane;                // query row of the tile = TMEM lane
    const int pos = pos0 + r;
    const bool live = r < n_rows;
    const uint32_t t_lane = tmem + ((uint32_t)(32 * grp) << 16);
    float m_used = -INFINITY, l = 0.0f;  // running (stale) max, partial sum over this half's keys
    for (int j = 0; j < n_pages; j++) {
      const int b = j % NS;
      mbar_wait(&s_full[b], (j / NS) & 1);
      if (tid == 0) PT_STAMP(16 + 16 * j);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float s[32];
      tmem_ld32(t_lane + (uint32_t)(b * 64 + hf * 32), s);
      const int kb0 = j * FE_PAGE + hf * 32;      // key position of s[0]
      // causal / tail mask: only the diagonal pages (and a ragged tile's dead
      // rows) need it -- warp-uniform test
      if (__any_sync(0xffffffffu, !live || kb0 + 31 > pos)) {
        const int lim = live ? pos - kb0 : -1;
#pragma unroll
        for (int i = 0; i < 32; i++) s[i] = i <= lim ? s[i] : -INFINITY;
      }
      float mx8[8];
#pragma unroll
      for (int e = 0; e < 8; e++) mx8[e] = fmaxf(fmaxf(s[e], s[e + 8]), fmaxf(s[e + 16], s[e + 24]));
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[4]), fmaxf(mx8[2], mx8[6])),
                       fmaxf(fmaxf(mx8[1], mx8[5]), fmaxf(mx8[3], mx8[7])));
      // row max over both key halves (double-buffered by page parity)
      red[((j & 1) * 2 + hf) * 128 + r] = mx;
      pair_sync(1 + grp);
      mx = fmaxf(mx, red[((j & 1) * 2 + (hf ^ 1)) * 128 + r]);
      if (tid == 0) PT_STAMP(16 + 16 * j + 2);
      // raise the running max only when the new scores would overflow the
      // headroom (both warps of the pair decide identically)
      const bool raise = mx > m_used + kRescale;
      if (__any_sync(0xffffffffu, raise && j > 0)) {
        // the P V of page j - 1 must have landed in O before O is rescaled
        mbar_wait(&pv_done[(j - 1) % NS], ((j - 1) / NS) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float f = raise ? exp2f(m_used - mx) : 1.0f;  // m_used = -inf -> 0 (O is still 0)
#pragma unroll 1
        for (int c = hf * 64; c < hf * 64 + 64; c += 32) {  // this half's O columns
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
      float sum4[4];
      unsigned char* pb = sp + b * kP;
      // P buffer b is free once the P V that read it (page j - 3) completed
      if (j >= NS) mbar_wait(&pv_done[b], ((j - NS) / NS) & 1);
      if (tid == 0) PT_STAMP(16 + 16 * j + 3);
#pragma unroll
      for (int c = 0; c < 4; c++) {
        float p[8];
#pragma unroll
        for (int e = 0; e < 8; e++) p[e] = ex2_approx(s[8 * c + e] - mu);
        sum4[c] = ((p[0] + p[4]) + (p[2] + p[6])) + ((p[1] + p[5]) + (p[3] + p[7]));
        const uint4 v = make_uint4(pack2(p[0], p[1]), pack2(p[2], p[3]), pack2(p[4], p[5]), pack2(p[6], p[7]));
        const int ch = 4 * hf + c;                // 16-byte chunk of the row's 64 keys
        *reinterpret_cast<uint4*>(pb + r * 128 + ((ch ^ (r & 7)) << 4)) = v;
      }
      l += (sum4[0] + sum4[2]) + (sum4[1] + sum4[3]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);  // this warp's half of 32 rows of P (and O) are in place
      if (lane == 0) PT_STAMP(16 + 16 * j + 4 + warp);
    }
    // O / l -> bf16 attention output; l = both halves' partial sums
    red[512 + hf * 128 + r] = l;
    const int jl = n_pages - 1;
    mbar_wait(&pv_done[jl % NS], (jl / NS) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    pair_sync(1 + grp);
    const float lt = red[512 + r] + red[640 + r];
    const float inv = lt > 0.0f ? 1.0f / lt : 0.0f;
    // this half's 64 O columns -> bf16 in the (now idle) Q buffer, then
    // coalesced stores: row r's 16-byte chunk k at r * 256 + ((k ^ (r & 7)) << 4)
    unsigned char* so = sq;
#pragma unroll 1
    for (int c = hf * 64; c < hf * 64 + 64; c += 32) {
      float o[32];
      tmem_ld32(t_lane + t_o + c, o);
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        const int k = (c + i) >> 3;
        *reinterpret_cast<uint4*>(so + r * 256 + ((k ^ (r & 7)) << 4)) =
            make_uint4(pack2(o[i] * inv, o[i + 1] * inv), pack2(o[i + 2] * inv, o[i + 3] * inv),
                       pack2(o[i + 4] * inv, o[i + 5] * inv), pack2(o[i + 6] * inv, o[i + 7] * inv));
      }
    }
    __syncwarp();
#pragma unroll 4
    for (int i = 0; i < 32; i += 4) {      // four half-rows per instruction, 8 lanes x 16 B each
      const int row = 32 * grp + i + (lane >> 3), k = 8 * hf + (lane & 7);
      if (row < n_rows)
        *reinterpret_cast<uint4*>(out + (size_t)(tile.row0 + row) * d + h * HD + 8 * k) =
            *reinterpret_cast<const uint4*>(so + row * 256 + ((k ^ (row & 7)) << 4));
    }
  }
  if (tid == 0) PT_STAMP(15);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == kIssuer) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
  }
}

}  // namespace

void launch_prefill_attention_tc(const Fwd& f, const ModelDims& m, const TmaMap& pool_map, const float* q, int layer,
                                 void* out, cudaStream_t s, unsigned long long* trace) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(prefill_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  launch_k(prefill_attn_tc_kernel, dim3(f.n_ptiles * m.H), dim3(kThreads), (size_t)kSmem, s,
           *reinterpret_cast<const CUtensorMap*>(pool_map.bytes), f.ptiles, f.ptab, q, m.L, layer, m.H, m.d,
           m.attn_scale * 1.4426950408889634f, (__nv_bfloat16*)out, trace);
}

}  // namespace fe
