// Persistent decode-tick kernel for the bf16 path (<= 16 rows per tick).
//
// One launch = one decode iteration of the whole model.  A decode tick is
// HBM-bound (13.2 GB of weights per tick for the 7B shape), and a chain of
// ~200 short kernels per tick loses a few microseconds of ramp-up and tail
// on every launch.  Here one CTA per SM streams weight tiles continuously
// through one TMA ring across every GEMM of every layer; the phases of the
// tick are separated by grid barriers that only gate the *activation*
// loads, so the weight stream never stops at a layer or matrix boundary.
//
// Warp roles (192 threads):
//   warp 0      TMA producer.  Issues the weight tile of every ring stage as
//               soon as the slot is free; the 16-row activation tile of a
//               stage is issued once the phase's grid barrier has been
//               passed (stages waiting for it are queued, at most one ring).
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue (swap-AB:
//               M = 128 weight rows, N = 16 batch rows, K = 16) into a
//               4-deep TMEM accumulator ring.
//   warps 2-5   epilogues and the non-GEMM phases (embedding, cascade
//               attention on mma.sync, argmax finalisation).
//
// Phases per tick (each ends with a grid barrier):
//   EMBED        x = embed[token]; xg = bf16(x * g_attn[0]); ss = sum x^2 per 128-column tile
//   per layer:   QKV   (epilogue: r = rsqrt(sum ss / d + eps), RoPE, q, paged K/V append)
//                ATTN  (cascade attention chunk partials of every (page, head) item, mma.sync)
//                AMERGE (chunk merge per (row, head) -> bf16 attention output)
//                O     (epilogue: residual add, xg = bf16(x * g_ffn), ss)
//                GU    (epilogue: r, SiLU(gate) * up -> act)
//                DOWN  (epilogue: residual add, xg = bf16(x * g_next), ss)
//   LM           lm_head + per-tile argmax keys (and fp32 logits in parity mode)
//   FINAL        greedy token per row -> out_tokens (fed back to the next tick)
//
// RMSNorm is folded: y = W (x * r * g) is computed as r * (W bf16(x * g)),
// with r from per-tile partial sums of squares written by the producing
// epilogue (fixed-order sums: deterministic).  Split-K partials are published
// with a release-add on a per-tile counter and reduced in split order by the
// tile's owner CTA after its own units (no CTA ever waits on a unit that is
// queued behind its wait), so results do not depend on timing.  Numerics are the bf16 path's (fp32 accumulation, bf16 operands);
// the fp32 canonical mode never uses this kernel.
//
// Grid barriers need every CTA resident: grid = SM count, one CTA per SM
// (shared memory forces it), no PDL, and only one lane runs this kernel.
#include "common.cuh"
#include "decode_mk.h"
#include "engine_internal.h"
#include "tc_util.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#ifndef MK_TRACE
#define MK_TRACE 0  // decode_mk_trace.cu builds the instrumented variant
#endif
#define MKTR(a) (MK_TRACE ? (a).trace : (unsigned long long*)nullptr)

namespace fe {
namespace {
using namespace tc;

constexpr int MT = 128;                    // weight rows per tile (UMMA M)
constexpr int KBK = 64;                    // K per ring stage
constexpr int XR = 16;                     // batch rows (UMMA N)
constexpr int kStages = 11;
constexpr int kAcc = 4;
constexpr int kWBytes = MT * KBK * 2;      // 16 KB
constexpr int kXBytes = XR * KBK * 2;      // 2 KB
constexpr int kThreads = 256;  // producer, MMA, 4 epilogue warps, helper, attention warp
constexpr int kAttnWarps = 5;   // the 4 epilogue warps + warp 7 stage and compute attention pairs
constexpr int HD = 128;                    // head dim (7B shape)
constexpr uint32_t kIdesc = idesc_bf16(MT, XR);
// attention phase: the (idle) ring holds K and V of up to 6 (page, head) pairs
constexpr int kAttnSlotBytes = 2 * FE_PAGE * HD * 2;  // 32 KB
constexpr int kAttnSlots = kStages * (kWBytes + kXBytes) / kAttnSlotBytes;
constexpr int kMaxPairs = kAttnSlots;
constexpr int kRing = 64;            // event / task rings (entries in flight per CTA << 64)
constexpr int kPartStride = HD + 4;  // attention chunk partial record: m, l, pad, pad, o[HD] (16-byte aligned)
constexpr int kStgStride = HD + 4;   // o staging rows in shared memory  // (page, head) pairs per CTA whose items are cached in smem
constexpr int kPtabOff = kStages * (kWBytes + kXBytes) + MT * (XR + 1) * 4 + XR * HD * 4 /* rope */ +
                         4096 /* barriers, scratch, rows, items */;
constexpr int kSmem = kPtabOff + 1024 /* phase table */ + 1024 /* align */;
static_assert(kAttnSlots >= 4, "attention staging needs >= 4 slots");

enum Kind { K_EMBED, K_QKV, K_RQKV, K_ATTN, K_AMERGE, K_O, K_RO, K_GU, K_RGU, K_DOWN, K_RDOWN, K_LM, K_RLM, K_FINAL };

struct Args {
  MkPlan plan[5];
  const CUtensorMap* wmaps;
  const float* const* norms;
  int d, F, H, L, V, n_text;
  float eps, scale_log2;
  const int32_t* hdr;
  const RowMeta* rows;
  const AttnItem* items;
  const ItemRow* item_rows;
  int B;
  const __nv_bfloat16* embed;
  int32_t* out_tokens;
  float* x;
  __nv_bfloat16* xg;
  float* ss;
  float* q;                  // holds bf16 q [16][d] (pre-scaled by scale_log2) in this kernel
  __nv_bfloat16* attn;
  __nv_bfloat16* kv_pool;
  size_t page_elems;
  const float* rope;
  float* partial;
  int* counters;
  float* apartial;
  int* acounters;
  unsigned long long* part_keys;
  float* logits;
  unsigned long long* bar;
  int flags;                  // diagnostics (engine option "mk_flags")
  int fused;                  // bit MK_*: GEMM finalised in-phase (option "mk_fused")
  int pf_stages;              // weight stages prefetched ahead of a phase's grid barrier (<= kStages)
  int* grab;                  // [P] chunk counters of the GEMM phases (reset by the last CTA to exit)
  unsigned long long* trace;  // diagnostics: [P][6][G] globaltimer: barrier pass, phase done, last weight load issued,
                             // first / last accumulator ready, segments drained
};

// per layer: QKV, RQKV, ATTN, AMERGE, O, RO, GU, DOWN, RDOWN.  Gate/up and
// lm_head (many tiles) finalise their tiles progressively inside the GEMM
// phase (role_helper); QKV, O and down (few, long-K tiles whose chunks all
// land at the end) reduce in a separate phase, which measured faster.
// a.fused: bit MK_* set = that GEMM finalises its tiles inside its own phase
// (helper warp), else a reduction phase follows it
__device__ __forceinline__ int layer_phases(const Args& a) {
  return 6 + !(a.fused >> MK_QKV & 1) + !(a.fused >> MK_O & 1) + !(a.fused >> MK_GU & 1) + !(a.fused >> MK_DOWN & 1);
}
__device__ __forceinline__ int n_phases(const Args& a) { return 3 + layer_phases(a) * a.L; }
__device__ __forceinline__ int phase_kind(const Args& a, int ph, int* layer) {
  *layer = 0;
  const int lp = layer_phases(a);
  if (ph == 0) return K_EMBED;
  if (ph == 1 + lp * a.L) return K_LM;
  if (ph == 2 + lp * a.L) return K_FINAL;
  *layer = (ph - 1) / lp;
  int k = (ph - 1) % lp;
  // QKV [RQKV] ATTN AMERGE O [RO] GU [RGU] DOWN [RDOWN]
  const int seq[10] = {K_QKV, K_RQKV, K_ATTN, K_AMERGE, K_O, K_RO, K_GU, K_RGU, K_DOWN, K_RDOWN};
  const bool has[10] = {true, !(a.fused >> MK_QKV & 1), true, true, true, !(a.fused >> MK_O & 1),
                        true, !(a.fused >> MK_GU & 1), true, !(a.fused >> MK_DOWN & 1)};
#pragma unroll
  for (int i = 0; i < 10; i++) {
    if (!has[i]) continue;
    if (k == 0) return seq[i];
    k--;
  }
  return K_FINAL;  // unreachable
}
// the GEMM whose chunk partials a reduction phase finalises
__device__ __forceinline__ int gemm_kind_of_reduce(int kind) {
  return kind == K_RQKV ? K_QKV : kind == K_RO ? K_O : kind == K_RGU ? K_GU : kind == K_RDOWN ? K_DOWN
       : kind == K_RLM ? K_LM : -1;
}
__device__ __forceinline__ int gemm_of(int kind) {
  return kind == K_QKV ? MK_QKV : kind == K_O ? MK_O : kind == K_GU ? MK_GU : kind == K_DOWN ? MK_DOWN
       : kind == K_LM ? MK_LM : -1;
}
// phase -> (kind, layer) from the table every CTA builds at launch
// (phase_kind's fused-mask walk stays out of the roles' code)
__device__ __forceinline__ int pkind(const unsigned char* ptab, int ph, int* layer) {
  *layer = ptab[512 + ph];
  return ptab[ph];
}
__device__ __forceinline__ bool fused_reduce_a(const Args& a, int kind) {
  const int gi = gemm_of(kind);
  return gi >= 0 && (a.fused >> gi & 1);
}
__device__ __forceinline__ const CUtensorMap* wmap_of(const Args& a, int gi, int l) {
  return gi == MK_LM ? &a.wmaps[4 * a.L] : &a.wmaps[4 * l + gi];
}
// Dynamic chunks: tile t's k-blocks are cut into nc chunks; CTAs grab chunk
// ids q = t * nc + j from a per-phase counter (tile-major, so tiles complete
// progressively through the phase and fast SMs simply take more chunks).
__device__ __forceinline__ void chunk_range(const MkPlan& p, int q, int* t, int* j, int* kb0, int* kb1) {
  *t = q / p.nc;
  *j = q - *t * p.nc;
  *kb0 = *j * p.kb_total / p.nc;
  *kb1 = (*j + 1) * p.kb_total / p.nc;
}
// producer -> MMA / epilogue queue of grabbed chunk ids (-1 ends a phase)
constexpr int kQueue = 32;
__device__ __forceinline__ int queue_read(volatile int* qseq, volatile int* qval, int n) {
  while (qseq[n % kQueue] != n) {
  }
  __threadfence_block();
  return qval[n % kQueue];
}

// ---- grid barrier (monotonic arrival counter, reset by the last CTA to exit)
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const unsigned long long* p, unsigned long long target) {
  if (ld_acquire(p) >= target) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned spins = 0;
  while (ld_acquire(p) < target) {
    if (++spins % 1024 == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 2000000000ull) __trap();  // 2 s: a lost CTA; abort instead of hanging the GPU
    }
  }
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// producer side: wait until the epilogue warps have seen phase `ph`'s grid barrier
__device__ __forceinline__ void wait_ready(volatile int* ready_ph, int ph) {
  if (*ready_ph >= ph) return;
  const uint64_t t0 = gtimer();
  unsigned spins = 0;
  while (*ready_ph < ph) {
    if (++spins % 1024 == 0 && gtimer() - t0 > 2000000000ull) __trap();
  }
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// ---- epilogue-group (warps 2-5) helpers
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// the attention phase's group: the 4 epilogue warps and warp 7
__device__ __forceinline__ void attn_sync() { asm volatile("bar.sync 2, 160;" ::: "memory"); }

// out[b * ostride] = sum over the 128 tile rows of tile[c][b]^2 (b < B), fixed
// order; the caller has synchronised the epilogue group after writing `tile`
__device__ __forceinline__ void epi_sumsq_cols(float* tile, float* red, int B, float* out, int ostride, int et) {
  // 8 groups of 16 tile rows per column b (thread et: b = et & 15, group et >> 4),
  // then the 8 group sums in order: short dependent chains, fixed order
  const int b = et & 15, grp = et >> 4;
  float acc = 0.0f;
  if (b < B) {
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const float v = tile[(16 * grp + c) * (XR + 1) + b];
      acc = fmaf(v, v, acc);
    }
  }
  red[grp * 16 + b] = acc;  // red: [8][16] scratch (rn / red / kred region)
  epi_sync();
  if (et < B) {
    float t = 0.0f;
#pragma unroll
    for (int g2 = 0; g2 < 8; g2++) t += red[g2 * 16 + et];
    out[et * ostride] = t;
  }
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ldcg4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ldcg4f(const float* p) {
  float4 r;
  asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// Cascade attention of one (page item, head) pair by one warp on mma.sync:
// S = Q K^T (M = 16 query rows, N = 8 keys, K = 16 dims), P = exp2(S - m),
// O = P V.  K and V of the (page, head) were staged in shared memory by one
// bulk copy each.  Head dims are permuted identically in Q and K so every
// lane's K fragment is one 16-byte load; V is read as 32-byte row slices and
// paired across keys with byte permutes.  Writes the chunk partial (m, l, o)
// of every row of the item; the chunks of a (row, head) are merged in the
// next phase.
// Q fragments of a pair: bf16, pre-scaled to the exp2 domain by the QKV epilogue;
// k-step s = 2i + j covers dims 32i + 8t + 4j + {0,1} | {2,3}
__device__ __forceinline__ void attn_load_q(const Args& a, const AttnItem& it, const ItemRow* irows, int h, int lane,
                                            uint4 (&q0)[4], uint4 (&q1)[4]) {
  const int g = lane >> 2, t = lane & 3;
  const __nv_bfloat16* qb = reinterpret_cast<const __nv_bfloat16*>(a.q);
  const int nr = it.row_count;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    q0[i] = g < nr ? ldcg4(qb + (size_t)irows[g].row * a.d + h * HD + 32 * i + 8 * t) : make_uint4(0u, 0u, 0u, 0u);
    q1[i] = g + 8 < nr ? ldcg4(qb + (size_t)irows[g + 8].row * a.d + h * HD + 32 * i + 8 * t)
                       : make_uint4(0u, 0u, 0u, 0u);
  }
}

__device__ void attn_pair(const Args& a, const RowMeta* srows, const AttnItem& it, const ItemRow* irows, int h,
                          const unsigned char* ks, const unsigned char* vs, const uint4 (&q0)[4],
                          const uint4 (&q1)[4], int lane, unsigned long long* dbg = nullptr) {
  if (dbg) { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory"); dbg[0] = t; }
  const int g = lane >> 2, t = lane & 3;
  const int H = a.H;
  const int nr = it.row_count;
  const int r0 = g, r1 = g + 8;
  const ItemRow ir0 = r0 < nr ? irows[r0] : ItemRow{0, 0};
  const ItemRow ir1 = r1 < nr ? irows[r1] : ItemRow{0, 0};
  const int v0 = r0 < nr ? ir0.valid : 0, v1 = r1 < nr ? ir1.valid : 0;
  const int vmax = it.valid_max;
  uint32_t qa[8][4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    qa[2 * i][0] = q0[i].x;
    qa[2 * i][1] = q1[i].x;
    qa[2 * i][2] = q0[i].y;
    qa[2 * i][3] = q1[i].y;
    qa[2 * i + 1][0] = q0[i].z;
    qa[2 * i + 1][1] = q1[i].z;
    qa[2 * i + 1][2] = q0[i].w;
    qa[2 * i + 1][3] = q1[i].w;
  }
  // S = Q K^T: k-step outer, the 8 key tiles inner (8 independent MMA chains)
  float s[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; nt++) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.0f;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint4 kv[8];
#pragma unroll
    for (int nt = 0; nt < 8; nt++)  // key 8nt + g (swizzle key & 7 = g), dims 32i + 8t .. +7
      kv[nt] = *reinterpret_cast<const uint4*>(ks + (size_t)(8 * nt + g) * HD * 2 + (((4 * i + t) ^ g) << 4));
#pragma unroll
    for (int nt = 0; nt < 8; nt++) mma_bf16(s[nt], qa[2 * i], kv[nt].x, kv[nt].y);  // keys past vmax masked below
#pragma unroll
    for (int nt = 0; nt < 8; nt++) mma_bf16(s[nt], qa[2 * i + 1], kv[nt].z, kv[nt].w);
  }
  if (dbg) { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory"); dbg[1] = t + (s[0][0] == 1234.5f); }
  // masked softmax (exp2 domain) per row; rows g (c0, c1) and g + 8 (c2, c3); tree reductions
#pragma unroll
  for (int nt = 0; nt < 8; nt++) {
    const int j = 8 * nt + 2 * t;
    s[nt][0] = j < v0 ? s[nt][0] : -INFINITY;
    s[nt][1] = j + 1 < v0 ? s[nt][1] : -INFINITY;
    s[nt][2] = j < v1 ? s[nt][2] : -INFINITY;
    s[nt][3] = j + 1 < v1 ? s[nt][3] : -INFINITY;
  }
  float mx0[8], mx1[8];
#pragma unroll
  for (int nt = 0; nt < 8; nt++) {
    mx0[nt] = fmaxf(s[nt][0], s[nt][1]);
    mx1[nt] = fmaxf(s[nt][2], s[nt][3]);
  }
#pragma unroll
  for (int w2 = 4; w2 >= 1; w2 >>= 1)
#pragma unroll
    for (int nt = 0; nt < w2; nt++) {
      mx0[nt] = fmaxf(mx0[nt], mx0[nt + w2]);
      mx1[nt] = fmaxf(mx1[nt], mx1[nt + w2]);
    }
  float m0 = mx0[0], m1 = mx1[0];
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
  m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
  const float mu0 = v0 > 0 ? m0 : 0.0f, mu1 = v1 > 0 ? m1 : 0.0f;
#pragma unroll
  for (int nt = 0; nt < 8; nt++) {  // exp2(-inf) = 0 for the masked keys
    s[nt][0] = exp2f(s[nt][0] - mu0);
    s[nt][1] = exp2f(s[nt][1] - mu0);
    s[nt][2] = exp2f(s[nt][2] - mu1);
    s[nt][3] = exp2f(s[nt][3] - mu1);
  }
  float sm0[8], sm1[8];
#pragma unroll
  for (int nt = 0; nt < 8; nt++) {
    sm0[nt] = s[nt][0] + s[nt][1];
    sm1[nt] = s[nt][2] + s[nt][3];
  }
#pragma unroll
  for (int w2 = 4; w2 >= 1; w2 >>= 1)
#pragma unroll
    for (int nt = 0; nt < w2; nt++) {
      sm0[nt] += sm0[nt + w2];
      sm1[nt] += sm1[nt + w2];
    }
  float l0 = sm0[0], l1 = sm1[0];
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

  if (dbg) { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory"); dbg[2] = t + (s[0][0] == 1234.5f); }
  // O = P V over 16-key steps kk; output dim of (n-tile nt, column n) = 16 n + nt.
  // Two passes over the output n-tiles (8 each) keep the accumulators at 32 registers.
  uint32_t pa[4][4];
#pragma unroll
  for (int kk = 0; kk < 4; kk++) {
    pa[kk][0] = pack_bf16(s[2 * kk][0], s[2 * kk][1]);
    pa[kk][1] = pack_bf16(s[2 * kk][2], s[2 * kk][3]);
    pa[kk][2] = pack_bf16(s[2 * kk + 1][0], s[2 * kk + 1][1]);
    pa[kk][3] = pack_bf16(s[2 * kk + 1][2], s[2 * kk + 1][3]);
  }
  // chunk partial records [m, l, -, -, o[128]] (kPartStride floats, 16-byte aligned)
  if (t == 0) {
    if (r0 < nr) {
      float* pp = a.apartial + ((size_t)(srows[ir0.row].chunk_base + it.chunk) * H + h) * kPartStride;
      pp[0] = mu0;
      pp[1] = l0;
    }
    if (r1 < nr) {
      float* pp = a.apartial + ((size_t)(srows[ir1.row].chunk_base + it.chunk) * H + h) * kPartStride;
      pp[0] = mu1;
      pp[1] = l1;
    }
  }
  // o is transposed through the (no longer needed) K tile so each row leaves as one 512-byte store
  float* stg = reinterpret_cast<float*>(const_cast<unsigned char*>(ks));
  __syncwarp();
  // V fragments by ldmatrix.x4.trans: matrices (keys 16kk + {0-7, 8-15}) x (dims 16np + {0-7, 8-15});
  // lane L addresses row L & 7 of matrix L >> 3 (staged rows beyond valid_max are zero-filled)
  const int lm = lane >> 3, lrow = lane & 7;
#pragma unroll
  for (int half = 0; half < 2; half++) {
    float o[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; nt++) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < 4; kk++) {  // P = 0 and V = 0 past vmax
      const int key = 16 * kk + lrow + 8 * (lm & 1);
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int np = 4 * half + q;  // dims 16 np .. 16 np + 15 = n-tiles 2 np, 2 np + 1
        const int c = 2 * np + (lm >> 1);
        uint32_t b0, b1, b2, b3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                     : "r"(su32(vs + (size_t)key * HD * 2 + ((c ^ (key & 7)) << 4))));
        mma_bf16(o[2 * q], pa[kk], b0, b1);
        mma_bf16(o[2 * q + 1], pa[kk], b2, b3);
      }
    }
    // n-tile nt of this half = dims 64 half + 8 nt .. +7; lane (g, t) holds columns 2t, 2t + 1 of rows g, g + 8
#pragma unroll
    for (int nt = 0; nt < 8; nt++) {
      const int dim = 64 * half + 8 * nt + 2 * t;
      *reinterpret_cast<float2*>(stg + g * kStgStride + dim) = make_float2(o[nt][0], o[nt][1]);
      *reinterpret_cast<float2*>(stg + (g + 8) * kStgStride + dim) = make_float2(o[nt][2], o[nt][3]);
    }
  }
  __syncwarp();
  for (int rr = 0; rr < nr; rr++) {
    float* pp = a.apartial + ((size_t)(srows[irows[rr].row].chunk_base + it.chunk) * H + h) * kPartStride;
    __stcg(reinterpret_cast<float4*>(pp + 4) + lane, *reinterpret_cast<const float4*>(stg + rr * kStgStride + 4 * lane));
  }
  if (dbg) { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) :: "memory"); dbg[3] = t; }
}

// Merge the chunk partials of one (row, head) in chunk order -> bf16 attention output.
__device__ void attn_merge(const Args& a, const RowMeta& m, int row, int h, int lane) {
  const size_t cs = (size_t)a.H * kPartStride;
  const float* mbase = a.apartial + ((size_t)m.chunk_base * a.H + h) * kPartStride;
  const float4* base = reinterpret_cast<const float4*>(mbase + 4) + lane;
  const int nch = m.n_chunks;
  float M = -INFINITY, L = 0.0f, acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  // batches of 16 chunks: (m, l) lane-parallel plus this lane's 4 dims of each
  // chunk, all requested together (a trunk row has ~10-20 chunks: one or two
  // L2 round trips); running-max rescale across batches
  for (int c0 = 0; c0 < nch; c0 += 16) {
    const int nb = min(16, nch - c0);
    const float mc = lane < nb ? __ldcg(mbase + (c0 + lane) * cs) : -INFINITY;
    const float lc = lane < nb ? __ldcg(mbase + (c0 + lane) * cs + 1) : 0.0f;
    float4 x[16];
#pragma unroll
    for (int u = 0; u < 16; u++) x[u] = u < nb ? __ldcg(base + (c0 + u) * (cs / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
    float Mb = mc;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) Mb = fmaxf(Mb, __shfl_xor_sync(0xffffffffu, Mb, off));
    const float Mn = fmaxf(M, Mb);
    const float rescale = M == -INFINITY ? 0.0f : exp2f(M - Mn);
    L *= rescale;
    acc0 *= rescale; acc1 *= rescale; acc2 *= rescale; acc3 *= rescale;
    const float wl = lane < nb ? exp2f(mc - Mn) : 0.0f;
    float ls = wl * lc;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, off);
    L += ls;
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const float wt = __shfl_sync(0xffffffffu, wl, u);
      acc0 = fmaf(wt, x[u].x, acc0); acc1 = fmaf(wt, x[u].y, acc1);
      acc2 = fmaf(wt, x[u].z, acc2); acc3 = fmaf(wt, x[u].w, acc3);
    }
    M = Mn;
  }
  const float inv = 1.0f / L;
  uint2 packed;
  packed.x = pack_bf16(acc0 * inv, acc1 * inv);
  packed.y = pack_bf16(acc2 * inv, acc3 * inv);
  *reinterpret_cast<uint2*>(a.attn + (size_t)row * a.d + h * HD + 4 * lane) = packed;
}

__device__ __forceinline__ int ld_acquire_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Final epilogue of one reduced [128 x B] tile (fp32 in shared memory):
// thread r <-> weight row r of the tile.
__device__ __forceinline__ void tile_epilogue(const Args& a, int kind, int l, int tl, const float* tile,
                                              const float* rn, float* red, unsigned long long* kred,
                                              const RowMeta* srows, const float* srope, float gw, int et, int warp,
                                              int lane) {
  const int r = 32 * (warp & 3) + lane;
  const int d = a.d, B = a.B;
  const int n0 = tl * MT;
  if (kind == K_QKV) {
    if (et < 64) {
      const int sec = n0 / d, h = (n0 % d) / HD, half = HD / 2;
      const size_t layer_off = (size_t)l * 2 * a.H * FE_PAGE * HD;
#pragma unroll 1
      for (int b = 0; b < B; b++) {
        const RowMeta& m = srows[b];
        float x1 = tile[et * (XR + 1) + b] * rn[b], x2 = tile[(et + half) * (XR + 1) + b] * rn[b];
        if (sec < 2) {
          const float co = srope[b * HD + et], sn = srope[b * HD + half + et];
          const float r1 = fmaf(x1, co, -(x2 * sn));
          const float r2 = fmaf(x2, co, x1 * sn);
          x1 = r1;
          x2 = r2;
        }
        if (sec == 0) {  // bf16, pre-scaled for exp2-domain scores (attention A operand)
          __nv_bfloat16* qr = reinterpret_cast<__nv_bfloat16*>(a.q) + (size_t)b * d + h * HD;
          qr[et] = __float2bfloat16_rn(x1 * a.scale_log2);
          qr[et + half] = __float2bfloat16_rn(x2 * a.scale_log2);
        } else {
          __nv_bfloat16* kv = a.kv_pool + (size_t)m.kv_page * a.page_elems + layer_off +
                              ((size_t)((sec - 1) * a.H + h) * FE_PAGE + m.kv_slot) * HD;
          kv[et] = __float2bfloat16_rn(x1);
          kv[et + half] = __float2bfloat16_rn(x2);
        }
      }
    }
  } else if (kind == K_O || kind == K_DOWN) {
    const int col = n0 + r;
#pragma unroll 1
    for (int b = 0; b < B; b++) {
      const float xv = tile[r * (XR + 1) + b];  // old x already folded into the sum
      a.x[(size_t)b * d + col] = xv;
      a.xg[(size_t)b * d + col] = __float2bfloat16_rn(xv * gw);
    }
    epi_sumsq_cols(const_cast<float*>(tile), red, B, a.ss + tl, a.d / MT, et);  // ss[row][tile]
  } else if (kind == K_GU) {
    if (et < 64 && tl * 64 + et < a.F)
#pragma unroll 4
      for (int b = 0; b < B; b++) {
        const float gt = tile[et * (XR + 1) + b] * rn[b], up = tile[(et + 64) * (XR + 1) + b] * rn[b];
        a.attn[(size_t)b * a.F + tl * 64 + et] = __float2bfloat16_rn(__fdividef(gt, 1.0f + __expf(-gt)) * up);
      }
  } else {  // K_LM
    const int nrow = n0 + r;
    const bool row_ok = nrow < a.V;
#pragma unroll 1
    for (int b = 0; b < B; b++) {
      const float v = tile[r * (XR + 1) + b] * rn[b];
      unsigned long long k = (row_ok && nrow < a.n_text) ? argmax_key(v, nrow) : 0ull;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, off));
      if (lane == 0) kred[b * 4 + (warp & 3)] = k;
      if (row_ok && a.logits && srows[b].logit_row >= 0) a.logits[(size_t)srows[b].logit_row * a.V + nrow] = v;
    }
    epi_sync();
    if (et < B)
      a.part_keys[(size_t)et * a.plan[MK_LM].tiles + tl] =
          max(max(kred[et * 4], kred[et * 4 + 1]), max(kred[et * 4 + 2], kred[et * 4 + 3]));
  }
}

#define MK_SMEM_LAYOUT(smem) \
  unsigned char* sw = smem; \
  const unsigned char* ptab = smem + kPtabOff; \
  unsigned char* sx = smem + kStages * kWBytes; \
  float* tile = (float*)(sx + kStages * kXBytes); \
  float* srope = tile + MT * (XR + 1); \
  uint64_t* full = (uint64_t*)(srope + XR * HD); \
  uint64_t* empty = full + kStages; \
  uint64_t* acc_full = empty + kStages; \
  uint64_t* acc_empty = acc_full + kAcc; \
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + kAcc); \
  int* last_flag = (int*)(tmem_slot + 1); \
  float* rn = (float*)(tmem_slot + 4); \
  float* red = rn + XR; \
  unsigned long long* kred = (unsigned long long*)(red + 8 * XR); \
  volatile int* ready_ph = (volatile int*)(kred + 4 * XR); \
  RowMeta* srows = (RowMeta*)(kred + 4 * XR + 2); \
  uint64_t* abar = (uint64_t*)(srows + XR); \
  volatile int* qseq = (volatile int*)(abar + kAttnSlots); \
  volatile int* qval = qseq + kQueue; \
  AttnItem* sitems = (AttnItem*)(qval + kQueue); \
  ItemRow* sirows = (ItemRow*)(sitems + kMaxPairs); \
  int* pend_slot = (int*)(sirows + kMaxPairs * XR); \
  int* pend_kb = pend_slot + kStages; \
  volatile int* evq = (volatile int*)(pend_kb + kStages); \
  volatile int* taskq = evq + kRing; \
  volatile int* ev_cnt = taskq + kRing; \
  volatile int* task_cnt = ev_cnt + 1; \
  volatile int* task_snap = ev_cnt + 2; \
  (void)0

__device__ __noinline__ void epi_embed(const Args& a, unsigned char* smem, int ph, int l, int kind) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int et = threadIdx.x - 64;
  const int r = 32 * (warp & 3) + lane;
  const int d = a.d, B = a.B;
  const int n_ss = d / MT;
  (void)r; (void)d; (void)B; (void)n_ss; (void)G;
      for (int ct = blockIdx.x; ct < n_ss; ct += G) {
        const int col = ct * MT + et;
        const float gw = __ldg(a.norms[0] + col);
        int tok[XR];
#pragma unroll
        for (int b = 0; b < XR; b++)
          tok[b] = b < B ? (srows[b].tok >= 0 ? srows[b].tok : __ldcg(a.out_tokens + srows[b].tok_src)) : 0;
        float xv[XR];
#pragma unroll
        for (int b = 0; b < XR; b++) xv[b] = b < B ? __bfloat162float(a.embed[(size_t)tok[b] * d + col]) : 0.0f;
#pragma unroll
        for (int b = 0; b < XR; b++) {
          tile[et * (XR + 1) + b] = xv[b];
          if (b < B) {
            a.x[(size_t)b * d + col] = xv[b];
            a.xg[(size_t)b * d + col] = __float2bfloat16_rn(xv[b] * gw);
          }
        }
        epi_sync();
        epi_sumsq_cols(tile, red, B, a.ss + ct, n_ss, et);
        epi_sync();
      }
}

__device__ __noinline__ void epi_attn(const Args& a, unsigned char* smem, int ph, int l, int kind) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int et = threadIdx.x - 64;
  const int r = 32 * (warp & 3) + lane;
  const int d = a.d, B = a.B;
  const int n_ss = d / MT;
  (void)r; (void)d; (void)B; (void)n_ss; (void)G;
      // The ring is idle (the producer holds the next weights back until this
      // phase ends): stage K and V of this CTA's (page, head) pairs into it with
      // bulk copies, all in flight at once, then one warp per pair computes.
      const int n_pairs = a.hdr[1] * a.H;
      const __nv_bfloat16* pool_l = a.kv_pool + (size_t)l * 2 * a.H * FE_PAGE * HD;
      if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 2) * G + blockIdx.x] = gtimer();
      for (int base = blockIdx.x, round = 0; base < n_pairs; base += kAttnSlots * G, round++) {
        auto item_of = [&](int j, int pr) -> AttnItem { return round == 0 ? sitems[j] : a.items[pr / a.H]; };
        // each warp stages K and V of its own pairs (j = warp, warp + 4) with
        // 16-byte cp.async, one commit group per pair (rows 256 B, 16-byte chunks
        // XOR-swizzled by key & 7: the fragment reads are bank-conflict free), and
        // starts computing as soon as its first pair has landed
        const int w = warp == 7 ? 4 : warp - 2;  // attention warp 0..4
        int ngroups = 0;
        for (int j = w; j < kAttnSlots; j += kAttnWarps) {
          const int pr = base + j * G;
          if (pr >= n_pairs) break;
          const AttnItem it = item_of(j, pr);
          const __nv_bfloat16* kg = pool_l + (size_t)it.page * a.page_elems + (size_t)(pr % a.H) * FE_PAGE * HD;
          const __nv_bfloat16* vg = kg + (size_t)a.H * FE_PAGE * HD;
          unsigned char* slot = sw + (size_t)j * kAttnSlotBytes;
          // every V row of the page is staged (rows past valid_max zero-filled):
          // the MMAs then run over all 64 keys without data-dependent branches
          // around mma.sync (which cost a warp re-convergence each)
          const int vpad = FE_PAGE;
          for (int x = lane; x < vpad * 16; x += 32) {
            const int key = x >> 4, c = x & 15;
            const uint32_t so = (uint32_t)(key * 256 + ((c ^ (key & 7)) << 4));
            const bool in = key < it.valid_max;
            const int keyc = in ? key : 0;
            if (in)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(slot + so)),
                           "l"(kg + (size_t)keyc * HD + c * 8) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(slot + kAttnSlotBytes / 2 + so)),
                         "l"(vg + (size_t)keyc * HD + c * 8), "r"(in ? 16 : 0) : "memory");
          }
          asm volatile("cp.async.commit_group;" ::: "memory");
          ngroups++;
        }
        uint4 q0[4], q1[4];
        int gi = 0;
        for (int j = w; j < kAttnSlots; j += kAttnWarps, gi++) {
          const int pr = base + j * G;
          if (pr >= n_pairs) break;
          const AttnItem it = item_of(j, pr);
          const ItemRow* irows = round == 0 ? sirows + j * XR : a.item_rows + it.row_begin;
          attn_load_q(a, it, irows, pr % a.H, lane, q0, q1);  // overlaps the K / V landing
          if (ngroups - gi - 1 >= 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
          else asm volatile("cp.async.wait_group 0;" ::: "memory");
          __syncwarp();
          if (MKTR(a) && et == 0 && round == 0 && gi == 0) MKTR(a)[((size_t)ph * 6 + 3) * G + blockIdx.x] = gtimer();
          const unsigned char* slot = sw + (size_t)j * kAttnSlotBytes;
          unsigned long long* dbg = nullptr;  // diagnostics (flags & 4): sub-step times of CTA 0's first pair
          if ((MK_TRACE && (a.flags & 4)) && MKTR(a) && blockIdx.x == 0 && et == 0 && j == 0 && round == 0)
            dbg = MKTR(a) + ((size_t)(n_phases(a) - 1) * 6 + 2) * G + 8 * l;  // FINAL phase slot 2, [layer][4]
          attn_pair(a, srows, it, irows, pr % a.H, slot, slot + kAttnSlotBytes / 2, q0, q1, lane, dbg);
        }
        if (MKTR(a) && et == 0 && round == 0) MKTR(a)[((size_t)ph * 6 + 4) * G + blockIdx.x] = gtimer();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem reads before async writes
        if (warp == 7) __threadfence();  // its partials, before the epilogue warps' barrier arrival
        attn_sync();  // slots reused by the next round
        if (MKTR(a) && et == 0 && round == 0) MKTR(a)[((size_t)ph * 6 + 5) * G + blockIdx.x] = gtimer();
      }
}

__device__ __noinline__ void epi_amerge(const Args& a, unsigned char* smem, int ph, int l, int kind) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int et = threadIdx.x - 64;
  const int r = 32 * (warp & 3) + lane;
  const int d = a.d, B = a.B;
  const int n_ss = d / MT;
  (void)r; (void)d; (void)B; (void)n_ss; (void)G;
      if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 2) * G + blockIdx.x] = gtimer();
      for (int pr = blockIdx.x * 4 + (et >> 5); pr < B * a.H; pr += G * 4) {
        attn_merge(a, srows[pr / a.H], pr / a.H, pr % a.H, lane);
        if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 3) * G + blockIdx.x] = gtimer();
      }
      if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 4) * G + blockIdx.x] = gtimer();
      epi_sync();
      if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 5) * G + blockIdx.x] = gtimer();
}

__device__ __noinline__ void epi_final(const Args& a, unsigned char* smem, int ph, int l, int kind) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int et = threadIdx.x - 64;
  const int r = 32 * (warp & 3) + lane;
  const int d = a.d, B = a.B;
  const int n_ss = d / MT;
  (void)r; (void)d; (void)B; (void)n_ss; (void)G;
      const int tiles = a.plan[MK_LM].tiles;
      for (int b = blockIdx.x; b < B; b += G) {
        unsigned long long k = 0ull;
        for (int t = et; t < tiles; t += 128) k = max(k, __ldcg(&a.part_keys[(size_t)b * tiles + t]));
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) k = max(k, __shfl_xor_sync(0xffffffffu, k, off));
        if (lane == 0) kred[et >> 5] = k;
        epi_sync();
        if (et == 0) {
          const unsigned long long kk = max(max(kred[0], kred[1]), max(kred[2], kred[3]));
          if (srows[b].out_idx >= 0) a.out_tokens[srows[b].out_idx] = argmax_index(kk);
        }
        epi_sync();
      }
}

__device__ __noinline__ void finalize_tile(const Args& a, unsigned char* smem, int l, int gk, int tl, bool with_rn,
                                          int ph);

__device__ __noinline__ void epi_gemm(const Args& a, unsigned char* smem, int ph, int l, int kind, uint32_t tmem, int& lu, int& n,
                                      int& task_r) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int et = threadIdx.x - 64;
  const int r = 32 * (warp & 3) + lane;
  const int d = a.d, B = a.B;
  const int n_ss = d / MT;
  (void)r; (void)d; (void)B; (void)n_ss; (void)G;
      // ---- GEMM phase: drain each grabbed chunk's accumulator into its partial
      // slot (no synchronisation; the grid barrier publishes them)
      const MkPlan p = a.plan[gemm_of(kind)];
      const bool scaled = kind == K_QKV || kind == K_GU || kind == K_LM;
      if (fused_reduce_a(a, kind) && scaled && et < B) {  // row norms r = rsqrt(sum x^2 / d + eps) of this GEMM's input
        const float4* sr = reinterpret_cast<const float4*>(a.ss + (size_t)et * n_ss);
        float sacc = 0.0f;
        for (int u = 0; u < n_ss / 4; u++) {
          const float4 v = __ldcg(sr + u);
          sacc += (v.x + v.y) + (v.z + v.w);
        }
        rn[et] = rsqrtf(sacc / (float)d + a.eps);
      }
      const bool fused = fused_reduce_a(a, kind);
      bool phase_tasks_done = false;
      const int ev_w_base = 0;
      (void)ev_w_base;
      // tasks (tiles to finalise) are consumed in order; task_r: next to run
      auto run_tasks = [&](int upto) {
        while (task_r < upto) {
          const int tl = taskq[task_r % kRing];
          task_r++;
          if (tl < 0) {
            phase_tasks_done = true;
            break;
          }
          finalize_tile(a, smem, l, kind, tl, false, -1);
        }
      };
      bool first_chunk = true;
      for (;; lu++) {
        const int q = queue_read(qseq, qval, n++);
        if (q < 0) break;
        int tl, j, kb0, kb1;
        chunk_range(p, q, &tl, &j, &kb0, &kb1);
        const int acc = lu % kAcc;
        // residual GEMMs: chunk 0 of a tile folds the old x into its partial
        // (loaded while the MMAs run), so the tile epilogue needs no x load
        const bool fold_x = (kind == K_O || kind == K_DOWN) && j == 0;
        float xo[XR];
#pragma unroll
        for (int b = 0; b < XR; b++) xo[b] = (fold_x && b < B) ? __ldcg(a.x + (size_t)b * d + tl * MT + r) : 0.0f;
        mbar_wait(&acc_full[acc], (lu / kAcc) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (MKTR(a) && et == 0) {
          const uint64_t tnow = gtimer();
          if (first_chunk) MKTR(a)[((size_t)ph * 6 + 3) * G + blockIdx.x] = tnow;
          MKTR(a)[((size_t)ph * 6 + 4) * G + blockIdx.x] = tnow;
        }
        first_chunk = false;
        uint32_t raw[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(raw[0]), "=r"(raw[1]), "=r"(raw[2]), "=r"(raw[3]), "=r"(raw[4]), "=r"(raw[5]), "=r"(raw[6]),
              "=r"(raw[7]), "=r"(raw[8]), "=r"(raw[9]), "=r"(raw[10]), "=r"(raw[11]), "=r"(raw[12]),
              "=r"(raw[13]), "=r"(raw[14]), "=r"(raw[15])
            : "r"(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(acc * XR)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        if (et == 0) *task_snap = *task_cnt;
        epi_sync();
        if (et == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&acc_empty[acc])) : "memory");
        const int tasks_now = *task_snap;
        // partial layout [chunk][batch rows / 4][128 weight rows] float4: coalesced
        float4* dst = reinterpret_cast<float4*>(a.partial) + (size_t)q * (XR / 4) * MT + r;
#pragma unroll
        for (int q4 = 0; q4 < XR / 4; q4++)
          if (4 * q4 < B)
            __stcg(dst + q4 * MT, make_float4(__uint_as_float(raw[4 * q4]) + xo[4 * q4],
                                         __uint_as_float(raw[4 * q4 + 1]) + xo[4 * q4 + 1],
                                         __uint_as_float(raw[4 * q4 + 2]) + xo[4 * q4 + 2],
                                         __uint_as_float(raw[4 * q4 + 3]) + xo[4 * q4 + 3]));
        if (fused) {
          epi_sync();  // the chunk's partial is issued by every thread before the helper's release
          if (et == 0) {
            evq[*ev_cnt % kRing] = tl;
            __threadfence_block();
            *ev_cnt = *ev_cnt + 1;
          }
          run_tasks(tasks_now);  // tiles completed meanwhile (uniform: snapshot taken before the sync)
        }
      }
      if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 5) * G + blockIdx.x] = gtimer();
      // no more chunks: tell the helper, then finalise the remaining tasks of this phase
      if (!fused) return;
      if (et == 0) {
        evq[*ev_cnt % kRing] = -1;
        __threadfence_block();
        *ev_cnt = *ev_cnt + 1;
      }
      while (!phase_tasks_done) {
        if (et == 0) {
          const int seen = task_r;
          if (*task_cnt <= seen) {
            const uint64_t t0 = gtimer();
            unsigned spins = 0;
            while (*task_cnt <= seen)
              if (++spins % 1024 == 0 && gtimer() - t0 > 2000000000ull) __trap();
          }
          __threadfence_block();
          *task_snap = *task_cnt;
        }
        epi_sync();
        const int upto = *task_snap;
        epi_sync();  // task_snap may be rewritten next iteration
        run_tasks(upto);
      }
}

// Reduction + fused epilogue of one tile whose nc chunk partials have all
// landed: sum in chunk order (deterministic), then RoPE + q / paged K/V,
// residual + norm inputs, SiLU * up or argmax keys (tile_epilogue).  rn holds
// the phase's row norms.
__device__ __noinline__ void finalize_tile(const Args& a, unsigned char* smem, int l, int gk, int tl, bool with_rn,
                                          int ph) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int et = threadIdx.x - 64;
  const int r = 32 * (warp & 3) + lane;
  const int B = a.B;
  // with_rn: this reduction phase also derives the row norms of the GEMM
  // input (r = rsqrt(sum x^2 / d + eps)); their loads go out with the partials'
  const bool do_rn = with_rn && et < B;
  const int nq = a.d / MT / 4;
  const float4* sr = reinterpret_cast<const float4*>(a.ss + (size_t)(do_rn ? et : 0) * (a.d / MT));
  float4 sv[8];
#pragma unroll
  for (int u = 0; u < 8; u++) sv[u] = (do_rn && u < nq) ? __ldcg(sr + u) : make_float4(0.f, 0.f, 0.f, 0.f);
  const MkPlan p = a.plan[gemm_of(gk)];
  const bool resid = gk == K_O || gk == K_DOWN;
  const float* gnext = gk == K_O ? a.norms[2 * l + 1]
                       : gk == K_DOWN ? (l + 1 < a.L ? a.norms[2 * (l + 1)] : a.norms[2 * a.L]) : nullptr;
        const float gw = resid ? __ldg(gnext + tl * MT + r) : 0.0f;
  float4 acc4[XR / 4];
#pragma unroll
  for (int q4 = 0; q4 < XR / 4; q4++) acc4[q4] = make_float4(0.f, 0.f, 0.f, 0.f);
  const size_t q0 = (size_t)tl * p.nc;
  if (B <= 8 && p.nc <= 12) {  // every chunk's 2 float4 requested together (straight-line registers)
    const float4* src = reinterpret_cast<const float4*>(a.partial) + q0 * (XR / 4) * MT + r;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const int nc = p.nc;
    const bool two = B > 4;
#define MK_P(u) const float4 pa##u = u < nc ? __ldcg(src + (size_t)(u) * (XR / 4) * MT) : z; \
          const float4 pb##u = (u < nc && two) ? __ldcg(src + (size_t)(u) * (XR / 4) * MT + MT) : z;
    MK_P(0) MK_P(1) MK_P(2) MK_P(3) MK_P(4) MK_P(5) MK_P(6) MK_P(7) MK_P(8) MK_P(9) MK_P(10) MK_P(11)
#undef MK_P
#define MK_S(u) acc4[0].x += pa##u.x; acc4[0].y += pa##u.y; acc4[0].z += pa##u.z; acc4[0].w += pa##u.w; \
          acc4[1].x += pb##u.x; acc4[1].y += pb##u.y; acc4[1].z += pb##u.z; acc4[1].w += pb##u.w;
    MK_S(0) MK_S(1) MK_S(2) MK_S(3) MK_S(4) MK_S(5) MK_S(6) MK_S(7) MK_S(8) MK_S(9) MK_S(10) MK_S(11)
#undef MK_S
  } else {
    for (int c0 = 0; c0 < p.nc; c0 += 4) {
      float4 v[4][XR / 4];
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int q4 = 0; q4 < XR / 4; q4++)
          if (c0 + u < p.nc && 4 * q4 < B)
            v[u][q4] = __ldcg(reinterpret_cast<const float4*>(a.partial) + ((q0 + c0 + u) * (XR / 4) + q4) * MT + r);
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int q4 = 0; q4 < XR / 4; q4++)
          if (c0 + u < p.nc && 4 * q4 < B) {
            acc4[q4].x += v[u][q4].x; acc4[q4].y += v[u][q4].y;
            acc4[q4].z += v[u][q4].z; acc4[q4].w += v[u][q4].w;
          }
    }
  }
  if (do_rn) {
    float sacc = 0.0f;
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (u < nq) sacc += (sv[u].x + sv[u].y) + (sv[u].z + sv[u].w);
    for (int u = 8; u < nq; u++) {
      const float4 v = __ldcg(sr + u);
      sacc += (v.x + v.y) + (v.z + v.w);
    }
    rn[et] = rsqrtf(sacc / (float)a.d + a.eps);
  }
#pragma unroll
  for (int q4 = 0; q4 < XR / 4; q4++) {
    tile[r * (XR + 1) + 4 * q4] = acc4[q4].x;
    tile[r * (XR + 1) + 4 * q4 + 1] = acc4[q4].y;
    tile[r * (XR + 1) + 4 * q4 + 2] = acc4[q4].z;
    tile[r * (XR + 1) + 4 * q4 + 3] = acc4[q4].w;
  }
  // trace (reduction phases): slot 3 = partials summed, slot 4 = epilogue done
  if (MKTR(a) && ph >= 0 && et == 0) MKTR(a)[((size_t)ph * 6 + 3) * gridDim.x + blockIdx.x] = gtimer();
  epi_sync();  // tile visible
  tile_epilogue(a, gk, l, tl, tile, rn, red, kred, srows, srope, gw, et, warp, lane);
  epi_sync();  // tile / reduction scratch reused
  if (MKTR(a) && ph >= 0 && et == 0) MKTR(a)[((size_t)ph * 6 + 4) * gridDim.x + blockIdx.x] = gtimer();
}

// Separate reduction phase (QKV, O, down): tiles t = cta (mod grid).
__device__ __noinline__ void epi_reduce(const Args& a, unsigned char* smem, int ph, int l, int kind) {
  MK_SMEM_LAYOUT(smem);
  const int G = gridDim.x;
  const int et = threadIdx.x - 64;
  const int d = a.d, B = a.B;
  const int n_ss = d / MT;
  const int gk = gemm_kind_of_reduce(kind);
  const MkPlan p = a.plan[gemm_of(gk)];
  if (blockIdx.x >= p.tiles) return;
  (void)d; (void)B; (void)n_ss; (void)et;
  if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 2) * G + blockIdx.x] = gtimer();
  const bool scaled = gk == K_QKV || gk == K_GU;  // row norms computed with the first tile's partials
  for (int tl = blockIdx.x; tl < p.tiles; tl += G) finalize_tile(a, smem, l, gk, tl, scaled, ph);
  if (MKTR(a) && et == 0) MKTR(a)[((size_t)ph * 6 + 5) * G + blockIdx.x] = gtimer();
}

// Helper warp (lane 0): for every chunk the epilogue drained it adds to the
// tile's arrival counter (acquire-release); the arrival that completes a tile
// queues it for finalisation by this CTA's epilogue warps.  Keeping these
// round trips off the epilogue keeps the accumulator drain (and with it the
// MMA and the weight stream) running; tiles are finalised progressively
// through the phase instead of in a separate reduction phase.
__device__ __noinline__ void role_helper(const Args& a, unsigned char* smem) {
  MK_SMEM_LAYOUT(smem);
  const int P = n_phases(a);
  int ev_pos = 0, task_w = 0;
  for (int ph = 0; ph < P; ph++) {
    int l;
    const int kind = pkind(ptab, ph, &l);
    const int gi = gemm_of(kind);
    if (gi < 0 || !fused_reduce_a(a, kind)) continue;
    const MkPlan p = a.plan[gi];
    while (true) {
      if (*ev_cnt <= ev_pos) {
        const uint64_t t0 = gtimer();
        unsigned spins = 0;
        while (*ev_cnt <= ev_pos)
          if (++spins % 1024 == 0 && gtimer() - t0 > 2000000000ull) __trap();
      }
      __threadfence_block();
      const int tl = evq[ev_pos % kRing];
      ev_pos++;
      if (tl >= 0) {
        const int prev = atom_add_acq_rel(&a.counters[tl], 1);  // releases this CTA's partial of the chunk
        if (prev != p.nc - 1) continue;
        a.counters[tl] = 0;  // next use is after a grid barrier
      }
      taskq[task_w % kRing] = tl;  // tile, or -1: no more tasks this phase
      __threadfence_block();
      *task_cnt = ++task_w;
      if (tl < 0) break;
    }
  }
}

// The three warp roles are separate non-inlined functions so each gets its own
// register allocation (the attention / reduction code of the epilogue warps
// would otherwise force the producer's and MMA's loop state into local memory).
__device__ __noinline__ void role_producer(const Args& a, unsigned char* smem, const CUtensorMap& map_xg,
                                           const CUtensorMap& map_attn, const CUtensorMap& map_act) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int P = n_phases(a);
  (void)warp; (void)lane; (void)G; (void)P;
      // ---------------- TMA producer
      const uint64_t wpol = policy_evict_first();  // weights are read once per tick
      int it = 0, n = 0;
      for (int ph = 0; ph < P; ph++) {
        int l;
        const int kind = pkind(ptab, ph, &l);
        const int gi = gemm_of(kind);
        if (gi < 0) continue;
        const MkPlan p = a.plan[gi];
        const CUtensorMap* wm = wmap_of(a, gi, l);
        const CUtensorMap* xm = gi == MK_O ? &map_attn : gi == MK_DOWN ? &map_act : &map_xg;
        // the attention phase borrows the ring: start the O weights only once this
        // CTA's epilogue warps have left it (they publish the AMERGE barrier)
        // -- and only once the merge's outputs are fenced: its stores then do not
        // queue behind the O weight stream (measured: merge 5.8 -> 3.5 us)
        if (kind == K_O) {
          // HBM idles through the QKV reduction: pull this CTA's attention K/V
          // blocks into L2 so the attention phase stages them from L2
          const int n_pairs = a.hdr[1] * a.H;
          const __nv_bfloat16* pool_l = a.kv_pool + (size_t)l * 2 * a.H * FE_PAGE * HD;
          for (int j = 0;; j++) {  // every round's pairs (round 0's items are in shared memory)
            const int pr = blockIdx.x + j * G;
            if (pr >= n_pairs) break;
            const AttnItem it = j < kAttnSlots ? sitems[j] : a.items[pr / a.H];
            const __nv_bfloat16* kg = pool_l + (size_t)it.page * a.page_elems + (size_t)(pr % a.H) * FE_PAGE * HD;
            const uint32_t bytes = (uint32_t)it.valid_max * HD * 2;
            bulk_prefetch_l2(kg, bytes);
            bulk_prefetch_l2(kg + (size_t)a.H * FE_PAGE * HD, bytes);
          }
          {  // then this CTA's share of the O weights (the ring is the attention's until the merge ends)
            const int boxes = p.tiles * p.kb_total;
            for (int b = blockIdx.x; b < boxes; b += G) tma_prefetch_l2(wm, (b % p.kb_total) * KBK, (b / p.kb_total) * MT);
          }
        }
        if (kind == K_O) wait_ready(ready_ph + 1, ph - 1);
        if (MK_TRACE && (a.flags & 1)) wait_ready(ready_ph, ph);  // diagnostics: no weight prefetch across barriers
        bool ready = false;
        int npend = 0;
        auto flush = [&]() {
          __threadfence_block();
          fence_proxy_async();
#pragma unroll 1
          for (int i = 0; i < npend; i++)
            tma_load_2d(sx + pend_slot[i] * kXBytes, xm, &full[pend_slot[i]], pend_kb[i] * KBK, 0);
          npend = 0;
          ready = true;
        };
        int q = atomicAdd(&a.grab[ph], 1);
        while (true) {
          const bool valid = q < p.chunks;
          const int q_next = valid ? atomicAdd(&a.grab[ph], 1) : 0;  // next grab in flight meanwhile
          qval[n % kQueue] = valid ? q : -1;
          __threadfence_block();
          qseq[n % kQueue] = n;
          n++;
          if (!valid) break;
          int tl, j, kb0, kb1;
          chunk_range(p, q, &tl, &j, &kb0, &kb1);
          for (int kb = kb0; kb < kb1; kb++, it++) {
            const int s = it % kStages;
            if (!ready && npend == a.pf_stages) {  // prefetch depth reached (<= kStages: the slot to refill waits)
              wait_ready(ready_ph, ph);
              flush();
            }
            mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
            mbar_expect_tx(&full[s], kWBytes + kXBytes);
            if (gi == MK_GU) {
              tma_load_2d_hint(sw + s * kWBytes, wm, &full[s], kb * KBK, tl * (MT / 2), wpol);
              tma_load_2d_hint(sw + s * kWBytes + kWBytes / 2, wm, &full[s], kb * KBK, a.F + tl * (MT / 2), wpol);
            } else {
              tma_load_2d_hint(sw + s * kWBytes, wm, &full[s], kb * KBK, tl * MT, wpol);
            }
            if (!ready && *ready_ph >= ph) flush();
            if (ready) {
              tma_load_2d(sx + s * kXBytes, xm, &full[s], kb * KBK, 0);
            } else {
              pend_slot[npend] = s;
              pend_kb[npend] = kb;
              npend++;
            }
          }
          q = q_next;
        }
        if (MKTR(a)) MKTR(a)[((size_t)ph * 6 + 2) * G + blockIdx.x] = gtimer();
        if (!ready) {
          wait_ready(ready_ph, ph);
          flush();
        }
      }
}

__device__ __noinline__ void role_mma(const Args& a, unsigned char* smem, uint32_t tmem) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int P = n_phases(a);
  (void)warp; (void)lane; (void)G; (void)P;
      // ---------------- MMA issuer
      int it = 0, lu = 0, n = 0;
      for (int ph = 0; ph < P; ph++) {
        int l;
        const int gi = gemm_of(pkind(ptab, ph, &l));
        if (gi < 0) continue;
        const MkPlan p = a.plan[gi];
        for (;; lu++) {
          const int q = queue_read(qseq, qval, n++);
          if (q < 0) break;
          int tl, j, kb0, kb1;
          chunk_range(p, q, &tl, &j, &kb0, &kb1);
          const int acc = lu % kAcc;
          mbar_wait(&acc_empty[acc], ((lu / kAcc) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t dst = tmem + (uint32_t)(acc * XR);
          for (int kb = kb0; kb < kb1; kb++, it++) {
            const int s = it % kStages;
            mbar_wait(&full[s], (it / kStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t da = smem_desc(sw + s * kWBytes);
            const uint64_t db = smem_desc(sx + s * kXBytes);
#pragma unroll
            for (int k = 0; k < KBK / 16; k++) {
              const uint64_t off = (uint64_t)((k * 32) >> 4);
              const uint32_t accum = (kb > kb0 || k > 0) ? 1u : 0u;
              asm volatile(
                  "{ .reg .pred p; setp.ne.b32 p, %4, 0;"
                  " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                  ::"r"(dst), "l"(da + off), "l"(db + off), "r"(kIdesc), "r"(accum));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                         ::"r"(su32(&empty[s])) : "memory");
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                       ::"r"(su32(&acc_full[acc])) : "memory");
        }
      }
}

__device__ __noinline__ void role_epilogue(const Args& a, unsigned char* smem, uint32_t tmem) {
  MK_SMEM_LAYOUT(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int P = n_phases(a);
  (void)warp; (void)lane; (void)G; (void)P;
    // ---------------- epilogue / non-GEMM phases (128 threads)
    const int et = threadIdx.x - 64;
    const int r = 32 * (warp & 3) + lane;  // TMEM lane = weight row of the tile
    const int d = a.d, B = a.B;
    const int n_ss = d / MT;
    int lu = 0, n = 0, task_r = 0;
    uint32_t apar = 0;  // phase parity of the attention staging barriers
    for (int ph = 0; ph < P; ph++) {
      int l;
      const int kind = pkind(ptab, ph, &l);
      if (et == 0) {
        spin_until(a.bar, (unsigned long long)ph * G);
        if (MKTR(a)) MKTR(a)[((size_t)ph * 6) * G + blockIdx.x] = gtimer();
        __threadfence_block();
        *ready_ph = ph;  // lets the producer issue this phase's activation loads
      }
      epi_sync();

      if (kind == K_EMBED) epi_embed(a, smem, ph, l, kind);
      else if (kind == K_ATTN) epi_attn(a, smem, ph, l, kind);
      else if (kind == K_AMERGE) epi_amerge(a, smem, ph, l, kind);
      else if (kind == K_FINAL) epi_final(a, smem, ph, l, kind);
      else if (gemm_of(kind) >= 0) epi_gemm(a, smem, ph, l, kind, tmem, lu, n, task_r);
      else epi_reduce(a, smem, ph, l, kind);
      // ---- phase done: publish and arrive at the grid barrier
      if (ph + 1 < P) {
        // (generic writes consumed by the next phase's TMA loads: the consumer
        // side orders them -- the producer issues fence.proxy.async after it
        // observes the barrier -- so no proxy fence here, which would also wait
        // for this SM's in-flight weight prefetch)
        if (MK_TRACE && (a.flags & 16)) fence_proxy_async();
        __threadfence();
        epi_sync();
        if (et == 0) {
          ready_ph[1] = ph;  // this phase's outputs are fenced (the producer starts the O weights on it)
          if (MKTR(a)) MKTR(a)[((size_t)ph * 6 + 1) * G + blockIdx.x] = gtimer();
          atomicAdd(a.bar, 1ull);
        }
      }
    }
}

// Warp 7: a fifth attention warp (the attention phase is latency-bound, one
// pair per warp halves the CTAs' critical path); idle in every other phase.
__device__ __noinline__ void role_attn(const Args& a, unsigned char* smem) {
  MK_SMEM_LAYOUT(smem);
  const int P = n_phases(a);
  for (int ph = 0; ph < P; ph++) {
    int l;
    const int kind = pkind(ptab, ph, &l);
    if (kind != K_ATTN) continue;
    wait_ready(ready_ph, ph);  // the epilogue warps passed this phase's grid barrier
    __syncwarp();
    epi_attn(a, smem, ph, l, kind);
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1) decode_mk_kernel(const __grid_constant__ CUtensorMap map_xg,
                                                                const __grid_constant__ CUtensorMap map_attn,
                                                                const __grid_constant__ CUtensorMap map_act,
                                                                const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ __align__(16) Args sargs[1];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  static_assert(sizeof(Args) % 4 == 0, "Args copy");
  for (int i = threadIdx.x; i < (int)(sizeof(Args) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(sargs)[i] = reinterpret_cast<const uint32_t*>(&a)[i];
  unsigned char* sw = smem;                                  // [kStages][128 x 64] weights
  const unsigned char* ptab = smem + kPtabOff;               // phase -> kind [512], layer [512]
  unsigned char* sx = smem + kStages * kWBytes;              // [kStages][16 x 64] activations
  float* tile = (float*)(sx + kStages * kXBytes);            // [128][17]
  float* srope = tile + MT * (XR + 1);                       // [16][128] RoPE cos | sin of the rows' positions
  uint64_t* full = (uint64_t*)(srope + XR * HD);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + kAcc;
  uint32_t* tmem_slot = (uint32_t*)(acc_empty + kAcc);
  int* last_flag = (int*)(tmem_slot + 1);
  float* rn = (float*)(tmem_slot + 4);                       // [16] row norms of the phase
  float* red = rn + XR;                                      // [8][16] epilogue reductions
  unsigned long long* kred = (unsigned long long*)(red + 8 * XR);  // [16][4]
  volatile int* ready_ph = (volatile int*)(kred + 4 * XR);    // last phase whose grid barrier was passed
  RowMeta* srows = (RowMeta*)(kred + 4 * XR + 2);            // [16] rows of the tick
  uint64_t* abar = (uint64_t*)(srows + XR);                  // [kAttnSlots] K/V staging barriers
  volatile int* qseq = (volatile int*)(abar + kAttnSlots);   // [kQueue] chunk queue: sequence numbers
  volatile int* qval = qseq + kQueue;                        // [kQueue] chunk ids
  AttnItem* sitems = (AttnItem*)(qval + kQueue);             // [kMaxPairs] items of this CTA's pairs
  ItemRow* sirows = (ItemRow*)(sitems + kMaxPairs);          // [kMaxPairs][16] their query rows
  int* pend_slot = (int*)(sirows + kMaxPairs * XR);          // [kStages] producer: stages awaiting activations
  int* pend_kb = pend_slot + kStages;                        // [kStages] their k-blocks
  volatile int* evq = (volatile int*)(pend_kb + kStages);    // [kRing] epilogue -> helper: drained chunks' tiles
  volatile int* taskq = evq + kRing;                         // [kRing] helper -> epilogue: tiles to finalise
  volatile int* ev_cnt = taskq + kRing;                      // events posted (monotonic)
  volatile int* task_cnt = ev_cnt + 1;                       // tasks posted (monotonic)
  volatile int* task_snap = ev_cnt + 2;                      // epilogue-group broadcast of task_cnt

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const int P = n_phases(a);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < kAcc; i++) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 1);
    }
    for (int i = 0; i < kAttnSlots; i++) mbar_init(&abar[i], 1);
    for (int i = 0; i < kQueue; i++) qseq[i] = -1;
    if ((const unsigned char*)(task_snap + 1) > ptab) __trap();  // scratch region overflows into the phase table
    *ev_cnt = 0;
    *task_cnt = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    ready_ph[0] = -1;
    ready_ph[1] = -1;
  }
  for (int ph = threadIdx.x; ph < P; ph += blockDim.x) {
    int l;
    const int k = phase_kind(a, ph, &l);
    smem[kPtabOff + ph] = (unsigned char)k;
    smem[kPtabOff + 512 + ph] = (unsigned char)l;
  }
  if (threadIdx.x >= 64 && threadIdx.x < 192) {  // per-tick constants: rows, RoPE rows, attention items
    const int et = threadIdx.x - 64;
    if (et < a.B) srows[et] = a.rows[et];
    for (int b = 0; b < a.B; b++) srope[b * HD + et] = __ldg(a.rope + (size_t)a.rows[b].pos * HD + et);
    const int n_pairs = a.hdr[1] * a.H;
    for (int j = 0; j < kMaxPairs; j++) {
      const int pr = blockIdx.x + j * gridDim.x;
      if (pr >= n_pairs) break;
      const AttnItem it = a.items[pr / a.H];
      if (et == 0) sitems[j] = it;
      if (et < it.row_count) sirows[j * XR + et] = a.item_rows[it.row_begin + et];
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "n"(kAcc * XR));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  // the roles read their arguments from a shared-memory copy (fast, and it keeps
  // kernel-parameter addresses out of the non-inlined role functions)
  const Args& as = *sargs;
  if (warp == 0) {
    if (lane == 0) role_producer(as, smem, map_xg, map_attn, map_act);
  } else if (warp == 1) {
    if (lane == 0) role_mma(as, smem, tmem);
  } else if (warp < 6) {
    role_epilogue(as, smem, tmem);
  } else if (warp == 6) {
    if (lane == 0) role_helper(as, smem);
  } else {
    role_attn(as, smem);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kAcc * XR));
  }
  if (threadIdx.x == 0) {
    // every thread of this CTA is past its last barrier wait
    if (atomicAdd(a.bar + 1, 1ull) == (unsigned long long)(G - 1)) {
      for (int ph = 0; ph < P; ph++) a.grab[ph] = 0;
      atomicExch(a.bar, 0ull);
      atomicExch(a.bar + 1, 0ull);
    }
  }
}


void launch_impl(const MkLaunch& l, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(decode_mk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  if (l.B < 1 || l.B > XR) throw std::runtime_error("decode_mk: 1..16 rows");
  if (mk_phases(l.L) > 512 || l.L > 255) throw std::runtime_error("decode_mk: too many layers for the phase table");
  if (l.d % (4 * MT) || l.F % 64 || l.H * HD != l.d) throw std::runtime_error("decode_mk: unsupported shape");
  Args a{};
  for (int i = 0; i < 5; i++) a.plan[i] = l.plan[i];
  a.wmaps = (const CUtensorMap*)l.wmaps;
  a.norms = l.norms;
  a.d = l.d; a.F = l.F; a.H = l.H; a.L = l.L; a.V = l.V; a.n_text = l.n_text;
  a.eps = l.eps; a.scale_log2 = l.scale_log2;
  a.hdr = l.hdr; a.rows = (const RowMeta*)l.rows; a.items = (const AttnItem*)l.items;
  a.item_rows = (const ItemRow*)l.item_rows; a.B = l.B;
  a.embed = l.embed; a.out_tokens = l.out_tokens; a.x = l.x; a.xg = l.xg; a.ss = l.ss; a.q = l.q;
  a.attn = l.attn; a.kv_pool = l.kv_pool; a.page_elems = l.page_elems; a.rope = l.rope;
  a.partial = l.partial; a.counters = l.counters; a.apartial = l.apartial; a.acounters = l.acounters;
  a.part_keys = l.part_keys; a.logits = l.logits; a.bar = l.bar; a.trace = l.trace;
  a.grab = l.grab;
  a.flags = l.flags;
  a.fused = l.fused | (1 << MK_LM);  // lm_head always finalises in-phase (FINAL follows)
  a.pf_stages = std::max(1, std::min(kStages, l.pf_stages > 0 ? l.pf_stages : kStages));
  // cooperative launch: the grid barriers need every CTA resident, which the
  // runtime then guarantees (or rejects the launch) instead of a spin timeout
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(l.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, decode_mk_kernel,
                                             *reinterpret_cast<const CUtensorMap*>(l.map_xg.bytes),
                                             *reinterpret_cast<const CUtensorMap*>(l.map_attn.bytes),
                                             *reinterpret_cast<const CUtensorMap*>(l.map_act.bytes), a);
  if (err != cudaSuccess)
    throw std::runtime_error(std::string("decode tick: cooperative launch failed: ") + cudaGetErrorString(err));
}

}  // namespace

#if MK_TRACE
void launch_decode_mk_traced(const MkLaunch& l, cudaStream_t s) { launch_impl(l, s); }
#else
int mk_phases(int L) { return 3 + 10 * L; }  // upper bound (any fused mask)
int mk_phases(int L, int fused) {
  return 3 + L * (6 + !(fused >> MK_QKV & 1) + !(fused >> MK_O & 1) + !(fused >> MK_GU & 1) + !(fused >> MK_DOWN & 1));
}

int mk_grid() {
  static int n_sm = 0;
  if (!n_sm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  return n_sm;
}

MkPlan mk_plan(int tiles, int kb_total, int grid, int per_cta, int cap) {
  // enough chunks for ~per_cta per CTA (dynamic balance), at least 4 k-blocks
  // each, at most min(cap, 16) per tile (one load round in the reduction)
  int nc = (per_cta * grid + tiles - 1) / tiles;
  nc = std::max(1, std::min({nc, cap, 16, std::max(1, kb_total / 4)}));
  return MkPlan{tiles, kb_total, nc, tiles * nc};
}

size_t mk_partial_floats(const MkPlan* plans) {
  int chunks = 0;
  for (int i = 0; i < 5; i++) chunks = std::max(chunks, plans[i].tiles * 16);  // any plan up to 16 per tile
  return (size_t)chunks * MT * XR;
}

// the lean kernel unless a trace or a diagnostic flag is requested: the
// instrumented one (decode_mk_trace.cu) is measurably slower (larger hot loops)
void launch_decode_mk(const MkLaunch& l, cudaStream_t s) {
  if (l.trace || l.flags) launch_decode_mk_traced(l, s);
  else launch_impl(l, s);
}
#endif

}  // namespace fe
