// Row-group cascade decode attention on tensor cores (bf16 path, head_dim
// 128): the attention of the decode ticks that run the per-matrix kernel
// chain (> 16 rows: config 4's batched episodes, the background lane).
//
// Work item = (row group, page range, head).  A row group is <= 16 query rows
// connected through shared KV pages (a trunk and the branches forked off it,
// engine.cu forward()); its item walks the union of the rows' pages in chunk
// order -- every page staged ONCE per head, whichever rows share it -- with
// one online-softmax state per row and a per-page row mask (rows that do not
// hold the page see no key of it; a row's last page is cut at its valid
// count).  So a row's whole attention is normally one item and its output is
// written directly: no partials, no merge.  Only when the groups alone do not
// fill the GPU are a group's pages split into ranges ("parts"); then each part
// writes a per-row partial and the CTA completing a row's last part merges
// the parts in part order (deterministic).
//
// Staging: an NST-stage TMA ring over the pool viewed as [rows][128] bf16,
// 64 x 64 boxes with 128-byte swizzle (bank-conflict-free ldmatrix); a
// partially filled page loads only its 16-key blocks that hold valid keys.
// Each of the 4 warps owns 16 keys of every page: S = Q K^T and O += P V on
// mma.sync m16n8k16 (rows padded to 16), softmax in the exp2 domain, and a
// warp whose keys no row can see skips the page (so unloaded rows are never
// read).  The four warps' states are combined in shared memory.
#include "common.cuh"
#include "engine_internal.h"
#include "gemm_tc.h"
#include "tc_util.cuh"

#include <cuda.h>
#include <cuda_bf16.h>

namespace fe {
namespace {

constexpr int HD = 128;
constexpr int NST = 3;                         // pipeline stages (pages)
constexpr int kBox = 64 * 64 * 2;              // 8 KB: 64 keys x 64 dims
constexpr int kStage = 4 * kBox;               // K lo, K hi, V lo, V hi
constexpr int kSmem = NST * kStage + 1024 + 1024;  // + alignment slack, barriers, warp states

using namespace tc;

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// byte offset of the 16-byte chunk `c16` (0..15 over the 128 dims) of `key`
// in a stage half (K or V): two 64-dim swizzled boxes
__device__ __forceinline__ uint32_t swz(int key, int c16) {
  return (uint32_t)((c16 >> 3) * kBox + key * 128 + (((c16 & 7) ^ (key & 7)) << 4));
}

__global__ void __launch_bounds__(128)
attn_span_kernel(const __grid_constant__ CUtensorMap pool_map, const __grid_constant__ CUtensorMap pool_map16,
                 const int32_t* __restrict__ hdr,
                 const AttnItem* __restrict__ items, const ItemRow* __restrict__ item_rows,
                 const int32_t* __restrict__ item_slots, const int32_t* __restrict__ span_pages,
                 const int32_t* __restrict__ span_masks,
                 const RowMeta* __restrict__ rows, const int32_t* __restrict__ row_nspans,
                 const float* __restrict__ q, int L, int layer, int H, int d, float scale_log2,
                 float* __restrict__ partial, int* __restrict__ counters, __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + NST * kStage);
  float* ml = (float*)(full + NST);          // [4 warps][16 rows][2]
  pdl_trigger();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int h = blockIdx.y;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&pool_map) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&pool_map16) : "memory");
    for (int s = 0; s < NST; s++) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // q and this tick's K/V rows come from the QKV GEMM
  const int item = blockIdx.x;
  if (item >= hdr[1]) return;
  const AttnItem it = items[item];
  const int n_pages = it.pad[0];
  const int32_t* pages = span_pages + it.pad[1];
  const int nr = it.row_count;
  __syncthreads();

  auto issue = [&](int j) {  // page j of the span -> stage j % NST (thread 0)
    const int s = j % NST;
    const int page = pages[j];
    const int rk = (((page * L + layer) * 2 + 0) * H + h) * 64;
    const int rv = rk + H * 64;
    unsigned char* st = smem + s * kStage;
    const int vmax = (int)((uint32_t)span_masks[it.pad[1] + j] >> 16);
    if (vmax == 64) {
      mbar_expect_tx(&full[s], kStage);
      tma_load_2d(st, &pool_map, &full[s], 0, rk);
      tma_load_2d(st + kBox, &pool_map, &full[s], 64, rk);
      tma_load_2d(st + 2 * kBox, &pool_map, &full[s], 0, rv);
      tma_load_2d(st + 3 * kBox, &pool_map, &full[s], 64, rv);
    } else {
      // partially filled last page: only the 16-key blocks holding valid
      // keys; a warp whose 16 keys are past every row's valid count skips
      // the page, so the rows never loaded are never read
      const int nb = (vmax + 15) >> 4;
      mbar_expect_tx(&full[s], nb * 4 * 16 * 128);
      for (int b = 0; b < nb; b++) {
        const int o = b * 16 * 128;
        tma_load_2d(st + o, &pool_map16, &full[s], 0, rk + 16 * b);
        tma_load_2d(st + kBox + o, &pool_map16, &full[s], 64, rk + 16 * b);
        tma_load_2d(st + 2 * kBox + o, &pool_map16, &full[s], 0, rv + 16 * b);
        tma_load_2d(st + 3 * kBox + o, &pool_map16, &full[s], 64, rv + 16 * b);
      }
    }
  };
  if (tid == 0)
    for (int j = 0; j < min(NST, n_pages); j++) issue(j);

  // this lane's rows (g, g + 8) of the item and their keys on the last page
  const int ra = g, rb = g + 8;
  int rowa = -1, rowb = -1, va = 0, vb = 0, lpa = -1, lpb = -1;  // last-page position in this item
  if (ra < nr) {
    const ItemRow ir = item_rows[it.row_begin + ra];
    rowa = ir.row; va = ir.valid; lpa = item_slots[it.row_begin + ra] >> 16;
  }
  if (rb < nr) {
    const ItemRow ir = item_rows[it.row_begin + rb];
    rowb = ir.row; vb = ir.valid; lpb = item_slots[it.row_begin + rb] >> 16;
  }
  // Q fragments (A operand, k-step ks: dims 16 ks + 2t + {0,1} | + 8), exp2 domain
  uint32_t qa[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ks++) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
    if (rowa >= 0) {
      const float* qp = q + (size_t)rowa * d + h * HD + 16 * ks + 2 * t;
      a0 = *reinterpret_cast<const float2*>(qp);
      a1 = *reinterpret_cast<const float2*>(qp + 8);
    }
    if (rowb >= 0) {
      const float* qp = q + (size_t)rowb * d + h * HD + 16 * ks + 2 * t;
      b0 = *reinterpret_cast<const float2*>(qp);
      b1 = *reinterpret_cast<const float2*>(qp + 8);
    }
    const float sc = scale_log2;
    qa[ks][0] = pack2(a0.x * sc, a0.y * sc);
    qa[ks][1] = pack2(b0.x * sc, b0.y * sc);
    qa[ks][2] = pack2(a1.x * sc, a1.y * sc);
    qa[ks][3] = pack2(b1.x * sc, b1.y * sc);
  }

  float o[16][4];
#pragma unroll
  for (int nt = 0; nt < 16; nt++) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.0f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
  const int lm = lane >> 3, lrow = lane & 7;
  const int kw = 16 * warp;  // this warp's keys of every page

  for (int j = 0; j < n_pages; j++) {
    const int s = j % NST;
    mbar_wait(&full[s], (j / NST) & 1);
    const unsigned char* ks_ = smem + s * kStage;
    const unsigned char* vs_ = ks_ + 2 * kBox;
    // keys visible per row: none if the row does not hold the page, its valid
    // count on its last page, else the whole page (padded rows see nothing)
    const uint32_t pmask = (uint32_t)span_masks[it.pad[1] + j] & 0xffffu;
    const int lima = (pmask >> ra & 1) ? (j == lpa ? va : 64) : 0;
    const int limb = (pmask >> rb & 1) ? (j == lpb ? vb : 64) : 0;
    if (__any_sync(0xffffffffu, kw < max(lima, limb))) {  // keys of this warp visible to some row (warp-uniform)
      // S = Q K^T over keys kw .. kw + 15 (two n-tiles of 8)
      float sc[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; nt++) sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.0f;
#pragma unroll
      for (int kk = 0; kk < 8; kk++) {
        // matrices: (keys +0-7, dims lo8), (keys +0-7, dims hi8), (keys +8-15, lo8), (keys +8-15, hi8)
        const int key = kw + 8 * (lm >> 1) + lrow;
        const int c16 = 2 * kk + (lm & 1);
        uint32_t b0, b1, b2, b3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                     : "r"(su32(ks_ + swz(key, c16))));
        mma16816(sc[0], qa[kk], b0, b1);
        mma16816(sc[1], qa[kk], b2, b3);
      }
      float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 2; nt++) {
        const int kp = kw + 8 * nt + 2 * t;
        sc[nt][0] = kp < lima ? sc[nt][0] : -INFINITY;
        sc[nt][1] = kp + 1 < lima ? sc[nt][1] : -INFINITY;
        sc[nt][2] = kp < limb ? sc[nt][2] : -INFINITY;
        sc[nt][3] = kp + 1 < limb ? sc[nt][3] : -INFINITY;
        mxa = fmaxf(mxa, fmaxf(sc[nt][0], sc[nt][1]));
        mxb = fmaxf(mxb, fmaxf(sc[nt][2], sc[nt][3]));
      }
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
      const float na = fmaxf(m0, mxa), nb = fmaxf(m1, mxb);
      const float ua = na == -INFINITY ? 0.0f : na, ub = nb == -INFINITY ? 0.0f : nb;
      const float ca = exp2f(m0 - ua), cb = exp2f(m1 - ub);
      float sa = 0.0f, sb = 0.0f;
#pragma unroll
      for (int nt = 0; nt < 2; nt++) {
        sc[nt][0] = exp2f(sc[nt][0] - ua);
        sc[nt][1] = exp2f(sc[nt][1] - ua);
        sc[nt][2] = exp2f(sc[nt][2] - ub);
        sc[nt][3] = exp2f(sc[nt][3] - ub);
        sa += sc[nt][0] + sc[nt][1];
        sb += sc[nt][2] + sc[nt][3];
      }
      sa += __shfl_xor_sync(0xffffffffu, sa, 1);
      sa += __shfl_xor_sync(0xffffffffu, sa, 2);
      sb += __shfl_xor_sync(0xffffffffu, sb, 1);
      sb += __shfl_xor_sync(0xffffffffu, sb, 2);
      l0 = l0 * ca + sa;
      l1 = l1 * cb + sb;
      m0 = na;
      m1 = nb;
#pragma unroll
      for (int nt = 0; nt < 16; nt++) {
        o[nt][0] *= ca;
        o[nt][1] *= ca;
        o[nt][2] *= cb;
        o[nt][3] *= cb;
      }
      // O += P V over the warp's 16 keys: V^T fragments by ldmatrix.x4.trans
      uint32_t pa4[4];
      pa4[0] = pack2(sc[0][0], sc[0][1]);
      pa4[1] = pack2(sc[0][2], sc[0][3]);
      pa4[2] = pack2(sc[1][0], sc[1][1]);
      pa4[3] = pack2(sc[1][2], sc[1][3]);
      const int vkey = kw + lrow + 8 * (lm & 1);
#pragma unroll
      for (int np = 0; np < 8; np++) {
        const int c16 = 2 * np + (lm >> 1);
        uint32_t b0, b1, b2, b3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                     : "r"(su32(vs_ + swz(vkey, c16))));
        mma16816(o[2 * np], pa4, b0, b1);
        mma16816(o[2 * np + 1], pa4, b2, b3);
      }
    }
    __syncthreads();  // every warp is done with stage s
    if (tid == 0 && j + NST < n_pages) issue(j + NST);
  }

  // ---- combine the four warps' states (rows g, g + 8 of every warp)
  if (t == 0) {
    ml[(warp * 16 + ra) * 2 + 0] = m0;
    ml[(warp * 16 + ra) * 2 + 1] = l0;
    ml[(warp * 16 + rb) * 2 + 0] = m1;
    ml[(warp * 16 + rb) * 2 + 1] = l1;
  }
  __syncthreads();
  float Ma = -INFINITY, Mb = -INFINITY;
#pragma unroll
  for (int w = 0; w < 4; w++) {
    Ma = fmaxf(Ma, ml[(w * 16 + ra) * 2]);
    Mb = fmaxf(Mb, ml[(w * 16 + rb) * 2]);
  }
  const float Ua = Ma == -INFINITY ? 0.0f : Ma, Ub = Mb == -INFINITY ? 0.0f : Mb;
  const float wa = exp2f(m0 - Ua), wb = exp2f(m1 - Ub);
  float* red = reinterpret_cast<float*>(smem);  // [4 warps][16 rows][128] (the ring is drained)
#pragma unroll
  for (int nt = 0; nt < 16; nt++) {
    const int dim = 8 * nt + 2 * t;
    *reinterpret_cast<float2*>(red + (warp * 16 + ra) * HD + dim) = make_float2(o[nt][0] * wa, o[nt][1] * wa);
    *reinterpret_cast<float2*>(red + (warp * 16 + rb) * HD + dim) = make_float2(o[nt][2] * wb, o[nt][3] * wb);
  }
  __syncthreads();
  // thread -> (row r = tid / 8, dims 16 (tid % 8) .. + 15)
  {
    const int r = tid >> 3, d0 = 16 * (tid & 7);
    if (r < nr) {
      const ItemRow ir = item_rows[it.row_begin + r];
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < 4; w++) M = fmaxf(M, ml[(w * 16 + r) * 2]);
      float Lr = 0.0f;
#pragma unroll
      for (int w = 0; w < 4; w++)  // a warp (or the whole part) that saw no key of the row has m = -inf, l = 0
        if (ml[(w * 16 + r) * 2 + 1] > 0.0f) Lr += ml[(w * 16 + r) * 2 + 1] * exp2f(ml[(w * 16 + r) * 2] - M);
      float acc[16];
#pragma unroll
      for (int e = 0; e < 16; e++) acc[e] = 0.0f;
#pragma unroll
      for (int w = 0; w < 4; w++) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          const float4 v = *reinterpret_cast<const float4*>(red + (w * 16 + r) * HD + d0 + e);
          acc[e] += v.x; acc[e + 1] += v.y; acc[e + 2] += v.z; acc[e + 3] += v.w;
        }
      }
      if (row_nspans[ir.row] == 1) {
        const float inv = 1.0f / Lr;
        __nv_bfloat16* dst = out + (size_t)ir.row * d + h * HD + d0;
        uint32_t w4[8];
#pragma unroll
        for (int e = 0; e < 8; e++) w4[e] = pack2(acc[2 * e] * inv, acc[2 * e + 1] * inv);
        *reinterpret_cast<uint4*>(dst) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        *reinterpret_cast<uint4*>(dst + 8) = make_uint4(w4[4], w4[5], w4[6], w4[7]);
      } else {
        const RowMeta m = rows[ir.row];
        float* pp = partial + ((size_t)(m.chunk_base + (item_slots[it.row_begin + r] & 0xffff)) * H + h) * (HD + 2);
        if ((tid & 7) == 0) { pp[0] = M; pp[1] = Lr; }
#pragma unroll
        for (int e = 0; e < 16; e++) pp[2 + d0 + e] = acc[e];
      }
    }
  }
  // ---- fused merge: the CTA delivering a row's last span merges its slots
  __syncthreads();
  __threadfence();
  for (int r = warp; r < nr; r += 4) {
    const ItemRow ir = item_rows[it.row_begin + r];
    const int ns = row_nspans[ir.row];
    if (ns == 1) continue;
    int prev = 0;
    if (lane == 0) prev = atomicAdd(&counters[ir.row * H + h], 1);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != ns - 1) continue;
    if (lane == 0) counters[ir.row * H + h] = 0;  // ready for the next launch
    __threadfence();
    const RowMeta m = rows[ir.row];
    const float* base = partial + ((size_t)m.chunk_base * H + h) * (HD + 2);
    const size_t stride = (size_t)H * (HD + 2);
    float M = -INFINITY;
    for (int c = 0; c < ns; c++) M = fmaxf(M, __ldcg(base + c * stride));
    float Lr = 0.0f, acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int c = 0; c < ns; c++) {
      const float mc = __ldcg(base + c * stride);
      if (mc == -INFINITY) continue;  // a part holding none of the row's pages
      const float wgt = exp2f(mc - M);
      Lr += wgt * __ldcg(base + c * stride + 1);
      const float2 v0 = __ldcg(reinterpret_cast<const float2*>(base + c * stride + 2 + 4 * lane));
      const float2 v1 = __ldcg(reinterpret_cast<const float2*>(base + c * stride + 4 + 4 * lane));
      acc[0] += wgt * v0.x; acc[1] += wgt * v0.y; acc[2] += wgt * v1.x; acc[3] += wgt * v1.y;
    }
    const float inv = 1.0f / Lr;
    __nv_bfloat16* dst = out + (size_t)ir.row * d + h * HD + 4 * lane;
    *reinterpret_cast<uint2*>(dst) = make_uint2(pack2(acc[0] * inv, acc[1] * inv), pack2(acc[2] * inv, acc[3] * inv));
  }
}

}  // namespace

int g_span_dbg = 0;  // engine option "span_dbg" (unused: diagnostics hook)

void launch_span_attention(const Fwd& f, const ModelDims& m, const TmaMap& pool_map, const TmaMap& pool_map16,
                           const float* q, int layer, float* partial, void* out, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attn_span_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  if (f.item_cap <= 0) return;
  launch_k(attn_span_kernel, dim3(f.item_cap, m.H), dim3(128), (size_t)kSmem, s,
           *reinterpret_cast<const CUtensorMap*>(pool_map.bytes),
           *reinterpret_cast<const CUtensorMap*>(pool_map16.bytes), f.hdr, f.items, f.item_rows, f.item_slots,
           f.span_pages, f.span_masks, f.rows, f.row_nspans, q, m.L, layer, m.H, m.d, m.attn_scale * 1.4426950408889634f,
           partial, f.attn_counters, (__nv_bfloat16*)out);
}

}  // namespace fe
