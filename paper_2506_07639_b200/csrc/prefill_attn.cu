// Causal prefill attention on tensor cores (bf16 path): the rows of a
// prefill forward are runs of consecutive positions of one or more sequences
// (a trunk prefill, or every trunk of a batched-episode timestep), cut into
// 64-row query tiles (engine.cu forward(): PrefillTile) attending over their
// sequence's paged K/V.
//
// Grid (query tiles, heads); 4 warps, 16 query rows each.  Per KV
// page (64 keys): K and V staged by cp.async into a double buffer (rows 256 B,
// 16-byte chunks XOR-swizzled by key & 7), S = Q K^T on mma.sync m16n8k16
// (Q scaled to the exp2 domain, head dims permuted identically in Q and K so a
// K fragment is one 16-byte load), causal mask, online softmax (running max /
// sum per row), O += P V with V fragments from ldmatrix.x4.trans.  Output: the
// bf16 attention rows the O projection consumes.
//
// Replaces the CUDA-core cascade kernel for prefill (one warp per query row,
// measured 187 us per layer for a 512-row chunk).
#include "common.cuh"
#include "engine_internal.h"

#include <cuda_bf16.h>

namespace fe {
namespace {

constexpr int HD = 128;
constexpr int QT = 64;                        // query rows per CTA
constexpr int kKV = FE_PAGE * HD * 2;         // 16 KB: one K or V page tile
constexpr int kSmem = 2 * 2 * kKV;            // double-buffered K + V

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

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

// stage K and V of one (page, layer, head) for keys [0, fill): 128 threads
__device__ __forceinline__ void stage(unsigned char* buf, const __nv_bfloat16* kg, const __nv_bfloat16* vg, int fill,
                                      int tid) {
  const int vpad = (fill + 15) & ~15;  // V rows up to the 16-key step are zero-filled
  for (int x = tid; x < vpad * 16; x += 128) {
    const int key = x >> 4, c = x & 15;
    const uint32_t so = (uint32_t)(key * 256 + ((c ^ (key & 7)) << 4));
    const bool in = key < fill;
    const int keyc = in ? key : 0;
    if (in)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(buf + so)),
                   "l"(kg + (size_t)keyc * HD + c * 8) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s32(buf + kKV + so)),
                 "l"(vg + (size_t)keyc * HD + c * 8), "r"(in ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(128) prefill_attn_kernel(const PrefillTile* __restrict__ tiles,
                                                           const int32_t* __restrict__ ptab,
                                                           const float* __restrict__ q,
                                                           const __nv_bfloat16* __restrict__ pool, size_t page_elems,
                                                           size_t layer_off, int H, int d, float scale_log2,
                                                           __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  pdl_trigger();
  pdl_wait();  // q and the K/V pages come from the QKV GEMM before this kernel
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int h = blockIdx.y;
  const PrefillTile tile = tiles[blockIdx.x];
  const int32_t* pages = ptab + tile.pages;          // the tile's sequence page table
  const int pos0 = tile.pos0, n_rows = tile.n;       // tile rows: forward rows row0 .., positions pos0 ..
  const int wrow0 = 16 * warp;                       // first tile-local query row of the warp
  const int seq_len = pos0 + n_rows;                 // keys any row of the tile can see
  const int n_pages = (seq_len - 1) / FE_PAGE + 1;
  const int ra = wrow0 + g, rb = wrow0 + g + 8;      // this lane's tile-local rows
  const int pa = pos0 + ra, pb = pos0 + rb;          // their positions
  const size_t fra = (size_t)(tile.row0 + ra), frb = (size_t)(tile.row0 + rb);  // forward rows

  auto kv_src = [&](int c, const __nv_bfloat16** kg, const __nv_bfloat16** vg, int* fill) {
    *kg = pool + (size_t)pages[c] * page_elems + layer_off + (size_t)h * FE_PAGE * HD;
    *vg = *kg + (size_t)H * FE_PAGE * HD;
    *fill = min(FE_PAGE, seq_len - c * FE_PAGE);
  };
  {
    const __nv_bfloat16 *kg, *vg;
    int fill;
    kv_src(0, &kg, &vg, &fill);
    stage(smem, kg, vg, fill, tid);
  }

  // Q fragments (k-step 2i + j: dims 32i + 8t + 4j + {0,1} | {2,3}), exp2 domain
  uint32_t qa[8][4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    float4 f[4];
#pragma unroll
    for (int u = 0; u < 4; u++) f[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ra < n_rows) {
      const float* qp = q + fra * d + h * HD + 32 * i + 8 * t;
      f[0] = *reinterpret_cast<const float4*>(qp);
      f[1] = *reinterpret_cast<const float4*>(qp + 4);
    }
    if (rb < n_rows) {
      const float* qp = q + frb * d + h * HD + 32 * i + 8 * t;
      f[2] = *reinterpret_cast<const float4*>(qp);
      f[3] = *reinterpret_cast<const float4*>(qp + 4);
    }
    const float sc = scale_log2;
    qa[2 * i][0] = pack2(f[0].x * sc, f[0].y * sc);
    qa[2 * i][1] = pack2(f[2].x * sc, f[2].y * sc);
    qa[2 * i][2] = pack2(f[0].z * sc, f[0].w * sc);
    qa[2 * i][3] = pack2(f[2].z * sc, f[2].w * sc);
    qa[2 * i + 1][0] = pack2(f[1].x * sc, f[1].y * sc);
    qa[2 * i + 1][1] = pack2(f[3].x * sc, f[3].y * sc);
    qa[2 * i + 1][2] = pack2(f[1].z * sc, f[1].w * sc);
    qa[2 * i + 1][3] = pack2(f[3].z * sc, f[3].w * sc);
  }

  float o[16][4];
#pragma unroll
  for (int nt = 0; nt < 16; nt++) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.0f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.0f, l1 = 0.0f;
  const int warp_last_pos = pos0 + min(n_rows - 1, wrow0 + 15);
  const int lm = lane >> 3, lrow = lane & 7;

  for (int c = 0; c < n_pages; c++) {
    if (c + 1 < n_pages) {  // prefetch the next page into the other buffer
      const __nv_bfloat16 *kg, *vg;
      int fill;
      kv_src(c + 1, &kg, &vg, &fill);
      stage(smem + ((c + 1) & 1) * 2 * kKV, kg, vg, fill, tid);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const unsigned char* ks = smem + (c & 1) * 2 * kKV;
    const unsigned char* vs = ks + kKV;
    const int kbase = c * FE_PAGE;
    if (kbase <= warp_last_pos) {  // some key of the page is visible to some row of the warp
      float s[8][4];
#pragma unroll
      for (int nt = 0; nt < 8; nt++) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.0f;
#pragma unroll
      for (int i = 0; i < 4; i++) {
        uint4 kv[8];
#pragma unroll
        for (int nt = 0; nt < 8; nt++)
          kv[nt] = *reinterpret_cast<const uint4*>(ks + (size_t)(8 * nt + g) * HD * 2 + (((4 * i + t) ^ g) << 4));
#pragma unroll
        for (int nt = 0; nt < 8; nt++) {
          if (kbase + 8 * nt > warp_last_pos) continue;
          mma16816(s[nt], qa[2 * i], kv[nt].x, kv[nt].y);
          mma16816(s[nt], qa[2 * i + 1], kv[nt].z, kv[nt].w);
        }
      }
      // causal mask + online softmax (rows a: c0, c1; b: c2, c3)
      float mxa = -INFINITY, mxb = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; nt++) {
        const int kp = kbase + 8 * nt + 2 * t;
        s[nt][0] = (kp <= pa && ra < n_rows) ? s[nt][0] : -INFINITY;
        s[nt][1] = (kp + 1 <= pa && ra < n_rows) ? s[nt][1] : -INFINITY;
        s[nt][2] = (kp <= pb && rb < n_rows) ? s[nt][2] : -INFINITY;
        s[nt][3] = (kp + 1 <= pb && rb < n_rows) ? s[nt][3] : -INFINITY;
        mxa = fmaxf(mxa, fmaxf(s[nt][0], s[nt][1]));
        mxb = fmaxf(mxb, fmaxf(s[nt][2], s[nt][3]));
      }
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 1));
      mxa = fmaxf(mxa, __shfl_xor_sync(0xffffffffu, mxa, 2));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 1));
      mxb = fmaxf(mxb, __shfl_xor_sync(0xffffffffu, mxb, 2));
      const float na = fmaxf(m0, mxa), nb = fmaxf(m1, mxb);
      const float ua = na == -INFINITY ? 0.0f : na, ub = nb == -INFINITY ? 0.0f : nb;  // fully masked rows
      const float ca = exp2f(m0 - ua), cb = exp2f(m1 - ub);                              // exp2(-inf) = 0
      float sa = 0.0f, sb = 0.0f;
#pragma unroll
      for (int nt = 0; nt < 8; nt++) {
        s[nt][0] = exp2f(s[nt][0] - ua);
        s[nt][1] = exp2f(s[nt][1] - ua);
        s[nt][2] = exp2f(s[nt][2] - ub);
        s[nt][3] = exp2f(s[nt][3] - ub);
        sa += s[nt][0] + s[nt][1];
        sb += s[nt][2] + s[nt][3];
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
      // O += P V: V fragments by ldmatrix.x4.trans (keys 16kk + {0-7, 8-15}) x (dims 16np + {0-7, 8-15})
#pragma unroll
      for (int kk = 0; kk < 4; kk++) {
        if (kbase + 16 * kk > warp_last_pos) break;
        uint32_t pa4[4];
        pa4[0] = pack2(s[2 * kk][0], s[2 * kk][1]);
        pa4[1] = pack2(s[2 * kk][2], s[2 * kk][3]);
        pa4[2] = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
        pa4[3] = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
        const int key = 16 * kk + lrow + 8 * (lm & 1);
#pragma unroll
        for (int np = 0; np < 8; np++) {
          const int cc = 2 * np + (lm >> 1);
          uint32_t b0, b1, b2, b3;
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                       : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                       : "r"(s32(vs + (size_t)key * HD * 2 + ((cc ^ (key & 7)) << 4))));
          mma16816(o[2 * np], pa4, b0, b1);
          mma16816(o[2 * np + 1], pa4, b2, b3);
        }
      }
    }
    __syncthreads();  // the buffer is restaged two pages later
  }
  const float ia = l0 > 0.0f ? 1.0f / l0 : 0.0f, ib = l1 > 0.0f ? 1.0f / l1 : 0.0f;
#pragma unroll
  for (int nt = 0; nt < 16; nt++) {
    const int dim = 8 * nt + 2 * t;
    if (ra < n_rows)
      *reinterpret_cast<uint32_t*>(out + fra * d + h * HD + dim) = pack2(o[nt][0] * ia, o[nt][1] * ia);
    if (rb < n_rows)
      *reinterpret_cast<uint32_t*>(out + frb * d + h * HD + dim) = pack2(o[nt][2] * ib, o[nt][3] * ib);
  }
}

}  // namespace

void launch_prefill_attention(const Fwd& f, const ModelDims& m, const float* q, const void* pool, int layer,
                              void* out, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  const size_t pe = kv_page_elems(m);
  const size_t lo = (size_t)layer * 2 * m.H * FE_PAGE * m.hd;
  const dim3 grid(f.n_ptiles, m.H);
  launch_k(prefill_attn_kernel, grid, dim3(128), (size_t)kSmem, s, f.ptiles, f.ptab, q,
           (const __nv_bfloat16*)pool, pe, lo, m.H, m.d, m.attn_scale * 1.4426950408889634f, (__nv_bfloat16*)out);
}

}  // namespace fe
