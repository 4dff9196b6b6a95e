// Decode/prefill kernels of the Fast-ECoT B200 engine (sm_100a).
//
//   embed          token / vision-row gather into the fp32 residual stream
//   rmsnorm        canonical RMSNorm, writes the GEMV staging dtype
//   gemv<EPI>      HBM-streaming batched GEMV: one warp owns 4 weight rows,
//                  16-byte non-allocating weight loads, activations staged in
//                  shared memory, canonical per-lane partials + xor butterfly;
//                  fused epilogues: RoPE + paged-KV append (QKV), residual add
//                  (O, down), SiLU*up (gate/up), greedy argmax partials (lm_head)
//   attention      cascade decode/prefill attention over 64-token KV pages:
//                  one CTA per (page, head) stages the page's K/V once with a
//                  1-D TMA bulk copy and serves every query row whose block
//                  table maps that chunk to the page; warp-level two-pass
//                  softmax per chunk; in-order LSE merge of chunk partials
//   finalize       argmax partial reduction -> token feedback
//
// Arithmetic follows DESIGN.md §3 exactly (compiled with --fmad=false).
#include "common.cuh"
#include "engine_internal.h"

#include <algorithm>

namespace fe {

bool g_pdl = true;

// ---------------------------------------------------------------- init ----
template <typename WT>
__global__ void init_linear_kernel(WT* w, uint64_t key, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    w[i] = Elem<WT>::from_f(__fmul_rn(centered(key, i), kLinearMult));
}

__global__ void init_norm_kernel(float* w, uint64_t key, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    w[i] = __fadd_rn(1.0f, __fmul_rn(centered(key, i), kNormMult));
}

void launch_init_linear(int dtype, void* w, uint64_t key, size_t n, cudaStream_t s) {
  if (dtype == F32) init_linear_kernel<float><<<148 * 16, 256, 0, s>>>((float*)w, key, n);
  else init_linear_kernel<__nv_bfloat16><<<148 * 16, 256, 0, s>>>((__nv_bfloat16*)w, key, n);
}
void launch_init_norm(float* w, uint64_t key, size_t n, cudaStream_t s) {
  init_norm_kernel<<<64, 256, 0, s>>>(w, key, n);
}

// --------------------------------------------------------------- embed ----
template <typename WT>
__global__ void embed_kernel(Fwd f, int d, const WT* embed, const int32_t* out_tokens, float* x) {
  pdl_trigger();
  pdl_wait();
  const RowMeta m = f.rows[blockIdx.x];
  float* xr = x + (size_t)blockIdx.x * d;
  if (m.vis_row >= 0) {
    const uint64_t base = (uint64_t)m.vis_row * d;
    const uint64_t key = f.vision_keys ? f.vision_keys[m.pad] : f.vision_key;
    if (f.vis_ptrs) {  // the vision tower's rows
      const float* src = reinterpret_cast<const float*>(key) + base;
      for (int k = threadIdx.x; k < d; k += blockDim.x) xr[k] = src[k];
    } else {
      for (int k = threadIdx.x; k < d; k += blockDim.x)
        xr[k] = __fmul_rn(centered(key, base + k), kVisionMult);
    }
  } else {
    const int tok = m.tok >= 0 ? m.tok : out_tokens[m.tok_src];
    const WT* e = embed + (size_t)tok * d;
    for (int k = threadIdx.x; k < d; k += blockDim.x) xr[k] = Elem<WT>::to_f(e[k]);
  }
}

void launch_embed(int dtype, const Fwd& f, const ModelDims& m, const void* embed, const int32_t* out_tokens,
                  float* x, cudaStream_t s) {
  if (f.n_rows == 0) return;
  if (dtype == F32) embed_kernel<float><<<f.n_rows, 256, 0, s>>>(f, m.d, (const float*)embed, out_tokens, x);
  else embed_kernel<__nv_bfloat16><<<f.n_rows, 256, 0, s>>>(f, m.d, (const __nv_bfloat16*)embed, out_tokens, x);
}

// ------------------------------------------------------------- rmsnorm ----
// One warp per row: ss = canonical dot(x, x); r = 1/sqrt(ss/d + eps);
// out = (x * r) * w, stored in the staging dtype.
template <typename XT>
__global__ void rmsnorm_kernel(const float* __restrict__ x, const float* __restrict__ w, XT* __restrict__ out,
                               int n, int d, int ld_out, float eps, const int32_t* __restrict__ row_index) {
  pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const int src = row_index ? row_index[warp] : warp;
  const float* xr = x + (size_t)src * d;
  float a = 0.0f;
  for (int j = 0; j < d; j += 128) {
    const int k = j + 4 * lane;
    if (k < d) {
      const float4 v = *reinterpret_cast<const float4*>(xr + k);
      a = __fmaf_rn(v.x, v.x, a);
      a = __fmaf_rn(v.y, v.y, a);
      a = __fmaf_rn(v.z, v.z, a);
      a = __fmaf_rn(v.w, v.w, a);
    }
  }
  const float ss = xor_butterfly(a);
  const float r = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)d), eps)));
  XT* o = out + (size_t)warp * ld_out;
  for (int k = lane; k < d; k += 32) o[k] = Elem<XT>::from_f(__fmul_rn(__fmul_rn(xr[k], r), w[k]));
}

// bf16 mode: one 256-thread block per row, 8 elements per thread-step,
// block-wide sum of squares (free reduction order).
__global__ void __launch_bounds__(256)
rmsnorm_bf16_kernel(const float* __restrict__ x, const float* __restrict__ w, __nv_bfloat16* __restrict__ out,
                    int d, int ld_out, float eps, const int32_t* __restrict__ row_index) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8];
  const int row = blockIdx.x;
  const int src = row_index ? row_index[row] : row;
  const float* xr = x + (size_t)src * d;
  float ss = 0.0f;
  for (int k = 8 * threadIdx.x; k < d; k += 8 * blockDim.x) {
    const float4 a = *reinterpret_cast<const float4*>(xr + k);
    const float4 b = *reinterpret_cast<const float4*>(xr + k + 4);
    ss = fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, fmaf(a.w, a.w, ss))));
    ss = fmaf(b.x, b.x, fmaf(b.y, b.y, fmaf(b.z, b.z, fmaf(b.w, b.w, ss))));
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int i = 0; i < 8; i++) tot += red[i];
  const float r = rsqrtf(tot / (float)d + eps);
  __nv_bfloat16* o = out + (size_t)row * ld_out;
  for (int k = 8 * threadIdx.x; k < d; k += 8 * blockDim.x) {
    const float4 a = *reinterpret_cast<const float4*>(xr + k);
    const float4 b = *reinterpret_cast<const float4*>(xr + k + 4);
    const float4 wa = *reinterpret_cast<const float4*>(w + k);
    const float4 wb = *reinterpret_cast<const float4*>(w + k + 4);
    __nv_bfloat162 v[4];
    v[0] = __floats2bfloat162_rn(a.x * r * wa.x, a.y * r * wa.y);
    v[1] = __floats2bfloat162_rn(a.z * r * wa.z, a.w * r * wa.w);
    v[2] = __floats2bfloat162_rn(b.x * r * wb.x, b.y * r * wb.y);
    v[3] = __floats2bfloat162_rn(b.z * r * wb.z, b.w * r * wb.w);
    *reinterpret_cast<uint4*>(o + k) = *reinterpret_cast<const uint4*>(v);
  }
}

void launch_rmsnorm(int dtype, const float* x, const float* w, void* out, int n_rows, int d, int ld_out,
                    float eps, const int32_t* row_index, cudaStream_t s) {
  if (n_rows == 0) return;
  if (dtype == BF16) {
    launch_k(rmsnorm_bf16_kernel, dim3(n_rows), dim3(256), 0, s, x, w, (__nv_bfloat16*)out, d, ld_out, eps, row_index);
    return;
  }
  const int blocks = (n_rows + 7) / 8;
  if (dtype == F32) launch_k(rmsnorm_kernel<float>, dim3(blocks), dim3(256), 0, s, x, w, (float*)out, n_rows, d, ld_out, eps, row_index);
  else launch_k(rmsnorm_kernel<__nv_bfloat16>, dim3(blocks), dim3(256), 0, s, x, w, (__nv_bfloat16*)out, n_rows, d, ld_out, eps, row_index);
}

// ---------------------------------------------------------------- gemv ----
enum Epi { EPI_STORE = 0, EPI_QKV = 1, EPI_RESID = 2, EPI_SWIGLU = 3, EPI_ARGMAX = 4 };

struct GemvArgs {
  const void* W;
  int N, K;
  const void* x;           // [rows][K] staging dtype
  int n_rows;
  float* y;                // STORE: [rows][N]; RESID: residual stream [rows][N]
  void* act;               // SWIGLU: [rows][N/2] staging dtype
  // QKV
  float* q;                // [rows][d]
  void* kv_pool;
  size_t page_elems, layer_off;
  const float* rope;
  int H, hd, d;
  const RowMeta* rows;
  // ARGMAX
  const int32_t* head_rows;
  unsigned long long* part_keys;
  float* logits;
  int V, n_text;
};

constexpr int kGemvWarps = 8;

template <typename WT, typename XT, int BMAX, int EPI>
__global__ void __launch_bounds__(kGemvWarps * 32)
gemv_kernel(const GemvArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = Elem<WT>::kVec;          // elements per 16-byte weight vector
  constexpr int KC = 32 * V * 8;             // K chunk staged per pass
  constexpr int XV = 16 / sizeof(XT);        // staging elements per 16 bytes
  static_assert(V == XV, "weights and staging must share the vector width");
  extern __shared__ __align__(16) unsigned char smem[];
  XT* xs = reinterpret_cast<XT*>(smem);      // [BMAX][KC]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = blockIdx.x * kGemvWarps + warp;
  const int row0 = blockIdx.y * BMAX;
  const int B = min(BMAX, a.n_rows - row0);
  const bool active = quad < (a.N >> 2);

  int wrow[4];
  if (EPI == EPI_QKV) {
    const int per = a.hd >> 2, sh = quad / per, pp = 2 * (quad % per);
    const int sec = sh / a.H, h = sh % a.H;
    wrow[0] = sec * a.d + h * a.hd + pp;
    wrow[1] = wrow[0] + (a.hd >> 1);
    wrow[2] = wrow[0] + 1;
    wrow[3] = wrow[1] + 1;
  } else if (EPI == EPI_SWIGLU) {
    const int F = a.N >> 1;
    wrow[0] = 2 * quad; wrow[1] = F + 2 * quad; wrow[2] = 2 * quad + 1; wrow[3] = F + 2 * quad + 1;
  } else {
#pragma unroll
    for (int r = 0; r < 4; r++) wrow[r] = 4 * quad + r;
  }
  const WT* W = reinterpret_cast<const WT*>(a.W);
  const XT* X = reinterpret_cast<const XT*>(a.x);

  float acc[4][BMAX];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int b = 0; b < BMAX; b++) acc[r][b] = 0.0f;

  for (int k0 = 0; k0 < a.K; k0 += KC) {
    const int kc = min(KC, a.K - k0);
    __syncthreads();
    {  // stage x[row0 .. row0+B)[k0 .. k0+kc) into shared memory, 16 B per thread-step
      const int vecs = kc / XV;
      for (int i = threadIdx.x; i < B * vecs; i += blockDim.x) {
        const int b = i / vecs, v = i % vecs;
        reinterpret_cast<uint4*>(xs + b * KC)[v] =
            *reinterpret_cast<const uint4*>(X + (size_t)(row0 + b) * a.K + k0 + v * XV);
      }
    }
    __syncthreads();
    if (!active) continue;
#pragma unroll
    for (int it0 = 0; it0 < 8; it0 += 4) {
      uint4 wv[4][4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int k = (it0 + u) * 32 * V + lane * V;
#pragma unroll
        for (int r = 0; r < 4; r++)
          wv[u][r] = k < kc ? ldg_stream(W + (size_t)wrow[r] * a.K + k0 + k) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int k = (it0 + u) * 32 * V + lane * V;
        if (k >= kc) continue;
        float wf[4][V];
#pragma unroll
        for (int r = 0; r < 4; r++) unpack(wv[u][r], wf[r]);
#pragma unroll
        for (int b = 0; b < BMAX; b++) {
          if (b >= B) break;
          float xf[V];
          unpack(*reinterpret_cast<const uint4*>(xs + b * KC + k), xf);
#pragma unroll
          for (int r = 0; r < 4; r++)
#pragma unroll
            for (int c = 0; c < V; c++) acc[r][b] = __fmaf_rn(wf[r][c], xf[c], acc[r][b]);
        }
      }
    }
  }

  // ---- epilogue: butterfly every partial, then lane b finishes batch row b
  unsigned long long best[BMAX];
#pragma unroll
  for (int b = 0; b < BMAX; b++) best[b] = 0ull;
  if (active) {
#pragma unroll
    for (int b = 0; b < BMAX; b++) {
      if (b >= B) break;
      float s[4];
#pragma unroll
      for (int r = 0; r < 4; r++) s[r] = xor_butterfly(acc[r][b]);
      const int row = row0 + b;
      if (EPI == EPI_STORE) {
        if (lane == 0) {
#pragma unroll
          for (int r = 0; r < 4; r++) a.y[(size_t)row * a.N + wrow[r]] = s[r];
        }
      } else if (EPI == EPI_RESID) {
        if (lane == 0) {
          float4* p = reinterpret_cast<float4*>(a.y + (size_t)row * a.N + wrow[0]);
          float4 v = *p;
          v.x = __fadd_rn(v.x, s[0]); v.y = __fadd_rn(v.y, s[1]);
          v.z = __fadd_rn(v.z, s[2]); v.w = __fadd_rn(v.w, s[3]);
          *p = v;
        }
      } else if (EPI == EPI_SWIGLU) {
        if (lane == 0) {
          XT* o = reinterpret_cast<XT*>(a.act) + (size_t)row * (a.N >> 1) + 2 * quad;
          o[0] = Elem<XT>::from_f(silu_mul(s[0], s[1]));
          o[1] = Elem<XT>::from_f(silu_mul(s[2], s[3]));
        }
      } else if (EPI == EPI_QKV) {
        if (lane == 0) {
          const RowMeta m = a.rows[row];
          const int per = a.hd >> 2, sh = quad / per, pp = 2 * (quad % per);
          const int sec = sh / a.H, h = sh % a.H, half = a.hd >> 1;
          float o[4] = {s[0], s[1], s[2], s[3]};
          if (sec < 2) {
            const float* cs = a.rope + (size_t)m.pos * a.hd;
#pragma unroll
            for (int t = 0; t < 2; t++) {
              const float c = cs[pp + t], sn = cs[half + pp + t];
              const float x1 = s[2 * t], x2 = s[2 * t + 1];
              o[2 * t] = __fmaf_rn(x1, c, -__fmul_rn(x2, sn));
              o[2 * t + 1] = __fmaf_rn(x2, c, __fmul_rn(x1, sn));
            }
          }
          if (sec == 0) {
            float* qr = a.q + (size_t)row * a.d + h * a.hd;
            qr[pp] = o[0]; qr[pp + half] = o[1]; qr[pp + 1] = o[2]; qr[pp + 1 + half] = o[3];
          } else {
            XT* kv = reinterpret_cast<XT*>(a.kv_pool) + (size_t)m.kv_page * a.page_elems + a.layer_off +
                     ((size_t)((sec - 1) * a.H + h) * FE_PAGE + m.kv_slot) * a.hd;
            kv[pp] = Elem<XT>::from_f(o[0]); kv[pp + half] = Elem<XT>::from_f(o[1]);
            kv[pp + 1] = Elem<XT>::from_f(o[2]); kv[pp + 1 + half] = Elem<XT>::from_f(o[3]);
          }
        }
      } else if (EPI == EPI_ARGMAX) {
        const RowMeta m = a.rows[a.head_rows[row]];
        unsigned long long k = 0ull;
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int n = wrow[r];
          if (n < a.n_text) k = max(k, argmax_key(s[r], n));
        }
        best[b] = k;
        if (m.logit_row >= 0 && lane == 0) {
#pragma unroll
          for (int r = 0; r < 4; r++) a.logits[(size_t)m.logit_row * a.V + wrow[r]] = s[r];
        }
      }
    }
  }
  if (EPI == EPI_ARGMAX) {
    __syncthreads();
    unsigned long long* red = reinterpret_cast<unsigned long long*>(smem);  // [warps][BMAX]
    if (lane == 0)
#pragma unroll
      for (int b = 0; b < BMAX; b++) red[warp * BMAX + b] = best[b];
    __syncthreads();
    if (threadIdx.x < B) {
      unsigned long long k = 0ull;
      for (int w = 0; w < kGemvWarps; w++) k = max(k, red[w * BMAX + threadIdx.x]);
      a.part_keys[(size_t)(row0 + threadIdx.x) * gridDim.x + blockIdx.x] = k;
    }
  }
}

template <typename WT, typename XT, int EPI>
static void gemv_dispatch(const GemvArgs& a, cudaStream_t s) {
  if (a.n_rows <= 0) return;
  constexpr int V = Elem<WT>::kVec;
  constexpr int KC = 32 * V * 8;
  const int gx = ((a.N >> 2) + kGemvWarps - 1) / kGemvWarps;
  auto go = [&](auto bmax_tag) {
    constexpr int BM = decltype(bmax_tag)::value;
    const size_t smem = std::max<size_t>((size_t)BM * KC * sizeof(XT), (size_t)kGemvWarps * BM * 8);
    auto kern = gemv_kernel<WT, XT, BM, EPI>;
    static bool configured = false;  // per instantiation
    if (!configured) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured = true;
    }
    dim3 grid(gx, (a.n_rows + BM - 1) / BM);
    launch_k(kern, grid, dim3(kGemvWarps * 32), smem, s, a);
  };
  if (a.n_rows <= 1) go(std::integral_constant<int, 1>{});
  else if (a.n_rows <= 2) go(std::integral_constant<int, 2>{});
  else if (a.n_rows <= 4) go(std::integral_constant<int, 4>{});
  else if (a.n_rows <= 8) go(std::integral_constant<int, 8>{});
  else go(std::integral_constant<int, 16>{});
}

template <int EPI>
static void gemv_any(int dtype, const GemvArgs& a, cudaStream_t s) {
  if (dtype == F32) gemv_dispatch<float, float, EPI>(a, s);
  else gemv_dispatch<__nv_bfloat16, __nv_bfloat16, EPI>(a, s);
}

size_t kv_page_elems(const ModelDims& m) { return (size_t)m.L * 2 * m.H * FE_PAGE * m.hd; }

int lm_head_ctas(const ModelDims& m) { return ((m.V >> 2) + kGemvWarps - 1) / kGemvWarps; }

void launch_qkv(int dtype, const Fwd& f, const ModelDims& m, const void* w, const void* xn, float* q,
                void* kv_pool, int layer, const float* rope, cudaStream_t s) {
  GemvArgs a{};
  a.W = w; a.N = 3 * m.d; a.K = m.d; a.x = xn; a.n_rows = f.n_rows;
  a.q = q; a.kv_pool = kv_pool; a.page_elems = kv_page_elems(m);
  a.layer_off = (size_t)layer * 2 * m.H * FE_PAGE * m.hd;
  a.rope = rope; a.H = m.H; a.hd = m.hd; a.d = m.d; a.rows = f.rows;
  gemv_any<EPI_QKV>(dtype, a, s);
}

void launch_resid(int dtype, const Fwd& f, int N, int K, const void* w, const void* xin, float* x, cudaStream_t s) {
  GemvArgs a{};
  a.W = w; a.N = N; a.K = K; a.x = xin; a.n_rows = f.n_rows; a.y = x;
  gemv_any<EPI_RESID>(dtype, a, s);
}

void launch_swiglu(int dtype, const Fwd& f, int F, int K, const void* w, const void* xin, void* act, cudaStream_t s) {
  GemvArgs a{};
  a.W = w; a.N = 2 * F; a.K = K; a.x = xin; a.n_rows = f.n_rows; a.act = act;
  gemv_any<EPI_SWIGLU>(dtype, a, s);
}

void launch_gemv_store(int dtype, const void* w, int N, int K, const void* x, int n_rows, float* y, cudaStream_t s) {
  GemvArgs a{};
  a.W = w; a.N = N; a.K = K; a.x = x; a.n_rows = n_rows; a.y = y;
  gemv_any<EPI_STORE>(dtype, a, s);
}

// ----------------------------------------------------- lm_head + argmax ----
__global__ void finalize_kernel(const RowMeta* rows, const int32_t* head_rows, const unsigned long long* part_keys,
                                int n_ctas, int32_t* out_tokens) {
  pdl_trigger();
  pdl_wait();
  __shared__ unsigned long long red[256];
  const int i = blockIdx.x;
  unsigned long long k = 0ull;
  for (int c = threadIdx.x; c < n_ctas; c += blockDim.x) k = max(k, part_keys[(size_t)i * n_ctas + c]);
  red[threadIdx.x] = k;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] = max(red[threadIdx.x], red[threadIdx.x + off]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const RowMeta m = rows[head_rows[i]];
    if (m.out_idx >= 0) out_tokens[m.out_idx] = argmax_index(red[0]);
  }
}

void launch_finalize(const Fwd& f, const unsigned long long* part_keys, int n_ctas, int32_t* out_tokens,
                     cudaStream_t s) {
  if (f.n_head_rows > 0)
    launch_k(finalize_kernel, dim3(f.n_head_rows), dim3(256), 0, s, f.rows, f.head_rows, part_keys, n_ctas, out_tokens);
}

void launch_lm_head(int dtype, const Fwd& f, const ModelDims& m, const void* w, const void* xn,
                    unsigned long long* part_keys, float* logits, int32_t* out_tokens, cudaStream_t s) {
  if (f.n_head_rows == 0) return;
  GemvArgs a{};
  a.W = w; a.N = m.V; a.K = m.d; a.x = xn; a.n_rows = f.n_head_rows;
  a.rows = f.rows; a.head_rows = f.head_rows; a.part_keys = part_keys; a.logits = logits;
  a.V = m.V; a.n_text = m.n_text;
  gemv_any<EPI_ARGMAX>(dtype, a, s);
  launch_k(finalize_kernel, dim3(f.n_head_rows), dim3(256), 0, s, f.rows, f.head_rows, part_keys, lm_head_ctas(m), out_tokens);
}

// ----------------------------------------------------------- attention ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <typename KT, int HD>
__global__ void __launch_bounds__(128)
attn_partial_kernel(const int32_t* __restrict__ hdr, const AttnItem* __restrict__ items, const ItemRow* __restrict__ item_rows,
                    const RowMeta* __restrict__ rows, const float* __restrict__ q, const KT* __restrict__ pool,
                    size_t page_elems, size_t layer_off, int H, int d, float scale, float* __restrict__ partial) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_kv[];
  __shared__ __align__(8) uint64_t bar;
  KT* ks = reinterpret_cast<KT*>(smem_kv);
  KT* vs = ks + FE_PAGE * HD;
  const int h = blockIdx.y;
  const int n_items = hdr[1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t phase = 0;
  // persistent over work items: grid.x CTAs per head stride through hdr[1] items
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, phase ^= 1) {
  __syncthreads();  // previous item's shared-memory reads done / barrier init visible
  const AttnItem it = items[item];
  // valid keys the CTA needs = max over its rows
  int vmax = 0;
  for (int i = 0; i < it.row_count; i++) vmax = max(vmax, item_rows[it.row_begin + i].valid);
  const KT* kg = pool + (size_t)it.page * page_elems + layer_off + (size_t)h * FE_PAGE * HD;
  const KT* vg = kg + (size_t)H * FE_PAGE * HD;
  const uint32_t bytes = (uint32_t)(vmax * HD * sizeof(KT));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(2 * bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(ks)), "l"(kg), "r"(bytes), "r"(smem_u32(&bar)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(vs)), "l"(vg), "r"(bytes), "r"(smem_u32(&bar)) : "memory");
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
    }
  }

  const bool own = 4 * lane < HD;  // lanes owning 4 head-dim elements
  for (int i = warp; i < it.row_count; i += 4) {
    const ItemRow ir = item_rows[it.row_begin + i];
    const RowMeta m = rows[ir.row];
    float qv[4] = {0.f, 0.f, 0.f, 0.f};
    if (own) {
      const float4 t = *reinterpret_cast<const float4*>(q + (size_t)ir.row * d + h * HD + 4 * lane);
      qv[0] = t.x; qv[1] = t.y; qv[2] = t.z; qv[3] = t.w;
    }
    // pass 1: scores; lane j%32 keeps s_j
    float mys[2] = {-INFINITY, -INFINITY};
    float mx = -INFINITY;
#pragma unroll
    for (int jb = 0; jb < 2; jb++) {
      for (int jj = 0; jj < 32; jj++) {
        const int j = jb * 32 + jj;
        if (j >= ir.valid) break;
        float a = 0.0f;
        if (own) {
          const KT* kr = ks + j * HD + 4 * lane;
#pragma unroll
          for (int c = 0; c < 4; c++) a = __fmaf_rn(Elem<KT>::to_f(kr[c]), qv[c], a);
        }
        // note: canonical dot is w=q, x=k order-insensitive per fmaf(a*b) commutativity
        const float sj = __fmul_rn(xor_butterfly(a), scale);
        if (lane == jj) mys[jb] = sj;
        mx = fmaxf(mx, sj);
      }
    }
    // pass 2: p_j, l, o
    float l = 0.0f, o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int jb = 0; jb < 2; jb++) {
      for (int jj = 0; jj < 32; jj++) {
        const int j = jb * 32 + jj;
        if (j >= ir.valid) break;
        const float p = fe_exp(__fsub_rn(__shfl_sync(0xffffffffu, mys[jb], jj), mx));
        l = __fadd_rn(l, p);
        if (own) {
          const KT* vr = vs + j * HD + 4 * lane;
#pragma unroll
          for (int c = 0; c < 4; c++) o[c] = __fmaf_rn(p, Elem<KT>::to_f(vr[c]), o[c]);
        }
      }
    }
    float* pp = partial + ((size_t)(m.chunk_base + it.chunk) * H + h) * (HD + 2);
    if (lane == 0) { pp[0] = mx; pp[1] = l; }
    if (own) {
      pp[2 + 4 * lane + 0] = o[0]; pp[2 + 4 * lane + 1] = o[1];
      pp[2 + 4 * lane + 2] = o[2]; pp[2 + 4 * lane + 3] = o[3];
    }
  }
  }  // item loop
}

template <typename XT, int HD>
__global__ void __launch_bounds__(128)
attn_merge_kernel(const RowMeta* __restrict__ rows, const float* __restrict__ partial, int H, int d,
                  XT* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x, h = blockIdx.y * 4 + warp;
  if (h >= H) return;
  const RowMeta m = rows[row];
  const bool own = 4 * lane < HD;
  float M = -INFINITY;
  for (int c = 0; c < m.n_chunks; c++) M = fmaxf(M, partial[((size_t)(m.chunk_base + c) * H + h) * (HD + 2)]);
  float L = 0.0f, o[4] = {0.f, 0.f, 0.f, 0.f};
  for (int c = 0; c < m.n_chunks; c++) {
    const float* pp = partial + ((size_t)(m.chunk_base + c) * H + h) * (HD + 2);
    const float sc = fe_exp(__fsub_rn(pp[0], M));
    L = __fmaf_rn(sc, pp[1], L);
    if (own) {
#pragma unroll
      for (int i = 0; i < 4; i++) o[i] = __fmaf_rn(sc, pp[2 + 4 * lane + i], o[i]);
    }
  }
  if (own) {
    XT* dst = out + (size_t)row * d + h * HD + 4 * lane;
#pragma unroll
    for (int i = 0; i < 4; i++) dst[i] = Elem<XT>::from_f(__fdiv_rn(o[i], L));
  }
}

// ------------------------------------------------- bf16 (fast) attention ----
// Same cascade work items as the canonical kernel, but free reduction order:
// 8 warps per (page, head) CTA, one query row per warp.  K and V land through
// two 1-D TMA bulk copies with separate mbarriers, so q.K^T starts while V is
// still in flight; scores for 8 keys at a time are reduced with a
// reduce-scatter butterfly (9 shuffles per 8 keys); softmax in the exp2 domain.
// The chunk merge is fused: after writing its chunk partial, a warp bumps the
// (row, head) arrival counter and the warp that completes the set merges all
// chunks of that (row, head) in chunk order (deterministic) and writes the
// attention output -- no separate merge launch.
template <int HD>
__global__ void __launch_bounds__(256)
attn_fused_bf16_kernel(const int32_t* __restrict__ hdr, const AttnItem* __restrict__ items,
                       const ItemRow* __restrict__ item_rows, const RowMeta* __restrict__ rows,
                       const float* __restrict__ q, const __nv_bfloat16* __restrict__ pool, size_t page_elems,
                       size_t layer_off, int H, int d, float scale_log2, float* __restrict__ partial,
                       int* __restrict__ counters, __nv_bfloat16* __restrict__ out) {
  constexpr int DPL = HD / 32;  // head dims per lane
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_kv[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ float pbuf[8][FE_PAGE];
  __nv_bfloat16* ks = reinterpret_cast<__nv_bfloat16*>(smem_kv);
  __nv_bfloat16* vs = ks + FE_PAGE * HD;
  const int h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();
  const int n_items = hdr[1];
  uint32_t phase = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, phase ^= 1) {
    __syncthreads();  // previous item's shared-memory reads done / barrier init visible
    const AttnItem it = items[item];
    const int vmax = it.valid_max;
    const __nv_bfloat16* kg = pool + (size_t)it.page * page_elems + layer_off + (size_t)h * FE_PAGE * HD;
    const __nv_bfloat16* vg = kg + (size_t)H * FE_PAGE * HD;
    const uint32_t bytes = (uint32_t)(vmax * HD * 2);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(ks)), "l"(kg), "r"(bytes), "r"(smem_u32(&bar[0])) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[1])), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(vs)), "l"(vg), "r"(bytes), "r"(smem_u32(&bar[1])) : "memory");
    }
    for (int i = warp; i < it.row_count; i += 8) {
      const ItemRow ir = item_rows[it.row_begin + i];
      const RowMeta m = rows[ir.row];
      float qv[DPL];
#pragma unroll
      for (int c = 0; c < DPL; c++) qv[c] = q[(size_t)ir.row * d + h * HD + DPL * lane + c] * scale_log2;
      if (i == warp) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(smem_u32(&bar[0])), "r"(phase) : "memory");
      }
      for (int j0 = 0; j0 < ir.valid; j0 += 8) {
        float part[8];
#pragma unroll
        for (int t = 0; t < 8; t++) {
          const __nv_bfloat16* kr = ks + (j0 + t) * HD + DPL * lane;
          float a = 0.0f;
          if (DPL == 4) {
            const uint2 raw = *reinterpret_cast<const uint2*>(kr);
            a = fmaf(qv[0], __uint_as_float(raw.x << 16), a);
            a = fmaf(qv[1], __uint_as_float(raw.x & 0xffff0000u), a);
            a = fmaf(qv[2], __uint_as_float(raw.y << 16), a);
            a = fmaf(qv[3], __uint_as_float(raw.y & 0xffff0000u), a);
          } else {
            const uint32_t raw = *reinterpret_cast<const uint32_t*>(kr);
            a = fmaf(qv[0], __uint_as_float(raw << 16), a);
            a = fmaf(qv[DPL - 1], __uint_as_float(raw & 0xffff0000u), a);
          }
          part[t] = a;
        }
#pragma unroll
        for (int t = 0; t < 4; t++) {
          const bool up = lane & 16;
          const float send = up ? part[t] : part[t + 4];
          const float keep = up ? part[t + 4] : part[t];
          part[t] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int t = 0; t < 2; t++) {
          const bool up = lane & 8;
          const float send = up ? part[t] : part[t + 2];
          const float keep = up ? part[t + 2] : part[t];
          part[t] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        {
          const bool up = lane & 4;
          const float send = up ? part[0] : part[1];
          const float keep = up ? part[1] : part[0];
          part[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        float sc = part[0];
        sc += __shfl_xor_sync(0xffffffffu, sc, 2);
        sc += __shfl_xor_sync(0xffffffffu, sc, 1);
        const int j = j0 + ((lane >> 2) & 7);
        if ((lane & 3) == 0) pbuf[warp][j] = j < ir.valid ? sc : -INFINITY;
      }
      __syncwarp();
      const float s0 = lane < ir.valid ? pbuf[warp][lane] : -INFINITY;
      const float s1 = lane + 32 < ir.valid ? pbuf[warp][lane + 32] : -INFINITY;
      float mx = fmaxf(s0, s1);
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float p0 = lane < ir.valid ? exp2f(s0 - mx) : 0.0f;
      const float p1 = lane + 32 < ir.valid ? exp2f(s1 - mx) : 0.0f;
      float l = p0 + p1;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
      __syncwarp();
      pbuf[warp][lane] = p0;
      pbuf[warp][lane + 32] = p1;
      __syncwarp();
      if (i == warp) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(smem_u32(&bar[1])), "r"(phase) : "memory");
      }
      float o[DPL];
#pragma unroll
      for (int c = 0; c < DPL; c++) o[c] = 0.0f;
#pragma unroll 8
      for (int j = 0; j < ir.valid; j++) {
        const float p = pbuf[warp][j];
        const __nv_bfloat16* vr = vs + j * HD + DPL * lane;
        if (DPL == 4) {
          const uint2 raw = *reinterpret_cast<const uint2*>(vr);
          o[0] = fmaf(p, __uint_as_float(raw.x << 16), o[0]);
          o[1] = fmaf(p, __uint_as_float(raw.x & 0xffff0000u), o[1]);
          o[2] = fmaf(p, __uint_as_float(raw.y << 16), o[2]);
          o[3] = fmaf(p, __uint_as_float(raw.y & 0xffff0000u), o[3]);
        } else {
          const uint32_t raw = *reinterpret_cast<const uint32_t*>(vr);
          o[0] = fmaf(p, __uint_as_float(raw << 16), o[0]);
          o[DPL - 1] = fmaf(p, __uint_as_float(raw & 0xffff0000u), o[DPL - 1]);
        }
      }
      float* pp = partial + ((size_t)(m.chunk_base + it.chunk) * H + h) * (HD + 2);
      if (lane == 0) { pp[0] = mx; pp[1] = l; }
#pragma unroll
      for (int c = 0; c < DPL; c++) pp[2 + DPL * lane + c] = o[c];

      // ---- fused merge: the warp that delivers the last chunk of (row, head)
      int prev = 0;
      __syncwarp();
      __threadfence();  // every lane publishes its slice of the partial
      if (lane == 0) prev = atomicAdd(&counters[ir.row * H + h], 1);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev == m.n_chunks - 1) {
        if (lane == 0) counters[ir.row * H + h] = 0;  // ready for the next launch
        __threadfence();
        const float* base = partial + ((size_t)m.chunk_base * H + h) * (HD + 2);
        const size_t stride = (size_t)H * (HD + 2);
        // chunk weights lane-parallel (lane c <-> chunk c, c + 32, ...), then
        // every lane accumulates its head dims over all chunks with the loads
        // of a group of 8 chunks in flight together
        float M = -INFINITY;
        for (int c = lane; c < m.n_chunks; c += 32) M = fmaxf(M, __ldcg(base + c * stride));
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
        float L = 0.0f, acc[DPL];
#pragma unroll
        for (int c = 0; c < DPL; c++) acc[c] = 0.0f;
        for (int c0 = 0; c0 < m.n_chunks; c0 += 32) {
          const int c = c0 + lane;
          const float wl = c < m.n_chunks ? exp2f(__ldcg(base + c * stride) - M) : 0.0f;
          float lsum = c < m.n_chunks ? wl * __ldcg(base + c * stride + 1) : 0.0f;
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
          L += lsum;
          const int nc = min(32, m.n_chunks - c0);
          for (int g = 0; g < nc; g += 8) {
            float v[8][DPL], w[8];
#pragma unroll
            for (int t = 0; t < 8; t++) {
              w[t] = __shfl_sync(0xffffffffu, wl, (g + t) & 31);
              if (g + t < nc) {
#pragma unroll
                for (int e = 0; e < DPL; e++) v[t][e] = __ldcg(base + (c0 + g + t) * stride + 2 + DPL * lane + e);
              }
            }
#pragma unroll
            for (int t = 0; t < 8; t++)
              if (g + t < nc) {
#pragma unroll
                for (int e = 0; e < DPL; e++) acc[e] = fmaf(w[t], v[t][e], acc[e]);
              }
          }
        }
        const float inv = 1.0f / L;
        __nv_bfloat16* dst = out + (size_t)ir.row * d + h * HD + DPL * lane;
#pragma unroll
        for (int e = 0; e < DPL; e++) dst[e] = __float2bfloat16_rn(acc[e] * inv);
      }
    }
  }  // item loop
}

template <int HD>
static void attention_bf16(const Fwd& f, const ModelDims& m, const float* q, const void* pool, int layer,
                           float* partial, void* out, cudaStream_t s) {
  const size_t pe = kv_page_elems(m);
  const size_t lo = (size_t)layer * 2 * m.H * FE_PAGE * m.hd;
  const size_t smem = 2 * (size_t)FE_PAGE * HD * 2;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attn_fused_bf16_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  const float scale_log2 = m.attn_scale * 1.4426950408889634f;
  if (f.item_cap > 0)
    launch_k(attn_fused_bf16_kernel<HD>, dim3(f.item_cap, m.H), dim3(256), smem, s, f.hdr, f.items, f.item_rows,
             f.rows, q, (const __nv_bfloat16*)pool, pe, lo, m.H, m.d, scale_log2, partial, f.attn_counters,
             (__nv_bfloat16*)out);
}

template <typename KT, int HD>
static void attention_t(const Fwd& f, const ModelDims& m, const float* q, const void* pool, int layer,
                        float* partial, void* out, cudaStream_t s) {
  const size_t pe = kv_page_elems(m);
  const size_t lo = (size_t)layer * 2 * m.H * FE_PAGE * m.hd;
  const size_t smem = 2 * (size_t)FE_PAGE * HD * sizeof(KT);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(attn_partial_kernel<KT, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured = true;
  }
  if (f.item_cap > 0)
    launch_k(attn_partial_kernel<KT, HD>, dim3(f.item_cap, m.H), dim3(128), smem, s, f.hdr, f.items, f.item_rows,
             f.rows, q, (const KT*)pool, pe, lo, m.H, m.d, m.attn_scale, partial);
  launch_k(attn_merge_kernel<KT, HD>, dim3(f.n_rows, (m.H + 3) / 4), dim3(128), 0, s, f.rows, (const float*)partial,
           m.H, m.d, (KT*)out);
}

void launch_attention(int dtype, const Fwd& f, const ModelDims& m, const float* q, const void* kv_pool,
                      int layer, float* partial, void* attn_out, cudaStream_t s) {
  if (f.n_rows == 0) return;
  if (dtype == F32) {
    if (m.hd == 64) attention_t<float, 64>(f, m, q, kv_pool, layer, partial, attn_out, s);
    else attention_t<float, 128>(f, m, q, kv_pool, layer, partial, attn_out, s);
  } else {
    if (m.hd == 64) attention_bf16<64>(f, m, q, kv_pool, layer, partial, attn_out, s);
    else attention_bf16<128>(f, m, q, kv_pool, layer, partial, attn_out, s);
  }
}

// ----------------------------------------------------------- page copy ----
// Copy-on-write at a fork: slots [0, n) of every (layer, K/V, head) block.
template <typename KT>
__global__ void page_copy_kernel(KT* pool, size_t page_elems, int src, int dst, int n_elems) {
  // block b = one (layer, K/V, head) block of FE_PAGE * hd elements
  const size_t block_elems = page_elems / gridDim.x;
  const KT* s = pool + (size_t)src * page_elems + (size_t)blockIdx.x * block_elems;
  KT* d = pool + (size_t)dst * page_elems + (size_t)blockIdx.x * block_elems;
  for (int i = threadIdx.x; i < n_elems; i += blockDim.x) d[i] = s[i];
}

void launch_page_copy(int dtype, void* pool, int src, int dst, int n_slots, const ModelDims& m, cudaStream_t s) {
  if (n_slots <= 0) return;
  const int blocks = m.L * 2 * m.H;
  const size_t pe = kv_page_elems(m);
  if (dtype == F32) page_copy_kernel<float><<<blocks, 256, 0, s>>>((float*)pool, pe, src, dst, n_slots * m.hd);
  else page_copy_kernel<__nv_bfloat16><<<blocks, 256, 0, s>>>((__nv_bfloat16*)pool, pe, src, dst, n_slots * m.hd);
}

}  // namespace fe
