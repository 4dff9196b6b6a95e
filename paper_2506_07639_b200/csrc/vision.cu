// Vision tower + projector: the observation's image ->
// the n_vision VIS rows of the LLM input, replacing the synthetic
// embeddings when enabled (fe_vision_enable).  A pre-LayerNorm ViT
// (DINOv2-L/14-shaped at 224 px: 256 patches, d 1024, 24 layers, 16 heads,
// MLP 4096) and a 2-layer GELU MLP projector into the LLM width; the image
// itself is synthetic (counter-based pixels keyed by the observation digest,
// random-init weights).  Definition: oracle/oracle.c `or_vision_encode`.
//
// fp32 mode: every contraction is the canonical dot (launch_gemv_store) and
// the other ops follow the oracle's order, so the rows are bit-identical to
// the CPU oracle.  bf16 mode: the linear layers run on the CTA-pair tcgen05
// GEMM (bf16 weights and staged activations, fp32 accumulate); LayerNorm,
// attention (256 patches x 16 heads, non-causal) and the activations stay in
// fp32.
#include "common.cuh"
#include "engine_internal.h"
#include "gemm_tc.h"
#include "vision.h"

#include <algorithm>
#include <stdexcept>
#include <vector>

namespace fe {
namespace {

constexpr uint64_t T_IMAGE = 5, T_VB = 1ull << 20;
enum { V_PE_W, V_PE_B, V_POS, V_LNF_G, V_LNF_B, V_P1_W, V_P1_B, V_P2_W, V_P2_B };
enum { VL_LN1_G, VL_LN1_B, VL_QKV_W, VL_QKV_B, VL_O_W, VL_O_B, VL_LN2_G, VL_LN2_B, VL_FC1_W, VL_FC1_B,
       VL_FC2_W, VL_FC2_B };

// canonical dot of one warp: lane l accumulates k = 128 j + 4 l + c, then the xor butterfly
__device__ __forceinline__ float warp_cdot(const float* w, const float* x, int K, int lane) {
  float a = 0.0f;
  for (int j = 0; j < K; j += 128) {
    const int k = j + 4 * lane;
    if (k < K) {
#pragma unroll
      for (int c = 0; c < 4; c++) a = __fmaf_rn(w[k + c], x[k + c], a);
    }
  }
  return xor_butterfly(a);
}

__global__ void patch_kernel(uint64_t vseed, int img, int ps, int grid, int kp, int P, float* patches) {
  const uint64_t key = tensor_key(vseed, T_IMAGE);
  const size_t n = (size_t)P * kp;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int p = (int)(i / kp), f = (int)(i % kp);
    float v = 0.0f;
    if (f < 3 * ps * ps) {
      const int c = f / (ps * ps), dy = (f / ps) % ps, dx = f % ps;
      const int y = (p / grid) * ps + dy, x = (p % grid) * ps + dx;
      v = __fmul_rn(centered(key, (uint64_t)((c * img + y) * img + x)), 2.0f);
    }
    patches[i] = v;
  }
}

// y = y + b (mode 0), gelu(y + b) (1), x = x + (y + b) (2), x = (y + b) + pos (3)
__global__ void bias_kernel(float* y, const float* b, float* x, const float* pos, int n, int N, int mode) {
  const size_t total = (size_t)n * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const float t = __fadd_rn(y[i], b[i % N]);
    if (mode == 0) y[i] = t;
    else if (mode == 1) y[i] = __fdiv_rn(t, __fadd_rn(1.0f, fe_exp(__fmul_rn(-1.702f, t))));
    else if (mode == 2) x[i] = __fadd_rn(x[i], t);
    else x[i] = __fadd_rn(t, pos[i]);
  }
}

__global__ void layernorm_kernel(const float* x, const float* g, const float* b, float* y, int n, int d, float eps) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const float* xr = x + (size_t)warp * d;
  float* yr = y + (size_t)warp * d;
  // the lane's elements k = 128 j + 4 lane + c, held in registers (d <= 2048)
  float4 v[16];
  float a = 0.0f;  // cdot(x, ones)
#pragma unroll
  for (int j = 0; j < 16; j++) {
    const int k = 128 * j + 4 * lane;
    v[j] = k < d ? *reinterpret_cast<const float4*>(xr + k) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (k < d) {
      a = __fmaf_rn(v[j].x, 1.0f, a);
      a = __fmaf_rn(v[j].y, 1.0f, a);
      a = __fmaf_rn(v[j].z, 1.0f, a);
      a = __fmaf_rn(v[j].w, 1.0f, a);
    }
  }
  const float mean = __fdiv_rn(xor_butterfly(a), (float)d);
  float s = 0.0f;  // cdot(xc, xc)
#pragma unroll
  for (int j = 0; j < 16; j++) {
    if (128 * j + 4 * lane < d) {
      v[j].x = __fsub_rn(v[j].x, mean); v[j].y = __fsub_rn(v[j].y, mean);
      v[j].z = __fsub_rn(v[j].z, mean); v[j].w = __fsub_rn(v[j].w, mean);
      s = __fmaf_rn(v[j].x, v[j].x, s);
      s = __fmaf_rn(v[j].y, v[j].y, s);
      s = __fmaf_rn(v[j].z, v[j].z, s);
      s = __fmaf_rn(v[j].w, v[j].w, s);
    }
  }
  const float var = __fdiv_rn(xor_butterfly(s), (float)d);
  const float r = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, eps)));
#pragma unroll
  for (int j = 0; j < 16; j++) {
    const int k = 128 * j + 4 * lane;
    if (k < d) {
      const float4 gg = *reinterpret_cast<const float4*>(g + k), bb = *reinterpret_cast<const float4*>(b + k);
      float4 o;
      o.x = __fadd_rn(__fmul_rn(__fmul_rn(v[j].x, r), gg.x), bb.x);
      o.y = __fadd_rn(__fmul_rn(__fmul_rn(v[j].y, r), gg.y), bb.y);
      o.z = __fadd_rn(__fmul_rn(__fmul_rn(v[j].z, r), gg.z), bb.z);
      o.w = __fadd_rn(__fmul_rn(__fmul_rn(v[j].w, r), gg.w), bb.w);
      *reinterpret_cast<float4*>(yr + k) = o;
    }
  }
}

// non-causal attention, one warp per (patch, head), keys in order (the oracle's vattention)
__global__ void __launch_bounds__(128) vattn_kernel(const float* qkv, float* out, int P, int H, int hd, int d,
                                                     float scale) {
  extern __shared__ float sbuf[];  // [4 warps][P]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 4 + warp;
  if (t >= P * H) return;
  const int p = t / H, h = t % H;
  float* s = sbuf + warp * P;
  const float* q = qkv + (size_t)p * 3 * d + h * hd;
  float m = -INFINITY;
  for (int j = 0; j < P; j++) {
    const float sj = __fmul_rn(warp_cdot(q, qkv + (size_t)j * 3 * d + d + h * hd, hd, lane), scale);
    if (lane == 0) s[j] = sj;
    m = fmaxf(m, sj);
  }
  __syncwarp();
  float l = 0.0f, o[8];
#pragma unroll
  for (int i = 0; i < 8; i++) o[i] = 0.0f;
  for (int j = 0; j < P; j++) {
    const float pj = fe_exp(__fsub_rn(s[j], m));
    l = __fadd_rn(l, pj);
    const float* vj = qkv + (size_t)j * 3 * d + 2 * d + h * hd;
#pragma unroll
    for (int i = 0; i < 8; i++)
      if (lane + 32 * i < hd) o[i] = __fmaf_rn(pj, vj[lane + 32 * i], o[i]);
  }
#pragma unroll
  for (int i = 0; i < 8; i++)
    if (lane + 32 * i < hd) out[(size_t)p * d + h * hd + lane + 32 * i] = __fdiv_rn(o[i], l);
}

// bf16 mode: the same attention on mma.sync m16n8k16 (bf16 operands, fp32
// accumulate): CTA = (64 query patches, head); K and V of all P <= 256
// patches staged in shared memory as bf16 (128-byte rows, 16-byte chunks
// XOR-swizzled, conflict-free ldmatrix); each warp holds its 16 rows' whole
// score row in registers (no online softmax needed at P <= 256).
__device__ __forceinline__ uint32_t vpack2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ void vmma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t vs32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) vattn_bf16_kernel(const float* __restrict__ qkv, float* __restrict__ out,
                                                         int P, int d, float scale_log2) {
  constexpr int HDV = 64, MAXP = 256;
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* sk = sm;                  // [P][128 B]
  unsigned char* sv = sm + MAXP * 128;     // [P][128 B]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int h = blockIdx.y, q0 = blockIdx.x * 64 + warp * 16;
  for (int i = tid; i < P * 8; i += 128) {  // 16-byte chunk c of patch j, K and V
    const int j = i >> 3, c = i & 7;
    const float* kp = qkv + (size_t)j * 3 * d + d + h * HDV + 8 * c;
    const float* vp = kp + d;
    const float4 k0 = *reinterpret_cast<const float4*>(kp), k1 = *reinterpret_cast<const float4*>(kp + 4);
    const float4 v0 = *reinterpret_cast<const float4*>(vp), v1 = *reinterpret_cast<const float4*>(vp + 4);
    const uint32_t off = (uint32_t)(j * 128 + ((c ^ (j & 7)) << 4));
    *reinterpret_cast<uint4*>(sk + off) = make_uint4(vpack2(k0.x, k0.y), vpack2(k0.z, k0.w), vpack2(k1.x, k1.y),
                                                     vpack2(k1.z, k1.w));
    *reinterpret_cast<uint4*>(sv + off) = make_uint4(vpack2(v0.x, v0.y), vpack2(v0.z, v0.w), vpack2(v1.x, v1.y),
                                                     vpack2(v1.z, v1.w));
  }
  // Q fragments (4 k-steps of 16 dims), exp2 domain
  const int ra = q0 + g, rb = q0 + g + 8;
  uint32_t qa[4][4];
#pragma unroll
  for (int ks = 0; ks < 4; ks++) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
    if (ra < P) {
      const float* qp = qkv + (size_t)ra * 3 * d + h * HDV + 16 * ks + 2 * t;
      a0 = *reinterpret_cast<const float2*>(qp);
      a1 = *reinterpret_cast<const float2*>(qp + 8);
    }
    if (rb < P) {
      const float* qp = qkv + (size_t)rb * 3 * d + h * HDV + 16 * ks + 2 * t;
      b0 = *reinterpret_cast<const float2*>(qp);
      b1 = *reinterpret_cast<const float2*>(qp + 8);
    }
    qa[ks][0] = vpack2(a0.x * scale_log2, a0.y * scale_log2);
    qa[ks][1] = vpack2(b0.x * scale_log2, b0.y * scale_log2);
    qa[ks][2] = vpack2(a1.x * scale_log2, a1.y * scale_log2);
    qa[ks][3] = vpack2(b1.x * scale_log2, b1.y * scale_log2);
  }
  __syncthreads();
  const int lm = lane >> 3, lrow = lane & 7;
  const int nts = P / 8;
  float sc[MAXP / 8][4];
#pragma unroll
  for (int nt = 0; nt < MAXP / 8; nt += 2) {
    sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.0f;
    sc[nt + 1][0] = sc[nt + 1][1] = sc[nt + 1][2] = sc[nt + 1][3] = 0.0f;
    if (nt >= nts) continue;
#pragma unroll
    for (int ks = 0; ks < 4; ks++) {
      const int key = 8 * nt + 8 * (lm >> 1) + lrow, c16 = 2 * ks + (lm & 1);
      uint32_t b0, b1, b2, b3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                   : "r"(vs32(sk + key * 128 + ((c16 ^ (key & 7)) << 4))));
      vmma(sc[nt], qa[ks], b0, b1);
      vmma(sc[nt + 1], qa[ks], b2, b3);
    }
  }
  float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
  for (int nt = 0; nt < MAXP / 8; nt++)
    if (nt < nts) {
      ma = fmaxf(ma, fmaxf(sc[nt][0], sc[nt][1]));
      mb = fmaxf(mb, fmaxf(sc[nt][2], sc[nt][3]));
    }
  ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, 1));
  ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, 2));
  mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 1));
  mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, 2));
  float la = 0.0f, lb = 0.0f;
#pragma unroll
  for (int nt = 0; nt < MAXP / 8; nt++)
    if (nt < nts) {
      sc[nt][0] = exp2f(sc[nt][0] - ma);
      sc[nt][1] = exp2f(sc[nt][1] - ma);
      sc[nt][2] = exp2f(sc[nt][2] - mb);
      sc[nt][3] = exp2f(sc[nt][3] - mb);
      la += sc[nt][0] + sc[nt][1];
      lb += sc[nt][2] + sc[nt][3];
    }
  la += __shfl_xor_sync(0xffffffffu, la, 1);
  la += __shfl_xor_sync(0xffffffffu, la, 2);
  lb += __shfl_xor_sync(0xffffffffu, lb, 1);
  lb += __shfl_xor_sync(0xffffffffu, lb, 2);
  float o[HDV / 8][4];
#pragma unroll
  for (int i = 0; i < HDV / 8; i++) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.0f;
#pragma unroll
  for (int kk = 0; kk < MAXP / 16; kk++) {
    if (kk >= P / 16) continue;
    uint32_t pa[4];
    pa[0] = vpack2(sc[2 * kk][0], sc[2 * kk][1]);
    pa[1] = vpack2(sc[2 * kk][2], sc[2 * kk][3]);
    pa[2] = vpack2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]);
    pa[3] = vpack2(sc[2 * kk + 1][2], sc[2 * kk + 1][3]);
    const int key = 16 * kk + lrow + 8 * (lm & 1);
#pragma unroll
    for (int np = 0; np < HDV / 16; np++) {
      const int c16 = 2 * np + (lm >> 1);
      uint32_t b0, b1, b2, b3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                   : "r"(vs32(sv + key * 128 + ((c16 ^ (key & 7)) << 4))));
      vmma(o[2 * np], pa, b0, b1);
      vmma(o[2 * np + 1], pa, b2, b3);
    }
  }
  const float ia = 1.0f / la, ib = 1.0f / lb;
#pragma unroll
  for (int nt = 0; nt < HDV / 8; nt++) {
    const int dim = 8 * nt + 2 * t;
    if (ra < P) *reinterpret_cast<float2*>(out + (size_t)ra * d + h * HDV + dim) = make_float2(o[nt][0] * ia, o[nt][1] * ia);
    if (rb < P) *reinterpret_cast<float2*>(out + (size_t)rb * d + h * HDV + dim) = make_float2(o[nt][2] * ib, o[nt][3] * ib);
  }
}

__global__ void to_bf16_kernel(const float* x, __nv_bfloat16* y, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

int blocks_for(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 8); }

}  // namespace

struct Vision::Lin {
  void* w = nullptr;   // [N][K] dtype
  float* b = nullptr;
  int N = 0, K = 0;
  TmaMap bmap{};       // bf16: B operand of the pair GEMM (64-row boxes)
};

Vision::Vision(const VisionDims& vd, int dtype, int out_d, uint64_t seed, cudaStream_t s,
               std::function<void*(size_t)> alloc)
    : v(vd), dtype(dtype), out_d(out_d) {
  grid = v.img / v.patch;
  P = grid * grid;
  hd = v.d / v.H;
  kp = (3 * v.patch * v.patch + 127) / 128 * 128;
  const size_t el = dtype == 1 ? 2 : 4;
  auto key = [&](uint64_t tid) { return tensor_key(seed, tid); };
  auto vec = [&](uint64_t tid, size_t n, bool norm) {
    float* p = (float*)alloc(n * 4);
    if (norm) launch_init_norm(p, key(tid), n, s);
    else launch_init_linear(0, p, key(tid), n, s);
    return p;
  };
  auto lin = [&](uint64_t wid, uint64_t bid, int N, int K) {
    auto L = std::make_unique<Lin>();
    L->N = N; L->K = K;
    L->w = alloc((size_t)N * K * el);
    launch_init_linear(dtype, L->w, key(wid), (size_t)N * K, s);
    L->b = vec(bid, N, false);
    if (dtype == 1) L->bmap = make_kmajor_map(L->w, N, K, K, 64);
    return L;
  };
  pe = lin(T_VB + V_PE_W, T_VB + V_PE_B, v.d, kp);
  pos = vec(T_VB + V_POS, (size_t)P * v.d, false);
  lnf_g = vec(T_VB + V_LNF_G, v.d, true);
  lnf_b = vec(T_VB + V_LNF_B, v.d, false);
  p1 = lin(T_VB + V_P1_W, T_VB + V_P1_B, v.ph, v.d);
  p2 = lin(T_VB + V_P2_W, T_VB + V_P2_B, out_d, v.ph);
  for (int l = 0; l < v.L; l++) {
    const uint64_t b = T_VB + 16 + 16 * (uint64_t)l;
    Layer y;
    y.ln1_g = vec(b + VL_LN1_G, v.d, true);
    y.ln1_b = vec(b + VL_LN1_B, v.d, false);
    y.qkv = lin(b + VL_QKV_W, b + VL_QKV_B, 3 * v.d, v.d);
    y.o = lin(b + VL_O_W, b + VL_O_B, v.d, v.d);
    y.ln2_g = vec(b + VL_LN2_G, v.d, true);
    y.ln2_b = vec(b + VL_LN2_B, v.d, false);
    y.fc1 = lin(b + VL_FC1_W, b + VL_FC1_B, v.mlp, v.d);
    y.fc2 = lin(b + VL_FC2_W, b + VL_FC2_B, v.d, v.mlp);
    layers.push_back(std::move(y));
  }
  const int wide = std::max({v.mlp, v.ph, 3 * v.d, kp, out_d});
  patches = (float*)alloc((size_t)P * kp * 4);
  x = (float*)alloc((size_t)P * v.d * 4);
  ln = (float*)alloc((size_t)P * wide * 4);
  big = (float*)alloc((size_t)P * wide * 4);
  att = (float*)alloc((size_t)P * v.d * 4);
  if (dtype == 1) {
    stage = (__nv_bfloat16*)alloc((size_t)std::max(P, 256) * wide * 2);
    stage_maps[0] = make_kmajor_map(stage, std::max(P, 256), kp, kp, 128);
    stage_maps[1] = make_kmajor_map(stage, std::max(P, 256), v.d, v.d, 128);
    stage_maps[2] = make_kmajor_map(stage, std::max(P, 256), v.mlp, v.mlp, 128);
    stage_maps[3] = make_kmajor_map(stage, std::max(P, 256), v.ph, v.ph, 128);
    split_floats = (size_t)8 * std::max(P, 256) * wide;
    split = (float*)alloc(split_floats * 4);
    cudaFuncSetAttribute(vattn_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 256 * 128);
  }
  CK_VIS(cudaGetLastError());
}

Vision::~Vision() = default;

// y[P][N] = x[P][K] . W^T (+ bias / activation / residual by `mode`, see bias_kernel)
void Vision::linear(const Lin& L, const float* xin, float* y, int mode, float* resid, const float* posv,
                    cudaStream_t s) {
  if (dtype == 0) {
    launch_gemv_store(0, L.w, L.N, L.K, xin, P, y, s);
  } else {
    to_bf16_kernel<<<blocks_for((size_t)P * L.K), 256, 0, s>>>(xin, stage, (size_t)P * L.K);
    const TmaMap& am = L.K == kp ? stage_maps[0] : L.K == v.d ? stage_maps[1] : L.K == v.mlp ? stage_maps[2]
                                                                                               : stage_maps[3];
    TcLaunch t{};
    t.M = P; t.N = L.N; t.K = L.K; t.epi = TC_STORE; t.y = y; t.ldy = L.N;
    t.split_scratch = split; t.split_floats = split_floats;  // few tiles at P = 256: split-K fills the GPU
    launch_gemm_tc(am, L.bmap, t, s);
  }
  bias_kernel<<<blocks_for((size_t)P * L.N), 256, 0, s>>>(y, L.b, resid, posv, P, L.N, mode);
}

void Vision::encode(uint64_t vseed, float* out, cudaStream_t s) {
  const int d = v.d;
  patch_kernel<<<blocks_for((size_t)P * kp), 256, 0, s>>>(vseed, v.img, v.patch, grid, kp, P, patches);
  linear(*pe, patches, big, 3, x, pos, s);                      // x = (pe(patch) + b) + pos
  const int ln_blocks = (P * 32 + 127) / 128;
  const float scale = 1.0f / sqrtf((float)hd);
  for (const Layer& y : layers) {
    layernorm_kernel<<<ln_blocks, 128, 0, s>>>(x, y.ln1_g, y.ln1_b, ln, P, d, v.eps);
    linear(*y.qkv, ln, big, 0, nullptr, nullptr, s);            // qkv
    if (dtype == 1 && hd == 64 && P % 16 == 0 && P <= 256)
      vattn_bf16_kernel<<<dim3((P + 63) / 64, v.H), 128, 2 * 256 * 128, s>>>(big, att, P, d,
                                                                           scale * 1.4426950408889634f);
    else
      vattn_kernel<<<(P * v.H + 3) / 4, 128, 4 * P * sizeof(float), s>>>(big, att, P, v.H, hd, d, scale);
    linear(*y.o, att, ln, 2, x, nullptr, s);                    // x += o(att) + b
    layernorm_kernel<<<ln_blocks, 128, 0, s>>>(x, y.ln2_g, y.ln2_b, ln, P, d, v.eps);
    linear(*y.fc1, ln, big, 1, nullptr, nullptr, s);            // gelu(fc1 + b)
    linear(*y.fc2, big, ln, 2, x, nullptr, s);                  // x += fc2 + b
  }
  layernorm_kernel<<<ln_blocks, 128, 0, s>>>(x, lnf_g, lnf_b, ln, P, d, v.eps);
  linear(*p1, ln, big, 1, nullptr, nullptr, s);                 // gelu(p1 + b)
  linear(*p2, big, out, 0, nullptr, nullptr, s);                // out = p2 + b
  CK_VIS(cudaGetLastError());
}

}  // namespace fe
