// tcgen05 GEMM interface (gemm_tc.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace fe {

struct RowMeta;

enum TcEpi { TC_STORE = 0, TC_QKV = 1, TC_RESID = 2, TC_SWIGLU = 3, TC_ARGMAX = 4 };

// Opaque CUtensorMap storage (128 bytes, 64-byte aligned).
struct alignas(64) TmaMap {
  unsigned char bytes[128];
};

struct TcLaunch {
  int M, N, K, epi;
  float* y;
  int ldy;
  __nv_bfloat16* act;
  int F;
  float* q;
  __nv_bfloat16* kv_pool;
  size_t page_elems, layer_off;
  const float* rope;
  const RowMeta* rows;
  int H, hd, d;
  float* sk_scratch;   // stream-K partials of the pair GEMM (pair_sk_scratch_floats()), or null: no stream-K
  int* sk_counters;    // pair_sk_counters() ints, zero-initialised
  float* split_scratch;  // split-K partial planes (split_floats floats), or null: no split-K
  size_t split_floats;
  // RESID only: the RMSNorm that follows (bf16 out = norm(y) * norm_w).  When
  // the GEMM runs split-K, the reduce applies it too and launch_gemm_tc
  // returns true (the caller then skips its own norm launch)
  const float* norm_w;
  __nv_bfloat16* norm_out;
  float norm_eps;
};

// skinny decode GEMM (swap-AB, <= skinny_max_rows() batch rows)
struct SkLaunch {
  int N, K, B, epi;
  float* partial;
  int* counters;
  float* y;
  int ldy;
  __nv_bfloat16* act;
  int F;
  float* q;
  __nv_bfloat16* kv_pool;
  size_t page_elems, layer_off;
  const float* rope;
  const RowMeta* rows;
  const int32_t* head_rows;
  int H, hd, d;
  unsigned long long* part_keys;
  float* logits;
  int V, n_text;
};

// 2-D K-major bf16 tensor [rows][K] with row stride ld_elems, box [box_rows x 64], 128B swizzle
TmaMap make_kmajor_map(const void* base, int rows, int K, int ld_elems, int box_rows);
int tc_box_rows(int epi);
// CTA-pair persistent tcgen05 GEMM (B map: 64-row boxes)
bool launch_gemm_tc(const TmaMap& a_map, const TmaMap& b_map64, const TcLaunch& l, cudaStream_t s);
// round-1 1-CTA 128 x 128 tile GEMM (B map: 128-row boxes, SwiGLU 64), kept for A/B (option "tc_pair" 0)
void launch_gemm_tc_v1(const TmaMap& a_map, const TmaMap& b_map, const TcLaunch& l, cudaStream_t s);
extern int g_pair_bn;
extern int g_pair_sk;
extern int g_pair_maxp;
extern int g_pair_split;
size_t pair_sk_scratch_floats();
int pair_sk_counters();
int skinny_max_rows();      // widest batch of the skinny GEMM (rows; > 256 run as 256-row slices)
int skinny_cols(int rows);  // MMA N used for `rows` batch rows (16/32/64/128/256)
size_t skinny_partial_floats(int N, int K);  // split-K scratch the skinny GEMM may use for one matrix
int skinny_tiles(int epi, int N, int F);
void launch_skinny_tc(const TmaMap& w_map, const TmaMap& x_map, const SkLaunch& l, cudaStream_t s);

}  // namespace fe
