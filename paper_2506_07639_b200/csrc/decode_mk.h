// Persistent decode-tick kernel (decode_mk.cu): one launch runs a whole
// bf16 decode iteration (embedding, all layers, lm_head + greedy argmax) for
// up to 16 rows.  Host-side interface for engine.cu.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "gemm_tc.h"

namespace fe {

struct Fwd;
struct ModelDims;

// One GEMM of the tick: `tiles` tiles of 128 weight rows; the k-blocks of a
// tile are cut into `nc` chunks that CTAs grab dynamically (chunks = tiles * nc).
struct MkPlan {
  int tiles, kb_total, nc, chunks;
};
enum MkGemm { MK_QKV = 0, MK_O = 1, MK_GU = 2, MK_DOWN = 3, MK_LM = 4 };

struct MkLaunch {
  int grid;                      // persistent CTAs (one per SM)
  MkPlan plan[5];
  const void* wmaps;             // device CUtensorMap[4 L + 1]: per layer qkv, o, gate/up, down; lm_head
  const float* const* norms;     // device float*[2 L + 1]: attn_norm l, ffn_norm l, ..., final_norm
  TmaMap map_xg, map_attn, map_act;  // 16-row boxes over the lane's staging buffers
  // model
  int d, F, H, L, V, n_text;
  float eps, scale_log2;
  // forward
  const int32_t* hdr;            // device header (n_items at [1])
  const void* rows;              // RowMeta[B]
  const void* items;             // AttnItem[]
  const void* item_rows;         // ItemRow[]
  int B;                         // rows of the tick (<= 16), every row samples a token
  const __nv_bfloat16* embed;
  int32_t* out_tokens;
  float* x;                      // [16][d] residual stream
  __nv_bfloat16* xg;             // [16][d] x * norm gain (bf16), the GEMM input of QKV / gate-up / lm_head
  float* ss;                     // [16][d / 128] per-tile sums of squares of x (16-byte aligned rows)
  float* q;                      // [16][d]
  __nv_bfloat16* attn;           // [16][max(d, F)] attention output, then the SwiGLU activation
  __nv_bfloat16* kv_pool;
  size_t page_elems;
  const float* rope;
  float* partial;                // chunk partials [chunks][128][16]
  int* counters;                 // per-tile chunk arrival counters (self-resetting)
  float* apartial;               // attention chunk partials
  int* acounters;                // attention merge counters (self-resetting)
  unsigned long long* part_keys; // [16][lm tiles]
  float* logits;                 // parity mode: rows with logit_row >= 0
  unsigned long long* bar;       // [2]: grid barrier arrivals, exits (self-resetting)
  int* grab;                     // [phases] chunk counters (self-resetting)
  int flags;                     // diagnostics: 1 = no weight prefetch across grid barriers
  int fused;                     // bit MK_*: that GEMM's tiles are finalised inside its phase
  int pf_stages;                 // weight stages prefetched ahead of a grid barrier (0 = whole ring)
  unsigned long long* trace;     // diagnostics (null): [phases][2][grid] globaltimer at barrier pass / phase end
};

MkPlan mk_plan(int tiles, int kb_total, int grid, int per_cta = 4, int cap = 16);
size_t mk_partial_floats(const MkPlan* plans);
void launch_decode_mk(const MkLaunch& l, cudaStream_t s);
void launch_decode_mk_traced(const MkLaunch& l, cudaStream_t s);  // decode_mk_trace.cu
int mk_grid();
int mk_phases(int L);             // upper bound over fused masks (buffer sizing)
int mk_phases(int L, int fused);  // phases of a tick with that fused mask

}  // namespace fe
