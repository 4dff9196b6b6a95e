// Internal structures shared by the host engine (engine.cu) and the kernels
// (kernels.cu).  Not part of the C ABI (see include/fastecot.h).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <utility>

namespace fe {

enum DType { F32 = 0, BF16 = 1 };

// One query row of a forward pass (prefill token or decode row).
struct RowMeta {
  int32_t pos;         // absolute position in its sequence
  int32_t tok;         // explicit input id (>= 0), else take out_tokens[tok_src]
  int32_t tok_src;     // feedback index into out_tokens
  int32_t vis_row;     // >= 0: vision embedding row (input is a VIS placeholder)
  int32_t kv_page;     // page receiving this row's K/V
  int32_t kv_slot;     // slot within that page
  int32_t out_idx;     // >= 0: write the greedy token to out_tokens[out_idx]
  int32_t chunk_base;  // first attention partial of this row
  int32_t n_chunks;    // pos / 64 + 1
  int32_t logit_row;   // >= 0: dump fp32 logits to logits[logit_row] (parity mode)
  int32_t head_row;    // >= 0: index among rows that need the lm_head
  int32_t pad;
};

// A cascade-attention work item: one KV page (= one 64-position chunk)
// shared by `row_count` query rows whose block tables map that chunk to it.
struct AttnItem {
  int32_t page;
  int32_t chunk;
  int32_t row_begin;   // into ItemRow[]
  int32_t row_count;
  int32_t valid_max;   // keys of the page any of the rows needs (bytes to stage)
  int32_t pad[3];
};
struct ItemRow {
  int32_t row;
  int32_t valid;       // keys of this page visible to the row (causal)
};

struct ModelDims {
  int d, L, H, hd, F, V, n_text, max_pos;
  float eps, attn_scale;
};

// A query tile of the tensor-core prefill attention: rows [row0, row0 + n) of
// the forward are consecutive positions pos0 .. of one sequence whose page
// table starts at ptab[pages].
struct PrefillTile {
  int32_t row0, n, pos0, pages;
};

// Device-side view of a forward pass.
struct Fwd {
  const int32_t* hdr;      // device header: [n_rows, n_items, n_head_rows, 0]
  const RowMeta* rows;
  int n_rows;
  const AttnItem* items;
  int n_items;             // host-side count (eager launches); kernels read hdr[1]
  int item_cap;            // attention CTAs per head (persistent over items)
  const ItemRow* item_rows;
  int* attn_counters;      // [max_rows][H] arrival counters of the fused attention merge
  int n_head_rows;         // rows that need the lm_head
  const int32_t* head_rows;  // row index of each lm_head row
  uint64_t vision_key;
  const uint64_t* vision_keys;  // per-row vision keys (RowMeta.pad indexes them), or null: vision_key
  bool vis_ptrs;                // vision_keys hold device pointers to VIS rows (the vision tower's output)
  // prefill forwards: 64-row query tiles of consecutive positions of one
  // sequence each (several sequences per forward), their page tables; else null
  const PrefillTile* ptiles;
  int n_ptiles;
  const int32_t* ptab;
  // span attention (bf16 chain decode ticks; attn_span.cu): an item is a
  // row group (<= 16 rows sharing pages) and a range of its pages
  // (AttnItem.pad[0] pages listed from span_pages[pad[1]], span_masks: per
  // page the group-local rows that see it | valid-key max << 16); each item
  // row carries (part | last-page position << 16) in item_slots, rows their
  // part count in row_nspans (1: the item writes the attention output)
  bool span_mode;
  const int32_t* item_slots;   // parallel to item_rows
  const int32_t* span_pages;
  const int32_t* span_masks;   // parallel to span_pages
  const int32_t* row_nspans;   // [n_rows]
};

struct Weights {
  void* embed;      // [V][d] WT
  void* lm_head;    // [V][d] WT
  float* final_norm;
  struct Layer {
    float* attn_norm;
    void* wqkv;     // [3d][d] WT (q rows, k rows, v rows)
    void* wo;       // [d][d]
    float* ffn_norm;
    void* wgu;      // [2F][d] (gate rows, then up rows)
    void* wdown;    // [d][F]
  } * layers;
};

struct Workspace {
  float* x;          // [max_rows][d] residual stream (fp32)
  void* xn;          // [max_rows][max(d,F)] staging (XT)
  float* q;          // [max_rows][d]
  void* attn;        // [max_rows][d] (XT)
  float* partial;    // [max_partials][H][hd + 2]
  unsigned long long* part_keys;  // [max_head_rows][max_ctas]
  float* logits;     // [max_logit_rows][V]
  int32_t* out_tokens;
  void* meta;        // device copy of the per-forward metadata
};

// --- programmatic dependent launch -------------------------------------------
extern bool g_pdl;       // engine option "pdl"
extern int g_sk_stages;  // engine option "sk_stages" (5 or 10)
extern int g_sk_splits;  // engine option "sk_splits" (0: cost model)

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// --- kernel launchers (kernels.cu) -----------------------------------------
void launch_init_linear(int dtype, void* w, uint64_t key, size_t n, cudaStream_t s);
void launch_init_norm(float* w, uint64_t key, size_t n, cudaStream_t s);
void launch_embed(int dtype, const Fwd& f, const ModelDims& m, const void* embed, const int32_t* out_tokens,
                  float* x, cudaStream_t s);
void launch_rmsnorm(int dtype, const float* x, const float* w, void* out, int n_rows, int d, int ld_out,
                    float eps, const int32_t* row_index, cudaStream_t s);
void launch_qkv(int dtype, const Fwd& f, const ModelDims& m, const void* w, const void* xn, float* q,
                void* kv_pool, int layer, const float* rope, cudaStream_t s);
void launch_attention(int dtype, const Fwd& f, const ModelDims& m, const float* q, const void* kv_pool,
                      int layer, float* partial, void* attn_out, cudaStream_t s);
// bf16, head_dim 128, f.seq_pages set (prefill_attn.cu)
void launch_prefill_attention(const Fwd& f, const ModelDims& m, const float* q, const void* kv_pool, int layer,
                              void* attn_out, cudaStream_t s);
struct TmaMap;
// bf16, head_dim 128, f.span_mode (attn_span.cu); pool_map: the KV pool as [rows][128] bf16, 64 x 64 boxes
extern int g_span_dbg;
// bf16, head_dim 128, f.ptiles of <= 128 rows (prefill_attn_tc.cu: tcgen05 + TMEM + TMA)
void launch_prefill_attention_tc(const Fwd& f, const ModelDims& m, const TmaMap& pool_map, const float* q, int layer,
                                 void* attn_out, cudaStream_t s,
                                 unsigned long long* trace = nullptr);
void launch_span_attention(const Fwd& f, const ModelDims& m, const TmaMap& pool_map, const TmaMap& pool_map16,
                           const float* q, int layer, float* partial, void* attn_out, cudaStream_t s);
void launch_resid(int dtype, const Fwd& f, int N, int K, const void* w, const void* xin, float* x,
                  cudaStream_t s);
void launch_swiglu(int dtype, const Fwd& f, int F, int K, const void* w, const void* xin, void* act,
                   cudaStream_t s);
void launch_lm_head(int dtype, const Fwd& f, const ModelDims& m, const void* w, const void* xn,
                    unsigned long long* part_keys, float* logits, int32_t* out_tokens, cudaStream_t s);
void launch_finalize(const Fwd& f, const unsigned long long* part_keys, int n_ctas, int32_t* out_tokens,
                     cudaStream_t s);
void launch_page_copy(int dtype, void* pool, int src, int dst, int n_slots, const ModelDims& m,
                      cudaStream_t s);
// plain y[n][N] = x[n][K] . W^T (parity tests)
void launch_gemv_store(int dtype, const void* w, int N, int K, const void* x, int n_rows, float* y,
                       cudaStream_t s);

size_t kv_page_elems(const ModelDims& m);
int lm_head_ctas(const ModelDims& m);

}  // namespace fe
