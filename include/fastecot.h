/*
 * fastecot.h -- C ABI of the B200 Fast-ECoT engine (libfastecot.so).
 *
 * The reference has no FFI: its hot path crosses one Python protocol,
 * `GenerationBackend` (pkg/src/ecot_sched/backends.py:98-110), whose
 * `begin_step(context, prefix, step, prev_content)` the runners call through
 * `_generate_step` (schedulers.py:217-225).  These entry points are what a
 * backend implementing that protocol binds (ctypes in
 * paper_2506_07639_b200/engine.py; a cgo/JNI/N-API stub would bind the same
 * symbols):
 *
 *   encode(instruction, observation)     -> fe_prefill of the context trunk
 *                                           (backends.py:102, :113-117)
 *   begin_step(ctx, prefix, step, prev)  -> fe_seq_fork + fe_prefill of the
 *                                           uncached prefix + fe_submit +
 *                                           fe_run + fe_request_tokens
 *                                           (backends.py:104-110)
 *   StepGenerator.drain()                -> fe_request_tokens (backends.py:93-95)
 *   runner-level batching                -> fe_submit / fe_run: continuous
 *     (_MicroEngine, schedulers.py:244-299;  batcher with the reference's
 *      ParallelSync fan-out :399-420)        action-first admission
 *
 * Conventions: every function returns 0 on success and a non-zero status on
 * failure, with a message retrievable through fe_last_error() (thread-local).
 * No C++ exceptions cross the ABI.  Host pointers are caller-owned; the
 * engine owns weights, the paged KV pool and its work buffers.  All device
 * work is ordered on the engine's CUDA stream; only fe_request_tokens,
 * fe_request_logits and fe_synchronize block the host.
 */
#ifndef FASTECOT_H
#define FASTECOT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fe_engine fe_engine;

enum { FE_F32 = 0, FE_BF16 = 1 };
enum { FE_PRIO_ACTION = 0, FE_PRIO_REASONING = 1 };  /* batching.py:21-22 */

typedef struct fe_config {
  int32_t d_model, n_layers, n_heads, head_dim, d_ffn;
  int32_t vocab;        /* rows of embed / lm_head */
  int32_t n_text;       /* greedy argmax range [0, n_text) */
  int32_t max_pos;      /* rows of the RoPE table */
  float rms_eps;
  float attn_scale;     /* 1/sqrt(head_dim) as fp32 */
  int32_t dtype;        /* FE_F32 (canonical, bit-exact) or FE_BF16 */
  int32_t max_rows;     /* rows per forward pass (prefill chunk) */
  int32_t kv_pages;     /* 64-token pages in the KV pool; 0 = size from free memory */
  int32_t max_slots;    /* capacity of the continuous batcher */
} fe_config;

/* engine lifetime; `rope` = host [max_pos][2][head_dim/2] fp32 (cos, sin) */
int fe_engine_create(const fe_config* cfg, int32_t device, const float* rope, fe_engine** out);
int fe_engine_destroy(fe_engine* e);
int fe_weights_init_random(fe_engine* e, uint64_t seed);
const char* fe_last_error(void);

/* paged KV sequences (64-token pages, refcounted, copy-on-write at forks) */
int fe_seq_create(fe_engine* e, int32_t* seq);
int fe_seq_fork(fe_engine* e, int32_t parent, int32_t len, int32_t* child);
int fe_seq_free(fe_engine* e, int32_t seq);
int fe_seq_len(fe_engine* e, int32_t seq, int32_t* len);

/* append n input ids to `seq` (positions len .. len+n-1); ids equal to
 * `vis_id` take row (pos-1) of the vision embedding seeded by `vision_seed` */
int fe_prefill(fe_engine* e, int32_t seq, const int32_t* ids, int32_t n, uint64_t vision_seed, int32_t vis_id);

/* vision tower + projector: VIS placeholders take the
 * rows a ViT (pre-LayerNorm, `layers` x `heads`, patch `patch` over an
 * img x img synthetic image of the observation) and a 2-layer GELU projector
 * produce, instead of the synthetic embeddings; the patch count must equal
 * the framing's VIS count.  `slots` observations stay cached. */
typedef struct {
  int32_t img, patch, d, layers, heads, mlp, proj_hidden;
  float eps;
} fe_vision_config;
int fe_vision_enable(fe_engine* e, const fe_vision_config* vc, uint64_t seed, int32_t slots);
int fe_vision_encode(fe_engine* e, uint64_t vision_seed, float* out_host);  /* [P][d_model] rows (tests) */

/* batched prefill: seqs[i] gets counts[i] ids (concatenated in `ids`),
 * vision placeholders seeded by vision_seeds[i]; rows of all sequences are
 * packed into as few forwards as the engine holds (one GEMM pass per
 * forward for every trunk of a batched-episode timestep) */
int fe_prefill_batch(fe_engine* e, int32_t n_seqs, const int32_t* seqs, const int32_t* counts, const int32_t* ids,
                     const uint64_t* vision_seeds, int32_t vis_id);

/* the same, and every sequence with want[i] != 0 runs the lm_head on its
 * last row (a branch TAG riding along with its trunk prefill): out[i] = the
 * greedy token after it (synchronous; -1 where want[i] == 0) */
int fe_prefill_batch_heads(fe_engine* e, int32_t n_seqs, const int32_t* seqs, const int32_t* counts,
                           const int32_t* ids, const uint64_t* vision_seeds, int32_t vis_id, const int32_t* want,
                           int32_t* out);

/* reuse-as-draft verification (replaces nothing in the reference: the
 * SyntheticBackend's reuse draw, backends.py:202-204, returns prev_content
 * verbatim; here prev_content is checked as a greedy draft): one batched
 * forward extends seqs[i] by counts[i] ids (concatenated in `ids`); out[k] =
 * greedy token after input k.  Then keep the accepted prefix: */
int fe_verify(fe_engine* e, int32_t n_seqs, const int32_t* seqs, const int32_t* counts, const int32_t* ids,
              int32_t* out);
/* drop positions >= len (pages past the end are released) */
int fe_seq_truncate(fe_engine* e, int32_t seq, int32_t len);

/* continuous batcher: a request decodes `length` greedy tokens on `seq`,
 * the first iteration consuming `first_id` */
int fe_set_slots(fe_engine* e, int32_t slots);
int fe_submit(fe_engine* e, int32_t seq, int32_t first_id, int32_t length, int32_t priority, int32_t* req);
/* run decode iterations until request `stop_req` completes (-1: until idle);
 * per tick: occupancy[t]; completions in order: completed[i] at tick
 * completed_tick[i].  Arrays need room for `cap` entries. */
int fe_run(fe_engine* e, int32_t stop_req, int32_t cap, int32_t* n_ticks, int32_t* occupancy,
           int32_t* completed, int32_t* completed_tick, int32_t* n_completed);
/* lanes: 0 = foreground (highest stream priority; prefills, forks and the
 * calls above), 1 = background (lowest priority; reasoning refresh of the
 * two-stream async scheduler).  Each lane has its own stream, batcher and
 * decode graphs; fe_run_lane locks the engine per tick, so two host threads
 * may drive the two lanes concurrently.  max_ticks <= 0: unbounded. */
int fe_set_slots_lane(fe_engine* e, int32_t lane, int32_t slots);
int fe_submit_lane(fe_engine* e, int32_t lane, int32_t seq, int32_t first_id, int32_t length, int32_t priority,
                   int32_t* req);
int fe_run_lane(fe_engine* e, int32_t lane, int32_t stop_req, int32_t max_ticks, int32_t cap, int32_t* n_ticks,
                int32_t* occupancy, int32_t* completed, int32_t* completed_tick, int32_t* n_completed);
int fe_stream_lane(fe_engine* e, int32_t lane, void** stream);
int fe_request_tokens(fe_engine* e, int32_t req, int32_t* out, int32_t cap);
int fe_request_release(fe_engine* e, int32_t req);
int fe_request_capture_logits(fe_engine* e, int32_t req);  /* parity mode: keep fp32 logits */
int fe_request_logits(fe_engine* e, int32_t req, float* out, int32_t rows);
int fe_in_flight(fe_engine* e, int32_t* n);

int fe_synchronize(fe_engine* e);
int fe_stream(fe_engine* e, void** stream);
/* ticks, forwards, rows, pages used, pages total, page bytes, H2D bytes, D2H bytes, kernel launches */
int fe_stats(fe_engine* e, int64_t* out, int32_t n);
/* CUDA-event timing of launches on the engine stream, per category
 * (0 decode GEMVs, 1 decode attention, 2 decode forwards, 3 prefill forwards):
 * out[3c] = ms, out[3c+1] = launches, out[3c+2] = algorithmic bytes */
int fe_profile(fe_engine* e, int32_t enable);
int fe_profile_read(fe_engine* e, double* out, int32_t n);

/* kernel-level entry points (device pointers, engine stream), for parity tests */
int fe_weight_ptr(fe_engine* e, int32_t tensor, int32_t layer, void** ptr, size_t* bytes);
int fe_memcpy(fe_engine* e, void* dst, const void* src, size_t bytes);  /* any direction, synchronous */
int fe_op_gemv(fe_engine* e, const void* w, int32_t N, int32_t K, const void* x, int32_t rows, float* y);
int fe_op_rmsnorm(fe_engine* e, const float* x, const float* w, void* out, int32_t rows, int32_t d);
/* bf16 tcgen05 GEMM: y[M][N] (fp32) = x[M][K] . w[N][K]^T */
int fe_op_gemm_tc(fe_engine* e, const void* x, const void* w, int32_t M, int32_t N, int32_t K, float* y);
/* bf16 tcgen05 swap-AB decode GEMM (M <= 16 rows): y[M][N] = x[M][K] . w[N][K]^T */
int fe_op_skinny_tc(fe_engine* e, const void* x, const void* w, int32_t M, int32_t N, int32_t K, float* y);
/* diagnostics of the persistent decode-tick kernel (option "mk_trace" = 1):
 * globaltimer ns of the last traced tick, out[(6 ph + k) * grid + cta]: k = 0
 * barrier passed, 1 phase done, 2 last weight load issued, 3 / 4 first / last
 * accumulator ready, 5 segments drained */
int fe_debug_trace(fe_engine* e, uint64_t* out, int32_t n, int32_t* n_phases, int32_t* grid);
/* engine options: "tc_min_rows" (rows from which a forward uses the tcgen05
 * GEMMs, bf16 only), "use_tc" (0/1), "mk" (0/1: persistent decode-tick
 * kernel), "mk_trace", "graphs", "pdl", "sk_mask", "sk_stages", "op_reps",
 * "debug_skip"; tick tuning: "mk_per_cta", "mk_nc_cap", "mk_nc_cap_o" (chunk
 * plans), "mk_pf" (weight stages prefetched across a barrier), "mk_fused"
 * (bit per GEMM: finalise its tiles in-phase), "mk_flags" (diagnostics) */
int fe_set_option(fe_engine* e, const char* key, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* FASTECOT_H */
