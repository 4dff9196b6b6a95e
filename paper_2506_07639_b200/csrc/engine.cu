// Host side of the Fast-ECoT B200 engine: weights, paged KV pool, forward
// passes, the continuous batcher(s) and the C ABI (include/fastecot.h).
//
// Reference anchors: the batcher's admission policy restates the simulated
// `_MicroEngine.tick` (pkg/src/ecot_sched/schedulers.py:277-299: admit
// waiting requests into free slots, action class first then FIFO by seqno;
// every occupied slot emits one token per tick; a slot freed at tick k is
// reusable at k+1).  Token generation itself has no reference counterpart
// (SPEC.md:166, :250): it is the decoder of DESIGN.md.
//
// Lanes.  The engine owns two lanes, each a CUDA stream with its own work
// buffers, metadata ring, decode graphs and continuous batcher; weights, the
// paged KV pool, sequences and the token arena are shared.  Lane 0 (highest
// stream priority) serves prefills and everything synchronous; lane 1
// (lowest priority) serves the background reasoning refresh of the two-stream
// async scheduler (north_star item 4).  Lane 1 orders itself after lane 0's
// prefills/forks with an event; freed KV pages are recycled only after both
// lanes have passed the point of release.
#include "common.cuh"
#include "engine_internal.h"
#include "gemm_tc.h"
#include "vision.h"
#include "decode_mk.h"
#include "../../include/fastecot.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <functional>
#include <mutex>
#include <thread>
#include <chrono>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <functional>
#include <vector>

namespace {

thread_local std::string g_last_error;

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t _e = (x);                                                                  \
    if (_e != cudaSuccess)                                                                 \
      throw Error(std::string(#x) + ": " + cudaGetErrorString(_e) + " @" + std::to_string(__LINE__)); \
  } while (0)

constexpr int kRequestCap = 1024;   // tokens per request (out_tokens arena slot)
constexpr int kMetaRing = 4;
constexpr int kItemRows = 16;       // query rows per cascade work item
constexpr int kLogitRows = 256;
constexpr int kMaxGraphRows = 64;   // decode ticks with <= this many rows replay CUDA graphs
constexpr int kLanes = 2;
constexpr int kLane1Rows = 64;      // background lane: decode rows only

struct MetaLayout {
  size_t o_rows, o_items, o_irows, o_heads, o_pages, o_slots, o_nspans, o_spages, o_smasks, o_ptiles, o_vkeys,
      total;
  int cap_rows, cap_items, cap_irows, cap_pages;
};

struct Seq {
  std::vector<int> pages;
  int len = 0;
  bool live = false;
};

struct Request {
  int seq = -1;
  int first_id = 0;
  int length = 0;
  int produced = 0;
  int priority = 1;
  uint64_t seqno = 0;
  int arena = -1;
  int lane = 0;
  int state = 0;      // 0 waiting, 1 running, 2 done
  bool capture = false;
  int logit_base = 0;  // first row of its logits in the capture buffer
  bool live = false;
};

struct RowIn {
  int seq, pos, tok, tok_src, vis_row, out_idx, logit_row;
  bool head;
  int vk;  // index into the forward's vision seeds (multi-sequence prefill)
};

enum ProfCat { PROF_GEMV = 0, PROF_ATTN = 1, PROF_DECODE_FWD = 2, PROF_PREFILL_FWD = 3, PROF_TICK = 4, PROF_NCAT = 5 };

struct ProfRec {
  int cat;
  cudaEvent_t a, b;
  double bytes;
};

struct GraphSlot {
  bool seen = false;
  cudaGraphExec_t exec = nullptr;
};

struct PendingPage {
  int page;
  cudaEvent_t ev[kLanes];
};

// One stream with everything a forward pass needs.
struct Lane {
  int id = 0;
  cudaStream_t stream = nullptr;
  int max_rows = 0;
  int max_partials = 0;
  int max_items = 0;
  fe::Workspace ws{};
  int* attn_counters = nullptr;
  float* sk_partial = nullptr;
  int* sk_counters = nullptr;
  float* pair_scratch = nullptr;  // stream-K partials of the CTA-pair GEMM
  int* pair_counters = nullptr;
  float* split_scratch = nullptr;  // split-K planes of the CTA-pair GEMM
  size_t split_floats = 0;
  // persistent decode-tick kernel scratch (lane 0)
  float* mk_ss = nullptr;
  unsigned long long* mk_bar = nullptr;
  float* mk_partial = nullptr;
  int* mk_counters = nullptr;
  unsigned long long* mk_keys = nullptr;
  int* mk_grab = nullptr;
  MetaLayout layout{};
  unsigned char* meta_host[kMetaRing] = {};
  cudaEvent_t meta_ev[kMetaRing] = {};
  int meta_next = 0;
  fe::TmaMap map_xn{}, map_attn{}, map_act{};        // 128-row boxes (tile GEMM A operand)
  fe::TmaMap map_xn16{}, map_attn16{}, map_act16{};  // 16-row boxes (skinny GEMM B operand)
  std::unordered_map<long, GraphSlot> graphs;       // key: rows * 4096 + attention item bucket
  cudaEvent_t tick_ev[2] = {};                      // tick pacing (run_lane)
  long pace_n = 0;                                  // ticks recorded for pacing (across run calls)
  // continuous batcher
  int slots = 8;
  std::vector<int> slot_req;
  std::vector<int> waiting;
};

}  // namespace

struct fe_engine {
  fe::ModelDims m{};
  int dtype = 0;
  int device = 0;
  size_t elem = 4;
  int max_slots = 0;
  std::mutex mu;

  // weights
  std::vector<void*> allocs;
  fe::Weights w{};
  std::vector<fe::Weights::Layer> layers;
  float* rope = nullptr;

  // KV pool (shared by the lanes)
  void* kv_pool = nullptr;
  int n_pages = 0;
  size_t page_elems = 0;
  std::vector<int> page_ref;
  std::vector<int> free_pages;
  std::vector<PendingPage> pending_pages;
  std::vector<cudaEvent_t> free_events;
  std::vector<Seq> seqs;
  std::vector<int> free_seqs;
  cudaEvent_t lane0_ev = nullptr;  // lane 0's latest prefill / fork, awaited by lane 1

  // requests and the token arena (shared)
  std::vector<Request> reqs;
  std::vector<int> free_reqs;
  uint64_t seqno = 0;
  std::vector<int> free_arena;
  int32_t* out_tokens = nullptr;
  float* logits = nullptr;  // lane 0 capture buffer
  int logit_next = 0;    // next free row of the logit capture buffer
  int capture_live = 0;  // live requests holding capture rows

  Lane lanes[kLanes];

  // tcgen05 path (bf16)
  struct LayerMaps {
    fe::TmaMap qkv, wo, wgu, wdown;   // 128-row boxes (wgu: 64), skinny A operand / v1 tile GEMM
    fe::TmaMap qkv64, wo64, wdown64;  // 64-row boxes: B operand of the CTA-pair GEMM (wgu shared)
  };
  bool use_tc = false;
  bool tc_pair = true;  // option "tc_pair": CTA-pair persistent GEMM (0: round-1 128x128 tile GEMM)
  bool span_attn = true;  // option "span_attn": tensor-core span attention for chain decode ticks (bf16)
  int span_cap = 8;       // option "span_cap": most page-range parts per row group (1: never split)
  int n_sm = 148;
  fe::TmaMap pool_map{};    // the KV pool as [rows][128] bf16, 64 x 64 boxes (span attention)
  fe::TmaMap pool_map16{};  // same, 64 x 16 boxes (partially filled last pages)
  // vision tower (fe_vision_enable): VIS rows from the observation's image
  std::unique_ptr<fe::Vision> vis;
  std::vector<float*> vis_buf;       // [slots] P x d fp32
  std::vector<uint64_t> vis_seed;
  std::vector<int64_t> vis_stamp;
  int64_t vis_clock = 0;
  int64_t vis_encodes = 0;
  int tc_min_rows = 17;
  // forwards up to this many rows use the skinny GEMM, wider ones the tile
  // GEMM (option "sk_max_rows"; measured in the engine at 7B: skinny ahead
  // up to ~32 rows, the tile GEMM at 56 and for prefill)
  int sk_max_rows = 32;
  // per matrix (QKV, O, gate/up, down; options "sk_rows_*"): rows up to which
  // the skinny swap-AB GEMM is used instead of the CTA-pair GEMM.  The
  // isolated sweeps favour skinny QKV up to 128 rows and gate/up up to 64,
  // but inside config-4 ticks that measured 795 vs 765 ms of decode GEMMs per
  // step, so every matrix switches at 32
  int sk_rows[4] = {32, 32, 32, 32};
  int sk_mask = 31;  // skinny path per matrix: 1 QKV, 2 O, 4 gate/up, 8 down, 16 lm_head
  std::vector<LayerMaps> tc_maps;
  fe::TmaMap map_lm{};
  // persistent decode-tick kernel (bf16 decode ticks of <= 16 rows on lane 0)
  bool mk_on = false;
  int mk_grid = 0;
  fe::MkPlan mk_plans[5] = {};
  void* mk_maps = nullptr;        // device CUtensorMap[4 L + 1]
  const float** mk_norms = nullptr;  // device float*[2 L + 1]
  unsigned long long* mk_trace = nullptr;  // diagnostics: per-phase barrier timestamps of the last tick
  size_t mk_trace_n = 0;
  bool mk_trace_on = false;
  bool pattn_trace_on = false;
  bool fuse_norm = true;  // option "fuse_norm": split-K residual reduces apply the following RMSNorm  // diagnostics: prefill attention stamps into mk_trace (option "pattn_trace")
  int mk_flags = 0;
  int mk_fused = (1 << fe::MK_GU) | (1 << fe::MK_LM);  // option "mk_fused"
  cudaEvent_t mk_ev[kLanes] = {};  // last persistent tick of each lane
  bool mk_ev_used[kLanes] = {};
  int mk_pf_stages = 0;  // 0 = the whole ring
  int mk_per_cta = 4, mk_nc_cap = 8, mk_nc_cap_o = 0;  // chunk plans (mk_make_plans; swept in tools/mk_sweep.sh)
  // per-GEMM chunks per tile (options "mk_nc_qkv" ... "mk_nc_lm"; 0 = the per_cta / cap plan), measured
  // on the B200 (bench config 2, decode tick): QKV and gate/up at 6 (3.062 -> 2.993 ms), down at 9 with
  // the 12-partial straight-line reduction (2.993 -> 2.969 ms); O and lm_head keep their plan
  int mk_nc_force[5] = {6, 0, 6, 9, 0};
  bool graphs_on = true;
  bool lane1_yields = true;
  int lane0_pace = 0;  // option "lane0_pace": lane-0 ticks kept queued (1 or 2; 0: unpaced)
  bool prefill_fa = true;  // option "prefill_fa": tensor-core causal prefill attention (bf16)
  bool prefill_tc = true;  // option "prefill_tc": its tcgen05 kernel (prefill_attn_tc.cu), else mma.sync
  float* op_partial = nullptr;  // fe_op_skinny_tc scratch
  size_t op_bytes = 0;
  int* op_counters = nullptr;
  int op_reps = 1;     // fe_op_skinny_tc: back-to-back launches (device-side timing of one kernel)
  int debug_skip = 0;  // timing experiments only: 1 attention, 2 rmsnorm, 4 layer GEMMs, 8 lm_head

  // stats
  int64_t n_ticks = 0, n_forwards = 0, n_rows_total = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0, n_launches = 0;

  // profiling (fe_profile), lane 0 only
  bool prof_on = false;
  std::vector<ProfRec> prof_recs;
  int prof_used = 0;
  double prof_ms[PROF_NCAT] = {}, prof_bytes[PROF_NCAT] = {};
  int64_t prof_n[PROF_NCAT] = {};

  void* dalloc(size_t bytes) {
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    allocs.push_back(p);
    return p;
  }
};

namespace {

const fe_engine::LayerMaps& EngineMapsDummy() {
  static fe_engine::LayerMaps d{};
  return d;
}

Lane& lane_at(fe_engine* e, int lane) {
  if (lane < 0 || lane >= kLanes) throw Error("lane must be 0 or 1");
  return e->lanes[lane];
}

// ---- KV pages ---------------------------------------------------------------
void reclaim_pages(fe_engine* e) {
  for (size_t i = 0; i < e->pending_pages.size();) {
    PendingPage& pp = e->pending_pages[i];
    bool done = true;
    for (int l = 0; l < kLanes; l++) done = done && cudaEventQuery(pp.ev[l]) == cudaSuccess;
    if (done) {
      e->free_pages.push_back(pp.page);
      for (int l = 0; l < kLanes; l++) e->free_events.push_back(pp.ev[l]);
      pp = e->pending_pages.back();
      e->pending_pages.pop_back();
    } else {
      i++;
    }
  }
}

// Make `need` pages allocatable (waiting for in-flight frees if necessary);
// throws before anything is allocated when the pool cannot supply them.
void ensure_free_pages(fe_engine* e, int need) {
  if (need <= 0 || (int)e->free_pages.size() >= need) return;
  reclaim_pages(e);
  if ((int)e->free_pages.size() < need && !e->pending_pages.empty()) {
    for (int l = 0; l < kLanes; l++) CK(cudaStreamSynchronize(e->lanes[l].stream));
    reclaim_pages(e);
  }
  if ((int)e->free_pages.size() < need)
    throw Error("KV pool exhausted (" + std::to_string(e->n_pages) + " pages, " + std::to_string(need) +
                " needed, " + std::to_string(e->free_pages.size()) + " free)");
}

int alloc_page(fe_engine* e) {
  if (e->free_pages.empty()) reclaim_pages(e);
  if (e->free_pages.empty() && !e->pending_pages.empty()) {
    for (int l = 0; l < kLanes; l++) CK(cudaStreamSynchronize(e->lanes[l].stream));
    reclaim_pages(e);
  }
  if (e->free_pages.empty()) throw Error("KV pool exhausted (" + std::to_string(e->n_pages) + " pages)");
  int p = e->free_pages.back();
  e->free_pages.pop_back();
  e->page_ref[p] = 1;
  return p;
}

cudaEvent_t take_event(fe_engine* e) {
  if (!e->free_events.empty()) {
    cudaEvent_t ev = e->free_events.back();
    e->free_events.pop_back();
    return ev;
  }
  cudaEvent_t ev;
  CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  return ev;
}

// A page whose last reference is dropped may still be read by kernels queued
// on either lane: recycle it once both lanes pass this point.
void release_page(fe_engine* e, int p) {
  if (--e->page_ref[p] != 0) return;
  PendingPage pp;
  pp.page = p;
  for (int l = 0; l < kLanes; l++) {
    pp.ev[l] = take_event(e);
    CK(cudaEventRecord(pp.ev[l], e->lanes[l].stream));
  }
  e->pending_pages.push_back(pp);
}

Seq& seq_at(fe_engine* e, int s) {
  if (s < 0 || s >= (int)e->seqs.size() || !e->seqs[s].live) throw Error("invalid sequence " + std::to_string(s));
  return e->seqs[s];
}

int new_seq(fe_engine* e) {
  int s;
  if (!e->free_seqs.empty()) {
    s = e->free_seqs.back();
    e->free_seqs.pop_back();
  } else {
    s = (int)e->seqs.size();
    e->seqs.emplace_back();
  }
  e->seqs[s] = Seq();
  e->seqs[s].live = true;
  return s;
}

// ---- profiling: CUDA events on lane 0 around launches ------------------------
void flush_profile(fe_engine* e) {
  if (e->prof_used == 0) return;
  CK(cudaStreamSynchronize(e->lanes[0].stream));
  for (int i = 0; i < e->prof_used; i++) {
    const ProfRec& r = e->prof_recs[i];
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    e->prof_ms[r.cat] += ms;
    e->prof_bytes[r.cat] += r.bytes;
    e->prof_n[r.cat]++;
  }
  e->prof_used = 0;
}

int prof_begin(fe_engine* e, const Lane& ln, int cat) {
  if (!e->prof_on || ln.id != 0) return -1;
  if (e->prof_used == (int)e->prof_recs.size()) {
    ProfRec r{};
    CK(cudaEventCreate(&r.a));
    CK(cudaEventCreate(&r.b));
    e->prof_recs.push_back(r);
  }
  const int i = e->prof_used++;
  e->prof_recs[i].cat = cat;
  CK(cudaEventRecord(e->prof_recs[i].a, ln.stream));
  return i;
}

void prof_end(fe_engine* e, const Lane& ln, int i, double bytes) {
  if (i < 0) return;
  e->prof_recs[i].bytes = bytes;
  CK(cudaEventRecord(e->prof_recs[i].b, ln.stream));
}

// Pinned staging buffer for one forward's metadata; waits for the buffer's
// previous H2D copy to finish before reuse.
unsigned char* next_meta(Lane& ln, int* idx) {
  int i = ln.meta_next;
  ln.meta_next = (i + 1) % kMetaRing;
  CK(cudaEventSynchronize(ln.meta_ev[i]));
  *idx = i;
  return ln.meta_host[i];
}

void clear_graphs(fe_engine* e) {
  for (auto& ln : e->lanes) {
    for (auto& g : ln.graphs)
      if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    ln.graphs.clear();
  }
}

// Chunk plans of the persistent decode-tick kernel's GEMMs (options "mk_per_cta",
// "mk_nc_cap" retune them; the partial buffers are sized for any plan).
void mk_make_plans(fe_engine* e) {
  const fe::ModelDims& m = e->m;
  const int G = e->mk_grid, pc = e->mk_per_cta, cap = e->mk_nc_cap;
  e->mk_plans[fe::MK_QKV] = fe::mk_plan(3 * m.d / 128, m.d / 64, G, pc, cap);
  e->mk_plans[fe::MK_O] = fe::mk_plan(m.d / 128, m.d / 64, G, pc, e->mk_nc_cap_o > 0 ? e->mk_nc_cap_o : cap);
  e->mk_plans[fe::MK_GU] = fe::mk_plan(m.F / 64, m.d / 64, G, pc, cap);
  e->mk_plans[fe::MK_DOWN] = fe::mk_plan(m.d / 128, m.F / 64, G, pc, cap);
  e->mk_plans[fe::MK_LM] = fe::mk_plan((m.V + 127) / 128, m.d / 64, G, pc, cap);
  for (int i = 0; i < 5; i++) {
    fe::MkPlan& p = e->mk_plans[i];
    if (e->mk_nc_force[i] > 0) {
      p.nc = std::max(1, std::min({e->mk_nc_force[i], 16, std::max(1, p.kb_total / 4)}));
      p.chunks = p.tiles * p.nc;
    }
  }
}

// ---- forward pass -----------------------------------------------------------
// The persistent decode-tick kernel takes bf16 decode ticks of <= 16 rows on
// lane 0 where every row samples a token (it needs every SM: one lane only).
bool mk_eligible(fe_engine* e, const Lane& ln, const fe::Fwd& f, int n) {
  (void)ln;
  return e->mk_on && n <= 16 && f.n_head_rows == n && e->debug_skip == 0;
}

// The kernel sequence of one forward pass (eager or under graph capture).
template <typename GB>
void launch_layers(fe_engine* e, Lane& ln, const fe::Fwd& f, int n, bool decode, double kv_bytes, GB gemv_bytes,
                   double flops = 0.0) {
  const fe::ModelDims& m = e->m;
  cudaStream_t st = ln.stream;
  const int dt = e->dtype;
  fe::Workspace& ws = ln.ws;
  const int whole = prof_begin(e, ln, decode ? PROF_DECODE_FWD : PROF_PREFILL_FWD);
  if (decode && mk_eligible(e, ln, f, n)) {
    // one persistent kernel for the whole tick (decode_mk.cu)
    fe::MkLaunch k{};
    k.grid = e->mk_grid;
    for (int i = 0; i < 5; i++) k.plan[i] = e->mk_plans[i];
    k.wmaps = e->mk_maps;
    k.norms = e->mk_norms;
    k.map_xg = ln.map_xn16;
    k.map_attn = ln.map_attn16;
    k.map_act = ln.map_act16;
    k.d = m.d; k.F = m.F; k.H = m.H; k.L = m.L; k.V = m.V; k.n_text = m.n_text;
    k.eps = m.eps;
    k.scale_log2 = m.attn_scale * 1.4426950408889634f;
    k.hdr = f.hdr; k.rows = f.rows; k.items = f.items; k.item_rows = f.item_rows; k.B = n;
    k.embed = (const __nv_bfloat16*)e->w.embed;
    k.out_tokens = e->out_tokens;
    k.x = ws.x; k.xg = (__nv_bfloat16*)ws.xn; k.ss = ln.mk_ss; k.q = ws.q; k.attn = (__nv_bfloat16*)ws.attn;
    k.kv_pool = (__nv_bfloat16*)e->kv_pool; k.page_elems = e->page_elems; k.rope = e->rope;
    k.partial = ln.mk_partial; k.counters = ln.mk_counters;
    k.apartial = ws.partial; k.acounters = f.attn_counters;
    k.part_keys = ln.mk_keys; k.logits = ws.logits; k.bar = ln.mk_bar;
    k.trace = e->mk_trace_on ? e->mk_trace : nullptr;
    k.grab = ln.mk_grab;
    k.flags = e->mk_flags;
    k.fused = e->mk_fused;
    k.pf_stages = e->mk_pf_stages;
    const int p = prof_begin(e, ln, PROF_TICK);
    fe::launch_decode_mk(k, st);
    // algorithmic bytes of the tick: every weight once, the K/V pages the
    // cascade items stage in every layer (shared pages once per head;
    // `kv_bytes` is one layer's), the new K/V rows
    const double el = (double)e->elem;
    const double w_bytes = (double)m.L * (4.0 * m.d * m.d + 3.0 * m.F * m.d) * el + (double)m.V * m.d * el;
    const double kv_write = (double)n * m.L * 2.0 * m.d * el;
    prof_end(e, ln, p, w_bytes + (double)m.L * kv_bytes + kv_write);
    prof_end(e, ln, whole, 0.0);
    return;
  }
  fe::launch_embed(dt, f, m, e->w.embed, e->out_tokens, ws.x, st);
  // bf16: the persistent swap-AB tcgen05 GEMM (decode batches of any width
  // and, up to `sk_max_rows`, prefill), else the tile tcgen05 GEMM; fp32: the
  // canonical CUDA-core GEMV
  const int sk_cap = std::min(e->sk_max_rows, fe::skinny_max_rows());
  auto sk_on = [&](int bit) {
    return e->use_tc && n <= std::min(sk_cap, e->sk_rows[bit]) && (e->sk_mask >> bit & 1);
  };
  auto tc_on = [&](int bit) { return e->use_tc && !sk_on(bit) && n >= e->tc_min_rows; };
  auto tc_launch = [&](int epi, int N, int K) {
    fe::TcLaunch t{};
    t.M = n; t.N = N; t.K = K; t.epi = epi;
    t.y = ws.x; t.ldy = m.d;
    t.act = (__nv_bfloat16*)ws.attn; t.F = m.F;
    t.q = ws.q; t.kv_pool = (__nv_bfloat16*)e->kv_pool; t.page_elems = e->page_elems;
    t.rope = e->rope; t.rows = f.rows; t.H = m.H; t.hd = m.hd; t.d = m.d;
    t.sk_scratch = ln.pair_scratch; t.sk_counters = ln.pair_counters;
    t.split_scratch = ln.split_scratch; t.split_floats = ln.split_floats;
    return t;
  };
  auto sk_launch = [&](int epi, int N, int K) {
    fe::SkLaunch t{};
    t.N = N; t.K = K; t.B = n; t.epi = epi;
    t.partial = ln.sk_partial; t.counters = ln.sk_counters;
    t.y = ws.x; t.ldy = m.d;
    t.act = (__nv_bfloat16*)ws.attn; t.F = m.F;
    t.q = ws.q; t.kv_pool = (__nv_bfloat16*)e->kv_pool; t.page_elems = e->page_elems;
    t.rope = e->rope; t.rows = f.rows; t.head_rows = f.head_rows; t.H = m.H; t.hd = m.hd; t.d = m.d;
    t.part_keys = ws.part_keys; t.logits = ws.logits; t.V = m.V; t.n_text = m.n_text;
    return t;
  };
  // a split-K residual GEMM (O, down) can apply the RMSNorm that follows it in
  // its reduce (launch_gemm_tc returns true); the norm launch is then skipped
  bool normed = false;
  auto with_norm = [&](fe::TcLaunch t, const float* w) {
    if (dt == FE_BF16 && w && e->fuse_norm && !(e->debug_skip & 2)) {
      t.norm_w = w;
      t.norm_out = (__nv_bfloat16*)ws.xn;
      t.norm_eps = m.eps;
    }
    return t;
  };
  for (int l = 0; l < m.L; l++) {
    const fe::Weights::Layer& ly = e->layers[l];
    const auto& mp = e->tc_maps.empty() ? EngineMapsDummy() : e->tc_maps[l];
    const size_t layer_off = (size_t)l * 2 * m.H * FE_PAGE * m.hd;
    const bool skip_norm = e->debug_skip & 2, skip_gemm = e->debug_skip & 4;
    int p;
    if (!skip_norm && !normed) fe::launch_rmsnorm(dt, ws.x, ly.attn_norm, ws.xn, n, m.d, m.d, m.eps, nullptr, st);
    normed = false;
    p = decode ? prof_begin(e, ln, PROF_GEMV) : -1;
    if (skip_gemm) {
    } else if (sk_on(0)) {
      fe::SkLaunch t = sk_launch(fe::TC_QKV, 3 * m.d, m.d);
      t.layer_off = layer_off;
      fe::launch_skinny_tc(mp.qkv, ln.map_xn16, t, st);
    } else if (tc_on(0)) {
      fe::TcLaunch t = tc_launch(fe::TC_QKV, 3 * m.d, m.d);
      t.layer_off = layer_off;
      if (e->tc_pair) fe::launch_gemm_tc(ln.map_xn, mp.qkv64, t, st);
      else fe::launch_gemm_tc_v1(ln.map_xn, mp.qkv, t, st);
    } else {
      fe::launch_qkv(dt, f, m, ly.wqkv, ws.xn, ws.q, e->kv_pool, l, e->rope, st);
    }
    prof_end(e, ln, p, gemv_bytes(3.0 * m.d, m.d, n));
    p = decode ? prof_begin(e, ln, PROF_ATTN) : -1;
    if (e->debug_skip & 1) {
    } else if (f.span_mode) {
      fe::launch_span_attention(f, m, e->pool_map, e->pool_map16, ws.q, l, ws.partial, ws.attn, st);
    } else if (f.ptiles && dt == FE_BF16 && m.hd == 128 && e->prefill_fa) {
      if (e->prefill_tc && e->use_tc) fe::launch_prefill_attention_tc(f, m, e->pool_map, ws.q, l, ws.attn, st,
                                                                        e->pattn_trace_on ? e->mk_trace : nullptr);
      else fe::launch_prefill_attention(f, m, ws.q, e->kv_pool, l, ws.attn, st);
    } else {
      fe::launch_attention(dt, f, m, ws.q, e->kv_pool, l, ws.partial, ws.attn, st);
    }
    prof_end(e, ln, p, kv_bytes);
    p = decode ? prof_begin(e, ln, PROF_GEMV) : -1;
    if (skip_gemm) {
    } else if (sk_on(1)) fe::launch_skinny_tc(mp.wo, ln.map_attn16, sk_launch(fe::TC_RESID, m.d, m.d), st);
    else if (tc_on(1) && e->tc_pair)
      normed = fe::launch_gemm_tc(ln.map_attn, mp.wo64, with_norm(tc_launch(fe::TC_RESID, m.d, m.d), ly.ffn_norm), st);
    else if (tc_on(1)) fe::launch_gemm_tc_v1(ln.map_attn, mp.wo, tc_launch(fe::TC_RESID, m.d, m.d), st);
    else fe::launch_resid(dt, f, m.d, m.d, ly.wo, ws.attn, ws.x, st);
    prof_end(e, ln, p, gemv_bytes(m.d, m.d, n));
    if (!skip_norm && !normed) fe::launch_rmsnorm(dt, ws.x, ly.ffn_norm, ws.xn, n, m.d, m.d, m.eps, nullptr, st);
    normed = false;
    p = decode ? prof_begin(e, ln, PROF_GEMV) : -1;
    if (skip_gemm) {
    } else if (sk_on(2)) fe::launch_skinny_tc(mp.wgu, ln.map_xn16, sk_launch(fe::TC_SWIGLU, 2 * m.F, m.d), st);
    else if (tc_on(2) && e->tc_pair) fe::launch_gemm_tc(ln.map_xn, mp.wgu, tc_launch(fe::TC_SWIGLU, 2 * m.F, m.d), st);
    else if (tc_on(2)) fe::launch_gemm_tc_v1(ln.map_xn, mp.wgu, tc_launch(fe::TC_SWIGLU, 2 * m.F, m.d), st);
    else fe::launch_swiglu(dt, f, m.F, m.d, ly.wgu, ws.xn, ws.attn /* reused as the SwiGLU activation */, st);
    prof_end(e, ln, p, gemv_bytes(2.0 * m.F, m.d, n));
    p = decode ? prof_begin(e, ln, PROF_GEMV) : -1;
    if (skip_gemm) {
    } else if (sk_on(3)) fe::launch_skinny_tc(mp.wdown, ln.map_act16, sk_launch(fe::TC_RESID, m.d, m.F), st);
    else if (tc_on(3) && e->tc_pair)
      normed = fe::launch_gemm_tc(ln.map_act, mp.wdown64,
                                  with_norm(tc_launch(fe::TC_RESID, m.d, m.F),
                                            l + 1 < m.L ? e->layers[l + 1].attn_norm : nullptr), st);
    else if (tc_on(3)) fe::launch_gemm_tc_v1(ln.map_act, mp.wdown, tc_launch(fe::TC_RESID, m.d, m.F), st);
    else fe::launch_resid(dt, f, m.d, m.F, ly.wdown, ws.attn, ws.x, st);
    prof_end(e, ln, p, gemv_bytes(m.d, m.F, n));
  }
  if (f.n_head_rows > 0 && !(e->debug_skip & 8)) {
    fe::launch_rmsnorm(dt, ws.x, e->w.final_norm, ws.xn, f.n_head_rows, m.d, m.d, m.eps, f.head_rows, st);
    const int p = prof_begin(e, ln, PROF_GEMV);
    if (e->use_tc && (e->sk_mask >> 4 & 1) && f.n_head_rows <= fe::skinny_max_rows()) {
      fe::SkLaunch t = sk_launch(fe::TC_ARGMAX, m.V, m.d);
      t.B = f.n_head_rows;
      fe::launch_skinny_tc(e->map_lm, ln.map_xn16, t, st);
      fe::launch_finalize(f, ws.part_keys, fe::skinny_tiles(fe::TC_ARGMAX, m.V, m.F), e->out_tokens, st);
    } else {
      fe::launch_lm_head(dt, f, m, e->w.lm_head, ws.xn, ws.part_keys, ws.logits, e->out_tokens, st);
    }
    prof_end(e, ln, p, gemv_bytes(m.V, m.d, f.n_head_rows));
  }
  prof_end(e, ln, whole, decode ? 0.0 : flops);  // prefill: algorithmic FLOPs (the profile's "bytes" slot)
}

// One forward pass over `rows` on a lane (positions must extend each
// sequence contiguously, in order).  Builds row metadata and the cascade work
// list, then launches the layer stack (or replays the lane's decode graph).
void forward(fe_engine* e, Lane& ln, const std::vector<RowIn>& rows, uint64_t vision_seed,
             const std::vector<uint64_t>* vseeds = nullptr, bool vis_ptrs = false, bool prefill_rows = false) {
  const fe::ModelDims& m = e->m;
  const int n = (int)rows.size();
  if (n == 0) return;
  if (n > ln.max_rows) throw Error("forward: too many rows for lane " + std::to_string(ln.id));
  if (e->prof_on && e->prof_used > 8192) flush_profile(e);  // only between forwards: all records closed
  if (ln.id != 0) CK(cudaStreamWaitEvent(ln.stream, e->lane0_ev, 0));  // trunks prefilled / forked on lane 0

  // Pass 1: validate every row and count the pages this forward appends,
  // without touching any sequence -- a rejected forward (bad position, shared
  // page, pool exhausted, workspace too small) leaves the engine unchanged.
  std::unordered_map<int, std::pair<int, int>> vlen;  // seq -> (length, pages) as the rows extend it
  int new_pages = 0, chunk_need = 0;
  for (int i = 0; i < n; i++) {
    const RowIn& r = rows[i];
    const Seq& s = seq_at(e, r.seq);
    auto it = vlen.find(r.seq);
    const int len = it == vlen.end() ? s.len : it->second.first;
    int np = it == vlen.end() ? (int)s.pages.size() : it->second.second;
    if (r.pos != len) throw Error("forward: non-contiguous append");
    if (r.pos >= m.max_pos) throw Error("forward: position beyond max_pos");
    const int pg = r.pos / FE_PAGE;
    if (pg == np) {
      np++;
      new_pages++;
    } else if (pg < (int)s.pages.size() && e->page_ref[s.pages[pg]] != 1) {
      throw Error("forward: write into a shared page");
    }
    vlen[r.seq] = {r.pos + 1, np};
    chunk_need += pg + 1;
  }
  if (chunk_need > ln.max_partials) throw Error("forward: partial workspace too small");
  ensure_free_pages(e, new_pages);

  // Pass 2: commit (cannot fail); undone below if a later check rejects.
  std::vector<std::tuple<int, int, int>> undo;  // seq, length, pages before this forward
  for (const auto& kv : vlen) {
    const Seq& s = e->seqs[kv.first];
    undo.emplace_back(kv.first, s.len, (int)s.pages.size());
  }
  auto rollback = [&]() {
    for (const auto& u : undo) {
      Seq& s = e->seqs[std::get<0>(u)];
      while ((int)s.pages.size() > std::get<2>(u)) {
        release_page(e, s.pages.back());
        s.pages.pop_back();
      }
      s.len = std::get<1>(u);
    }
  };
  std::vector<fe::RowMeta> meta(n);
  std::vector<int32_t> head_rows;
  int chunk_total = 0;
  for (int i = 0; i < n; i++) {
    const RowIn& r = rows[i];
    Seq& s = e->seqs[r.seq];
    const int pg = r.pos / FE_PAGE;
    if (pg == (int)s.pages.size()) s.pages.push_back(alloc_page(e));
    s.len = r.pos + 1;
    fe::RowMeta& mm = meta[i];
    mm.pos = r.pos;
    mm.tok = r.tok;
    mm.tok_src = r.tok_src;
    mm.vis_row = r.vis_row;
    mm.kv_page = s.pages[pg];
    mm.kv_slot = r.pos % FE_PAGE;
    mm.out_idx = r.out_idx;
    mm.chunk_base = chunk_total;
    mm.n_chunks = pg + 1;
    mm.logit_row = r.logit_row;
    mm.head_row = -1;
    mm.pad = vseeds ? r.vk : 0;
    chunk_total += pg + 1;
    if (r.head) {
      mm.head_row = (int)head_rows.size();
      head_rows.push_back(i);
    }
  }

  // cascade work list: group rows by the physical page their chunk maps to.
  // Rows sharing a trunk point at the same pages, so each shared page is
  // staged once per (page, head) CTA and serves all of them.
  std::map<int, std::vector<std::pair<int, int>>> by_page;  // page -> (row, valid)
  std::unordered_map<int, int> page_chunk;
  for (int i = 0; i < n; i++) {
    const Seq& s = e->seqs[rows[i].seq];
    const int pos = rows[i].pos;
    for (int c = 0; c <= pos / FE_PAGE; c++) {
      const int pg = s.pages[c];
      by_page[pg].push_back({i, std::min(FE_PAGE, pos + 1 - c * FE_PAGE)});
      page_chunk[pg] = c;
    }
  }
  // span mode (bf16 chain decode ticks, attn_span.cu): runs of consecutive
  // pages with the same rows, every page but the last full for all of them
  int n_head = 0;
  for (const RowIn& r : rows) n_head += r.head ? 1 : 0;
  const bool span_mode = !prefill_rows && n_head > 0 && e->span_attn && e->use_tc && m.hd == 128 &&
                         !(e->mk_on && n <= 16 && n_head == n && e->debug_skip == 0);
  std::vector<fe::AttnItem> items;
  std::vector<fe::ItemRow> irows;
  std::vector<int32_t> islots, nspans, spages, smasks;
  if (span_mode) {
    // Row groups (attn_span.cu): rows connected through shared pages (a trunk
    // and the branches forked off it), <= 16 per group; a group's unit walks
    // the union of its rows' pages once per head with one softmax state per
    // row, so a row's whole attention is one unit -- no partials -- unless
    // the group's pages are split into `parts` ranges to fill the GPU.
    std::vector<int> parent(n);
    for (int i = 0; i < n; i++) parent[i] = i;
    std::function<int(int)> find = [&](int x) { return parent[x] == x ? x : parent[x] = find(parent[x]); };
    for (auto& kv : by_page)
      for (size_t k = 1; k < kv.second.size(); k++) {
        const int ra = find(kv.second[0].first), rb = find(kv.second[k].first);
        if (ra != rb) parent[std::max(ra, rb)] = std::min(ra, rb);
      }
    std::map<int, std::vector<int>> comps;  // root -> rows (ascending)
    for (int i = 0; i < n; i++) comps[find(i)].push_back(i);
    std::vector<std::vector<int>> groups;
    for (auto& kv : comps)
      for (size_t b = 0; b < kv.second.size(); b += kItemRows)
        groups.emplace_back(kv.second.begin() + b, kv.second.begin() + std::min(kv.second.size(), b + kItemRows));
    // page-range splits: enough units for ~4 CTAs per SM
    const int target = 4 * e->n_sm;
    const int base_units = (int)groups.size() * m.H;
    const int want_parts = std::max(1, std::min(e->span_cap, (target + base_units - 1) / base_units));
    nspans.assign(n, 0);
    for (const auto& grp : groups) {
      // the union of the group's pages in chunk order, with per page the rows that see it
      std::map<std::pair<int, int>, std::pair<uint32_t, int>> pg;  // (chunk, page) -> (row mask, valid max)
      std::vector<int> last_chunk(grp.size());
      for (size_t k = 0; k < grp.size(); k++) {
        const Seq& sq = e->seqs[rows[grp[k]].seq];
        const int pos = rows[grp[k]].pos;
        last_chunk[k] = pos / FE_PAGE;
        for (int c = 0; c <= last_chunk[k]; c++) {
          auto& ent = pg[{c, sq.pages[c]}];
          ent.first |= 1u << k;
          ent.second = std::max(ent.second, std::min(FE_PAGE, pos + 1 - c * FE_PAGE));
        }
      }
      std::vector<std::pair<int, int>> plist;  // (chunk, page)
      for (auto& kv : pg) plist.push_back(kv.first);
      const int np = (int)plist.size();
      // a row's partial slots are its n_chunks (chunk_base ..): parts <= every row's chunk count
      int parts = std::min(want_parts, np);
      for (size_t k = 0; k < grp.size(); k++) parts = std::min(parts, last_chunk[k] + 1);
      for (int part = 0; part < parts; part++) {
        const int p0 = (int)((long)np * part / parts), p1 = (int)((long)np * (part + 1) / parts);
        fe::AttnItem it;
        it.page = plist[p0].second;
        it.chunk = plist[p0].first;
        it.row_begin = (int)irows.size();
        it.row_count = (int)grp.size();
        it.valid_max = 0;
        it.pad[0] = p1 - p0;
        it.pad[1] = (int)spages.size();
        it.pad[2] = 0;
        for (int j = p0; j < p1; j++) {
          const auto& ent = pg[plist[j]];
          spages.push_back(plist[j].second);
          smasks.push_back((int32_t)(ent.first | ((uint32_t)ent.second << 16)));
          it.valid_max = std::max(it.valid_max, ent.second);
        }
        for (size_t k = 0; k < grp.size(); k++) {
          const int row = grp[k];
          // the row's last page inside this part (position in the part's list), else -1
          int lastpos = -1, valid = FE_PAGE;
          const Seq& sq = e->seqs[rows[row].seq];
          for (int j = p0; j < p1; j++)
            if (plist[j].first == last_chunk[k] && plist[j].second == sq.pages[last_chunk[k]]) {
              lastpos = j - p0;
              valid = rows[row].pos + 1 - last_chunk[k] * FE_PAGE;
            }
          irows.push_back({row, valid});
          islots.push_back(part | (lastpos << 16));
        }
        items.push_back(it);
      }
      for (int row : grp) nspans[row] = parts;
    }
  } else {
    for (auto& kv : by_page) {
      const auto& lst = kv.second;
      for (size_t b = 0; b < lst.size(); b += kItemRows) {
        fe::AttnItem it;
        it.page = kv.first;
        it.chunk = page_chunk[kv.first];
        it.row_begin = (int)irows.size();
        it.row_count = (int)std::min<size_t>(kItemRows, lst.size() - b);
        it.valid_max = 0;
        it.pad[0] = it.pad[1] = it.pad[2] = 0;
        for (int j = 0; j < it.row_count; j++) {
          irows.push_back({lst[b + j].first, lst[b + j].second});
          it.valid_max = std::max(it.valid_max, lst[b + j].second);
        }
        items.push_back(it);
      }
    }
  }

  // Metadata at fixed offsets of the lane's device buffer (header, rows,
  // items, item rows, head rows) so a captured decode graph can be replayed
  // with new contents: counts that vary per tick are read on device.
  const MetaLayout& L = ln.layout;
  if (n > L.cap_rows || (int)items.size() > L.cap_items || (int)irows.size() > L.cap_irows) {
    rollback();
    throw Error("forward: metadata capacity exceeded");
  }
  int mi;
  unsigned char* hbuf = next_meta(ln, &mi);
  int32_t* hdr = reinterpret_cast<int32_t*>(hbuf);
  hdr[0] = n;
  hdr[1] = (int)items.size();
  hdr[2] = (int)head_rows.size();
  hdr[3] = 0;
  std::memcpy(hbuf + L.o_rows, meta.data(), sizeof(fe::RowMeta) * n);
  std::memcpy(hbuf + L.o_items, items.data(), sizeof(fe::AttnItem) * items.size());
  std::memcpy(hbuf + L.o_irows, irows.data(), sizeof(fe::ItemRow) * irows.size());
  std::memcpy(hbuf + L.o_heads, head_rows.data(), sizeof(int32_t) * head_rows.size());
  unsigned char* dbuf = (unsigned char*)ln.ws.meta;
  size_t h2d = 0;
  auto copy = [&](size_t off, size_t bytes) {
    if (bytes == 0) return;
    CK(cudaMemcpyAsync(dbuf + off, hbuf + off, bytes, cudaMemcpyHostToDevice, ln.stream));
    h2d += bytes;
  };
  copy(0, L.o_rows + sizeof(fe::RowMeta) * n);  // header + rows
  copy(L.o_items, sizeof(fe::AttnItem) * items.size());
  copy(L.o_irows, sizeof(fe::ItemRow) * irows.size());
  copy(L.o_heads, sizeof(int32_t) * head_rows.size());
  if (span_mode) {
    std::memcpy(hbuf + L.o_slots, islots.data(), sizeof(int32_t) * islots.size());
    std::memcpy(hbuf + L.o_nspans, nspans.data(), sizeof(int32_t) * nspans.size());
    std::memcpy(hbuf + L.o_spages, spages.data(), sizeof(int32_t) * spages.size());
    std::memcpy(hbuf + L.o_smasks, smasks.data(), sizeof(int32_t) * smasks.size());
    copy(L.o_smasks, sizeof(int32_t) * smasks.size());
    copy(L.o_slots, sizeof(int32_t) * islots.size());
    copy(L.o_nspans, sizeof(int32_t) * nspans.size());
    copy(L.o_spages, sizeof(int32_t) * spages.size());
  }
  // prefill forwards (no lm_head rows): runs of consecutive positions of one
  // sequence, cut into 64-row query tiles with their sequence's page table,
  // for the tensor-core causal attention (prefill_attn.cu; several trunks per
  // forward in a batched prefill)
  std::vector<fe::PrefillTile> ptiles;
  std::vector<int32_t> ptab;
  if ((head_rows.empty() || prefill_rows) && !span_mode) {
    for (int i = 0; i < n;) {
      int j = i + 1;
      while (j < n && rows[j].seq == rows[i].seq && rows[j].pos == rows[j - 1].pos + 1) j++;
      const Seq& sq = e->seqs[rows[i].seq];
      const int np = rows[j - 1].pos / FE_PAGE + 1;
      const int off = (int)ptab.size();
      ptab.insert(ptab.end(), sq.pages.begin(), sq.pages.begin() + np);
      const int tr = e->prefill_tc && e->use_tc ? 128 : 64;  // query rows per attention tile
      for (int t = i; t < j; t += tr) ptiles.push_back({t, std::min(tr, j - t), rows[t].pos, off});
      i = j;
    }
    if ((int)ptab.size() > ln.max_partials) ptiles.clear();  // table does not fit: cascade kernel
    else {
      std::memcpy(hbuf + L.o_spages, ptab.data(), sizeof(int32_t) * ptab.size());
      std::memcpy(hbuf + L.o_ptiles, ptiles.data(), sizeof(fe::PrefillTile) * ptiles.size());
      copy(L.o_spages, sizeof(int32_t) * ptab.size());
      copy(L.o_ptiles, sizeof(fe::PrefillTile) * ptiles.size());
    }
  }
  if (vseeds) {
    std::vector<uint64_t> keys(vseeds->size());
    for (size_t k = 0; k < keys.size(); k++)
      keys[k] = vis_ptrs ? (*vseeds)[k] : fe::tensor_key((*vseeds)[k], 4 /* T_VISION */);
    std::memcpy(hbuf + L.o_vkeys, keys.data(), 8 * keys.size());
    copy(L.o_vkeys, 8 * keys.size());
  }
  CK(cudaEventRecord(ln.meta_ev[mi], ln.stream));
  e->h2d_bytes += h2d;

  fe::Fwd f{};
  f.hdr = reinterpret_cast<const int32_t*>(dbuf);
  f.rows = (const fe::RowMeta*)(dbuf + L.o_rows);
  f.n_rows = n;
  f.items = (const fe::AttnItem*)(dbuf + L.o_items);
  f.n_items = (int)items.size();
  // one attention CTA per (item, head); decode graphs are keyed by (rows,
  // item bucket of 8) so the grid tracks the item count without re-capture
  // every tick (CTAs beyond the device-side count exit immediately)
  const int item_bucket = ((int)items.size() + 7) / 8;
  f.item_cap = items.empty() ? 0 : (head_rows.empty() ? (int)items.size() : item_bucket * 8);
  f.item_rows = (const fe::ItemRow*)(dbuf + L.o_irows);
  f.n_head_rows = (int)head_rows.size();
  f.head_rows = (const int32_t*)(dbuf + L.o_heads);
  f.attn_counters = ln.attn_counters;
  f.vision_key = fe::tensor_key(vision_seed, 4 /* T_VISION */);
  f.ptiles = ptiles.empty() ? nullptr : (const fe::PrefillTile*)(dbuf + L.o_ptiles);
  f.n_ptiles = (int)ptiles.size();
  f.ptab = (const int32_t*)(dbuf + L.o_spages);
  f.vision_keys = vseeds ? (const uint64_t*)(dbuf + L.o_vkeys) : nullptr;
  f.vis_ptrs = vis_ptrs;
  f.span_mode = span_mode;
  f.item_slots = (const int32_t*)(dbuf + L.o_slots);
  f.row_nspans = (const int32_t*)(dbuf + L.o_nspans);
  f.span_pages = (const int32_t*)(dbuf + L.o_spages);
  f.span_masks = (const int32_t*)(dbuf + L.o_smasks);

  // a prefill forward may carry lm_head rows (a branch's TAG riding along with
  // its trunk): it is still a prefill (prefill attention tiles, no graph)
  const bool decode = f.n_head_rows > 0 && !prefill_rows;
  // algorithmic FLOPs of the forward (prefill roofline): every row through
  // every linear, causal attention over its own prefix, lm_head rows
  double fwd_flops = 0.0;
  {
    const double lin = (double)m.L * (4.0 * m.d * m.d + 3.0 * m.d * m.F);
    fwd_flops = 2.0 * n * lin + 2.0 * f.n_head_rows * (double)m.V * m.d;
    for (const RowIn& r : rows) fwd_flops += 4.0 * (r.pos + 1) * (double)m.d * m.L;
  }
  const double el = (double)e->elem;
  // algorithmic bytes of one GEMV launch: weights + staged input + fp32 output
  auto gemv_bytes = [&](double N, double K, int rws) { return N * K * el + rws * K * el + rws * N * 4.0; };
  double kv_bytes = 0;  // K+V bytes the cascade items stage (each shared page once per head)
  for (const auto& it : items)
    if (!span_mode) kv_bytes += 2.0 * it.valid_max * m.hd * m.H * el;
  for (size_t j = 0; j < smasks.size(); j++) kv_bytes += 2.0 * ((uint32_t)smasks[j] >> 16) * m.hd * m.H * el;

  // decode ticks replay a CUDA graph per (rows, item bucket), captured on the
  // second tick with that key; prefill and profiled runs launch eagerly
  const bool graphable = decode && e->graphs_on && !(e->prof_on && ln.id == 0) && n <= kMaxGraphRows;
  const long key = (long)n * 4096 + item_bucket;
  auto it_g = ln.graphs.find(key);
  // a persistent tick needs every SM: it never overlaps the other lane's
  // persistent tick (grid-barrier deadlock); order them with events
  const bool mk_tick = decode && mk_eligible(e, ln, f, n);
  if (mk_tick && e->mk_ev_used[1 - ln.id]) CK(cudaStreamWaitEvent(ln.stream, e->mk_ev[1 - ln.id], 0));
  if (graphable && it_g != ln.graphs.end() && it_g->second.exec) {
    CK(cudaGraphLaunch(it_g->second.exec, ln.stream));
  } else if (graphable && it_g != ln.graphs.end() && it_g->second.seen) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(ln.stream, cudaStreamCaptureModeThreadLocal));
    launch_layers(e, ln, f, n, decode, kv_bytes, gemv_bytes, fwd_flops);
    CK(cudaStreamEndCapture(ln.stream, &g));
    CK(cudaGraphInstantiate(&it_g->second.exec, g, 0));
    CK(cudaGraphDestroy(g));
    CK(cudaGraphLaunch(it_g->second.exec, ln.stream));
  } else {
    if (graphable) ln.graphs[key].seen = true;
    launch_layers(e, ln, f, n, decode, kv_bytes, gemv_bytes, fwd_flops);
  }
  CK(cudaGetLastError());
  if (mk_tick) {
    CK(cudaEventRecord(e->mk_ev[ln.id], ln.stream));
    e->mk_ev_used[ln.id] = true;
  }
  const int attn_kernels = e->dtype == FE_BF16 ? 1 : 2;  // bf16: merge fused into the attention kernel
  if (mk_tick) e->n_launches += 1;
  else e->n_launches += 1 + (6 + attn_kernels) * m.L + (decode ? 3 : 0) - (items.empty() ? m.L : 0);
  e->n_forwards++;
  e->n_rows_total += n;
}

// Append ids to one or more sequences (positions len .. len + n - 1 each),
// packing the rows of all of them into as few forwards as the lane holds:
// a batched trunk prefill runs its GEMMs at M = the packed row count.
struct PrefillSeg {
  int seq;
  const int32_t* ids;
  int n;
  uint64_t vseed;
  int out_idx = -1;  // >= 0: the last row runs the lm_head, greedy token -> out_tokens[out_idx]
};

void prefill_multi(fe_engine* e, const std::vector<PrefillSeg>& segs, int vis_id) {
  Lane& ln = e->lanes[0];
  for (const auto& sg : segs) {
    seq_at(e, sg.seq);
    for (int i = 0; i < sg.n; i++) {
      if (sg.ids[i] == vis_id && e->seqs[sg.seq].len + i < 1) throw Error("prefill: vision placeholder at position 0");
      if (sg.ids[i] != vis_id && (sg.ids[i] < 0 || sg.ids[i] >= e->m.V)) throw Error("prefill: token id out of range");
    }
    for (const auto& o : segs)
      if (&o != &sg && o.seq == sg.seq) throw Error("prefill: a sequence listed twice");
  }
  std::vector<RowIn> rows;
  std::vector<uint64_t> vseeds;  // per-forward table: vision seeds, or (tower on) VIS-row buffer pointers
  std::vector<int> pinned;       // tower slots the pending forward reads
  int chunks = 0;
  auto flush = [&]() {
    if (rows.empty()) return;
    forward(e, ln, rows, 0, &vseeds, e->vis != nullptr, /*prefill_rows=*/true);
    rows.clear();
    vseeds.clear();
    pinned.clear();
    chunks = 0;
  };
  // VIS rows of an observation: the tower's output, encoded once per seed
  // (LRU slots; a slot the pending forward reads is never recycled)
  auto vis_rows = [&](uint64_t vseed) -> uint64_t {
    int slot = -1;
    for (size_t i = 0; i < e->vis_seed.size(); i++)
      if (e->vis_stamp[i] >= 0 && e->vis_seed[i] == vseed) slot = (int)i;
    if (slot < 0) {
      for (size_t i = 0; i < e->vis_seed.size(); i++) {
        if (std::find(pinned.begin(), pinned.end(), (int)i) != pinned.end()) continue;
        if (slot < 0 || e->vis_stamp[i] < e->vis_stamp[slot]) slot = (int)i;
      }
      if (slot < 0) {  // every slot feeds the pending forward
        flush();
        slot = 0;
      }
      e->vis->encode(vseed, e->vis_buf[slot], ln.stream);
      e->vis_seed[slot] = vseed;
      e->vis_encodes++;
    }
    e->vis_stamp[slot] = ++e->vis_clock;
    pinned.push_back(slot);
    return (uint64_t)(uintptr_t)e->vis_buf[slot];
  };
  for (const auto& sg : segs) {
    int pos = e->seqs[sg.seq].len;
    int vk = -1;
    for (int i = 0; i < sg.n; i++, pos++) {
      const int c = pos / FE_PAGE + 1;
      if (!rows.empty() && ((int)rows.size() >= ln.max_rows || chunks + c > ln.max_partials)) {
        flush();
        vk = -1;
      }
      if (vk < 0) {
        const uint64_t tag = e->vis ? vis_rows(sg.vseed) : sg.vseed;  // (may flush the pending forward)
        vk = (int)vseeds.size();
        vseeds.push_back(tag);
      }
      RowIn r{};
      r.seq = sg.seq;
      r.pos = pos;
      r.tok = sg.ids[i] == vis_id ? -1 : sg.ids[i];
      r.tok_src = -1;
      r.vis_row = sg.ids[i] == vis_id ? pos - 1 : -1;
      r.out_idx = -1;
      r.logit_row = -1;
      r.head = sg.out_idx >= 0 && i == sg.n - 1;
      r.out_idx = r.head ? sg.out_idx : -1;
      r.vk = vk;
      rows.push_back(r);
      chunks += c;
    }
  }
  flush();
  CK(cudaEventRecord(e->lane0_ev, ln.stream));
}

void prefill(fe_engine* e, int seq, const int32_t* ids, int n, uint64_t vseed, int vis_id) {
  prefill_multi(e, {PrefillSeg{seq, ids, n, vseed}}, vis_id);
}

int new_request_slot(fe_engine* e) {
  int r;
  if (!e->free_reqs.empty()) {
    r = e->free_reqs.back();
    e->free_reqs.pop_back();
  } else {
    r = (int)e->reqs.size();
    e->reqs.emplace_back();
  }
  return r;
}

Request& req_at(fe_engine* e, int r) {
  if (r < 0 || r >= (int)e->reqs.size() || !e->reqs[r].live) throw Error("invalid request " + std::to_string(r));
  return e->reqs[r];
}

bool lane_busy(const Lane& ln) {
  if (!ln.waiting.empty()) return true;
  for (int s = 0; s < ln.slots; s++)
    if (ln.slot_req[s] >= 0) return true;
  return false;
}

// One decode iteration of a lane (= one tick of the reference _MicroEngine).
int tick(fe_engine* e, Lane& ln, std::vector<int>* completed) {
  // admission: action class first, then FIFO by seqno (schedulers.py:279-285)
  if (!ln.waiting.empty()) {
    std::stable_sort(ln.waiting.begin(), ln.waiting.end(), [&](int a, int b) {
      const Request &ra = e->reqs[a], &rb = e->reqs[b];
      if (ra.priority != rb.priority) return ra.priority < rb.priority;
      return ra.seqno < rb.seqno;
    });
    for (int s = 0; s < ln.slots && !ln.waiting.empty(); s++) {
      if (ln.slot_req[s] < 0) {
        ln.slot_req[s] = ln.waiting.front();
        e->reqs[ln.waiting.front()].state = 1;
        ln.waiting.erase(ln.waiting.begin());
      }
    }
  }
  std::vector<RowIn> rows;
  for (int s = 0; s < ln.slots; s++) {
    const int ri = ln.slot_req[s];
    if (ri < 0) continue;
    Request& q = e->reqs[ri];
    RowIn r{};
    r.seq = q.seq;
    r.pos = e->seqs[q.seq].len;
    r.tok = q.produced == 0 ? q.first_id : -1;
    r.tok_src = q.produced == 0 ? -1 : q.arena * kRequestCap + q.produced - 1;
    r.vis_row = -1;
    r.out_idx = q.arena * kRequestCap + q.produced;
    r.logit_row = (q.capture && q.produced < q.length) ? q.logit_base + q.produced : -1;
    r.head = true;
    rows.push_back(r);
  }
  const int occupied = (int)rows.size();
  forward(e, ln, rows, 0);
  for (int s = 0; s < ln.slots; s++) {
    const int ri = ln.slot_req[s];
    if (ri < 0) continue;
    Request& q = e->reqs[ri];
    if (++q.produced == q.length) {
      q.state = 2;
      ln.slot_req[s] = -1;
      completed->push_back(ri);
    }
  }
  e->n_ticks++;
  return occupied;
}

void init_weights(fe_engine* e, uint64_t seed) {
  const fe::ModelDims& m = e->m;
  cudaStream_t st = e->lanes[0].stream;
  const size_t d = m.d, F = m.F, V = m.V;
  auto key = [&](uint64_t tid) { return fe::tensor_key(seed, tid); };
  fe::launch_init_linear(e->dtype, e->w.embed, key(1), V * d, st);
  fe::launch_init_linear(e->dtype, e->w.lm_head, key(2), V * d, st);
  fe::launch_init_norm(e->w.final_norm, key(3), d, st);
  for (int l = 0; l < m.L; l++) {
    const uint64_t b = 16 + 16 * (uint64_t)l;
    fe::Weights::Layer& ly = e->layers[l];
    char* qkv = (char*)ly.wqkv;
    char* gu = (char*)ly.wgu;
    fe::launch_init_norm(ly.attn_norm, key(b + 0), d, st);
    fe::launch_init_linear(e->dtype, qkv, key(b + 1), d * d, st);
    fe::launch_init_linear(e->dtype, qkv + d * d * e->elem, key(b + 2), d * d, st);
    fe::launch_init_linear(e->dtype, qkv + 2 * d * d * e->elem, key(b + 3), d * d, st);
    fe::launch_init_linear(e->dtype, ly.wo, key(b + 4), d * d, st);
    fe::launch_init_norm(ly.ffn_norm, key(b + 5), d, st);
    fe::launch_init_linear(e->dtype, gu, key(b + 6), F * d, st);
    fe::launch_init_linear(e->dtype, gu + F * d * e->elem, key(b + 7), F * d, st);
    fe::launch_init_linear(e->dtype, ly.wdown, key(b + 8), d * F, st);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
}

void create_lane(fe_engine* e, Lane& ln, int id, int rows, int priority) {
  const fe::ModelDims& m = e->m;
  const size_t d = m.d, F = m.F, V = m.V, el = e->elem, R = rows;
  ln.id = id;
  ln.max_rows = rows;
  CK(cudaStreamCreateWithPriority(&ln.stream, cudaStreamNonBlocking, priority));
  ln.ws.x = (float*)e->dalloc(R * d * 4);
  ln.ws.xn = e->dalloc(R * std::max(d, F) * el);
  ln.ws.q = (float*)e->dalloc(R * d * 4);
  ln.ws.attn = e->dalloc(R * std::max(d, F) * el);
  ln.max_partials = (int)std::min<size_t>(R * (size_t)(m.max_pos / FE_PAGE), 65536);
  ln.max_items = ln.max_partials;
  ln.ws.partial = (float*)e->dalloc((size_t)ln.max_partials * m.H * (m.hd + 4) * 4);  // decode_mk: hd + 4 records
  ln.ws.part_keys = (unsigned long long*)e->dalloc(R * (size_t)fe::lm_head_ctas(m) * 8);
  ln.ws.logits = id == 0 ? e->logits : nullptr;
  ln.attn_counters = (int*)e->dalloc(R * m.H * sizeof(int));
  CK(cudaMemset(ln.attn_counters, 0, R * m.H * sizeof(int)));
  if (e->mk_on) {
    ln.mk_ss = (float*)e->dalloc((size_t)(m.d / 128) * 16 * 4);
    ln.mk_bar = (unsigned long long*)e->dalloc(2 * sizeof(unsigned long long));
    CK(cudaMemset(ln.mk_bar, 0, 2 * sizeof(unsigned long long)));
    ln.mk_partial = (float*)e->dalloc(fe::mk_partial_floats(e->mk_plans) * 4);
    ln.mk_grab = (int*)e->dalloc((size_t)fe::mk_phases(m.L) * sizeof(int));
    CK(cudaMemset(ln.mk_grab, 0, (size_t)fe::mk_phases(m.L) * sizeof(int)));
    ln.mk_counters = (int*)e->dalloc(4096 * sizeof(int));
    CK(cudaMemset(ln.mk_counters, 0, 4096 * sizeof(int)));
    ln.mk_keys = (unsigned long long*)e->dalloc((size_t)16 * e->mk_plans[fe::MK_LM].tiles * 8);
  }
  {  // fixed-offset metadata layout (16-byte aligned sections)
    MetaLayout& L = ln.layout;
    auto up16 = [](size_t v) { return (v + 15) & ~(size_t)15; };
    L.cap_rows = (int)R;
    L.cap_items = ln.max_items;
    L.cap_irows = ln.max_partials;
    L.o_rows = 64;
    L.o_items = up16(L.o_rows + R * sizeof(fe::RowMeta));
    L.o_irows = up16(L.o_items + (size_t)L.cap_items * sizeof(fe::AttnItem));
    L.o_heads = up16(L.o_irows + (size_t)L.cap_irows * sizeof(fe::ItemRow));
    L.cap_pages = m.max_pos / FE_PAGE + 1;
    L.o_pages = up16(L.o_heads + R * 4);
    L.o_slots = up16(L.o_pages + (size_t)L.cap_pages * 4);
    L.o_nspans = up16(L.o_slots + (size_t)L.cap_irows * 4);
    L.o_spages = up16(L.o_nspans + R * 4);
    L.o_smasks = up16(L.o_spages + (size_t)ln.max_partials * 4);
    L.o_ptiles = up16(L.o_smasks + (size_t)ln.max_partials * 4);
    L.o_vkeys = up16(L.o_ptiles + R * sizeof(fe::PrefillTile));
    L.total = up16(L.o_vkeys + R * 8);
  }
  ln.ws.meta = e->dalloc(ln.layout.total);
  for (int i = 0; i < 2; i++) CK(cudaEventCreateWithFlags(&ln.tick_ev[i], cudaEventDisableTiming));
  for (int i = 0; i < kMetaRing; i++) {
    CK(cudaMallocHost((void**)&ln.meta_host[i], ln.layout.total));
    CK(cudaEventCreateWithFlags(&ln.meta_ev[i], cudaEventDisableTiming));
    CK(cudaEventRecord(ln.meta_ev[i], ln.stream));
  }
  ln.slot_req.assign(e->max_slots, -1);
  ln.slots = std::min(8, e->max_slots);
  if (e->use_tc) {
    ln.map_xn = fe::make_kmajor_map(ln.ws.xn, rows, m.d, m.d, 128);
    ln.map_attn = fe::make_kmajor_map(ln.ws.attn, rows, m.d, m.d, 128);
    ln.map_act = fe::make_kmajor_map(ln.ws.attn, rows, m.F, m.F, 128);
    ln.map_xn16 = fe::make_kmajor_map(ln.ws.xn, rows, m.d, m.d, 16);
    ln.map_attn16 = fe::make_kmajor_map(ln.ws.attn, rows, m.d, m.d, 16);
    ln.map_act16 = fe::make_kmajor_map(ln.ws.attn, rows, m.F, m.F, 16);
    const size_t part_floats = std::max({fe::skinny_partial_floats(3 * m.d, m.d), fe::skinny_partial_floats(m.d, m.d),
                                         fe::skinny_partial_floats(2 * m.F, m.d), fe::skinny_partial_floats(m.d, m.F),
                                         fe::skinny_partial_floats(m.V, m.d)});  // any skinny split plan
    ln.sk_partial = (float*)e->dalloc(part_floats * 4);
    ln.sk_counters = (int*)e->dalloc(4096 * sizeof(int));
    CK(cudaMemset(ln.sk_counters, 0, 4096 * sizeof(int)));
    ln.pair_scratch = (float*)e->dalloc(fe::pair_sk_scratch_floats() * 4);
    ln.pair_counters = (int*)e->dalloc(fe::pair_sk_counters() * sizeof(int));
    CK(cudaMemset(ln.pair_counters, 0, fe::pair_sk_counters() * sizeof(int)));
    // split-K planes: 4 splits of a 256-row gate/up output
    ln.split_floats = (size_t)4 * 256 * std::max<size_t>(2 * F, 3 * d);
    ln.split_scratch = (float*)e->dalloc(ln.split_floats * 4);
  }
  (void)V;
}

fe_engine* create(const fe_config* c, int device, const float* rope_host) {
  if (c->head_dim != 64 && c->head_dim != 128) throw Error("head_dim must be 64 or 128");
  if (c->n_heads * c->head_dim != c->d_model) throw Error("n_heads * head_dim != d_model");
  if (c->d_model % 8 || c->d_ffn % 8 || c->vocab % 4) throw Error("dimensions must be multiples of 8");
  if (c->dtype != FE_F32 && c->dtype != FE_BF16) throw Error("dtype must be FE_F32 or FE_BF16");
  auto* e = new fe_engine();
  try {
    e->device = device;
    CK(cudaSetDevice(device));
    e->m = {c->d_model, c->n_layers, c->n_heads, c->head_dim, c->d_ffn, c->vocab, c->n_text, c->max_pos,
            c->rms_eps, c->attn_scale};
    e->dtype = c->dtype;
    e->elem = c->dtype == FE_F32 ? 4 : 2;
    const int max_rows = c->max_rows > 0 ? c->max_rows : 512;
    e->max_slots = c->max_slots > 0 ? c->max_slots : 64;
    const fe::ModelDims& m = e->m;
    const size_t d = m.d, F = m.F, V = m.V, el = e->elem;

    e->w.embed = e->dalloc(V * d * el);
    e->w.lm_head = e->dalloc(V * d * el);
    e->w.final_norm = (float*)e->dalloc(d * 4);
    e->layers.resize(m.L);
    for (int l = 0; l < m.L; l++) {
      auto& ly = e->layers[l];
      ly.attn_norm = (float*)e->dalloc(d * 4);
      ly.ffn_norm = (float*)e->dalloc(d * 4);
      ly.wqkv = e->dalloc(3 * d * d * el);
      ly.wo = e->dalloc(d * d * el);
      ly.wgu = e->dalloc(2 * F * d * el);
      ly.wdown = e->dalloc(d * F * el);
    }
    e->w.layers = e->layers.data();
    e->rope = (float*)e->dalloc(sizeof(float) * (size_t)m.max_pos * m.hd);
    CK(cudaMemcpy(e->rope, rope_host, sizeof(float) * (size_t)m.max_pos * m.hd, cudaMemcpyHostToDevice));

    // shared token arena and logits capture
    e->logits = (float*)e->dalloc((size_t)kLogitRows * V * 4);
    const int n_arena = std::max(4 * e->max_slots, 256);
    e->out_tokens = (int32_t*)e->dalloc((size_t)n_arena * kRequestCap * 4);
    CK(cudaMemset(e->out_tokens, 0, (size_t)n_arena * kRequestCap * 4));
    for (int i = n_arena - 1; i >= 0; i--) e->free_arena.push_back(i);

    // tcgen05 path: weight tensor maps (A operand of the skinny GEMM, B of the tile GEMM)
    e->use_tc = e->dtype == FE_BF16 && m.hd == 128 && m.d % 128 == 0 && m.F % 64 == 0 && max_rows >= 64;
    if (e->use_tc) {
      e->map_lm = fe::make_kmajor_map(e->w.lm_head, m.V, m.d, m.d, 128);
      e->tc_maps.resize(m.L);
      for (int l = 0; l < m.L; l++) {
        auto& ly = e->layers[l];
        e->tc_maps[l].qkv = fe::make_kmajor_map(ly.wqkv, 3 * m.d, m.d, m.d, 128);
        e->tc_maps[l].wo = fe::make_kmajor_map(ly.wo, m.d, m.d, m.d, 128);
        e->tc_maps[l].wgu = fe::make_kmajor_map(ly.wgu, 2 * m.F, m.d, m.d, fe::tc_box_rows(fe::TC_SWIGLU));
        e->tc_maps[l].wdown = fe::make_kmajor_map(ly.wdown, m.d, m.F, m.F, 128);
        e->tc_maps[l].qkv64 = fe::make_kmajor_map(ly.wqkv, 3 * m.d, m.d, m.d, 64);
        e->tc_maps[l].wo64 = fe::make_kmajor_map(ly.wo, m.d, m.d, m.d, 64);
        e->tc_maps[l].wdown64 = fe::make_kmajor_map(ly.wdown, m.d, m.F, m.F, 64);
      }
    }

    // persistent decode-tick kernel: per-GEMM split plans over one CTA per SM,
    // weight tensor maps and norm vectors in device memory
    e->mk_on = e->use_tc && m.H * m.hd == m.d && m.d % 512 == 0;
    if (e->mk_on) {
      e->mk_grid = fe::mk_grid();
      mk_make_plans(e);
      std::vector<fe::TmaMap> maps(4 * m.L + 1);
      for (int l = 0; l < m.L; l++) {
        maps[4 * l + 0] = e->tc_maps[l].qkv;
        maps[4 * l + 1] = e->tc_maps[l].wo;
        maps[4 * l + 2] = e->tc_maps[l].wgu;
        maps[4 * l + 3] = e->tc_maps[l].wdown;
      }
      maps[4 * m.L] = e->map_lm;
      e->mk_maps = e->dalloc(maps.size() * sizeof(fe::TmaMap));
      CK(cudaMemcpy(e->mk_maps, maps.data(), maps.size() * sizeof(fe::TmaMap), cudaMemcpyHostToDevice));
      std::vector<const float*> norms(2 * m.L + 1);
      for (int l = 0; l < m.L; l++) {
        norms[2 * l] = e->layers[l].attn_norm;
        norms[2 * l + 1] = e->layers[l].ffn_norm;
      }
      norms[2 * m.L] = e->w.final_norm;
      e->mk_norms = (const float**)e->dalloc(norms.size() * sizeof(float*));
      CK(cudaMemcpy(e->mk_norms, norms.data(), norms.size() * sizeof(float*), cudaMemcpyHostToDevice));
    }

    // lanes: 0 = foreground (highest priority), 1 = background reasoning
    int prio_low = 0, prio_high = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
    create_lane(e, e->lanes[0], 0, max_rows, prio_high);
    create_lane(e, e->lanes[1], 1, std::min(max_rows, kLane1Rows), prio_low);
    CK(cudaEventCreateWithFlags(&e->lane0_ev, cudaEventDisableTiming));
    for (int i = 0; i < kLanes; i++) CK(cudaEventCreateWithFlags(&e->mk_ev[i], cudaEventDisableTiming));
    CK(cudaEventRecord(e->lane0_ev, e->lanes[0].stream));

    // KV pool: 64-token pages [L][2][H][64][hd]
    e->page_elems = fe::kv_page_elems(m);
    CK(cudaDeviceGetAttribute(&e->n_sm, cudaDevAttrMultiProcessorCount, device));
    size_t pages = c->kv_pages;
    if (pages == 0) {
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      const size_t reserve = (size_t)4 << 30;
      const size_t avail = free_b > reserve ? free_b - reserve : free_b / 2;
      pages = std::max<size_t>(16, std::min<size_t>(avail / 2 / (e->page_elems * el), 8192));
    }
    e->n_pages = (int)pages;
    e->kv_pool = e->dalloc(pages * e->page_elems * el);
    // zeroed once: attention kernels that stage whole pages multiply the keys
    // past a row's valid count by p = 0, which needs finite contents
    CK(cudaMemset(e->kv_pool, 0, pages * e->page_elems * el));
    if (e->use_tc)
    {
      e->pool_map = fe::make_kmajor_map(e->kv_pool, (int)(pages * e->page_elems / 128), 128, 128, 64);
      e->pool_map16 = fe::make_kmajor_map(e->kv_pool, (int)(pages * e->page_elems / 128), 128, 128, 16);
    }
    e->page_ref.assign(pages, 0);
    for (int p = (int)pages - 1; p >= 0; p--) e->free_pages.push_back(p);
  } catch (...) {
    for (void* p : e->allocs) cudaFree(p);
    delete e;
    throw;
  }
  return e;
}

void destroy(fe_engine* e) {
  cudaSetDevice(e->device);
  for (auto& ln : e->lanes)
    if (ln.stream) cudaStreamSynchronize(ln.stream);
  clear_graphs(e);
  for (void* p : e->allocs) cudaFree(p);
  for (auto& r : e->prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto& pp : e->pending_pages)
    for (int l = 0; l < kLanes; l++) cudaEventDestroy(pp.ev[l]);
  for (auto ev : e->free_events) cudaEventDestroy(ev);
  for (auto& ln : e->lanes) {
    for (int i = 0; i < kMetaRing; i++) {
      if (ln.meta_host[i]) cudaFreeHost(ln.meta_host[i]);
      if (ln.meta_ev[i]) cudaEventDestroy(ln.meta_ev[i]);
    }
    if (ln.stream) cudaStreamDestroy(ln.stream);
  }
  if (e->lane0_ev) cudaEventDestroy(e->lane0_ev);
  delete e;
}

template <typename Fn>
int guarded(fe_engine* e, Fn&& fn) {
  try {
    if (!e) throw Error("null engine");
    std::lock_guard<std::mutex> lk(e->mu);
    cudaSetDevice(e->device);
    fn();
    return 0;
  } catch (const std::exception& ex) {
    g_last_error = ex.what();
    return 1;
  }
}

int submit(fe_engine* e, int lane, int32_t seq, int32_t first_id, int32_t length, int32_t priority) {
  Lane& ln = lane_at(e, lane);
  Seq& s = seq_at(e, seq);
  if (length < 1 || length > kRequestCap) throw Error("request length outside [1, 1024]");
  if (s.len + length > e->m.max_pos) throw Error("request would exceed max_pos");
  if (first_id < 0 || first_id >= e->m.V) throw Error("first token id out of range");
  if (e->free_arena.empty()) throw Error("too many live requests");
  const int r = new_request_slot(e);
  Request& q = e->reqs[r];
  q = Request();
  q.live = true;
  q.seq = seq;
  q.first_id = first_id;
  q.length = length;
  q.lane = lane;
  q.priority = priority == FE_PRIO_ACTION ? 0 : 1;
  q.seqno = e->seqno++;
  q.arena = e->free_arena.back();
  e->free_arena.pop_back();
  ln.waiting.push_back(r);
  return r;
}

// Tick a lane until `stop_req` completes (-1: until idle) or `max_ticks`
// (<= 0: unbounded).  The engine lock is held per tick, so the two lanes can
// be driven by two host threads concurrently.
int run_lane(fe_engine* e, int lane, int32_t stop_req, int32_t max_ticks, int32_t cap, int32_t* n_ticks,
             int32_t* occupancy, int32_t* completed, int32_t* completed_tick, int32_t* n_completed) {
  try {
    if (!e) throw Error("null engine");
    int t = 0, nc = 0;
    bool yield = false, paced = false;
    cudaEvent_t pace = nullptr;
    while (true) {
      if (paced) {
        CK(cudaEventSynchronize(pace));
        paced = false;
      }
      if (yield) {  // lane 1 waiting for the action lane: outside the lock
        std::this_thread::sleep_for(std::chrono::microseconds(50));
        yield = false;
        if (stop_req < 0 && max_ticks > 0) break;  // a bounded background call returns to its driver
      }
      std::lock_guard<std::mutex> lk(e->mu);
      cudaSetDevice(e->device);
      Lane& ln = lane_at(e, lane);
      if (stop_req >= 0) {
        Request& q = req_at(e, stop_req);
        if (q.lane != lane) throw Error("run: stop request belongs to the other lane");
        if (q.state == 2) break;
      } else if (!lane_busy(ln)) {
        break;
      }
      if (max_ticks > 0 && t >= max_ticks) break;
      if (!lane_busy(ln)) throw Error("run: stop request is not in flight");
      if (lane == 1 && e->lane1_yields && lane_busy(e->lanes[0])) {
        // the action lane has work: the reasoning lane does not add ticks
        // (the action decodes on an uncontended GPU); retry shortly
        yield = true;
        continue;
      }
      if (t >= cap) throw Error("run: tick capacity exceeded");
      std::vector<int> done;
      occupancy[t] = tick(e, ln, &done);
      for (int r : done) {
        if (nc >= cap) throw Error("run: completion capacity exceeded");
        completed[nc] = r;
        completed_tick[nc] = t;
        nc++;
      }
      if ((lane == 1 && e->lane1_yields) || (lane == 0 && e->lane0_pace)) {
        // keep <= 2 ticks queued on the device: a background ticker (lane 0,
        // option "lane0_pace") or the reasoning lane would otherwise run
        // arbitrarily far ahead of the GPU, and a later action would queue
        // behind all of those ticks
        CK(cudaEventRecord(ln.tick_ev[ln.pace_n & 1], ln.stream));
        const bool one = lane == 0 && e->lane0_pace == 1;  // depth 1: this tick done before returning
        pace = ln.tick_ev[(ln.pace_n + (one ? 0 : 1)) & 1];
        paced = one || ln.pace_n > 0;
        ln.pace_n++;
      }
      t++;
    }
    *n_ticks = t;
    *n_completed = nc;
    return 0;
  } catch (const std::exception& ex) {
    g_last_error = ex.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* fe_last_error(void) { return g_last_error.c_str(); }

int fe_engine_create(const fe_config* cfg, int32_t device, const float* rope, fe_engine** out) {
  try {
    if (!cfg || !out || !rope) throw Error("null argument");
    *out = create(cfg, device, rope);
    return 0;
  } catch (const std::exception& ex) {
    g_last_error = ex.what();
    return 1;
  }
}

int fe_engine_destroy(fe_engine* e) {
  if (!e) return 0;
  destroy(e);
  return 0;
}

int fe_weights_init_random(fe_engine* e, uint64_t seed) {
  return guarded(e, [&] { init_weights(e, seed); });
}

int fe_seq_create(fe_engine* e, int32_t* seq) {
  return guarded(e, [&] { *seq = new_seq(e); });
}

int fe_seq_fork(fe_engine* e, int32_t parent, int32_t len, int32_t* child) {
  return guarded(e, [&] {
    Seq& p = seq_at(e, parent);
    if (len < 0 || len > p.len) throw Error("fork length outside the parent");
    const std::vector<int> ppages = p.pages;  // copy: new_seq may reallocate
    const int c = new_seq(e);
    Seq& s = e->seqs[c];
    const int full = len / FE_PAGE, rem = len % FE_PAGE;
    for (int i = 0; i < full; i++) {
      s.pages.push_back(ppages[i]);
      e->page_ref[ppages[i]]++;
    }
    if (rem) {  // copy-on-write of the partially filled page (lane 0)
      const int np = alloc_page(e);
      fe::launch_page_copy(e->dtype, e->kv_pool, ppages[full], np, rem, e->m, e->lanes[0].stream);
      CK(cudaEventRecord(e->lane0_ev, e->lanes[0].stream));
      s.pages.push_back(np);
      e->n_launches++;
    }
    s.len = len;
    *child = c;
  });
}

int fe_seq_free(fe_engine* e, int32_t seq) {
  return guarded(e, [&] {
    Seq& s = seq_at(e, seq);
    for (int p : s.pages) release_page(e, p);
    s = Seq();
    e->free_seqs.push_back(seq);
  });
}

int fe_seq_len(fe_engine* e, int32_t seq, int32_t* len) {
  return guarded(e, [&] { *len = seq_at(e, seq).len; });
}

// Draft verification (reuse-as-draft): every listed
// sequence is extended by counts[i] input ids in ONE batched forward whose
// rows all run the lm_head; the greedy token after each input lands in
// out[] (same order as ids).  The caller keeps the verified prefix and
// truncates the rest (fe_seq_truncate).  Rows beyond the lane's capacity run
// as further forwards (each sequence's rows stay in order).
int fe_verify(fe_engine* e, int32_t n_seqs, const int32_t* seqs, const int32_t* counts, const int32_t* ids,
              int32_t* out) {
  return guarded(e, [&] {
    Lane& ln = e->lanes[0];
    int total = 0;
    for (int i = 0; i < n_seqs; i++) {
      if (counts[i] < 1) throw Error("verify: every sequence needs >= 1 input");
      seq_at(e, seqs[i]);
      total += counts[i];
    }
    const int n_slots = (total + kRequestCap - 1) / kRequestCap;
    if ((int)e->free_arena.size() < n_slots) throw Error("verify: token arena exhausted");
    std::vector<int> arena(e->free_arena.end() - n_slots, e->free_arena.end());
    e->free_arena.resize(e->free_arena.size() - n_slots);
    auto give_back = [&]() { for (int a : arena) e->free_arena.push_back(a); };
    try {
      std::vector<RowIn> rows;
      int chunks = 0, k = 0;
      for (int i = 0; i < n_seqs; i++) {
        int pos = e->seqs[seqs[i]].len;
        for (int j = 0; j < counts[i]; j++, k++, pos++) {
          const int c = pos / FE_PAGE + 1;
          if (!rows.empty() && ((int)rows.size() >= ln.max_rows || chunks + c > ln.max_partials)) {
            forward(e, ln, rows, 0);
            rows.clear();
            chunks = 0;
          }
          if (ids[k] < 0 || ids[k] >= e->m.V) throw Error("verify: token id out of range");
          RowIn r{};
          r.seq = seqs[i];
          r.pos = pos;
          r.tok = ids[k];
          r.tok_src = -1;
          r.vis_row = -1;
          r.out_idx = arena[k / kRequestCap] * kRequestCap + k % kRequestCap;
          r.logit_row = -1;
          r.head = true;
          rows.push_back(r);
          chunks += c;
        }
      }
      if (!rows.empty()) forward(e, ln, rows, 0);
      CK(cudaStreamSynchronize(ln.stream));
      for (int a = 0; a < n_slots; a++) {
        const int n = std::min(kRequestCap, total - a * kRequestCap);
        CK(cudaMemcpy(out + (size_t)a * kRequestCap, e->out_tokens + (size_t)arena[a] * kRequestCap,
                      sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
      }
      e->d2h_bytes += (int64_t)sizeof(int32_t) * total;
      e->h2d_bytes += 0;
    } catch (...) {
      give_back();
      throw;
    }
    give_back();
  });
}

// Drop positions >= len of a sequence (its pages past the new end are released).
int fe_seq_truncate(fe_engine* e, int32_t seq, int32_t len) {
  return guarded(e, [&] {
    Seq& s = seq_at(e, seq);
    if (len < 0 || len > s.len) throw Error("truncate: length outside the sequence");
    const int keep = (len + FE_PAGE - 1) / FE_PAGE;
    while ((int)s.pages.size() > keep) {
      release_page(e, s.pages.back());
      s.pages.pop_back();
    }
    s.len = len;
  });
}

int fe_prefill(fe_engine* e, int32_t seq, const int32_t* ids, int32_t n, uint64_t vision_seed, int32_t vis_id) {
  return guarded(e, [&] { prefill(e, seq, ids, n, vision_seed, vis_id); });
}

int fe_vision_enable(fe_engine* e, const fe_vision_config* vc, uint64_t seed, int32_t slots) {
  return guarded(e, [&] {
    if (!vc) throw Error("null vision config");
    if (vc->img % vc->patch || vc->d % vc->heads || (vc->d / vc->heads) > 256 || vc->d % 128 || vc->d > 2048)
      throw Error("bad vision shape (d a multiple of 128, <= 2048; head_dim <= 256)");
    fe::VisionDims vd{vc->img, vc->patch, vc->d, vc->layers, vc->heads, vc->mlp, vc->proj_hidden, vc->eps};
    cudaStream_t st = e->lanes[0].stream;
    e->vis = std::make_unique<fe::Vision>(vd, e->dtype, e->m.d, seed, st, [&](size_t b) { return e->dalloc(b); });
    const int P = e->vis->patches_count();
    const int n = std::max(2, (int)slots);
    e->vis_buf.assign(n, nullptr);
    for (int i = 0; i < n; i++) e->vis_buf[i] = (float*)e->dalloc((size_t)P * e->m.d * 4);
    e->vis_seed.assign(n, 0);
    e->vis_stamp.assign(n, -1);
    CK(cudaStreamSynchronize(st));
  });
}

int fe_vision_encode(fe_engine* e, uint64_t vision_seed, float* out_host) {
  return guarded(e, [&] {
    if (!e->vis) throw Error("vision tower not enabled");
    Lane& ln = e->lanes[0];
    float* tmp = (float*)e->dalloc((size_t)e->vis->patches_count() * e->m.d * 4);
    e->vis->encode(vision_seed, tmp, ln.stream);
    CK(cudaStreamSynchronize(ln.stream));
    CK(cudaMemcpy(out_host, tmp, (size_t)e->vis->patches_count() * e->m.d * 4, cudaMemcpyDeviceToHost));
    e->allocs.pop_back();
    CK(cudaFree(tmp));
  });
}

int fe_prefill_batch_heads(fe_engine* e, int32_t n_seqs, const int32_t* seqs, const int32_t* counts,
                           const int32_t* ids, const uint64_t* vision_seeds, int32_t vis_id, const int32_t* want,
                           int32_t* out) {
  return guarded(e, [&] {
    if ((int)e->free_arena.empty()) throw Error("prefill_batch_heads: token arena exhausted");
    if (n_seqs > kRequestCap) throw Error("prefill_batch_heads: too many sequences");
    const int slot = e->free_arena.back();
    e->free_arena.pop_back();
    try {
      std::vector<PrefillSeg> segs;
      size_t off = 0;
      for (int i = 0; i < n_seqs; i++) {
        if (counts[i] < 0 || (want[i] && counts[i] < 1)) throw Error("prefill_batch_heads: bad count");
        if (counts[i]) segs.push_back({seqs[i], ids + off, counts[i], vision_seeds[i],
                                       want[i] ? slot * kRequestCap + i : -1});
        off += counts[i];
      }
      prefill_multi(e, segs, vis_id);
      Lane& ln = e->lanes[0];
      CK(cudaStreamSynchronize(ln.stream));
      std::vector<int32_t> tok(n_seqs);
      CK(cudaMemcpy(tok.data(), e->out_tokens + (size_t)slot * kRequestCap, sizeof(int32_t) * n_seqs,
                    cudaMemcpyDeviceToHost));
      for (int i = 0; i < n_seqs; i++) out[i] = want[i] ? tok[i] : -1;
      e->d2h_bytes += (int64_t)sizeof(int32_t) * n_seqs;
    } catch (...) {
      e->free_arena.push_back(slot);
      throw;
    }
    e->free_arena.push_back(slot);
  });
}

int fe_prefill_batch(fe_engine* e, int32_t n_seqs, const int32_t* seqs, const int32_t* counts, const int32_t* ids,
                     const uint64_t* vision_seeds, int32_t vis_id) {
  return guarded(e, [&] {
    std::vector<PrefillSeg> segs;
    size_t off = 0;
    for (int i = 0; i < n_seqs; i++) {
      if (counts[i] < 0) throw Error("prefill_batch: negative count");
      if (counts[i]) segs.push_back({seqs[i], ids + off, counts[i], vision_seeds[i]});
      off += counts[i];
    }
    prefill_multi(e, segs, vis_id);
  });
}

int fe_set_slots(fe_engine* e, int32_t slots) { return fe_set_slots_lane(e, 0, slots); }

int fe_set_slots_lane(fe_engine* e, int32_t lane, int32_t slots) {
  return guarded(e, [&] {
    Lane& ln = lane_at(e, lane);
    if (slots < 1 || slots > e->max_slots || slots > ln.max_rows) throw Error("slots outside [1, lane capacity]");
    for (int s = slots; s < ln.slots; s++)
      if (ln.slot_req[s] >= 0) throw Error("cannot shrink slots while they are occupied");
    ln.slots = slots;
  });
}

int fe_submit(fe_engine* e, int32_t seq, int32_t first_id, int32_t length, int32_t priority, int32_t* req) {
  return guarded(e, [&] { *req = submit(e, 0, seq, first_id, length, priority); });
}

int fe_submit_lane(fe_engine* e, int32_t lane, int32_t seq, int32_t first_id, int32_t length, int32_t priority,
                   int32_t* req) {
  return guarded(e, [&] { *req = submit(e, lane, seq, first_id, length, priority); });
}

int fe_run(fe_engine* e, int32_t stop_req, int32_t cap, int32_t* n_ticks, int32_t* occupancy, int32_t* completed,
           int32_t* completed_tick, int32_t* n_completed) {
  return run_lane(e, 0, stop_req, 0, cap, n_ticks, occupancy, completed, completed_tick, n_completed);
}

int fe_run_lane(fe_engine* e, int32_t lane, int32_t stop_req, int32_t max_ticks, int32_t cap, int32_t* n_ticks,
                int32_t* occupancy, int32_t* completed, int32_t* completed_tick, int32_t* n_completed) {
  return run_lane(e, lane, stop_req, max_ticks, cap, n_ticks, occupancy, completed, completed_tick, n_completed);
}

int fe_request_tokens(fe_engine* e, int32_t req, int32_t* out, int32_t cap) {
  // enqueue the completion marker under the lock, wait and copy outside it so
  // the other lane's driver is not blocked behind this synchronisation
  cudaEvent_t ev = nullptr;
  const int32_t* src = nullptr;
  int length = 0;
  int rc = guarded(e, [&] {
    Request& q = req_at(e, req);
    if (q.state != 2) throw Error("request not complete");
    if (cap < q.length) throw Error("output buffer too small");
    ev = take_event(e);
    CK(cudaEventRecord(ev, e->lanes[q.lane].stream));
    src = e->out_tokens + (size_t)q.arena * kRequestCap;
    length = q.length;
    e->d2h_bytes += (int64_t)sizeof(int32_t) * q.length;
  });
  if (rc) return rc;
  try {
    cudaSetDevice(e->device);
    CK(cudaEventSynchronize(ev));
    CK(cudaMemcpy(out, src, sizeof(int32_t) * length, cudaMemcpyDeviceToHost));
  } catch (const std::exception& ex) {
    g_last_error = ex.what();
    rc = 1;
  }
  std::lock_guard<std::mutex> lk(e->mu);
  e->free_events.push_back(ev);
  return rc;
}

int fe_request_release(fe_engine* e, int32_t req) {
  return guarded(e, [&] {
    Request& q = req_at(e, req);
    if (q.state == 0 || q.state == 1) throw Error("request still in flight");
    e->free_arena.push_back(q.arena);
    if (q.capture && --e->capture_live == 0) e->logit_next = 0;  // buffer rows recycled when none is held
    q = Request();
    e->free_reqs.push_back(req);
  });
}

int fe_request_capture_logits(fe_engine* e, int32_t req) {
  return guarded(e, [&] {
    Request& q = req_at(e, req);
    if (q.lane != 0) throw Error("logit capture is a lane-0 feature");
    if (q.capture) return;
    if (q.state != 0 || q.produced != 0) throw Error("logit capture must be requested before decoding starts");
    if (e->logit_next + q.length > kLogitRows) throw Error("logit capture buffer full (" + std::to_string(kLogitRows) + " rows)");
    q.capture = true;
    q.logit_base = e->logit_next;
    e->logit_next += q.length;
    e->capture_live++;
  });
}

int fe_request_logits(fe_engine* e, int32_t req, float* out, int32_t rows) {
  return guarded(e, [&] {
    Request& q = req_at(e, req);
    if (!q.capture) throw Error("request did not capture logits");
    if (rows > q.produced) throw Error("more logit rows than captured");
    CK(cudaStreamSynchronize(e->lanes[0].stream));
    CK(cudaMemcpy(out, e->logits + (size_t)q.logit_base * e->m.V, sizeof(float) * (size_t)rows * e->m.V,
                  cudaMemcpyDeviceToHost));
  });
}

int fe_in_flight(fe_engine* e, int32_t* n) {
  return guarded(e, [&] {
    int c = 0;
    for (auto& ln : e->lanes) {
      c += (int)ln.waiting.size();
      for (int s = 0; s < ln.slots; s++) c += ln.slot_req[s] >= 0;
    }
    *n = c;
  });
}

int fe_synchronize(fe_engine* e) {
  return guarded(e, [&] {
    for (auto& ln : e->lanes) CK(cudaStreamSynchronize(ln.stream));
  });
}

int fe_stream(fe_engine* e, void** stream) {
  return guarded(e, [&] { *stream = (void*)e->lanes[0].stream; });
}

int fe_stream_lane(fe_engine* e, int32_t lane, void** stream) {
  return guarded(e, [&] { *stream = (void*)lane_at(e, lane).stream; });
}

int fe_profile(fe_engine* e, int32_t enable) {
  return guarded(e, [&] {
    flush_profile(e);
    e->prof_on = enable != 0;
    for (int c = 0; c < PROF_NCAT; c++) {
      e->prof_ms[c] = 0.0;
      e->prof_bytes[c] = 0.0;
      e->prof_n[c] = 0;
    }
  });
}

int fe_profile_read(fe_engine* e, double* out, int32_t n) {
  return guarded(e, [&] {
    flush_profile(e);
    for (int c = 0; c < PROF_NCAT && 3 * c + 2 < n; c++) {
      out[3 * c] = e->prof_ms[c];
      out[3 * c + 1] = (double)e->prof_n[c];
      out[3 * c + 2] = e->prof_bytes[c];
    }
  });
}

int fe_stats(fe_engine* e, int64_t* out, int32_t n) {
  return guarded(e, [&] {
    const int64_t used = e->n_pages - (int)e->free_pages.size() - (int)e->pending_pages.size();
    const int64_t v[] = {e->n_ticks, e->n_forwards, e->n_rows_total, used, (int64_t)e->n_pages,
                         (int64_t)(e->page_elems * e->elem), e->h2d_bytes, e->d2h_bytes, e->n_launches};
    for (int i = 0; i < n && i < (int)(sizeof(v) / sizeof(v[0])); i++) out[i] = v[i];
  });
}

int fe_weight_ptr(fe_engine* e, int32_t tensor, int32_t layer, void** ptr, size_t* bytes) {
  return guarded(e, [&] {
    const size_t d = e->m.d, F = e->m.F, V = e->m.V, el = e->elem;
    if (tensor == 1) { *ptr = e->w.embed; *bytes = V * d * el; return; }
    if (tensor == 2) { *ptr = e->w.lm_head; *bytes = V * d * el; return; }
    if (tensor == 3) { *ptr = e->w.final_norm; *bytes = d * 4; return; }
    if (layer < 0 || layer >= e->m.L) throw Error("layer out of range");
    const auto& ly = e->layers[layer];
    switch ((tensor - 16) % 16) {
      case 0: *ptr = ly.attn_norm; *bytes = d * 4; return;
      case 1: *ptr = ly.wqkv; *bytes = d * d * el; return;
      case 2: *ptr = (char*)ly.wqkv + d * d * el; *bytes = d * d * el; return;
      case 3: *ptr = (char*)ly.wqkv + 2 * d * d * el; *bytes = d * d * el; return;
      case 4: *ptr = ly.wo; *bytes = d * d * el; return;
      case 5: *ptr = ly.ffn_norm; *bytes = d * 4; return;
      case 6: *ptr = ly.wgu; *bytes = F * d * el; return;
      case 7: *ptr = (char*)ly.wgu + F * d * el; *bytes = F * d * el; return;
      case 8: *ptr = ly.wdown; *bytes = d * F * el; return;
    }
    throw Error("unknown tensor id");
  });
}

int fe_memcpy(fe_engine* e, void* dst, const void* src, size_t bytes) {
  return guarded(e, [&] {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, e->lanes[0].stream));
    CK(cudaStreamSynchronize(e->lanes[0].stream));
  });
}

int fe_op_gemv(fe_engine* e, const void* w, int32_t N, int32_t K, const void* x, int32_t rows, float* y) {
  return guarded(e, [&] {
    if (N % 4 || K % 8) throw Error("gemv: N % 4 and K % 8 must be 0");
    fe::launch_gemv_store(e->dtype, w, N, K, x, rows, y, e->lanes[0].stream);
    CK(cudaGetLastError());
  });
}

int fe_op_gemm_tc(fe_engine* e, const void* x, const void* w, int32_t M, int32_t N, int32_t K, float* y) {
  return guarded(e, [&] {
    if (N % 128 || K % 64) throw Error("gemm_tc: N % 128 and K % 64 must be 0");
    const fe::TmaMap am = fe::make_kmajor_map(x, M, K, K, 128);
    const fe::TmaMap bm = fe::make_kmajor_map(w, N, K, K, e->tc_pair ? 64 : 128);
    fe::TcLaunch t{};
    t.M = M; t.N = N; t.K = K; t.epi = fe::TC_STORE; t.y = y; t.ldy = N;
    t.sk_scratch = e->lanes[0].pair_scratch; t.sk_counters = e->lanes[0].pair_counters;
    t.split_scratch = e->lanes[0].split_scratch; t.split_floats = e->lanes[0].split_floats;
    for (int r = 0; r < e->op_reps; r++) {
      if (e->tc_pair) fe::launch_gemm_tc(am, bm, t, e->lanes[0].stream);
      else fe::launch_gemm_tc_v1(am, bm, t, e->lanes[0].stream);
    }
    CK(cudaGetLastError());
  });
}

int fe_op_skinny_tc(fe_engine* e, const void* x, const void* w, int32_t M, int32_t N, int32_t K, float* y) {
  return guarded(e, [&] {
    if (M > fe::skinny_max_rows() || N % 128 || K % 64) throw Error("skinny_tc: M <= 128, N % 128, K % 64");
    Lane& ln = e->lanes[0];
    // kernel-test scratch, separate from the lanes' (graph-captured) buffers
    const size_t need = std::max(fe::skinny_partial_floats(N, K), (size_t)((N + 127) / 128) * 16 * 128 * 256) * 4;
    if (e->op_bytes < need) {
      e->op_partial = (float*)e->dalloc(need);
      e->op_bytes = need;
    }
    if (!e->op_counters) {
      e->op_counters = (int*)e->dalloc(4096 * sizeof(int));
      CK(cudaMemset(e->op_counters, 0, 4096 * sizeof(int)));
    }
    const fe::TmaMap xm = fe::make_kmajor_map(x, M, K, K, 16);
    const fe::TmaMap wm = fe::make_kmajor_map(w, N, K, K, 128);
    fe::SkLaunch t{};
    t.N = N; t.K = K; t.B = M; t.epi = fe::TC_STORE; t.y = y; t.ldy = N;
    t.partial = e->op_partial; t.counters = e->op_counters;
    for (int r = 0; r < e->op_reps; r++) fe::launch_skinny_tc(wm, xm, t, ln.stream);
    CK(cudaGetLastError());
  });
}

int fe_set_option(fe_engine* e, const char* key, int64_t value) {
  return guarded(e, [&] {
    const std::string k = key ? key : "";
    // every option that changes the kernel selection baked into captured
    // decode graphs drops them (a graphed tick would keep the old choice)
    if (k == "tc_min_rows") {
      e->tc_min_rows = (int)value;
      clear_graphs(e);
    } else if (k == "sk_splits") {
      fe::g_sk_splits = (int)value;
      clear_graphs(e);
    } else if (k == "sk_rows_qkv" || k == "sk_rows_o" || k == "sk_rows_gu" || k == "sk_rows_down") {
      e->sk_rows[k == "sk_rows_qkv" ? 0 : k == "sk_rows_o" ? 1 : k == "sk_rows_gu" ? 2 : 3] = (int)value;
      clear_graphs(e);
    } else if (k == "sk_max_rows") {
      e->sk_max_rows = (int)value;
      clear_graphs(e);
    } else if (k == "use_tc") {
      e->use_tc = value != 0 && !e->tc_maps.empty();
      e->mk_on = e->use_tc && e->mk_maps != nullptr;
      clear_graphs(e);
    } else if (k == "mk_trace") {
      if (value && !e->mk_trace && e->mk_on) {
        e->mk_trace_n = (size_t)fe::mk_phases(e->m.L) * 6 * e->mk_grid;
        e->mk_trace = (unsigned long long*)e->dalloc(e->mk_trace_n * 8);
        CK(cudaMemset(e->mk_trace, 0, e->mk_trace_n * 8));
      }
      e->mk_trace_on = value != 0 && e->mk_trace != nullptr;
      clear_graphs(e);
    } else if (k == "fuse_norm") {
      e->fuse_norm = value != 0;
      clear_graphs(e);
    } else if (k == "pattn_trace") {
      if (value && !e->mk_trace) {
        e->mk_trace_n = 1 << 14;
        e->mk_trace = (unsigned long long*)e->dalloc(e->mk_trace_n * 8);
        CK(cudaMemset(e->mk_trace, 0, e->mk_trace_n * 8));
      }
      e->pattn_trace_on = value != 0 && e->mk_trace != nullptr;
      clear_graphs(e);
    } else if (k == "mk_fused") {
      e->mk_fused = (int)value;
      clear_graphs(e);
    } else if (k == "mk_flags") {
      e->mk_flags = (int)value;
      clear_graphs(e);
    } else if (k == "mk_pf") {
      e->mk_pf_stages = (int)value;
      clear_graphs(e);
    } else if (k == "mk_per_cta" || k == "mk_nc_cap" || k == "mk_nc_cap_o" || k == "mk_nc_qkv" || k == "mk_nc_o" ||
               k == "mk_nc_gu" || k == "mk_nc_down" || k == "mk_nc_lm") {
      int* slot = k == "mk_per_cta" ? &e->mk_per_cta : k == "mk_nc_cap" ? &e->mk_nc_cap
                  : k == "mk_nc_cap_o" ? &e->mk_nc_cap_o : k == "mk_nc_qkv" ? &e->mk_nc_force[fe::MK_QKV]
                  : k == "mk_nc_o" ? &e->mk_nc_force[fe::MK_O] : k == "mk_nc_gu" ? &e->mk_nc_force[fe::MK_GU]
                  : k == "mk_nc_down" ? &e->mk_nc_force[fe::MK_DOWN] : &e->mk_nc_force[fe::MK_LM];
      *slot = (int)value;
      if (e->mk_on) mk_make_plans(e);
      clear_graphs(e);
    } else if (k == "span_attn") {
      e->span_attn = value != 0;
      clear_graphs(e);
    } else if (k == "span_dbg") {
      fe::g_span_dbg = (int)value;
      clear_graphs(e);
    } else if (k == "span_cap") {
      e->span_cap = (int)std::max<int64_t>(1, value);
      clear_graphs(e);
    } else if (k == "tc_pair") {
      e->tc_pair = value != 0;
      clear_graphs(e);
    } else if (k == "tc_split") {
      fe::g_pair_split = (int)value;
      clear_graphs(e);
    } else if (k == "tc_maxp") {
      fe::g_pair_maxp = (int)value;
      clear_graphs(e);
    } else if (k == "tc_sk") {
      fe::g_pair_sk = (int)value;
      clear_graphs(e);
    } else if (k == "tc_bn") {
      fe::g_pair_bn = (int)value;
      clear_graphs(e);
    } else if (k == "prefill_tc") {
      e->prefill_tc = value != 0 && e->use_tc;
    } else if (k == "prefill_fa") {
      e->prefill_fa = value != 0;
    } else if (k == "lane0_pace") {
      e->lane0_pace = (int)std::max<int64_t>(0, std::min<int64_t>(2, value));
    } else if (k == "lane1_yields") {
      e->lane1_yields = value != 0;
    } else if (k == "mk") {
      e->mk_on = value != 0 && e->use_tc && e->mk_maps != nullptr;
      clear_graphs(e);
    }
    else if (k == "sk_mask") {
      e->sk_mask = (int)value;
      clear_graphs(e);
    } else if (k == "graphs") e->graphs_on = value != 0;
    else if (k == "pdl") {
      fe::g_pdl = value != 0;
      clear_graphs(e);
    }
    else if (k == "op_reps") e->op_reps = (int)std::max<int64_t>(1, value);
    else if (k == "sk_stages") {
      fe::g_sk_stages = (int)value;
      clear_graphs(e);
    } else if (k == "debug_skip") {
      e->debug_skip = (int)value;
      clear_graphs(e);
    } else {
      throw Error("unknown option " + k);
    }
  });
}

int fe_debug_trace(fe_engine* e, uint64_t* out, int32_t n, int32_t* n_phases, int32_t* grid) {
  return guarded(e, [&] {
    if (!e->mk_trace) throw Error("debug_trace: enable option mk_trace first");
    CK(cudaStreamSynchronize(e->lanes[0].stream));
    const size_t k = std::min<size_t>((size_t)std::max(n, 0), e->mk_trace_n);
    CK(cudaMemcpy(out, e->mk_trace, k * 8, cudaMemcpyDeviceToHost));
    *n_phases = fe::mk_phases(e->m.L, e->mk_fused | (1 << fe::MK_LM));
    *grid = e->mk_grid;
  });
}

int fe_op_rmsnorm(fe_engine* e, const float* x, const float* w, void* out, int32_t rows, int32_t d) {
  return guarded(e, [&] {
    fe::launch_rmsnorm(e->dtype, x, w, out, rows, d, d, e->m.eps, nullptr, e->lanes[0].stream);
    CK(cudaGetLastError());
  });
}

}  // extern "C"
