/*
 * CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library, and only as the checker or
 * the CPU baseline.  The product path (paper_2506_07639_b200/) never links or
 * imports anything under oracle/.
 *
 * What it restates.  The reference (`/root/reference/pkg/src/ecot_sched`) has
 * no model: `begin_step` (backends.py:98-110) is served by an RNG or an HTTP
 * server (backends.py:190-209, :355-379).  BASELINE.json's "tiny random-init
 * ECoT transformer" and the 7B-shaped decoder are builder-defined (SURVEY.md
 * finding 0.5), so this file is the *definition* of the model arithmetic that
 * the B200 engine must reproduce bit for bit in fp32 mode:
 *
 *   - Llama-style decoder (RMSNorm, RoPE rotate-half, MHA, SwiGLU, untied
 *     lm_head), weights from the counter-based init of model.py;
 *   - canonical dot product `cdot` (32 lane partials, float4-strided, fmaf in
 *     order, then the xor-butterfly 16/8/4/2/1) used for every contraction;
 *   - attention in aligned 64-position chunks: two-pass softmax inside a
 *     chunk, then an in-order log-sum-exp merge of the chunk partials;
 *   - a deterministic exp (`fe_exp`) built from fmaf, rintf and exponent bits;
 *   - greedy argmax over the first n_text logits, lowest index on ties.
 *
 * Parity anchors: request framing and lengths follow the reference's call
 * sites (schedulers.py:329-351 sequential prefixes, :399-404 branch prefixes,
 * :471-509 async snapshot prefixes) through oracle/backend.py; golden traces
 * are produced by the reference runners over this model (tests/golden/).
 *
 * Build: oracle/Makefile (gcc -O3 -fopenmp -ffp-contract=off); the explicit
 * fmaf() calls are the only fused operations.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>
#include <immintrin.h>

#define CHUNK 64

/* ---------------- counter-based init (model.py) ---------------- */
static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static uint64_t tensor_key(uint64_t seed, uint64_t tid) { return splitmix64(splitmix64(seed) ^ tid); }
static inline float centered(uint64_t key, uint64_t i) {
    float u = (float)(splitmix64(key + i) >> 40);
    return u * 0x1p-24f - 0.5f;
}
static const float LINEAR_MULT = 0x1.1bc77ap-4f;
static const float VISION_MULT = 0x1.bb67aep+1f;
static const float NORM_MULT = 0x1.99999ap-3f;

enum { T_EMBED = 1, T_LM_HEAD = 2, T_FINAL_NORM = 3, T_VISION = 4, T_LAYER_BASE = 16, T_LAYER_STRIDE = 16 };
enum { L_ATTN_NORM, L_WQ, L_WK, L_WV, L_WO, L_FFN_NORM, L_WGATE, L_WUP, L_WDOWN };

static void fill_linear(float* w, uint64_t seed, uint64_t tid, size_t n) {
    uint64_t key = tensor_key(seed, tid);
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i++) w[i] = centered(key, i) * LINEAR_MULT;
}
static void fill_norm(float* w, uint64_t seed, uint64_t tid, size_t n) {
    uint64_t key = tensor_key(seed, tid);
    for (size_t i = 0; i < n; i++) w[i] = 1.0f + centered(key, i) * NORM_MULT;
}

/* ---------------- canonical arithmetic ---------------- */
static inline float cdot(const float* w, const float* x, int K) {
    float a[32];
    for (int l = 0; l < 32; l++) a[l] = 0.0f;
    for (int j = 0; j < K; j += 128)
        for (int l = 0; l < 32; l++) {
            int k = j + 4 * l;
            if (k < K) {
                a[l] = fmaf(w[k + 0], x[k + 0], a[l]);
                a[l] = fmaf(w[k + 1], x[k + 1], a[l]);
                a[l] = fmaf(w[k + 2], x[k + 2], a[l]);
                a[l] = fmaf(w[k + 3], x[k + 3], a[l]);
            }
        }
    for (int off = 16; off >= 1; off >>= 1)
        for (int l = 0; l < off; l++) a[l] = a[l] + a[l + off];
    return a[0];
}

static inline float fe_exp(float x) {
    if (!(x > -87.0f)) return 0.0f;
    if (x > 88.0f) x = 88.0f;
    float y = x * 0x1.715476p+0f;
    float n = rintf(y);
    float f = y - n;
    float p = 0x1.ffcbfcp-17f;
    p = fmaf(p, f, 0x1.430912p-13f);
    p = fmaf(p, f, 0x1.5d87fep-10f);
    p = fmaf(p, f, 0x1.3b2ab6p-7f);
    p = fmaf(p, f, 0x1.c6b08ep-5f);
    p = fmaf(p, f, 0x1.ebfbe0p-3f);
    p = fmaf(p, f, 0x1.62e430p-1f);
    p = fmaf(p, f, 1.0f);
    int32_t bits = ((int32_t)n + 127) << 23;
    float scale;
    memcpy(&scale, &bits, 4);
    return p * scale;
}

static inline void rmsnorm(float* y, const float* x, const float* w, int d, float eps) {
    float ss = cdot(x, x, d);
    float mean = ss / (float)d;
    float r = 1.0f / sqrtf(mean + eps);
    for (int k = 0; k < d; k++) y[k] = (x[k] * r) * w[k];
}

/* ---------------- model ---------------- */
typedef struct {
    float *attn_norm, *wq, *wk, *wv, *wo, *ffn_norm, *wg, *wu, *wd;
} layer_t;

typedef struct {
    int32_t* ids;     /* input ids of the cached sequence */
    uint64_t vseed;
    int n;            /* positions held */
    float* kv;        /* [L][2][n_cap][d] */
    int n_cap;
    uint64_t stamp;
} entry_t;

#define N_ENTRIES 16

typedef struct {
    int d, L, H, hd, F, V, n_text, max_pos;
    float eps, attn_scale;
    uint64_t seed;
    float *embed, *lm_head, *final_norm;
    layer_t* layers;
    float* rope;      /* [max_pos][2][hd/2] */
    entry_t cache[N_ENTRIES];
    uint64_t clock;
    struct or_vision* vision;   /* optional vision tower: VIS rows take its output */
} or_model;

typedef struct or_vision or_vision;
static const float* vision_rows(or_vision* v, uint64_t vseed);

or_model* or_create(int d, int L, int H, int hd, int F, int V, int n_text, float eps,
                    float attn_scale, uint64_t seed, const float* rope, int max_pos, int n_threads) {
    if (n_threads > 0) omp_set_num_threads(n_threads);
    or_model* m = (or_model*)calloc(1, sizeof(or_model));
    m->d = d; m->L = L; m->H = H; m->hd = hd; m->F = F; m->V = V; m->n_text = n_text;
    m->eps = eps; m->attn_scale = attn_scale; m->seed = seed; m->max_pos = max_pos;
    m->embed = (float*)malloc(sizeof(float) * (size_t)V * d);
    m->lm_head = (float*)malloc(sizeof(float) * (size_t)V * d);
    m->final_norm = (float*)malloc(sizeof(float) * d);
    fill_linear(m->embed, seed, T_EMBED, (size_t)V * d);
    fill_linear(m->lm_head, seed, T_LM_HEAD, (size_t)V * d);
    fill_norm(m->final_norm, seed, T_FINAL_NORM, d);
    m->layers = (layer_t*)calloc(L, sizeof(layer_t));
    for (int l = 0; l < L; l++) {
        layer_t* ly = &m->layers[l];
        uint64_t b = T_LAYER_BASE + (uint64_t)T_LAYER_STRIDE * l;
        size_t dd = (size_t)d * d, fd = (size_t)F * d;
        ly->attn_norm = (float*)malloc(sizeof(float) * d);
        ly->ffn_norm = (float*)malloc(sizeof(float) * d);
        ly->wq = (float*)malloc(sizeof(float) * dd);
        ly->wk = (float*)malloc(sizeof(float) * dd);
        ly->wv = (float*)malloc(sizeof(float) * dd);
        ly->wo = (float*)malloc(sizeof(float) * dd);
        ly->wg = (float*)malloc(sizeof(float) * fd);
        ly->wu = (float*)malloc(sizeof(float) * fd);
        ly->wd = (float*)malloc(sizeof(float) * fd);
        fill_norm(ly->attn_norm, seed, b + L_ATTN_NORM, d);
        fill_norm(ly->ffn_norm, seed, b + L_FFN_NORM, d);
        fill_linear(ly->wq, seed, b + L_WQ, dd);
        fill_linear(ly->wk, seed, b + L_WK, dd);
        fill_linear(ly->wv, seed, b + L_WV, dd);
        fill_linear(ly->wo, seed, b + L_WO, dd);
        fill_linear(ly->wg, seed, b + L_WGATE, fd);
        fill_linear(ly->wu, seed, b + L_WUP, fd);
        fill_linear(ly->wd, seed, b + L_WDOWN, fd);
    }
    m->rope = (float*)malloc(sizeof(float) * (size_t)max_pos * hd);
    memcpy(m->rope, rope, sizeof(float) * (size_t)max_pos * hd);
    return m;
}

void or_destroy(or_model* m) {
    if (!m) return;
    for (int l = 0; l < m->L; l++) {
        layer_t* ly = &m->layers[l];
        free(ly->attn_norm); free(ly->ffn_norm); free(ly->wq); free(ly->wk); free(ly->wv);
        free(ly->wo); free(ly->wg); free(ly->wu); free(ly->wd);
    }
    for (int e = 0; e < N_ENTRIES; e++) { free(m->cache[e].ids); free(m->cache[e].kv); }
    free(m->layers); free(m->embed); free(m->lm_head); free(m->final_norm); free(m->rope); free(m);
}

/*
 * Canonical dots of one weight row against 32 tokens at once (AVX2): the
 * 8-wide vectors run across TOKENS, so every (row, token) dot keeps exactly
 * cdot's order -- lane l accumulates k = 128j + 4l + c (j, then c ascending)
 * with one fused multiply-add each, then the xor butterfly.  Only the loop
 * order over lanes changes (lanes are independent), so results are
 * bit-identical to cdot.  xT holds 4 blocks of 8 tokens as [block][K][8].
 */
static void cdot_rows32(float* out, const float* w, const float* xT, int K, int N_out_stride) {
    __m256 part[4][32];
    for (int l = 0; l < 32; l++) {
        __m256 a0 = _mm256_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
        for (int j = 0; j + 4 * l < K; j += 128) {
            int k = j + 4 * l;
            for (int c = 0; c < 4; c++) {
                __m256 wv = _mm256_set1_ps(w[k + c]);
                const float* xp = xT + (size_t)(k + c) * 8;
                a0 = _mm256_fmadd_ps(wv, _mm256_loadu_ps(xp), a0);
                a1 = _mm256_fmadd_ps(wv, _mm256_loadu_ps(xp + (size_t)K * 8), a1);
                a2 = _mm256_fmadd_ps(wv, _mm256_loadu_ps(xp + (size_t)K * 16), a2);
                a3 = _mm256_fmadd_ps(wv, _mm256_loadu_ps(xp + (size_t)K * 24), a3);
            }
        }
        part[0][l] = a0; part[1][l] = a1; part[2][l] = a2; part[3][l] = a3;
    }
    for (int b = 0; b < 4; b++) {
        for (int off = 16; off >= 1; off >>= 1)
            for (int l = 0; l < off; l++) part[b][l] = _mm256_add_ps(part[b][l], part[b][l + off]);
        float tmp[8];
        _mm256_storeu_ps(tmp, part[b][0]);
        for (int i = 0; i < 8; i++) out[(size_t)(8 * b + i) * N_out_stride] = tmp[i];
    }
}

/* y[n][N] = x[n][K] . W[N][K]^T, every element a canonical dot */
static void matmul(float* y, const float* x, const float* W, int n, int N, int K) {
    int n32 = (K % 4 == 0) ? n / 32 * 32 : 0;
    if (n32) {
        float* xT = (float*)malloc(sizeof(float) * (size_t)32 * K);
        for (int t0 = 0; t0 < n32; t0 += 32) {
            for (int b = 0; b < 4; b++)
                for (int k = 0; k < K; k++)
                    for (int i = 0; i < 8; i++)
                        xT[((size_t)b * K + k) * 8 + i] = x[(size_t)(t0 + 8 * b + i) * K + k];
#pragma omp parallel for schedule(static)
            for (int r = 0; r < N; r++) cdot_rows32(y + (size_t)t0 * N + r, W + (size_t)r * K, xT, K, N);
        }
        free(xT);
    }
#pragma omp parallel for schedule(static)
    for (int r = 0; r < N; r++)
        for (int t = n32; t < n; t++) y[(size_t)t * N + r] = cdot(W + (size_t)r * K, x + (size_t)t * K, K);
}

static void rope_apply(const or_model* m, float* v, int pos) {
    int half = m->hd / 2;
    const float* cs = m->rope + (size_t)pos * m->hd;   /* cos[half], sin[half] */
    for (int h = 0; h < m->H; h++) {
        float* x = v + h * m->hd;
        for (int i = 0; i < half; i++) {
            float c = cs[i], s = cs[half + i];
            float x1 = x[i], x2 = x[i + half];
            float t1 = x2 * s, t2 = x1 * s;
            x[i] = fmaf(x1, c, -t1);
            x[i + half] = fmaf(x2, c, t2);
        }
    }
}

/* attention of one query row (all heads) at position pos over kvK/kvV [pos+1][d] */
static void attend(const or_model* m, float* out, const float* q, const float* kK, const float* kV, int pos) {
    int hd = m->hd, d = m->d, nc = pos / CHUNK + 1;
    float s[CHUNK];
    float* pm = (float*)malloc(sizeof(float) * nc);
    float* pl = (float*)malloc(sizeof(float) * nc);
    float* po = (float*)malloc(sizeof(float) * (size_t)nc * hd);
    for (int h = 0; h < m->H; h++) {
        const float* qh = q + h * hd;
        for (int c = 0; c < nc; c++) {
            int a = c * CHUNK, b = a + CHUNK;
            if (b > pos + 1) b = pos + 1;
            float mx = -INFINITY;
            for (int j = a; j < b; j++) {
                s[j - a] = cdot(qh, kK + (size_t)j * d + h * hd, hd) * m->attn_scale;
                mx = fmaxf(mx, s[j - a]);
            }
            float l = 0.0f;
            float* o = po + (size_t)c * hd;
            for (int i = 0; i < hd; i++) o[i] = 0.0f;
            for (int j = a; j < b; j++) {
                float p = fe_exp(s[j - a] - mx);
                l = l + p;
                const float* vv = kV + (size_t)j * d + h * hd;
                for (int i = 0; i < hd; i++) o[i] = fmaf(p, vv[i], o[i]);
            }
            pm[c] = mx; pl[c] = l;
        }
        float M = -INFINITY;
        for (int c = 0; c < nc; c++) M = fmaxf(M, pm[c]);
        float L = 0.0f;
        float* oh = out + h * hd;
        for (int i = 0; i < hd; i++) oh[i] = 0.0f;
        for (int c = 0; c < nc; c++) {
            float sc = fe_exp(pm[c] - M);
            L = fmaf(sc, pl[c], L);
            for (int i = 0; i < hd; i++) oh[i] = fmaf(sc, po[(size_t)c * hd + i], oh[i]);
        }
        for (int i = 0; i < hd; i++) oh[i] = oh[i] / L;
    }
    free(pm); free(pl); free(po);
}

static void embed_rows(const or_model* m, float* x, const int32_t* ids, int p0, int n, uint64_t vseed,
                       int vis_id) {
    uint64_t vkey = tensor_key(vseed, T_VISION);
    const float* vis = m->vision ? vision_rows(m->vision, vseed) : NULL;
    for (int t = 0; t < n; t++) {
        int pos = p0 + t;
        float* row = x + (size_t)t * m->d;
        if (ids[pos] == vis_id && vis) {
            memcpy(row, vis + (size_t)(pos - 1) * m->d, sizeof(float) * m->d);
        } else if (ids[pos] == vis_id) {
            uint64_t base = (uint64_t)(pos - 1) * m->d;
            for (int k = 0; k < m->d; k++) row[k] = centered(vkey, base + k) * VISION_MULT;
        } else {
            memcpy(row, m->embed + (size_t)ids[pos] * m->d, sizeof(float) * m->d);
        }
    }
}

/* forward rows [p0, p0+n) of one sequence; kv = [L][2][cap][d]; returns final hidden in x */
static void forward(const or_model* m, float* x, int p0, int n, float* kv, int cap) {
    int d = m->d, F = m->F;
    float* xn = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* q = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* k = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* v = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* att = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* g = (float*)malloc(sizeof(float) * (size_t)n * F);
    float* u = (float*)malloc(sizeof(float) * (size_t)n * F);
    for (int l = 0; l < m->L; l++) {
        const layer_t* ly = &m->layers[l];
        float* kK = kv + ((size_t)l * 2 + 0) * cap * d;
        float* kV = kv + ((size_t)l * 2 + 1) * cap * d;
        for (int t = 0; t < n; t++) rmsnorm(xn + (size_t)t * d, x + (size_t)t * d, ly->attn_norm, d, m->eps);
        matmul(q, xn, ly->wq, n, d, d);
        matmul(k, xn, ly->wk, n, d, d);
        matmul(v, xn, ly->wv, n, d, d);
        for (int t = 0; t < n; t++) {
            rope_apply(m, q + (size_t)t * d, p0 + t);
            rope_apply(m, k + (size_t)t * d, p0 + t);
            memcpy(kK + (size_t)(p0 + t) * d, k + (size_t)t * d, sizeof(float) * d);
            memcpy(kV + (size_t)(p0 + t) * d, v + (size_t)t * d, sizeof(float) * d);
        }
#pragma omp parallel for schedule(dynamic)
        for (int t = 0; t < n; t++) attend(m, att + (size_t)t * d, q + (size_t)t * d, kK, kV, p0 + t);
        matmul(q, att, ly->wo, n, d, d);
        for (size_t i = 0; i < (size_t)n * d; i++) x[i] = x[i] + q[i];
        for (int t = 0; t < n; t++) rmsnorm(xn + (size_t)t * d, x + (size_t)t * d, ly->ffn_norm, d, m->eps);
        matmul(g, xn, ly->wg, n, F, d);
        matmul(u, xn, ly->wu, n, F, d);
        for (size_t i = 0; i < (size_t)n * F; i++) {
            float e = fe_exp(-g[i]);
            float sg = g[i] / (1.0f + e);
            g[i] = sg * u[i];
        }
        matmul(q, g, ly->wd, n, d, F);
        for (size_t i = 0; i < (size_t)n * d; i++) x[i] = x[i] + q[i];
    }
    free(xn); free(q); free(k); free(v); free(att); free(g); free(u);
}

static int head_argmax(const or_model* m, const float* h, float* logits_out) {
    float* xn = (float*)malloc(sizeof(float) * m->d);
    float* lg = logits_out ? logits_out : (float*)malloc(sizeof(float) * m->V);
    rmsnorm(xn, h, m->final_norm, m->d, m->eps);
    matmul(lg, xn, m->lm_head, 1, m->V, m->d);
    int best = 0;
    for (int i = 1; i < m->n_text; i++)
        if (lg[i] > lg[best]) best = i;
    free(xn);
    if (!logits_out) free(lg);
    return best;
}

/*
 * Greedy generation for one request: `ids[0:n_in]` is the framed input
 * (context, prefix, step tag), VIS placeholders take vision row pos-1 of the
 * embedding seeded by `vseed`.  Emits n_out tokens; `logits` (nullable)
 * receives [n_out][V].  A prefix cache of recent sequences supplies the KV of
 * the longest shared input prefix (exact: KV at p depends on ids[0..p] only).
 */
int or_generate(or_model* m, const int32_t* ids, int n_in, uint64_t vseed, int vis_id,
                int n_out, int32_t* out, float* logits) {
    if (n_in < 1 || n_out < 1 || n_in + n_out > m->max_pos) return -1;
    int d = m->d, cap = n_in + n_out;
    float* kv = (float*)malloc(sizeof(float) * (size_t)m->L * 2 * cap * d);
    int32_t* seq = (int32_t*)malloc(sizeof(int32_t) * cap);
    memcpy(seq, ids, sizeof(int32_t) * n_in);
    /* longest common prefix with a cached sequence (keep >= 1 row to compute) */
    int best = -1, lcp = 0;
    for (int e = 0; e < N_ENTRIES; e++) {
        entry_t* en = &m->cache[e];
        if (!en->ids || en->vseed != vseed) continue;
        int lim = en->n < n_in - 1 ? en->n : n_in - 1, p = 0;
        while (p < lim && en->ids[p] == ids[p]) p++;
        if (p > lcp) { lcp = p; best = e; }
    }
    if (best >= 0)
        for (int l = 0; l < m->L; l++)
            for (int s = 0; s < 2; s++)
                memcpy(kv + ((size_t)l * 2 + s) * cap * d,
                       m->cache[best].kv + ((size_t)l * 2 + s) * m->cache[best].n_cap * d,
                       sizeof(float) * (size_t)lcp * d);
    int n = n_in - lcp;
    float* x = (float*)malloc(sizeof(float) * (size_t)n * d);
    embed_rows(m, x, seq, lcp, n, vseed, vis_id);
    forward(m, x, lcp, n, kv, cap);
    const float* last = x + (size_t)(n - 1) * d;
    float* h = (float*)malloc(sizeof(float) * d);
    memcpy(h, last, sizeof(float) * d);
    for (int s = 0; s < n_out; s++) {
        int tok = head_argmax(m, h, logits ? logits + (size_t)s * m->V : NULL);
        out[s] = tok;
        if (s + 1 == n_out) break;
        int pos = n_in + s;
        seq[pos] = tok;
        embed_rows(m, h, seq, pos, 1, vseed, vis_id);
        forward(m, h, pos, 1, kv, cap);
    }
    /* remember this request's input KV (LRU replacement) */
    int slot = 0;
    for (int e = 0; e < N_ENTRIES; e++) {
        if (!m->cache[e].ids) { slot = e; break; }
        if (m->cache[e].stamp < m->cache[slot].stamp) slot = e;
    }
    entry_t* en = &m->cache[slot];
    free(en->ids); free(en->kv);
    en->ids = seq; en->kv = kv; en->n = n_in; en->n_cap = cap; en->vseed = vseed; en->stamp = ++m->clock;
    free(x); free(h);
    return 0;
}

/* ---- kernel-level restatements, for per-kernel parity tests ---- */
float or_cdot(const float* w, const float* x, int K) { return cdot(w, x, K); }
float or_exp(float x) { return fe_exp(x); }
void or_rmsnorm(float* y, const float* x, const float* w, int d, float eps) { rmsnorm(y, x, w, d, eps); }
void or_matmul(float* y, const float* x, const float* W, int n, int N, int K) { matmul(y, x, W, n, N, K); }

/* attention of `n` query rows at positions pos[t] over per-position K/V [*, H*hd] */
void or_attention(const or_model* m, float* out, const float* q, const float* K, const float* V,
                  const int32_t* pos, int n) {
    for (int t = 0; t < n; t++) attend(m, out + (size_t)t * m->d, q + (size_t)t * m->d, K, V, pos[t]);
}

/* copy of a weight tensor, for engine-vs-oracle weight checks */
const float* or_tensor(const or_model* m, int which, int layer) {
    if (which == T_EMBED) return m->embed;
    if (which == T_LM_HEAD) return m->lm_head;
    if (which == T_FINAL_NORM) return m->final_norm;
    const layer_t* ly = &m->layers[layer];
    switch ((which - T_LAYER_BASE) % T_LAYER_STRIDE) {
        case L_ATTN_NORM: return ly->attn_norm;
        case L_WQ: return ly->wq;
        case L_WK: return ly->wk;
        case L_WV: return ly->wv;
        case L_WO: return ly->wo;
        case L_FFN_NORM: return ly->ffn_norm;
        case L_WGATE: return ly->wg;
        case L_WUP: return ly->wu;
        case L_WDOWN: return ly->wd;
    }
    return NULL;
}

/* ================= vision tower + projector ===========
 * A pre-LayerNorm ViT over a synthetic image of the observation, then a
 * 2-layer MLP projector into the LLM width: the 256 (n_vision) VIS rows.
 * Restated by csrc/vision.cu in the same canonical arithmetic (fp32 mode
 * bit-exact).  Definition:
 *   pixel(c, y, x)  = 2 * centered(key(vseed, T_IMAGE), (c * img + y) * img + x)
 *   patch p (row-major grid), feature f = (c * P + dy) * P + dx, zero-padded to kp
 *   x = cdot(pe_w, patch) ; x = x + pe_b ; x = x + pos[p]
 *   layer: x += O(attn(LN1 x)) ; x += fc2(gelu(fc1(LN2 x)))   (linears add their bias after the dot)
 *   LN(x) = ((x - mean) * r) * g + b, mean = cdot(x, 1) / d, r = 1 / sqrt(cdot(xc, xc) / d + eps)
 *   attn: non-causal over all P patches, s = cdot(q, k) * hd^-1/2, fe_exp softmax, in order
 *   gelu(z) = z / (1 + fe_exp(-1.702 z))
 *   out = p2(gelu(p1(LN_f x)))
 */
enum { T_IMAGE = 5, T_VB = 1 << 20 };
enum { V_PE_W, V_PE_B, V_POS, V_LNF_G, V_LNF_B, V_P1_W, V_P1_B, V_P2_W, V_P2_B };
enum { VL_LN1_G, VL_LN1_B, VL_QKV_W, VL_QKV_B, VL_O_W, VL_O_B, VL_LN2_G, VL_LN2_B, VL_FC1_W, VL_FC1_B,
       VL_FC2_W, VL_FC2_B };

typedef struct {
    float *ln1_g, *ln1_b, *qkv_w, *qkv_b, *o_w, *o_b, *ln2_g, *ln2_b, *fc1_w, *fc1_b, *fc2_w, *fc2_b;
} vlayer_t;

#define V_CACHE 8
struct or_vision {
    int img, patch, grid, P, d, L, H, hd, mlp, ph, out, kp;
    float eps;
    uint64_t seed;
    float *pe_w, *pe_b, *pos, *lnf_g, *lnf_b, *p1_w, *p1_b, *p2_w, *p2_b;
    vlayer_t* layers;
    uint64_t cache_seed[V_CACHE];
    float* cache_out[V_CACHE];
    int cache_next;
};

static float* vfill(uint64_t seed, uint64_t tid, size_t n, int norm) {
    float* w = (float*)malloc(sizeof(float) * n);
    if (norm) fill_norm(w, seed, tid, n);
    else fill_linear(w, seed, tid, n);
    return w;
}

or_vision* or_vision_create(int img, int patch, int d, int L, int H, int mlp, int ph, int out, float eps,
                            uint64_t seed) {
    or_vision* v = (or_vision*)calloc(1, sizeof(or_vision));
    v->img = img; v->patch = patch; v->grid = img / patch; v->P = v->grid * v->grid;
    v->d = d; v->L = L; v->H = H; v->hd = d / H; v->mlp = mlp; v->ph = ph; v->out = out; v->eps = eps;
    v->kp = (3 * patch * patch + 127) / 128 * 128;
    v->seed = seed;
    v->pe_w = vfill(seed, T_VB + V_PE_W, (size_t)d * v->kp, 0);
    v->pe_b = vfill(seed, T_VB + V_PE_B, d, 0);
    v->pos = vfill(seed, T_VB + V_POS, (size_t)v->P * d, 0);
    v->lnf_g = vfill(seed, T_VB + V_LNF_G, d, 1);
    v->lnf_b = vfill(seed, T_VB + V_LNF_B, d, 0);
    v->p1_w = vfill(seed, T_VB + V_P1_W, (size_t)ph * d, 0);
    v->p1_b = vfill(seed, T_VB + V_P1_B, ph, 0);
    v->p2_w = vfill(seed, T_VB + V_P2_W, (size_t)out * ph, 0);
    v->p2_b = vfill(seed, T_VB + V_P2_B, out, 0);
    v->layers = (vlayer_t*)calloc(L, sizeof(vlayer_t));
    for (int l = 0; l < L; l++) {
        vlayer_t* y = &v->layers[l];
        uint64_t b = T_VB + 16 + 16 * (uint64_t)l;
        y->ln1_g = vfill(seed, b + VL_LN1_G, d, 1);
        y->ln1_b = vfill(seed, b + VL_LN1_B, d, 0);
        y->qkv_w = vfill(seed, b + VL_QKV_W, (size_t)3 * d * d, 0);
        y->qkv_b = vfill(seed, b + VL_QKV_B, (size_t)3 * d, 0);
        y->o_w = vfill(seed, b + VL_O_W, (size_t)d * d, 0);
        y->o_b = vfill(seed, b + VL_O_B, d, 0);
        y->ln2_g = vfill(seed, b + VL_LN2_G, d, 1);
        y->ln2_b = vfill(seed, b + VL_LN2_B, d, 0);
        y->fc1_w = vfill(seed, b + VL_FC1_W, (size_t)mlp * d, 0);
        y->fc1_b = vfill(seed, b + VL_FC1_B, mlp, 0);
        y->fc2_w = vfill(seed, b + VL_FC2_W, (size_t)d * mlp, 0);
        y->fc2_b = vfill(seed, b + VL_FC2_B, d, 0);
    }
    return v;
}

void or_vision_destroy(or_vision* v) {
    if (!v) return;
    for (int l = 0; l < v->L; l++) {
        vlayer_t* y = &v->layers[l];
        free(y->ln1_g); free(y->ln1_b); free(y->qkv_w); free(y->qkv_b); free(y->o_w); free(y->o_b);
        free(y->ln2_g); free(y->ln2_b); free(y->fc1_w); free(y->fc1_b); free(y->fc2_w); free(y->fc2_b);
    }
    for (int i = 0; i < V_CACHE; i++) free(v->cache_out[i]);
    free(v->layers); free(v->pe_w); free(v->pe_b); free(v->pos); free(v->lnf_g); free(v->lnf_b);
    free(v->p1_w); free(v->p1_b); free(v->p2_w); free(v->p2_b); free(v);
}

static void vlinear(float* y, const float* x, const float* W, const float* b, int n, int N, int K) {
    matmul(y, x, W, n, N, K);
    for (size_t i = 0; i < (size_t)n * N; i++) y[i] = y[i] + b[i % N];
}

static void vlayernorm(float* y, const float* x, const float* g, const float* b, int n, int d, float eps) {
    float* ones = (float*)malloc(sizeof(float) * d);
    float* xc = (float*)malloc(sizeof(float) * d);
    for (int k = 0; k < d; k++) ones[k] = 1.0f;
    for (int t = 0; t < n; t++) {
        const float* xr = x + (size_t)t * d;
        float mean = cdot(xr, ones, d) / (float)d;
        for (int k = 0; k < d; k++) xc[k] = xr[k] - mean;
        float var = cdot(xc, xc, d) / (float)d;
        float r = 1.0f / sqrtf(var + eps);
        for (int k = 0; k < d; k++) {
            float u = xc[k] * r;
            u = u * g[k];
            y[(size_t)t * d + k] = u + b[k];
        }
    }
    free(ones); free(xc);
}

static inline float vgelu(float z) { return z / (1.0f + fe_exp(-1.702f * z)); }

static void vattention(const or_vision* v, float* out, const float* qkv) {
    const int P = v->P, d = v->d, hd = v->hd;
    const float scale = 1.0f / sqrtf((float)hd);
#pragma omp parallel for schedule(static)
    for (int t = 0; t < P * v->H; t++) {
        int p = t / v->H, h = t % v->H;
        const float* q = qkv + (size_t)p * 3 * d + h * hd;
        float* s = (float*)malloc(sizeof(float) * P);
        float m = -INFINITY;
        for (int j = 0; j < P; j++) {
            s[j] = cdot(q, qkv + (size_t)j * 3 * d + d + h * hd, hd) * scale;
            if (s[j] > m) m = s[j];
        }
        float l = 0.0f;
        float o[256];
        for (int i = 0; i < hd; i++) o[i] = 0.0f;
        for (int j = 0; j < P; j++) {
            float pj = fe_exp(s[j] - m);
            l = l + pj;
            const float* vj = qkv + (size_t)j * 3 * d + 2 * d + h * hd;
            for (int i = 0; i < hd; i++) o[i] = fmaf(pj, vj[i], o[i]);
        }
        for (int i = 0; i < hd; i++) out[(size_t)p * d + h * hd + i] = o[i] / l;
        free(s);
    }
}

/* out[P][out] = vision rows of the observation seeded vseed */
int or_vision_encode(or_vision* v, uint64_t vseed, float* out) {
    const int P = v->P, d = v->d, kp = v->kp, ps = v->patch, img = v->img;
    float* patches = (float*)calloc((size_t)P * kp, sizeof(float));
    uint64_t ikey = tensor_key(vseed, T_IMAGE);
    for (int p = 0; p < P; p++) {
        int gy = p / v->grid, gx = p % v->grid;
        for (int c = 0; c < 3; c++)
            for (int dy = 0; dy < ps; dy++)
                for (int dx = 0; dx < ps; dx++) {
                    int y = gy * ps + dy, xx = gx * ps + dx;
                    patches[(size_t)p * kp + (c * ps + dy) * ps + dx] =
                        centered(ikey, (uint64_t)((c * img + y) * img + xx)) * 2.0f;
                }
    }
    float* x = (float*)malloc(sizeof(float) * (size_t)P * d);
    float* ln = (float*)malloc(sizeof(float) * (size_t)P * d);
    float* qkv = (float*)malloc(sizeof(float) * (size_t)P * 3 * d);
    float* att = (float*)malloc(sizeof(float) * (size_t)P * d);
    float* tmp = (float*)malloc(sizeof(float) * (size_t)P * d);
    float* hid = (float*)malloc(sizeof(float) * (size_t)P * (v->mlp > v->ph ? v->mlp : v->ph));
    vlinear(x, patches, v->pe_w, v->pe_b, P, d, kp);
    for (size_t i = 0; i < (size_t)P * d; i++) x[i] = x[i] + v->pos[i];
    for (int l = 0; l < v->L; l++) {
        const vlayer_t* y = &v->layers[l];
        vlayernorm(ln, x, y->ln1_g, y->ln1_b, P, d, v->eps);
        vlinear(qkv, ln, y->qkv_w, y->qkv_b, P, 3 * d, d);
        vattention(v, att, qkv);
        vlinear(tmp, att, y->o_w, y->o_b, P, d, d);
        for (size_t i = 0; i < (size_t)P * d; i++) x[i] = x[i] + tmp[i];
        vlayernorm(ln, x, y->ln2_g, y->ln2_b, P, d, v->eps);
        vlinear(hid, ln, y->fc1_w, y->fc1_b, P, v->mlp, d);
        for (size_t i = 0; i < (size_t)P * v->mlp; i++) hid[i] = vgelu(hid[i]);
        vlinear(tmp, hid, y->fc2_w, y->fc2_b, P, d, v->mlp);
        for (size_t i = 0; i < (size_t)P * d; i++) x[i] = x[i] + tmp[i];
    }
    vlayernorm(ln, x, v->lnf_g, v->lnf_b, P, d, v->eps);
    vlinear(hid, ln, v->p1_w, v->p1_b, P, v->ph, d);
    for (size_t i = 0; i < (size_t)P * v->ph; i++) hid[i] = vgelu(hid[i]);
    vlinear(out, hid, v->p2_w, v->p2_b, P, v->out, v->ph);
    free(patches); free(x); free(ln); free(qkv); free(att); free(tmp); free(hid);
    return 0;
}

static const float* vision_rows(or_vision* v, uint64_t vseed) {
    for (int i = 0; i < V_CACHE; i++)
        if (v->cache_out[i] && v->cache_seed[i] == vseed) return v->cache_out[i];
    int i = v->cache_next;
    v->cache_next = (v->cache_next + 1) % V_CACHE;
    if (!v->cache_out[i]) v->cache_out[i] = (float*)malloc(sizeof(float) * (size_t)v->P * v->out);
    or_vision_encode(v, vseed, v->cache_out[i]);
    v->cache_seed[i] = vseed;
    return v->cache_out[i];
}

/* VIS rows of every later generate take the tower's output (n_vision == P) */
int or_set_vision(or_model* m, or_vision* v) {
    if (v && v->out != m->d) return 1;
    m->vision = v;
    for (int e = 0; e < N_ENTRIES; e++) m->cache[e].n = 0;   /* KV cached under the old embeddings */
    return 0;
}
