/*
 * phub_oracle.c -- plain, slow, obviously-correct CPU oracle for the PHub
 * data-parallel hot path (arXiv 1805.07891).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_1805_07891_b200/), and it never reads anything the CUDA path wrote.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *   -ffp-contract=off : every fp32 add/mul below is rounded separately (no FMA),
 *                        DESIGN.md reading R5.
 *   x86-64 SSE arithmetic: no x87 excess precision, no FTZ/DAZ (reading R6).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 *
 * Functions and what pins them (tests/test_oracle_*.py):
 *   oracle_chunk_plan     P:693-698, P:703 ("chunks a gradient array into
 *                         mini-chunks of predefined sizes", 32KB default);
 *                         S:73-81.  Pinned: closed form ceil(n/ce),
 *                         S:80 (10000 -> 8192+1808), S:167 (137e6 -> 16,724),
 *                         coverage/bijection.
 *   oracle_owners_lpt     P:717 ("4/3 approximation set partition"); S:85 LPT
 *                         with index tie-breaks.  Pinned: S:89/S:106 worked
 *                         example, 4/3 bound vs brute force, totality.
 *   oracle_owners_contig  DESIGN.md reading R10 (contiguous owner ranges for
 *                         the NCCL path).  Pinned: monotone, balance bound.
 *   oracle_bruteforce     S:100-104 (exhaustive optimum, tiny instances).
 *                         Pinned: S:104 examples, hand-enumerated cases.
 *   oracle_round          P:657 (aggregation + optimization are element-wise),
 *                         P:677-686 (tall aggregation: one thread owns a chunk,
 *                         sums it over all workers, then the same thread
 *                         optimizes it), P:783 (Nesterov SGD).
 *                         Pinned: dyadic inputs == exact float64 sum, S:175,
 *                         signed-zero rule, S:193 hex values, multi-round
 *                         closed form, lr=0 identity, mu=0 SGD, convergence
 *                         bound, chunk-size / order invariance.
 *   oracle_elems          the same per-element arithmetic on gathered
 *                         elements (for sampled full-size parity).
 *   oracle_hier_round     P:746-763 (rack deployment, hierarchical reduction:
 *   oracle_hier_elems     per-rack aggregation, cross-rack aggregation, then
 *                         the optimizer), P:1008 (cross-rack accumulation one
 *                         rack after another).  Pinned: R = 1 and one worker
 *                         per rack reduce to oracle_round; dyadic inputs ==
 *                         exact float64 sum; a hand-computed case where the
 *                         two-level order differs from the flat one.
 *
 * The Nesterov recurrence is not printed in the paper (P:783 only names
 * "Nesterov's accelerated gradient method"); this oracle implements SPEC's
 * reading (R1):  v' = mu*v + g ;  w' = w - lr*(g + mu*v').
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_ERR_MANIFEST   (-2)
#define ORACLE_ERR_CHUNK_SIZE (-3)
#define ORACLE_ERR_CAPACITY   (-4)
#define ORACLE_ERR_ARG        (-1)

/* ---------------------------------------------------------------- chunking */
/* per key, count = ceil(n_k / ce) with ce = chunk_size_bytes / 4. */
int64_t oracle_chunk_count(const uint64_t* n, int32_t K, uint64_t chunk_bytes)
{
    if (K <= 0 || n == NULL) return ORACLE_ERR_MANIFEST;
    if (chunk_bytes == 0 || chunk_bytes % 4 != 0) return ORACLE_ERR_CHUNK_SIZE;
    uint64_t ce = chunk_bytes / 4, total = 0;
    for (int32_t k = 0; k < K; ++k) {
        if (n[k] == 0) return ORACLE_ERR_MANIFEST;
        total += (n[k] + ce - 1) / ce;
    }
    return (int64_t)total;
}

/* for each key in key order, chunks in offset order;
 * vkey ids dense; every chunk has length ce except a short last one. */
int64_t oracle_chunk_plan(const uint64_t* n, int32_t K, uint64_t chunk_bytes,
                          uint32_t* vkey_id, uint32_t* key_id, uint64_t* offset,
                          uint64_t* length, uint64_t cap)
{
    int64_t count = oracle_chunk_count(n, K, chunk_bytes);
    if (count < 0) return count;
    if ((uint64_t)count > cap) return ORACLE_ERR_CAPACITY;
    uint64_t ce = chunk_bytes / 4, j = 0;
    for (int32_t k = 0; k < K; ++k) {
        for (uint64_t off = 0; off < n[k]; off += ce) {
            vkey_id[j] = (uint32_t)j;
            key_id[j] = (uint32_t)k;
            offset[j] = off;
            length[j] = (n[k] - off < ce) ? (n[k] - off) : ce;
            ++j;
        }
    }
    return count;
}

/* ------------------------------------------------------------------ owners */
/* S:85 LPT: order chunks by length descending, ties lower vkey_id first; put
 * each on the currently least-loaded bin, ties lower bin index first. */
int oracle_owners_lpt(const uint64_t* length, uint64_t count, int32_t G, int32_t* owner)
{
    if (G < 1 || (count > 0 && (length == NULL || owner == NULL))) return ORACLE_ERR_ARG;
    uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * (count ? count : 1));
    uint64_t* load = (uint64_t*)calloc((size_t)G, sizeof(uint64_t));
    if (!order || !load) { free(order); free(load); return ORACLE_ERR_ARG; }
    for (uint64_t i = 0; i < count; ++i) order[i] = i;
    /* insertion sort: slow and obviously right */
    for (uint64_t i = 1; i < count; ++i) {
        uint64_t x = order[i], j = i;
        while (j > 0) {
            uint64_t y = order[j - 1];
            int before = (length[x] > length[y]) || (length[x] == length[y] && x < y);
            if (!before) break;
            order[j] = y;
            --j;
        }
        order[j] = x;
    }
    for (uint64_t i = 0; i < count; ++i) {
        int32_t best = 0;
        for (int32_t b = 1; b < G; ++b)
            if (load[b] < load[best]) best = b;
        owner[order[i]] = best;
        load[best] += length[order[i]];
    }
    free(order);
    free(load);
    return 0;
}

/* DESIGN.md R10: owner = min(G-1, floor((p + l/2) * G / E)) where p is the
 * element prefix before the chunk and l its length, in exact integers as
 * floor((2p + l) * G / (2E)). */
int oracle_owners_contig(const uint64_t* length, uint64_t count, int32_t G, int32_t* owner)
{
    if (G < 1 || (count > 0 && (length == NULL || owner == NULL))) return ORACLE_ERR_ARG;
    unsigned __int128 E = 0;
    for (uint64_t i = 0; i < count; ++i) E += length[i];
    unsigned __int128 p = 0;
    for (uint64_t i = 0; i < count; ++i) {
        unsigned __int128 num = (2 * p + length[i]) * (unsigned __int128)G;
        unsigned __int128 o = num / (2 * E);
        owner[i] = (o > (unsigned __int128)(G - 1)) ? G - 1 : (int32_t)o;
        p += length[i];
    }
    return 0;
}

/* exhaustive minimum of the maximum bin load (tiny instances). */
static void bf_rec(const uint64_t* len, uint64_t count, int32_t G, uint64_t i,
                   uint64_t* load, uint64_t cur_max, uint64_t* best)
{
    if (cur_max >= *best) return;
    if (i == count) { *best = cur_max; return; }
    for (int32_t b = 0; b < G; ++b) {
        load[b] += len[i];
        bf_rec(len, count, G, i + 1, load, load[b] > cur_max ? load[b] : cur_max, best);
        load[b] -= len[i];
    }
}

int64_t oracle_bruteforce_max_load(const uint64_t* length, uint64_t count, int32_t G)
{
    if (count > 14 || G < 1 || G > 4) return ORACLE_ERR_ARG;   /* S:100 guard */
    uint64_t load[4] = {0, 0, 0, 0};
    uint64_t best = UINT64_MAX;
    if (count == 0) return 0;
    bf_rec(length, count, G, 0, load, 0, &best);
    return (int64_t)best;
}

/* --------------------------------------------------- aggregation + optimizer */
/* One chunk, in the paper's tall order:
 *   1. merge buffer starts zeroed: +0.0f;
 *   2. workers' chunks are added in worker-id order (reading R3);
 *   3. the same thread then optimizes the chunk:
 *        g  = merge * rescale            (reading R2; rescale = 1/N default)
 *        v' = mu*v + g
 *        w' = w - lr*(g + mu*v')
 *      each operation rounded separately to fp32. */
static void oracle_chunk(int32_t N, const float* const* grads, uint64_t base,
                         uint64_t len, float* w, float* v, float* agg,
                         float lr, float mu, float rescale, float* merge)
{
    for (uint64_t j = 0; j < len; ++j) merge[j] = 0.0f;
    for (int32_t wk = 0; wk < N; ++wk) {
        const float* g = grads[wk] + base;
        for (uint64_t j = 0; j < len; ++j) {
            float s = merge[j] + g[j];
            merge[j] = s;
        }
    }
    for (uint64_t j = 0; j < len; ++j) {
        float g = merge[j] * rescale;
        float t1 = mu * v[base + j];
        float vn = t1 + g;
        float t2 = mu * vn;
        float t3 = g + t2;
        float t4 = lr * t3;
        float wn = w[base + j] - t4;
        v[base + j] = vn;
        w[base + j] = wn;
        if (agg) agg[base + j] = merge[j];
    }
}

/* One full push/aggregate/optimize round over every vkey of the model.
 * grads[wk]: worker wk's gradient, E elements, key-major, unpadded.
 * w, v: E elements each, updated in place.  agg: optional E-element output of
 * the worker-order sum.  vkey_order: optional permutation of vkey ids in
 * which chunks are processed (cross-chunk order independence).
 * nthreads > 1: chunks distributed statically over OpenMP threads, PHub's
 * chunk -> core mapping. */
int oracle_round(const uint64_t* n, int32_t K, uint64_t chunk_bytes, int32_t N,
                 const float* const* grads, float* w, float* v, float* agg,
                 float lr, float mu, float rescale, const uint32_t* vkey_order,
                 int32_t nthreads)
{
    if (N < 1 || grads == NULL || w == NULL || v == NULL) return ORACLE_ERR_ARG;
    int64_t count = oracle_chunk_count(n, K, chunk_bytes);
    if (count < 0) return (int)count;
    uint64_t cnt = (uint64_t)count, ce = chunk_bytes / 4;
    uint64_t* kbase = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)K);
    uint64_t* cbase = (uint64_t*)malloc(sizeof(uint64_t) * cnt);
    uint64_t* clen = (uint64_t*)malloc(sizeof(uint64_t) * cnt);
    if (!kbase || !cbase || !clen) { free(kbase); free(cbase); free(clen); return ORACLE_ERR_ARG; }
    uint64_t acc = 0, j = 0;
    for (int32_t k = 0; k < K; ++k) {
        kbase[k] = acc;
        for (uint64_t off = 0; off < n[k]; off += ce, ++j) {
            cbase[j] = acc + off;
            clen[j] = (n[k] - off < ce) ? (n[k] - off) : ce;
        }
        acc += n[k];
    }
    if (rescale == 0.0f) rescale = 1.0f / (float)N;
    int nt = nthreads < 1 ? 1 : nthreads;
#pragma omp parallel num_threads(nt)
    {
        float* merge = (float*)malloc(sizeof(float) * (size_t)ce);
#pragma omp for schedule(static)
        for (int64_t i = 0; i < (int64_t)cnt; ++i) {
            uint64_t c = vkey_order ? vkey_order[i] : (uint64_t)i;
            oracle_chunk(N, grads, cbase[c], clen[c], w, v, agg, lr, mu, rescale, merge);
        }
        free(merge);
    }
    free(kbase);
    free(cbase);
    free(clen);
    return 0;
}

/* Per-element arithmetic of oracle_chunk on gathered elements (sampled parity
 * at full size).  g is worker-major: g[wk*count + i]. */
void oracle_elems(uint64_t count, int32_t N, const float* g, float* w, float* v,
                  float* agg, float lr, float mu, float rescale)
{
    if (rescale == 0.0f) rescale = 1.0f / (float)N;
    for (uint64_t i = 0; i < count; ++i) {
        float merge = 0.0f;
        for (int32_t wk = 0; wk < N; ++wk) merge = merge + g[(uint64_t)wk * count + i];
        float gg = merge * rescale;
        float t1 = mu * v[i];
        float vn = t1 + gg;
        float t2 = mu * vn;
        float t3 = gg + t2;
        float t4 = lr * t3;
        w[i] = w[i] - t4;
        v[i] = vn;
        if (agg) agg[i] = merge;
    }
}

/* ------------------------------------------- hierarchical reduction (NEXT-4) */
/* PHub's rack deployment: "each PBox centrally aggregates gradient
 * updates from workers in the same rack; then, the PBox nodes start
 * cross-rack aggregation and compute globally aggregated gradients; finally,
 * each per-rack PBox runs an optimizer on this gradient".  The
 * paper's own emulation of the cross-rack step sends "N chunk-size messages
 * sequentially, each performing one additional aggregation", i.e. the
 * racks' aggregates are accumulated one rack after another (reading R17):
 *   rack r:   S_r = ((+0 + g_{rP}) + g_{rP+1}) + ... + g_{rP+P-1}
 *   global:   s   = ((+0 + S_0) + S_1) + ... + S_{R-1}
 *   then the same optimizer as oracle_chunk, rescale default 1/(R*P).
 * grads[r*P + k] is worker k of rack r.  Same layout/outputs as oracle_round. */
int oracle_hier_round(const uint64_t* n, int32_t K, uint64_t chunk_bytes, int32_t R, int32_t P,
                      const float* const* grads, float* w, float* v, float* agg,
                      float lr, float mu, float rescale)
{
    if (R < 1 || P < 1 || grads == NULL || w == NULL || v == NULL) return ORACLE_ERR_ARG;
    int64_t count = oracle_chunk_count(n, K, chunk_bytes);
    if (count < 0) return (int)count;
    uint64_t ce = chunk_bytes / 4;
    if (rescale == 0.0f) rescale = 1.0f / (float)(R * P);
    float* merge = (float*)malloc(sizeof(float) * (size_t)ce);
    float* rack = (float*)malloc(sizeof(float) * (size_t)ce);
    if (!merge || !rack) { free(merge); free(rack); return ORACLE_ERR_ARG; }
    uint64_t acc = 0;
    for (int32_t k = 0; k < K; ++k) {
        for (uint64_t off = 0; off < n[k]; off += ce) {          /* one chunk (vkey) */
            const uint64_t base = acc + off;
            const uint64_t len = (n[k] - off < ce) ? (n[k] - off) : ce;
            for (uint64_t j = 0; j < len; ++j) merge[j] = 0.0f;
            for (int32_t r = 0; r < R; ++r) {                      /* step 1: per rack */
                for (uint64_t j = 0; j < len; ++j) rack[j] = 0.0f;
                for (int32_t wk = 0; wk < P; ++wk) {
                    const float* g = grads[r * P + wk] + base;
                    for (uint64_t j = 0; j < len; ++j) rack[j] = rack[j] + g[j];
                }
                for (uint64_t j = 0; j < len; ++j) merge[j] = merge[j] + rack[j];  /* step 2 */
            }
            for (uint64_t j = 0; j < len; ++j) {                   /* step 3: optimizer */
                float g = merge[j] * rescale;
                float t1 = mu * v[base + j];
                float vn = t1 + g;
                float t2 = mu * vn;
                float t3 = g + t2;
                float t4 = lr * t3;
                float wn = w[base + j] - t4;
                v[base + j] = vn;
                w[base + j] = wn;
                if (agg) agg[base + j] = merge[j];
            }
        }
        acc += n[k];
    }
    free(merge);
    free(rack);
    return 0;
}

/* oracle_hier_round's arithmetic on gathered elements: g[(r*P + k)*count + i]. */
void oracle_hier_elems(uint64_t count, int32_t R, int32_t P, const float* g, float* w, float* v,
                       float* agg, float lr, float mu, float rescale)
{
    if (rescale == 0.0f) rescale = 1.0f / (float)(R * P);
    for (uint64_t i = 0; i < count; ++i) {
        float merge = 0.0f;
        for (int32_t r = 0; r < R; ++r) {
            float rack = 0.0f;
            for (int32_t wk = 0; wk < P; ++wk) rack = rack + g[(uint64_t)(r * P + wk) * count + i];
            merge = merge + rack;
        }
        float gg = merge * rescale;
        float t1 = mu * v[i];
        float vn = t1 + gg;
        float t2 = mu * vn;
        float t3 = gg + t2;
        float t4 = lr * t3;
        w[i] = w[i] - t4;
        v[i] = vn;
        if (agg) agg[i] = merge;
    }
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
