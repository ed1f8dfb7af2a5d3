// phub_core.cpp -- host side of libphub: the C ABI of include/phub.h.
//
//   manifest -> chunk plan -> chunk -> owner table
//   (LPT S:85 or CONTIG, reading R10) -> padded device layout ->
//   one-shot arenas -> per-(worker, key) receipts (P:686,
//   S:137-142) -> one fused kernel launch per round (phub_kernels.cu).
//
// Nothing here computes on the model data: every step of the numeric path
// runs in the sm_100a kernels.  Errors never throw across the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "phub.h"
#include "phub_kernels.cuh"

using phub::Tile;

namespace {

constexpr uint64_t kKeyAlign = 32;   // key starts rounded to 32 elements (128 B)
constexpr uint64_t kDefaultChunkBytes = 32768;

struct DeviceGuard {
    int prev = -1, dev;
    explicit DeviceGuard(int d) : dev(d) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

}  // namespace

struct phub_ctx_s {
    // configuration
    int device = 0;
    int N = 0, K = 0, G = 1, rank = 0, policy = PHUB_OWNER_CONTIG;
    uint64_t chunk_bytes = kDefaultChunkBytes, ce = kDefaultChunkBytes / 4;
    float lr = 0.f, mu = 0.f, rescale = 0.f;
    bool keep_agg = false;
    int num_sms = 148;

    // layout
    std::vector<uint64_t> n;          // key sizes
    std::vector<uint64_t> key_off;    // padded device offset of each key
    uint64_t E = 0, E_pad = 0;

    // chunk table + ownership
    std::vector<phub_chunk> chunks;
    std::vector<uint64_t> own_begin, own_end;   // CONTIG ranges per owner (padded layout)
    uint64_t owned_elems = 0;
    uint64_t n_tiles = 0;
    Tile* d_tiles = nullptr;
    std::vector<uint64_t> key_tile_begin, key_tile_end;   // owned tiles of key k, in order
    uint32_t tile_elems = 1024;       // measured best (profiles/r01_tune: tiles1024)

    // arenas
    float* d_w = nullptr;
    float* d_v = nullptr;
    float* d_agg = nullptr;
    float* d_recv = nullptr;          // N x E_pad, allocated on first COPY push

    // push state (iteration-scoped)
    std::vector<uint8_t> got;         // K x N receipts
    uint64_t got_count = 0;
    std::vector<uint8_t> done;        // key aggregated this iteration (streaming, NEXT-1)
    uint64_t done_count = 0;
    std::vector<uintptr_t> base;      // N x K: base + 4*dev_off = byte address
    std::vector<uintptr_t> base_uploaded;
    uintptr_t* d_base = nullptr;
    std::vector<float*> replicas;     // peer weight replicas written by the kernel
    uint64_t range_cursor = UINT64_MAX;   // phub_aggregate_range progress (UINT64_MAX: none)
    uint32_t* d_sync = nullptr;           // [0] CTA counter, [1] timeouts, [2] abandoned wait value,
                                          // [5] consumer-lane ticket (k_sched), [6] spare,
                                          // [3] block ticket, [4] CTAs done (block streaming)
    uint32_t* h_err = nullptr;            // host-mapped word a kernel sets on an expired wait
    uint32_t* d_err = nullptr;            // its device address (kernel argument)

    // options + counters
    int kernel = PHUB_KERNEL_AUTO;
    int grid_override = 0;
    int flat_oneshot = -1;            // -1 auto: one-shot for local HBM streams (profiles/
                                      // r01_tune2), persistent grid when peer replicas are
                                      // registered (NVLink latency; profiles/r01_multi2)
    int cache = PHUB_CACHE_RESIDENT;  // a fixed L2-resident slice of w, the rest evict-first:
                                      // measured fastest on B200 (R14, NEXT-2)
    uint64_t resident_bytes = 32ull << 20;   // PHUB_OPT_L2_RESIDENT (profiles/r02_l2/: 32 MiB best)
    int flat_grid[2][2] = {{0, 0}, {0, 0}};   // [vec8?][agg]
    int blocks_occ[2][phub::kMaxWorkers + 1] = {};      // resident CTAs/SM [nag][nw]
    int hier_occ[2] = {0, 0};                          // resident CTAs/SM of k_hier [worker_order]
    // scheduled exchange (phub_sched_load / phub_sched_exchange)
    phub::SchedItem* d_items = nullptr;
    uint64_t n_items = 0, n_prod = 0;    // items [0, n_prod) producer lane, the rest consumers
    double cons_frac = 0.0;               // consumer share of the items' elements
    uint64_t* sched_trace = nullptr;      // PHUB_OPT_SCHED_TRACE (diagnostic)
    int sched_ranks = 0, sched_rank = -1;
    uint32_t sched_flags = 0;
    int sched_occ = 0;
    uint64_t iteration = 0;
    int launches = 0;
    uint64_t launches_total = 0;
    bool failed = false;
    phub_status sticky = PHUB_OK;     // status every later call returns once failed
    std::string err;

    phub_status fail(phub_status s, const char* fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        return s;
    }
    phub_status cuda_fail(cudaError_t e, const char* where) {
        failed = true;
        sticky = PHUB_ERR_CUDA;
        err = std::string(where) + ": " + cudaGetErrorString(e);
        return e == cudaErrorMemoryAllocation ? PHUB_ERR_OUT_OF_MEMORY : PHUB_ERR_CUDA;
    }
    // Entry check of every state-changing or data-returning call: a sticky
    // failure, or a device-side wait that expired since the last call (the
    // kernel raised the host-mapped word; reading it needs no synchronize).
    phub_status guard() {
        if (!failed && h_err && *reinterpret_cast<volatile uint32_t*>(h_err)) {
            failed = true;
            sticky = PHUB_ERR_SYNC_TIMEOUT;
            err = "a device-side flag wait expired (~2 s): that launch skipped work, so the "
                  "round's results are incomplete; the context is sticky-failed";
        }
        return failed ? sticky : PHUB_OK;
    }
};

static const char* kStatusNames[] = {
    "PHUB_OK",
    "PHUB_ERR_INVALID_ARGUMENT",
    "PHUB_ERR_INVALID_MANIFEST",
    "PHUB_ERR_INVALID_CHUNK_SIZE",
    "PHUB_ERR_INVALID_INIT",
    "PHUB_ERR_BAD_WORKER",
    "PHUB_ERR_BAD_KEY",
    "PHUB_ERR_LENGTH_MISMATCH",
    "PHUB_ERR_DUPLICATE_PUSH",
    "PHUB_ERR_INCOMPLETE",
    "PHUB_ERR_CUDA",
    "PHUB_ERR_OUT_OF_MEMORY",
    "PHUB_ERR_UNSUPPORTED",
    "PHUB_ERR_SYNC_TIMEOUT",
};

// ------------------------------------------------------------ table logic
// Chunk plan: per key in key order, ceil(n_k / ce) chunks;
// then owners: G == 1 -> 0; LPT or CONTIG (reading R10).
static std::vector<phub_chunk> plan_chunks(const std::vector<uint64_t>& n, uint64_t ce, int G,
                                           int policy) {
    std::vector<phub_chunk> chunks;
    uint64_t E = 0;
    for (size_t k = 0; k < n.size(); ++k) {
        E += n[k];
        for (uint64_t off = 0; off < n[k]; off += ce) {
            phub_chunk ch{};
            ch.vkey_id = (uint32_t)chunks.size();
            ch.key_id = (uint32_t)k;
            ch.offset = off;
            ch.length = std::min(ce, n[k] - off);
            ch.owner = 0;
            chunks.push_back(ch);
        }
    }
    if (G == 1) return chunks;
    if (policy == PHUB_OWNER_LPT) {
        // length desc, ties lower vkey_id; least-loaded owner, ties lower index
        std::vector<uint32_t> order(chunks.size());
        for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
            return chunks[a].length > chunks[b].length;
        });
        std::vector<uint64_t> load(G, 0);
        for (uint32_t i : order) {
            int best = 0;
            for (int b = 1; b < G; ++b)
                if (load[b] < load[best]) best = b;
            chunks[i].owner = best;
            load[best] += chunks[i].length;
        }
    } else {
        // owner = min(G-1, floor((2p + l) G / 2E)), p = element prefix before the chunk
        unsigned __int128 p = 0;
        const unsigned __int128 twoE = (unsigned __int128)2 * E;
        for (auto& ch : chunks) {
            unsigned __int128 o = ((2 * p + ch.length) * (unsigned __int128)G) / twoE;
            ch.owner = o > (unsigned __int128)(G - 1) ? G - 1 : (int32_t)o;
            p += ch.length;
        }
    }
    return chunks;
}

// Padded key-major layout: every key starts on a 128-B boundary.
static void layout_keys(phub_ctx c) {
    c->key_off.resize(c->K);
    uint64_t off = 0;
    c->E = 0;
    for (int k = 0; k < c->K; ++k) {
        off = (off + kKeyAlign - 1) / kKeyAlign * kKeyAlign;
        c->key_off[k] = off;
        off += c->n[k];
        c->E += c->n[k];
    }
    c->E_pad = (off + kKeyAlign - 1) / kKeyAlign * kKeyAlign;
}

static uint64_t chunk_dev_off(phub_ctx c, const phub_chunk& ch) {
    return c->key_off[ch.key_id] + ch.offset;
}

// CONTIG ranges in the padded layout: owner o covers from its first chunk's
// device offset up to the next owner's first chunk (padding included).
static void build_ranges(phub_ctx c) {
    c->own_begin.assign(c->G, 0);
    c->own_end.assign(c->G, 0);
    if (!(c->G == 1 || c->policy == PHUB_OWNER_CONTIG)) return;
    std::vector<int64_t> first(c->G, -1);
    for (const auto& ch : c->chunks)
        if (first[ch.owner] < 0) first[ch.owner] = (int64_t)chunk_dev_off(c, ch);
    uint64_t next = c->E_pad;
    for (int o = c->G - 1; o >= 0; --o) {
        if (first[o] < 0) {
            c->own_begin[o] = c->own_end[o] = next;
        } else {
            c->own_begin[o] = (uint64_t)first[o];
            c->own_end[o] = next;
            next = (uint64_t)first[o];
        }
    }
}

static bool contig_mode(phub_ctx c) { return c->G == 1 || c->policy == PHUB_OWNER_CONTIG; }

// Owned chunks split into CTA tiles of <= tile_elems (chunk-tile kernel).
// Tiles stay in vkey order, so each key's tiles are one index range.
static std::vector<Tile> build_tiles(phub_ctx c) {
    std::vector<Tile> tiles;
    c->key_tile_begin.assign(c->K, 0);
    c->key_tile_end.assign(c->K, 0);
    for (const auto& ch : c->chunks) {
        if (ch.owner != c->rank) continue;
        if (c->key_tile_end[ch.key_id] == 0) c->key_tile_begin[ch.key_id] = tiles.size();
        for (uint64_t o = 0; o < ch.length; o += c->tile_elems) {
            Tile t;
            t.off = chunk_dev_off(c, ch) + o;
            t.len = (uint32_t)std::min<uint64_t>(c->tile_elems, ch.length - o);
            t.key = ch.key_id;
            tiles.push_back(t);
        }
        c->key_tile_end[ch.key_id] = tiles.size();
    }
    return tiles;
}

// ------------------------------------------------------------------ C ABI
extern "C" {

void phub_config_default(phub_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof *cfg);
    cfg->chunk_size_bytes = kDefaultChunkBytes;
    cfg->num_workers = 1;
    cfg->lr = 0.1f;
    cfg->momentum = 0.9f;
    cfg->rescale = 0.0f;
    cfg->num_owners = 1;
    cfg->owner_policy = PHUB_OWNER_CONTIG;
}

const char* phub_status_string(phub_status s) {
    if ((int)s < 0 || (size_t)s >= sizeof kStatusNames / sizeof kStatusNames[0])
        return "PHUB_ERR_UNKNOWN";
    return kStatusNames[s];
}

static thread_local std::string g_init_err;

const char* phub_last_error(phub_ctx ctx) { return ctx ? ctx->err.c_str() : g_init_err.c_str(); }

static phub_status validate_config(const phub_config* cfg, std::string& why) {
    auto bad = [&](phub_status s, const char* m) { why = m; return s; };
    if (!cfg) return bad(PHUB_ERR_INVALID_ARGUMENT, "cfg is NULL");
    if (cfg->num_keys <= 0 || !cfg->key_num_elements)
        return bad(PHUB_ERR_INVALID_MANIFEST, "manifest has no keys (S:68)");
    for (int k = 0; k < cfg->num_keys; ++k)
        if (cfg->key_num_elements[k] == 0)
            return bad(PHUB_ERR_INVALID_MANIFEST, "a key has zero elements (S:68)");
    if (cfg->chunk_size_bytes % 4 != 0)
        return bad(PHUB_ERR_INVALID_CHUNK_SIZE, "chunk_size_bytes must be a multiple of 4 (S:77)");
    if (cfg->num_workers < 1) return bad(PHUB_ERR_INVALID_ARGUMENT, "num_workers < 1");
    if (!std::isfinite(cfg->lr)) return bad(PHUB_ERR_INVALID_ARGUMENT, "lr not finite");
    if (!std::isfinite(cfg->momentum) || cfg->momentum < 0.f || cfg->momentum >= 1.f)
        return bad(PHUB_ERR_INVALID_ARGUMENT, "momentum must be in [0,1) (S:144)");
    if (!std::isfinite(cfg->rescale)) return bad(PHUB_ERR_INVALID_ARGUMENT, "rescale not finite");
    if (cfg->num_owners < 1 || cfg->owner_rank < 0 || cfg->owner_rank >= cfg->num_owners)
        return bad(PHUB_ERR_INVALID_ARGUMENT, "owner_rank must be in [0, num_owners)");
    if (cfg->owner_policy != PHUB_OWNER_LPT && cfg->owner_policy != PHUB_OWNER_CONTIG)
        return bad(PHUB_ERR_INVALID_ARGUMENT, "unknown owner_policy");
    if (cfg->device < 0) return bad(PHUB_ERR_INVALID_ARGUMENT, "device < 0");
    return PHUB_OK;
}

static void free_ctx(phub_ctx c) {
    if (!c) return;
    DeviceGuard g(c->device);
    cudaFree(c->d_w);
    cudaFree(c->d_v);
    cudaFree(c->d_agg);
    cudaFree(c->d_recv);
    cudaFree(c->d_tiles);
    cudaFree(c->d_base);
    cudaFree(c->d_sync);
    cudaFree(c->d_items);
    if (c->h_err) cudaFreeHost(c->h_err);
    delete c;
}

phub_status phub_init(const phub_config* cfg, phub_ctx* out) {
    std::string& why = g_init_err;
    why.clear();
    if (!out) return why = "out is NULL", PHUB_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    phub_status st = validate_config(cfg, why);
    if (st != PHUB_OK) return st;

    phub_ctx c = new (std::nothrow) phub_ctx_s();
    if (!c) return PHUB_ERR_OUT_OF_MEMORY;
    c->device = cfg->device;
    c->N = cfg->num_workers;
    c->K = cfg->num_keys;
    c->G = cfg->num_owners;
    c->rank = cfg->owner_rank;
    c->policy = cfg->owner_policy;
    c->chunk_bytes = cfg->chunk_size_bytes ? cfg->chunk_size_bytes : kDefaultChunkBytes;
    c->ce = c->chunk_bytes / 4;
    c->lr = cfg->lr;
    c->mu = cfg->momentum;
    c->rescale = cfg->rescale != 0.f ? cfg->rescale : 1.0f / (float)c->N;
    c->keep_agg = cfg->keep_aggregate != 0;
    c->n.assign(cfg->key_num_elements, cfg->key_num_elements + c->K);

    layout_keys(c);
    if (cfg->init_weights && cfg->init_num_elements != c->E) {
        delete c;
        why = "init_num_elements != E (S:163)";
        return PHUB_ERR_INVALID_INIT;
    }

    c->chunks = plan_chunks(c->n, c->ce, c->G, c->policy);
    build_ranges(c);

    for (const auto& ch : c->chunks)
        if (ch.owner == c->rank) c->owned_elems += ch.length;
    std::vector<Tile> tiles = build_tiles(c);
    c->n_tiles = tiles.size();
    c->got.assign((size_t)c->K * c->N, 0);
    c->done.assign(c->K, 0);
    c->base.assign((size_t)c->K * c->N, 0);

    DeviceGuard g(c->device);
    cudaError_t e;
    int cnt = 0;
    if ((e = cudaGetDeviceCount(&cnt)) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        why = std::string("no CUDA device: ") + cudaGetErrorString(e);
        return PHUB_ERR_CUDA;
    }
    if (c->device >= cnt) {
        delete c;
        why = "device ordinal out of range";
        return PHUB_ERR_INVALID_ARGUMENT;
    }
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device);
    {
        // every kernel loaded before any flag protocol can spin (lazy loading), once per device
        static std::mutex mu;
        static std::vector<int> loaded;
        std::lock_guard<std::mutex> lk(mu);
        if (std::find(loaded.begin(), loaded.end(), c->device) == loaded.end()) {
            if ((e = phub::preload_kernels()) != cudaSuccess) {
                cudaGetLastError();
                delete c;
                why = std::string("kernel preload: ") + cudaGetErrorString(e);
                return PHUB_ERR_CUDA;
            }
            loaded.push_back(c->device);
        }
    }
    const size_t bytes = c->E_pad * sizeof(float);
    if ((e = cudaMalloc(&c->d_w, bytes)) != cudaSuccess ||
        (e = cudaMalloc(&c->d_v, bytes)) != cudaSuccess ||
        (c->keep_agg && (e = cudaMalloc(&c->d_agg, bytes)) != cudaSuccess) ||
        (e = cudaMalloc(&c->d_base, sizeof(uintptr_t) * c->base.size())) != cudaSuccess ||
        (e = cudaMalloc(&c->d_sync, 7 * sizeof(uint32_t))) != cudaSuccess ||
        (e = cudaHostAlloc(&c->h_err, sizeof(uint32_t), cudaHostAllocMapped)) != cudaSuccess ||
        (e = cudaHostGetDevicePointer(&c->d_err, c->h_err, 0)) != cudaSuccess ||
        (c->n_tiles && (e = cudaMalloc(&c->d_tiles, sizeof(Tile) * c->n_tiles)) != cudaSuccess)) {
        cudaGetLastError();
        free_ctx(c);
        why = std::string("device arenas: ") + cudaGetErrorString(e);
        return PHUB_ERR_OUT_OF_MEMORY;
    }
    *c->h_err = 0;
    bool ok = cudaMemset(c->d_sync, 0, 7 * sizeof(uint32_t)) == cudaSuccess &&
              cudaMemset(c->d_w, 0, bytes) == cudaSuccess &&
              cudaMemset(c->d_v, 0, bytes) == cudaSuccess &&
              (!c->d_agg || cudaMemset(c->d_agg, 0, bytes) == cudaSuccess) &&
              (!c->n_tiles || cudaMemcpy(c->d_tiles, tiles.data(), sizeof(Tile) * c->n_tiles,
                                         cudaMemcpyHostToDevice) == cudaSuccess);
    if (ok && cfg->init_weights) {
        uint64_t src = 0;
        for (int k = 0; ok && k < c->K; ++k) {
            ok = cudaMemcpy(c->d_w + c->key_off[k], cfg->init_weights + src,
                            c->n[k] * sizeof(float), cudaMemcpyDefault) == cudaSuccess;
            src += c->n[k];
        }
    }
    if (!ok || (e = cudaDeviceSynchronize()) != cudaSuccess) {
        why = std::string("init copies: ") + cudaGetErrorString(cudaGetLastError());
        free_ctx(c);
        return PHUB_ERR_CUDA;
    }
    for (int vec8 = 0; vec8 < 2; ++vec8)
        for (int agg = 0; agg < 2; ++agg)
            c->flat_grid[vec8][agg] =
                c->num_sms * phub::flat_blocks_per_sm(vec8 ? 8 : 4, c->N, agg, c->cache);
    *out = c;
    return PHUB_OK;
}

phub_status phub_plan_chunks(const uint64_t* key_num_elements, int32_t num_keys,
                             uint64_t chunk_size_bytes, int32_t num_owners, int32_t owner_policy,
                             phub_chunk* out, uint64_t cap, uint64_t* count) {
    std::string& why = g_init_err;
    why.clear();
    phub_config cfg;
    phub_config_default(&cfg);
    cfg.key_num_elements = key_num_elements;
    cfg.num_keys = num_keys;
    cfg.chunk_size_bytes = chunk_size_bytes;
    cfg.num_owners = num_owners;
    cfg.owner_policy = owner_policy;
    phub_status st = validate_config(&cfg, why);
    if (st != PHUB_OK) return st;
    if (!count || (cap && !out)) return why = "count/out is NULL", PHUB_ERR_INVALID_ARGUMENT;
    const uint64_t ce = (chunk_size_bytes ? chunk_size_bytes : kDefaultChunkBytes) / 4;
    std::vector<uint64_t> n(key_num_elements, key_num_elements + num_keys);
    std::vector<phub_chunk> ch = plan_chunks(n, ce, num_owners, owner_policy);
    *count = ch.size();
    if (cap == 0) return PHUB_OK;
    if (cap < ch.size()) return why = "cap < number of chunks", PHUB_ERR_LENGTH_MISMATCH;
    std::copy(ch.begin(), ch.end(), out);
    return PHUB_OK;
}

phub_status phub_plan_ranges(const uint64_t* key_num_elements, int32_t num_keys,
                             uint64_t chunk_size_bytes, int32_t num_owners, uint64_t* E_padded,
                             uint64_t* key_offsets, uint64_t* owner_begin, uint64_t* owner_end) {
    std::string& why = g_init_err;
    why.clear();
    phub_config cfg;
    phub_config_default(&cfg);
    cfg.key_num_elements = key_num_elements;
    cfg.num_keys = num_keys;
    cfg.chunk_size_bytes = chunk_size_bytes;
    cfg.num_owners = num_owners;
    phub_status st = validate_config(&cfg, why);
    if (st != PHUB_OK) return st;
    // a host-only context: layout + table + ranges, no device state
    phub_ctx_s c;
    c.K = num_keys;
    c.G = num_owners;
    c.policy = PHUB_OWNER_CONTIG;
    c.ce = (chunk_size_bytes ? chunk_size_bytes : kDefaultChunkBytes) / 4;
    c.n.assign(key_num_elements, key_num_elements + num_keys);
    layout_keys(&c);
    c.chunks = plan_chunks(c.n, c.ce, c.G, c.policy);
    build_ranges(&c);
    if (E_padded) *E_padded = c.E_pad;
    if (key_offsets) std::copy(c.key_off.begin(), c.key_off.end(), key_offsets);
    if (owner_begin) std::copy(c.own_begin.begin(), c.own_begin.end(), owner_begin);
    if (owner_end) std::copy(c.own_end.begin(), c.own_end.end(), owner_end);
    return PHUB_OK;
}

phub_status phub_destroy(phub_ctx ctx) {
    if (!ctx) return PHUB_ERR_INVALID_ARGUMENT;
    free_ctx(ctx);
    return PHUB_OK;
}

static bool is_device_ptr(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

phub_status phub_push(phub_ctx c, int32_t worker, int32_t key, const float* grad, uint64_t n,
                      int32_t mode, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (worker < 0 || worker >= c->N)
        return c->fail(PHUB_ERR_BAD_WORKER, "worker %d not in [0,%d) (S:170)", worker, c->N);
    const bool ranged = key == PHUB_OWNED_RANGE;
    const bool all = key == PHUB_ALL_KEYS || ranged;
    if (!all && (key < 0 || key >= c->K))
        return c->fail(PHUB_ERR_BAD_KEY, "key %d not in [0,%d), PHUB_ALL_KEYS or PHUB_OWNED_RANGE",
                       key, c->K);
    if (ranged && !contig_mode(c))
        return c->fail(PHUB_ERR_UNSUPPORTED, "PHUB_OWNED_RANGE needs CONTIG ownership");
    const uint64_t rb = ranged ? c->own_begin[c->rank] : 0;
    const uint64_t want = ranged ? c->own_end[c->rank] - rb : (all ? c->E_pad : c->n[key]);
    if (n != want)
        return c->fail(PHUB_ERR_LENGTH_MISMATCH, "push length %llu != %llu (S:172)",
                       (unsigned long long)n, (unsigned long long)want);
    if (!grad && n) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "grad is NULL");
    if (mode != PHUB_COPY && mode != PHUB_BORROW)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "mode must be PHUB_COPY or PHUB_BORROW");
    const int k0 = all ? 0 : key, k1 = all ? c->K : key + 1;
    for (int k = k0; k < k1; ++k)
        if (c->got[(size_t)k * c->N + worker])
            return c->fail(PHUB_ERR_DUPLICATE_PUSH,
                           "worker %d already pushed key %d this iteration (S:176)", worker, k);
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (mode == PHUB_BORROW && n == 0) {
        // an empty owned range: nothing will be read (the owner has no chunk)
    } else if (mode == PHUB_BORROW) {
        if (!is_device_ptr(grad))
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "PHUB_BORROW needs device memory");
        if (reinterpret_cast<uintptr_t>(grad) % 16 != 0)
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "PHUB_BORROW pointer must be 16-B aligned");
        // base + 4*dev_off is the byte address of padded element dev_off
        for (int k = k0; k < k1; ++k)
            c->base[(size_t)worker * c->K + k] =
                ranged ? reinterpret_cast<uintptr_t>(grad) - 4 * rb
                : all  ? reinterpret_cast<uintptr_t>(grad)
                       : reinterpret_cast<uintptr_t>(grad) - 4 * c->key_off[k];
    } else {
        if (!c->d_recv) {
            // two slots: iteration i lands in slot i % 2, so the copies of
            // iteration i+1 may overlap the kernel of iteration i
            cudaError_t e = cudaMalloc(&c->d_recv, sizeof(float) * c->E_pad * c->N * 2);
            if (e != cudaSuccess) {
                cudaGetLastError();
                c->d_recv = nullptr;
                return c->fail(PHUB_ERR_OUT_OF_MEMORY, "receive arena: %s", cudaGetErrorString(e));
            }
            if ((e = cudaMemset(c->d_recv, 0, sizeof(float) * c->E_pad * c->N * 2)) != cudaSuccess)
                return c->cuda_fail(e, "cudaMemset(recv)");
        }
        float* slot = c->d_recv + ((c->iteration & 1) * (uint64_t)c->N + worker) * c->E_pad;
        cudaError_t e = cudaSuccess;
        if (ranged) {
            if (n) e = cudaMemcpyAsync(slot + rb, grad, n * sizeof(float), cudaMemcpyDefault, s);
        } else if (all) {
            uint64_t b = 0, eend = c->E_pad;
            if (contig_mode(c)) {
                b = c->own_begin[c->rank];
                eend = c->own_end[c->rank];
            }
            if (eend > b)
                e = cudaMemcpyAsync(slot + b, grad + b, (eend - b) * sizeof(float),
                                    cudaMemcpyDefault, s);
        } else {
            e = cudaMemcpyAsync(slot + c->key_off[key], grad, c->n[key] * sizeof(float),
                                cudaMemcpyDefault, s);
        }
        if (e != cudaSuccess) return c->cuda_fail(e, "cudaMemcpyAsync(push)");
        for (int k = k0; k < k1; ++k)
            c->base[(size_t)worker * c->K + k] = reinterpret_cast<uintptr_t>(slot);
    }
    for (int k = k0; k < k1; ++k) c->got[(size_t)k * c->N + worker] = 1;
    c->got_count += (uint64_t)(k1 - k0);
    return PHUB_OK;
}

// Chunk-tile kernel over owned tiles [t0, t1) (per-(worker,key) base table).
static cudaError_t launch_tile_range(phub_ctx c, cudaStream_t s, uint64_t t0, uint64_t t1) {
    if (t1 <= t0) return cudaSuccess;
    if (c->base != c->base_uploaded) {
        // pageable source: returns once staged, so `base` may change afterwards
        cudaError_t e = cudaMemcpyAsync(c->d_base, c->base.data(),
                                        sizeof(uintptr_t) * c->base.size(),
                                        cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return e;
        c->base_uploaded = c->base;
    }
    phub::TileArgs a{};
    a.tiles = c->d_tiles + t0;
    a.ntiles = t1 - t0;
    a.base = c->d_base;
    a.K = c->K;
    a.nw = c->N;
    a.w = c->d_w;
    a.v = c->d_v;
    a.agg = c->keep_agg ? c->d_agg : nullptr;
    a.lr = c->lr;
    a.mu = c->mu;
    a.rescale = c->rescale;
    int grid = c->grid_override ? c->grid_override : (int)std::min<uint64_t>(t1 - t0, 1u << 30);
    return phub::launch_tiles(a, std::max(grid, 1), s, &c->launches);
}

// Tiles of every key in [k0, k1) that is not yet aggregated, as maximal runs.
static cudaError_t launch_keys(phub_ctx c, cudaStream_t s, const std::vector<uint8_t>& pick) {
    cudaError_t e = cudaSuccess;
    int k = 0;
    while (k < c->K && e == cudaSuccess) {
        if (!pick[k]) { ++k; continue; }
        int k1 = k;
        uint64_t t0 = UINT64_MAX, t1 = 0;
        while (k1 < c->K && pick[k1]) {
            if (c->key_tile_end[k1] > c->key_tile_begin[k1]) {
                t0 = std::min(t0, c->key_tile_begin[k1]);
                t1 = std::max(t1, c->key_tile_end[k1]);
            }
            ++k1;
        }
        if (t1 > 0) e = launch_tile_range(c, s, t0, t1);
        k = k1;
    }
    return e;
}

// PHUB_CACHE_RESIDENT: first vector (relative to `lo`, in `vec`-element units)
// of the kept slice -- the last resident_bytes of this context's owned range
// [ob, oe) -- for a launch over [lo, hi); UINT64_MAX when the launch holds none.
static uint64_t keep_from(phub_ctx c, uint64_t ob, uint64_t oe, uint64_t lo, uint64_t hi, int vec) {
    const uint64_t keep = std::min<uint64_t>(oe - ob, c->resident_bytes / 4) / vec * vec;
    const uint64_t ks = oe - keep;                    // first kept element
    if (keep == 0 || ks >= hi) return UINT64_MAX;
    // rounded up to a whole warp of vectors: the kernel's L2 policy operand is
    // warp-uniform (it is moved into a uniform register, R2UR)
    return ks > lo ? ((ks - lo + vec - 1) / vec + 31) / 32 * 32 : 0;
}

static void end_iteration(phub_ctx c) {
    std::fill(c->got.begin(), c->got.end(), 0);
    c->got_count = 0;
    std::fill(c->done.begin(), c->done.end(), 0);
    c->done_count = 0;
    ++c->iteration;
}

phub_status phub_aggregate_ready(phub_ctx c, void* stream, uint64_t* keys_done) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (c->range_cursor != UINT64_MAX)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "iteration is being aggregated by ranges");
    if (!c->replicas.empty())
        return c->fail(PHUB_ERR_UNSUPPORTED, "streaming aggregation does not store replicas");
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<uint8_t> pick(c->K, 0);
    uint64_t n = 0;
    for (int k = 0; k < c->K; ++k) {
        if (c->done[k]) continue;
        bool all = true;
        for (int w = 0; all && w < c->N; ++w) all = c->got[(size_t)k * c->N + w] != 0;
        if (all) {
            pick[k] = 1;
            ++n;
        }
    }
    c->launches = 0;
    cudaError_t e = n ? launch_keys(c, s, pick) : cudaSuccess;
    c->launches_total += (uint64_t)c->launches;
    if (e != cudaSuccess) return c->cuda_fail(e, "kernel launch");
    for (int k = 0; k < c->K; ++k)
        if (pick[k]) c->done[k] = 1;
    c->done_count += n;
    if (keys_done) *keys_done = n;
    if (c->done_count == (uint64_t)c->K) end_iteration(c);
    return PHUB_OK;
}

static void apply_sync(phub_ctx c, phub::FlatArgs& a, const phub_sync* sync) {
    a.cta_counter = c->d_sync;
    a.timeouts = c->d_sync + 1;
    a.ticket = c->d_sync + 3;
    a.err_host = c->d_err;
    if (!sync) return;
    a.wait_flag = sync->wait_flag;
    a.wait_value = sync->wait_value;
    a.signal_flag = sync->signal_flag;
    a.signal_value = sync->signal_value;
    a.block = sync->block_elems;
}

// Flags must be 4-B aligned; blocks whole multiples of one 256-thread x 8-element pass.
static phub_status check_sync(phub_ctx c, const phub_sync* sync) {
    if (!sync) return PHUB_OK;
    if ((sync->wait_flag && reinterpret_cast<uintptr_t>(sync->wait_flag) % 4) ||
        (sync->signal_flag && reinterpret_cast<uintptr_t>(sync->signal_flag) % 4))
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "flags must be 4-B aligned");
    if (sync->block_elems % 2048)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "block_elems must be a multiple of 2048");
    return PHUB_OK;
}

// Persistent grid of a block-streaming launch: every SM x resident CTAs, at most one CTA per block.
static int blocks_grid(phub_ctx c, int nw, bool nag, uint64_t begin, uint64_t end, uint64_t B) {
    int& occ = c->blocks_occ[nag ? 1 : 0][std::min(nw, phub::kMaxWorkers)];
    if (!occ) occ = phub::blocks_per_sm(nw, nag);
    const uint64_t nblk = (end + B - 1) / B - begin / B;
    const int grid = c->grid_override ? c->grid_override : c->num_sms * occ;
    return (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)grid, nblk));
}

phub_status phub_sync_timeouts(phub_ctx c, uint32_t* count) {
    if (!c || !count) return PHUB_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    cudaError_t e = cudaMemcpy(count, c->d_sync + 1, sizeof(uint32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return c->cuda_fail(e, "cudaMemcpy(timeouts)");
    c->guard();            // the count is reported either way; a timeout also makes ctx sticky
    return PHUB_OK;
}

phub_status phub_check(phub_ctx c) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    return c->guard();
}

phub_status phub_synchronize(phub_ctx c, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    DeviceGuard g(c->device);
    cudaError_t e = stream ? cudaStreamSynchronize(static_cast<cudaStream_t>(stream))
                           : cudaDeviceSynchronize();
    if (e != cudaSuccess && !c->failed) return c->cuda_fail(e, "synchronize");
    return c->guard();
}

phub_status phub_push_batch(phub_ctx c, int32_t count, const int32_t* workers,
                            const int32_t* keys, const float* const* grads,
                            const uint64_t* lens, int32_t mode, void* stream,
                            int32_t* failed_index) {
    if (failed_index) *failed_index = -1;
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (count < 0 || (count && (!workers || !keys || !grads || !lens)))
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "batch arrays are NULL");
    // all-or-nothing: validate every entry (including duplicates inside the
    // batch) against a scratch copy of the receipts before recording anything
    std::vector<uint8_t> got = c->got;
    for (int32_t j = 0; j < count; ++j) {
        const int32_t w = workers[j], k = keys[j];
        phub_status st = PHUB_OK;
        if (w < 0 || w >= c->N) st = PHUB_ERR_BAD_WORKER;
        else if (k != PHUB_ALL_KEYS && k != PHUB_OWNED_RANGE && (k < 0 || k >= c->K))
            st = PHUB_ERR_BAD_KEY;
        else {
            const int k0 = k < 0 ? 0 : k, k1 = k < 0 ? c->K : k + 1;
            for (int kk = k0; kk < k1 && st == PHUB_OK; ++kk) {
                if (got[(size_t)kk * c->N + w]) st = PHUB_ERR_DUPLICATE_PUSH;
                got[(size_t)kk * c->N + w] = 1;
            }
        }
        if (st != PHUB_OK) {
            if (failed_index) *failed_index = j;
            return c->fail(st, "batch entry %d (worker %d, key %d) rejected", j, w, k);
        }
    }
    // lengths / pointers / modes are checked by phub_push itself; the first
    // failure there is reported, and the pushes before it are rolled back
    std::vector<uint8_t> got_before = c->got;
    const uint64_t count_before = c->got_count;
    std::vector<uintptr_t> base_before = c->base;
    for (int32_t j = 0; j < count; ++j) {
        phub_status st = phub_push(c, workers[j], keys[j], grads[j], lens[j], mode, stream);
        if (st != PHUB_OK) {
            if (c->failed) return st;
            c->got = got_before;
            c->got_count = count_before;
            c->base = base_before;
            if (failed_index) *failed_index = j;
            return st;
        }
    }
    return PHUB_OK;
}

phub_status phub_partial_sum(phub_ctx c, const float* const* srcs, int32_t count, float* dst,
                             uint64_t begin, uint64_t end, const phub_sync* sync, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (count < 1 || count > phub::kMaxWorkers || !srcs || !dst)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "need 1..%d sources and a destination",
                       phub::kMaxWorkers);
    if (end < begin || end > c->E_pad || begin % 8 || (end % 8 && end != c->E_pad))
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "range must lie in [0, E_padded), 8-aligned");
    if (reinterpret_cast<uintptr_t>(dst) % 32)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "dst must be 32-B aligned");
    phub::FlatArgs a{};
    for (int k = 0; k < count; ++k) {
        if (!srcs[k] || reinterpret_cast<uintptr_t>(srcs[k]) % 32)
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "source %d NULL or not 32-B aligned", k);
        a.g[k] = srcs[k];
    }
    a.nw = count;
    a.begin = begin;
    a.end = end;
    if (phub_status bs = check_sync(c, sync)) return bs;
    apply_sync(c, a, sync);
    DeviceGuard g(c->device);
    c->launches = 0;
    cudaError_t e;
    if (a.block) {
        e = phub::launch_blocks(a, dst, blocks_grid(c, count, false, begin, end, a.block),
                                static_cast<cudaStream_t>(stream), &c->launches);
    } else {
        const uint64_t nvec = (end - begin) / 8;
        const int grid = (int)std::max<uint64_t>(
            1, std::min<uint64_t>((uint64_t)c->flat_grid[1][0], (nvec + phub::kThreads - 1) / phub::kThreads));
        e = phub::launch_prefix(a, dst, grid, static_cast<cudaStream_t>(stream), &c->launches);
    }
    c->launches_total += (uint64_t)c->launches;
    if (e != cudaSuccess) return c->cuda_fail(e, "partial-sum launch");
    return PHUB_OK;
}

phub_status phub_aggregate_range(phub_ctx c, uint64_t begin, uint64_t end,
                                 const phub_sync* sync, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (c->got_count != (uint64_t)c->K * c->N)
        return c->fail(PHUB_ERR_INCOMPLETE, "%llu of %llu (worker,key) pushes received (S:181)",
                       (unsigned long long)c->got_count,
                       (unsigned long long)((uint64_t)c->K * c->N));
    if (!contig_mode(c) || c->done_count)
        return c->fail(PHUB_ERR_UNSUPPORTED, "range aggregation needs CONTIG ownership and no "
                       "streamed keys in this iteration");
    const uint64_t ob = c->own_begin[c->rank], oe = c->own_end[c->rank];
    const uint64_t cur = c->range_cursor == UINT64_MAX ? ob : c->range_cursor;
    const uint64_t b = std::max(begin, ob), e_ = std::min(end, oe);
    if (begin > cur || end < begin || (e_ > b && (b % 8 || (e_ % 8 && e_ != oe))))
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "ranges must abut in increasing order, 8-aligned");
    bool flat = c->ce % 8 == 0 && c->N <= phub::kMaxWorkers;
    for (int w = 0; flat && w < c->N; ++w) {
        const uintptr_t b0 = c->base[(size_t)w * c->K];
        for (int k = 1; k < c->K && flat; ++k) flat = c->base[(size_t)w * c->K + k] == b0;
        flat = flat && b0 % 32 == 0;
    }
    if (!flat)
        return c->fail(PHUB_ERR_UNSUPPORTED, "range aggregation needs whole-model / owned-range "
                       "pushes, 32-B aligned");
    if (phub_status bs = check_sync(c, sync)) return bs;
    DeviceGuard g(c->device);
    c->launches = 0;
    cudaError_t e = cudaSuccess;
    const uint64_t lo = std::max(b, cur);
    if (e_ > lo || (sync && sync->signal_flag)) {
        phub::FlatArgs a{};
        apply_sync(c, a, sync);
        for (int w = 0; w < c->N; ++w) a.g[w] = reinterpret_cast<const float*>(c->base[(size_t)w * c->K]);
        a.w = c->d_w;
        a.v = c->d_v;
        a.agg = c->keep_agg ? c->d_agg : nullptr;
        a.begin = lo;
        a.end = e_;
        a.lr = c->lr;
        a.mu = c->mu;
        a.rescale = c->rescale;
        a.nw = c->N;
        a.nrep = (int)c->replicas.size();
        for (int r = 0; r < a.nrep; ++r) a.rep[r] = c->replicas[r];
        const uint64_t nvec = (e_ - lo) / 8;
        const uint64_t cover = (nvec + phub::kThreads - 1) / phub::kThreads;
        if (a.block) {
            e = e_ > lo ? phub::launch_blocks(a, nullptr, blocks_grid(c, c->N, true, lo, e_, a.block),
                                              static_cast<cudaStream_t>(stream), &c->launches)
                        : cudaSuccess;
        } else {
            int grid = c->grid_override ? c->grid_override
                       : (c->flat_oneshot > 0 || (c->flat_oneshot < 0 && c->replicas.empty()))
                             ? (int)std::min<uint64_t>(cover, 0x7fffffffULL)
                             : c->flat_grid[1][c->keep_agg];
            grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(grid, cover));
            a.keep_from = keep_from(c, ob, oe, lo, e_, 8);
            e = phub::launch_flat(a, 8, c->cache, grid, static_cast<cudaStream_t>(stream),
                                  &c->launches);
        }
    }
    c->launches_total += (uint64_t)c->launches;
    if (e != cudaSuccess) return c->cuda_fail(e, "kernel launch");
    c->range_cursor = std::max(cur, std::min(std::max(end, cur), oe));
    if (c->range_cursor >= oe) {
        c->range_cursor = UINT64_MAX;
        end_iteration(c);
    }
    return PHUB_OK;
}

phub_status phub_aggregate_optimize(phub_ctx c, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (c->got_count != (uint64_t)c->K * c->N)
        return c->fail(PHUB_ERR_INCOMPLETE, "%llu of %llu (worker,key) pushes received (S:181)",
                       (unsigned long long)c->got_count,
                       (unsigned long long)((uint64_t)c->K * c->N));
    DeviceGuard g(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);

    // Flat eligibility: contiguous ownership and every worker's keys share one base.
    bool flat = contig_mode(c) && c->N <= phub::kMaxWorkers && c->ce % 4 == 0;
    bool align32 = c->ce % 8 == 0;
    for (int w = 0; flat && w < c->N; ++w) {
        const uintptr_t b0 = c->base[(size_t)w * c->K];
        for (int k = 1; k < c->K; ++k)
            if (c->base[(size_t)w * c->K + k] != b0) {
                flat = false;
                break;
            }
        align32 &= b0 % 32 == 0;
    }
    int variant = c->kernel;
    if (variant == PHUB_KERNEL_AUTO)
        variant = !flat ? PHUB_KERNEL_TILES : (align32 ? PHUB_KERNEL_FLAT : PHUB_KERNEL_FLAT128);
    if (variant == PHUB_KERNEL_BULK && !(flat && align32 && c->N <= 8))
        return c->fail(PHUB_ERR_UNSUPPORTED, "bulk kernel needs whole-model pushes, contiguous "
                       "ownership, 32-B aligned chunks and N <= 8");
    if ((variant == PHUB_KERNEL_FLAT && !(flat && align32)) ||
        ((variant == PHUB_KERNEL_FLAT128 || variant == PHUB_KERNEL_WIDE) && !flat))
        return c->fail(PHUB_ERR_UNSUPPORTED, "forced kernel variant %d needs whole-model pushes, "
                       "contiguous ownership and aligned chunks", variant);
    if (!c->replicas.empty() && variant != PHUB_KERNEL_FLAT && variant != PHUB_KERNEL_FLAT128 &&
        variant != PHUB_KERNEL_BULK)
        return c->fail(PHUB_ERR_UNSUPPORTED, "replica stores need the flat kernel (whole-model "
                       "or owned-range pushes under CONTIG ownership)");
    if (variant == PHUB_KERNEL_WIDE && !c->keep_agg)
        return c->fail(PHUB_ERR_UNSUPPORTED, "wide ablation needs keep_aggregate (merge buffer)");

    cudaError_t e = cudaSuccess;
    c->launches = 0;
    if (c->done_count > 0) {
        // part of the iteration was already aggregated by phub_aggregate_ready
        if (!c->replicas.empty())
            return c->fail(PHUB_ERR_UNSUPPORTED, "streaming aggregation does not store replicas");
        std::vector<uint8_t> pick(c->K, 0);
        for (int k = 0; k < c->K; ++k) pick[k] = !c->done[k];
        e = launch_keys(c, s, pick);
        c->launches_total += (uint64_t)c->launches;
        if (e != cudaSuccess) return c->cuda_fail(e, "kernel launch");
        end_iteration(c);
        return PHUB_OK;
    }
    const uint64_t b = contig_mode(c) ? c->own_begin[c->rank] : 0;
    const uint64_t eend = contig_mode(c) ? c->own_end[c->rank] : 0;
    if (c->range_cursor != UINT64_MAX)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "iteration is being aggregated by ranges");
    if (variant == PHUB_KERNEL_FLAT || variant == PHUB_KERNEL_FLAT128 ||
        variant == PHUB_KERNEL_BULK) {
        phub::FlatArgs a{};
        for (int w = 0; w < c->N; ++w) a.g[w] = reinterpret_cast<const float*>(c->base[(size_t)w * c->K]);
        a.w = c->d_w;
        a.v = c->d_v;
        a.agg = c->keep_agg ? c->d_agg : nullptr;
        a.begin = b;
        a.end = eend;
        a.lr = c->lr;
        a.mu = c->mu;
        a.rescale = c->rescale;
        a.nw = c->N;
        a.nrep = (int)c->replicas.size();
        for (int r = 0; r < a.nrep; ++r) a.rep[r] = c->replicas[r];
        a.err_host = c->d_err;
        const int vec = variant == PHUB_KERNEL_FLAT ? 8 : 4;
        const uint64_t nvec = (eend - b) / vec;
        const uint64_t cover = (nvec + phub::kThreads - 1) / phub::kThreads;
        int grid = c->grid_override ? c->grid_override
                   : (c->flat_oneshot > 0 || (c->flat_oneshot < 0 && c->replicas.empty()))
                         ? (int)std::min<uint64_t>(cover, 0x7fffffffULL)
                                     : c->flat_grid[vec == 8][c->keep_agg];
        grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(grid, cover));
        a.keep_from = keep_from(c, b, eend, b, eend, vec);
        if (variant == PHUB_KERNEL_BULK)
            e = phub::launch_bulk(a, c->grid_override ? c->grid_override : c->num_sms, s,
                                  &c->launches);
        else
            e = phub::launch_flat(a, vec, c->cache, grid, s, &c->launches);
    } else if (variant == PHUB_KERNEL_WIDE) {
        phub::WideArgs a{};
        for (int w = 0; w < c->N; ++w) a.g[w] = reinterpret_cast<const float*>(c->base[(size_t)w * c->K]);
        a.w = c->d_w;
        a.v = c->d_v;
        a.agg = c->d_agg;
        a.begin = b;
        a.end = eend;
        a.lr = c->lr;
        a.mu = c->mu;
        a.rescale = c->rescale;
        a.nw = c->N;
        int grid = c->grid_override ? c->grid_override : c->num_sms * 8;
        e = phub::launch_wide(a, grid, s, &c->launches);
    } else {
        e = launch_tile_range(c, s, 0, c->n_tiles);
    }
    c->launches_total += (uint64_t)c->launches;
    if (e != cudaSuccess) return c->cuda_fail(e, "kernel launch");
    end_iteration(c);
    return PHUB_OK;
}

phub_status phub_pull(phub_ctx c, int32_t key, float* dst, uint64_t n, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    const bool all = key == PHUB_ALL_KEYS;
    if (!all && (key < 0 || key >= c->K))
        return c->fail(PHUB_ERR_BAD_KEY, "key %d not in [0,%d) and not PHUB_ALL_KEYS", key, c->K);
    const uint64_t want = all ? c->E_pad : c->n[key];
    if (n != want)
        return c->fail(PHUB_ERR_LENGTH_MISMATCH, "pull length %llu != %llu",
                       (unsigned long long)n, (unsigned long long)want);
    if (!dst) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "dst is NULL");
    DeviceGuard g(c->device);
    cudaError_t e = cudaMemcpyAsync(dst, c->d_w + (all ? 0 : c->key_off[key]), n * sizeof(float),
                                    cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return c->cuda_fail(e, "cudaMemcpyAsync(pull)");
    return PHUB_OK;
}

phub_status phub_pushpull(phub_ctx c, int32_t worker, const float* grad, uint64_t n,
                          int32_t mode, float* dst, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    phub_status st = phub_push(c, worker, PHUB_ALL_KEYS, grad, n, mode, stream);
    if (st != PHUB_OK) return st;
    if (c->got_count != (uint64_t)c->K * c->N) return PHUB_OK;
    st = phub_aggregate_optimize(c, stream);
    if (st != PHUB_OK || !dst) return st;
    return phub_pull(c, PHUB_ALL_KEYS, dst, c->E_pad, stream);
}

phub_status phub_weights(phub_ctx c, float** w_dev) {
    if (!c || !w_dev) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    *w_dev = c->d_w;
    return PHUB_OK;
}

phub_status phub_layout(phub_ctx c, uint64_t* E, uint64_t* E_padded, uint64_t* key_offsets) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (E) *E = c->E;
    if (E_padded) *E_padded = c->E_pad;
    if (key_offsets) std::copy(c->key_off.begin(), c->key_off.end(), key_offsets);
    return PHUB_OK;
}

phub_status phub_num_chunks(phub_ctx c, uint64_t* n) {
    if (!c || !n) return PHUB_ERR_INVALID_ARGUMENT;
    *n = c->chunks.size();
    return PHUB_OK;
}

phub_status phub_chunk_table(phub_ctx c, phub_chunk* out, uint64_t cap) {
    if (!c || !out) return PHUB_ERR_INVALID_ARGUMENT;
    if (cap < c->chunks.size())
        return c->fail(PHUB_ERR_LENGTH_MISMATCH, "capacity %llu < %zu chunks",
                       (unsigned long long)cap, c->chunks.size());
    std::copy(c->chunks.begin(), c->chunks.end(), out);
    return PHUB_OK;
}

phub_status phub_owner_range(phub_ctx c, int32_t owner, uint64_t* begin, uint64_t* end) {
    if (!c || !begin || !end) return PHUB_ERR_INVALID_ARGUMENT;
    if (owner < 0 || owner >= c->G) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "bad owner %d", owner);
    if (!contig_mode(c))
        return c->fail(PHUB_ERR_UNSUPPORTED, "owner ranges exist only under CONTIG ownership");
    *begin = c->own_begin[owner];
    *end = c->own_end[owner];
    return PHUB_OK;
}

phub_status phub_owned_elements(phub_ctx c, uint64_t* n) {
    if (!c || !n) return PHUB_ERR_INVALID_ARGUMENT;
    *n = c->owned_elems;
    return PHUB_OK;
}

static phub_status scatter_keys(phub_ctx c, float* dst_dev, const float* src) {
    uint64_t s = 0;
    for (int k = 0; k < c->K; ++k) {
        cudaError_t e = cudaMemcpy(dst_dev + c->key_off[k], src + s, c->n[k] * sizeof(float),
                                   cudaMemcpyDefault);
        if (e != cudaSuccess) return c->cuda_fail(e, "cudaMemcpy(load_state)");
        s += c->n[k];
    }
    return PHUB_OK;
}

static phub_status gather_keys(phub_ctx c, float* dst, const float* src_dev) {
    uint64_t s = 0;
    for (int k = 0; k < c->K; ++k) {
        cudaError_t e = cudaMemcpy(dst + s, src_dev + c->key_off[k], c->n[k] * sizeof(float),
                                   cudaMemcpyDefault);
        if (e != cudaSuccess) return c->cuda_fail(e, "cudaMemcpy(read_state)");
        s += c->n[k];
    }
    return PHUB_OK;
}

phub_status phub_load_state(phub_ctx c, const float* w, const float* v) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return c->cuda_fail(e, "cudaDeviceSynchronize");
    if (phub_status st1 = c->guard()) return st1;      // a wait expired in the launches waited for
    phub_status st = PHUB_OK;
    if (w && (st = scatter_keys(c, c->d_w, w)) != PHUB_OK) return st;
    if (v && (st = scatter_keys(c, c->d_v, v)) != PHUB_OK) return st;
    return PHUB_OK;
}

phub_status phub_read_state(phub_ctx c, float* w, float* v, float* agg) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (agg && !c->keep_agg)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "agg requested but keep_aggregate is off");
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return c->cuda_fail(e, "cudaDeviceSynchronize");
    if (phub_status st1 = c->guard()) return st1;      // never return a partly skipped round
    phub_status st = PHUB_OK;
    if (w && (st = gather_keys(c, w, c->d_w)) != PHUB_OK) return st;
    if (v && (st = gather_keys(c, v, c->d_v)) != PHUB_OK) return st;
    if (agg && (st = gather_keys(c, agg, c->d_agg)) != PHUB_OK) return st;
    return PHUB_OK;
}

phub_status phub_iteration(phub_ctx c, uint64_t* it) {
    if (!c || !it) return PHUB_ERR_INVALID_ARGUMENT;
    *it = c->iteration;
    return PHUB_OK;
}

phub_status phub_kernel_launches(phub_ctx c, uint64_t* n) {
    if (!c || !n) return PHUB_ERR_INVALID_ARGUMENT;
    *n = c->launches_total;
    return PHUB_OK;
}

phub_status phub_set_replicas(phub_ctx c, float* const* replicas, int32_t count) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (count < 0 || count > phub::kMaxReplicas || (count && !replicas))
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "replica count must be in [0,%d]",
                       phub::kMaxReplicas);
    for (int r = 0; r < count; ++r) {
        if (!replicas[r] || reinterpret_cast<uintptr_t>(replicas[r]) % 32 != 0)
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "replica %d is NULL or not 32-B aligned", r);
        DeviceGuard g(c->device);
        if (!is_device_ptr(replicas[r]))
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "replica %d is not device memory", r);
    }
    if (count && !contig_mode(c))
        return c->fail(PHUB_ERR_UNSUPPORTED, "replicas need CONTIG ownership");
    c->replicas.assign(replicas, replicas + count);
    return PHUB_OK;
}

phub_status phub_hier_exchange(phub_ctx c, const phub_hier* h, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (!h || h->num_racks != c->G || h->num_racks > phub::kMaxRacks)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "num_racks must equal the context's owners (<= %d)",
                       phub::kMaxRacks);
    if (!contig_mode(c) || c->ce % 8 || c->N > phub::kMaxWorkers)
        return c->fail(PHUB_ERR_UNSUPPORTED, "hierarchical exchange needs CONTIG ownership, "
                       "chunks of a multiple of 32 B and <= %d local workers", phub::kMaxWorkers);
    if (!h->block_elems || h->block_elems % 2048)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "block_elems must be a positive multiple of 2048");
    if (h->epoch == 0) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "epoch must be >= 1");
    const int R = h->num_racks, me = c->rank;
    if (R > 1 && (!h->inbox || !h->peer_inbox || !h->flags || !h->peer_flags))
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "inbox / flag pointers required for > 1 rack");
    for (int q = 0; R > 1 && q < R; ++q) {
        if (q == me) continue;
        if (!h->inbox[q] || !h->peer_inbox[q] || !h->peer_flags[q])
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "rack %d: inbox / peer pointers missing", q);
        // 256-bit accesses at padded offsets that are multiples of 8 elements
        if (reinterpret_cast<uintptr_t>(h->inbox[q]) % 32 ||
            reinterpret_cast<uintptr_t>(h->peer_inbox[q]) % 32 ||
            reinterpret_cast<uintptr_t>(h->peer_flags[q]) % 4)
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "rack %d: inbox pointers must be 32-B "
                           "aligned, flags 4-B aligned", q);
    }
    if (R > 1 && reinterpret_cast<uintptr_t>(h->flags) % 4)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "flags must be 4-B aligned");
    if (c->got_count != (uint64_t)c->K * c->N)
        return c->fail(PHUB_ERR_INCOMPLETE, "%llu of %llu (worker,key) pushes received (S:181)",
                       (unsigned long long)c->got_count,
                       (unsigned long long)((uint64_t)c->K * c->N));
    if (c->range_cursor != UINT64_MAX || c->done_count)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "iteration is being aggregated otherwise");
    phub::HierArgs a{};
    for (int w = 0; w < c->N; ++w) {
        const uintptr_t b0 = c->base[(size_t)w * c->K];
        for (int k = 1; k < c->K; ++k)
            if (c->base[(size_t)w * c->K + k] != b0 || b0 % 32)
                return c->fail(PHUB_ERR_UNSUPPORTED, "worker %d: whole-model 32-B aligned push "
                               "required", w);
        a.g[w] = reinterpret_cast<const float*>(b0);
    }
    a.nw = c->N;
    a.R = R;
    a.rack = me;
    a.w = c->d_w;
    a.v = c->d_v;
    a.agg = c->keep_agg ? c->d_agg : nullptr;
    a.lr = c->lr;
    a.mu = c->mu;
    a.rescale = c->rescale;
    a.nrep = (int)c->replicas.size();
    for (int r = 0; r < a.nrep; ++r) a.rep[r] = c->replicas[r];
    for (int o = 0; o < R; ++o) {
        a.own_begin[o] = c->own_begin[o];
        a.own_end[o] = c->own_end[o];
        if (o != me && R > 1) {
            a.inbox[o] = h->inbox[o];
            a.peer_inbox[o] = h->peer_inbox[o];
            a.peer_flags[o] = h->peer_flags[o];
        }
    }
    a.block = h->block_elems;
    a.flags = R > 1 ? h->flags : nullptr;
    a.epoch = h->epoch;
    a.worker_order = h->worker_order ? 1 : 0;
    a.device_barrier = h->device_barrier ? 1 : 0;
    if (a.device_barrier && R < 2) a.device_barrier = 0;   // one rack: nothing to order
    a.ticket = c->d_sync + 3;
    a.timeouts = c->d_sync + 1;
    a.err_host = c->d_err;
    DeviceGuard g(c->device);
    c->launches = 0;
    int& occ = c->hier_occ[a.worker_order];
    if (!occ) occ = phub::hier_blocks_per_sm(c->N, a.worker_order != 0);
    const int grid = c->grid_override ? c->grid_override : c->num_sms * occ;
    cudaError_t e = phub::launch_hier(a, grid, static_cast<cudaStream_t>(stream), &c->launches);
    c->launches_total += (uint64_t)c->launches;
    if (e != cudaSuccess) return c->cuda_fail(e, "hierarchical exchange launch");
    end_iteration(c);
    return PHUB_OK;
}

// ------------------------------------------- scheduled exchange (DESIGN 8.6)
static_assert(sizeof(phub_sched_item) == sizeof(phub::SchedItem), "item layout");
static_assert(offsetof(phub_sched_item, type) == offsetof(phub::SchedItem, type), "item layout");
static_assert(offsetof(phub_sched_item, signal_flag) == offsetof(phub::SchedItem, signal_flag),
              "item layout");

phub_status phub_sched_plan(int32_t ranks, int32_t rank, int32_t workers_per_rank,
                            const uint64_t* bounds, const uint64_t* split, uint64_t block_elems,
                            uint64_t lag_blocks, uint64_t taper_blocks, phub_sched_item* out,
                            uint64_t cap, uint64_t* count, uint32_t* num_flags) {
    const int G = ranks, p = rank, W = workers_per_rank;
    if (G < 1 || G > phub::kMaxRacks || p < 0 || p >= G || W < 1 || W > phub::kMaxWorkers ||
        !bounds || !split || !count || !block_elems || block_elems % 2048 || (cap && !out))
        return PHUB_ERR_INVALID_ARGUMENT;
    if (bounds[0] != 0) return PHUB_ERR_INVALID_ARGUMENT;
    for (int o = 0; o < G; ++o)
        if (bounds[o + 1] < bounds[o] || bounds[o] % 8 || bounds[o + 1] % 8 || split[o] % 8 ||
            split[o] < bounds[o] || split[o] > bounds[o + 1])
            return PHUB_ERR_INVALID_ARGUMENT;
    struct Blk { int o; uint64_t lo, hi; uint64_t j, J; };
    // Cut a part [b, e) into blocks: block_elems each, except its first and last
    // taper_blocks * block_elems elements, cut 4x finer (multiples of 8) so the
    // pipeline fills and drains in smaller steps.
    const uint64_t fine = std::max<uint64_t>(256, block_elems / 4 / 8 * 8);
    auto cut = [&](int o, uint64_t b, uint64_t e, std::vector<Blk>& outv) {
        const uint64_t L = e - b, span = taper_blocks * block_elems;
        const uint64_t head = std::min(span, L / 2 / 8 * 8);
        const uint64_t tail = std::min(span, (L - head) / 8 * 8);
        std::vector<std::pair<uint64_t, uint64_t>> r;
        for (uint64_t x = b; x < b + head; x += fine) r.push_back({x, std::min(x + fine, b + head)});
        for (uint64_t x = b + head; x < e - tail; x += block_elems)
            r.push_back({x, std::min(x + block_elems, e - tail)});
        for (uint64_t x = e - tail; x < e; x += fine) r.push_back({x, std::min(x + fine, e)});
        for (size_t j = 0; j < r.size(); ++j) outv.push_back({o, r[j].first, r[j].second, j, r.size()});
    };
    std::vector<Blk> chain, raw;
    for (int o = 0; o < G; ++o) cut(o, split[o], bounds[o + 1], chain);   // chain parts, owner-major
    for (int o = 0; o < G; ++o) cut(o, bounds[o], split[o], raw);         // raw parts, owner-major
    const uint64_t C = chain.size(), R = raw.size();
    // + 2G round-barrier flags at the end (phub_sched.device_barrier):
    //   [2C + RG + q]     rank q's replica is free for this epoch (its kernel started)
    //   [2C + RG + G + q] rank q finished storing into this rank's replica
    const uint64_t nflags = 2 * C + R * (uint64_t)G + 2 * (uint64_t)G;
    if (nflags >= 0xffffffffull) return PHUB_ERR_INVALID_ARGUMENT;
    // (progress key, stage, item): progress = fraction of the block's own part
    // done before it, plus stage * lag; the same doubles on every rank.  Every
    // part -- each owner's RAW part and each owner's CHAIN part -- advances at
    // the same relative pace, so at any moment each rank mixes all its kinds of
    // work (e.g. the last rank's Nesterov + replica stores for its own chain
    // part are spread over the round instead of trailing the other owners').
    struct Keyed { double t; int stage; phub_sched_item it; };
    std::vector<Keyed> v;
    const double lag_c = C ? (double)lag_blocks / (double)C : 0.0;
    for (uint64_t c = 0; c < C; ++c) {
        const Blk& b = chain[c];
        const double t = (double)b.j / (double)b.J;
        phub_sched_item it{};
        it.lo = b.lo;
        it.hi = b.hi;
        it.type = PHUB_ITEM_CHAIN;
        it.wait_flag = p > 0 ? (uint32_t)c : phub::kNoFlag;
        if (p < G - 1) {
            it.dst = p + 1;                           // partial into the next rank's inbox
            it.signal_flag = (uint32_t)c;
        } else if (b.o == G - 1) {
            it.dst = -1;                              // sum complete here: Nesterov
            it.signal_flag = phub::kNoFlag;
        } else {
            it.dst = b.o;                             // s into the owner's inbox
            it.signal_flag = (uint32_t)(C + c);
        }
        v.push_back({t + p * lag_c, p, it});
        if (p == b.o && b.o != G - 1) {
            phub_sched_item f{};
            f.lo = b.lo;
            f.hi = b.hi;
            f.type = PHUB_ITEM_CONSUME_FINAL;
            f.dst = -1;
            f.wait_flag = (uint32_t)(C + c);
            f.signal_flag = phub::kNoFlag;
            v.push_back({t + G * lag_c, G, f});
        }
    }
    for (uint64_t jg = 0; jg < R; ++jg) {
        const Blk& b = raw[jg];
        const double t = (double)b.j / (double)b.J;
        phub_sched_item it{};
        it.lo = b.lo;
        it.hi = b.hi;
        it.base = bounds[b.o];
        it.len = split[b.o] - bounds[b.o];
        if (p != b.o) {
            it.type = PHUB_ITEM_RAW_PUSH;
            it.dst = b.o;
            it.wait_flag = phub::kNoFlag;
            it.signal_flag = (uint32_t)(2 * C + jg * G + p);
            v.push_back({t, 0, it});
        } else {
            it.type = PHUB_ITEM_CONSUME_RAW;
            it.dst = -1;
            it.wait_flag = (uint32_t)(2 * C + jg * G);
            it.signal_flag = phub::kNoFlag;
            v.push_back({t + (double)lag_blocks / (double)b.J, 1, it});
        }
    }
    std::stable_sort(v.begin(), v.end(), [](const Keyed& a, const Keyed& b) {
        return a.t < b.t || (a.t == b.t && a.stage < b.stage);
    });
    *count = v.size();
    if (num_flags) *num_flags = (uint32_t)nflags;
    if (cap == 0) return PHUB_OK;
    if (cap < v.size()) return PHUB_ERR_LENGTH_MISMATCH;
    for (size_t i = 0; i < v.size(); ++i) out[i] = v[i].it;
    return PHUB_OK;
}

phub_status phub_sched_load(phub_ctx c, int32_t ranks, int32_t rank, const phub_sched_item* items,
                            uint64_t count, uint32_t num_flags) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (ranks < 1 || ranks > phub::kMaxRacks || rank < 0 || rank >= ranks || (count && !items))
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "bad ranks / rank / items");
    for (uint64_t t = 0; t < count; ++t) {
        const phub_sched_item& it = items[t];
        const bool raw = it.type == PHUB_ITEM_RAW_PUSH || it.type == PHUB_ITEM_CONSUME_RAW;
        bool ok = it.type >= PHUB_ITEM_RAW_PUSH && it.type <= PHUB_ITEM_CONSUME_FINAL &&
                  it.lo % 8 == 0 && it.hi % 8 == 0 && it.lo < it.hi && it.hi <= c->E_pad &&
                  it.dst >= -1 && it.dst < ranks;
        if (raw) ok = ok && it.base % 8 == 0 && it.lo >= it.base && it.hi <= it.base + it.len;
        if (it.type == PHUB_ITEM_RAW_PUSH)
            ok = ok && it.dst >= 0 && it.dst != rank && it.signal_flag < num_flags;
        if (it.type == PHUB_ITEM_CHAIN)
            ok = ok && (it.wait_flag == phub::kNoFlag || it.wait_flag < num_flags) &&
                 (it.dst < 0 || (it.dst != rank && it.signal_flag < num_flags));
        if (it.type == PHUB_ITEM_CONSUME_RAW)
            ok = ok && it.dst == -1 && (uint64_t)it.wait_flag + ranks <= num_flags;
        if (it.type == PHUB_ITEM_CONSUME_FINAL) ok = ok && it.dst == -1 && it.wait_flag < num_flags;
        if (!ok)
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "item %llu: invalid (type %u, [%llu, %llu), "
                           "dst %d)", (unsigned long long)t, it.type, (unsigned long long)it.lo,
                           (unsigned long long)it.hi, it.dst);
    }
    // two lanes, each in ticket (key) order: producers (RAW_PUSH, CHAIN) first,
    // then consumers (CONSUME_RAW, CONSUME_FINAL) -- see k_sched.  A program
    // without CHAIN items (the push plan) keeps ONE lane in key order: its
    // producers never wait, so a waiting consumer cannot hold up anything a
    // CTA taking the next ticket would not reach anyway (k_hier's scheme), and
    // the CTAs balance between pushes and consumers dynamically.
    bool chain = false;
    for (uint64_t t = 0; t < count; ++t) chain |= items[t].type == PHUB_ITEM_CHAIN;
    std::vector<phub_sched_item> lanes;
    lanes.reserve(count);
    uint64_t prod_elems = 0, cons_elems = 0;
    for (int pass = 0; pass < (chain ? 2 : 1); ++pass)
        for (uint64_t t = 0; t < count; ++t) {
            const bool cons = items[t].type == PHUB_ITEM_CONSUME_RAW ||
                              items[t].type == PHUB_ITEM_CONSUME_FINAL;
            if (chain && cons != (pass == 1)) continue;
            lanes.push_back(items[t]);
            (cons ? cons_elems : prod_elems) += items[t].hi - items[t].lo;
        }
    uint64_t n_prod = count;
    if (chain) {
        n_prod = 0;
        while (n_prod < count && lanes[n_prod].type != PHUB_ITEM_CONSUME_RAW &&
               lanes[n_prod].type != PHUB_ITEM_CONSUME_FINAL)
            ++n_prod;
    }
    DeviceGuard g(c->device);
    phub::SchedItem* d = nullptr;
    if (count) {
        cudaError_t e = cudaMalloc(&d, count * sizeof(phub::SchedItem));
        if (e == cudaSuccess) e = cudaMemcpy(d, lanes.data(), count * sizeof(phub::SchedItem),
                                             cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(d);
            return c->cuda_fail(e, "sched item upload");
        }
    }
    cudaFree(c->d_items);
    c->d_items = d;
    c->n_items = count;
    c->n_prod = n_prod;
    c->cons_frac = (prod_elems + cons_elems) ? (double)cons_elems / (double)(prod_elems + cons_elems)
                                             : 0.0;
    c->sched_ranks = ranks;
    c->sched_rank = rank;
    c->sched_flags = num_flags;
    return PHUB_OK;
}

phub_status phub_sched_exchange(phub_ctx c, const phub_sched* s, void* stream) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    if (phub_status st0 = c->guard()) return st0;
    if (!s || s->epoch == 0) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "epoch must be >= 1");
    if (c->sched_rank < 0) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "no item program loaded");
    if (c->G != 1 || c->N > phub::kMaxWorkers || c->ce % 8)
        return c->fail(PHUB_ERR_UNSUPPORTED, "scheduled exchange needs num_owners == 1, chunks of "
                       "a multiple of 32 B and <= %d local workers", phub::kMaxWorkers);
    const int R = c->sched_ranks, me = c->sched_rank;
    if (!s->inbox || !s->raw_inbox || !s->flags)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "inbox / raw_inbox / flags arrays required");
    for (int q = 0; q < R; ++q)
        if (reinterpret_cast<uintptr_t>(s->inbox[q]) % 32 ||
            reinterpret_cast<uintptr_t>(s->raw_inbox[q]) % 32 ||
            reinterpret_cast<uintptr_t>(s->flags[q]) % 4 || (R > 1 && !s->flags[q]))
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "rank %d: inboxes must be 32-B aligned, "
                           "flags 4-B aligned and non-null", q);
    if (c->got_count != (uint64_t)c->K * c->N)
        return c->fail(PHUB_ERR_INCOMPLETE, "%llu of %llu (worker,key) pushes received (S:181)",
                       (unsigned long long)c->got_count,
                       (unsigned long long)((uint64_t)c->K * c->N));
    if (c->range_cursor != UINT64_MAX || c->done_count)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "iteration is being aggregated otherwise");
    phub::SchedArgs a{};
    for (int w = 0; w < c->N; ++w) {
        const uintptr_t b0 = c->base[(size_t)w * c->K];
        for (int k = 1; k < c->K; ++k)
            if (c->base[(size_t)w * c->K + k] != b0 || b0 % 32)
                return c->fail(PHUB_ERR_UNSUPPORTED, "worker %d: whole-model 32-B aligned push "
                               "required", w);
        a.g[w] = reinterpret_cast<const float*>(b0);
    }
    a.nw = c->N;
    a.R = R;
    a.rank = me;
    a.w = c->d_w;
    a.v = c->d_v;
    a.agg = c->keep_agg ? c->d_agg : nullptr;
    a.lr = c->lr;
    a.mu = c->mu;
    a.rescale = c->rescale;
    a.nrep = (int)c->replicas.size();
    for (int r = 0; r < a.nrep; ++r) a.rep[r] = c->replicas[r];
    a.items = c->d_items;
    a.nitems = c->n_items;
    a.nprod = c->n_prod;
    a.trace = c->sched_trace;
    for (int q = 0; q < R; ++q) {
        a.inbox[q] = s->inbox[q];
        a.raw_inbox[q] = s->raw_inbox[q];
        a.flags[q] = s->flags[q];
    }
    a.epoch = s->epoch;
    a.ticket = c->d_sync + 3;
    a.timeouts = c->d_sync + 1;
    a.err_host = c->d_err;
    if (s->device_barrier) {
        if (c->sched_flags < 2u * (uint32_t)R)
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "device_barrier needs the program's 2 x ranks "
                           "barrier flags (plans from phub_sched_plan carry them)");
        a.bar = (int64_t)c->sched_flags - 2 * R;
    } else {
        a.bar = -1;
    }
    DeviceGuard g(c->device);
    c->launches = 0;
    if (!c->sched_occ) c->sched_occ = phub::sched_blocks_per_sm(c->N);
    const int grid = c->grid_override ? c->grid_override : c->num_sms * c->sched_occ;
    // CTAs [0, grid_prod) take producer items, the rest consumer items: a CTA
    // blocked on a consumer's wait never holds up the chain it waits for
    const bool has_p = c->n_prod > 0, has_c = c->n_items > c->n_prod;
    int cons_ctas = s->consumer_ctas > 0 ? s->consumer_ctas
                                         : (int)std::lround(grid * std::min(0.5, std::max(0.125,
                                                                              c->cons_frac)));
    if (!has_c) cons_ctas = 0;
    else if (!has_p) cons_ctas = grid;
    cons_ctas = std::min(std::max(cons_ctas, has_c ? 1 : 0), grid - (has_p ? 1 : 0));
    if (has_p && has_c && grid < 2)
        return c->fail(PHUB_ERR_INVALID_ARGUMENT, "two item lanes need a grid of >= 2 CTAs");
    a.grid_prod = grid - cons_ctas;
    cudaError_t e = phub::launch_sched(a, grid, static_cast<cudaStream_t>(stream), &c->launches);
    c->launches_total += (uint64_t)c->launches;
    if (e != cudaSuccess) return c->cuda_fail(e, "scheduled exchange launch");
    end_iteration(c);
    return PHUB_OK;
}

phub_status phub_alloc_shared(int32_t device, uint64_t bytes, void** dev_ptr) {
    if (!dev_ptr || device < 0) return PHUB_ERR_INVALID_ARGUMENT;
    DeviceGuard g(device);
    cudaError_t e = cudaMalloc(dev_ptr, bytes ? bytes : 1);
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_init_err = cudaGetErrorString(e);
        *dev_ptr = nullptr;
        return PHUB_ERR_OUT_OF_MEMORY;
    }
    return PHUB_OK;
}

phub_status phub_free_shared(int32_t device, void* dev_ptr) {
    if (device < 0) return PHUB_ERR_INVALID_ARGUMENT;
    DeviceGuard g(device);
    cudaError_t e = cudaFree(dev_ptr);
    if (e != cudaSuccess) {
        g_init_err = cudaGetErrorString(e);
        return PHUB_ERR_CUDA;
    }
    return PHUB_OK;
}

phub_status phub_ipc_get_handle(int32_t device, const void* dev_ptr, void* handle64) {
    if (!dev_ptr || !handle64 || device < 0) return PHUB_ERR_INVALID_ARGUMENT;
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_init_err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
        return PHUB_ERR_CUDA;
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, sizeof h);
    return PHUB_OK;
}

phub_status phub_ipc_open(int32_t device, const void* handle64, void** dev_ptr) {
    if (!handle64 || !dev_ptr || device < 0) return PHUB_ERR_INVALID_ARGUMENT;
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_init_err = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
        *dev_ptr = nullptr;
        return PHUB_ERR_CUDA;
    }
    return PHUB_OK;
}

phub_status phub_ipc_close(int32_t device, void* dev_ptr) {
    if (!dev_ptr || device < 0) return PHUB_ERR_INVALID_ARGUMENT;
    DeviceGuard g(device);
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        g_init_err = std::string("cudaIpcCloseMemHandle: ") + cudaGetErrorString(e);
        return PHUB_ERR_CUDA;
    }
    return PHUB_OK;
}

phub_status phub_set_option(phub_ctx c, int32_t option, int64_t value) {
    if (!c) return PHUB_ERR_INVALID_ARGUMENT;
    switch (option) {
        case PHUB_OPT_KERNEL:
            if (value < PHUB_KERNEL_AUTO || value > PHUB_KERNEL_BULK)
                return c->fail(PHUB_ERR_INVALID_ARGUMENT, "unknown kernel variant");
            c->kernel = (int)value;
            return PHUB_OK;
        case PHUB_OPT_GRID:
            if (value < 0 || value > (1 << 30)) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "bad grid");
            c->grid_override = (int)value;
            return PHUB_OK;
        case PHUB_OPT_SCHED_TRACE:
            if (value % 8) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "trace buffer must be 8-B aligned");
            c->sched_trace = reinterpret_cast<uint64_t*>(value);
            return PHUB_OK;
        case PHUB_OPT_L2_RESIDENT:
            if (value < 0) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "resident bytes must be >= 0");
            c->resident_bytes = (uint64_t)value;
            return PHUB_OK;
        case PHUB_OPT_CACHE: {
            if (value != PHUB_CACHE_ENABLED && value != PHUB_CACHE_BYPASS &&
                value != PHUB_CACHE_RESIDENT)
                return c->fail(PHUB_ERR_INVALID_ARGUMENT, "unknown cache mode");
            c->cache = (int)value;
            DeviceGuard g(c->device);
            for (int vec8 = 0; vec8 < 2; ++vec8)
                for (int agg = 0; agg < 2; ++agg)
                    c->flat_grid[vec8][agg] =
                        c->num_sms * phub::flat_blocks_per_sm(vec8 ? 8 : 4, c->N, agg, c->cache);
            return PHUB_OK;
        }
        case PHUB_OPT_FLAT_ONESHOT:
            if (value < -1 || value > 1) return c->fail(PHUB_ERR_INVALID_ARGUMENT, "-1, 0 or 1");
            c->flat_oneshot = (int)value;
            return PHUB_OK;
        case PHUB_OPT_TILE_ELEMS: {
            if (value < 1 || value > (1 << 30))
                return c->fail(PHUB_ERR_INVALID_ARGUMENT, "tile elements must be in [1, 2^30]");
            if (phub_status st0 = c->guard()) return st0;
            DeviceGuard g(c->device);
            const uint32_t old = c->tile_elems;
            c->tile_elems = (uint32_t)value;
            std::vector<Tile> tiles = build_tiles(c);
            Tile* d = nullptr;
            cudaError_t e = cudaSuccess;
            if (!tiles.empty()) {
                if ((e = cudaMalloc(&d, sizeof(Tile) * tiles.size())) != cudaSuccess) {
                    cudaGetLastError();
                    c->tile_elems = old;
                    return c->fail(PHUB_ERR_OUT_OF_MEMORY, "tile table: %s", cudaGetErrorString(e));
                }
                if ((e = cudaDeviceSynchronize()) != cudaSuccess ||
                    (e = cudaMemcpy(d, tiles.data(), sizeof(Tile) * tiles.size(),
                                    cudaMemcpyHostToDevice)) != cudaSuccess)
                    return c->cuda_fail(e, "tile table upload");
            }
            cudaFree(c->d_tiles);
            c->d_tiles = d;
            c->n_tiles = tiles.size();
            return PHUB_OK;
        }
        default:
            return c->fail(PHUB_ERR_INVALID_ARGUMENT, "unknown option %d", option);
    }
}

// Hierarchical-reduction benefit model, PAPER.md P:760-763 (S 3.4 "Rack
// Deployment and Topology-Aware Reduction"), as printed (R18):
//   B_bn = min((r-1) B_PBox, B_Core)
//   beneficial  <=>  max((N-1)/B_bn, 1/(N B_Wkr)) > max(1/B_PBox, N/B_Wkr) + C
//   C = (N-1)/(N B_bn)  sharded cross-rack step,  C = (r-1)/(r B_bn)  ring.
phub_status phub_hier_beneficial(int32_t workers_per_rack, int32_t racks, double b_pbox,
                                 double b_wkr, double b_core, int32_t cross_rack,
                                 int32_t* beneficial, double* lhs, double* rhs) {
    std::string& why = g_init_err;
    why.clear();
    if (!beneficial) return why = "beneficial is NULL", PHUB_ERR_INVALID_ARGUMENT;
    if (workers_per_rack < 1 || racks < 2)
        return why = "need >= 1 worker per rack and >= 2 racks", PHUB_ERR_INVALID_ARGUMENT;
    if (!(std::isfinite(b_pbox) && b_pbox > 0) || !(std::isfinite(b_wkr) && b_wkr > 0) ||
        !(std::isfinite(b_core) && b_core > 0))
        return why = "bandwidths must be finite and > 0", PHUB_ERR_INVALID_ARGUMENT;
    if (cross_rack != PHUB_CROSS_RACK_SHARDED && cross_rack != PHUB_CROSS_RACK_RING)
        return why = "cross_rack must be PHUB_CROSS_RACK_SHARDED or _RING", PHUB_ERR_INVALID_ARGUMENT;
    const double N = workers_per_rack, r = racks;
    const double b_bn = std::min((r - 1) * b_pbox, b_core);
    const double C = cross_rack == PHUB_CROSS_RACK_SHARDED ? (N - 1) / (N * b_bn)
                                                           : (r - 1) / (r * b_bn);
    const double L = std::max((N - 1) / b_bn, 1.0 / (N * b_wkr));
    const double R = std::max(1.0 / b_pbox, N / b_wkr) + C;
    *beneficial = L > R ? 1 : 0;
    if (lhs) *lhs = L;
    if (rhs) *rhs = R;
    return PHUB_OK;
}

}  // extern "C"
