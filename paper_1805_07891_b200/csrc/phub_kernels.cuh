// Internal launch interface between the host core (phub_core.cpp) and the
// sm_100a kernels (phub_kernels.cu).  Not part of the C ABI.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace phub {

constexpr int kMaxWorkers = 64;       // flat-kernel pointer array capacity
constexpr int kMaxReplicas = 16;      // peer weight replicas written by the flat kernel
constexpr int kThreads = 256;         // CTA size of every hot kernel

// One CTA tile of an owned chunk (chunk-tile kernel).  `off` is the element
// offset in the padded device layout, `key` the key the chunk belongs to.
struct Tile {
    uint64_t off;
    uint32_t len;
    uint32_t key;
};

struct FlatArgs {
    const float* g[kMaxWorkers];      // worker bases in the padded layout
    float* w;
    float* v;
    float* agg;                       // nullptr unless keep_aggregate
    uint64_t begin, end;              // owned padded range [begin, end), elements
    float lr, mu, rescale;
    int nw;
    int nrep;                         // extra replicas (peer-mapped) that also receive w'
    float* rep[kMaxReplicas];
    // optional device-side stage ordering (chained exchange)
    const uint32_t* wait_flag;
    uint32_t wait_value;
    uint32_t* signal_flag;
    uint32_t signal_value;
    uint32_t* cta_counter;            // local counter: last CTA raises signal_flag
    uint32_t* timeouts;               // [0] expired waits, [1] highest wait value given up on
    volatile uint32_t* err_host;      // host-mapped word set to 1 on any expired wait: the
                                      // host turns it into a sticky PHUB_ERR_SYNC_TIMEOUT
    uint64_t block;                   // > 0: block-streaming flags (one per `block` elements)
    uint32_t* ticket;                 // [0] next block, [1] CTAs done (block streaming, zeroed)
    uint64_t keep_from;               // PHUB_CACHE_RESIDENT: vectors >= keep_from (relative to
                                      // begin) are the L2-kept slice of w
};

// Hierarchical reduction: one GPU = one rack's PBox with its P
// local workers; R racks exchange rack aggregates over NVLink by owner range.
constexpr int kMaxRacks = 16;
struct HierArgs {
    const float* g[kMaxWorkers];      // this rack's workers (padded-layout bases)
    int nw;                           // P
    int R, rack;
    float* w;
    float* v;
    float* agg;                       // nullptr unless keep_aggregate (owned range)
    float lr, mu, rescale;
    int nrep;
    float* rep[kMaxReplicas];         // peer replicas receiving w' of the owned range
    uint64_t own_begin[kMaxRacks], own_end[kMaxRacks];
    uint64_t block;                   // elements per block (multiple of 2048)
    const float* inbox[kMaxRacks];    // this owner's inbox per source rack (padded-based)
    float* peer_inbox[kMaxRacks];     // owner o's inbox slot for this rack (padded-based)
    const uint32_t* flags;            // this owner's arrival flags [block * R + source rack]
    uint32_t* peer_flags[kMaxRacks];  // owner o's arrival flags (peer-mapped)
    uint32_t epoch;
    uint32_t* ticket;                 // [0] next item, [1] CTAs done
    uint32_t* timeouts;               // [0] expired waits, [1] abandoned epoch
    volatile uint32_t* err_host;      // host-mapped sticky-error word (see FlatArgs)
    int worker_order;                 // 1: flat worker-order sum of raw slices (M3 exchange)
    int device_barrier;               // 1: in-kernel round barrier over flags [J*R, J*R + 2R)
};
cudaError_t launch_hier(const HierArgs& a, int grid, cudaStream_t s, int* launches);
int hier_blocks_per_sm(int nw, bool worker_order);

// Scheduled exchange (phub_sched_exchange): one persistent
// launch per GPU executes a host-built item program in ticket order.  The item
// layout is phub_sched_item's (static_assert in phub_core.cpp).
struct SchedItem {
    uint64_t lo, hi, base, len;
    uint32_t type;
    int32_t dst;
    uint32_t wait_flag, signal_flag;
};
constexpr uint32_t kNoFlag = 0xffffffffu;
struct SchedArgs {
    const float* g[kMaxWorkers];      // this rank's workers (padded-layout bases)
    int nw;                           // W
    int R, rank;
    float* w;
    float* v;
    float* agg;                       // nullptr unless keep_aggregate
    float lr, mu, rescale;
    int nrep;
    float* rep[kMaxReplicas];         // peer replicas receiving w' of every NAG item
    const SchedItem* items;           // [0, nprod) producer lane, [nprod, nitems) consumer lane
    uint64_t nitems, nprod;
    int grid_prod;                    // CTAs [0, grid_prod) serve the producer lane
    uint64_t* trace;                  // diagnostic: per item (in lane order) 4 x u64 -- ticket,
                                      // wait done, item done (%globaltimer ns), CTA << 32 | SM
    float* inbox[kMaxRacks];          // rank q's partial/sum inbox (padded-based)
    float* raw_inbox[kMaxRacks];      // rank q's raw inbox
    uint32_t* flags[kMaxRacks];       // rank q's flags
    uint32_t epoch;
    int64_t bar;                      // >= 0: index of the 2R round-barrier flags (in-kernel
                                      // start / end barriers instead of the caller's); -1: off
    uint32_t* ticket;                 // [0] next producer item, [1] CTAs done, [2] next consumer
    uint32_t* timeouts;               // [0] expired waits, [1] abandoned epoch
    volatile uint32_t* err_host;
};
cudaError_t launch_sched(const SchedArgs& a, int grid, cudaStream_t s, int* launches);
int sched_blocks_per_sm(int nw);

struct TileArgs {
    const Tile* tiles;
    uint64_t ntiles;
    const uintptr_t* base;            // [nw * K]: base[w*K+k] + 4*off = byte address
    int K;
    int nw;
    float* w;
    float* v;
    float* agg;
    float lr, mu, rescale;
};

struct WideArgs {                     // ablation: wide aggregation
    const float* g[kMaxWorkers];
    float* w;
    float* v;
    float* agg;                       // required scratch: the merge buffer
    uint64_t begin, end;
    float lr, mu, rescale;
    int nw;
};

// vec = 8 (256-bit LDG/STG, sm_100a) or 4 (128-bit).  cache = PHUB_CACHE_*.
cudaError_t launch_flat(const FlatArgs& a, int vec, int cache, int grid, cudaStream_t s,
                        int* launches);
cudaError_t launch_tiles(const TileArgs& a, int grid, cudaStream_t s, int* launches);
// Worker-order partial sum (no optimizer): dst[i] = ((+0 + g0[i]) + g1[i]) + ...
// over [a.begin, a.end); dst may be a peer-mapped pointer (chained exchange).
cudaError_t launch_prefix(const FlatArgs& a, float* dst, int grid, cudaStream_t s, int* launches);
// Block-streaming forms (a.block > 0): one persistent launch over [begin, end)
// walking blocks of a.block elements in order, waiting on a.wait_flag[b] and
// raising a.signal_flag[b] per block.  dst == nullptr: fused Nesterov (w, v,
// replicas); else the worker-order partial sum stored into dst.
cudaError_t launch_blocks(const FlatArgs& a, float* dst, int grid, cudaStream_t s, int* launches);
int blocks_per_sm(int nw, bool nag);
// TMA-style staging: 1-D bulk async copies into a shared-memory ring (nw <= 8).
cudaError_t launch_bulk(const FlatArgs& a, int grid, cudaStream_t s, int* launches);
size_t bulk_smem_bytes(int nw);
cudaError_t launch_wide(const WideArgs& a, int grid, cudaStream_t s, int* launches);

// Load every kernel into the current device's context (lazy-loading safety for
// the flag protocols; see phub_kernels.cu).
cudaError_t preload_kernels();

// Resident CTAs per SM of the flat kernel for (vec, nw, agg) -- grid sizing.
int flat_blocks_per_sm(int vec, int nw, bool agg, int cache);

}  // namespace phub
