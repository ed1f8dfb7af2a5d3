/*
 * phub.h -- C ABI of the B200-native PHub parameter-exchange hot path.
 *
 * PHub (arXiv 1805.07891) is a parameter server: N workers push per-key
 * gradients, the server sums them per fixed-size chunk ("tall aggregation")
 * and applies a Nesterov-SGD update to the chunk's weights and momentum, and
 * workers pull the updated weights back.  This library implements that hot
 * path on one B200 (sm_100a) per context; several contexts (one per GPU /
 * process) shard the chunks by owner.
 *
 * Citations: P:n = PAPER.md line n (canonical copy P:377-1120), S:n = SPEC.md
 * line n.  DESIGN.md lists every reading of the paper used here (R1..R18).
 *
 *   problem statement ........ P:634-638 (InitService allocates receive and
 *                               merge buffers; Push / Pull / PushPull)
 *   chunking .................. P:693-703 (32 KB mini-chunks, "virtual keys")
 *   chunk -> owner ............ P:708-717 (assignment computed at init; 4/3
 *                               set partition)
 *   aggregation + optimizer ... P:657, P:677-686 (tall: the thread that sums a
 *                               chunk over all workers also optimizes it),
 *                               P:783 (Nesterov SGD; recurrence from S:189)
 *
 * Conventions (all entry points):
 *   - extern "C", no C++ exception ever crosses the boundary; every call
 *     returns a phub_status.  On any validation error the context state is
 *     unchanged and phub_last_error() explains it.
 *   - A CUDA runtime error makes the context sticky-failed: the failing call
 *     and every later call (except the introspection/destroy calls) return
 *     PHUB_ERR_CUDA.
 *   - Device-side flag waits (phub_sync, phub_hier_exchange) are bounded
 *     (~2 s).  A launch whose wait expires skips that work and raises a
 *     host-mapped error word; the context then becomes sticky-failed with
 *     PHUB_ERR_SYNC_TIMEOUT, reported by the first call that starts after the
 *     expiry -- like an asynchronous CUDA error.  Every synchronizing call
 *     (phub_synchronize, phub_read_state, phub_load_state) reports it for all
 *     work enqueued before it, so a partly skipped round is never returned as
 *     PHUB_OK by a call that waited for it.
 *   - `stream` arguments are a cudaStream_t passed as void* (NULL = legacy
 *     default stream).  Work is enqueued on it; validation is synchronous on
 *     the host before anything is enqueued.
 *   - One host thread per context at a time.  Any number of contexts
 *     may coexist in a process (multi-tenant analog).
 *   - Element type is IEEE-754 binary32 ("single-precision").
 *   - Device layout: keys are stored key-major; key k starts at element
 *     key_offsets[k] (phub_layout), each start rounded up to 32 elements
 *     (128 B) so every key is 128-B aligned; E_padded is the padded total.
 *     Padding elements carry no meaning and are never returned by pull or
 *     read_state.
 */
#ifndef PHUB_H
#define PHUB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct phub_ctx_s* phub_ctx;    /* opaque; owns every device arena */

typedef enum {
    PHUB_OK = 0,
    PHUB_ERR_INVALID_ARGUMENT = 1,   /* null ptr, N<1, lr/mu not finite, mu outside [0,1),
                                        bad owner/rank/policy/mode, misaligned BORROW pointer */
    PHUB_ERR_INVALID_MANIFEST = 2,   /* num_keys==0 or some key has 0 elements     */
    PHUB_ERR_INVALID_CHUNK_SIZE = 3, /* chunk_size_bytes % 4 != 0             */
    PHUB_ERR_INVALID_INIT = 4,       /* init_num_elements != E                      */
    PHUB_ERR_BAD_WORKER = 5,         /* worker_id >= N                              */
    PHUB_ERR_BAD_KEY = 6,            /* key >= num_keys and != PHUB_ALL_KEYS        */
    PHUB_ERR_LENGTH_MISMATCH = 7,    /* n != n_k, or != E_padded for PHUB_ALL_KEYS  */
    PHUB_ERR_DUPLICATE_PUSH = 8,     /* same (worker, key) twice in one iteration   */
    PHUB_ERR_INCOMPLETE = 9,         /* aggregate before all N x K pushes arrived   */
    PHUB_ERR_CUDA = 10,              /* CUDA runtime/launch error; context sticky-failed    */
    PHUB_ERR_OUT_OF_MEMORY = 11,     /* device allocation failed                            */
    PHUB_ERR_UNSUPPORTED = 12,       /* option/variant not available for this context       */
    PHUB_ERR_SYNC_TIMEOUT = 13       /* a device-side flag wait expired; sticky              */
} phub_status;

#define PHUB_ALL_KEYS (-1)            /* whole-model push/pull in the padded layout        */
#define PHUB_OWNED_RANGE (-2)         /* push of exactly this context's owned padded range  */

enum { PHUB_COPY = 0, PHUB_BORROW = 1 };          /* ownership mode of a pushed buffer   */
enum { PHUB_OWNER_LPT = 0, PHUB_OWNER_CONTIG = 1 };  /* chunk -> owner policy    */

/* One virtual key: chunk `vkey_id` of key `key_id` covers elements
 * [offset, offset+length) of that key; `owner` is the owning rank. */
typedef struct {
    uint32_t vkey_id;
    uint32_t key_id;
    uint64_t offset;
    uint64_t length;
    int32_t owner;
    int32_t reserved;
} phub_chunk;

typedef struct {
    const uint64_t* key_num_elements; /* manifest: n_k for k in [0,num_keys), key order = id */
    int32_t num_keys;
    int32_t num_workers;              /* N >= 1                                            */
    uint64_t chunk_size_bytes;        /* 0 -> 32768 ("default is 32KB")       */
    float lr;                         /* eta, finite                                       */
    float momentum;                   /* mu in [0,1)                               */
    float rescale;                    /* optimizer input g = s * rescale; 0 -> 1.0f/N      */
                                      /* (mean of the gradients; reading R2)        */
    int32_t device;                   /* CUDA device ordinal the context lives on          */
    int32_t num_owners;               /* G >= 1: ranks the chunks are sharded over         */
    int32_t owner_rank;               /* this context's rank in [0, G)                     */
    int32_t owner_policy;             /* PHUB_OWNER_LPT or PHUB_OWNER_CONTIG               */
    int32_t keep_aggregate;           /* nonzero: also store the sum s (test mode)         */
    const float* init_weights;        /* NULL -> zeros; else E elements,       */
                                      /* key-major unpadded, host or device memory         */
    uint64_t init_num_elements;       /* must equal E when init_weights != NULL            */
} phub_config;

/* Fill `cfg` with defaults: chunk 32 KB, lr 0.1, mu 0.9, rescale 0 (=1/N),
 * device 0, G=1, rank 0, CONTIG, no aggregate, zero init weights. */
void phub_config_default(phub_config* cfg);

/* InitService analog: build the chunk plan, the chunk -> owner
 * table, the padded device layout, and allocate w, v (and s) in
 * one shot on cfg->device.  w = init weights or 0, v = 0.
 * On success *out owns everything; release with phub_destroy. */
phub_status phub_init(const phub_config* cfg, phub_ctx* out);
phub_status phub_destroy(phub_ctx ctx);

/* Push: make worker `worker`'s gradient for key `key`
 * (or PHUB_ALL_KEYS) available for this iteration.
 *   key == PHUB_ALL_KEYS: `grad` holds n == E_padded elements in the padded
 *     layout (keys at phub_layout offsets).  Only this context's owned chunks
 *     are read.
 *   key == PHUB_OWNED_RANGE (CONTIG ownership or G == 1): `grad` holds
 *     n == end - begin elements, the padded range phub_owner_range() gives
 *     for this context's rank -- what an owner receives from a remote worker.
 *     If that range is empty (an owner with no chunk) n == 0 and `grad`
 *     may be NULL.
 *   key in [0, num_keys): `grad` holds n == n_k contiguous elements.
 *   mode PHUB_BORROW: zero copy -- the pointer is recorded and read by
 *     the next phub_aggregate_optimize.  `grad` must be device memory
 *     (this or a peer-mapped GPU), 16-byte aligned.  The caller must keep it
 *     valid and unmodified until that aggregate has completed on its stream.
 *   mode PHUB_COPY: the data (host or device memory) is copied into the
 *     context's receive arena on `stream`; the caller may reuse `grad` once
 *     the copy has completed on `stream`.  The arena has two slots (iteration
 *     i uses slot i % 2, 2 x N x E_padded floats, allocated on the first COPY
 *     push), so iteration i+1's copies may run on another stream while
 *     iteration i's kernel runs; the caller orders the streams (the copies of
 *     i+1 must not start before the kernel of i-1 has finished).
 * Errors: BAD_WORKER, BAD_KEY, LENGTH_MISMATCH, DUPLICATE_PUSH (this
 * (worker, key) already pushed in this iteration), INVALID_ARGUMENT. */
phub_status phub_push(phub_ctx ctx, int32_t worker, int32_t key, const float* grad,
                      uint64_t n, int32_t mode, void* stream);

/* Batched push: `count` pushes in one call (per-key framework pushes, e.g.
 * one per layer as a backward pass produces them -- P:638).  Entry j
 * is phub_push(ctx, workers[j], keys[j], grads[j], lens[j], mode, stream).
 * Validated all-or-nothing: on any error nothing is recorded (no receipts,
 * no copies) and *failed_index (nullable) names the offending entry. */
phub_status phub_push_batch(phub_ctx ctx, int32_t count, const int32_t* workers,
                            const int32_t* keys, const float* const* grads,
                            const uint64_t* lens, int32_t mode, void* stream,
                            int32_t* failed_index);

/* Aggregate + optimize every owned chunk: for each element i
 *   s  = (((+0.0f + g_0[i]) + g_1[i]) + ...) + g_{N-1}[i]   (worker-id order)
 *   g  = s * rescale
 *   v' = mu * v[i] + g
 *   w' = w[i] - lr * (g + mu * v')
 * every operation separately rounded to nearest-even in fp32, no contraction
 * (readings R3-R6).  One fused kernel launch on `stream`.  Requires every
 * (worker, key) pushed (else PHUB_ERR_INCOMPLETE, nothing enqueued).  Then
 * clears the receipts and advances the iteration counter. */
phub_status phub_aggregate_optimize(phub_ctx ctx, void* stream);

/* Streaming aggregation ("when a chunk is received from all workers, it
 * can be optimized"; "streaming aggregation and optimization"): launch
 * the fused kernel on the chunks of every key whose N pushes have all arrived
 * and that has not been aggregated in this iteration (chunk-tile kernel, one
 * launch per run of consecutive ready keys); *keys_done (nullable) receives
 * how many keys were launched.  When every key of the iteration has been
 * aggregated the receipts clear and the iteration advances.  A later
 * phub_aggregate_optimize processes only the keys not yet aggregated.
 * Results are bit-identical to one phub_aggregate_optimize (element-wise,
 * P:657).  Not combinable with phub_set_replicas (PHUB_ERR_UNSUPPORTED). */
phub_status phub_aggregate_ready(phub_ctx ctx, void* stream, uint64_t* keys_done);

/* Pull: copy the current weights of `key` (n == n_k) or of
 * the whole padded model (PHUB_ALL_KEYS, n == E_padded) into `dst` (host or
 * device memory) on `stream`.  Before any aggregate it returns the initial
 * weights; after k aggregates, iteration k's result. */
phub_status phub_pull(phub_ctx ctx, int32_t key, float* dst, uint64_t n, void* stream);

/* PushPull: push `grad` for `worker` (COPY or BORROW, as
 * phub_push with key == PHUB_ALL_KEYS); when that push completes the
 * iteration (all N x K receipts), run phub_aggregate_optimize and copy the
 * updated padded model into `dst` (may be NULL).  Otherwise only pushes. */
phub_status phub_pushpull(phub_ctx ctx, int32_t worker, const float* grad, uint64_t n,
                          int32_t mode, float* dst, void* stream);

/* Zero-copy pull: the device pointer of the padded weight replica (E_padded
 * elements).  Valid until phub_destroy.  Writes by the caller (e.g. an
 * all-gather of other owners' ranges at G > 1) are allowed. */
phub_status phub_weights(phub_ctx ctx, float** w_dev);

/* Layout: E (real elements), E_padded, and key_offsets[num_keys] (may be NULL). */
phub_status phub_layout(phub_ctx ctx, uint64_t* E, uint64_t* E_padded, uint64_t* key_offsets);

/* Host-only planning (no device needed): the chunk table phub_init would
 * build for this manifest, chunk size, G and policy, written to out[0..cap).
 * *count receives the number of chunks; cap may be 0 (count query).
 * Errors as phub_init's validation; LENGTH_MISMATCH if cap < count. */
phub_status phub_plan_chunks(const uint64_t* key_num_elements, int32_t num_keys,
                             uint64_t chunk_size_bytes, int32_t num_owners, int32_t owner_policy,
                             phub_chunk* out, uint64_t cap, uint64_t* count);

/* Host-only layout planning (no device): E_padded, key_offsets[num_keys]
 * (may be NULL) and the CONTIG owner ranges owner_begin/end[num_owners] (may
 * be NULL) exactly as phub_init / phub_owner_range would give them. */
phub_status phub_plan_ranges(const uint64_t* key_num_elements, int32_t num_keys,
                             uint64_t chunk_size_bytes, int32_t num_owners, uint64_t* E_padded,
                             uint64_t* key_offsets, uint64_t* owner_begin, uint64_t* owner_end);

/* Chunk table (S:125 order: vkey_id, key_id, offset, length, owner). */
phub_status phub_num_chunks(phub_ctx ctx, uint64_t* n);
phub_status phub_chunk_table(phub_ctx ctx, phub_chunk* out, uint64_t cap);

/* Padded-layout element range [begin, end) owned by `owner` under the CONTIG
 * policy (G == 1 or PHUB_OWNER_CONTIG); PHUB_ERR_UNSUPPORTED under LPT.
 * Ranges of consecutive owners abut; an owner with no chunk gets begin==end. */
phub_status phub_owner_range(phub_ctx ctx, int32_t owner, uint64_t* begin, uint64_t* end);

/* Owned elements (real, padding excluded) of this context. */
phub_status phub_owned_elements(phub_ctx ctx, uint64_t* n);

/* Overwrite w and/or v (each E elements, key-major unpadded, host or device,
 * NULL = leave unchanged).  Synchronous.  Checkpoint-restore analog. */
phub_status phub_load_state(phub_ctx ctx, const float* w, const float* v);

/* Read w, v and (keep_aggregate) the last sum s into E-element key-major
 * unpadded buffers (host or device; NULL = skip).  Synchronous (device-wide
 * synchronize first).  agg must be NULL unless keep_aggregate. */
phub_status phub_read_state(phub_ctx ctx, float* w, float* v, float* agg);

/* Iterations completed, and kernels this context has launched. */
phub_status phub_iteration(phub_ctx ctx, uint64_t* iteration);
phub_status phub_kernel_launches(phub_ctx ctx, uint64_t* launches);

/* ---------------------------------------------------------------------------
 * Peer-memory exchange (multi-GPU, one process per GPU)
 *
 * The owner's fused kernel can read remote workers' gradients and write the
 * updated weights into remote replicas directly over NVLink: push a peer-mapped
 * gradient pointer with PHUB_BORROW, and register peer-mapped replicas here.
 * Then one kernel does aggregate + optimize + the all-gather of the pull
 * ("transmitted back to the workers on its originating path").
 * The caller orders rounds across GPUs (e.g. a stream-ordered barrier before
 * and after phub_aggregate_optimize); the library never spins on peers.
 * ------------------------------------------------------------------------- */

/* Device-side ordering between the stages of a chained exchange (one GPU per
 * process).  `wait_flag` (nullable) is a uint32 in this GPU's memory that a
 * previous stage raises; every CTA of the launch first waits until
 * *wait_flag >= wait_value (system-scope acquire; bounded: after ~2 s it
 * gives up, skips its work and the context becomes sticky-failed with
 * PHUB_ERR_SYNC_TIMEOUT -- see the conventions above and phub_sync_timeouts).
 * `signal_flag` (nullable, typically peer-mapped) is written with
 * `signal_value` (system-scope release) once every CTA of the launch has
 * finished its stores -- and never if any CTA of the launch gave up its wait,
 * so a downstream stage cannot consume a partly computed partial.  At most one
 * signalling (or block-streaming) launch per context in flight.
 *
 * Block-streaming form (`block_elems` > 0, a multiple of 2048): the model is
 * cut into blocks b = [b*block_elems, (b+1)*block_elems) of the padded layout
 * and `wait_flag` / `signal_flag` point at ARRAYS with one uint32 per block
 * (ceil(E_padded / block_elems) entries).  One persistent launch walks its
 * range block by block: before reading block b a CTA waits for
 * wait_flag[b] >= wait_value; once block b's stores are performed it raises
 * signal_flag[b] = signal_value (a skipped block is never raised).  A
 * downstream stage can then start on block b while this launch still works on
 * later blocks -- the pipelining of PHub's streaming aggregation
 * without one launch per piece.  Flags must be 4-B aligned. */
typedef struct {
    const uint32_t* wait_flag;
    uint32_t wait_value;
    uint32_t* signal_flag;
    uint32_t signal_value;
    uint64_t block_elems;       /* 0: one flag per launch; > 0: one flag per block */
} phub_sync;

/* Chained exchange (workers hosted in rank order): the
 * worker-order partial sum of `count` (<= 64) padded-layout sources over
 * [begin, end), stored into `dst` (padded layout; typically a peer-mapped
 * buffer of the next rank):  dst[i] = ((+0 + src0[i]) + src1[i]) + ...
 * Because the sum starts from +0 and adds in order, chaining partials rank
 * by rank reproduces the global worker-order sum bit for bit (reading R3).
 * All pointers 32-B aligned device memory; begin, end multiples of 8.
 * Uses ctx's device; no receipts are involved. */
phub_status phub_partial_sum(phub_ctx ctx, const float* const* srcs, int32_t count, float* dst,
                             uint64_t begin, uint64_t end, const phub_sync* sync, void* stream);

/* Range-wise aggregation of one iteration (pipelined exchange): requires all
 * N x K pushes, whole-model / owned-range pushes under CONTIG ownership;
 * runs the fused kernel on the owned elements of [begin, end).  Calls must
 * cover the owned range in increasing, abutting order starting at its begin
 * (begin == previous end); the call that reaches the owned range's end
 * completes the iteration.  begin/end multiples of 8 (or the range bounds). */
phub_status phub_aggregate_range(phub_ctx ctx, uint64_t begin, uint64_t end,
                                 const phub_sync* sync, void* stream);

/* Number of device-side waits (phub_sync, phub_hier_exchange) that expired on
 * this context (synchronous; reported even when the context is failed --
 * a nonzero count also makes it sticky-failed with PHUB_ERR_SYNC_TIMEOUT). */
phub_status phub_sync_timeouts(phub_ctx ctx, uint32_t* count);

/* The context's status now, without synchronizing: PHUB_OK, or the sticky
 * PHUB_ERR_SYNC_TIMEOUT / PHUB_ERR_CUDA (a wait that expired after this call
 * shows up in a later one). */
phub_status phub_check(phub_ctx ctx);

/* Wait for `stream` (NULL: the whole device) and return the context's status:
 * PHUB_OK, or the sticky PHUB_ERR_SYNC_TIMEOUT / PHUB_ERR_CUDA of any work
 * waited for. */
phub_status phub_synchronize(phub_ctx ctx, void* stream);

/* Every later phub_aggregate_optimize also stores w' of the owned range into
 * replicas[0..count) (padded layout, E_padded elements each; device pointers,
 * typically peer-mapped with phub_ipc_open).  count == 0 clears.  count <= 16.
 * Requires CONTIG ownership (or G == 1) and the flat kernel (whole-model or
 * owned-range pushes, 32-B aligned chunk layout), else PHUB_ERR_UNSUPPORTED
 * at aggregate time. */
phub_status phub_set_replicas(phub_ctx ctx, float* const* replicas, int32_t count);

/* Hierarchical reduction across racks: each
 * GPU (context) is one rack's PBox whose N local workers pushed their whole
 * model (PHUB_ALL_KEYS, BORROW, 32-B aligned) this iteration; the context has
 * CONTIG ownership over G = num_racks owners and owner_rank = this rack.
 * One launch performs the paper's three steps for the whole model:
 *   1. per rack:   S_rack = ((+0 + g_0) + g_1) + ... + g_{N-1}  (local workers)
 *   2. cross rack: every other rack's S over this owner's range arrives in
 *                  this owner's inbox (their launches store it over NVLink);
 *                  s = ((+0 + S_0) + S_1) + ... + S_{G-1}  in rack order, the
 *                  rack-by-rack accumulation of the paper's emulation (P:1008,
 *                  reading R17)
 *   3. optimizer:  Nesterov on the owned range with g = s * rescale (set
 *                  rescale = 1/(G*N) for the mean over all workers), w'
 *                  stored locally and into every replica registered with
 *                  phub_set_replicas (the per-rack broadcast).
 * while its own step-1 sums for the OTHER owners' ranges are stored into their
 * inboxes.  Work is cut into blocks of `block_elems` (multiple of 2048) of each
 * owner range; per block and source rack a uint32 flag (system-scope release /
 * acquire, value `epoch`) orders arrival.  Bounded waits as phub_sync.
 *   inbox[q]       device pointer such that inbox[q] + x is this owner's
 *                  receive slot for rack q's element x (x in the owned padded
 *                  range); inbox[rack] unused.  Two slots alternated by the
 *                  caller per epoch parity (a rack may run one round ahead).
 *   peer_inbox[o]  peer-mapped: owner o's receive slot for THIS rack, same
 *                  addressing over o's range; [rack] unused.
 *   flags          this owner's flags, ceil(owned / block_elems) x num_racks
 *                  uint32, zero before the first epoch; never reset.
 *   peer_flags[o]  peer-mapped flags of owner o.
 *   epoch          1, 2, 3, ... (strictly increasing per round).
 * Completes the iteration.  The caller orders rounds so every replica write
 * of round k is complete before its replica is read (e.g. a barrier after). */
typedef struct {
    int32_t num_racks;
    uint64_t block_elems;
    const float* const* inbox;
    float* const* peer_inbox;
    const uint32_t* flags;
    uint32_t* const* peer_flags;
    uint32_t epoch;
    /* 0: hierarchical (rack-grouped) sum as above.  != 0: the flat worker-order
     * sum over all num_racks x N workers -- rack q's local worker k is global
     * worker q*N + k -- i.e. the owner-sharded exchange of ONE job whose
     * workers are spread over the GPUs (reading R3), with every transfer an
     * NVLink store: each rack stores its workers' raw slices of owner o's
     * range into o's inbox (worker k at inbox + k*L + x, L = o's owned
     * length, so each slot holds N slices) and o sums them in worker order. */
    int32_t worker_order;
    /* nonzero: in-kernel round barriers as phub_sched.device_barrier -- flags and
     * peer_flags then hold 2 x num_racks more entries after the block flags, at
     * [J*num_racks, J*num_racks + 2*num_racks), J = the block count of the
     * LARGEST owner range (every rack's flag arrays sized alike).  0: the
     * caller orders rounds. */
    int32_t device_barrier;
} phub_hier;
phub_status phub_hier_exchange(phub_ctx ctx, const phub_hier* h, void* stream);

/* Hierarchical-reduction benefit model (S 3.4; R18),
 * host-only, as printed in the paper: with N = workers_per_rack, r = racks,
 *   B_bn = min((r-1) * B_PBox, B_Core)
 *   lhs  = max((N-1)/B_bn, 1/(N*B_Wkr))         time of the flat cross-rack step
 *   rhs  = max(1/B_PBox, N/B_Wkr) + C           local aggregation + cross-rack cost
 *   C    = (N-1)/(N*B_bn)   PHUB_CROSS_RACK_SHARDED (sharded PSs; this build's
 *                           k_hier cross-rack step)
 *        = (r-1)/(r*B_bn)   PHUB_CROSS_RACK_RING (racks in a ring; the paper's
 *                           emulation)
 * *beneficial = lhs > rhs.  Bandwidths in any one consistent unit (> 0,
 * finite); lhs/rhs (nullable) are in its reciprocal (time per model byte).
 * INVALID_ARGUMENT for N < 1, r < 2 (no cross-rack step), bad bandwidths or
 * mode.  Needs no device. */
enum { PHUB_CROSS_RACK_SHARDED = 0, PHUB_CROSS_RACK_RING = 1 };
phub_status phub_hier_beneficial(int32_t workers_per_rack, int32_t racks, double b_pbox,
                                 double b_wkr, double b_core, int32_t cross_rack,
                                 int32_t* beneficial, double* lhs, double* rhs);

/* ---------------------------------------------------------------------------
 * Scheduled owner-sharded exchange ("chunks ...
 * assigned to owners", P:698 streaming aggregation; reading R3 worker order)
 *
 * One persistent launch per GPU executes a host-built ITEM PROGRAM for the
 * N-worker job whose workers are hosted in rank order (rank p hosts global
 * workers [p*W, (p+1)*W)).  The padded model is cut into owner ranges
 * [bounds[o], bounds[o+1]); each owner range into a RAW part [bounds[o],
 * split[o]) and a CHAIN part [split[o], bounds[o+1]):
 *   RAW part:   every other rank stores its W workers' raw slices into the
 *               owner's raw inbox; the owner sums all N workers in worker
 *               order (CONSUME_RAW) -- the push exchange;
 *   CHAIN part: the worker-order sum is built rank by rank: rank 0 sums its
 *               workers from +0 and stores the partial into rank 1's inbox,
 *               rank p adds its workers to the incoming partial and stores it
 *               into rank p+1's, the last rank completes the sum and either
 *               runs the Nesterov step itself (owner == last rank) or stores
 *               s into the owner's inbox (CONSUME_FINAL).
 * Both give the flat worker-order sum s = ((+0 + g_0) + g_1) + ... bit for
 * bit (R3, R4).  The split of each owner range trades NVLink bytes between
 * ports: all-RAW is the push exchange (byte-optimal at W = 1), all-CHAIN on
 * the last owner the chained exchange (byte-optimal at G = 2); in between a
 * mix lowers the busiest port's bytes (G = 4, W = 2: 1.79 vs 2.25 model sizes,
 * scripts/sched_lp.py).  Every NAG item stores w' locally and into every
 * replica registered with phub_set_replicas.
 * ------------------------------------------------------------------------- */
enum {
    PHUB_ITEM_RAW_PUSH = 1,      /* store local workers' raw slices of [lo,hi) into rank dst's
                                    raw inbox, raise dst's flag signal_flag                   */
    PHUB_ITEM_CHAIN = 2,         /* [wait flag] partial(inbox or +0) + local workers; dst >= 0:
                                    store into rank dst's inbox and raise its signal_flag;
                                    dst < 0: Nesterov here                                   */
    PHUB_ITEM_CONSUME_RAW = 3,   /* wait flags wait_flag + q (q != rank); worker-order sum of
                                    local workers and raw inbox slots; Nesterov              */
    PHUB_ITEM_CONSUME_FINAL = 4  /* wait flag; s = inbox; Nesterov                            */
};
typedef struct {
    uint64_t lo, hi;             /* padded-layout element range, multiples of 8              */
    uint64_t base, len;          /* RAW items: the owner's raw part [base, base + len)       */
    uint32_t type;               /* PHUB_ITEM_*                                              */
    int32_t dst;                 /* destination rank, or -1                                  */
    uint32_t wait_flag;          /* index into this rank's flags, UINT32_MAX = none          */
    uint32_t signal_flag;        /* index into dst's flags                                   */
} phub_sched_item;

/* Host-only planner: the item program of `rank` (ticket order) for `ranks`
 * GPUs with `workers_per_rank` workers each.  bounds[ranks+1] (bounds[0] = 0,
 * non-decreasing, bounds[ranks] = E_padded), split[ranks] (bounds[o] <=
 * split[o] <= bounds[o+1]); every bound and split a multiple of 8.  Parts are
 * cut into blocks of block_elems (multiple of 2048).  Items are ordered by a
 * key every rank shares -- (normalized progress of the block in its part +
 * stage * lag, stage) -- so each item waits only on items with strictly
 * smaller keys on other ranks: deadlock-free with any number of co-resident
 * CTAs taking tickets in order.  The first and last
 * taper_blocks * block_elems elements of every part are cut into blocks 4x
 * smaller (multiples of 8) so the pipeline fills and drains in finer steps
 * (0 = uniform blocks).  lag_blocks shifts the chain
 * stages and consumers by that many blocks of progress (pipeline fill).
 * Flag layout (identical on every rank, *num_flags entries, zero initially):
 * chain block c: [c] partial arrival, [C + c] final arrival; raw block j
 * (numbered owner-major): [2C + j*ranks + q] slices of rank q arrived; the
 * last 2 x ranks: the round barrier of phub_sched.device_barrier.
 * *count receives the item count (cap may be 0: count query; LENGTH_MISMATCH
 * if cap < count).  INVALID_ARGUMENT on bad geometry. */
phub_status phub_sched_plan(int32_t ranks, int32_t rank, int32_t workers_per_rank,
                            const uint64_t* bounds, const uint64_t* split, uint64_t block_elems,
                            uint64_t lag_blocks, uint64_t taper_blocks, phub_sched_item* out,
                            uint64_t cap, uint64_t* count, uint32_t* num_flags);

/* Upload an item program (host array) to the context's device; validated
 * (types, ranges within E_padded and multiples of 8, dst < ranks, flag
 * indices < num_flags).  Replaces the previous program. */
phub_status phub_sched_load(phub_ctx ctx, int32_t ranks, int32_t rank, const phub_sched_item* items,
                            uint64_t count, uint32_t num_flags);

/* One round of the loaded program (one launch on `stream`).  Requires the
 * context's W = N workers pushed whole-model (PHUB_ALL_KEYS, BORROW, 32-B
 * aligned) and num_owners == 1 (the items, not the context's owner table,
 * say which ranges this rank optimizes; v is meaningful on those ranges).
 *   inbox[q]     rank q's partial/sum inbox (E_padded floats, 32-B aligned;
 *                peer-mapped for q != rank), addressed by padded element.
 *   raw_inbox[q] rank q's raw inbox: slot (src rank s, worker k) of owner q's
 *                raw part at raw_inbox[q] + ((s*W + k)*len + (x - base)).
 *   flags[q]     rank q's flags (num_flags uint32, never reset).
 *   epoch        1, 2, 3, ... strictly increasing per round (flags hold it).
 * Bounded waits as phub_sync (sticky PHUB_ERR_SYNC_TIMEOUT; a skipped item
 * never raises its flag).  The caller orders rounds (a barrier before: every
 * replica and inbox free; after: replicas complete).  Completes the
 * iteration. */
typedef struct {
    float* const* inbox;
    float* const* raw_inbox;
    uint32_t* const* flags;
    uint32_t epoch;
    int32_t consumer_ctas;       /* CTAs serving the consumer lane (CONSUME_* items); the
                                    rest serve the producers (RAW_PUSH, CHAIN), each lane in
                                    ticket order, so a consumer waiting for late data never
                                    holds a CTA the chain needs.  0 = auto (the consumers'
                                    share of the items' elements, clamped to [1/8, 1/2]).
                                    A program without CHAIN items runs as ONE lane in
                                    ticket order (the field is ignored). */
    int32_t device_barrier;      /* nonzero: the launch brackets the round with in-kernel
                                    barriers over the last 2 x ranks flags of the program
                                    -- it tells every peer its replica is free when it
                                    starts (so the caller orders its own replica reads
                                    before the launch on `stream`), stores w' into a peer
                                    replica only after that peer's launch has started,
                                    and completes only once every peer has finished
                                    storing into this rank's replica and reading its
                                    inboxes -- replacing the caller's start and end
                                    barriers (collectives).  0: the caller orders rounds. */
} phub_sched;
phub_status phub_sched_exchange(phub_ctx ctx, const phub_sched* s, void* stream);

/* Shared device allocations that can be exported to peer processes.
 * phub_alloc_shared: cudaMalloc of `bytes` on `device` (whole allocation, so an
 * IPC handle maps exactly this buffer).  phub_free_shared releases it. */
phub_status phub_alloc_shared(int32_t device, uint64_t bytes, void** dev_ptr);
phub_status phub_free_shared(int32_t device, void* dev_ptr);

/* CUDA IPC: export a phub_alloc_shared pointer (or phub_weights) as a 64-byte
 * handle; open a peer's handle on `device` (peer access enabled lazily);
 * close an opened mapping. */
phub_status phub_ipc_get_handle(int32_t device, const void* dev_ptr, void* handle64);
phub_status phub_ipc_open(int32_t device, const void* handle64, void** dev_ptr);
phub_status phub_ipc_close(int32_t device, void* dev_ptr);

/* Options (ablations / tuning).  Values are validated; PHUB_ERR_UNSUPPORTED
 * when a forced variant cannot run this context's layout. */
enum {
    PHUB_OPT_KERNEL = 1,      /* PHUB_KERNEL_*                                           */
    PHUB_OPT_GRID = 2,        /* CTAs for the flat kernels, 0 = auto (SMs x occupancy)   */
    PHUB_OPT_TILE_ELEMS = 3,  /* max elements per CTA tile in the chunk-tile kernel (1024) */
    PHUB_OPT_CACHE = 4,       /* PHUB_CACHE_*: L2 policy of the pulled weights   */
                              /* (5, 6: removed in round 2 -- measured without gain)     */
    PHUB_OPT_SCHED_TRACE = 9, /* diagnostic: device pointer to 4 x n_items uint64 that    */
                              /* phub_sched_exchange fills per item (lane order: producers */
                              /* then consumers): ticket taken, wait done, item done       */
                              /* (%globaltimer ns), CTA << 32 | SM id; 0 = off             */
    PHUB_OPT_L2_RESIDENT = 8, /* PHUB_CACHE_RESIDENT: bytes of w kept L2-resident across  */
                              /* rounds (the tail of the owned range; default 32 MiB)    */
    PHUB_OPT_FLAT_ONESHOT = 7 /* flat kernels: 1 = one vector per thread, grid covering */
                              /* the range (the hardware CTA scheduler balances like     */
                              /* PHub's chunk -> core map); 0 = persistent grid (SMs x   */
                              /* resident CTAs, grid-stride); -1 (default) = one-shot    */
                              /* unless peer replicas are registered (NVLink latency     */
                              /* favours the persistent grid)                            */
};
enum {
    PHUB_KERNEL_AUTO = 0,     /* flat 256-bit kernel when eligible, else chunk tiles     */
    PHUB_KERNEL_FLAT = 1,     /* flat owned range, 256-bit LDG/STG (needs 32-B alignment) */
    PHUB_KERNEL_TILES = 2,    /* one CTA per chunk tile, per-(worker,key) pointers       */
    PHUB_KERNEL_FLAT128 = 3,  /* flat owned range, 128-bit LDG/STG                       */
    PHUB_KERNEL_WIDE = 4,     /* ablation: wide aggregation, N-1 pairwise passes + NAG   */
                              /* pass (MXNet style)                           */
    PHUB_KERNEL_BULK = 5      /* flat range staged through shared memory by 1-D bulk     */
                              /* async copies (TMA engine, mbarrier ring); N <= 8        */
};
enum {
    PHUB_CACHE_ENABLED = 0,   /* all of w' stored evict-last (kept in L2 for the pull),  */
                              /* grads evict-first ("cache-enabled")        */
    PHUB_CACHE_BYPASS = 1,    /* every stream evict-first (the cache-bypass analog)     */
    PHUB_CACHE_RESIDENT = 2   /* DEFAULT: a FIXED slice of w (the last                 */
                              /* PHUB_OPT_L2_RESIDENT bytes of the owned range) is loaded */
                              /* and stored evict-last, so it stays in L2 from round to  */
                              /* round; everything else evict-first.  VGG-19, N = 8:     */
                              /* 0.978 vs 1.003 (BYPASS) vs 1.009 ms (ENABLED): the model */
                              /* (>> 126 MB of L2) never fits, so caching all of w' only */
                              /* crowds L2, a fixed resident slice is hit every round    */
                              /* (R14, profiles/r02_l2/)                       */
};
phub_status phub_set_option(phub_ctx ctx, int32_t option, int64_t value);

const char* phub_status_string(phub_status s);
/* Detail of the last failed call on `ctx`; with ctx == NULL, of the calling
 * thread's last failed phub_init / phub_plan_chunks. */
const char* phub_last_error(phub_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* PHUB_H */
