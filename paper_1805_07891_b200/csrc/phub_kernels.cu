// phub_kernels.cu -- sm_100a kernels of the PHub hot path.
//
// The one hot operation is the fused "tall" aggregation + Nesterov update
// (the thread that sums a chunk across all workers also
// optimizes it; P:783 Nesterov SGD; recurrence S:189, reading R1):
//
//   s  = (((+0.0f + g_0) + g_1) + ...) + g_{N-1}      worker-id order (R3, R4)
//   g  = s * rescale                                  (R2)
//   v' = mu*v + g ;  w' = w - lr*(g + mu*v')
//
// every op rounded separately (__fadd_rn/__fmul_rn/__fsub_rn: no FMA
// contraction, R5; no FTZ, R6).  It is a streaming element-wise update at
// ~0.3 flop/B, so it is HBM-bound: (4N+16) B per element (N gradient reads,
// w and v read and written), no tensor cores (nothing is a contraction).
//
// Kernels:
//   k_flat   owned padded range walked as 256-bit (LDG.E.256/STG.E.256, new on
//            sm_100a) or 128-bit vectors; one-shot grid (one vector per
//            thread, the hardware CTA scheduler hands out 2048-element pieces
//            like PHub's chunk -> core map), or a persistent grid when peer
//            replicas are registered; workers' bases in kernel params.  Bases
//            may be peer-mapped (NVLink loads) and w' may also be stored into
//            peer replicas: the push, the aggregate+optimize and the pull's
//            all-gather fused in one kernel over peer memory.
//   k_blocks block-streamed chain stage (per-block device flags)
//   k_hier   owner-sharded push exchange / hierarchical reduction (one
//            ticket-ordered launch per GPU)
//   k_bulk   TMA-engine staging variant (1-D cp.async.bulk into a smem ring)
//   k_tiles  one CTA per chunk tile (PHub's chunk -> core mapping, P:708-713,
//            with the hardware CTA scheduler as the "core" assigner); worker
//            pointers per (worker, key) for per-key pushes; 128-bit body +
//            scalar tail per tile.
//   k_wide_* ablation of MXNet-style wide aggregation: N-1
//            pairwise passes then a separate optimizer pass; same arithmetic,
//            12(N-1)+20 B/elt instead of 4N+16.
#include <vector>

#include "phub_kernels.cuh"
#include "phub.h"

namespace phub {
namespace {

template <int VEC>
struct alignas(VEC * 4) VecT {
    float x[VEC];
};
using V8 = VecT<8>;
using V4 = VecT<4>;

// ------------------------------------------------------------ memory access
// Gradients are read exactly once per round: non-coherent path, no L1
// allocation, L2 evict-first (the 256-bit form is the one that takes an L2
// eviction-priority qualifier on sm_100a).
__device__ __forceinline__ V8 ld_grad(const V8* p) {
    V8 r;
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]),
          "=f"(r.x[6]), "=f"(r.x[7])
        : "l"(p));
    return r;
}
__device__ __forceinline__ V4 ld_grad(const V4* p) {
    V4 r;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3])
        : "l"(p));
    return r;
}

// Model state (w, v): read then rewritten by the same thread.  ENABLED: no
// L2 hint; BYPASS: evict-first.  (RESIDENT accesses w through a run-time
// policy operand, ld_state_pol below.)
template <int CACHE>
__device__ __forceinline__ V8 ld_state(const V8* p) {
    V8 r;
    if (CACHE == PHUB_CACHE_BYPASS)
        asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                       "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
                     : "l"(p));
    else
        asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                       "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
                     : "l"(p));
    return r;
}
template <int CACHE>
__device__ __forceinline__ V4 ld_state(const V4* p) {
    V4 r;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3])
                 : "l"(p));
    return r;
}

// PHUB_CACHE_RESIDENT: w is loaded and stored with a run-time L2 policy
// operand (createpolicy + .L2::cache_hint), evict-last on the kept slice and
// evict-first elsewhere -- one instruction form for both, so the choice costs
// no registers (a branch between two qualifier forms cost 20).  The policy must
// be warp-uniform: the host rounds keep_from to a whole warp of vectors.
__device__ __forceinline__ uint64_t l2_policy(bool keep) {
    uint64_t p;
    if (keep)
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else
        asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
template <int VEC>
__device__ __forceinline__ VecT<VEC> ld_state_pol(const VecT<VEC>* p, uint64_t pol) {
    VecT<VEC> r;
    if constexpr (VEC == 8)
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                     : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                       "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
                     : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3])
                     : "l"(p), "l"(pol));
    return r;
}
template <int VEC>
__device__ __forceinline__ void st_state_pol(VecT<VEC>* p, const VecT<VEC>& r, uint64_t pol) {
    if constexpr (VEC == 8)
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;"
                     :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]),
                        "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]), "l"(pol) : "memory");
    else
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                     :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "l"(pol)
                     : "memory");
}

// Updated weights: under PHUB_CACHE_ENABLED (and for the kept slice under
// RESIDENT) they are stored L2 evict-last so a pull / the next round is served
// from L2 ("models can be sent directly from cache after being updated",
// P:911); under BYPASS (and outside the kept slice) they stream.
template <int CACHE>
__device__ __forceinline__ void st_w(V8* p, const V8& r) {
    if (CACHE == PHUB_CACHE_BYPASS)
        asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]),
                        "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]) : "memory");
    else
        asm volatile("st.global.L1::no_allocate.L2::evict_last.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                     :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]),
                        "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]) : "memory");
}
template <int CACHE>
__device__ __forceinline__ void st_w(V4* p, const V4& r) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]) : "memory");
}
// Momentum and the test-mode sum are only re-read next round: stream them.
__device__ __forceinline__ void st_stream(V8* p, const V8& r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]),
                    "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]) : "memory");
}
__device__ __forceinline__ void st_stream(V4* p, const V4& r) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]) : "memory");
}

// ----------------------------------------------- stage ordering (chain)
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// An expired wait: counted on the device (timeouts[0]), the value given up on
// recorded (timeouts[1], so the rest of the launch stops waiting for it), and
// the host-mapped error word raised -- the host makes the context
// sticky-failed (PHUB_ERR_SYNC_TIMEOUT) on its next call, so skipped work is
// never reported as a completed round.
__device__ __forceinline__ void record_timeout(uint32_t* timeouts, volatile uint32_t* err_host,
                                               uint32_t value) {
    atomicAdd(timeouts, 1u);
    atomicMax(timeouts + 1, value);
    if (err_host) {
        *err_host = 1u;
        __threadfence_system();
    }
}

// Every CTA waits for the previous stage's flag (bounded); returns false when
// the wait expired (the CTA then skips its work; the timeout is recorded).
__device__ __forceinline__ bool stage_wait(const FlatArgs& a) {
    if (!a.wait_flag) return true;
    __shared__ int ok;
    if (threadIdx.x == 0) {
        // timeouts[0]: expired waits; timeouts[1]: highest wait value given up on,
        // so once one CTA gives up, the rest of the grid does not wait again
        volatile uint32_t* abandoned = a.timeouts + 1;
        const uint64_t t0 = globaltimer_ns();
        int good = 1;
        while (ld_acquire_sys(a.wait_flag) < a.wait_value) {
            if (*abandoned >= a.wait_value) {
                good = 0;
                break;
            }
            if (globaltimer_ns() - t0 > 2000000000ull) {
                record_timeout(a.timeouts, a.err_host, a.wait_value);
                good = 0;
                break;
            }
            __nanosleep(64);
        }
        ok = good;
    }
    __syncthreads();
    return ok != 0;
}

// After all CTAs' stores: the last CTA to finish raises the next stage's flag
// -- unless a CTA of this launch gave up its wait (its work was skipped): then
// the flag stays down, the downstream stage times out too and records its own
// error instead of consuming a stale partial (every CTA still counts itself,
// so the counter resets for the next launch).
__device__ __forceinline__ void stage_signal(const FlatArgs& a) {
    if (!a.signal_flag) return;
    __threadfence_system();                       // this thread's (peer) stores are visible
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t done = atomicAdd(a.cta_counter, 1u);
        if (done == gridDim.x - 1) {
            *a.cta_counter = 0;
            // every other CTA's atomicMax (if any) preceded its fence + counter add
            const bool abandoned = a.wait_flag && atomicAdd(a.timeouts + 1, 0u) >= a.wait_value;
            __threadfence_system();
            if (!abandoned) st_release_sys(a.signal_flag, a.signal_value);
        }
    }
}

// ------------------------------------------------------------- arithmetic
// Nesterov step on one element, each op rounded separately (R5).
__device__ __forceinline__ void nag(float s, float& w, float& v, float lr, float mu,
                                    float rescale) {
    const float g = __fmul_rn(s, rescale);
    const float vn = __fadd_rn(__fmul_rn(mu, v), g);
    const float t3 = __fadd_rn(g, __fmul_rn(mu, vn));
    w = __fsub_rn(w, __fmul_rn(lr, t3));
    v = vn;
}

// ------------------------------------------------------------ flat kernel
// NW > 0: worker count fixed at compile time; NW == 0: any count <= 64, in
// groups of 8 loads issued before their in-order adds.
// One vector position i of the owned range: N gradient loads, in-order sum,
// Nesterov, stores (local w, v, optional s, optional peer replicas).
template <int NW, int VEC, int CACHE, bool AGG>
__device__ __forceinline__ void flat_body(const FlatArgs& a, uint64_t i) {
    using V = VecT<VEC>;
    V* __restrict__ w = reinterpret_cast<V*>(a.w + a.begin);
    V* __restrict__ v = reinterpret_cast<V*>(a.v + a.begin);
    V* __restrict__ sa = AGG ? reinterpret_cast<V*>(a.agg + a.begin) : nullptr;
    {
        // RESIDENT: vectors >= keep_from are the L2-kept slice of w (warp-uniform)
        const uint64_t wpol = CACHE == PHUB_CACHE_RESIDENT ? l2_policy(i >= a.keep_from) : 0;
        float acc[VEC];
        if constexpr (NW > 0) {
            V gv[NW];
#pragma unroll
            for (int k = 0; k < NW; ++k)
                gv[k] = ld_grad(reinterpret_cast<const V*>(a.g[k] + a.begin) + i);
#pragma unroll
            for (int j = 0; j < VEC; ++j) {
                float s = __fadd_rn(0.0f, gv[0].x[j]);
#pragma unroll
                for (int k = 1; k < NW; ++k) s = __fadd_rn(s, gv[k].x[j]);
                acc[j] = s;
            }
        } else {
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc[j] = 0.0f;
            for (int k0 = 0; k0 < a.nw; k0 += 8) {
                V gv[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k0 + k < a.nw)
                        gv[k] = ld_grad(reinterpret_cast<const V*>(a.g[k0 + k] + a.begin) + i);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (k0 + k < a.nw) {
#pragma unroll
                        for (int j = 0; j < VEC; ++j) acc[j] = __fadd_rn(acc[j], gv[k].x[j]);
                    }
            }
        }
        constexpr int C_OUT = CACHE == PHUB_CACHE_RESIDENT ? PHUB_CACHE_BYPASS : CACHE;
        V wv = CACHE == PHUB_CACHE_RESIDENT ? ld_state_pol<VEC>(w + i, wpol) : ld_state<C_OUT>(w + i);
        V vv = ld_state<C_OUT>(v + i);
        V sv;
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            sv.x[j] = acc[j];
            nag(acc[j], wv.x[j], vv.x[j], a.lr, a.mu, a.rescale);
        }
        if constexpr (CACHE == PHUB_CACHE_RESIDENT)
            st_state_pol<VEC>(w + i, wv, wpol);           // kept slice: evict-last, stays resident
        else
            st_w<C_OUT>(w + i, wv);
        st_stream(v + i, vv);
        if constexpr (AGG) st_stream(sa + i, sv);
        // fused pull: w' straight into every registered (peer) replica over NVLink
        for (int r = 0; r < a.nrep; ++r)
            reinterpret_cast<V*>(a.rep[r] + a.begin)[i] = wv;
    }
}

// Grid-stride over vectors: with a grid covering the range (one-shot, the
// default) every thread handles one vector; with a persistent grid (SMs x
// resident CTAs) the CTAs sweep the range together.
template <int NW, int VEC, int CACHE, bool AGG>
__device__ __forceinline__ void flat_loop(const FlatArgs& a) {
    const uint64_t n = (a.end - a.begin) / VEC;
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride)
        flat_body<NW, VEC, CACHE, AGG>(a, i);
    if (a.nrep) __threadfence_system();   // peer stores performed before the grid retires
}

template <int NW, int VEC, int CACHE, bool AGG>
__global__ void __launch_bounds__(kThreads) k_flat(const __grid_constant__ FlatArgs a) {
    if (stage_wait(a)) flat_loop<NW, VEC, CACHE, AGG>(a);
    stage_signal(a);
}

// ---------------------------------------------------------- chunk tiles
template <int NW, bool AGG>
__global__ void __launch_bounds__(kThreads) k_tiles(const __grid_constant__ TileArgs a) {
    for (uint64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const Tile tl = a.tiles[t];
        const int nw = NW > 0 ? NW : a.nw;
        // Vector body only if every stream of this tile is 16-B aligned.
        bool aligned = (tl.off % 4) == 0;
        for (int k = 0; k < nw; ++k)
            aligned &= ((a.base[(uint64_t)k * a.K + tl.key] + 4 * tl.off) % 16) == 0;
        const uint32_t nvec = aligned ? tl.len / 4 : 0;
        float* w = a.w + tl.off;
        float* v = a.v + tl.off;
        for (uint32_t j = threadIdx.x; j < nvec; j += kThreads) {
            float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            if constexpr (NW > 0) {
                V4 gv[NW];
#pragma unroll
                for (int k = 0; k < NW; ++k)
                    gv[k] = ld_grad(reinterpret_cast<const V4*>(
                                        a.base[(uint64_t)k * a.K + tl.key] + 4 * tl.off) + j);
#pragma unroll
                for (int k = 0; k < NW; ++k)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[e] = __fadd_rn(acc[e], gv[k].x[e]);
            } else {
                for (int k = 0; k < nw; ++k) {
                    const V4 gk = ld_grad(reinterpret_cast<const V4*>(
                                              a.base[(uint64_t)k * a.K + tl.key] + 4 * tl.off) + j);
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[e] = __fadd_rn(acc[e], gk.x[e]);
                }
            }
            V4 wv = ld_state<PHUB_CACHE_ENABLED>(reinterpret_cast<const V4*>(w) + j);
            V4 vv = ld_state<PHUB_CACHE_ENABLED>(reinterpret_cast<const V4*>(v) + j);
            V4 sv;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                sv.x[e] = acc[e];
                nag(acc[e], wv.x[e], vv.x[e], a.lr, a.mu, a.rescale);
            }
            st_w<PHUB_CACHE_ENABLED>(reinterpret_cast<V4*>(w) + j, wv);
            st_stream(reinterpret_cast<V4*>(v) + j, vv);
            if constexpr (AGG) st_stream(reinterpret_cast<V4*>(a.agg + tl.off) + j, sv);
        }
        // scalar tail (short last chunk of a key, or a misaligned tile)
        for (uint32_t e = nvec * 4 + threadIdx.x; e < tl.len; e += kThreads) {
            float s = 0.0f;
            for (int k = 0; k < nw; ++k) {
                const float* gk = reinterpret_cast<const float*>(
                    a.base[(uint64_t)k * a.K + tl.key] + 4 * tl.off);
                s = __fadd_rn(s, __ldg(gk + e));
            }
            float wv = w[e], vv = v[e];
            nag(s, wv, vv, a.lr, a.mu, a.rescale);
            w[e] = wv;
            v[e] = vv;
            if constexpr (AGG) a.agg[tl.off + e] = s;
        }
    }
}

// ---------------------------------------------- partial (prefix) sum only
// One stage of the chained exchange: the worker-order prefix of this rank's
// workers (the first source may be the incoming partial of the previous
// rank), stored -- typically over NVLink -- into the next rank's buffer.
template <int NW>
__global__ void __launch_bounds__(kThreads) k_prefix(const __grid_constant__ FlatArgs a,
                                                     float* __restrict__ dst) {
    const bool go = stage_wait(a);
    const uint64_t n = go ? (a.end - a.begin) / 8 : 0;
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
        const int nw = NW > 0 ? NW : a.nw;
        for (int k0 = 0; k0 < nw; k0 += 8) {
            V8 gv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < nw) gv[k] = ld_grad(reinterpret_cast<const V8*>(a.g[k0 + k] + a.begin) + i);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < nw) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], gv[k].x[j]);
                }
        }
        V8 out;
#pragma unroll
        for (int j = 0; j < 8; ++j) out.x[j] = acc[j];
        reinterpret_cast<V8*>(dst + a.begin)[i] = out;
    }
    __threadfence_system();
    stage_signal(a);                              // held back if any CTA's wait expired
}

// ------------------------------------------- block-streaming chain stages
// One persistent launch per stage and round.  CTA i walks blocks i, i+grid, ...
// of `a.block` elements; per block it waits for the upstream stage's flag
// (a.wait_flag[b], system-scope acquire, bounded), reads its sources, and
// raises a.signal_flag[b] (system-scope release) once the block's stores are
// performed.  The downstream stage therefore starts on block b while this one
// still works on later blocks (streaming aggregation) -- no launch per
// piece.  Sources are read with coherent loads (not the .nc path): the
// upstream partial is written by another GPU while this kernel runs.
__device__ __forceinline__ V8 ld_coherent(const V8* p) {
    V8 r;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                   "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
                 : "l"(p) : "memory");
    return r;
}

// One 256-bit vector i of a block-streamed stage: the worker-order sum of the
// sources, then either the fused Nesterov (w, v, replicas) or the partial sum
// stored into dst.
template <int NW, bool NAG>
__device__ __forceinline__ void blocks_body(const FlatArgs& a, float* __restrict__ dst, uint64_t i) {
    const int nw = NW > 0 ? NW : a.nw;
    float acc[8];
    if constexpr (NW > 0) {
        V8 gv[NW];
#pragma unroll
        for (int k = 0; k < NW; ++k) gv[k] = ld_coherent(reinterpret_cast<const V8*>(a.g[k]) + i);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float s = __fadd_rn(0.0f, gv[0].x[j]);
#pragma unroll
            for (int k = 1; k < NW; ++k) s = __fadd_rn(s, gv[k].x[j]);
            acc[j] = s;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
        for (int k0 = 0; k0 < nw; k0 += 8) {
            V8 gv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < nw) gv[k] = ld_coherent(reinterpret_cast<const V8*>(a.g[k0 + k]) + i);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < nw) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], gv[k].x[j]);
                }
        }
    }
    V8 out;
    if constexpr (NAG) {
        V8* w = reinterpret_cast<V8*>(a.w);
        V8* v = reinterpret_cast<V8*>(a.v);
        // read once per round: evict-first, so an incoming partial keeps its L2 lines
        V8 wv = ld_state<PHUB_CACHE_BYPASS>(w + i);
        V8 vv = ld_state<PHUB_CACHE_BYPASS>(v + i);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            out.x[j] = acc[j];
            nag(acc[j], wv.x[j], vv.x[j], a.lr, a.mu, a.rescale);
        }
        st_stream(w + i, wv);     // the pull is the replica stores below: keep L2
        st_stream(v + i, vv);     // for the incoming partial, not for w'
        if (a.agg) st_stream(reinterpret_cast<V8*>(a.agg) + i, out);
        for (int r = 0; r < a.nrep; ++r) reinterpret_cast<V8*>(a.rep[r])[i] = wv;
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) out.x[j] = acc[j];
        reinterpret_cast<V8*>(dst)[i] = out;
    }
}

// Bounded wait of one thread for *flag >= value (0 = gave up, counted).
__device__ __forceinline__ int wait_bounded(const FlatArgs& a, const uint32_t* flag, uint32_t value) {
    if (ld_acquire_sys(flag) >= value) return 1;
    volatile uint32_t* abandoned = a.timeouts + 1;
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(flag) < value) {
        if (*abandoned >= value) return 0;
        if (globaltimer_ns() - t0 > 2000000000ull) {
            record_timeout(a.timeouts, a.err_host, value);
            return 0;
        }
        __nanosleep(100);
    }
    return 1;
}

// CTA-granular: each CTA takes a block (multiple of 2048 elements) per ticket.
template <int NW, bool NAG>
__global__ void __launch_bounds__(kThreads) k_blocks(const __grid_constant__ FlatArgs a,
                                                     float* __restrict__ dst) {
    const uint64_t B = a.block;
    const uint64_t b0 = a.begin / B, b1 = (a.end + B - 1) / B;
    __shared__ uint64_t s_blk;
    __shared__ int s_go;
    for (;;) {
        // dynamic ticket: CTAs take blocks in global order as they free up, so
        // this stage's front follows the upstream stage's front closely
        if (threadIdx.x == 0) {
            const uint64_t blk = b0 + atomicAdd(a.ticket, 1u);
            int go = 1;
            if (blk < b1 && a.wait_flag) go = wait_bounded(a, a.wait_flag + blk, a.wait_value);
            s_blk = blk;
            s_go = go;
        }
        __syncthreads();
        const uint64_t blk = s_blk;
        const bool go = s_go != 0;
        if (blk >= b1) break;
        const uint64_t lo = (blk * B > a.begin ? blk * B : a.begin) / 8;
        const uint64_t hi = ((blk + 1) * B < a.end ? (blk + 1) * B : a.end) / 8;
        for (uint64_t i = lo + threadIdx.x; go && i < hi; i += kThreads) blocks_body<NW, NAG>(a, dst, i);
        // bar.sync (also retires s_blk / s_go before the next ticket) then one
        // system-scope fence: cumulative over the CTA's stores (the
        // cooperative-groups grid-sync pattern)
        __syncthreads();
        if (threadIdx.x == 0 && a.signal_flag && go) {   // a skipped block is never signalled
            __threadfence_system();
            st_release_sys(a.signal_flag + blk, a.signal_value);
        }
    }
    if (NAG && a.nrep) __threadfence_system();
    // the last CTA out resets the tickets for the next launch (stream-ordered)
    if (threadIdx.x == 0 && atomicAdd(a.ticket + 1, 1u) == gridDim.x - 1) {
        a.ticket[0] = 0;
        a.ticket[1] = 0;
    }
}

template <bool NAG>
void* pick_blocks(int nw) {
    switch (nw) {
        case 1: return (void*)k_blocks<1, NAG>;
        case 2: return (void*)k_blocks<2, NAG>;
        case 3: return (void*)k_blocks<3, NAG>;
        case 4: return (void*)k_blocks<4, NAG>;
        case 5: return (void*)k_blocks<5, NAG>;
        case 6: return (void*)k_blocks<6, NAG>;
        case 7: return (void*)k_blocks<7, NAG>;
        case 8: return (void*)k_blocks<8, NAG>;
        case 9: return (void*)k_blocks<9, NAG>;
        default: return (void*)k_blocks<0, NAG>;
    }
}

// ------------------------------------------- hierarchical reduction (NEXT-4)
// PHub's rack deployment: each GPU is one rack's PBox holding its
// P workers' gradients.  One persistent launch per rack and round walks a
// ticket-ordered item list; for block index j the items are
//   produce(o, j), o != rack:  S_rack = worker-order sum of the local workers
//                              over owner o's block j, stored straight into o's
//                              inbox over NVLink, then o's flag [j][rack] raised;
//   consume(j):                once every other rack's flag for block j is up,
//                              s = ((+0 + S_0) + S_1) + ... + S_{R-1} in rack
//                              order (own S computed here), Nesterov, w' stored
//                              locally and into every peer replica.
// Deadlock-free: produce items never wait, and tickets are taken in item order,
// so every produce item a waiting consume item needs has already been taken by
// a running CTA on its rack.
// acc = ((+0 + g_0) + g_1) + ... over the local workers (ZERO), or acc += g_0, g_1, ...
// in order onto a running sum (!ZERO: the flat worker-order exchange)
template <int NW, bool ZERO = true>
__device__ __forceinline__ void local_sum(const HierArgs& a, uint64_t i, float acc[8]) {
    const int nw = NW > 0 ? NW : a.nw;
    if constexpr (ZERO) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
    }
    if constexpr (NW > 0) {
        // batches of 4 loads keep the kernel at <= 64 registers (4 CTAs/SM), so a
        // CTA stalled in its per-block fence leaves three others streaming
#pragma unroll
        for (int k0 = 0; k0 < NW; k0 += 4) {
            V8 gv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k0 + k < NW) gv[k] = ld_grad(reinterpret_cast<const V8*>(a.g[k0 + k]) + i);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k0 + k < NW) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], gv[k].x[j]);
                }
        }
    } else {
        for (int k0 = 0; k0 < nw; k0 += 8) {
            V8 gv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < nw) gv[k] = ld_grad(reinterpret_cast<const V8*>(a.g[k0 + k]) + i);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < nw) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], gv[k].x[j]);
                }
        }
    }
}

// Thread 0: bounded wait for *f >= epoch (0 = gave up or abandoned), as sched_wait.
__device__ __forceinline__ int hier_wait(const HierArgs& a, const uint32_t* f, const uint64_t t0) {
    volatile uint32_t* abandoned = a.timeouts + 1;
    while (ld_acquire_sys(f) < a.epoch) {
        if (*abandoned >= a.epoch) return 0;
        if (globaltimer_ns() - t0 > 2000000000ull) {
            record_timeout(a.timeouts, a.err_host, a.epoch);
            return 0;
        }
        __nanosleep(100);
    }
    return 1;
}

template <int NW, bool WO>
__global__ void __launch_bounds__(kThreads, 3) k_hier(const __grid_constant__ HierArgs a) {
    const uint64_t B = a.block;
    const int R = a.R;
    uint64_t J = 0;                                    // blocks of the largest owner range
    for (int o = 0; o < R; ++o) {
        const uint64_t n = (a.own_end[o] - a.own_begin[o] + B - 1) / B;
        J = n > J ? n : J;
    }
    const uint64_t items = J * (uint64_t)R;
    // in-kernel round barrier (a.device_barrier; the k_sched scheme): flags
    // [J*R + q] "rank q's replica is free", [J*R + R + q] "rank q is done
    // storing into this rank's replica"
    const uint64_t bar = J * (uint64_t)R;
    __shared__ uint64_t s_item;
    __shared__ int ok;
    __shared__ int s_free;
    if (threadIdx.x == 0) s_free = !a.device_barrier;
    if (a.device_barrier && blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = 0; q < R; ++q)
            if (q != a.rack) st_release_sys(a.peer_flags[q] + bar + a.rack, a.epoch);
    __syncthreads();
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(a.ticket, 1u);
        __syncthreads();
        const uint64_t t = s_item;
        if (t >= items) break;
        const uint64_t j = t / R;
        const int k = (int)(t % R);
        if (k < R - 1) {                               // ---- produce(o, j)
            const int o = (a.rack + 1 + k) % R;
            const uint64_t lo = a.own_begin[o] + j * B;
            const uint64_t hi = lo + B < a.own_end[o] ? lo + B : a.own_end[o];
            if (lo < hi) {
                if constexpr (WO) {
                    // worker-order exchange: each local worker's raw slice goes to o's
                    // inbox (worker k at +k*L_o); o sums all workers in worker order
                    const int nw = NW > 0 ? NW : a.nw;
                    const uint64_t L = a.own_end[o] - a.own_begin[o];
                    for (uint64_t i = lo / 8 + threadIdx.x; i < hi / 8; i += kThreads)
                        for (int k0 = 0; k0 < nw; k0 += 4) {
                            V8 gv[4];
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                if (k0 + k < nw)
                                    gv[k] = ld_grad(reinterpret_cast<const V8*>(a.g[k0 + k]) + i);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                if (k0 + k < nw)
                                    reinterpret_cast<V8*>(a.peer_inbox[o] + (k0 + k) * L)[i] = gv[k];
                        }
                } else {
                    V8* dst = reinterpret_cast<V8*>(a.peer_inbox[o]);
                    for (uint64_t i = lo / 8 + threadIdx.x; i < hi / 8; i += kThreads) {
                        float acc[8];
                        local_sum<NW>(a, i, acc);
                        V8 out;
#pragma unroll
                        for (int e = 0; e < 8; ++e) out.x[e] = acc[e];
                        dst[i] = out;
                    }
                }
                __syncthreads();                       // bar.sync + one fence (cumulative)
                if (threadIdx.x == 0) {
                    __threadfence_system();
                    st_release_sys(a.peer_flags[o] + j * R + a.rack, a.epoch);
                }
            }
        } else {                                       // ---- consume(j)
            const uint64_t lo = a.own_begin[a.rack] + j * B;
            const uint64_t hi = lo + B < a.own_end[a.rack] ? lo + B : a.own_end[a.rack];
            if (lo < hi) {
                if (threadIdx.x == 0) {
                    int good = 1;
                    const uint64_t t0 = globaltimer_ns();
                    for (int q = 0; q < R && good; ++q)
                        if (q != a.rack) good = hier_wait(a, a.flags + j * R + q, t0);
                    // w' goes into every peer replica: each must be free (barrier)
                    if (good && !s_free) {
                        for (int q = 0; q < R && good; ++q)
                            if (q != a.rack) good = hier_wait(a, a.flags + bar + q, t0);
                        s_free = good;
                    }
                    ok = good;
                }
                __syncthreads();
                if (ok) {
                    V8* w = reinterpret_cast<V8*>(a.w);
                    V8* v = reinterpret_cast<V8*>(a.v);
                    for (uint64_t i = lo / 8 + threadIdx.x; i < hi / 8; i += kThreads) {
                        float acc[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
                        for (int q = 0; q < R; ++q) {
                            if constexpr (WO) {                    // worker order (R3)
                                if (q == a.rack) {
                                    local_sum<NW, false>(a, i, acc);
                                } else {
                                    const int nw = NW > 0 ? NW : a.nw;
                                    const uint64_t L = a.own_end[a.rack] - a.own_begin[a.rack];
                                    for (int k = 0; k < nw; ++k) {
                                        const V8 rv = ld_coherent(
                                            reinterpret_cast<const V8*>(a.inbox[q] + k * L) + i);
#pragma unroll
                                        for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], rv.x[e]);
                                    }
                                }
                            } else if (q == a.rack) {              // rack order (R17)
                                float own[8];
                                local_sum<NW>(a, i, own);          // S_rack, from +0
#pragma unroll
                                for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], own[e]);
                            } else {
                                const V8 rv = ld_coherent(reinterpret_cast<const V8*>(a.inbox[q]) + i);
#pragma unroll
                                for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], rv.x[e]);
                            }
                        }
                        V8 wv = ld_state<PHUB_CACHE_BYPASS>(w + i);   // read once: evict-first
                        V8 vv = ld_state<PHUB_CACHE_BYPASS>(v + i);
                        V8 sv;
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            sv.x[e] = acc[e];
                            nag(acc[e], wv.x[e], vv.x[e], a.lr, a.mu, a.rescale);
                        }
                        st_stream(w + i, wv);
                        st_stream(v + i, vv);
                        if (a.agg) st_stream(reinterpret_cast<V8*>(a.agg) + i, sv);
                        for (int r = 0; r < a.nrep; ++r) reinterpret_cast<V8*>(a.rep[r])[i] = wv;
                    }
                }
            }
        }
        __syncthreads();                               // s_item / ok retire before the next item
    }
    if (a.nrep) __threadfence_system();
    if (threadIdx.x == 0 && atomicAdd(a.ticket + 1, 1u) == gridDim.x - 1) {
        if (a.device_barrier) {                        // end half (see k_sched)
            __threadfence_system();
            const bool abandoned = *(volatile uint32_t*)(a.timeouts + 1) >= a.epoch;
            for (int q = 0; q < R && !abandoned; ++q)
                if (q != a.rack) st_release_sys(a.peer_flags[q] + bar + R + a.rack, a.epoch);
            const uint64_t t0 = globaltimer_ns();
            for (int q = 0; q < R; ++q)
                if (q != a.rack && !hier_wait(a, a.flags + bar + R + q, t0)) break;
        }
        a.ticket[0] = 0;
        a.ticket[1] = 0;
    }
}

template <bool WO>
void* pick_hier_wo(int nw) {
    switch (nw) {
        case 1: return (void*)k_hier<1, WO>;
        case 2: return (void*)k_hier<2, WO>;
        case 4: return (void*)k_hier<4, WO>;
        case 8: return (void*)k_hier<8, WO>;
        default: return (void*)k_hier<0, WO>;
    }
}
void* pick_hier(int nw, bool wo) { return wo ? pick_hier_wo<true>(nw) : pick_hier_wo<false>(nw); }

// ------------------------------------------------ scheduled exchange (8.6)
// One persistent launch per GPU walks the host-built item program in ticket
// order (phub_sched_plan): RAW_PUSH, CHAIN (first / middle / last stage of the
// rank-by-rank worker-order partial sum), CONSUME_RAW, CONSUME_FINAL.  Every
// item waits only on items of other ranks with strictly smaller keys in the
// shared order, and tickets are taken in that order, so a waited-on item has
// always been taken by a running CTA: no deadlock with co-resident CTAs (the
// k_hier argument).  Waits are bounded; a skipped item never
// raises its flag, so downstream stages time out too.

// acc += g_0, g_1, ... (this rank's workers, in order), batches of 4 loads
template <int NW>
__device__ __forceinline__ void sched_local(const SchedArgs& a, uint64_t i, float acc[8]) {
    const int nw = NW > 0 ? NW : a.nw;
#pragma unroll
    for (int k0 = 0; k0 < (NW > 0 ? NW : kMaxWorkers); k0 += 4) {
        if (k0 >= nw) break;
        V8 gv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k0 + k < nw) gv[k] = ld_grad(reinterpret_cast<const V8*>(a.g[k0 + k]) + i);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k0 + k < nw) {
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], gv[k].x[j]);
            }
    }
}

// s = acc: Nesterov on vector i, w' stored locally and into every replica
__device__ __forceinline__ void sched_nag(const SchedArgs& a, uint64_t i, const float acc[8]) {
    V8* w = reinterpret_cast<V8*>(a.w);
    V8* v = reinterpret_cast<V8*>(a.v);
    V8 wv = ld_state<PHUB_CACHE_BYPASS>(w + i);
    V8 vv = ld_state<PHUB_CACHE_BYPASS>(v + i);
    V8 sv;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        sv.x[e] = acc[e];
        float s = acc[e];
        nag(s, wv.x[e], vv.x[e], a.lr, a.mu, a.rescale);
    }
    st_stream(w + i, wv);
    st_stream(v + i, vv);
    if (a.agg) st_stream(reinterpret_cast<V8*>(a.agg) + i, sv);
    for (int r = 0; r < a.nrep; ++r) reinterpret_cast<V8*>(a.rep[r])[i] = wv;
}

// Thread 0: bounded wait for flags[f] >= epoch (0 = gave up or abandoned)
__device__ __forceinline__ int sched_wait(const SchedArgs& a, const uint32_t* f, const uint64_t t0) {
    volatile uint32_t* abandoned = a.timeouts + 1;
    while (ld_acquire_sys(f) < a.epoch) {
        if (*abandoned >= a.epoch) return 0;
        if (globaltimer_ns() - t0 > 2000000000ull) {
            record_timeout(a.timeouts, a.err_host, a.epoch);
            return 0;
        }
        __nanosleep(100);
    }
    return 1;
}

template <int NW>
__global__ void __launch_bounds__(kThreads, 3) k_sched(const __grid_constant__ SchedArgs a) {
    __shared__ uint64_t s_t;
    __shared__ int s_ok;
    __shared__ int s_free;                             // every peer replica writable (barrier)
    const uint32_t* my_flags = a.flags[a.rank];
    // In-kernel round barrier (a.bar >= 0), start half: this launch is stream-ordered
    // after this rank's reads of its replica from the previous round, so it tells
    // every peer "my replica is free for this epoch"; a CTA waits for every peer's
    // such flag before its first replica store (below).
    if (threadIdx.x == 0) s_free = a.bar < 0;
    if (a.bar >= 0 && blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = 0; q < a.R; ++q)
            if (q != a.rank) st_release_sys(a.flags[q] + a.bar + a.rank, a.epoch);
    __syncthreads();
    // two lanes with their own tickets: producers (RAW_PUSH, CHAIN) never wait on
    // a consumer, so consumers blocked on late data cannot stall the chain
    const bool cons_lane = (int)blockIdx.x >= a.grid_prod;
    uint32_t* const tk = cons_lane ? a.ticket + 2 : a.ticket;
    const uint64_t first = cons_lane ? a.nprod : 0, last = cons_lane ? a.nitems : a.nprod;
    for (;;) {
        if (threadIdx.x == 0) s_t = first + atomicAdd(tk, 1u);
        __syncthreads();
        const uint64_t t = s_t;
        if (t >= last) break;
        const SchedItem it = a.items[t];
        if (threadIdx.x == 0) {
            int good = 1;
            const uint64_t t0 = globaltimer_ns();
            if (a.trace) {
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                a.trace[4 * t] = t0;
                a.trace[4 * t + 3] = ((uint64_t)blockIdx.x << 32) | smid;
            }
            if (it.type == PHUB_ITEM_CONSUME_RAW) {
                for (int q = 0; q < a.R && good; ++q)
                    if (q != a.rank) good = sched_wait(a, my_flags + it.wait_flag + q, t0);
            } else if (it.wait_flag != kNoFlag) {
                good = sched_wait(a, my_flags + it.wait_flag, t0);
            }
            // a Nesterov item stores w' into every peer replica: they must be free
            if (good && !s_free && it.dst < 0) {
                for (int q = 0; q < a.R && good; ++q)
                    if (q != a.rank) good = sched_wait(a, my_flags + a.bar + q, t0);
                s_free = good;
            }
            s_ok = good;
            if (a.trace) a.trace[4 * t + 1] = globaltimer_ns();
        }
        __syncthreads();
        const bool ok = s_ok != 0;
        const uint64_t lo = it.lo / 8, hi = it.hi / 8;
        if (ok) {
            if (it.type == PHUB_ITEM_RAW_PUSH) {
                // worker k of this rank -> slot (rank, k) of owner dst's raw part
                float* dst = a.raw_inbox[it.dst];
                const int nw = NW > 0 ? NW : a.nw;
                if constexpr (NW == 1 || NW == 2) {
                    // few workers: U = 4 / NW vectors per thread and iteration, so four
                    // NVLink stores are in flight per thread (G = 8: one worker per GPU)
                    constexpr int U = 4 / NW;
                    for (uint64_t i0 = lo + threadIdx.x; i0 < hi; i0 += U * kThreads) {
                        V8 gv[U][NW];
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int k = 0; k < NW; ++k)
                                if (i0 + u * kThreads < hi)
                                    gv[u][k] = ld_grad(reinterpret_cast<const V8*>(a.g[k]) + i0 +
                                                       u * kThreads);
#pragma unroll
                        for (int u = 0; u < U; ++u)
#pragma unroll
                            for (int k = 0; k < NW; ++k) {
                                const uint64_t i = i0 + u * kThreads;
                                if (i < hi)
                                    *reinterpret_cast<V8*>(dst + ((uint64_t)(a.rank * NW + k) * it.len +
                                                                  8 * i - it.base)) = gv[u][k];
                            }
                    }
                } else
                for (uint64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
                    const uint64_t x = 8 * i - it.base;
                    for (int k0 = 0; k0 < nw; k0 += 4) {
                        V8 gv[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (k0 + k < nw) gv[k] = ld_grad(reinterpret_cast<const V8*>(a.g[k0 + k]) + i);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (k0 + k < nw)
                                *reinterpret_cast<V8*>(
                                    dst + ((uint64_t)(a.rank * nw + k0 + k) * it.len + x)) = gv[k];
                    }
                }
            } else if (it.type == PHUB_ITEM_CHAIN) {
                const bool first = it.wait_flag == kNoFlag;
                const V8* in = reinterpret_cast<const V8*>(a.inbox[a.rank]);
                for (uint64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
                    float acc[8];
                    if (first) {
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[e] = 0.0f;           // +0 (R4)
                    } else {
                        const V8 p = ld_coherent(in + i);                      // ranks 0..p-1
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[e] = p.x[e];
                    }
                    sched_local<NW>(a, i, acc);
                    if (it.dst >= 0) {
                        V8 out;
#pragma unroll
                        for (int e = 0; e < 8; ++e) out.x[e] = acc[e];
                        reinterpret_cast<V8*>(a.inbox[it.dst])[i] = out;
                    } else {
                        sched_nag(a, i, acc);
                    }
                }
            } else if (it.type == PHUB_ITEM_CONSUME_RAW) {
                const int nw = NW > 0 ? NW : a.nw;
                const float* rin = a.raw_inbox[a.rank];
                for (uint64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
                    const uint64_t x = 8 * i - it.base;
                    float acc[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
                    for (int q = 0; q < a.R; ++q) {                        // worker order (R3)
                        if (q == a.rank) {
                            sched_local<NW>(a, i, acc);
                        } else {
                            for (int k = 0; k < nw; ++k) {
                                const V8 r = ld_coherent(reinterpret_cast<const V8*>(
                                    rin + ((uint64_t)(q * nw + k) * it.len + x)));
#pragma unroll
                                for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], r.x[e]);
                            }
                        }
                    }
                    sched_nag(a, i, acc);
                }
            } else {                                                   // CONSUME_FINAL
                const V8* in = reinterpret_cast<const V8*>(a.inbox[a.rank]);
                for (uint64_t i = lo + threadIdx.x; i < hi; i += kThreads) {
                    const V8 p = ld_coherent(in + i);
                    float acc[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) acc[e] = p.x[e];
                    sched_nag(a, i, acc);
                }
            }
        }
        __syncthreads();                               // bar.sync + one fence (cumulative)
        if (threadIdx.x == 0 && ok && it.dst >= 0 && it.signal_flag != kNoFlag) {
            __threadfence_system();
            st_release_sys(a.flags[it.dst] + it.signal_flag, a.epoch);
        }
        if (threadIdx.x == 0 && a.trace) a.trace[4 * t + 2] = globaltimer_ns();
    }
    if (a.nrep) __threadfence_system();
    if (threadIdx.x == 0 && atomicAdd(a.ticket + 1, 1u) == gridDim.x - 1) {
        if (a.bar >= 0) {
            // end half: every CTA's replica stores are performed (each fenced before
            // counting itself); tell every peer, then wait until every peer has done
            // so -- the launch completes only once this rank's replica is complete
            // and every peer has finished reading this round's inboxes.  A peer whose
            // launch gave up never raises its flag, so this wait expires too.
            __threadfence_system();
            // a launch that skipped work (a wait given up) never reports done: its
            // peers' end waits expire and fail loudly instead of trusting stale w'
            const bool abandoned = *(volatile uint32_t*)(a.timeouts + 1) >= a.epoch;
            for (int q = 0; q < a.R && !abandoned; ++q)
                if (q != a.rank) st_release_sys(a.flags[q] + a.bar + a.R + a.rank, a.epoch);
            const uint64_t t0 = globaltimer_ns();
            for (int q = 0; q < a.R; ++q)
                if (q != a.rank && !sched_wait(a, my_flags + a.bar + a.R + q, t0)) break;
        }
        a.ticket[0] = 0;
        a.ticket[1] = 0;
        a.ticket[2] = 0;
    }
}

void* pick_sched(int nw) {
    switch (nw) {
        case 1: return (void*)k_sched<1>;
        case 2: return (void*)k_sched<2>;
        case 4: return (void*)k_sched<4>;
        case 8: return (void*)k_sched<8>;
        default: return (void*)k_sched<0>;
    }
}

// ------------------------------------------------ bulk-copy (TMA) staging
// Variant with the loads taken off the register file: one producer thread per
// CTA streams each tile's N gradient slices and the w, v slices into a
// shared-memory ring with 1-D bulk async copies (cp.async.bulk, SASS UBLKCP,
// completion counted on an mbarrier), while 8 consumer warps compute from
// shared memory and store w', v' with 256-bit STG.  Same arithmetic and order.
constexpr int kBulkTile = 2048;                  // elements per stream per stage (8 KB)
constexpr int kBulkStages = 2;
constexpr int kBulkConsumers = 256;              // 8 warps; +1 producer warp

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}"
        :: "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;"
        :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}

template <int NW, bool AGG>
__global__ void __launch_bounds__(kBulkConsumers + 32, 1) k_bulk(const __grid_constant__ FlatArgs a) {
    constexpr int S = NW + 2;                           // streams per tile: grads, w, v
    extern __shared__ __align__(128) float smem[];      // [stage][stream][kBulkTile]
    __shared__ uint64_t full[kBulkStages], empty[kBulkStages];
    const uint64_t n = a.end - a.begin;
    const uint64_t ntiles = (n + kBulkTile - 1) / kBulkTile;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kBulkStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kBulkConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kBulkConsumers / 32) {                   // ---- producer warp
        if ((threadIdx.x & 31) == 0) {
            uint64_t pol_first;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
            int stage = 0;
            uint32_t phase = 0;
            for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(&empty[stage], phase ^ 1);
                const uint64_t off = a.begin + t * kBulkTile;
                const uint32_t len = (uint32_t)(a.end - off < (uint64_t)kBulkTile ? a.end - off : (uint64_t)kBulkTile);
                const uint32_t bytes = len * 4;
                mbar_expect_tx(&full[stage], bytes * S);
                float* st = smem + (size_t)stage * S * kBulkTile;
#pragma unroll
                for (int k = 0; k < NW; ++k)
                    bulk_g2s(st + k * kBulkTile, a.g[k] + off, bytes, &full[stage], pol_first);
                bulk_g2s(st + NW * kBulkTile, a.w + off, bytes, &full[stage], pol_first);
                bulk_g2s(st + (NW + 1) * kBulkTile, a.v + off, bytes, &full[stage], pol_first);
                if (++stage == kBulkStages) { stage = 0; phase ^= 1; }
            }
        }
        return;
    }
    // ---- consumer warps: 8 elements per thread per tile (one 256-bit vector)
    int stage = 0;
    uint32_t phase = 0;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&full[stage], phase);
        const uint64_t off = a.begin + t * kBulkTile;
        const uint32_t len = (uint32_t)(a.end - off < (uint64_t)kBulkTile ? a.end - off : (uint64_t)kBulkTile);
        const float* st = smem + (size_t)stage * S * kBulkTile;
        for (uint32_t e = threadIdx.x * 8; e < len; e += kBulkConsumers * 8) {
            V8 acc = *reinterpret_cast<const V8*>(st + e);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc.x[j] = __fadd_rn(0.0f, acc.x[j]);
#pragma unroll
            for (int k = 1; k < NW; ++k) {
                const V8 gk = *reinterpret_cast<const V8*>(st + k * kBulkTile + e);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc.x[j] = __fadd_rn(acc.x[j], gk.x[j]);
            }
            V8 wv = *reinterpret_cast<const V8*>(st + NW * kBulkTile + e);
            V8 vv = *reinterpret_cast<const V8*>(st + (NW + 1) * kBulkTile + e);
            V8 sv = acc;
#pragma unroll
            for (int j = 0; j < 8; ++j) nag(acc.x[j], wv.x[j], vv.x[j], a.lr, a.mu, a.rescale);
            st_w<PHUB_CACHE_ENABLED>(reinterpret_cast<V8*>(a.w + off + e), wv);
            st_stream(reinterpret_cast<V8*>(a.v + off + e), vv);
            if constexpr (AGG) st_stream(reinterpret_cast<V8*>(a.agg + off + e), sv);
            for (int r = 0; r < a.nrep; ++r) *reinterpret_cast<V8*>(a.rep[r] + off + e) = wv;
        }
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[stage]);
        if (++stage == kBulkStages) { stage = 0; phase ^= 1; }
    }
    if (a.nrep) __threadfence_system();
}

template <bool AGG>
void* pick_bulk(int nw) {
    switch (nw) {
        case 1: return (void*)k_bulk<1, AGG>;
        case 2: return (void*)k_bulk<2, AGG>;
        case 3: return (void*)k_bulk<3, AGG>;
        case 4: return (void*)k_bulk<4, AGG>;
        case 5: return (void*)k_bulk<5, AGG>;
        case 6: return (void*)k_bulk<6, AGG>;
        case 7: return (void*)k_bulk<7, AGG>;
        case 8: return (void*)k_bulk<8, AGG>;
        default: return nullptr;
    }
}

// -------------------------------------------------------- wide (ablation)
// pass 1: merge = (+0 + g0) [+ g1];  pass k: merge = merge + gk;  NAG pass.
__global__ void __launch_bounds__(kThreads) k_wide_first(const __grid_constant__ WideArgs a) {
    const uint64_t n = (a.end - a.begin) / 4;
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
        const V4 g0 = ld_grad(reinterpret_cast<const V4*>(a.g[0] + a.begin) + i);
        V4 s;
        if (a.nw > 1) {
            const V4 g1 = ld_grad(reinterpret_cast<const V4*>(a.g[1] + a.begin) + i);
#pragma unroll
            for (int e = 0; e < 4; ++e) s.x[e] = __fadd_rn(__fadd_rn(0.0f, g0.x[e]), g1.x[e]);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) s.x[e] = __fadd_rn(0.0f, g0.x[e]);
        }
        reinterpret_cast<V4*>(a.agg + a.begin)[i] = s;
    }
}

__global__ void __launch_bounds__(kThreads) k_wide_add(const __grid_constant__ WideArgs a, int k) {
    const uint64_t n = (a.end - a.begin) / 4;
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
        const V4 gk = ld_grad(reinterpret_cast<const V4*>(a.g[k] + a.begin) + i);
        V4 s = reinterpret_cast<V4*>(a.agg + a.begin)[i];
#pragma unroll
        for (int e = 0; e < 4; ++e) s.x[e] = __fadd_rn(s.x[e], gk.x[e]);
        reinterpret_cast<V4*>(a.agg + a.begin)[i] = s;
    }
}

__global__ void __launch_bounds__(kThreads) k_wide_nag(const __grid_constant__ WideArgs a) {
    const uint64_t n = (a.end - a.begin) / 4;
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += stride) {
        const V4 s = reinterpret_cast<const V4*>(a.agg + a.begin)[i];
        V4 wv = reinterpret_cast<V4*>(a.w + a.begin)[i];
        V4 vv = reinterpret_cast<V4*>(a.v + a.begin)[i];
#pragma unroll
        for (int e = 0; e < 4; ++e) nag(s.x[e], wv.x[e], vv.x[e], a.lr, a.mu, a.rescale);
        reinterpret_cast<V4*>(a.w + a.begin)[i] = wv;
        reinterpret_cast<V4*>(a.v + a.begin)[i] = vv;
    }
}

// ------------------------------------------------------------- dispatch
using FlatFn = void (*)(FlatArgs);
using TileFn = void (*)(TileArgs);

template <int VEC, int CACHE, bool AGG>
FlatFn pick_flat_nw(int nw) {
    switch (nw) {
        case 1: return k_flat<1, VEC, CACHE, AGG>;
        case 2: return k_flat<2, VEC, CACHE, AGG>;
        case 3: return k_flat<3, VEC, CACHE, AGG>;
        case 4: return k_flat<4, VEC, CACHE, AGG>;
        case 5: return k_flat<5, VEC, CACHE, AGG>;
        case 6: return k_flat<6, VEC, CACHE, AGG>;
        case 7: return k_flat<7, VEC, CACHE, AGG>;
        case 8: return k_flat<8, VEC, CACHE, AGG>;
        default: return k_flat<0, VEC, CACHE, AGG>;
    }
}

FlatFn pick_flat(int vec, int nw, bool agg, int cache) {
    if (vec == 8) {
        if (cache == PHUB_CACHE_RESIDENT)
            return agg ? pick_flat_nw<8, PHUB_CACHE_RESIDENT, true>(nw)
                       : pick_flat_nw<8, PHUB_CACHE_RESIDENT, false>(nw);
        if (cache == PHUB_CACHE_BYPASS)
            return agg ? pick_flat_nw<8, PHUB_CACHE_BYPASS, true>(nw)
                       : pick_flat_nw<8, PHUB_CACHE_BYPASS, false>(nw);
        return agg ? pick_flat_nw<8, PHUB_CACHE_ENABLED, true>(nw)
                   : pick_flat_nw<8, PHUB_CACHE_ENABLED, false>(nw);
    }
    return agg ? pick_flat_nw<4, PHUB_CACHE_ENABLED, true>(nw)
               : pick_flat_nw<4, PHUB_CACHE_ENABLED, false>(nw);
}

template <bool AGG>
TileFn pick_tiles_nw(int nw) {
    switch (nw) {
        case 1: return k_tiles<1, AGG>;
        case 2: return k_tiles<2, AGG>;
        case 3: return k_tiles<3, AGG>;
        case 4: return k_tiles<4, AGG>;
        case 5: return k_tiles<5, AGG>;
        case 6: return k_tiles<6, AGG>;
        case 7: return k_tiles<7, AGG>;
        case 8: return k_tiles<8, AGG>;
        default: return k_tiles<0, AGG>;
    }
}

}  // namespace

int flat_blocks_per_sm(int vec, int nw, bool agg, int cache) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &nb, reinterpret_cast<const void*>(pick_flat(vec, nw, agg, cache)), kThreads, 0) !=
        cudaSuccess)
        return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_flat(const FlatArgs& a, int vec, int cache, int grid, cudaStream_t s,
                        int* launches) {
    if (a.end <= a.begin && !a.signal_flag) return cudaSuccess;
    pick_flat(vec, a.nw, a.agg != nullptr, cache)<<<grid, kThreads, 0, s>>>(a);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_tiles(const TileArgs& a, int grid, cudaStream_t s, int* launches) {
    if (a.ntiles == 0) return cudaSuccess;
    TileFn fn = a.agg ? pick_tiles_nw<true>(a.nw) : pick_tiles_nw<false>(a.nw);
    fn<<<grid, kThreads, 0, s>>>(a);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_prefix(const FlatArgs& a, float* dst, int grid, cudaStream_t s, int* launches) {
    if (a.end <= a.begin && !a.signal_flag) return cudaSuccess;
    switch (a.nw) {
        case 1: k_prefix<1><<<grid, kThreads, 0, s>>>(a, dst); break;
        case 2: k_prefix<2><<<grid, kThreads, 0, s>>>(a, dst); break;
        case 3: k_prefix<3><<<grid, kThreads, 0, s>>>(a, dst); break;
        case 4: k_prefix<4><<<grid, kThreads, 0, s>>>(a, dst); break;
        case 5: k_prefix<5><<<grid, kThreads, 0, s>>>(a, dst); break;
        default: k_prefix<0><<<grid, kThreads, 0, s>>>(a, dst); break;
    }
    ++*launches;
    return cudaGetLastError();
}

int blocks_per_sm(int nw, bool nag) {
    int nb = 0;
    const void* fn = nag ? pick_blocks<true>(nw) : pick_blocks<false>(nw);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, 0) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_blocks(const FlatArgs& a, float* dst, int grid, cudaStream_t s, int* launches) {
    if (a.end <= a.begin || a.block == 0) return cudaSuccess;
    void* fn = dst ? pick_blocks<false>(a.nw) : pick_blocks<true>(a.nw);
    void* args[] = {const_cast<FlatArgs*>(&a), &dst};
    cudaError_t e = cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, 0, s);
    ++*launches;
    return e;
}

int hier_blocks_per_sm(int nw, bool worker_order) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pick_hier(nw, worker_order), kThreads, 0) !=
        cudaSuccess)
        return 1;
    return nb > 0 ? nb : 1;
}

int sched_blocks_per_sm(int nw) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pick_sched(nw), kThreads, 0) != cudaSuccess)
        return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_sched(const SchedArgs& a, int grid, cudaStream_t s, int* launches) {
    void* args[] = {const_cast<SchedArgs*>(&a)};
    cudaError_t e = cudaLaunchKernel(pick_sched(a.nw), dim3(grid), dim3(kThreads), args, 0, s);
    ++*launches;
    return e;
}

cudaError_t launch_hier(const HierArgs& a, int grid, cudaStream_t s, int* launches) {
    void* args[] = {const_cast<HierArgs*>(&a)};
    cudaError_t e = cudaLaunchKernel(pick_hier(a.nw, a.worker_order != 0), dim3(grid),
                                     dim3(kThreads), args, 0, s);
    ++*launches;
    return e;
}

// Load every kernel of the library into the context now.  Under CUDA's lazy
// loading (the CUDA 12 default) a kernel's code is loaded on its first use,
// and a load can wait for the device -- including for a kernel spinning on a
// device flag that only the not-yet-loaded kernel would raise (a producer and
// consumer of one chain on two streams of one GPU, or any first exchange
// round): a deadlock until the bounded wait expires.  phub_init calls this
// once per device, before any flag protocol can run.
cudaError_t preload_kernels() {
    std::vector<const void*> fns;
    for (int nw = 0; nw <= 9; ++nw) {
        fns.push_back(pick_blocks<true>(nw));
        fns.push_back(pick_blocks<false>(nw));
        fns.push_back(pick_hier(nw, true));
        fns.push_back(pick_hier(nw, false));
        fns.push_back(pick_sched(nw));
        for (int vec : {4, 8})
            for (int cache : {PHUB_CACHE_ENABLED, PHUB_CACHE_BYPASS, PHUB_CACHE_RESIDENT})
                for (bool agg : {false, true})
                    fns.push_back(reinterpret_cast<const void*>(pick_flat(vec, nw, agg, cache)));
        fns.push_back(reinterpret_cast<const void*>(pick_tiles_nw<false>(nw)));
        fns.push_back(reinterpret_cast<const void*>(pick_tiles_nw<true>(nw)));
        if (void* b = pick_bulk<false>(nw)) fns.push_back(b);
        if (void* b = pick_bulk<true>(nw)) fns.push_back(b);
    }
    for (const void* f : {(const void*)k_prefix<0>, (const void*)k_prefix<1>, (const void*)k_prefix<2>,
                          (const void*)k_prefix<3>, (const void*)k_prefix<4>, (const void*)k_prefix<5>,
                          (const void*)k_wide_first, (const void*)k_wide_add, (const void*)k_wide_nag})
        fns.push_back(f);
    for (const void* f : fns) {
        cudaFuncAttributes at;
        cudaError_t e = cudaFuncGetAttributes(&at, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

size_t bulk_smem_bytes(int nw) { return (size_t)kBulkStages * (nw + 2) * kBulkTile * sizeof(float); }

cudaError_t launch_bulk(const FlatArgs& a, int grid, cudaStream_t s, int* launches) {
    if (a.end <= a.begin) return cudaSuccess;
    void* fn = a.agg ? pick_bulk<true>(a.nw) : pick_bulk<false>(a.nw);
    if (!fn) return cudaErrorInvalidValue;
    const size_t smem = bulk_smem_bytes(a.nw);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<FlatArgs*>(&a)};
    e = cudaLaunchKernel(fn, dim3(grid), dim3(kBulkConsumers + 32), args, smem, s);
    ++*launches;
    return e;
}

cudaError_t launch_wide(const WideArgs& a, int grid, cudaStream_t s, int* launches) {
    if (a.end <= a.begin) return cudaSuccess;
    k_wide_first<<<grid, kThreads, 0, s>>>(a);
    ++*launches;
    for (int k = 2; k < a.nw; ++k) {
        k_wide_add<<<grid, kThreads, 0, s>>>(a, k);
        ++*launches;
    }
    k_wide_nag<<<grid, kThreads, 0, s>>>(a);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace phub
