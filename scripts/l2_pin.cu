// l2_pin.cu (derived from l2_keep.cu) -- pin a tail of w/v in L2 ONCE (evict_last store), then all-evict-first rounds of the fused aggregate + Nesterov step
// (k_flat's one-shot 256-bit schedule, N = 8, VGG-19 size) on one B200.
//
// Scratch experiment for NEXT-2 (P:691 / P:908-935 "cache-enabled vs
// cache-bypass"): which L2 eviction hints on which stream make the streaming
// kernel fastest, alone and followed by the pull of w' (a D2D copy)?
//   G: gradient loads   0 = .nc L1::no_allocate L2::evict_first (k_flat)
//                       1 = .nc L1::no_allocate (no L2 hint)
//                       2 = .nc L1::no_allocate L2::evict_first L2::256B prefetch
//   S: w, v loads       0 = L1::no_allocate            1 = + L2::evict_first
//   W: w' store         0 = L2::evict_last (k_flat "cache enabled")
//                       1 = L2::evict_first (k_flat "bypass")   2 = no hint
//   V: v' store         0 = L2::evict_first (k_flat)   1 = no hint
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cache_sweep cache_sweep.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

struct alignas(32) V8 { float x[8]; };

template <int G> __device__ __forceinline__ V8 ldg(const V8* p) {
    V8 r;
    if (G == 0)
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    else if (G == 1)
        asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    return r;
}
template <int S> __device__ __forceinline__ V8 lds(const V8* p) {
    V8 r;
    if (S == 0)
        asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    else
        asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    return r;
}
template <int W> __device__ __forceinline__ void stw(V8* p, const V8& r) {
    if (W == 0)
        asm volatile("st.global.L1::no_allocate.L2::evict_last.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
            :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]), "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]) : "memory");
    else if (W == 1)
        asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
            :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]), "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]) : "memory");
    else
        asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
            :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]), "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]) : "memory");
}

struct Args { const float* g[8]; float* w; float* v; uint64_t nvec; float lr, mu, resc;
              uint64_t keep_w, keep_v; };   // vectors i >= keep_* are stored evict_last (resident)

__global__ void __launch_bounds__(256) kk(const __grid_constant__ Args a) {
    const uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= a.nvec) return;
    V8 gv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) gv[q] = ldg<0>(reinterpret_cast<const V8*>(a.g[q]) + i);
    const bool kw = i >= a.keep_w, kv = i >= a.keep_v;
    V8 wv = kw ? lds<0>(reinterpret_cast<const V8*>(a.w) + i) : lds<1>(reinterpret_cast<const V8*>(a.w) + i);
    V8 vv = kv ? lds<0>(reinterpret_cast<const V8*>(a.v) + i) : lds<1>(reinterpret_cast<const V8*>(a.v) + i);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float s = __fadd_rn(0.0f, gv[0].x[j]);
#pragma unroll
        for (int q = 1; q < 8; ++q) s = __fadd_rn(s, gv[q].x[j]);
        const float g = __fmul_rn(s, a.resc);
        const float vn = __fadd_rn(__fmul_rn(a.mu, vv.x[j]), g);
        wv.x[j] = __fsub_rn(wv.x[j], __fmul_rn(a.lr, __fadd_rn(g, __fmul_rn(a.mu, vn))));
        vv.x[j] = vn;
    }
    if (kw) stw<0>(reinterpret_cast<V8*>(a.w) + i, wv); else stw<1>(reinterpret_cast<V8*>(a.w) + i, wv);
    if (kv) stw<0>(reinterpret_cast<V8*>(a.v) + i, vv); else stw<1>(reinterpret_cast<V8*>(a.v) + i, vv);
}

// value-preserving pin: load the tail and store it back with L2::evict_last
__global__ void pin(float* p, uint64_t from, uint64_t nvec) {
    const uint64_t i = from + (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (i < nvec) { V8 r = lds<0>(reinterpret_cast<const V8*>(p) + i); stw<0>(reinterpret_cast<V8*>(p) + i, r); }
}

__global__ void fill(float* p, uint64_t n, uint64_t seed) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        uint32_t b = (uint32_t)((z >> 63) << 31) | (uint32_t)((127 - (z >> 23) % 20) << 23) | (uint32_t)(z & 0x7FFFFF);
        p[i] = __uint_as_float(b) * 1e-3f;
    }
}

// usage: l2_pin W_MB V_MB MODE ROUNDS  MODE 0: kept tail stored evict_last every round (l2_keep);
//        1: pinned once, then every round all-evict-first; 2: re-pinned before every round
int main(int argc, char** argv) {
    const uint64_t E = 143667264, nvec = E / 8;
    const double wmb = argc > 1 ? atof(argv[1]) : 0, vmb = argc > 2 ? atof(argv[2]) : 0;
    std::vector<float*> bufs(11);
    for (int b = 0; b < 11; ++b) { cudaMalloc(&bufs[b], E * 4); fill<<<4096, 256>>>(bufs[b], E, 1000003ull * b); }
    Args a{};
    for (int q = 0; q < 8; ++q) a.g[q] = bufs[q];
    a.w = bufs[8]; a.v = bufs[9]; a.nvec = nvec; a.lr = 0.1f; a.mu = 0.9f; a.resc = 0.125f;
    const int mode = argc > 3 ? atoi(argv[3]) : 0;
    const int reps = argc > 4 ? atoi(argv[4]) : 4;
    const uint64_t kwv = (uint64_t)(wmb * (1 << 20) / 32), kvv = (uint64_t)(vmb * (1 << 20) / 32);
    const uint64_t pw = nvec - (kwv < nvec ? kwv : nvec), pv = nvec - (kvv < nvec ? kvv : nvec);
    a.keep_w = mode == 0 ? pw : nvec;
    a.keep_v = mode == 0 ? pv : nvec;
    auto do_pin = [&]() {
        if (kwv) pin<<<(unsigned)((kwv + 255) / 256), 256>>>(a.w, pw, nvec);
        if (kvv) pin<<<(unsigned)((kvv + 255) / 256), 256>>>(a.v, pv, nvec);
    };
    const unsigned grid = (unsigned)((nvec + 255) / 256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaDeviceSynchronize();
    if (mode == 1) do_pin();
    for (int rep = 0; rep < reps; ++rep) {
        for (int t = 0; t < 3; ++t) { if (mode == 2) do_pin(); kk<<<grid, 256>>>(a); }
        cudaEventRecord(e0);
        for (int t = 0; t < 20; ++t) { if (mode == 2) do_pin(); kk<<<grid, 256>>>(a); }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
        // pull: D2D copy of w right after (is the resident part served from L2?)
        cudaEventRecord(e0);
        for (int t = 0; t < 20; ++t) { kk<<<grid, 256>>>(a); cudaMemcpyAsync(bufs[10], a.w, E * 4, cudaMemcpyDeviceToDevice); }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms2 = 0; cudaEventElapsedTime(&ms2, e0, e1);
        printf("{\"w_mb\": %.0f, \"v_mb\": %.0f, \"mode\": %d, \"rep\": %d, \"kernel_ms\": %.4f, \"kernel_pull_ms\": %.4f}\n",
               wmb, vmb, mode, rep, ms / 20, ms2 / 20);
    }
    cudaError_t err = cudaGetLastError();
    return err == cudaSuccess ? 0 : 1;
}
