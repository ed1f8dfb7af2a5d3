// cache_sweep.cu -- L2 policy sweep of the fused aggregate + Nesterov step
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

struct Args { const float* g[8]; float* w; float* v; uint64_t nvec; float lr, mu, resc; };

template <int G, int S, int W, int V>
__global__ void __launch_bounds__(256) k(const __grid_constant__ Args a) {
    const uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x;
    if (i >= a.nvec) return;
    V8 gv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) gv[q] = ldg<G>(reinterpret_cast<const V8*>(a.g[q]) + i);
    V8 wv = lds<S>(reinterpret_cast<const V8*>(a.w) + i);
    V8 vv = lds<S>(reinterpret_cast<const V8*>(a.v) + i);
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
    stw<W>(reinterpret_cast<V8*>(a.w) + i, wv);
    if (V == 0) stw<1>(reinterpret_cast<V8*>(a.v) + i, vv);
    else stw<2>(reinterpret_cast<V8*>(a.v) + i, vv);
}

typedef void (*Fn)(Args);
struct Var { int g, s, w, v; Fn fn; };

template <int G, int S, int W, int V> void add(std::vector<Var>& out) { out.push_back({G, S, W, V, k<G, S, W, V>}); }
template <int G, int S, int W> void addV(std::vector<Var>& o) { add<G, S, W, 0>(o); add<G, S, W, 1>(o); }
template <int G, int S> void addW(std::vector<Var>& o) { addV<G, S, 0>(o); addV<G, S, 1>(o); addV<G, S, 2>(o); }
template <int G> void addS(std::vector<Var>& o) { addW<G, 0>(o); addW<G, 1>(o); }

int main() {
    const uint64_t E = 143667264;                 // VGG-19 padded
    const uint64_t nvec = E / 8;
    std::vector<float*> bufs(11);
    for (auto& b : bufs) { cudaMalloc(&b, E * 4); cudaMemset(b, 0, E * 4); }
    Args a{};
    for (int q = 0; q < 8; ++q) a.g[q] = bufs[q];
    a.w = bufs[8]; a.v = bufs[9]; a.nvec = nvec; a.lr = 0.1f; a.mu = 0.9f; a.resc = 0.125f;
    float* pull = bufs[10];
    std::vector<Var> vars;
    addS<0>(vars); addS<1>(vars); addS<2>(vars);
    const unsigned grid = (unsigned)((nvec + 255) / 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 30;
    printf("{\"bytes_per_launch\": %llu, \"reps\": %d}\n", (unsigned long long)(48 * E), reps);
    for (int pass = 0; pass < 2; ++pass)
        for (const Var& v : vars) {
            for (int t = 0; t < 3; ++t) v.fn<<<grid, 256>>>(a);
            cudaEventRecord(e0);
            for (int t = 0; t < reps; ++t) v.fn<<<grid, 256>>>(a);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms_k = 0;
            cudaEventElapsedTime(&ms_k, e0, e1);
            cudaEventRecord(e0);
            for (int t = 0; t < reps; ++t) {
                v.fn<<<grid, 256>>>(a);
                cudaMemcpyAsync(pull, a.w, E * 4, cudaMemcpyDeviceToDevice);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms_kp = 0;
            cudaEventElapsedTime(&ms_kp, e0, e1);
            printf("{\"pass\": %d, \"G\": %d, \"S\": %d, \"W\": %d, \"V\": %d, \"kernel_ms\": %.4f, "
                   "\"kernel_tbs\": %.3f, \"kernel_pull_ms\": %.4f}\n", pass, v.g, v.s, v.w, v.v,
                   ms_k / reps, 48.0 * E / (ms_k / reps * 1e-3) / 1e12, ms_kp / reps);
        }
    cudaError_t err = cudaGetLastError();
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
