// Standalone probe of the fused one-shot kernel's instruction schedule (not
// the library): VGG-19 size, 8 gradient streams + w + v, the
// same arithmetic and cache hints as k_flat<8,8,BYPASS>, in variants that
// differ only in how many loads a thread has in flight before its first add:
//   A  as the library compiles it (ptxas interleaves loads with adds: ~3 loads
//      in flight, 44-48 registers, 5 CTAs/SM)
//   B  __launch_bounds__(256, 3): registers for all 10 loads up front
//   C  all 8 gradient loads issued in ONE asm block (outputs defined together)
//   D  C + w, v loads in the same block
// Mean kernel ms of 30 launches (CUDA events), VGG-19 E = 143,667,264.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o flat_variants flat_variants.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(32) V8 { float x[8]; };

__device__ __forceinline__ V8 ldg(const V8* p) {
    V8 r;
    asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]),
          "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    return r;
}
__device__ __forceinline__ V8 lds(const V8* p) {
    V8 r;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]), "=f"(r.x[5]),
          "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    return r;
}
__device__ __forceinline__ void sts(V8* p, const V8& r) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
        :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]), "f"(r.x[5]),
           "f"(r.x[6]), "f"(r.x[7]) : "memory");
}
// two v8 loads in one asm block: both issued before either result is used
__device__ __forceinline__ void ldg2(const V8* p, const V8* q, V8& a, V8& b) {
    asm("{\n\t"
        "ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%16];\n\t"
        "ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%8,%9,%10,%11,%12,%13,%14,%15}, [%17];\n\t"
        "}"
        : "=f"(a.x[0]), "=f"(a.x[1]), "=f"(a.x[2]), "=f"(a.x[3]), "=f"(a.x[4]), "=f"(a.x[5]),
          "=f"(a.x[6]), "=f"(a.x[7]), "=f"(b.x[0]), "=f"(b.x[1]), "=f"(b.x[2]), "=f"(b.x[3]),
          "=f"(b.x[4]), "=f"(b.x[5]), "=f"(b.x[6]), "=f"(b.x[7])
        : "l"(p), "l"(q));
}

struct Args { const float* g[8]; float* w; float* v; uint64_t n; float lr, mu, rs; };

__device__ __forceinline__ void nag(float s, float& w, float& v, float lr, float mu, float rs) {
    const float g = __fmul_rn(s, rs);
    const float vn = __fadd_rn(__fmul_rn(mu, v), g);
    w = __fsub_rn(w, __fmul_rn(lr, __fadd_rn(g, __fmul_rn(mu, vn))));
    v = vn;
}

template <int MODE>
__device__ __forceinline__ void body(const Args& a, uint64_t i) {
    V8 g[8];
    if (MODE >= 2) {
        for (int k = 0; k < 8; k += 2)
            ldg2(reinterpret_cast<const V8*>(a.g[k]) + i, reinterpret_cast<const V8*>(a.g[k + 1]) + i,
                 g[k], g[k + 1]);
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k] = ldg(reinterpret_cast<const V8*>(a.g[k]) + i);
    }
    V8* w = reinterpret_cast<V8*>(a.w) + i;
    V8* v = reinterpret_cast<V8*>(a.v) + i;
    V8 wv, vv;
    if (MODE == 3) { wv = lds(w); vv = lds(v); }
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float s = __fadd_rn(0.0f, g[0].x[j]);
#pragma unroll
        for (int k = 1; k < 8; ++k) s = __fadd_rn(s, g[k].x[j]);
        acc[j] = s;
    }
    if (MODE != 3) { wv = lds(w); vv = lds(v); }
#pragma unroll
    for (int j = 0; j < 8; ++j) nag(acc[j], wv.x[j], vv.x[j], a.lr, a.mu, a.rs);
    sts(w, wv);
    sts(v, vv);
}

__global__ void __launch_bounds__(256) kA(const __grid_constant__ Args a) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < a.n) body<0>(a, i);
}
__global__ void __launch_bounds__(256, 3) kB(const __grid_constant__ Args a) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < a.n) body<1>(a, i);
}
__global__ void __launch_bounds__(256) kC(const __grid_constant__ Args a) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < a.n) body<2>(a, i);
}
__global__ void __launch_bounds__(256) kD(const __grid_constant__ Args a) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < a.n) body<3>(a, i);
}
__global__ void __launch_bounds__(256, 4) kE(const __grid_constant__ Args a) {
    const uint64_t i = blockIdx.x * 256ull + threadIdx.x;
    if (i < a.n) body<2>(a, i);
}

__global__ void fill(float* p, uint64_t n, uint64_t seed) {
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        p[i] = (float)((int64_t)(z >> 40) - (1ll << 23)) * 1e-9f;   // random, full mantissa
    }
}

int main(int argc, char** argv) {
    const bool zeros = argc > 1 && argv[1][0] == 'z';
    const uint64_t E = 143667264ull, n = E / 8;
    Args a{};
    auto init = [&](float* p, uint64_t seed) {
        if (zeros) cudaMemset(p, 0, E * 4);
        else fill<<<148 * 8, 256>>>(p, E, seed * 1000003ull);
    };
    for (int k = 0; k < 8; ++k) {
        float* p;
        cudaMalloc(&p, E * 4);
        init(p, k + 1);
        a.g[k] = p;
    }
    cudaMalloc(&a.w, E * 4);
    cudaMalloc(&a.v, E * 4);
    init(a.w, 11);
    init(a.v, 12);
    cudaDeviceSynchronize();
    printf("{\"data\": \"%s\"}\n", zeros ? "zeros" : "random");
    a.n = n; a.lr = 0.1f; a.mu = 0.9f; a.rs = 0.125f;
    const unsigned grid = (unsigned)((n + 255) / 256);
    void (*ks[])(Args) = {kA, kB, kC, kD, kE};
    const char* names[] = {"A library schedule", "B launch_bounds(256,3)", "C grads in asm pairs",
                           "D C + w,v first", "E C + launch_bounds(256,4)"};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int pass = 0; pass < 3; ++pass)
        for (int v = 0; v < 5; ++v) {
            for (int w = 0; w < 5; ++w) ks[v]<<<grid, 256>>>(a);
            cudaEventRecord(e0);
            for (int r = 0; r < 30; ++r) ks[v]<<<grid, 256>>>(a);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaFuncAttributes at;
            cudaFuncGetAttributes(&at, ks[v]);
            printf("{\"pass\": %d, \"variant\": \"%s\", \"regs\": %d, \"ms\": %.4f, \"TBps\": %.3f}\n",
                   pass, names[v], at.numRegs, ms / 30, 48.0 * E / 8 * 8 / (ms / 30) / 1e9);
        }
    return cudaGetLastError() != cudaSuccess;
}
