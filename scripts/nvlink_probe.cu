// nvlink_probe.cu -- NVLink 5 peer-access microbenchmark (single process,
// cudaDeviceEnablePeerAccess), used to pick the denominators and the data
// direction (peer loads vs peer stores) of the multi-GPU exchange kernels.
//
// Patterns (SM-driven 256-bit accesses, grid = SMs x CTAs/SM, CUDA events):
//   load1    GPU1 loads a GPU0 buffer               (one direction, pull)
//   store1   GPU0 stores into a GPU1 buffer          (one direction, push)
//   loadbi   GPU0 loads GPU1 and GPU1 loads GPU0     (both directions at once)
//   chain    GPU1 loads GPU0's buffer AND stores the same bytes into GPU0
//   a2a      every GPU loads a slice from every peer (G >= 3)
//   ce       cudaMemcpyPeerAsync GPU0 -> GPU1        (copy engine)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvlink_probe nvlink_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

struct alignas(32) V8 { float x[8]; };

__device__ __forceinline__ V8 ld8(const V8* p) {
    V8 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                   "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(V8* p, const V8& r) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]),
                    "f"(r.x[5]), "f"(r.x[6]), "f"(r.x[7]) : "memory");
}

// copy n vectors from src to dst (either may be a peer pointer); dst==nullptr: load only
template <int U>
__global__ void k_copy(const V8* __restrict__ src, V8* __restrict__ dst, uint64_t n, float* sink) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        V8 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = ld8(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (dst) st8(dst + i + u * stride, r[u]);
            else acc += r[u].x[0];
        }
    }
    for (; i < n; i += stride) {
        V8 r = ld8(src + i);
        if (dst) st8(dst + i, r); else acc += r.x[0];
    }
    if (acc == 1234.5f) *sink = acc;
}

// store-only: fill n vectors of dst
__global__ void k_fill(V8* __restrict__ dst, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    V8 r;
    for (int j = 0; j < 8; ++j) r.x[j] = 1.0f;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) st8(dst + i, r);
}

// mode 0: load 1/G slice from each peer; 1: store 1/G slice into each peer; 2: load from
// peer p AND store into peer p (same kernel, same link)
struct PeerPtrs { V8* p[8]; };
__global__ void k_multi(int me, int G, PeerPtrs a, PeerPtrs b, uint64_t n, int mode, float* sink) {
    const int q0 = blockIdx.y;
    const int q = q0 >= me ? q0 + 1 : q0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    V8 r;
    for (int j = 0; j < 8; ++j) r.x[j] = 1.0f;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if (mode == 0) acc += ld8(a.p[q] + me * n + i).x[0];
        else if (mode == 1) st8(b.p[q] + me * n + i, r);
        else st8(b.p[q] + me * n + i, ld8(a.p[q] + me * n + i));
    }
    if (acc == 1234.5f) *sink = acc;
}

// TMA bulk-copy all-to-all: each CTA streams 16 KB chunks of its local slice
// global -> shared (cp.async.bulk, mbarrier) -> peer global (cp.async.bulk
// bulk_group), double-buffered; one elected thread drives the copy engine.
__device__ __forceinline__ unsigned su32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__global__ void k_bulk_a2a(int me, int G, PeerPtrs a, PeerPtrs b, uint64_t n_vec) {
    constexpr unsigned CH = 16384;                       // bytes per chunk
    __shared__ __align__(128) unsigned char buf[2][CH];
    __shared__ __align__(8) unsigned long long bar[2];
    const int q0 = blockIdx.y;
    const int q = q0 >= me ? q0 + 1 : q0;
    if (threadIdx.x != 0) return;
    const char* src = reinterpret_cast<const char*>(a.p[me] + q * n_vec);   // local slice for q
    char* dst = reinterpret_cast<char*>(b.p[q] + me * n_vec);               // peer q's slot for me
    const uint64_t bytes = n_vec * 32;
    for (int s = 0; s < 2; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned phase[2] = {0, 0};
    int it = 0;
    for (uint64_t off = (uint64_t)blockIdx.x * CH; off < bytes; off += (uint64_t)gridDim.x * CH, ++it) {
        const int s = it & 1;
        const unsigned len = (unsigned)(bytes - off < CH ? bytes - off : CH);
        // the store that last read buf[s] (two chunks ago) must have finished reading smem
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     :: "r"(su32(&bar[s])), "r"(len) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(su32(buf[s])), "l"(src + off), "r"(len), "r"(su32(&bar[s])) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                     :: "r"(su32(&bar[s])), "r"(phase[s]) : "memory");
        phase[s] ^= 1;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     :: "l"(dst + off), "r"(su32(buf[s])), "r"(len) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int G, nsm;
std::vector<cudaStream_t> st;
std::vector<cudaEvent_t> e0, e1;

template <class F>
double timed(F launch_all, int reps = 10) {
    for (int w = 0; w < 3; ++w) launch_all();
    for (int d = 0; d < G; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
        for (int d = 0; d < G; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e0[d], st[d])); }
        launch_all();
        for (int d = 0; d < G; ++d) { CK(cudaSetDevice(d)); CK(cudaEventRecord(e1[d], st[d])); }
        double mx = 0;
        for (int d = 0; d < G; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaEventSynchronize(e1[d]));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
            if (ms > mx) mx = ms;
        }
        if (mx < best) best = mx;
    }
    return best;  // ms, max over GPUs of the best repetition
}

int main(int argc, char** argv) {
    CK(cudaGetDeviceCount(&G));
    if (G < 2) { printf("{\"error\": \"need >= 2 GPUs\"}\n"); return 0; }
    const uint64_t bytes = argc > 1 ? strtoull(argv[1], 0, 10) : (512ull << 20);
    const uint64_t n = bytes / 32;
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    nsm = p.multiProcessorCount;
    std::vector<V8*> a(G), b(G);
    struct { PeerPtrs data_dev[8]; } a_, b_;
    std::vector<float*> sink(G);
    st.resize(G); e0.resize(G); e1.resize(G);
    for (int d = 0; d < G; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < G; ++q)
            if (q != d) {
                int ok = 0;
                CK(cudaDeviceCanAccessPeer(&ok, d, q));
                if (ok) CK(cudaDeviceEnablePeerAccess(q, 0));
            }
        CK(cudaMalloc(&a[d], bytes));
        CK(cudaMalloc(&b[d], bytes));
        CK(cudaMalloc(&sink[d], 4));
        CK(cudaMemset(a[d], 0, bytes));
        CK(cudaMemset(b[d], 0, bytes));
        CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
    }
    for (int d = 0; d < G; ++d)
        for (int q = 0; q < G && q < 8; ++q) { a_.data_dev[d].p[q] = a[q]; b_.data_dev[d].p[q] = b[q]; }
    const double gb = bytes / 1e9;
    printf("{\"gpus\": %d, \"sms\": %d, \"bytes\": %llu, \"results\": [\n", G, nsm,
           (unsigned long long)bytes);
    bool first = true;
    auto out = [&](const char* pat, int cta, double ms, double moved_gb) {
        printf("%s{\"pattern\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.4f, \"GBps_per_dir\": %.1f}",
               first ? "" : ",\n", pat, cta, ms, moved_gb / (ms * 1e-3));
        first = false;
    };
    const int ctas[] = {1, 2, 4, 8, 16};
    for (int cta : ctas) {
        const int grid = nsm * cta;
        // local copy for reference (HBM read+write)
        double ms = timed([&] { CK(cudaSetDevice(0)); k_copy<4><<<grid, 256, 0, st[0]>>>(a[0], b[0], n, sink[0]); });
        out("local_copy_rw", cta, ms, 2 * gb);
        ms = timed([&] { CK(cudaSetDevice(1)); k_copy<4><<<grid, 256, 0, st[1]>>>(a[0], nullptr, n, sink[1]); });
        out("load1", cta, ms, gb);
        ms = timed([&] { CK(cudaSetDevice(1)); k_copy<4><<<grid, 256, 0, st[1]>>>(a[0], b[1], n, sink[1]); });
        out("load1_store_local", cta, ms, gb);
        ms = timed([&] { CK(cudaSetDevice(0)); k_fill<<<grid, 256, 0, st[0]>>>(b[1], n); });
        out("store1", cta, ms, gb);
        ms = timed([&] { CK(cudaSetDevice(0)); k_copy<4><<<grid, 256, 0, st[0]>>>(a[0], b[1], n, sink[0]); });
        out("store1_from_local", cta, ms, gb);
        ms = timed([&] {
            CK(cudaSetDevice(0)); k_copy<4><<<grid, 256, 0, st[0]>>>(a[1], nullptr, n, sink[0]);
            CK(cudaSetDevice(1)); k_copy<4><<<grid, 256, 0, st[1]>>>(a[0], nullptr, n, sink[1]);
        });
        out("loadbi", cta, ms, gb);
        ms = timed([&] {
            CK(cudaSetDevice(0)); k_fill<<<grid, 256, 0, st[0]>>>(b[1], n);
            CK(cudaSetDevice(1)); k_fill<<<grid, 256, 0, st[1]>>>(b[0], n);
        });
        out("storebi", cta, ms, gb);
        // chain: GPU1 pulls GPU0's buffer and pushes the same bytes back into GPU0
        ms = timed([&] { CK(cudaSetDevice(1)); k_copy<4><<<grid, 256, 0, st[1]>>>(a[0], b[0], n, sink[1]); });
        out("chain_load_and_store_same_gpu", cta, ms, gb);
        if (G >= 3) {
            // every GPU moves 1/G of its buffer to/from EACH peer in ONE kernel
            // (blockIdx.y = peer slot): load-only, store-only, and mixed
            ms = timed([&] {
                for (int d = 0; d < G; ++d) {
                    CK(cudaSetDevice(d));
                    k_multi<<<dim3(grid / (G - 1) > 0 ? grid / (G - 1) : 1, G - 1), 256, 0, st[d]>>>(
                        d, G, a_.data_dev[d], b_.data_dev[d], n / G, 0, sink[d]);
                }
            });
            out("a2a_load", cta, ms, gb * (G - 1) / G);
            ms = timed([&] {
                for (int d = 0; d < G; ++d) {
                    CK(cudaSetDevice(d));
                    k_multi<<<dim3(grid / (G - 1) > 0 ? grid / (G - 1) : 1, G - 1), 256, 0, st[d]>>>(
                        d, G, a_.data_dev[d], b_.data_dev[d], n / G, 1, sink[d]);
                }
            });
            out("a2a_store", cta, ms, gb * (G - 1) / G);
            ms = timed([&] {
                for (int d = 0; d < G; ++d) {
                    CK(cudaSetDevice(d));
                    k_multi<<<dim3(grid / (G - 1) > 0 ? grid / (G - 1) : 1, G - 1), 256, 0, st[d]>>>(
                        d, G, a_.data_dev[d], b_.data_dev[d], n / G, 2, sink[d]);
                }
            });
            out("a2a_load_and_store", cta, ms, gb * (G - 1) / G);
            ms = timed([&] {
                for (int d = 0; d < G; ++d) {
                    CK(cudaSetDevice(d));
                    k_bulk_a2a<<<dim3(nsm * cta / (G - 1) > 0 ? nsm * cta / (G - 1) : 1, G - 1), 32, 0,
                                 st[d]>>>(d, G, a_.data_dev[d], b_.data_dev[d], n / G);
                }
            });
            out("a2a_tma_bulk_store", cta, ms, gb * (G - 1) / G);
        }
    }
    // copy engine
    double ms = timed([&] { CK(cudaSetDevice(0)); CK(cudaMemcpyPeerAsync(b[1], 1, a[0], 0, bytes, st[0])); });
    out("ce_copy", 0, ms, gb);
    ms = timed([&] {
        CK(cudaSetDevice(0)); CK(cudaMemcpyPeerAsync(b[1], 1, a[0], 0, bytes, st[0]));
        CK(cudaSetDevice(1)); CK(cudaMemcpyPeerAsync(b[0], 0, a[1], 1, bytes, st[1]));
    });
    out("ce_copy_bi", 0, ms, gb);
    if (G >= 3) {
        // copy engines: every GPU copies 1/G of its buffer into each peer (one stream per peer)
        std::vector<std::vector<cudaStream_t>> ps(G, std::vector<cudaStream_t>(G));
        for (int d = 0; d < G; ++d) {
            CK(cudaSetDevice(d));
            for (int q = 0; q < G; ++q) CK(cudaStreamCreateWithFlags(&ps[d][q], cudaStreamNonBlocking));
        }
        const uint64_t sl = bytes / G;
        ms = timed([&] {
            for (int d = 0; d < G; ++d) {
                CK(cudaSetDevice(d));
                std::vector<cudaEvent_t> evs;
                for (int q = 0; q < G; ++q) {
                    if (q == d) continue;
                    cudaEvent_t e0x, e1x;
                    CK(cudaEventCreateWithFlags(&e0x, cudaEventDisableTiming));
                    CK(cudaEventCreateWithFlags(&e1x, cudaEventDisableTiming));
                    CK(cudaEventRecord(e0x, st[d]));
                    CK(cudaStreamWaitEvent(ps[d][q], e0x, 0));
                    CK(cudaMemcpyPeerAsync((char*)b[q] + d * sl, q, (char*)a[d] + q * sl, d, sl, ps[d][q]));
                    CK(cudaEventRecord(e1x, ps[d][q]));
                    CK(cudaStreamWaitEvent(st[d], e1x, 0));
                    evs.push_back(e0x); evs.push_back(e1x);
                }
                for (auto e : evs) CK(cudaEventDestroy(e));
            }
        });
        out("a2a_ce_copy", 0, ms, gb * (G - 1) / G);
    }
    printf("\n]}\n");
    return 0;
}
