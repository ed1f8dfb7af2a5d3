/* The library's fused kernel timed from plain C (no Python, no torch): VGG-19
 * sized padded model, N = 8 cudaMalloc'd gradient buffers pushed BORROW,
 * 30 phub_aggregate_optimize rounds back to back after 10 warm-up, for each
 * L2 policy given on the command line (0 enabled, 1 bypass, 2 resident).
 * Companion of scripts/flat_variants.cu and scripts/flat_gap_probe.py. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "phub.h"

__attribute__((unused)) static const char* st(phub_status s) { return phub_status_string(s); }

int main(int argc, char** argv) {
    const int cache = argc > 1 ? atoi(argv[1]) : 2;
    const int data = argc > 2 ? atoi(argv[2]) : 0;   /* 0 zeros; 1 random grads; 2 + random w, v */
    const int vgg = argc > 3 && atoi(argv[3]);       /* 1: the 38-key VGG-19 manifest */
    static const uint64_t vgg19[38] = {
        1728, 64, 36864, 64, 73728, 128, 147456, 128, 294912, 256, 589824, 256, 589824, 256,
        589824, 256, 1179648, 512, 2359296, 512, 2359296, 512, 2359296, 512, 2359296, 512,
        2359296, 512, 2359296, 512, 2359296, 512, 102760448, 4096, 16777216, 4096, 4096000, 1000};
    uint64_t keys[1] = {143667264ull};          /* one key = E_padded of VGG-19 */
    phub_config cfg;
    phub_config_default(&cfg);
    cfg.key_num_elements = vgg ? vgg19 : keys;
    cfg.num_keys = vgg ? 38 : 1;
    cfg.num_workers = 8;
    phub_ctx ctx = NULL;
    if (phub_init(&cfg, &ctx) != PHUB_OK) return 1;
    phub_set_option(ctx, PHUB_OPT_CACHE, cache);
    float* g[8];
    float* h = (float*)malloc(keys[0] * 4);
    uint64_t z = 88172645463325252ull;
    for (uint64_t i = 0; i < keys[0]; ++i) {      /* xorshift, ~1e-3 scale, full mantissa */
        z ^= z << 13; z ^= z >> 7; z ^= z << 17;
        h[i] = (float)((int64_t)(z >> 40) - (1ll << 23)) * 1.2e-10f;
    }
    for (int w = 0; w < 8; ++w) {
        if (cudaMalloc((void**)&g[w], keys[0] * 4) != cudaSuccess) return 1;
        if (data) cudaMemcpy(g[w], h, keys[0] * 4, cudaMemcpyHostToDevice);
        else cudaMemset(g[w], 0, keys[0] * 4);
    }
    uint64_t Ereal = 0, Epad = 0;
    phub_layout(ctx, &Ereal, &Epad, NULL);
    if (Epad != keys[0]) return 2;
    if (data == 2 && phub_load_state(ctx, h, h) != PHUB_OK) return 1;
    free(h);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int r = 0; r < 40; ++r) {
        if (r == 10) cudaEventRecord(a, NULL);
        for (int w = 0; w < 8; ++w)
            if (phub_push(ctx, w, PHUB_ALL_KEYS, g[w], keys[0], PHUB_BORROW, NULL) != PHUB_OK) return 1;
        if (phub_aggregate_optimize(ctx, NULL) != PHUB_OK) return 1;
    }
    cudaEventRecord(b, NULL);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"harness\": \"C\", \"keys\": %d, \"cache\": %d, \"data\": %d, \"ms\": %.4f}\n",
           cfg.num_keys, cache, data, ms / 30);
    phub_destroy(ctx);
    return 0;
}
