/* Host-side fuzz of libphub's planning code under ASan + UBSan (SURVEY 5:
 * "host ASan/UBSan on the table code").  Plain C client of include/phub.h.
 *
 * For pseudo-random manifests (up to 200 keys of up to 2e5 elements, some tiny),
 * chunk sizes (4 B .. 1 MiB and invalid ones), owner counts 1..8 and both
 * owner policies it calls phub_plan_chunks (count query + fill),
 * phub_plan_ranges and phub_init (which plans on the host and then fails
 * without a GPU, or succeeds and is destroyed with one), and checks the
 * table invariants: coverage of every key in order, owner in range, ranges
 * abutting over [0, E_padded), offsets 32-element aligned.  Exit 0 = clean.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "phub.h"

static uint64_t rng = 0x1805078910ull;
static uint64_t next(void) {
    rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
    return rng;
}

#define CHECK(c, ...) do { if (!(c)) { fprintf(stderr, __VA_ARGS__); fputc('\n', stderr); return 1; } } while (0)

int main(int argc, char** argv) {
    const int iters = argc > 1 ? atoi(argv[1]) : 400;
    for (int it = 0; it < iters; ++it) {
        static const uint64_t cbs[] = {4, 12, 64, 4096, 8192, 32768, 65536, 1 << 20, 0, 6, 3};
        const uint64_t cb = cbs[next() % (sizeof cbs / sizeof cbs[0])];
        /* keep the chunk count moderate: tiny chunks get small manifests */
        const int small = cb != 0 && cb < 4096;
        const int K = 1 + (int)(next() % (small ? 12 : 200));
        uint64_t* n = (uint64_t*)malloc(sizeof(uint64_t) * K);
        for (int k = 0; k < K; ++k)
            n[k] = (next() % 4 == 0) ? 1 + next() % 7 : 1 + next() % (small ? 3000 : 200000);
        const int G = 1 + (int)(next() % 8);
        const int policy = (int)(next() % 2);
        const int valid_cb = cb == 0 || cb % 4 == 0;

        uint64_t cnt = 0;
        phub_status st = phub_plan_chunks(n, K, cb, G, policy, NULL, 0, &cnt);
        if (!valid_cb) {
            CHECK(st == PHUB_ERR_INVALID_CHUNK_SIZE, "iter %d: chunk %llu accepted", it,
                  (unsigned long long)cb);
            free(n);
            continue;
        }
        CHECK(st == PHUB_OK || st == PHUB_ERR_LENGTH_MISMATCH, "iter %d: count query -> %d", it, st);
        phub_chunk* ch = (phub_chunk*)malloc(sizeof(phub_chunk) * (cnt ? cnt : 1));
        uint64_t cnt2 = 0;
        CHECK(phub_plan_chunks(n, K, cb, G, policy, ch, cnt, &cnt2) == PHUB_OK && cnt2 == cnt,
              "iter %d: fill", it);
        /* coverage: chunks are dense in (key, offset) order and cover every key */
        uint64_t j = 0;
        for (int k = 0; k < K; ++k) {
            uint64_t off = 0;
            while (off < n[k]) {
                CHECK(j < cnt, "iter %d: ran out of chunks", it);
                CHECK(ch[j].vkey_id == j && ch[j].key_id == (uint32_t)k && ch[j].offset == off,
                      "iter %d: chunk %llu out of order", it, (unsigned long long)j);
                CHECK(ch[j].length >= 1 && off + ch[j].length <= n[k], "iter %d: bad length", it);
                CHECK(ch[j].owner >= 0 && ch[j].owner < G, "iter %d: owner %d", it, ch[j].owner);
                off += ch[j].length;
                ++j;
            }
        }
        CHECK(j == cnt, "iter %d: %llu extra chunks", it, (unsigned long long)(cnt - j));

        uint64_t Ep = 0;
        uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * K);
        uint64_t* ob = (uint64_t*)malloc(sizeof(uint64_t) * G);
        uint64_t* oe = (uint64_t*)malloc(sizeof(uint64_t) * G);
        CHECK(phub_plan_ranges(n, K, cb, G, &Ep, offs, ob, oe) == PHUB_OK, "iter %d: ranges", it);
        uint64_t prev = 0;
        for (int k = 0; k < K; ++k) {
            CHECK(offs[k] % 32 == 0 && offs[k] >= prev, "iter %d: key offset", it);
            prev = offs[k] + n[k];
        }
        CHECK(Ep >= prev && Ep % 32 == 0, "iter %d: E_padded", it);
        CHECK(ob[0] == 0 && oe[G - 1] == Ep, "iter %d: range ends", it);
        for (int g = 0; g < G; ++g) {
            CHECK(ob[g] <= oe[g], "iter %d: range %d inverted", it, g);
            if (g) CHECK(ob[g] == oe[g - 1], "iter %d: ranges do not abut", it);
        }

        phub_config cfg;
        phub_config_default(&cfg);
        cfg.key_num_elements = n;
        cfg.num_keys = K;
        cfg.chunk_size_bytes = cb;
        cfg.num_workers = 1 + (int)(next() % 9);
        cfg.num_owners = G;
        cfg.owner_rank = (int)(next() % G);
        cfg.owner_policy = policy;
        phub_ctx ctx = NULL;
        st = phub_init(&cfg, &ctx);
        if (st == PHUB_OK) phub_destroy(ctx);
        else CHECK(st == PHUB_ERR_CUDA || st == PHUB_ERR_INVALID_ARGUMENT ||
                   st == PHUB_ERR_OUT_OF_MEMORY, "iter %d: init -> %s", it, phub_status_string(st));
        free(n); free(ch); free(offs); free(ob); free(oe);
    }
    /* invalid manifests / arguments */
    uint64_t zero[2] = {5, 0};
    uint64_t c = 0;
    CHECK(phub_plan_chunks(zero, 2, 32768, 1, 0, NULL, 0, &c) == PHUB_ERR_INVALID_MANIFEST, "zero key");
    CHECK(phub_plan_chunks(zero, 0, 32768, 1, 0, NULL, 0, &c) == PHUB_ERR_INVALID_MANIFEST, "no keys");
    CHECK(phub_plan_chunks(zero, 1, 32768, 0, 0, NULL, 0, &c) != PHUB_OK, "0 owners");
    printf("host fuzz ok: %d manifests\n", iters);
    return 0;
}
