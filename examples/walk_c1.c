/*
 * A C host of the C ABI alone (no Python, no torch): the reference sampler's first n
 * config-1 starts (lc_reference_candidates = random_candidate(random.Random(0), A51,
 * 0x2AAA00), pipeline.py:301-310) walked to their next special node at the paper's stride
 * (lc_walk = bitslice.forward_to_candidate), printed as one line:
 *     <n> <sum of dist> <min> <max> <fnv1a-64 of the (dst, dist) pairs>
 * tests/test_gpu_abi_c.py builds this against include/lfsr_b200.h and the in-tree library
 * and compares the line with the C restatement of the reference.
 *
 *     gcc -O2 -I include examples/walk_c1.c -L paper_1210_6411_b200/_lib -llfsr_b200 -o walk_c1
 */
#include <stdio.h>
#include <stdlib.h>

#include "lfsr_b200.h"

static void die(const char *what, int rc) {
    fprintf(stderr, "%s failed (%d): %s\n", what, rc, lc_last_error());
    exit(1);
}

int main(int argc, char **argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], NULL, 10) : 4096;
    const lc_spec a51 = {{19, 22, 23},
                         {(1u << 13) | (1u << 16) | (1u << 17) | (1u << 18), (1u << 20) | (1u << 21),
                          (1u << 7) | (1u << 20) | (1u << 21) | (1u << 22)},
                         {8, 10, 10}};
    /* the reference's default cap for A5/1, 16 * int(expected chain length) + 64
     * (bitslice.py:273-274) */
    const uint64_t fixed_r3 = 0x2AAA00, stride = 11170000, max_clocks = 178957008;
    uint64_t *starts = malloc(n * 8), *dst = malloc(n * 8), *dist = malloc(n * 8);
    uint64_t stats[LC_ST_HEADER + 2];
    lc_ctx *ctx = NULL;
    int rc;
    if (lc_abi_version() != LC_ABI_VERSION) die("lc_abi_version", -1);
    if ((rc = lc_reference_candidates(&a51, fixed_r3, 0, n, starts, NULL))) die("lc_reference_candidates", rc);
    if ((rc = lc_ctx_create(0, &ctx))) die("lc_ctx_create", rc);
    /* legs 1; refill 0: auto; no histogram bins */
    if ((rc = lc_walk(ctx, &a51, fixed_r3, starts, n, stride, max_clocks, 1, 0, dst, dist, 0, 0, 0, stats)))
        die("lc_walk", rc);
    uint64_t h = 1469598103934665603ull, sum = 0;
    for (uint64_t i = 0; i < n; i++) {
        h = (h ^ dst[i]) * 1099511628211ull;
        h = (h ^ dist[i]) * 1099511628211ull;
        sum += dist[i];
    }
    if (sum != stats[LC_ST_TRANSITIONS] || stats[LC_ST_EDGES] != n) {
        fprintf(stderr, "statistics block disagrees with the outputs\n");
        return 1;
    }
    printf("%llu %llu %llu %llu %016llx\n", (unsigned long long)n, (unsigned long long)sum,
           (unsigned long long)stats[LC_ST_MIN], (unsigned long long)stats[LC_ST_MAX], (unsigned long long)h);
    lc_ctx_destroy(ctx);
    free(starts);
    free(dst);
    free(dist);
    return 0;
}
