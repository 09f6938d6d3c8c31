/* Plain-C host of the drop-in ABI (include/uuvsim.h): what a non-Python caller of
 * the reference's libuuvsim_core.so (capi.rs) does, unchanged, against this library.
 *
 *   gcc -O2 -I include examples/host_step.c -L paper_2410_14117_b200/_lib \
 *       -luuvsim_core -Wl,-rpath,$PWD/paper_2410_14117_b200/_lib -o host_step
 *   ./host_step config.json [steps]
 *
 * Prints one line: envs, steps, env-steps/s, sum of rewards, done count.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "uuvsim.h"

static char* slurp(const char* path) {
    FILE* f = fopen(path, "rb");
    if (!f) return NULL;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    char* buf = (char*)malloc((size_t)n + 1);
    if (fread(buf, 1, (size_t)n, f) != (size_t)n) { fclose(f); free(buf); return NULL; }
    buf[n] = 0;
    fclose(f);
    return buf;
}

static int fail(const char* what) {
    char msg[1024];
    int64_t n = uuvsim_last_error(msg, sizeof msg - 1);
    msg[n < (int64_t)sizeof msg - 1 ? n : (int64_t)sizeof msg - 1] = 0;
    fprintf(stderr, "%s failed: %s\n", what, msg);
    return 1;
}

int main(int argc, char** argv) {
    if (argc < 2) { fprintf(stderr, "usage: %s config.json [steps]\n", argv[0]); return 2; }
    int steps = argc > 2 ? atoi(argv[2]) : 200;
    if (uuvsim_abi_version() != UUVSIM_ABI_VERSION) { fprintf(stderr, "ABI mismatch\n"); return 1; }
    char* cfg = slurp(argv[1]);
    if (!cfg) { fprintf(stderr, "cannot read %s\n", argv[1]); return 2; }
    uint64_t h = 0, spec[4];
    if (uuvsim_create(cfg, &h) != UUVSIM_OK) return fail("uuvsim_create");
    free(cfg);
    if (uuvsim_spec(h, spec) != UUVSIM_OK) return fail("uuvsim_spec");
    const uint64_t m = spec[0], od = spec[1], ad = spec[2];
    double* obs = (double*)malloc(m * od * sizeof(double));
    double* act = (double*)malloc(m * ad * sizeof(double));
    double* rew = (double*)malloc(m * sizeof(double));
    uint8_t* done = (uint8_t*)malloc(m);
    for (uint64_t i = 0; i < m * ad; ++i) act[i] = ((i * 2654435761u) % 2001) / 1000.0 - 1.0;
    if (uuvsim_reset(h, 7, obs, m * od) != UUVSIM_OK) return fail("uuvsim_reset");
    double rsum = 0.0;
    uint64_t ndone = 0;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (int s = 0; s < steps; ++s) {
        if (uuvsim_step(h, act, m * ad, obs, m * od, rew, m, done, m) != UUVSIM_OK)
            return fail("uuvsim_step");
        for (uint64_t e = 0; e < m; ++e) { rsum += rew[e]; ndone += done[e]; }
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double sec = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    /* misuse paths of the contract: wrong length -> 3, stale handle -> 2 */
    int bad = uuvsim_step(h, act, m * ad - 1, obs, m * od, rew, m, done, m);
    if (uuvsim_destroy(h) != UUVSIM_OK) return fail("uuvsim_destroy");
    int stale = uuvsim_destroy(h);
    printf("envs %llu steps %d env_steps_per_s %.3e reward_sum %.6e dones %llu bad_len_code %d "
           "stale_code %d\n", (unsigned long long)m, steps, (double)m * steps / sec, rsum,
           (unsigned long long)ndone, bad, stale);
    free(obs); free(act); free(rew); free(done);
    return bad == UUVSIM_ERR_SIZE && stale == UUVSIM_ERR_HANDLE ? 0 : 1;
}
