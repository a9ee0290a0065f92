/* c_api_example.c — the C ABI of libmig.so used from plain C (no Python, no torch): the paper's A30 example
 * queue ("example W") under the four Scheme B policies through
 * mig_simulate_host (host buffers in, host results out).
 *
 * Build: gcc -std=c11 -O2 -Iinclude examples/c_api_example.c -Lpaper_2508_18556_b200 -lmig
 *            -Wl,-rpath,$PWD/paper_2508_18556_b200 -o build/c_api_example
 * Prints one line per policy; exits 0, or 2 with the library's message when the call fails (e.g. no GPU:
 * MIG_E_CUDA — there is no CPU fallback). */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "mig.h"

int main(void) {
    mig_geometry* g = NULL;
    if (mig_geometry_load("builtin:a30-24gb", &g) != MIG_OK) {
        fprintf(stderr, "geometry: %s\n", mig_last_error());
        return 2;
    }
    /* example W (GB x 1024 = MiB): est, true, iterations, iteration ticks; all STATIC-class estimates */
    const uint32_t w[8][4] = {{10, 5, 1, 100}, {5, 5, 1, 60}, {4, 4, 1, 80}, {20, 20, 1, 50},
                              {6, 8, 4, 10},   {3, 3, 1, 30}, {11, 11, 1, 70}, {2, 2, 1, 20}};
    uint32_t jobs[8][4];
    for (int j = 0; j < 8; ++j) {
        jobs[j][0] = w[j][0] * 1024u;
        jobs[j][1] = w[j][1] * 1024u;
        jobs[j][2] = w[j][2];  /* iterations | class 0 << 16 */
        jobs[j][3] = w[j][3];
    }
    const uint64_t off[2] = {0, 8};
    mig_traces tr;
    memset(&tr, 0, sizeof(tr));
    tr.jobs = jobs;
    tr.trace_off = off;
    tr.n_traces = 1;
    tr.n_jobs = 8;
    tr.max_jobs = 8;
    mig_policy pols[4];
    const char* names[4] = {"BASELINE", "STATIC", "DYNAMIC", "FUSION_FISSION"};
    for (int k = 0; k < 4; ++k) {
        memset(&pols[k], 0, sizeof(pols[k]));
        pols[k].kind = (uint32_t)k;
        pols[k].ctx_mib = 0;
        pols[k].reconfig_ticks = 0;
        pols[k].idle_w = 30;
        pols[k].w_per_slice = 25;
        pols[k].z = 2.326;
        pols[k].eps_num = 1;
        pols[k].eps_den = 100;
        pols[k].conv_k = 3;
        pols[k].min_n = 3;
    }
    mig_trace_result res[4];
    mig_policy_totals tot[4];
    if (mig_simulate_host(g, &tr, pols, 4, res, tot) != MIG_OK) {
        fprintf(stderr, "mig_simulate_host: %s\n", mig_last_error());
        mig_geometry_free(g);
        return 2;
    }
    for (int k = 0; k < 4; ++k)
        printf("%-15s makespan %u completed %u rejected %u ooms %u decisions %u energy %llu W*ticks\n", names[k],
               res[k].makespan, res[k].completed, res[k].rejected, res[k].ooms,
               res[k].placements + res[k].waits + res[k].rejected, (unsigned long long)res[k].energy_wticks);
    mig_geometry_free(g);
    return 0;
}
