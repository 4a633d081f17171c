/* c_abi_demo.c — the C ABI used from plain C (no Python, no torch).
 *
 * Builds a 3-op chain on 2 devices, evaluates every placement on the GPU and
 * prints the best one; without a GPU it reports MP_ERR_NO_GPU and exits 0.
 *
 *   gcc -std=c11 -I include examples/c_abi_demo.c -L paper_2312_04025_b200 \
 *       -lmoirai_b200 -Wl,-rpath,$PWD/paper_2312_04025_b200 -o c_abi_demo
 */
#include <stdint.h>
#include <stdio.h>

#include "moirai_b200.h"

int main(void) {
    /* op i on device k takes cost[i*2+k] seconds; flows 0->1, 1->2 */
    const double cost[6] = {2.0, 4.0, 1.0, 0.5, 3.0, 1.0};
    const int64_t mem[3] = {10, 10, 10};
    const int32_t src[2] = {0, 1}, dst[2] = {1, 2};
    const int64_t payload[2] = {10000000, 20000000};
    const int64_t cap[2] = {100, 100};
    const double bw[4] = {0.0, 5e6, 5e6, 0.0};
    mp_problem prob = {3, 2, 2, cost, mem, src, dst, payload, cap, bw};
    mp_instance *inst = NULL;
    mp_error err;
    int32_t rc = mp_instance_create(&prob, 0, &inst, &err);
    if (rc == MP_ERR_NO_GPU) {
        printf("no GPU visible: %s (status %d, no CPU fallback)\n", err.msg, rc);
        return 0;
    }
    if (rc != MP_OK) {
        printf("mp_instance_create failed: %d %s\n", rc, err.msg);
        return 1;
    }
    uint8_t rows[8 * 3];
    for (int p = 0; p < 8; ++p)
        for (int i = 0; i < 3; ++i) rows[p * 3 + i] = (uint8_t)((p >> (2 - i)) & 1);
    double ms[8];
    int8_t st[8];
    int64_t best = -1;
    double best_ms = 0.0;
    rc = mp_evaluate_batch(inst, rows, 8, ms, st, NULL, NULL, 0, NULL, &err);
    if (rc == MP_OK) rc = mp_evaluate_argmin(inst, rows, 8, NULL, NULL, &best, &best_ms, 0, NULL, &err);
    if (rc != MP_OK) {
        printf("evaluation failed: %d %s\n", rc, err.msg);
        mp_instance_destroy(inst);
        return 1;
    }
    for (int p = 0; p < 8; ++p) printf("placement %d%d%d  makespan %a  status %d\n", rows[p * 3], rows[p * 3 + 1],
                                       rows[p * 3 + 2], ms[p], st[p]);
    printf("best row %lld makespan %a\n", (long long)best, best_ms);
    mp_instance_destroy(inst);
    return 0;
}
