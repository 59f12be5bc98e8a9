/* solve_panda.c — a plain-C user of the HJCD-IK C ABI (include/hjcd.h): no
 * Python, no torch.  Builds a Panda-like 7-DoF chain from its modified-DH table,
 * makes reachable targets by FK of random in-limit configurations (hjcd_fk), and
 * solves them with hjcd_solve_host (host buffers; the library copies, solves,
 * copies back and synchronises).
 *
 *   gcc -O2 examples/solve_panda.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2510_07514_b200 -lhjcd -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_2510_07514_b200 -o solve_panda
 *   ./solve_panda [T]
 * Prints one line: "targets T success S max_pos_err E ms M" and exits 0 when
 * every target reached 1 mm / 1 degree. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include <cuda_runtime.h>

#include "hjcd.h"

#define CHECK(x)                                                                   \
    do {                                                                           \
        hjcd_status s_ = (x);                                                      \
        if (s_ != HJCD_OK) {                                                       \
            fprintf(stderr, "%s: %s (%s)\n", #x, hjcd_status_string(s_), hjcd_last_cuda_error()); \
            return 2;                                                              \
        }                                                                          \
    } while (0)

int main(int argc, char** argv) {
    const int T = argc > 1 ? atoi(argv[1]) : 256;
    /* Craig modified DH: a_{i-1}, d_i, alpha_{i-1}, lo, hi */
    const double mdh[7][5] = {{0.0, 0.333, 0.0, -2.8973, 2.8973},
                              {0.0, 0.0, -M_PI / 2, -1.7628, 1.7628},
                              {0.0, 0.316, M_PI / 2, -2.8973, 2.8973},
                              {0.0825, 0.0, M_PI / 2, -3.0718, -0.0698},
                              {-0.0825, 0.384, -M_PI / 2, -2.8973, 2.8973},
                              {0.0, 0.0, M_PI / 2, -0.0175, 3.7525},
                              {0.088, 0.0, M_PI / 2, -2.8973, 2.8973}};
    hjcd_joint j[7];
    for (int i = 0; i < 7; ++i) {
        const double a = mdh[i][0], d = mdh[i][1], al = mdh[i][2];
        memset(&j[i], 0, sizeof(j[i]));
        j[i].type = HJCD_REVOLUTE;
        j[i].origin_xyz[0] = a;
        j[i].origin_xyz[1] = -d * sin(al);
        j[i].origin_xyz[2] = d * cos(al);
        j[i].origin_quat_wxyz[0] = cos(al / 2);
        j[i].origin_quat_wxyz[1] = sin(al / 2);
        j[i].axis[2] = 1.0;
        j[i].lo = mdh[i][3];
        j[i].hi = mdh[i][4];
    }
    const double ee_xyz[3] = {0.0, 0.0, 0.107}, ee_q[4] = {1.0, 0.0, 0.0, 0.0};
    hjcd_robot* robot = NULL;
    CHECK(hjcd_robot_create(j, 7, ee_xyz, ee_q, &robot));
    const int n = hjcd_robot_dof(robot);

    /* reachable targets: FK of random in-limit configurations */
    float* q_h = (float*)malloc(sizeof(float) * T * n);
    srand(7);
    for (int t = 0; t < T; ++t)
        for (int k = 0; k < n; ++k) {
            const double u = (rand() + 0.5) / ((double)RAND_MAX + 1.0);
            q_h[t * n + k] = (float)(j[k].lo + u * (j[k].hi - j[k].lo));
        }
    float *q_d, *tg_d;
    cudaMalloc((void**)&q_d, sizeof(float) * T * n);
    cudaMalloc((void**)&tg_d, sizeof(float) * T * 7);
    cudaMemcpy(q_d, q_h, sizeof(float) * T * n, cudaMemcpyHostToDevice);
    CHECK(hjcd_fk(robot, q_d, T, tg_d, NULL, NULL));
    float* tg_h = (float*)malloc(sizeof(float) * T * 7);
    cudaMemcpy(tg_h, tg_d, sizeof(float) * T * 7, cudaMemcpyDeviceToHost);

    hjcd_config cfg;
    hjcd_config_default(&cfg);   /* M = 1000, K = 50, B = 100, readings */
    size_t ws_bytes = 0;
    CHECK(hjcd_workspace_size_host(robot, T, &cfg, &ws_bytes));
    void* ws = NULL;
    cudaMalloc(&ws, ws_bytes);   /* cudaMalloc is 256-byte aligned */

    float* sol = (float*)malloc(sizeof(float) * T * n);
    float* pe = (float*)malloc(sizeof(float) * T);
    float* oe = (float*)malloc(sizeof(float) * T);
    int32_t* st = (int32_t*)malloc(sizeof(int32_t) * T);
    CHECK(hjcd_solve_host(robot, &cfg, tg_h, T, sol, pe, oe, st, ws, ws_bytes, NULL));   /* warm-up */
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    CHECK(hjcd_solve_host(robot, &cfg, tg_h, T, sol, pe, oe, st, ws, ws_bytes, NULL));
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double ms = (t1.tv_sec - t0.tv_sec) * 1e3 + (t1.tv_nsec - t0.tv_nsec) * 1e-6;

    int ok = 0;
    float emax = 0.f;
    for (int t = 0; t < T; ++t) {
        if (st[t] <= HJCD_TARGET_SUCCESS) ok++;
        if (pe[t] > emax) emax = pe[t];
    }
    printf("targets %d success %d max_pos_err %.3g ms %.3f\n", T, ok, emax, ms);
    cudaFree(ws);
    cudaFree(q_d);
    cudaFree(tg_d);
    free(q_h); free(tg_h); free(sol); free(pe); free(oe); free(st);
    hjcd_robot_destroy(robot);
    return ok == T ? 0 : 1;
}
