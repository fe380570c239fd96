/* Plain-C use of the boundary (include/rfk.h): one Randers solve on host
 * buffers, the way a cgo/JNI/FFI binding would call it.
 *
 *   gcc -O2 -Iinclude examples/solve.c -Lpaper_2603_00035_b200 -lrfk \
 *       -Wl,-rpath,$PWD/paper_2603_00035_b200 -o solve_c
 *   ./solve_c 64 48 out.bin     # rows cols output: g11 g12 g22 b1 b2 T, rows*cols doubles each
 *
 * Fields: a smooth anisotropic metric with a constant drift (feasible), point
 * source at the centre, h = 1/rows, SolveOptions defaults. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "rfk.h"

int main(int argc, char** argv) {
    const int rows = argc > 1 ? atoi(argv[1]) : 64, cols = argc > 2 ? atoi(argv[2]) : 48;
    const char* out_path = argc > 3 ? argv[3] : NULL;
    const size_t n = (size_t)rows * cols;
    double *g11 = malloc(n * 8), *g12 = malloc(n * 8), *g22 = malloc(n * 8), *b1 = malloc(n * 8), *b2 = malloc(n * 8);
    double* t = malloc(n * 8);
    unsigned char* src = calloc(n, 1);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const size_t i = (size_t)r * cols + c;
            g11[i] = 1.0 + 0.25 * sin(0.11 * r);
            g12[i] = 0.1 * cos(0.07 * c);
            g22[i] = 1.2 + 0.2 * cos(0.05 * (r + c));
            b1[i] = 0.15;
            b2[i] = -0.05;
        }
    src[(size_t)(rows / 2) * cols + cols / 2] = 1;

    rfk_context* ctx = NULL;
    rfk_status st = rfk_create(&ctx, 0);
    if (st != RFK_OK) {
        fprintf(stderr, "rfk_create: %s\n", rfk_status_string(st));
        return 2;
    }
    rfk_fields f = {1, rows, cols, 1.0 / rows, g11, g12, g22, b1, b2, 0, src, 0, NULL};
    rfk_solve_options opt = {1e-6, 50, {0, 1, 2, 3}};
    int32_t iters = 0, conv = 0;
    st = rfk_solve(ctx, RFK_MEM_HOST, &f, &opt, t, &iters, &conv, NULL);
    if (st != RFK_OK) {
        fprintf(stderr, "rfk_solve: %s (%s)\n", rfk_status_string(st), rfk_last_error(ctx));
        return 1;
    }
    double tmax = 0.0;
    for (size_t i = 0; i < n; ++i)
        if (t[i] < 1e9 && t[i] > tmax) tmax = t[i];
    printf("iterations %d converged %d max_T %.17g launches %lld\n", iters, conv, tmax,
           (long long)rfk_launch_count(ctx));
    if (out_path) {
        FILE* fp = fopen(out_path, "wb");
        const double* planes[6] = {g11, g12, g22, b1, b2, t};
        for (int k = 0; k < 6; ++k)
            if (!fp || fwrite(planes[k], 8, n, fp) != n) return 3;
        fclose(fp);
    }
    rfk_destroy(ctx);
    free(g11), free(g12), free(g22), free(b1), free(b2), free(t), free(src);
    return 0;
}
