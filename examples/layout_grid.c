/*
 * layout_grid.c -- the C ABI used from plain C (no Python, no torch): lay out an
 * R x C grid graph (BASELINE config C1 is 10 x 10) with Algorithm 2 and print the
 * run summary and the first positions.
 *
 * Build: gcc -O2 -I include examples/layout_grid.c -o layout_grid \
 *            -L paper_1711_01228_b200/lib -lfdl -Wl,-rpath,$PWD/paper_1711_01228_b200/lib
 * Run:   ./layout_grid [rows cols]            (needs a GPU)
 *        ./layout_grid --check-errors         (no GPU needed: input validation only)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "fdl.h"

/* CSR of the rows x cols grid (4-neighbourhood), both directions stored */
static void grid_csr(int rows, int cols, int64_t* rp, int32_t* col)
{
    int64_t e = 0;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            const int v = r * cols + c;
            rp[v] = e;
            if (r > 0) col[e++] = v - cols;
            if (c > 0) col[e++] = v - 1;
            if (c + 1 < cols) col[e++] = v + 1;
            if (r + 1 < rows) col[e++] = v + cols;
        }
    rp[rows * cols] = e;
}

static int check_errors(void)
{
    /* two disconnected edges: rejected before any GPU work */
    const int64_t rp[5] = {0, 1, 2, 3, 4};
    const int32_t col[4] = {1, 0, 3, 2};
    fdl_params p;
    fdl_params_default(&p);
    fdl_ctx* ctx = (fdl_ctx*)1;
    fdl_status s = fdl_create(4, rp, col, NULL, &p, NULL, &ctx);
    printf("disconnected: %s, ctx %s\n", fdl_status_str(s), ctx == NULL ? "NULL" : "set");
    if (s != FDL_E_DISCONNECTED || ctx != NULL) return 1;
    /* a self-loop */
    const int64_t rp2[3] = {0, 2, 3};
    const int32_t col2[3] = {0, 1, 0};
    s = fdl_create(2, rp2, col2, NULL, &p, NULL, &ctx);
    printf("self loop: %s\n", fdl_status_str(s));
    if (s != FDL_E_SELF_LOOP) return 1;
    /* a bad parameter */
    p.omega = -1.0;
    const int64_t rp3[3] = {0, 1, 2};
    const int32_t col3[2] = {1, 0};
    s = fdl_create(2, rp3, col3, NULL, &p, NULL, &ctx);
    printf("omega < 0: %s\n", fdl_status_str(s));
    if (s != FDL_E_INVALID_ARG) return 1;
    printf("abi %d ok\n", fdl_abi_version());
    return 0;
}

int main(int argc, char** argv)
{
    if (argc > 1 && argv[1][0] == '-') return check_errors();
    /* layout_grid ROWS COLS [X0_FILE OUT_FILE]: the optional files hold n*2 doubles
       (row-major): the initial placement, and the final one written back */
    const int rows = argc > 2 ? atoi(argv[1]) : 10, cols = argc > 2 ? atoi(argv[2]) : 10;
    const char* x0_file = argc > 4 ? argv[3] : NULL;
    const char* out_file = argc > 4 ? argv[4] : NULL;
    const int n = rows * cols;
    int64_t* rp = malloc(sizeof(int64_t) * (n + 1));
    int32_t* col = malloc(sizeof(int32_t) * 4 * n);
    double* X = malloc(sizeof(double) * 2 * n);
    grid_csr(rows, cols, rp, col);

    fdl_params p;
    fdl_params_default(&p); /* omega 1.5, tol 1e-4, w = d^-2 */
    p.dim = 2;
    p.k = sqrt(1.0 / n); /* C1's ideal edge length */
    p.tol = 1e-6;        /* Table 1's rel err for n <= 86 .. C1 (DESIGN R5) */
    p.seed = 7;          /* initial placement uniform in the unit square */

    double* X0 = NULL;
    if (x0_file) {
        FILE* f = fopen(x0_file, "rb");
        X0 = malloc(sizeof(double) * 2 * n);
        if (!f || fread(X0, sizeof(double), (size_t)2 * n, f) != (size_t)2 * n) {
            fprintf(stderr, "cannot read %s\n", x0_file);
            return 1;
        }
        fclose(f);
    }
    fdl_ctx* ctx = NULL;
    fdl_status s = fdl_create(n, rp, col, NULL, &p, X0, &ctx);
    if (s != FDL_OK) {
        fprintf(stderr, "fdl_create: %s\n", fdl_status_str(s));
        return 1;
    }
    fdl_run_info info;
    s = fdl_run_until_converged(ctx, &info);
    if (s != FDL_OK) {
        fprintf(stderr, "fdl_run_until_converged: %s (%s)\n", fdl_status_str(s), fdl_last_error(ctx));
        fdl_destroy(ctx);
        return 1;
    }
    fdl_get_positions(ctx, X, (size_t)2 * n);
    printf("grid %dx%d: %d iterations, %d relaxations accepted, %d PCG iterations, f %.6g -> %.6g\n", rows, cols,
           info.iterations, info.accepted, info.cg_iters, info.f_initial, info.f_final);
    printf("x_0 = (%.3g, %.3g)  x_1 = (%.6f, %.6f)  |x_1 - x_0| / k = %.4f\n", X[0], X[1], X[2], X[3],
           sqrt(X[2] * X[2] + X[3] * X[3]) / p.k);
    if (out_file) {
        FILE* f = fopen(out_file, "wb");
        if (!f || fwrite(X, sizeof(double), (size_t)2 * n, f) != (size_t)2 * n) {
            fprintf(stderr, "cannot write %s\n", out_file);
            return 1;
        }
        fclose(f);
    }
    fdl_destroy(ctx);
    free(rp);
    free(col);
    free(X);
    free(X0);
    return info.f_final < info.f_initial ? 0 : 1;
}
