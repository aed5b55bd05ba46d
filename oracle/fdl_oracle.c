/*
 * fdl_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU reference of the quantities the SOR stress-majorization
 * layout computes (Wang & Wang, PAPER.md).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header or table with the CUDA path
 * (paper_1711_01228_b200/csrc), and the CUDA path never calls it.
 *
 * Every routine is the definition written out as scalar loops, in the paper's
 * notation, with no blocking or reordering beyond "rows may run on different
 * threads"; each row (or each i<j pair list of a row) is summed sequentially by
 * one thread, so results do not depend on the thread count.
 *
 * Citations: "P:n" = line n of PAPER.md, "S:n" = line n of SPEC.md.
 *   ideal distance   d_ij = k * hop(i,j)   ("predefined ideal distance";
 *                                            reading S:49-57)
 *   weight           w_ij = d_ij^alpha, alpha = -2
 *   stress  f(X) = sum_{i<j} w_ij (||x_i - x_j|| - d_ij)^2            Eq. 1
 *   L^W   l_ij = -w_ij (i != j), l_ii = -sum_{k!=i} l_ik
 *   L^Y   l_ij = 0 if y_i == y_j, else -w_ij d_ij / ||y_i - y_j||
 *   so (L^W X)_i = sum_{j!=i} w_ij (x_i - x_j)
 *      (L^Y Y)_i = sum_{j!=i, y_j!=y_i} w_ij d_ij (y_i - y_j)/||y_i - y_j||
 *
 * Hop matrices are passed as uint16 (n_rows x n, row-major); 0 on the diagonal.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ BFS --
 * Unweighted single-source shortest paths (breadth-first search), the ideal
 * distance reading of S:52 ("BFS when all lengths are unit").  dist[v] = -1
 * for unreached vertices.  Returns the number of reached vertices. */
int64_t orc_bfs(int32_t n, const int64_t* row_ptr, const int32_t* col, int32_t src, int32_t* dist)
{
    int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int64_t head = 0, tail = 0;
    for (int32_t v = 0; v < n; ++v) dist[v] = -1;
    dist[src] = 0;
    queue[tail++] = src;
    while (head < tail) {
        int32_t u = queue[head++];
        for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e) {
            int32_t v = col[e];
            if (dist[v] < 0) {
                dist[v] = dist[u] + 1;
                queue[tail++] = v;
            }
        }
    }
    free(queue);
    return tail;
}

/* Hop rows for a list of sources: out[s*n + v] = hop(srcs[s], v).
 * Returns the largest hop seen, -1 if some source does not reach every vertex
 * (disconnected graph), -2 if a hop exceeds 65535. */
int32_t orc_hop_rows(int32_t n, const int64_t* row_ptr, const int32_t* col,
                     int32_t nsrc, const int32_t* srcs, uint16_t* out)
{
    int32_t worst = 0;
    int bad = 0, big = 0;
#pragma omp parallel
    {
        int32_t* dist = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        int32_t local_max = 0;
#pragma omp for schedule(dynamic, 4)
        for (int32_t s = 0; s < nsrc; ++s) {
            int64_t reached = orc_bfs(n, row_ptr, col, srcs[s], dist);
            if (reached != n) {
#pragma omp atomic write
                bad = 1;
            }
            uint16_t* row = out + (size_t)s * (size_t)n;
            for (int32_t v = 0; v < n; ++v) {
                int32_t h = dist[v];
                if (h > 65535) {
#pragma omp atomic write
                    big = 1;
                    h = 65535;
                }
                if (h < 0) h = 0;
                row[v] = (uint16_t)h;
                if (h > local_max) local_max = h;
            }
        }
#pragma omp critical
        {
            if (local_max > worst) worst = local_max;
        }
        free(dist);
    }
    if (bad) return -1;
    if (big) return -2;
    return worst;
}

static inline double ideal_d(double k, uint16_t h) { return k * (double)h; }
static inline double weight(double d, double alpha) { return pow(d, alpha); }

/* Per-call table of (d_h, w_h) for h = 0..hmax, filled from the two
 * definitions above (d = k*h, w = d^alpha); entry 0 is never used for i != j.
 * Only a cache of the same values -- pow() per pair is 20x slower. */
typedef struct { double* d; double* w; } dw_table;

/* Largest hop of a matrix (sizes the table); a max over threads -- the table's values
 * do not depend on how it is found.  (A serial scan of a full C4 matrix, 4.8 GB, cost
 * ~1 s per call, i.e. most of an oracle iteration.) */
static uint16_t max_hop(const uint16_t* h, size_t count)
{
    uint16_t m = 0;
#pragma omp parallel for reduction(max : m) schedule(static)
    for (size_t t = 0; t < count; ++t) if (h[t] > m) m = h[t];
    return m;
}

static dw_table make_table(double k, double alpha, uint16_t hmax)
{
    dw_table t;
    t.d = (double*)malloc(sizeof(double) * ((size_t)hmax + 1));
    t.w = (double*)malloc(sizeof(double) * ((size_t)hmax + 1));
    for (uint32_t h = 0; h <= hmax; ++h) {
        t.d[h] = ideal_d(k, (uint16_t)h);
        t.w[h] = h ? weight(t.d[h], alpha) : 0.0;
    }
    return t;
}

static void free_table(dw_table t) { free(t.d); free(t.w); }

static inline double dist_ij(const double* X, int32_t dim, int64_t i, int64_t j)
{
    double s = 0.0;
    for (int32_t c = 0; c < dim; ++c) {
        double t = X[i * dim + c] - X[j * dim + c];
        s += t * t;
    }
    return sqrt(s);
}

static inline int same_point(const double* X, int32_t dim, int64_t i, int64_t j)
{
    for (int32_t c = 0; c < dim; ++c)
        if (X[i * dim + c] != X[j * dim + c]) return 0;
    return 1;
}

/* ---------------------------------------------------------------- stress --
 * Eq. 1 over all pairs i<j.  hop is the full n x n matrix.
 * Row i sums j = i+1..n-1 sequentially; row partials are then summed in
 * increasing i. */
double orc_stress(int32_t n, int32_t dim, const double* X, const uint16_t* hop,
                  double k, double alpha)
{
    dw_table t = make_table(k, alpha, max_hop(hop, (size_t)n * (size_t)n));
    double* part = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t j = i + 1; j < n; ++j) {
            uint16_t h = hop[i * (int64_t)n + j];
            double d = t.d[h], w = t.w[h];
            double r = dist_ij(X, dim, i, j);
            acc += w * (r - d) * (r - d);
        }
        part[i] = acc;
    }
    double f = 0.0;
    for (int64_t i = 0; i < n; ++i) f += part[i];
    free(part);
    free_table(t);
    return f;
}

/* Per-row ordered stress s_i = sum_{j != i} w_ij (||x_i - x_j|| - d_ij)^2, so that
 * f = 1/2 sum_i s_i (Eq. 1).  rows[] lists global row ids, hoprows[r*n + j] is
 * hop(rows[r], j).  Used for sampled parity at sizes where the full matrix
 * does not fit. */
void orc_stress_rows(int32_t n, int32_t dim, const double* X, int32_t nrows, const int32_t* rows,
                     const uint16_t* hoprows, double k, double alpha, double* s_out)
{
    dw_table t = make_table(k, alpha, max_hop(hoprows, (size_t)nrows * (size_t)n));
#pragma omp parallel for schedule(dynamic, 4)
    for (int32_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        const uint16_t* hrow = hoprows + (size_t)r * (size_t)n;
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double d = t.d[hrow[j]], w = t.w[hrow[j]];
            double rr = dist_ij(X, dim, i, j);
            acc += w * (rr - d) * (rr - d);
        }
        s_out[r] = acc;
    }
    free_table(t);
}

/* ------------------------------------------------------------- L^Y Y rows --
 * (L^Y Y)_i for Y = X (the right-hand side of Eq. 2-5; L^Y from
 * Prop. 2.1, including the coincident rule y_i = y_j -> 0). */
void orc_ly_rows(int32_t n, int32_t dim, const double* X, int32_t nrows, const int32_t* rows,
                 const uint16_t* hoprows, double k, double alpha, double* out)
{
    dw_table t = make_table(k, alpha, max_hop(hoprows, (size_t)nrows * (size_t)n));
#pragma omp parallel for schedule(dynamic, 4)
    for (int32_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        const uint16_t* hrow = hoprows + (size_t)r * (size_t)n;
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            if (same_point(X, dim, i, j)) continue;       /* l_ij = 0 branch */
            double d = t.d[hrow[j]], w = t.w[hrow[j]];
            double rr = dist_ij(X, dim, i, j);
            double c = w * d / rr;                         /* -l^Y_ij */
            for (int32_t q = 0; q < dim; ++q) acc[q] += c * (X[i * dim + q] - X[j * dim + q]);
        }
        for (int32_t q = 0; q < dim; ++q) out[(size_t)r * dim + q] = acc[q];
    }
    free_table(t);
}

/* ------------------------------------------------------------- L^W X rows --
 * (L^W X)_i = sum_{j != i} w_ij (x_i - x_j), from l_ij = -w_ij and
 * l_ii = sum_{k != i} w_ik. */
void orc_lw_rows(int32_t n, int32_t dim, const double* X, int32_t nrows, const int32_t* rows,
                 const uint16_t* hoprows, double k, double alpha, double* out)
{
    dw_table t = make_table(k, alpha, max_hop(hoprows, (size_t)nrows * (size_t)n));
#pragma omp parallel for schedule(dynamic, 4)
    for (int32_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        const uint16_t* hrow = hoprows + (size_t)r * (size_t)n;
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double w = t.w[hrow[j]];
            for (int32_t q = 0; q < dim; ++q) acc[q] += w * (X[i * dim + q] - X[j * dim + q]);
        }
        for (int32_t q = 0; q < dim; ++q) out[(size_t)r * dim + q] = acc[q];
    }
    free_table(t);
}

/* Dense L^W (n x n, row-major) from the full hop matrix. */
void orc_lw_dense(int32_t n, const uint16_t* hop, double k, double alpha, double* L)
{
    dw_table t = make_table(k, alpha, max_hop(hop, (size_t)n * (size_t)n));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double diag = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) { L[i * n + j] = 0.0; continue; }
            double w = t.w[hop[i * (int64_t)n + j]];
            L[i * n + j] = -w;
            diag += w;
        }
        L[i * n + i] = diag;
    }
    free_table(t);
}

/* Gansner's reduced matrix: L^W with its first row and first column
 * removed, (n-1) x (n-1) row-major, written directly so no n x n copy is
 * needed before factorisation. */
void orc_lw_red_dense(int32_t n, const uint16_t* hop, double k, double alpha, double* Lr)
{
    dw_table t = make_table(k, alpha, max_hop(hop, (size_t)n * (size_t)n));
    int64_t m = (int64_t)n - 1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 1; i < n; ++i) {
        double diag = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double w = t.w[hop[i * (int64_t)n + j]];
            diag += w;                                   /* l_ii = sum_{k != i} w_ik */
            if (j >= 1) Lr[(i - 1) * m + (j - 1)] = -w;  /* l_ij = -w_ij */
        }
        Lr[(i - 1) * m + (i - 1)] = diag;
    }
    free_table(t);
}

/* Reduced matrix-vector product for Gansner's pinned system:
 * vertex 0 fixed at the origin, row/column 0 deleted.  For i >= 1 and each
 * column c,
 *   y_ic = (sum_{j != i} w_ij) p_ic - sum_{j >= 1, j != i} w_ij p_jc ,
 * p is n x ncols row-major with row 0 ignored (treated as 0); y row 0 = 0.
 * hop is the full matrix. */
void orc_lw_red_matvec(int32_t n, int32_t ncols, const double* p, const uint16_t* hop,
                       double k, double alpha, double* y)
{
    dw_table t = make_table(k, alpha, max_hop(hop, (size_t)n * (size_t)n));
    for (int32_t c = 0; c < ncols; ++c) y[c] = 0.0;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 1; i < n; ++i) {
        double diag = 0.0, off[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double w = t.w[hop[i * (int64_t)n + j]];
            diag += w;
            if (j >= 1)
                for (int32_t c = 0; c < ncols; ++c) off[c] += w * p[j * ncols + c];
        }
        for (int32_t c = 0; c < ncols; ++c) y[i * ncols + c] = diag * p[i * ncols + c] - off[c];
    }
    free_table(t);
}

/* Diagonal of L^W: sum_{j != i} w_ij (Jacobi preconditioner). */
void orc_lw_diag(int32_t n, const uint16_t* hop, double k, double alpha, double* diag)
{
    dw_table t = make_table(k, alpha, max_hop(hop, (size_t)n * (size_t)n));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            s += t.w[hop[i * (int64_t)n + j]];
        }
        diag[i] = s;
    }
    free_table(t);
}

/* Diagonal entries sum_{j != i} w_ij of L^W for listed rows (hoprows as in
 * orc_stress_rows). */
void orc_lw_diag_rows(int32_t n, int32_t nrows, const int32_t* rows, const uint16_t* hoprows,
                      double k, double alpha, double* out)
{
    dw_table t = make_table(k, alpha, max_hop(hoprows, (size_t)nrows * (size_t)n));
#pragma omp parallel for schedule(dynamic, 4)
    for (int32_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        const uint16_t* hrow = hoprows + (size_t)r * (size_t)n;
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j)
            if (j != i) s += t.w[hrow[j]];
        out[r] = s;
    }
    free_table(t);
}

/* C = sum_{i<j} w_ij d_ij^2, the constant of Eq. 2. */
double orc_const_c(int32_t n, const uint16_t* hop, double k, double alpha)
{
    dw_table t = make_table(k, alpha, max_hop(hop, (size_t)n * (size_t)n));
    double* part = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t j = i + 1; j < n; ++j) {
            uint16_t h = hop[i * (int64_t)n + j];
            acc += t.w[h] * t.d[h] * t.d[h];
        }
        part[i] = acc;
    }
    double c = 0.0;
    for (int64_t i = 0; i < n; ++i) c += part[i];
    free(part);
    free_table(t);
    return c;
}

int32_t orc_num_threads(void)
{
#ifdef _OPENMP
    return (int32_t)omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_threads(int32_t t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
