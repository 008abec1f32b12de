/*
 * oracle_kernels.c -- CPU restatement of the reference's compiled kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is part of the parity oracle: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path (paper_1706_05988_b200)
 * never links or calls it.
 *
 * Every function restates one numba kernel of the reference package `kpl`
 * (pkg/src/kpl/_kernels.py) with the same floating-point operation order.
 * Build flags (oracle/Makefile) pin -O2 -ffp-contract=off -fno-fast-math so
 * that no multiply-add is contracted: the reference's numba asm has separate
 * vmulsd / vaddsd.
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>

/* pkg/src/kpl/_kernels.py:15-41  blocked_dot: 8 interleaved lanes over k mod 8,
 * fixed merge ((a0+a1)+(a2+a3))+((a4+a5)+(a6+a7)), then + sequential tail. */
double orc_blocked_dot(int64_t n, const double *u, const double *v)
{
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    double a4 = 0.0, a5 = 0.0, a6 = 0.0, a7 = 0.0;
    int64_t lim = n - (n % 8);
    int64_t k = 0;
    while (k < lim) {
        a0 += u[k] * v[k];
        a1 += u[k + 1] * v[k + 1];
        a2 += u[k + 2] * v[k + 2];
        a3 += u[k + 3] * v[k + 3];
        a4 += u[k + 4] * v[k + 4];
        a5 += u[k + 5] * v[k + 5];
        a6 += u[k + 6] * v[k + 6];
        a7 += u[k + 7] * v[k + 7];
        k += 8;
    }
    double tail = 0.0;
    for (int64_t j = lim; j < n; ++j)
        tail += u[j] * v[j];
    return (((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7))) + tail;
}

/* pkg/src/kpl/_kernels.py:44-52  csr_matvec: acc starts at +0.0 and
 * accumulates values[k]*v[col_idx[k]] left to right within each row. */
void orc_csr_matvec(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                    const double *values, const double *v, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
            acc += values[k] * v[col_idx[k]];
        out[i] = acc;
    }
}

/* Matrix-free form of csr_matvec applied to the unscaled Dirichlet Laplacian
 * (pkg/src/kpl/sparse.py:188-214 for 2D; the 3D 7-point analogue of
 * SURVEY.md Appendix C).  Grid (NX, NY, NZ), id = x + NX*(y + NY*z); the 2D
 * grid nx-by-ny is (NX, NY, NZ) = (nx, 1, ny).  Terms are added in ascending
 * column order (id-NX*NY, id-NX, id-1, id, id+1, id+NX, id+NX*NY) starting
 * from +0.0 and only for neighbours that exist, exactly like the CSR rows the
 * generator assembles, so the result equals csr_matvec bit for bit. */
void orc_stencil_matvec(int64_t NX, int64_t NY, int64_t NZ, double diag,
                        const double *v, double *out)
{
    const int64_t sxy = NX * NY;
    for (int64_t z = 0; z < NZ; ++z)
        for (int64_t y = 0; y < NY; ++y)
            for (int64_t x = 0; x < NX; ++x) {
                const int64_t id = x + NX * (y + NY * z);
                double acc = 0.0;
                if (z > 0) acc += -1.0 * v[id - sxy];
                if (y > 0) acc += -1.0 * v[id - NX];
                if (x > 0) acc += -1.0 * v[id - 1];
                acc += diag * v[id];
                if (x < NX - 1) acc += -1.0 * v[id + 1];
                if (y < NY - 1) acc += -1.0 * v[id + NX];
                if (z < NZ - 1) acc += -1.0 * v[id + sxy];
                out[id] = acc;
            }
}

/* pkg/src/kpl/_kernels.py:55-63  lower_solve: forward substitution with a
 * lower-triangular CSR factor whose diagonal is the last entry of each row;
 * acc starts at b[i] and subtracts values[k]*out[col] in stored order, then
 * one division by the diagonal. */
void orc_lower_solve(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                     const double *values, const double *b, double *out)
{
    for (int64_t i = 0; i < n; ++i) {
        const int64_t d = row_ptr[i + 1] - 1;
        double acc = b[i];
        for (int64_t k = row_ptr[i]; k < d; ++k)
            acc -= values[k] * out[col_idx[k]];
        out[i] = acc / values[d];
    }
}

/* pkg/src/kpl/_kernels.py:66-74  upper_solve: backward substitution with the
 * transposed factor (diagonal first in each row), rows from n-1 down. */
void orc_upper_solve(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                     const double *values, const double *b, double *out)
{
    for (int64_t i = n - 1; i >= 0; --i) {
        const int64_t d = row_ptr[i];
        double acc = b[i];
        for (int64_t k = d + 1; k < row_ptr[i + 1]; ++k)
            acc -= values[k] * out[col_idx[k]];
        out[i] = acc / values[d];
    }
}

/* pkg/src/kpl/_kernels.py:77-115  ic0_factor: row-by-row IC(0) on the
 * lower pattern (sorted columns, diagonal last).  Off-diagonal (i, c):
 * s = a - sum over the shared strictly-lower columns (merge walk, ascending)
 * of l[i,*] * l[c,*], then s / l[c,c]; the pivot is a[i,i] - sum l[i,k]^2 in
 * row order, square-rooted.  Returns -1, or the first row with pivot <= 0. */
int64_t orc_ic0_factor(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                       const double *a_values, double *l_values)
{
    for (int64_t i = 0; i < n; ++i) {
        const int64_t lo = row_ptr[i], di = row_ptr[i + 1] - 1;
        for (int64_t kk = lo; kk < di; ++kk) {
            const int64_t c = col_idx[kk];
            const int64_t dc = row_ptr[c + 1] - 1;
            double s = a_values[kk];
            int64_t p = lo, q = row_ptr[c];
            while (p < kk && q < dc) {
                if (col_idx[p] == col_idx[q]) { s -= l_values[p] * l_values[q]; ++p; ++q; }
                else if (col_idx[p] < col_idx[q]) ++p;
                else ++q;
            }
            l_values[kk] = s / l_values[dc];
        }
        double d = a_values[di];
        for (int64_t kk = lo; kk < di; ++kk)
            d -= l_values[kk] * l_values[kk];
        if (d <= 0.0)
            return i;
        l_values[di] = sqrt(d);
    }
    return -1;
}
