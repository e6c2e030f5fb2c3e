/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the sparse arithmetic on the BSGD-TV epoch path, used
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm as the checker and the CPU baseline.  Never linked into, loaded by, or
 * called from the product package (paper_1812_01307_b200/).
 *
 * The reference reaches these products through `blk @ x` and `blk.T @ r`
 * (`pkg/src/bsgdtv/blockops.py:207-223`), i.e. scipy's C++ sparsetools, a
 * third-party dependency absent from /root/reference (scipy >= 1.8 unpinned
 * in `pkg/pyproject.toml:13`; 1.18.1 installed here and on the GPU box).
 * Restated published algorithms:
 *   csr_matvec (sparsetools/csr.h): y[i] = 0; y[i] += A[k] * x[col[k]] for k
 *       ascending inside row i -- one multiply and one add per term, no FMA.
 *   csc_matvec applied to blk.T (a CSC view of the CSR block): for every block
 *       row in ascending order, out[col] += A[k] * r[row].
 * Block (i, j) is the row range [r0, r1) restricted to columns [c0, c1); since
 * every row's indices are sorted (`blockops.py:125-126`) the block's entries
 * in a row are one contiguous run, found here by binary search.  Products run
 * in exactly the reference order, so results are bit-identical to scipy
 * (compile with -ffp-contract=off, see oracle/Makefile).
 *
 * OpenMP parallelism is over independent (i, j) block pairs only, mirroring
 * the reference's executor (`solvers.py:281-290`); each pair writes its own
 * output slot, so results do not depend on the thread count.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int64_t lower_bound_i32(const int32_t *a, int64_t lo, int64_t hi, int64_t key)
{
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if ((int64_t)a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

#define VAL(k) (vdt == 4 ? (double)((const float *)data)[k] : ((const double *)data)[k])

/* z = A[r0:r1, c0:c1] @ xj  (csr_matvec order) */
void orc_block_matvec(int vdt, const int64_t *indptr, const int32_t *indices, const void *data,
                      int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                      const double *xj, double *out)
{
    for (int64_t row = r0; row < r1; ++row) {
        int64_t lo = lower_bound_i32(indices, indptr[row], indptr[row + 1], c0);
        int64_t hi = lower_bound_i32(indices, lo, indptr[row + 1], c1);
        double s = 0.0;
        for (int64_t k = lo; k < hi; ++k) {
            double prod = VAL(k) * xj[indices[k] - c0];
            s = s + prod;
        }
        out[row - r0] = s;
    }
}

/* g = A[r0:r1, c0:c1]^T @ ri  (csc_matvec order on the transposed view) */
void orc_block_rmatvec(int vdt, const int64_t *indptr, const int32_t *indices, const void *data,
                       int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                       const double *ri, double *out)
{
    memset(out, 0, sizeof(double) * (size_t)(c1 - c0));
    for (int64_t row = r0; row < r1; ++row) {
        int64_t lo = lower_bound_i32(indices, indptr[row], indptr[row + 1], c0);
        int64_t hi = lower_bound_i32(indices, lo, indptr[row + 1], c1);
        const double rv = ri[row - r0];
        for (int64_t k = lo; k < hi; ++k) {
            double prod = VAL(k) * rv;
            out[indices[k] - c0] = out[indices[k] - c0] + prod;
        }
    }
}

/*
 * All per-pair products of one epoch (`solvers.py:281-290`).  For pair k =
 * (pi[k], pj[k]): zbuf[zoff[k] : zoff[k] + |I_i|] = A_ij x_k[J_j] and
 * gbuf[goff[k] : goff[k] + |J_j|] = A_ij^T r_k[I_i].  Returns the nnz charged.
 */
int64_t orc_pair_products(int vdt, const int64_t *indptr, const int32_t *indices, const void *data,
                          const int64_t *row_bounds, const int64_t *col_bounds,
                          int64_t npairs, const int64_t *pi, const int64_t *pj,
                          const double *x, const double *r,
                          const int64_t *zoff, double *zbuf,
                          const int64_t *goff, double *gbuf, int nthreads)
{
    int64_t charged = 0;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(+ : charged)
#endif
    for (int64_t k = 0; k < npairs; ++k) {
        const int64_t i = pi[k], j = pj[k];
        const int64_t r0 = row_bounds[i], r1 = row_bounds[i + 1];
        const int64_t c0 = col_bounds[j], c1 = col_bounds[j + 1];
        orc_block_rmatvec(vdt, indptr, indices, data, r0, r1, c0, c1, r + r0, gbuf + goff[k]);
        orc_block_matvec(vdt, indptr, indices, data, r0, r1, c0, c1, x + c0, zbuf + zoff[k]);
        int64_t nz = 0;
        for (int64_t row = r0; row < r1; ++row) {
            int64_t lo = lower_bound_i32(indices, indptr[row], indptr[row + 1], c0);
            nz += lower_bound_i32(indices, lo, indptr[row + 1], c1) - lo;
        }
        charged += 2 * nz;
    }
    return charged;
}

/*
 * Full A @ x assembled from block products in ascending j
 * (`blockops.py:237-243`: acc = z_0; acc = acc + z_j), parallel over row blocks.
 * scratch must hold N * max|I_i| doubles per thread-free row block: we use
 * one |I_i| accumulator per row computed on the fly instead.
 */
void orc_matvec(int vdt, const int64_t *indptr, const int32_t *indices, const void *data,
                int64_t M, int64_t N, const int64_t *row_bounds, const int64_t *col_bounds,
                const double *x, double *out, int nthreads)
{
    (void)M;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int64_t row = 0; row < row_bounds[M]; ++row) {
        double acc = 0.0;
        int64_t lo = indptr[row];
        for (int64_t j = 0; j < N; ++j) {
            const int64_t c0 = col_bounds[j], c1 = col_bounds[j + 1];
            int64_t hi = lower_bound_i32(indices, lo, indptr[row + 1], c1);
            double s = 0.0;
            for (int64_t k = lo; k < hi; ++k) {
                double prod = VAL(k) * x[indices[k]];
                s = s + prod;
            }
            (void)c0;
            acc = (j == 0) ? s : acc + s;
            lo = hi;
        }
        out[row] = acc;
    }
}

/*
 * Full A^T @ w assembled from block products in ascending i
 * (`blockops.py:254-260`: acc = t_0; acc = acc + t_i), parallel over column
 * blocks.  tscratch holds cols doubles.
 */
void orc_rmatvec(int vdt, const int64_t *indptr, const int32_t *indices, const void *data,
                 int64_t M, int64_t N, const int64_t *row_bounds, const int64_t *col_bounds,
                 const double *w, double *out, double *tscratch, int nthreads)
{
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
    for (int64_t j = 0; j < N; ++j) {
        const int64_t c0 = col_bounds[j], c1 = col_bounds[j + 1];
        double *t = tscratch + c0;
        for (int64_t i = 0; i < M; ++i) {
            const int64_t r0 = row_bounds[i], r1 = row_bounds[i + 1];
            orc_block_rmatvec(vdt, indptr, indices, data, r0, r1, c0, c1, w + r0, t);
            if (i == 0) {
                memcpy(out + c0, t, sizeof(double) * (size_t)(c1 - c0));
            } else {
                for (int64_t c = 0; c < c1 - c0; ++c) out[c0 + c] = out[c0 + c] + t[c];
            }
        }
    }
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
