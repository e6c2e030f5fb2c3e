/*
 * bsgd_b200 -- C ABI of the B200-native BSGD-TV epoch path.
 *
 * Plain C types only (no torch, no C++ in the signatures).  All vector
 * pointers are DEVICE pointers to float64 arrays owned by the caller unless a
 * parameter says "host".  Every compute call is asynchronous on `stream` (a
 * cudaStream_t passed as void*, NULL = legacy default stream) and is safe to
 * capture into a CUDA graph; none of them synchronises the device.
 *
 * Status codes: BSGD_OK, BSGD_EINVAL (the reference raises ValueError),
 * BSGD_ECUDA / BSGD_ENOMEM (RuntimeError).  bsgd_last_error() returns the
 * calling thread's last message.  No C++ exception crosses this boundary.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/bsgdtv/).
 */
#ifndef BSGD_B200_H
#define BSGD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSGD_OK 0
#define BSGD_EINVAL 1
#define BSGD_ECUDA 2
#define BSGD_ENOMEM 3

/* value dtype codes = element size in bytes */
#define BSGD_F32 4
#define BSGD_F64 8

/* epoch flags */
#define BSGD_EP_R_NEXT 1u     /* compute r_next = y - A x_k (lookahead r invalid) */
#define BSGD_EP_LOOKAHEAD 2u  /* compute r_ahead = y - A x_next and f_next = ||r_ahead||^2 */
#define BSGD_EP_MONITOR 4u    /* Eq. 9 test + f_curr update (solvers.py:316-334) */
#define BSGD_EP_SKIP_GRAD 8u  /* reuse g already in args->g (step re-try, solvers.py:327-332) */
#define BSGD_EP_NO_TAIL 16u   /* caller runs bsgd_epoch_tail itself (multi-GPU) */

/* history row layout (doubles), one row per epoch */
#define BSGD_H_FNEXT 0      /* ||y - A x_next||^2 (NaN if not computed) */
#define BSGD_H_HOLDS 1      /* 1 / 0, or -1 when the monitor is off */
#define BSGD_H_XX 2         /* ||x_next||^2 */
#define BSGD_H_XE 3         /* ||x_next - x_true||^2 (0 without x_true) */
#define BSGD_H_TV 4         /* TV(image of x_next) when lam > 0, else 0 */
#define BSGD_H_PITER 5      /* prox iterations */
#define BSGD_H_PRESTART 6   /* prox restarts */
#define BSGD_H_PCONV 7      /* prox converged */
#define BSGD_H_PFELL 8      /* prox fell back to the identity */
#define BSGD_H_DG 9         /* (x_next - x_k) . g */
#define BSGD_H_DD 10        /* ||x_next - x_k||^2 */
#define BSGD_H_FCURR 11     /* f_curr used by the test */
#define BSGD_HIST_COLS 12

/* device scratch needed by the reducing helpers (residual, dot, sqdist, tv_value) */
#define BSGD_SCRATCH_BYTES 65536

typedef struct bsgd_plan bsgd_plan;

/* ProxInfo (tv.py:155-163) as written by the device */
typedef struct bsgd_prox_info {
    int32_t iterations;
    int32_t converged;
    int32_t restarts;
    int32_t fell_back;
} bsgd_prox_info;

/* One BSGD-TV epoch (bsgd_tv_iteration, solvers.py:259-341) on a resident plan. */
typedef struct bsgd_epoch_args {
    const double *x_k;        /* [cols]  snapshot x_k (solvers.py:276) */
    const double *r_k;        /* [rows]  snapshot r_k = y - A x_{k-1} (solvers.py:277) */
    const double *y;          /* [rows] */
    double *g;                /* [cols]  out: 2 A^T r_k (solvers.py:299-303); in with SKIP_GRAD */
    double *x_next;           /* [cols]  out: prox(x_k + mu g) (solvers.py:307-314) */
    double *r_next;           /* [rows]  out with R_NEXT: y - A x_k (solvers.py:297) */
    double *r_ahead;          /* [rows]  out with LOOKAHEAD: y - A x_next (solvers.py:319-320) */
    const double *x_true;     /* [cols]  or NULL */
    const int64_t *perm;      /* [cols]  vector position -> row-major pixel, NULL = identity */
    double mu;                /* state.mu_eff */
    double lam;               /* cfg.lam; prox weight = mu * lam */
    int64_t height, width;    /* image grid, height * width == cols when lam > 0 */
    int32_t max_inner_iters;  /* ProxSettings.max_inner_iters */
    double tol;               /* ProxSettings.tol */
    double *f_curr;           /* device scalar, in/out with MONITOR */
    double *history;          /* device [history_capacity x BSGD_HIST_COLS] */
    int64_t *epoch_counter;   /* device scalar: history row index, incremented per epoch */
    int64_t history_capacity;
    double *dual_objectives;  /* device [max_inner_iters + 1] or NULL */
    void *workspace;          /* device, bsgd_epoch_workspace_bytes(), zero-filled once */
    size_t workspace_bytes;
    uint32_t flags;
    int64_t depth;            /* volumes (configs[4]): depth*height*width == cols, 3D TV;
                                 0 or 1 = image (2D TV, the reference's tv.py) */
} bsgd_epoch_args;

/* --- library ----------------------------------------------------------- */
const char *bsgd_last_error(void);
int bsgd_version(void);
int bsgd_device_count(int *out);

/* --- BlockOperator (blockops.py:112-261) ------------------------------ */
/* __init__ (blockops.py:123-152): canonical CSR (sorted, summed; host
 * arrays) + partition bounds.  Uploads A and builds A^T on the device. */
int bsgd_plan_create(bsgd_plan **out, int device, int64_t rows, int64_t cols, int64_t nnz,
                     const int64_t *indptr, const int32_t *indices, const void *values,
                     int value_dtype, int64_t num_row_blocks, int64_t num_col_blocks,
                     const int64_t *row_bounds, const int64_t *col_bounds, void *stream);
/* same, from a CSR already on the device (e.g. bsgd_siddon_csr output); the
 * plan ADOPTS the three arrays (they must come from this library's allocator)
 * and frees them with the plan */
int bsgd_plan_create_device(bsgd_plan **out, int device, int64_t rows, int64_t cols, int64_t nnz,
                            int64_t *indptr, int32_t *indices, void *values, int value_dtype,
                            int64_t num_row_blocks, int64_t num_col_blocks, const int64_t *row_bounds,
                            const int64_t *col_bounds, void *stream);
/* Slice-stacked plan (configs[4], 3-D parallel-beam CT): A = A2 (x) I_depth,
 * block-diagonal with the same 2-D matrix A2 (rows2 x cols2 CSR, canonical)
 * on every slice, in the INTERLEAVED order row r*depth + z, column
 * c*depth + z (csrc/stacked.cuh).  Only A2 and A2^T are stored; every other
 * entry point takes the logical (rows2*depth) x (cols2*depth) operator, and
 * products follow the reference's block-sequential arithmetic order exactly.
 * Partition bounds are over the logical rows / columns.  The _device variant
 * adopts the arrays like bsgd_plan_create_device. */
int bsgd_plan_create_stacked(bsgd_plan **out, int device, int64_t depth, int64_t rows2, int64_t cols2,
                             int64_t nnz2, const int64_t *indptr, const int32_t *indices, const void *values,
                             int value_dtype, int64_t num_row_blocks, int64_t num_col_blocks,
                             const int64_t *row_bounds, const int64_t *col_bounds, void *stream);
int bsgd_plan_create_stacked_device(bsgd_plan **out, int device, int64_t depth, int64_t rows2, int64_t cols2,
                                    int64_t nnz2, int64_t *indptr, int32_t *indices, void *values,
                                    int value_dtype, int64_t num_row_blocks, int64_t num_col_blocks,
                                    const int64_t *row_bounds, const int64_t *col_bounds, void *stream);
/* Tile-staged products for a stacked plan: group the stored rows of A2
 * (transposed = 0) or A2^T (1) into tiles of <= 16 rows that share columns
 * (tile t = rows tile_rows[tile_ptr[t] .. tile_ptr[t+1]), a permutation of all
 * stored rows; host arrays).  Products then stream each tile's distinct vector
 * rows through shared memory once instead of once per entry; results are
 * unchanged bit for bit.  ntiles = 0 removes the tiles. */
int bsgd_plan_stacked_tiles(bsgd_plan *plan, int transposed, int64_t ntiles, const int64_t *tile_ptr,
                            const int64_t *tile_rows, void *stream);
/* Gather-tiled products for an ordinary plan: group the rows of A (transposed = 0)
 * or A^T (1) into tiles of <= 16 rows that share columns (host arrays, a
 * permutation of all rows); each tile's distinct vector elements are gathered
 * once into shared memory.  Values agree with the CSR kernel to rounding (same
 * per-row reduction shape).  ntiles = 0 removes the tiles. */
int bsgd_plan_gather_tiles(bsgd_plan *plan, int transposed, int64_t ntiles, const int64_t *tile_ptr,
                           const int64_t *tile_rows, void *stream);
/* Blocked stream for A^T (the copy csr_blocked_kernel runs; A's own is built at plan
 * creation when its rows are long, and so is A^T's when A has >= 384 nonzeros per
 * column: on the row grid the plan infers from A^T's index gaps, else in A^T's own
 * column order).  grid_h x grid_w = rows of A is the grid the
 * gathered vector r lives on (row-major; a sinogram's angles x bins): the stream is
 * then gathered in 16-element grid tiles (one 128-byte line each; 4 x 4, 8 x 2 or 2 x 8,
 * chosen from the footprint of 16 consecutive entries on the grid) from r permuted into
 * that order before each launch, with 16-bit offset indices when they fit.  0, 0 =
 * no grid (A^T's own column order); a negative size removes the copy.  Between the
 * blocked copy and gather tiles of A^T the latest explicit request wins (requesting
 * gather tiles drops the blocked copy; a blocked copy built later runs instead of them).  Values agree with the CSR kernel to
 * rounding (lane-strided per-row sums, fixed shuffle tree). */
int bsgd_plan_blocked_transposed(bsgd_plan *plan, int64_t grid_h, int64_t grid_w, void *stream);
/* depth (1 for ordinary plans) and the stored CSR's shape / nnz */
int bsgd_plan_stacked_info(const bsgd_plan *plan, int64_t *depth, int64_t *rows2, int64_t *cols2,
                           int64_t *nnz2);
int bsgd_plan_destroy(bsgd_plan *plan);
/* tocsr (blockops.py:185-186): A's CSR copied to HOST buffers (rows+1, nnz, nnz) */
int bsgd_plan_csr_copy(const bsgd_plan *plan, int64_t *indptr_out, int32_t *indices_out, void *values_out,
                       void *stream);
/* shape / nnz / dtype / device bytes (blockops.py:156-162) */
int bsgd_plan_info(const bsgd_plan *plan, int64_t *rows, int64_t *cols, int64_t *nnz,
                   int *value_dtype, int64_t *device_bytes);
/* Which product kernels the plan runs (fixed at plan creation by structural
 * rules, never by timing; BlockOperator.kernel_info).  Lanes: lanes per row
 * for CSR / blocked / gather-tiled kernels, slices per lane for stacked ones. */
#define BSGD_K_CSR 0           /* dual_csr_kernel (spmv.cuh) */
#define BSGD_K_BLOCKED 1       /* csr_blocked_kernel, int32 indices */
#define BSGD_K_BLOCKED_CMP 2   /* csr_blocked_kernel, 16-bit offsets from two int32 bases per block */
#define BSGD_K_GTILE 3         /* gtile_kernel (gtile.cuh) */
#define BSGD_K_STACKED 4       /* stacked_kernel (stacked.cuh) */
#define BSGD_K_STACKED_TILE 5  /* stacked_tile_kernel (stacked.cuh) */
#define BSGD_ORDER_NATIVE 0     /* gathers in the matrix's own column order */
#define BSGD_ORDER_TILE4 1      /* blocked stream over a grid (n x n image; sinogram): 4 x 4 tiles */
#define BSGD_ORDER_TILE8X2 4    /* tiles of 8 grid rows x 2 columns (A^T on a sinogram: entries run along the angles) */
#define BSGD_ORDER_TILE2X8 5    /* tiles of 2 grid rows x 8 columns */
#define BSGD_ORDER_MORTON 2     /* (experiment, BSGD_BLK_ORDER=morton) Z order */
typedef struct bsgd_kernel_info {
    int32_t fwd_kernel, fwd_lanes;  /* A x  (K1) */
    int32_t tr_kernel, tr_lanes;    /* A^T r (K2) */
    int64_t depth;
    int32_t fwd_order;              /* BSGD_ORDER_*: pixel order of K1's gathers */
    int32_t tr_order;               /* BSGD_ORDER_*: order of K2's gathers from r */
} bsgd_kernel_info;
int bsgd_plan_kernel_info(const bsgd_plan *plan, bsgd_kernel_info *out);
/* In-epoch phase timing for measurement (bench.py): while enabled, every eager
 * bsgd_epoch on this plan records CUDA events on its stream between phases
 * (never inside a graph capture).  bsgd_plan_timing synchronises, returns the
 * summed milliseconds per phase over the recorded epochs and resets:
 * [0] K1(x_k) when the lookahead residual is invalid, [1] K2 (A^T r + step
 * epilogue), [2] TV prox, [3] K1(x_next) lookahead, [4] tail. */
#define BSGD_TIMING_PHASES 5
int bsgd_plan_set_timing(bsgd_plan *plan, int enable);
int bsgd_plan_timing(bsgd_plan *plan, double *ms_out, int64_t *epochs_out);
/* block_nnz (blockops.py:179-180), host out */
int bsgd_plan_block_nnz(const bsgd_plan *plan, int64_t i, int64_t j, int64_t *out);
/* block (blockops.py:176-177): block-local CSR copied to HOST buffers sized
 * (|I_i| + 1, block_nnz, block_nnz); values in the plan dtype. Synchronous. */
int bsgd_plan_block_copy(const bsgd_plan *plan, int64_t i, int64_t j, int64_t *indptr_out,
                         int32_t *indices_out, void *values_out, void *stream);
/* transposed pattern check: A^T rows (= A columns) [c0,c1) copied to HOST */
int bsgd_plan_transpose_copy(const bsgd_plan *plan, int64_t *indptr_out, int32_t *indices_out,
                             void *values_out, void *stream);

/* block_matvec (blockops.py:207-214): out[|I_i|] = A_ij x_j[|J_j|] */
int bsgd_block_matvec(const bsgd_plan *plan, int64_t i, int64_t j, const double *x_j, double *out,
                      void *stream);
/* block_matvec_transpose (blockops.py:216-223): out[|J_j|] = A_ij^T r_i[|I_i|] */
int bsgd_block_matvec_transpose(const bsgd_plan *plan, int64_t i, int64_t j, const double *r_i,
                                double *out, void *stream);
/* matvec / rmatvec (blockops.py:225-261) */
int bsgd_matvec(const bsgd_plan *plan, const double *x, double *out, void *stream);
int bsgd_rmatvec(const bsgd_plan *plan, const double *w, double *out, void *stream);
/* y - A x and ||y - A x||^2 (metrics.py:32-33, solvers.py:319-320); sumsq_out device scalar */
int bsgd_residual(const bsgd_plan *plan, const double *x, const double *y, double *r_out,
                  double *sumsq_out, void *scratch, void *stream);

/* assemble_residual (blockops.py:264-278): out = y - z[0] - ... - z[N-1] */
int bsgd_assemble_residual(int64_t rows, int64_t num_col_blocks, const double *y,
                           const double *z_cache, double *out, void *stream);

/* --- stochastic pair path (solvers.py:274-303 with alpha/gamma < 1) ---- */
/* z_cache[j, I_i] = A_ij x_k[J_j] for the selected pairs; g[J_j] = 2 sum_i A_ij^T r_k[I_i]
 * over selected i (zero for unselected column blocks); r_next = y - sum_j z_cache[j].
 * row_sel / col_sel: host arrays of selected block indices.  n_rows_sel may be 0 (a
 * row-slab shard owning none of the selected row blocks): g = 0, r_next from the cache. */
int bsgd_pair_products(const bsgd_plan *plan, int64_t n_rows_sel, const int64_t *row_sel,
                       int64_t n_cols_sel, const int64_t *col_sel, const double *x_k,
                       const double *r_k, const double *y, double *z_cache, double *g,
                       double *r_next, void *stream);

/* --- problem generation on the device ------------------ */
/* Parallel-beam Siddon intersection-length matrix, (num_angles*num_bins) x n^2,
 * rows angle-major then bin, bins of unit pitch centred on the axis, columns =
 * row-major pixels (row 0 at the top) -- the same matrix as
 * problems.parallel_beam_matrix (bit-identical given the same cos/sin, host).
 * Allocates device CSR arrays (free with bsgd_device_free or adopt them with
 * bsgd_plan_create_device). */
int bsgd_siddon_csr(int device, int64_t n, int64_t num_angles, int64_t num_bins, const double *cos_host,
                    const double *sin_host, int value_dtype, int64_t **indptr_out, int32_t **indices_out,
                    void **values_out, int64_t *nnz_out, void *stream);
int bsgd_device_free(void *ptr);

/* --- total variation (tv.py) ------------------------------------------- */
size_t bsgd_tv_prox_workspace_bytes(int64_t height, int64_t width);
/* tv_prox (tv.py:172-255): out = argmin ||t - img||^2 + 2 w TV(t).  info_out
 * (device) and dual_objectives (device [max_inner_iters + 1]) may be NULL. */
int bsgd_tv_prox(int64_t height, int64_t width, const double *img, double *out, double weight,
                 int32_t max_inner_iters, double tol, void *workspace, size_t workspace_bytes,
                 bsgd_prox_info *info_out, double *dual_objectives, void *stream);
/* tv_value (tv.py:149-152): device scalar out */
int bsgd_tv_value(int64_t height, int64_t width, const double *img, double *out, void *scratch,
                  void *stream);
/* discrete_gradient / discrete_divergence (tv.py:115-146) */
int bsgd_discrete_gradient(int64_t height, int64_t width, const double *img, double *dv, double *dh,
                           void *stream);
int bsgd_discrete_divergence(int64_t height, int64_t width, const double *pv, const double *ph,
                             double *out, void *stream);

/* 3D isotropic TV for volumes (z-major, then rows, then columns).  The reference
 * has 2D TV only (tv.py:28-56); these extend its conventions one axis up:
 * backward differences along z/rows/columns, div = negative adjoint, dual step
 * 1/(12 w), the same restart / stop / fallback rules (oracle/oracle.py tv_prox3). */
size_t bsgd_tv_prox3_workspace_bytes(int64_t depth, int64_t height, int64_t width);
int bsgd_tv_prox3(int64_t depth, int64_t height, int64_t width, const double *vol, double *out, double weight,
                  int32_t max_inner_iters, double tol, void *workspace, size_t workspace_bytes,
                  bsgd_prox_info *info_out, double *dual_objectives, void *stream);
int bsgd_tv_value3(int64_t depth, int64_t height, int64_t width, const double *vol, double *out, void *scratch,
                   void *stream);
int bsgd_discrete_gradient3(int64_t depth, int64_t height, int64_t width, const double *vol, double *dz,
                            double *dv, double *dh, void *stream);
int bsgd_discrete_divergence3(int64_t depth, int64_t height, int64_t width, const double *pz, const double *pv,
                              const double *ph, double *out, void *stream);

/* --- reductions (metrics.py, solvers.py:198-215, :517-518) ------------ */
/* out = sum_k a[k] * b[k]  (deterministic order); device scalar */
int bsgd_dot(int64_t n, const double *a, const double *b, double *out, void *scratch, void *stream);
/* out = sum_k (a[k] - b[k])^2; device scalar */
int bsgd_sqdist(int64_t n, const double *a, const double *b, double *out, void *scratch, void *stream);

/* --- the fused epoch ----------------------------------------------------- */
size_t bsgd_epoch_workspace_bytes(const bsgd_plan *plan, int64_t height, int64_t width);
/* bsgd_tv_iteration (solvers.py:259-341), alpha = gamma = 1 */
int bsgd_epoch(const bsgd_plan *plan, const bsgd_epoch_args *args, void *stream);
/* multi-GPU pieces of the same epoch (row-slab ownership):
 *   bsgd_grad:  g = 2 A_local^T r_local  (partial over this rank's rows)
 *   bsgd_step:  x_next = prox(x_k + mu g) with fused statistics (replicated)
 *   bsgd_epoch_forward: r_ahead/r_next over local rows + partial ||r||^2
 *   bsgd_epoch_tail: history row from the (all-reduced) scalars */
int bsgd_grad(const bsgd_plan *plan, const double *r, double *g, void *stream);
int bsgd_step(int64_t cols, const bsgd_epoch_args *args, void *stream);
int bsgd_epoch_forward(const bsgd_plan *plan, const double *x, const double *y, double *r_out,
                       const bsgd_epoch_args *args, void *stream);
/* scalars_out (device, 2 doubles): [0] = sum of the forward partials, [1] unused */
int bsgd_epoch_reduce_forward(const bsgd_plan *plan, const bsgd_epoch_args *args,
                              double *scalars_out, void *stream);
/* finish: f_next from fnext_dev (device scalar, may be NULL when no lookahead) */
int bsgd_epoch_tail(const bsgd_plan *plan, const bsgd_epoch_args *args, const double *fnext_dev,
                    void *stream);

/* --- slab-decomposed TV prox (multi-GPU, SURVEY.md §8 e "Prox") ---------
 * Replaces, on rank p of a multi-GPU run, the replicated prox inside
 * bsgd_step: tv_prox (tv.py:172-255, 3-D: oracle tv_prox3) over the rank's
 * voxels [offset, offset + count) of the C-order volume, with one-plane halos
 * (height*width voxels in 3-D, width in 2-D) exchanged by the caller between
 * passes.  Each pass that the FGP decisions need returns this slab's
 * numpy-order partial sums; when the slabs are nodes of numpy's pairwise
 * recursion over the whole volume the caller combines them in that order and
 * every decision is bit-identical to bsgd_tv_prox / bsgd_tv_prox3
 * (paper_1812_01307_b200/parallel.py: prox_slabs, pw_combine, SlabProx). */
typedef struct bsgd_slab {
    int64_t depth, height, width; /* global volume; depth 1 for an image */
    int64_t offset, count;        /* own voxels, C order */
    double weight;                /* prox weight w > 0 (mu * lam) */
    int32_t parity;               /* dual buffer (0 / 1) holding p; the other holds c (host decisions) */
    int32_t flags;                /* 0: host decisions.  BSGD_SLAB_DEVICE | (when << 1): decisions in the
                                     workspace's control block (bsgd_slab_decide); `when` = 0 always,
                                     BSGD_SLAB_MAIN / BSGD_SLAB_RESTART for the FGP passes */
    void *workspace;              /* bsgd_slab_workspace_bytes, device */
    size_t workspace_bytes;
} bsgd_slab;

#define BSGD_SLAB_SLOTS 12
/* offsets_out[BSGD_SLAB_SLOTS] (doubles from the workspace start) of the local
 * buffers, each count + 2*halo long and covering voxels
 * [offset - halo, offset + count + halo):
 *   [0] b   [1..3] dual buffer 0   [4..6] dual buffer 1   [7..9] q   [10] u
 * (2-D: entries 3, 6 and 9 are -1); [11] = a 16-double slot for sums. */
size_t bsgd_slab_workspace_bytes(int64_t depth, int64_t height, int64_t width, int64_t count);
int bsgd_slab_layout(int64_t depth, int64_t height, int64_t width, int64_t count, int64_t *offsets_out,
                     int64_t *halo_out);
/* b = x_k + mu g on the own voxels (x_k, g: full-length vectors in volume order) */
int bsgd_slab_step(const bsgd_slab *s, const double *x_k, const double *g, double mu, void *stream);
/* p = q = 0 (halos included); sums_out[0..2) = np.sum(b*b), TV(b)  (needs b's lower halo) */
int bsgd_slab_init(const bsgd_slab *s, double *sums_out, void *stream);
/* c = proj(src + step grad(b + w div src)), src = p (from_p) or q  (needs src halos) */
int bsgd_slab_candidate(const bsgd_slab *s, int32_t from_p, void *stream);
/* q = c + beta (c - p); sums_out[0 .. 1 + 2*DIM) = phi, |c_k - p_k|^2, |c_k|^2  (needs c's upper halo) */
int bsgd_slab_dual(const bsgd_slab *s, double beta, double *sums_out, void *stream);
/* u = b + w div p  (needs p's upper halo) */
int bsgd_slab_finalize(const bsgd_slab *s, void *stream);
/* sums_out[0..2) = np.sum((u - b)^2), TV(u)  (needs u's lower halo) */
int bsgd_slab_energy(const bsgd_slab *s, double *sums_out, void *stream);
/* x_next = fell_back ? b : u on the own voxels; stats_out[4] = partial |x|^2,
 * |x - x*|^2, (x - x_k).g, |x - x_k|^2 over them (x_true may be NULL) */
int bsgd_slab_output(const bsgd_slab *s, int32_t fell_back, double *x_next, const double *x_k, const double *g,
                     const double *x_true, double *stats_out, void *stream);
/* --- device-decided slab prox (graph-capturable, no host round trip) ------
 * With flags = BSGD_SLAB_DEVICE the FGP state (parity, beta, restart, done,
 * iterations, fallback) lives in the slab workspace; passes read it and return
 * at once when they do not apply, so the host issues a FIXED sequence per prox
 * (max_inner_iters blocks of candidate / dual / decide, then the restart
 * variants), collectives included.  The per-rank sums of a stage
 * (init: 2, dual: 1 + 2*DIM, energy: 2) are all-gathered rank-major into
 * `gathered` (device) and combined in numpy's recursion order by `program`
 * (host postfix: op >= 0 pushes rank op's sums, -1 adds the top two;
 * parallel.slab_program).  stage: 0 init, 1 main dual, 2 restart dual, 3 energy. */
#define BSGD_SLAB_DEVICE 1
#define BSGD_SLAB_MAIN 1
#define BSGD_SLAB_RESTART 2
/* flags bit: the x_k / g / x_next / x_true of bsgd_slab_step and bsgd_slab_output
 * are this rank's LOCAL vectors for its slices of a slice-stacked operator, in
 * the interleaved order pixel * (count / (H W)) + (slice - offset / (H W)) --
 * slice ownership of configs[4] (A = A2 (x) I_D is block diagonal in the slices,
 * so the products need no exchange); the slab must be whole slices */
#define BSGD_SLAB_INTERLEAVED 8
int bsgd_slab_decide(const bsgd_slab *s, int32_t stage, int32_t iteration, const double *gathered, int32_t world,
                     const int32_t *program, int32_t nprogram, double tol, void *stream);
/* bsgd_epoch_set_step with the prox scalars taken from the control block */
int bsgd_slab_set_step(const bsgd_slab *s, int64_t cols, const bsgd_epoch_args *args, const double *stats_dev,
                       void *stream);
/* host copy of the control block's ProxInfo (iterations, converged, restarts, fell_back) and TV; synchronises */
int bsgd_slab_info(const bsgd_slab *s, int32_t *info_out, double *tv_out, void *stream);
/* hand a distributed step's results to bsgd_epoch_tail: the all-reduced
 * statistics (device, 4 doubles) and the prox scalars */
int bsgd_epoch_set_step(int64_t cols, const bsgd_epoch_args *args, const double *stats_dev, double tv,
                        int32_t iterations, int32_t restarts, int32_t converged, int32_t fell_back,
                        void *stream);

#ifdef __cplusplus
}
#endif

#endif /* BSGD_B200_H */
