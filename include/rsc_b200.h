/*
 * rsc_b200.h -- C ABI of librsc_b200.so, the B200 (sm_100a) numeric engine of the
 * rank-structured supernodal Cholesky preconditioner (Chadwick & Bindel,
 * arXiv 1507.05593).
 *
 * Conventions (all entry points):
 *   - every matrix is FP64, ROW-MAJOR, addressed as X[i*ld + j];
 *   - pointers named *_dev are device pointers, everything else lives on the host;
 *   - `stream` is a cudaStream_t passed as void*; all work is stream-ordered and
 *     asynchronous, the library keeps no global state and allocates nothing
 *     persistent (caller-owned workspaces only);
 *   - return value: 0 ok, <0 bad argument (index of the offending argument, negated),
 *     >0 CUDA error code from the launch.  Numerical failures (a non-positive
 *     Cholesky pivot) are reported through per-matrix device `info` words with the
 *     LAPACK convention (1-based failing column, 0 = success), which the host turns
 *     into IndefiniteError(info-1) exactly like rschol.kernels.dense_cholesky
 *     (reference pkg/src/rschol/kernels.py:34-38).
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/pkg/src/rschol/).
 */
#ifndef RSC_B200_H
#define RSC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One GEMM problem (possibly a strided batch) of a grouped launch:
 *   C[b] (+)= alpha * op(A[b]) @ op(B[b]) + beta * C[b]      for b < batch
 * op(A) is M x K (A stored M x K, or K x M when transA), op(B) is K x N.
 * Optional index maps (device int32 arrays, NULL = identity):
 *   b_rows : row k of op(B) is read from B row b_rows[k]        (transB == 0 only)
 *   c_rows : row m of the result goes to C row c_rows[m]
 *   c_cols : column n of the result goes to C column c_cols[n]
 * atomic != 0: C += alpha*op(A)op(B) (beta ignored), and several problems of one
 * launch may scatter into the same target block.  These sums are DETERMINISTIC:
 * each such problem's product is stored to a private partial in the stream's GEMM
 * workspace (rsc_gemm_set_workspace), then an ordered reduction adds the partials
 * into C in problem order (for every element of C: C + P_first + ... + P_last,
 * the left-to-right order of rschol's `UD -= ...` loops, factor.py:389-398).
 * For accumulating problems c_cols must be strictly increasing and c_rows
 * non-decreasing (a repeated row is summed by one thread); ext_r x ext_c is the
 * extent of the target block C (0 = M x N, allowed only without maps), and rows
 * mapped at or beyond ext_r are dropped. */
typedef struct {
    const double *A;
    const double *B;
    double *C;
    long long strideA, strideB, strideC;
    const int *b_rows;
    const int *c_rows;
    const int *c_cols;
    int M, N, K;
    int lda, ldb, ldc;
    int batch;
    int atomic;
    double alpha, beta;
    int ext_r, ext_c;
} rsc_gemm_problem;

/* Device workspace for the ordered accumulation of a stream's grouped GEMMs
 * (partials of every atomic problem of a launch chunk).  as_default != 0 registers
 * it for every stream without its own workspace.  A launch whose chunk does not
 * fit is cut into several ordered chunks; a single problem larger than the
 * workspace returns -6.  No workspace and an atomic problem: -6. */
int rsc_gemm_set_workspace(void *stream, void *ws_dev, long long bytes, int as_default);

/* Grouped FP64 tensor-core (DMMA) GEMM.  Replaces every numpy `@` on the
 * factorization path: factor.py:383-398 (_assemble_schur), factor.py:444-455 and
 * 471-483 (off_diagonal_multiply[_trans]), diagblocks.py:220-262 (windowed source
 * products), blocks.py:35-39 (LowRankBlock.matmat/rmatmat), kernels.py:107-112. */
int rsc_gemm_grouped(int transA, int transB, const rsc_gemm_problem *problems,
                     int count, void *stream);
/* The same launch with K balancing (engine.balance_k): accumulating problems (atomic
 * or beta = 1) whose k-loop exceeds 1.5x the balanced per-CTA share of `ctas`
 * concurrent CTAs are cut into K slabs of that share, in place and in order. */
int rsc_gemm_grouped_balanced(int transA, int transB, const rsc_gemm_problem *problems, int count, int ctas,
                              void *stream);

/* Batched in-place lower Cholesky of `count` matrices (sizes may differ).
 * A[i] (n[i] x n[i], ld lda[i]) : lower triangle read, overwritten by L with the
 * strict upper triangle zeroed (dpotrf lower + clean).  Dinv[i] (n[i] x 64, ld 64)
 * receives the inverses of L's 64x64 diagonal blocks, used by rsc_trsm_batched.
 * info_dev[i] = 0 or the 1-based column of the first non-positive pivot.
 * Replaces kernels.py:22-39 dense_cholesky (called at factor.py:614,
 * diagblocks.py:300, interior.py:140). */
int rsc_potrf_batched(int count, double *const *A, const int *n, const int *lda,
                      double *const *Dinv, int *info_dev, void *stream);

/* Batched triangular solve with lower factors produced by rsc_potrf_batched.
 *   side = 0 (left):  B (n x cols)  <- L^{-1} B       (trans = 0)
 *                                   <- L^{-T} B       (trans = 1)
 *   side = 1 (right): B (rows x n)  <- B L^{-T}       (trans = 1 only)
 * `m[i]` is the number of right-hand-side columns (left) or rows (right).
 * Replaces kernels.py:42-64 tri_solve (factor.py:414,633; interior.py:60,74,141;
 * diagblocks.py:178). */
int rsc_trsm_batched(int side, int trans, int count, const double *const *L,
                     const int *n, const int *ldl, const double *const *Dinv,
                     double *const *B, const int *m, const int *ldb, void *stream);

/* Right-side solve X = Bsrc L^{-T} written to B (Bsrc == NULL: in place), for
 * panels with n <= 320: one launch, each CTA keeping a 64-row strip resident in
 * shared memory (rsc_trsm_batched side = 1 uses the same kernel when it can).
 * Returns -3 if some n > 320.  Replaces kernels.py:42-64 tri_solve at
 * factor.py:414,633. */
int rsc_trsm_right_batched(int count, const double *const *L, const int *n, const int *ldl,
                           const double *const *Dinv, const double *const *Bsrc,
                           double *const *B, const int *m, const int *ldb, void *stream);

/* Inverses of the 64x64 diagonal blocks of caller-supplied lower triangles
 * (Dinv[i]: n[i] x 64, ld 64), so rsc_trsm_batched can solve with them. */
int rsc_trtri_diag_batched(int count, const double *const *L, const int *n,
                           const int *ldl, double *const *Dinv, void *stream);

/* Batched column-pivoted Householder QR with the reference rank cutoff.
 * G[i] (m[i] x k[i], ld ldg[i]) is destroyed.  rank_dev[i] receives
 * #{ |R_jj| > max(m,k) * eps * |R_00| } (eps = 2^-52), and Q[i] (m[i] x k[i],
 * ld ldq[i]) receives the first rank_dev[i] columns of the orthonormal factor
 * and exact zeros in the remaining k[i] - rank_dev[i] columns (so a caller may keep
 * sketch-width panels without reading the ranks back).  Pivot selection, Householder vectors and the
 * partial-norm downdating follow LAPACK dgeqp3/dlaqp2 + dorg2r, which is what
 * scipy.linalg.qr(pivoting=True) runs.  work_dev: caller workspace of at least
 * rsc_qrcp_workspace_bytes(count, m, k) bytes.
 * Replaces kernels.py:67-82 orthonormalize. */
long long rsc_qrcp_workspace_bytes(int count, const int *m, const int *k);
int rsc_qrcp_batched(int count, double *const *G, const int *m, const int *k,
                     const int *ldg, double *const *Q, const int *ldq, int *rank_dev,
                     void *work_dev, void *stream);

/* Batched symmetric scatter of CSR blocks into dense row-major blocks:
 *   D[i][r, c] = values[p]  for the CSR block i (rows r < nrows[i]).
 * Used to materialize A(C_j, C_j), A(R_j, C_j) (factor.py:378-379,
 * diagblocks.py:294).  D must be zeroed by the caller. */
int rsc_csr_to_dense_batched(int count, const int *const *rowptr,
                             const int *const *colidx, const double *const *values,
                             const int *nrows, double *const *D, const int *ldd,
                             void *stream);

/* Y (nrows x r) = alpha * S @ X + beta * Y for a CSR block S (nrows x ncols)
 * and dense row-major X (ncols x r).  Replaces the scipy sparse block products
 * factor.py:444 and 471 (A(R_j,C_j) @ G1, A(R_j,C_j)^T @ G), interior.py:92-95. */
int rsc_spmm_csr(int nrows, int r, const int *rowptr_dev, const int *colidx_dev,
                 const double *values_dev, const double *X_dev, int ldx,
                 double alpha, double beta, double *Y_dev, int ldy, void *stream);

/* Grouped form of rsc_spmm_csr over `count` CSR blocks (host arrays of device
 * pointers / sizes); one launch for all A-block products of a level. */
int rsc_spmm_csr_batched(int count, const int *const *rowptr, const int *const *colidx,
                         const double *const *values, const int *nrows, const int *r,
                         const double *const *X, const int *ldx, double alpha, double beta,
                         double *const *Y, const int *ldy, void *stream);

/* Preconditioner-apply kernels (factor.py:187-218), HBM streaming:
 * rsc_trsv_batched: x[i] <- L_i^{-1} x[i] (trans=0) or L_i^{-T} x[i] (trans=1) for
 *   lower triangles from rsc_potrf_batched (their Dinv blocks); x[i] contiguous.
 * rsc_gemv_batched (mode bit 0 = transpose, bit 1 = M lower triangular, bit 2 =
 *   assign instead of accumulate (transpose 0 only), bit 3 = M upper triangular
 *   (transpose 0 only)):
 *                   mode&1==0: y[yidx[r]] += alpha * sum_c M[r,c] x[xidx[c]]
 *                   mode&1==1: y[yidx[c]] += alpha * sum_r M[r,c] x[xidx[r]]
 *   (index arrays optional, NULL = identity; FP64 atomics on y). */
int rsc_trsv_batched(int count, const double *const *L, const int *n, const int *ldl,
                     const double *const *Dinv, double *const *x, int trans, void *stream);
int rsc_gemv_batched(int count, const double *const *M, const int *rows, const int *cols,
                     const int *ldm, const double *const *x, const int *const *xidx,
                     double *const *y, const int *const *yidx, int mode, double alpha,
                     void *stream);
/* rsc_gemv_multi: the same products with a mode and alpha per problem, so one launch
 * covers a whole phase of an apply level (diagonal solves with mode 6 next to
 * couplings with mode 0, low-rank U^T w with mode 1, ...). */
int rsc_gemv_multi(int count, const double *const *M, const int *rows, const int *cols,
                   const int *ldm, const double *const *x, const int *const *xidx,
                   double *const *y, const int *const *yidx, const int *modes,
                   const double *alphas, void *stream);
/* Device-resident form of one rsc_gemv_multi phase for phases with more problems than
 * one kernel parameter block holds (the apply program is static after factorization,
 * factor.py:175-218): rsc_gemv_describe fills `desc` (count x rsc_gemv_desc_bytes()
 * bytes, host memory; the caller uploads it) and blocks[i] = CTAs of problem i;
 * rsc_gemv_multi_dev runs the phase as one launch from the uploaded descriptors and a
 * block -> problem map (int32, total_blocks entries = the repeat of i by blocks[i]). */
int rsc_gemv_desc_bytes(void);
int rsc_gemv_describe(int count, const double *const *M, const int *rows, const int *cols,
                      const int *ldm, const double *const *x, const int *const *xidx,
                      double *const *y, const int *const *yidx, const int *modes,
                      const double *alphas, void *desc, long long *blocks);
int rsc_gemv_multi_dev(const void *desc, const int *blk2prob, long long total_blocks, void *stream);

/* Subtree tasks of the preconditioner apply (factor.py:187-218): CTA t runs the
 * GEMV ops [task_ptr_dev[t], task_ptr_dev[t+1]) of descriptor array `ops` (from
 * rsc_gemv_describe over all tasks' ops followed by one empty sentinel op) in order,
 * a CTA barrier between ops.  One task = one nested-dissection subtree's interior
 * blocks and small separators (their update sources never leave the subtree);
 * mode bit 4 marks ops whose target rows the task owns (plain accumulate), other
 * accumulating ops use FP64 atomics.  Replaces the per-level launches of the
 * small units: one launch per sweep. */
int rsc_apply_tasks(const void *ops, const int *task_ptr_dev, int ntasks, void *stream);
/* The same op lists run by thread-block clusters of C <= 8 CTAs (one cluster per
 * task: the Alg. 4 chain of one diagonal block tree); each op's blocks are dealt to
 * the cluster's CTAs and a cluster barrier separates consecutive ops. */
int rsc_apply_cluster_tasks(const void *ops, const int *task_ptr_dev, int ntasks, int C, void *stream);



/* y = A x for the full symmetric CSR (pcg.py:105,116; sparse.py:86-97). */
int rsc_spmv_csr(int n, const int *rowptr_dev, const int *colidx_dev,
                 const double *values_dev, const double *x_dev, double *y_dev,
                 void *stream);

/* Gather / scatter of rows: dst[i, :] = src[idx[i], :]  (gather)
 *                           dst[idx[i], :] += alpha*src[i, :]  (scatter_add) */
/* Batched n x n identity fill / transpose (dst = src^T) of device squares: the apply
 * program's explicit inverses (apply.py refresh_inverses) in one launch each. */
int rsc_identity_batched(int count, double *const *dst, const int *n, const int *ldd, void *stream);
int rsc_transpose_batched(int count, const double *const *src, double *const *dst, const int *n,
                          const int *lds, const int *ldd, void *stream);
/* Batched rectangular copy (trans 0: dst = src) / transpose (trans 1: dst = src^T, src
 * rows x cols): stages V, U and the dense couplings of the diagonal block trees before
 * the tree solves that flatten each tree's inverse for the apply (apply.py
 * refresh_inverses; the block substitution of diagblocks.py:192-273 folded into the
 * factors once per factorization). */
int rsc_copy2d_batched(int count, const double *const *src, double *const *dst, const int *rows,
                       const int *cols, const int *lds, const int *ldd, int trans, void *stream);
int rsc_gather_rows(int nrows, int ncols, const int *idx_dev, const double *src_dev,
                    int lds, double *dst_dev, int ldd, void *stream);
int rsc_scatter_add_rows(int nrows, int ncols, const int *idx_dev, double alpha,
                         const double *src_dev, int lds, double *dst_dev, int ldd,
                         void *stream);

/* PCG vector kernels (pcg.py:104-128).  dot: out_dev[0] = x.y (deterministic
 * two-pass tree reduction).  axpy: y += alpha_dev[0]*scale * x.  xpby:
 * p = z + (num/den) * p with num/den read from device scalars. */
int rsc_dot(int n, const double *x_dev, const double *y_dev, double *out_dev,
            double *work_dev, void *stream);
int rsc_pcg_update_xr(int n, const double *rz_dev, const double *pap_dev,
                      double *x_dev, double *r_dev, const double *p_dev,
                      const double *ap_dev, void *stream);
int rsc_pcg_update_p(int n, const double *rznew_dev, const double *rz_dev,
                     const double *z_dev, double *p_dev, void *stream);

/* ---- host-only symbolic analysis (no device work; symbolic.py:44-151) ----
 * Inputs: the permuted matrix in lower CSC (col_ptr[n+1], row_idx[nnz], int64).
 * etree: parent[j] (-1 for roots).  postorder: children ascending, roots ascending.
 * colcounts: nonzeros per column of the Cholesky factor, diagonal included. */
int rsc_sym_etree(long long n, const long long *col_ptr, const long long *row_idx,
                  long long *parent);
/* The same etree with the rows of nr disjoint ND-subtree column ranges
 * [ranges[2r], ranges[2r+1]) on host threads first; returns 1 when the ranges are
 * not closed (parent then untouched: call rsc_sym_etree). */
int rsc_sym_etree_par(long long n, const long long *col_ptr, const long long *row_idx, long long nr,
                      const long long *ranges, long long *parent);
int rsc_sym_postorder(long long n, const long long *parent, long long *post);
int rsc_sym_colcounts(long long n, const long long *col_ptr, const long long *row_idx,
                      const long long *parent, const long long *post, long long *counts);
/* Relaxed amalgamation of one gap of fundamental supernodes (symbolic.py:244-277):
 * bounds[0..nb] fundamental boundaries, tiers (tw[i] max width or -1, tb[i] bound);
 * writes the kept starts to out and returns their count (<0: bad argument). */
long long rsc_sym_amalgamate(long long nb, const long long *bounds, const long long *parent,
                             const long long *counts, int ntier, const long long *tw, const double *tb,
                             long long *out);
/* Row structures of the M supernodes (symbolic.py:280-306), two calls: compute
 * returns a handle and the total row count, fetch writes ptr[M+1] and rows[total]
 * and frees the handle. */
void *rsc_sym_rows_compute(long long M, const long long *starts, const long long *col_ptr,
                           const long long *row_idx, long long *total);
/* The same with nr supernode ranges [ranges[2i], ranges[2i+1]) (disjoint ND
 * subtrees) swept on host threads first; falls back to the sequential sweep when a
 * range is not closed under the pass-up.  Identical output. */
void *rsc_sym_rows_compute_par(long long M, const long long *starts, const long long *col_ptr,
                               const long long *row_idx, long long nr, const long long *ranges, long long *total);
int rsc_sym_rows_fetch(void *handle, long long *ptr, long long *rows);
/* Full symmetric CSR of a lower-CSC matrix, rows sorted, stored zeros dropped
 * (sparse.py:86-97 _csr_full); adjacency != 0 also drops the diagonal (the ND
 * graph, ordering.py:113-119).  indices/data need 2*nnz_lower capacity; returns
 * the entry count. */
long long rsc_sym_full_csr(long long n, const long long *col_ptr, const long long *row_idx,
                           const double *values, int adjacency, long long *indptr, long long *indices,
                           double *data);
/* Symmetric permutation in lower storage (sparse.py:171-189): new rows / columns of
 * every entry sorted by (column, row) and the source position of each. */
int rsc_sym_permute_lower(long long n, const long long *col_ptr, const long long *row_idx, const long long *p,
                          long long *out_rows, long long *out_cols, long long *order);
/* One geometric bisection step of nested dissection (ordering.py:182-192): the
 * vertices are split at the median along the widest coordinate axis (ties by id);
 * the second half's members adjacent to the first form the separator.  indptr /
 * indices: full adjacency CSR without the diagonal; xyz: n x dim row-major;
 * mark: n zero bytes of scratch.  out <- side1 | separator | side2, counts <- sizes.
 * Returns 1 when a side is empty (no split). */
int rsc_nd_split_geometric(long long nv, const long long *verts, int dim, const double *xyz,
                           const long long *indptr, const long long *indices, unsigned char *mark,
                           long long *out, long long *counts);
/* Whole geometric nested dissection (ordering.py:277-368, replaces the Python
 * recursion over rsc_nd_split_geometric): subtrees run on host threads.
 * order[pos] <- vertex; separator-tree nodes in the arrays of capacity cap
 * (lo, hi, subtree_lo, level, left, right; -1 children = leaf), *root <- root id.
 * Returns the node count, -1 bad arguments, -3 capacity too small. */
long long rsc_nd_geometric(long long n, int dim, const double *xyz, const long long *indptr,
                           const long long *indices, long long leaf, long long *order, long long cap,
                           long long *n_lo, long long *n_hi, long long *n_sub, long long *n_lev,
                           long long *n_left, long long *n_right, long long *root);
/* Batched window cut of a CSR matrix (n rows, ascending column indices) whose
 * values are 1-based positions: request q = rows sel[r_off[q]..+r_n[q]) (or the
 * range [r_lo[q], +r_n[q]) when r_off[q] < 0) x columns likewise (ascending
 * lists), block-local numbering.  Pass 1 (rowptr == NULL) writes nnz[q]; pass 2
 * (nz_off = exclusive scan of nnz, rp_off[q] = sum of r_n[i]+1 over i < q) writes
 * rowptr (int32), colidx (int32) and val = position - 1 (int32).  Host threads. */
int rsc_csr_windows(long long nq, long long n, const long long *indptr, const long long *indices,
                    const double *data, const long long *sel, const long long *r_off,
                    const long long *r_n, const long long *r_lo, const long long *c_off,
                    const long long *c_n, const long long *c_lo, long long *nnz,
                    const long long *rp_off, const long long *nz_off, int *rowptr, int *colidx,
                    int *val);

/* ---- The apply as one dataflow launch (factor.py:175-218) -------------------------
 * rsc_flow_deps (host): the op graph of the apply's GEMV ops given in a valid
 * sequential order -- op o reads x elements (contiguous from xaddr[o], or
 * xaddr[o] + 8*idx[k] for an index list at device address xidx[o], xlen[o] of them)
 * and writes y elements likewise (yassign[o] != 0: assignment, else accumulation,
 * which commutes with other accumulations).  Vector addresses lie in the nbuf
 * buffers [buf_base, buf_base + 8*buf_len); index lists are read from idx_host, the
 * host copy of the device index buffer at idx_dev (idx_len ints).  Writes need[o]
 * (predecessor count) and the successor CSR (succ_ptr nops+1, succ); returns the
 * edge count (> succ_cap: nothing written to succ, call again with that capacity),
 * <0 on bad input.
 * rsc_flow_describe: descriptors (rsc_gemv_desc_bytes each) of the ops in queue
 * order, at least one item per op, items numbered globally; item_op (total ints,
 * may be null) = item -> op.  Returns the item count.
 * rsc_apply_flow: zeroes `state` (1 + 2*nops ints) and runs every item in one
 * persistent launch: an item waits until its op's predecessors have all completed. */
long long rsc_flow_deps(int nops, const long long *xaddr, const long long *xidx, const int *xlen,
                        const long long *yaddr, const long long *yidx, const int *ylen, const int *yassign,
                        int nbuf, const long long *buf_base, const long long *buf_len, const int *idx_host,
                        long long idx_dev, long long idx_len, int *need, int *succ_ptr, int *succ,
                        long long succ_cap);
long long rsc_flow_describe(int count, const double *const *M, const int *rows, const int *cols, const int *ldm,
                            const double *const *x, const int *const *xidx, double *const *y,
                            const int *const *yidx, const int *modes, const double *alphas, void *desc,
                            int *item_op);
int rsc_apply_flow(const void *ops, const int *item_op, const int *need, const int *succ_ptr, const int *succ,
                   int *state, int nops, int total, void *stream);
/* Diagnostics: the same launch recording, per item, 4 uint64 into `trace` (device,
 * 4*total): %globaltimer when taken, after its dependency wait, at completion; SM id. */
int rsc_apply_flow_trace(const void *ops, const int *item_op, const int *need, const int *succ_ptr,
                         const int *succ, int *state, int nops, int total, void *trace, void *stream);

/* ---- Plan compiler (plan.py NumericPlan; host threads) --------------------------
 * rsc_plan_pairs: every (target supernode j, update source s) pair with a row of s
 * inside C_j (is_target[j] != 0), grouped by target, sources by src_order within a
 * target (the bucket order of factor.py:545-554,572); lo/hi = the run of s's rows
 * in C_j; an int32 index chunk with cpos = rows[lo:hi] - c0 and
 * rpos = searchsorted(R_j, rows[hi:]) per pair (factor.py:389-398, 450-455).
 * Returns a handle; rsc_plan_pairs_fetch copies tgt, src, lo, hi, cpos offset,
 * rpos offset (npairs each) and the chunk (nidx ints), then frees it.
 * rsc_plan_tree_maps: the window maps of diagonal-tree blocks (diagblocks.py:
 * 231-262) for blocks with global spans (row lo, row hi, col lo, col hi) and the
 * pairs of each tree; rsc_plan_tree_maps_fetch writes 9 arrays (tree, block, src,
 * clo, chi, rlo, rhi, cidx offset, ridx offset) grouped by (tree, block), and the
 * chunk. */
void *rsc_plan_pairs(long long nsrc, const long long *src_ptr, const long long *src_rows,
                     const long long *src_order, long long M, const long long *starts,
                     const unsigned char *is_target, const long long *R_ptr, const long long *R_rows,
                     long long *npairs, long long *nidx);
int rsc_plan_pairs_fetch(void *h, long long *tgt, long long *src, long long *lo, long long *hi, long long *cpos,
                         long long *rpos, int *idx);
void *rsc_plan_tree_maps(long long ntree, const long long *blk_ptr, const long long *spans,
                         const long long *pair_ptr, const long long *pair_src, const long long *src_ptr,
                         const long long *src_rows, long long *nmaps, long long *nidx);
int rsc_plan_tree_maps_fetch(void *h, long long *const *out, int *idx);
/* 64-bit digest of a byte buffer (the pattern key load_values compares). */
unsigned long long rsc_hash64(const void *data, long long nbytes);

/* ---- Plan-level numeric steps ------------------
 * Composed from the batched kernels above, driven by the plan's index arrays (the
 * descendant maps of plan.py: per update source q of a target supernode, its panel
 * pair eff/raw (ld, width w), the row run lo, the counts nrd = rows inside C_j and
 * nro = rows beyond, and the int32 maps cpos (rows inside C_j, relative to c0) and
 * rpos (searchsorted positions in R_j)).  Sources in reference order.
 *
 * rsc_schur_update (factor.py:383-398 _assemble_schur): UD[cpos, cpos] -=
 *   eff[lo:lo+nrd] raw[lo:lo+nrd]^T and UO[rpos, cpos] -= eff[lo+nrd:] raw[lo:lo+nrd]^T,
 *   summed in source order (ordered accumulation, bit-reproducible).  UD (nc x nc)
 *   and UO (nr x nc) hold A's blocks on entry; either may be NULL.
 * rsc_offdiag_products (factor.py:444-455 / 471-482): the source terms of Alg. 2;
 *   trans = 0: W[rpos] -= E[hi:] (V[lo:hi]^T G[cpos]); trans = 1: W[cpos] -=
 *   V[lo:hi] (E[hi:]^T G[rpos]).  W (wr x wc), G (x r), T: workspace of
 *   sum_q w_q r doubles.  The caller adds A's term and the diagonal solve
 *   (rsc_spmm_csr, rsc_trsm_batched / rsc_tree_trsm).
 * rsc_interior_factor_batched (interior.py:105-156): L_B = chol(A_BB) in place
 *   (+ Dinv, LAPACK info words) and Y_B = A(off_rows, C_B) L_B^{-T} in place.
 * rsc_tree_trsm (diagblocks.py:192-273, Alg. 4): X (n x r) <- D^{-1} X (trans 0) or
 *   D^{-T} X (trans 1) for a block tree of nnodes nodes: node i spans [lo, hi) of the
 *   separator; split[i] < 0 marks a leaf (L, ldl, Dinv: its triangle), else the
 *   coupling of [lo, split) into [split, hi) is dense B (rows hi-split x cols
 *   split-lo) or, when k != NULL and V[i] != NULL, V U^T (V: rows x k[i], U: cols x
 *   k[i]); tws: k_max x r doubles of workspace.
 * rsc_apply_sweep (factor.py:187-218): one sweep of the apply program, phases of
 *   rsc_gemv_multi problems run in order (flattened arrays, phase_count[p] problems
 *   each); forward and backward sweeps are two programs (apply.py DeviceApply).
 * rsc_nccl_*: NCCL resolved at run time (libnccl.so.2 or RSC_NCCL_LIB); -20 if
 *   unavailable.  Communicator from a 128-byte unique id; FP64 sum all-reduce and
 *   broadcast (the multi-GPU top-separator sums and apply rows, distributed.py). */
int rsc_schur_update(double *UD, int ld_ud, int nc, double *UO, int ld_uo, int nr, int nsrc,
                     const double *const *eff, const double *const *raw, const int *ld, const int *w, const int *lo,
                     const int *nrd, const int *nro, const int *const *cpos, const int *const *rpos, void *stream);
int rsc_offdiag_products(int trans, double *W, int ldw, int wr, int wc, const double *G, int ldg, int r, int nsrc,
                         const double *const *eff, const double *const *raw, const int *ld, const int *w,
                         const int *lo, const int *nrd, const int *nro, const int *const *cpos,
                         const int *const *rpos, double *T, void *stream);
int rsc_interior_factor_batched(int count, double *const *L, const int *n, const int *ldl, double *const *Dinv,
                                double *const *Y, const int *m, const int *ldy, int *info_dev, void *stream);
int rsc_tree_trsm(int trans, int nnodes, int root, const int *lo, const int *hi, const int *split, const int *left,
                  const int *right, const double *const *L, const int *ldl, const double *const *Dinv,
                  const double *const *B, const int *ldb, const double *const *V, const double *const *U,
                  const int *ldv, const int *ldu, const int *k, double *X, int ldx, int r, double *tws,
                  void *stream);
int rsc_apply_sweep(int nphases, const int *phase_count, const double *const *M, const int *rows, const int *cols,
                    const int *ldm, const double *const *x, const int *const *xidx, double *const *y,
                    const int *const *yidx, const int *modes, const double *alphas, void *stream);
int rsc_nccl_available(void);
int rsc_nccl_unique_id(char *id128);
int rsc_nccl_comm_init(int nranks, const char *id128, int rank, void **comm);
int rsc_nccl_allreduce_sum_f64(void *comm, const double *send, double *recv, long long count, void *stream);
int rsc_nccl_broadcast_f64(void *comm, const double *send, double *recv, long long count, int root, void *stream);
int rsc_nccl_comm_destroy(void *comm);

/* ---- Gaussian sketches (replaces the host draw at reference kernels.py:85-92,
 * np.random.Generator(np.random.PCG64(seed)).standard_normal((m, r)), seeded per
 * block by factor.py:324-326 _block_seed) ---------------------------------------
 *
 * rsc_pcg64_block_states: for each i, keys[i*width .. +nkeys[i]] = (master, tags...)
 * -> seed = SeedSequence(keys).generate_state(1, uint64)[0] (seeds_out, optional)
 * -> PCG64(seed) state as 4 words (state_hi, state_lo, inc_hi, inc_lo).  Host only.
 * rsc_pcg64_seed_states: the same from ready-made seeds.
 * rsc_normal_pcg64: out[i][0 .. n[i]) = the first n[i] standard normals of stream i,
 * bit-identical to numpy's Generator.standard_normal (C order), generated on the
 * device.  `states` is HOST memory (4 words per stream); work is device memory of
 * rsc_normal_workspace_bytes(count, n) bytes.
 * rsc_log1p_fdlibm: the host copy of the device log1p (test hook). */
int rsc_pcg64_block_states(int count, int width, const uint64_t *keys, const int *nkeys,
                           uint64_t *seeds_out, uint64_t *states_out);
int rsc_pcg64_seed_states(int count, const uint64_t *seeds, uint64_t *states_out);
size_t rsc_normal_workspace_bytes(int count, const long long *n);
int rsc_normal_pcg64(int count, const unsigned long long *states, const long long *n,
                     double *const *out, void *work, size_t work_bytes, void *stream);
double rsc_log1p_fdlibm(double x);
/* Test hook: cand_cap (0..160) caps the slow positions a chunk may record and
 * slack = 0 scans only n/2 draws, forcing both exact sequential fallbacks.
 * Defaults (160, 1) restore the fast path. */
int rsc_normal_debug_limits(int cand_cap, int slack);

/* Number of kernels this process launched through the library (reset != 0
 * returns the count and zeroes it).  Diagnostic only. */
long long rsc_launch_counter(int reset);

/* Library self-description, for load checks. */
const char *rsc_version(void);
int rsc_device_arch(void);

#ifdef __cplusplus
}
#endif
#endif /* RSC_B200_H */
