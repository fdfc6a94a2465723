/*
 * laq_b200.h — C-ABI of the B200-native LAQ hot path.
 *
 * The reference (arxiv 2306.08367 artifact, /root/reference/proj) exposes a
 * C++20 operator API over host std::vectors (proj/include/laq/*.hpp).  This
 * header is the drop-in boundary underneath it: plain C, plain pointers and
 * sizes, no C++ or torch types.  Every entry point names the reference
 * function it replaces as  file:line  (paths relative to proj/).
 *
 * Conventions
 *  - Every call returns an int status: LAQ_OK or one of the LAQ_ERR_* codes,
 *    which map 1:1 onto the laq::Error subclasses of include/laq/error.hpp:10-74
 *    (the C++ shim in integration/ rethrows the matching type).  The message of
 *    the last failure on a context is available from laq_ctx_last_error().
 *  - "d_" arguments are DEVICE pointers owned by the caller; "h_" arguments are
 *    host pointers.  Scratch memory is owned by the context.
 *  - A context is bound to one device and one CUDA stream; calls on one context
 *    are serialised on that stream (asynchronous unless the call must return a
 *    data-dependent size through an h_ pointer, in which case it synchronises).
 *    Separate contexts are reentrant.
 *  - There is no CPU fallback: when the CUDA kernels cannot run, calls fail
 *    with LAQ_ERR_CUDA.
 */
#ifndef LAQ_B200_H
#define LAQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (error.hpp:10-74) ---------------------------------- */
enum laq_status {
  LAQ_OK = 0,
  LAQ_ERR_GENERIC = 1,        /* laq::Error            error.hpp:10  */
  LAQ_ERR_INDEX = 2,          /* laq::IndexError       error.hpp:15  */
  LAQ_ERR_SHAPE = 3,          /* laq::ShapeError       error.hpp:20  */
  LAQ_ERR_FORMAT = 4,         /* laq::FormatError      error.hpp:25  */
  LAQ_ERR_NAME = 5,           /* laq::NameError        error.hpp:30  */
  LAQ_ERR_TYPE = 6,           /* laq::TypeError        error.hpp:35  */
  LAQ_ERR_MAPPING = 7,        /* laq::MappingError     error.hpp:40  */
  LAQ_ERR_DOMAIN = 8,         /* laq::DomainError      error.hpp:45  */
  LAQ_ERR_DUPLICATE_KEY = 9,  /* laq::DuplicateKeyError error.hpp:51 */
  LAQ_ERR_TREE = 10,          /* laq::TreeError        error.hpp:56  */
  LAQ_ERR_MODEL = 11,         /* laq::ModelError       error.hpp:61  */
  LAQ_ERR_GEN = 12,           /* laq::GenError         error.hpp:66  */
  LAQ_ERR_CAPACITY = 13,      /* laq::CapacityError    error.hpp:71  */
  LAQ_ERR_CUDA = 100,         /* device / driver failure (no reference equivalent) */
  LAQ_ERR_UNSUPPORTED = 101   /* valid input outside this build's device paths */
};

typedef struct laq_ctx laq_ctx;
typedef struct laq_star laq_star;
typedef struct laq_plan laq_plan;

/* ---- context ----------------------------------------------------------- */
int laq_ctx_create(int device, laq_ctx** out);
int laq_ctx_destroy(laq_ctx* ctx);
/* Bind the context to an existing cudaStream_t (NULL = the legacy stream). */
int laq_ctx_set_stream(laq_ctx* ctx, void* cuda_stream);
int laq_ctx_synchronize(laq_ctx* ctx);
const char* laq_ctx_last_error(const laq_ctx* ctx);
/* Number of kernels this context has launched (bench/gpu_launches evidence). */
int64_t laq_ctx_launch_count(const laq_ctx* ctx);
/* Library build string (arch, version). */
const char* laq_version(void);

/* ---- row-sharded multi-GPU ---------------------------------
 * The reference is single-process (proj/README.md:115); these entry points are
 * the B200 build's own.  One process per GPU, each owning a contiguous row
 * shard of the fact table (dimension tables replicated).  Once a context has a
 * communicator, laq_run_query and laq_measure_selectivity sum their per-group
 * (count, sum) accumulators across the ranks before emitting, so every rank
 * returns the whole-table result; laq_allreduce_acc does the same for the
 * prepared-plan path (laq_plan_execute on each shard, then all-reduce, then
 * laq_plan_emit).  Integer accumulators: the merge is exact and order-free. */
/* NCCL (loaded at run time from libnccl.so.2): rank 0 creates the id, the
 * caller distributes its 128 bytes, every rank attaches. */
int laq_nccl_unique_id(uint8_t h_id[128]);
int laq_ctx_attach_nccl(laq_ctx* ctx, int32_t nranks, int32_t rank, const uint8_t h_id[128]);
/* Or any host-side transport: fn sums h_buf[0..count) in place across the
 * ranks (called with the context's stream synchronised).  NULL detaches. */
typedef int (*laq_allreduce_host_fn)(int64_t* h_buf, int64_t count, void* user);
int laq_ctx_set_allreduce_host(laq_ctx* ctx, int32_t nranks, int32_t rank, laq_allreduce_host_fn fn, void* user);
int laq_ctx_comm_info(const laq_ctx* ctx, int32_t* h_nranks, int32_t* h_rank);
/* Sum d_acc[0..count) (int64, device) across the ranks on the context stream. */
int laq_allreduce_acc(laq_ctx* ctx, int64_t* d_acc, int64_t count);

/* ---- key encoding (laqops.hpp:54-78) ----------------------------------- */

/* build_key_domain (laqops.cpp:142-155): ascending distinct union of keys_r and
 * keys_s into d_out_sorted (capacity n_r + n_s); size to *h_out_size.
 * LAQ_ERR_DOMAIN on a negative key. Synchronises. */
int laq_build_key_domain(laq_ctx* ctx, const int64_t* d_keys_r, int64_t n_r,
                         const int64_t* d_keys_s, int64_t n_s, int64_t* d_out_sorted,
                         int64_t* h_out_size);

/* update_key_domain (laqops.cpp:157-171): merge new keys into a sorted domain.
 * d_out capacity d + n_new. Synchronises. */
int laq_update_key_domain(laq_ctx* ctx, const int64_t* d_domain, int64_t d,
                          const int64_t* d_new_keys, int64_t n_new, int64_t* d_out,
                          int64_t* h_out_size);

/* KeyDomain::position over a batch (laqops.cpp:123-127) — the col_idx of
 * key_matrix(RowsByDomain) (laqops.cpp:181-195).  LAQ_ERR_DOMAIN if a key is
 * absent.  d_domain must be ascending and distinct. */
int laq_key_positions(laq_ctx* ctx, const int64_t* d_keys, int64_t n, const int64_t* d_domain,
                      int64_t d, int64_t* d_pos);

/* key_matrix(DomainByRows) (laqops.cpp:196-218): CSR d x n, counting sort by
 * domain position, columns ascending per row.  d_values may be NULL (all 1.0);
 * rows whose value is exactly 0.0 are validated but not stored (laqops.cpp:188-190),
 * so d_col_idx/d_out_values capacity is n and *h_nnz receives the stored count.
 * d_out_values may be NULL when d_values is NULL. Synchronises. */
int laq_key_matrix_dbr(laq_ctx* ctx, const int64_t* d_keys, int64_t n, const int64_t* d_domain,
                       int64_t d, const double* d_values, int64_t* d_row_ptr, int64_t* d_col_idx,
                       double* d_out_values, int64_t* h_nnz);

/* ---- join-MM (laqops.hpp:80-110) --------------------------------------- */

/* mm_join (laqops.cpp:222-231): equi-join as spmm(key_matrix(R), key_matrix(S)^T),
 * many-to-many, COO in canonical (r asc, s asc) order.  If capacity is too small
 * returns LAQ_ERR_CAPACITY with *h_nnz = required entries and writes nothing.
 * Synchronises. */
int laq_mm_join(laq_ctx* ctx, const int64_t* d_keys_r, int64_t n_r, const int64_t* d_keys_s,
                int64_t n_s, int64_t* d_out_r, int64_t* d_out_s, int64_t capacity, int64_t* h_nnz);

/* multiway_star_join (laqops.cpp:233-319): per fact row, the unique matching
 * row of every dimension; rows missing any dimension drop out.  Outputs, in
 * ascending fact-row order: d_survivors[m] (fact row) and d_dim_rows[j][m]
 * (row of dim j).  Capacities n_fact.  LAQ_ERR_DUPLICATE_KEY on a duplicate
 * pk (laqops.cpp:252-254).  d_survivors may be NULL. Synchronises. */
int laq_star_join(laq_ctx* ctx, int32_t n_links, const int64_t* const* d_fks, int64_t n_fact,
                  const int64_t* const* d_pks, const int64_t* h_pk_rows, int64_t* d_survivors,
                  int64_t* const* d_dim_rows, int64_t* h_nnz);

/* ---- dense / fused prediction (fusion.hpp:8-18, mlops.hpp:74) ----------- */

/* dense_matmul (matrix.cpp:158-174) / predict_linear (mlops.cpp:248-250):
 * C[m x n] = A[m x k] * B[k x n], fp64 row-major, sequential-k fp64 sums. */
int laq_dense_matmul(laq_ctx* ctx, const double* d_a, int64_t m, int64_t k, const double* d_b,
                     int64_t n, double* d_c);

/* spmm_dense (matrix.cpp:125-139) for a general CSR (rows x b_rows) times a
 * dense b_rows x n: each output is the row's entries in CSR order, each product
 * separately rounded (bit-identical).  Used for non-one-hot row/column maps. */
int laq_spmm_dense(laq_ctx* ctx, const int64_t* d_row_ptr, const int64_t* d_col_idx, const double* d_values,
                   int64_t rows, const double* d_b, int64_t b_rows, int64_t n, double* d_out);

/* materialize's column placement (laqops.cpp:364-371): for each ColumnMap entry
 * (src col, tgt col, v): d_dst[r, tgt] += v * d_src[r, src] (d_dst is rows x k). */
int laq_place_columns(laq_ctx* ctx, const double* d_src, int64_t rows, int64_t src_cols,
                      const int64_t* h_src_col, const int64_t* h_tgt_col, const double* h_val,
                      int64_t nnz, int64_t k, double* d_dst);

/* prefuse_linear (fusion.cpp:50-62) + linear_partial (fusion.cpp:31-36):
 * P_j = B_j * (M_j * L) where M_j is the placement of dim j's k_j columns into
 * the global width k (h_placements[j][c] = global column of local column c).
 * Placements must tile [0,k) exactly: LAQ_ERR_MAPPING on overlap, LAQ_ERR_SHAPE
 * on gaps (check_placements, fusion.cpp:11-25). fp64. */
int laq_prefuse_linear(laq_ctx* ctx, int32_t n_dims, const double* const* d_dims,
                       const int64_t* h_dim_rows, const int64_t* h_dim_cols,
                       const int64_t* const* h_placements, const double* d_L, int64_t k,
                       int64_t l, double* const* d_partials);

/* apply_fused_linear (fusion.cpp:64-77): Y[m] = ((P_0[i_0[m]] + P_1[i_1[m]]) + ...)
 * in the reference's association order, fp64.  d_idx[j] are the I_j row maps
 * (one source row per target row). */
int laq_apply_fused_linear(laq_ctx* ctx, int32_t n_parts, const int64_t* const* d_idx, int64_t rows,
                           const double* const* d_partials, const int64_t* h_partial_rows,
                           int64_t l, double* d_out);

/* materialize (laqops.cpp:338-374): T[m, place_j(c)] = B_j[i_j[m], c], fp64,
 * the non-fused plan's target table.  LAQ_ERR_MAPPING on overlapping targets. */
int laq_materialize(laq_ctx* ctx, int32_t n_parts, const int64_t* const* d_idx, int64_t rows,
                    const double* const* d_dims, const int64_t* h_dim_rows,
                    const int64_t* h_dim_cols, const int64_t* const* h_placements, int64_t k,
                    double* d_out);

/* Fused join + predict (north_star; PipelineRunner::run_fused cli.cpp:336-346
 * composed with prepare_joins cli.cpp:279-293): one pass over the fact keys
 * that probes every dimension, drops misses, and writes Y[m] = sum_j P_j[row_j]
 * for the m-th surviving fact row in ascending order.  d_survivors may be NULL.
 * Keys are int32 (range-checked narrowing of the reference's int64 keys).
 * Synchronises to report *h_nnz. */
int laq_fused_star_predict(laq_ctx* ctx, int32_t n_links, const int32_t* const* d_fks,
                           int64_t n_fact, const int32_t* const* d_pks, const int64_t* h_pk_rows,
                           const double* const* d_partials, int64_t l, double* d_out,
                           int64_t* d_survivors, int64_t* h_nnz);

/* Lower-level form of laq_fused_star_predict for repeated execution (CUDA-graph
 * capturable, no host sync): build the per-dimension probe tables once ... */
typedef struct laq_probe laq_probe;
int laq_probe_build(laq_ctx* ctx, int32_t n_links, const int32_t* const* d_pks,
                    const int64_t* h_pk_rows, laq_probe** out);
/* Optionally bind the partials once (re-laid out in key-slot order next to an
 * existence bitmap); later calls may then pass d_partials = NULL.  Binding
 * snapshots the values: rebind after the partials change (refresh_partial,
 * fusion.cpp:161-179). */
int laq_probe_bind_partials(laq_ctx* ctx, laq_probe* probe, const double* const* d_partials, int64_t l);
/* ... then stream the fact keys; the survivor count is written to d_nnz (device). */
int laq_probe_fused_predict(laq_ctx* ctx, const laq_probe* probe, const int32_t* const* d_fks,
                            int64_t n_fact, const double* const* d_partials, int64_t l,
                            double* d_out, int64_t* d_survivors, int64_t* d_nnz);
/* The same with HOST buffers (the reference-facing call: keys in, predictions
 * out in host memory): h_fks[j] are n_fact int32 keys, h_out has room for
 * n_fact * l doubles and receives the *h_nnz surviving rows in ascending fact
 * order.  The keys stream H2D and the predictions D2H in chunk_rows pieces
 * (0: one piece up to 4M rows, else n_fact / 8) on two copy streams,
 * overlapped with each other and with the probe kernel; pinned host memory
 * gives the full PCIe rate.
 * Needs direct probes and partials bound with laq_probe_bind_partials.
 * Synchronises before returning. */
int laq_probe_fused_predict_host(laq_ctx* ctx, const laq_probe* probe, const int32_t* const* h_fks,
                                 int64_t n_fact, int64_t l, double* h_out, int64_t chunk_rows, int64_t* h_nnz);
int laq_probe_destroy(laq_probe* probe);

/* Star join over prebuilt probe tables, compacted to int32 row maps
 * (multiway_star_join, laqops.cpp:233-319, for the tensor-core operators):
 * d_rows[j][m] = row of dim j matched by the m-th surviving fact row (ascending);
 * survivor count to d_nnz (device).  No host synchronisation. */
int laq_probe_join_rows(laq_ctx* ctx, const laq_probe* probe, const int32_t* const* d_fks, int64_t n_fact,
                        int32_t* const* d_rows, int64_t* d_survivors, int64_t* d_nnz);

/* ---- tensor-core FFN over a star join (BASELINE configs[2]) -------------
 * Y = ReLU(T W1) W2 with T = materialize(I_j, B_j, placements) (laqops.cpp:338-374)
 * and the products of predict_linear / dense_matmul (mlops.cpp:248-250,
 * matrix.cpp:158-174); the reference has no FFN, cfg3 composes these.  T is
 * gathered tile by tile into shared memory, never written.  fp64 inputs are
 * stored as a scaled fp16x2 split; tcgen05 MMAs accumulate fp32 in TMEM (SURVEY.md
 * Appendix B: condition-aware 1e-5).  Output fp32 [rows x l].
 * Limits: 1..4 dims, sum of 8-padded dim widths <= 128, h multiple of 32 in
 * [32,256], l in [1,8] (LAQ_ERR_UNSUPPORTED otherwise); placements as in
 * laq_prefuse_linear (LAQ_ERR_MAPPING / LAQ_ERR_SHAPE). */
typedef struct laq_ffn laq_ffn;
int laq_ffn_create(laq_ctx* ctx, int32_t n_dims, const double* const* d_dims, const int64_t* h_dim_rows,
                   const int64_t* h_dim_cols, const int64_t* const* h_placements, int64_t k, const double* d_W1,
                   int64_t h, const double* d_W2, int64_t l, laq_ffn** out);
/* Over explicit join row maps (one row of every dim per target row). Async. */
int laq_ffn_predict_rows(laq_ctx* ctx, const laq_ffn* f, const int32_t* const* d_rows, int64_t rows, float* d_out);
/* Join + FFN: probes the fact keys inside the kernel; if any fact row misses a
 * dimension, compacts with laq_probe_join_rows and reruns on the survivors.
 * Y[m] for the m-th surviving fact row (ascending).  Synchronises (*h_nnz). */
int laq_ffn_predict_star(laq_ctx* ctx, const laq_ffn* f, const laq_probe* probe, const int32_t* const* d_fks,
                         int64_t n_fact, float* d_out, int64_t* d_survivors, int64_t* h_nnz);
int laq_ffn_destroy(laq_ffn* f);

/* ---- tensor-core contractions for the wide shapes (BASELINE configs[4]) ----
 * A features object holds dims' tables B_j (fp64, rows x cols) in the fp16x2
 * split block layout with their placements into the global feature width k
 * (LAQ_ERR_MAPPING on overlap / out of range, as check_placements fusion.cpp:11-25).
 *   laq_tc_gemm: C[m x n] (fp32) = T . W, T[r] = sum_j B_j[d_rows[j][r]] M_j
 *     - prefuse_linear (fusion.cpp:50-62): one dim, d_rows = NULL (identity),
 *       m = dim rows -> P_j = B_j (M_j W);
 *     - non-fused predict (materialize laqops.cpp:338-374 + predict_linear
 *       mlops.cpp:248-250): d_rows = join row maps, T never written.
 *   W is k x n fp64 row-major.  tcgen05 fp16x2 split (3 MMAs), fp32 accumulate (condition-aware
 *   1e-5).  Asynchronous.
 *   laq_apply_fused_linear_f32: Y = ((P_0[i_0] + P_1[i_1]) + ...) over fp32 partials
 *     (fusion.cpp:64-77), int32 row maps.  Synchronises. */
typedef struct laq_tc_features laq_tc_features;
int laq_tc_features_create(laq_ctx* ctx, int32_t n_dims, const double* const* d_dims, const int64_t* h_dim_rows,
                           const int64_t* h_dim_cols, const int64_t* const* h_placements, int64_t k,
                           laq_tc_features** out);
int laq_tc_features_destroy(laq_tc_features* f);
int laq_tc_gemm(laq_ctx* ctx, const laq_tc_features* f, const int32_t* const* d_rows, int64_t m, const double* d_W,
                int64_t n, float* d_out);
int laq_apply_fused_linear_f32(laq_ctx* ctx, int32_t n_parts, const int32_t* const* d_idx, int64_t rows,
                               const float* const* d_partials, int64_t l, float* d_out);

/* ---- decision-tree fusion (fusion.hpp:20-55, mlops.hpp:49-80) ----------
 * laq_tree_partial: tree_partial (fusion.cpp:39-47) for one dimension B
 * (rows x cols fp64): P[r, c] = sum over nodes n (in order) with
 * B[r, node_col[n]] * scale[n] > thr[n] of 1 * path_rows[n, c]; node_col[n] = -1
 * for a node whose feature the dim does not place (reads 0); scale[n] = the
 * placement value (NULL = all 1).  Bit-identical to the
 * reference.  predict_tree's scores (mlops.cpp:254-268) are the same call on T
 * with every node.  d_out rows x l.  p <= 2048 nodes.  Synchronises.
 * laq_apply_fused_tree: apply_fused_tree (fusion.cpp:138-159) /
 * predict_tree's decode (mlops.cpp:269-280): scores = ((P_0[i_0] + P_1[i_1]) +
 * ...), label = labels[c] of the unique leaf with scores[c] == path_score[c].
 * d_idx NULL (or d_idx[j] NULL) = identity rows.  LAQ_ERR_MODEL for the first
 * row matching no leaf or several (*h_bad_row, *h_bad_several).  Synchronises. */
int laq_tree_partial(laq_ctx* ctx, const double* d_B, int64_t rows, int64_t cols, int64_t p,
                     const int64_t* h_node_col, const double* h_node_scale, const double* h_thr,
                     const double* h_path_rows, int64_t l, double* d_out);
int laq_apply_fused_tree(laq_ctx* ctx, int32_t n_parts, const int64_t* const* d_idx, int64_t rows,
                         const double* const* d_partials, int64_t l, const double* h_path_score,
                         const int64_t* h_labels, int64_t* d_out, int64_t* h_bad_row, int32_t* h_bad_several);

/* ---- aggregate-MM (laqops.hpp:112-166) --------------------------------- */

/* groupby_sum_single (laqops.cpp:376-413): join R and S on key, sum R's values
 * per S group; groups = distinct group_s ascending, zero-sum groups included.
 * Output capacity n_s.  Synchronises. */
int laq_groupby_sum_single(laq_ctx* ctx, const int64_t* d_keys_r, const double* d_vals_r,
                           int64_t n_r, const int64_t* d_keys_s, const int64_t* d_group_s,
                           int64_t n_s, int64_t* d_out_groups, double* d_out_sums,
                           int64_t* h_n_groups);

/* groupby_sum_multi (laqops.cpp:415-455): present tuples only, ascending.
 * d_out_keys is n_cols x capacity (column-major: key c of group g at
 * [c*capacity + g]); capacity n. Synchronises. */
int laq_groupby_sum_multi(laq_ctx* ctx, int32_t n_cols, const int64_t* const* d_cols,
                          const double* d_vals, int64_t n, int64_t* d_out_keys, double* d_out_sums,
                          int64_t capacity, int64_t* h_n_groups);

/* sort_rows (laqops.cpp:457-478): stable lexicographic sort of the rows of a
 * row-major fp64 rows x cols matrix on h_key_cols (h_desc[k] != 0: descending),
 * ties in the original row order, -0.0 == 0.0.  LAQ_ERR_INDEX on a bad key
 * column. Synchronises. */
int laq_sort_rows(laq_ctx* ctx, const double* d_t, int64_t rows, int64_t cols, const int64_t* h_key_cols,
                  const int32_t* h_desc, int32_t n_keys, double* d_out);

/* ---- sparse formats and SpGEMM (matrix.hpp:44-100) ------------------------ */

/* check_canonical(SparseCoo) (matrix.cpp:243-255): in bounds, sorted by
 * (row, col), no duplicates; LAQ_ERR_GENERIC with the reference's message for
 * the first offending entry. Synchronises. */
int laq_coo_check(laq_ctx* ctx, const int64_t* d_row_idx, const int64_t* d_col_idx, int64_t nnz, int64_t rows,
                  int64_t cols);
/* csr_from_coo (matrix.cpp:210-221): validates like laq_coo_check, then
 * d_row_ptr (rows + 1); col_idx / values are the COO's unchanged. */
int laq_csr_from_coo(laq_ctx* ctx, const int64_t* d_row_idx, const int64_t* d_col_idx, int64_t nnz, int64_t rows,
                     int64_t cols, int64_t* d_row_ptr);
/* coo_from_csr (matrix.cpp:198-208): the row index of every stored entry. */
int laq_coo_from_csr(laq_ctx* ctx, const int64_t* d_row_ptr, int64_t rows, int64_t nnz, int64_t* d_row_idx);
/* spmm (matrix.cpp:81-123): C = A B for canonical CSR operands, Gustavson
 * semantics bit for bit: every (i, j) sums its products a(i,k) b(k,j) from 0.0
 * in A-row then B-row order, exact zeros dropped, columns ascending.
 * d_c_row_ptr has a_rows + 1 entries; if *h_nnz > capacity returns
 * LAQ_ERR_CAPACITY (nothing written to d_c_col_idx / d_c_values).
 * LAQ_ERR_SHAPE when a_cols != b_rows. Synchronises. */
int laq_spmm(laq_ctx* ctx, const int64_t* d_a_row_ptr, const int64_t* d_a_col_idx, const double* d_a_values,
             int64_t a_rows, int64_t a_cols, const int64_t* d_b_row_ptr, const int64_t* d_b_col_idx,
             const double* d_b_values, int64_t b_rows, int64_t b_cols, int64_t* d_c_row_ptr, int64_t* d_c_col_idx,
             double* d_c_values, int64_t capacity, int64_t* h_nnz);

/* ---- selection (laqops.hpp:37-52; predicate.hpp:15-103) ------------------- */

/* A typed Predicate (predicate.hpp:15-57): integer constants (ilo/ihi/iset) or
 * float constants (flo/fhi/fset); sets are host arrays (any order). */
typedef struct {
  int32_t kind;     /* laq_pred_kind */
  int32_t is_float;
  int64_t ilo, ihi;
  double flo, fhi;
  const int64_t* iset;
  const double* fset;
  int64_t set_len;
} laq_pred;
/* build_selection_mask (laqops.cpp:65-79): d_mask[i] = pred.matches(col[i])
 * (1/0), or AND-ed into d_mask when and_into != 0 (mask_and).  d_col is int64
 * (col_is_float = 0) or double.  LAQ_ERR_TYPE on a typed mismatch (only for a
 * non-empty column, as the reference throws from matches()). Synchronises. */
int laq_selection_mask(laq_ctx* ctx, const void* d_col, int32_t col_is_float, int64_t n, const laq_pred* pred,
                       uint8_t* d_mask, int32_t and_into);
/* mask_and (laqops.cpp:87-93). */
int laq_mask_and(laq_ctx* ctx, const uint8_t* d_a, const uint8_t* d_b, int64_t n, uint8_t* d_out);
/* apply_mask's row selection (laqops.cpp:95-121): ascending positions of the
 * set mask entries into d_idx (capacity n; NULL to count only). Synchronises. */
int laq_mask_indices(laq_ctx* ctx, const uint8_t* d_mask, int64_t n, int64_t* d_idx, int64_t* h_count);
/* Row gather d_dst[r] = d_src[d_idx[r]] (d_idx NULL: identity) over rows of
 * row_elems elements: apply_mask for columns / DenseMat rows, the exact
 * one-hot spmm_dense(I, to_matrix(col)) of run_query_laq (cli.cpp:96-101) and
 * column_to_ints (cli.cpp:65-69).  src_kind 0 int32, 1 int64, 2 double;
 * out_kind 1 int64 (copy; integer sources), 2 double ((double) v), 3 int64
 * llround((double) v). */
int laq_gather(laq_ctx* ctx, const void* d_src, int32_t src_kind, int64_t row_elems, const int64_t* d_idx, int64_t n,
               void* d_dst, int32_t out_kind);
/* dense_matmul(ones(1 x n), v) (cli.cpp:103-107): the sequential fp64 sum in
 * row order (integral inputs whose partial sums stay below 2^53 are summed in
 * parallel, exactly). Synchronises. */
int laq_sum_f64(laq_ctx* ctx, const double* d_v, int64_t n, double* h_out);

/* ---- ingest: the reference's CSV table format parsed on the device
 *      (load_csv storage.cpp:112-150; load_dataset cli.cpp:483-513) ---- */

typedef struct laq_csv laq_csv;
/* Index the lines of a CSV text already in device memory (caller-owned, kept
 * alive until laq_csv_close): getline semantics -- '\n' separated, a final line
 * without '\n' counts, a trailing '\n' opens none.  *h_lines = rows. */
int laq_csv_open(laq_ctx* ctx, const char* d_text, int64_t nbytes, laq_csv** out, int64_t* h_lines);
/* Parse every line into n_cols device columns (d_cols[c]: int64 for
 * LAQ_COL_KEY / LAQ_COL_INT, double for LAQ_COL_FLOAT; capacity = lines),
 * std::from_chars semantics per field.  The first failing line in file order
 * returns LAQ_ERR_FORMAT with the reference's message ("line N: expected K
 * fields" / "missing value" / "bad integer 'x'" / "bad float 'x'").
 * LAQ_ERR_UNSUPPORTED for a float with > 19 significant digits whose dropped
 * digits decide the rounding. */
int laq_csv_parse(laq_ctx* ctx, const laq_csv* f, int32_t n_cols, const int32_t* h_kinds, void* const* d_cols);
int laq_csv_close(laq_csv* f);

/* ---- star schema + query plan driver (storage.hpp:75-100, cli.cpp:73-138) ---- */

enum laq_col_kind { LAQ_COL_KEY = 0, LAQ_COL_INT = 1, LAQ_COL_FLOAT = 2 }; /* storage.hpp:14 */

/* A StarSchema resident in HBM: integer columns are narrowed to int32 on the
 * device (range-checked; LAQ_ERR_CAPACITY if a value does not fit). */
int laq_star_create(laq_ctx* ctx, laq_star** out);
int laq_star_destroy(laq_star* star);
/* Add a table from host (or, through unified addressing, device) columns:
 * key/int kinds are int64 (the reference's
 * IntColumn, storage.hpp:35) when int_width == 8, or already-narrowed int32
 * when int_width == 4; float columns are double.  The table added with
 * is_fact=1 is the fact table.  Key columns must be non-negative
 * (LAQ_ERR_FORMAT, storage.cpp:54-56).  Synchronises. */
int laq_star_add_table(laq_star* star, const char* name, int32_t is_fact, int64_t rows,
                       int32_t n_cols, const char* const* col_names, const int32_t* col_kinds,
                       int32_t int_width, const void* const* h_cols);
/* Same, from int32 DEVICE columns already narrowed (no copy; caller keeps them alive). */
int laq_star_add_table_device(laq_star* star, const char* name, int32_t is_fact, int64_t rows,
                              int32_t n_cols, const char* const* col_names,
                              const int32_t* col_kinds, const int32_t* const* d_cols);
/* StarSchema link (storage.hpp:75-81); checks pk uniqueness (storage.cpp:200-214). */
/* Register a table whose integer columns are caller-owned device buffers in a
 * byte-packed layout (the compact transfer format): value = stored + offset[c],
 * stored as uint8 (width 1), uint16 (width 2) or int32 (width 4, offset 0); each
 * buffer has >= 16 readable bytes past its end.  Scans read packed columns
 * directly (the stream kernel); a query that needs another scan variant on a
 * packed-only column (fact InSet filter, fact group-by, G > 4096) fails with
 * LAQ_ERR_UNSUPPORTED. */
int laq_star_add_table_device_packed(laq_star* star, const char* name, int32_t is_fact, int64_t rows,
                                     int32_t n_cols, const char* const* col_names, const int32_t* col_kinds,
                                     const void* const* d_cols, const int32_t* widths, const int32_t* offsets);
/* Register a table whose integer columns are caller-owned device bitstreams
 * (the bit-packed transfer format): column c stores bits[c] (1..32) bits per
 * row, value = stored + offsets[c]; rows are little-endian bit fields packed
 * back to back, so a group of 32 rows is bits[c] consecutive 32-bit words.
 * Each buffer is 4-byte aligned and holds ceil(rows/128)*4*bits[c] words plus
 * 16 bytes.  Only the direct scan reads these, with every scanned column
 * bit-packed (LAQ_ERR_UNSUPPORTED otherwise); scan ranges start at multiples
 * of 32 rows. */
int laq_star_add_table_device_bitpacked(laq_star* star, const char* name, int32_t is_fact, int64_t rows,
                                        int32_t n_cols, const char* const* col_names, const int32_t* col_kinds,
                                        const void* const* d_cols, const int32_t* bits, const int32_t* offsets);
int laq_star_add_link(laq_star* star, const char* fact_fk, const char* dim_name,
                      const char* dim_pk);

/* Query description (benchgen.hpp:296-326).  Predicates are Predicate kinds
 * (predicate.hpp:15-28) over integer columns. */
enum laq_pred_kind {
  LAQ_PRED_LT = 0, LAQ_PRED_LE = 1, LAQ_PRED_EQ = 2, LAQ_PRED_GE = 3, LAQ_PRED_GT = 4,
  LAQ_PRED_BETWEEN = 5, LAQ_PRED_INSET = 6
};
typedef struct {
  int32_t target;        /* -1 = fact, else index into joins */
  const char* column;
  int32_t kind;          /* laq_pred_kind */
  int32_t is_float;      /* 1: float constants (TypeError against int columns) */
  int64_t lo, hi;        /* integer constants (hi used by BETWEEN) */
  const int64_t* set;    /* INSET values */
  int64_t set_len;
} laq_filter_desc;
typedef struct { const char* fact_fk; const char* dim_name; const char* dim_pk; } laq_link_desc;
typedef struct { int32_t target; const char* column; } laq_group_desc;
typedef struct {
  int32_t n_joins;
  const laq_link_desc* joins;
  int32_t n_filters;
  const laq_filter_desc* filters;
  const char* measure;
  int32_t n_group;
  const laq_group_desc* group_by;
  int32_t order_by;
} laq_query_desc;

/* Prepare a plan: resolves names (LAQ_ERR_NAME), types (LAQ_ERR_TYPE) and the
 * dense group-id space; *h_n_groups = number of group-id slots G.  A join with
 * no filter and no group column whose fact keys all have a dim row (checked once
 * per star on the device and cached) is left out of the scan: it cannot drop a
 * fact row.  Plans snapshot that check: re-prepare after rewriting fact key
 * columns registered with laq_star_add_table_device. */
int laq_query_prepare(laq_ctx* ctx, const laq_star* star, const laq_query_desc* q, laq_plan** out,
                      int64_t* h_n_groups);
/* Enqueue the plan on the context stream (no host sync; graph-capturable):
 * rebuild the per-link probe tables from the dimension filters, then one
 * fused scan of the fact table that accumulates, per group id, d_acc[2g] =
 * surviving row count and d_acc[2g+1] = SUM(measure) (exact int64).  d_acc
 * (2*G int64) is zeroed by the call unless accumulate != 0. */
int laq_plan_execute(laq_ctx* ctx, laq_plan* plan, int64_t* d_acc, int32_t accumulate);
/* The two halves of laq_plan_execute, for per-kernel timing: rebuild the
 * per-link code tables (dimension filters), then the fused fact scan. */
int laq_plan_build_codes(laq_ctx* ctx, laq_plan* plan);
/* The code tables of a batch of plans (e.g. one step of queries) in one launch
 * (falls back to one launch per plan beyond 24 links in total). */
int laq_plans_build_codes(laq_ctx* ctx, int32_t n_plans, laq_plan* const* plans);
/* Scan a batch of 2-3 plans that read the same fact columns in the same roles
 * (e.g. Q1.1-Q1.3) in ONE pass over the fact table: each column vector is
 * loaded once and every query evaluates its own filters, probes and group bins
 * into its own accumulator d_accs[q].  *h_shared = 1 when the batch qualified,
 * 0 when it was scanned one plan at a time (same results either way). */
int laq_plans_scan_shared(laq_ctx* ctx, int32_t n_plans, laq_plan* const* plans, int64_t* const* d_accs,
                          int32_t accumulate, int32_t* h_shared);
int laq_plan_scan(laq_ctx* ctx, laq_plan* plan, int64_t* d_acc, int32_t accumulate);
/* Batched scan: a batch of 1..4 prepared plans over the same fact table run
 * as ONE pass (scan_batch_kernel, csrc/ssb_batch.cuh) with one probe per row
 * per dimension link for the whole batch: each link's per-query codes are
 * dictionary-encoded on the device (laq_batch_build), staged in shared
 * memory, and decoded into every query's group id at once.  A batch the
 * fused pass cannot take (InSet / packed fact columns, > 4096 groups, > 6
 * links ...) is scanned plan by plan with identical results; *h_fused and
 * laq_batch_info say which.  Each plan keeps its own accumulator
 * (laq_plan_emit).  The reference runs the same queries one run_query_laq
 * (cli.cpp:73-138) at a time; the results are those of each query alone.
 * The batch borrows the plans: destroy it before them. */
typedef struct laq_batch laq_batch;
int laq_batch_prepare(laq_ctx* ctx, int32_t n_plans, laq_plan* const* plans, laq_batch** out, int32_t* h_fused);
/* Every plan's code tables (one launch) + the link dictionaries (3 launches). */
int laq_batch_build(laq_ctx* ctx, laq_batch* batch);
/* d_accs[q]: plan q's [2*G] int64 (count, sum) accumulator. */
int laq_batch_scan(laq_ctx* ctx, laq_batch* batch, int64_t* const* d_accs, int32_t accumulate);
int laq_batch_info(const laq_batch* batch, int32_t* fused, int64_t* bytes_per_row, int32_t* n_links, char* why,
                   size_t why_cap);
int laq_batch_destroy(laq_batch* batch);
/* Scan only fact rows [row0, row0 + rows) (row0 a multiple of 4) with the code
 * tables of the last build: lets a caller overlap the upload of later row
 * chunks with the scan of earlier ones (accumulate = 1 after the first chunk). */
int laq_plan_scan_range(laq_ctx* ctx, laq_plan* plan, int64_t row0, int64_t rows, int64_t* d_acc,
                        int32_t accumulate);
/* Bytes of fact columns the scan streams per row (the roofline unit). */
int64_t laq_plan_bytes_per_row(const laq_plan* plan);
/* Joins the plan's scan actually probes (after eliding covered filter-free links). */
int32_t laq_plan_scanned_links(const laq_plan* plan);
/* Turn an accumulator (host copy, e.g. after an all-reduce) into the
 * run_query_laq result rows [group cols..., sum] (row-major), present groups
 * only, ascending (groupby_sum_multi + sort_rows; laqops.cpp:415-478).  A plain
 * Sum query yields one 1x1 row (cli.cpp:103-107). */
int laq_plan_emit(const laq_plan* plan, const int64_t* h_acc, double* h_out, int64_t capacity,
                  int64_t* h_rows, int64_t* h_cols);
int laq_plan_destroy(laq_plan* plan);

/* run_query_laq (cli.cpp:73-138) in one call: prepare + execute + emit. */
int laq_run_query(laq_ctx* ctx, const laq_star* star, const laq_query_desc* q, double* h_out,
                  int64_t capacity, int64_t* h_rows, int64_t* h_cols);

/* measure_selectivity (benchgen.cpp:366-411) on the device: surviving fact
 * rows / fact rows. Synchronises. */
int laq_measure_selectivity(laq_ctx* ctx, const laq_star* star, const laq_query_desc* q,
                            double* h_out);

/* ---- fusion cost model (fusion.hpp:57-76; fusion.cpp:181-224) ----------- */
int laq_speedup_ratio_linear(int64_t i, int64_t k, int64_t l, const int64_t* dim_rows,
                             int32_t n_dims, double* h_out);
int laq_speedup_ratio_tree(int64_t i, int64_t k, int64_t l, int64_t p, const int64_t* dim_rows,
                           int32_t n_dims, double* h_out);
int laq_decide_fusion(double ratio, double threshold, int32_t* h_out);
/* The B200 plan model for the tensor-core operators (no reference function:
 * the paper's Eq. 2 above counts CPU sparse-matrix work; on the tensor cores
 * both plans are GEMM + gather and the winner is set by tensor time vs HBM
 * bytes).  Predicted seconds of the fused plan (prefuse P_j = B_j W on every
 * dim + the fp32 gather-apply) and of the non-fused plan (one GEMM over the
 * gathered rows), from the measured bf16 tensor rate (FLOP/s) and HBM
 * bandwidth (B/s); *h_fused = t_fused < t_nonfused.  Calibrated on the
 * 164-cell complexity sweep, checked on a disjoint hold-out grid
 * (profiles/round2/planner_holdout.json).  No device needed. */
int laq_plan_linear_device(int64_t target_rows, int64_t k, int64_t l, const int64_t* dim_rows, int32_t n_dims,
                           double tensor_flops, double hbm_bytes_per_s, double* h_t_fused, double* h_t_nonfused,
                           int32_t* h_fused);

#ifdef __cplusplus
}
#endif
#endif /* LAQ_B200_H */
