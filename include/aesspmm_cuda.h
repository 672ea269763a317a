/*
 * aesspmm_cuda.h — the C-ABI boundary of the B200-native AES-SpMM path.
 *
 * Implemented by paper_2503_18427_b200/libaescuda.so (hand-written sm_100a
 * CUDA; no CPU fallback).  Plain pointers and sizes only: no C++ or torch
 * types cross this boundary.  Every function returns an aes_status (0 = OK);
 * aes_last_error() gives the message for the calling thread, using the
 * reference's exception strings so a binding can re-raise them verbatim
 * ("ZeroWidth", "ShapeMismatch", "PlanMatrixMismatch", "EmptyMatrix",
 * "NonFinite", "invalid QuantParams", "bits must be 1..16",
 * "<CsrError> at row <i>" — proj/src/{sampling,spmm,quantize,matrix}.cpp).
 *
 * Two tiers:
 *   1. Handle API (host buffers in, host buffers out).  These are exactly the
 *      entry points the reference's FFI binds — proj/bindings/module.cpp:52-144
 *      — so a pybind11 / ctypes / cgo binding maps 1:1 onto them.  Objects
 *      (CSR, plan set, quantized features) live in HBM behind opaque handles.
 *   2. Device API (device pointers + a cudaStream_t passed as void*).  Used by
 *      the handle tier, the benchmark and the multi-GPU layer driver; it never
 *      synchronises the stream and never allocates unless it says so.
 *
 * Strategy values follow the reference enum order
 * (proj/include/aesspmm/sampling.hpp:14).
 */
#ifndef AESSPMM_CUDA_H
#define AESSPMM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AES_API __attribute__((visibility("default")))

typedef enum {
    AES_OK = 0,
    AES_ERR_ZERO_WIDTH = 1,      /* "ZeroWidth"              sampling.cpp:30,63,106 */
    AES_ERR_SHAPE = 2,           /* "ShapeMismatch"          spmm.cpp:13, gnn.cpp:13,44 */
    AES_ERR_PLAN_MISMATCH = 3,   /* "PlanMatrixMismatch"     spmm.cpp:44-46 */
    AES_ERR_EMPTY = 4,           /* "EmptyMatrix"            quantize.cpp:12 */
    AES_ERR_NONFINITE = 5,       /* "NonFinite"              quantize.cpp:16 */
    AES_ERR_QPARAMS = 6,         /* "invalid QuantParams"    quantize.cpp:24-26 */
    AES_ERR_BITS = 7,            /* "bits must be 1..16"     quantize.cpp:13 */
    AES_ERR_CSR_INVALID = 8,     /* ValidationResult::message()  matrix.cpp:11-26 */
    AES_ERR_INVALID_ARG = 9,     /* null handle / bad argument */
    AES_ERR_CUDA = 10,           /* CUDA runtime error (message has details) */
    AES_ERR_UNSUPPORTED = 11,    /* layout the kernels do not take */
    AES_ERR_NOT_SQUARE = 12,     /* "NotSquare"              matrix.cpp:131 */
    AES_ERR_IO = 13              /* std::runtime_error of io.cpp ("BadMagic: path", ...) */
} aes_status;

typedef enum { AES_ADAPTIVE = 0, AES_AFS = 1, AES_SFS = 2, AES_FULL = 3 } aes_strategy;

/* CsrError codes of proj/include/aesspmm/matrix.hpp:44-51. */
typedef enum {
    AES_CSR_OK = 0, AES_CSR_NON_MONOTONIC = 1, AES_CSR_COL_OUT_OF_RANGE = 2,
    AES_CSR_UNSORTED = 3, AES_CSR_LENGTH_MISMATCH = 4, AES_CSR_NOT_SQUARE = 5
} aes_csr_error;

AES_API const char* aes_last_error(void);
AES_API const char* aes_status_name(int status);
AES_API int aes_version(void);

/* ======================================================================
 * Scalar formulas (host-callable; the same __host__ __device__ code the
 * kernels run).
 * ====================================================================== */

/* select_strategy — proj/include/aesspmm/sampling.hpp:61, sampling.cpp:29-54 */
AES_API int aes_select_strategy(uint64_t row_nnz, uint32_t width, uint32_t* chunk_len,
                                uint32_t* sample_cnt);
/* hash_start — sampling.hpp:64-65, sampling.cpp:56-60 */
AES_API uint32_t aes_hash_start(uint32_t current_ind, uint64_t row_nnz, uint32_t chunk_len);

/* ======================================================================
 * Tier 1: handle API (host buffers) — mirrors proj/bindings/module.cpp
 * ====================================================================== */

typedef struct aes_csr_s* aes_csr_t;      /* CsrMatrix resident in HBM */
typedef struct aes_plan_s* aes_plan_t;    /* SamplePlanSet resident in HBM */
typedef struct aes_qfeat_s* aes_qfeat_t;  /* QuantizedFeatures resident in HBM */

/* CsrMatrix(n_rows, n_cols, row_ptr, col_ind, val) with validate_csr —
 * module.cpp:17-33 (copies in, validates on the GPU; on failure returns
 * AES_ERR_CSR_INVALID with ValidationResult::message()).  row_ptr_len,
 * nnz_len are the host array lengths (the reference checks them). */
AES_API int aes_csr_create(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                           uint64_t row_ptr_len, const uint32_t* col_ind, const float* val,
                           uint64_t nnz_len, aes_csr_t* out);
/* Same, without validation, from DEVICE arrays that stay owned by the caller
 * (no copy).  Used by the device tier / layer driver. */
AES_API int aes_csr_wrap_device(uint64_t n_rows, uint64_t n_cols, const uint64_t* d_row_ptr,
                                const uint32_t* d_col_ind, const float* d_val, uint64_t nnz,
                                aes_csr_t* out);
/* validate_csr on host arrays (matrix.cpp:28-52): *error = CsrError code,
 * *row = offending row; returns AES_ERR_CSR_INVALID with the message. */
AES_API int aes_validate_csr(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                             uint64_t row_ptr_len, const uint32_t* col_ind, uint64_t nnz_len,
                             int* error, uint64_t* row);
/* Structure-only CSR (row_ptr only): enough for row_stats, sampling_rate and
 * plan export; not for SpMM. */
AES_API int aes_csr_structure(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr,
                              aes_csr_t* out);
AES_API int aes_csr_destroy(aes_csr_t a);
AES_API int aes_csr_shape(aes_csr_t a, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz);
/* Device views of the CSR arrays (for zero-copy interop). */
AES_API int aes_csr_device_ptrs(aes_csr_t a, const uint64_t** row_ptr, const uint32_t** col_ind,
                                const float** val);
/* Copy the CSR back to host arrays (sizes n_rows+1 and nnz). */
AES_API int aes_csr_download(aes_csr_t a, uint64_t* row_ptr, uint32_t* col_ind, float* val);
/* row_stats — matrix.hpp:82, matrix.cpp:54-63 (row_nnz may be NULL). */
AES_API int aes_csr_row_stats(aes_csr_t a, uint64_t* row_nnz, uint64_t* max_row_nnz,
                              double* avg_degree);
/* gcn_normalize(a, add_self_loops) — matrix.hpp:76, matrix.cpp:130-144 */
AES_API int aes_gcn_normalize(aes_csr_t a, int add_self_loops, aes_csr_t* out);

/* build_plan_set(matrix, width, strategy) — sampling.hpp:70-72,
 * sampling.cpp:104-118, module.cpp:107-108.  Builds the per-row plan and the
 * sampled CSR (slot order) in HBM. */
AES_API int aes_build_plan_set(aes_csr_t a, uint32_t width, int strategy, aes_plan_t* out);
/* A plan set given as host data (SamplePlanSet built or edited by the
 * caller): per-row chunk_len/sample_cnt and starts in CSR form (starts_ptr
 * n+1).  Filled in slot order exactly like a built plan (spmm.cpp:54-76).
 * Validated first (the reference reads out of range instead): starts_ptr
 * must begin at 0 and be non-decreasing with at least sample_cnt starts per
 * row, and every window must fit its row (start + chunk_len <= row nnz);
 * otherwise AES_ERR_INVALID_ARG "invalid plan: ... row <i>". */
AES_API int aes_plan_from_host(aes_csr_t a, uint32_t width, int strategy, const uint32_t* chunk_len,
                               const uint32_t* sample_cnt, const uint64_t* starts_ptr,
                               const uint32_t* starts, aes_plan_t* out);
AES_API int aes_plan_destroy(aes_plan_t p);
AES_API int aes_plan_info(aes_plan_t p, uint32_t* width, int* strategy, uint64_t* n_rows,
                          uint64_t* total_slots, uint64_t* total_starts);
/* Export SamplePlanSet::plans (module.cpp:78-81) as flat host arrays:
 * chunk_len[n], sample_cnt[n], starts_ptr[n+1], starts[total_starts]. */
AES_API int aes_plan_export(aes_plan_t p, uint32_t* chunk_len, uint32_t* sample_cnt,
                            uint64_t* starts_ptr, uint32_t* starts);
/* Sampled CSR device views (srow_ptr n+1 u64, scol/sval total_slots). */
AES_API int aes_plan_device_ptrs(aes_plan_t p, const uint64_t** srow_ptr, const uint32_t** scol,
                                 const float** sval);
/* Copy the sampled CSR (srow_ptr n+1, scol/sval total_slots) to host. */
AES_API int aes_plan_download(aes_plan_t p, uint64_t* srow_ptr, uint32_t* scol, float* sval);
/* sampling_rate(plans, row_stats(matrix)) — sampling.cpp:120-152,
 * module.cpp:109-116.  per_row (n doubles) may be NULL. */
AES_API int aes_sampling_rate(aes_plan_t p, aes_csr_t a, double* aggregate,
                              double* unique_coverage, double* per_row);

/* spmm_exact(a, b) — spmm.hpp:19-20, spmm.cpp:18-36, module.cpp:118-123.
 * b: host row-major b_rows x f; c: host row-major a.n_rows x f. */
AES_API int aes_spmm_exact(aes_csr_t a, const float* b, uint64_t b_rows, uint64_t f, float* c);
/* cdf_stats(rates) — bench.hpp:58-59, bench.cpp:124-138: the empirical CDF
 * of per-row sampling rates as steps (rate, cumulative fraction), sorted by
 * rate, ties (==) merged into one step carrying the last fraction.
 * out_rate / out_frac hold up to n entries; *n_steps gets the step count.
 * n == 0: AES_ERR_INVALID_ARG "rates must be nonempty".  Bit-exact. */
AES_API int aes_cdf_stats(const double* rates, uint64_t n, double* out_rate, double* out_frac,
                          uint64_t* n_steps);
/* cdf_stats(sampling_rate(plans, row_stats(a)).per_row) with the per-row
 * rates kept on the device (outputs as above, capacity n_rows). */
AES_API int aes_sampling_rate_cdf(aes_plan_t p, aes_csr_t a, double* out_rate, double* out_frac,
                                  uint64_t* n_steps);
/* Device tier: rates, outputs and *n_steps in device memory; workspace of
 * aes_cdf_workspace_bytes(n) bytes; stream-ordered (radix sort + scan). */
AES_API uint64_t aes_cdf_workspace_bytes(uint64_t n);
AES_API int aes_dev_cdf_stats(const double* rates, uint64_t n, double* out_rate, double* out_frac,
                              uint64_t* n_steps, void* workspace, size_t workspace_bytes, void* stream);

/* spmm_sampled(a, b, plans) — spmm.hpp:25-26, spmm.cpp:40-107, module.cpp:124-131.
 * fma/loads counters (spmm_sampled_instrumented, spmm.cpp:109-114) may be NULL. */
AES_API int aes_spmm_sampled(aes_csr_t a, const float* b, uint64_t b_rows, uint64_t f,
                             aes_plan_t p, float* c, uint64_t* fma_count, uint64_t* loads_a,
                             uint64_t* loads_b);

/* Stream-ordered form of aes_spmm_sampled for pipelined callers: enqueues
 * H2D(b) -> SpMM -> D2H(c) on `stream` (NULL = library stream) and returns.
 * b and c should be pinned; they must stay valid until the stream reaches
 * this point.  Successive calls on two streams overlap one call's H2D with
 * the previous call's D2H (both copy engines busy).  The plan (and its
 * matrix) may be destroyed right after the call: aes_plan_destroy orders its
 * frees after the work enqueued here on `stream`.  The plan must have been
 * built on `a`. */
AES_API int aes_spmm_sampled_async(aes_csr_t a, const float* b, uint64_t b_rows, uint64_t f,
                                   aes_plan_t p, float* c, void* stream);

/* quantize(x, bits) = quantize(x, fit_params(x, bits)) — module.cpp:133-139,
 * quantize.cpp:11-51.  x: host rows x cols f32. */
AES_API int aes_quantize(const float* x, uint64_t rows, uint64_t cols, uint32_t bits,
                         aes_qfeat_t* out);
/* fit_params(x, bits) — quantize.hpp:28, quantize.cpp:11-21 */
AES_API int aes_fit_params(const float* x, uint64_t rows, uint64_t cols, uint32_t bits, float* x_min,
                           float* x_max);
/* quantize(x, p) with explicit params — quantize.hpp:31 */
AES_API int aes_quantize_with(const float* x, uint64_t rows, uint64_t cols, float x_min,
                              float x_max, uint32_t bits, aes_qfeat_t* out);
/* QuantizedFeatures from host uint16 codes (quantize.hpp:20-25). */
AES_API int aes_qfeat_from_codes(const uint16_t* codes, uint64_t rows, uint64_t cols,
                                 float x_min, float x_max, uint32_t bits, aes_qfeat_t* out);
AES_API int aes_qfeat_destroy(aes_qfeat_t q);
AES_API int aes_qfeat_info(aes_qfeat_t q, uint64_t* rows, uint64_t* cols, float* x_min,
                           float* x_max, uint32_t* bits);
/* codes as uint16 (the reference's in-memory type, module.cpp:96-101). */
AES_API int aes_qfeat_codes(aes_qfeat_t q, uint16_t* codes);
/* dequantize(qf) — quantize.hpp:34, quantize.cpp:53-64, module.cpp:140-143 */
AES_API int aes_dequantize(aes_qfeat_t q, float* x);
/* spmm_sampled(a, dequantize(q), plans) with the dequantization fused into
 * the gather (int8 feature bytes).  plans == NULL -> exact (spmm_exact). */
AES_API int aes_spmm_sampled_q8(aes_csr_t a, aes_qfeat_t q, aes_plan_t p, float* c);

/* dense_matmul(a, b) — gnn.hpp:64, gnn.cpp:11-31 (host buffers). */
AES_API int aes_dense_matmul(const float* a, uint64_t m, uint64_t k, const float* b, uint64_t n,
                             float* c);
/* gcn_forward(adj, features, model, plans) — gnn.hpp:37-40, gnn.cpp:66-78.
 * dims[0..n_layers]; weights/biases concatenated per layer (bias_len[l] is
 * 0 or dims[l+1]); p == NULL -> exact aggregation. */
AES_API int aes_gcn_forward(aes_csr_t adj, const float* x, const uint64_t* dims, int n_layers,
                            const float* weights, const float* biases, const uint64_t* bias_len,
                            aes_plan_t p, float* out);

/* sage_forward(adj_mean, features, model, plans) — gnn.hpp:43-46,
 * gnn.cpp:80-95: H <- act(concat(H, spmm(adj_mean, H)) @ W + b); layer l's
 * weight is (2*dims[l]) x dims[l+1]. */
AES_API int aes_sage_forward(aes_csr_t adj_mean, const float* x, const uint64_t* dims, int n_layers,
                             const float* weights, const float* biases, const uint64_t* bias_len,
                             aes_plan_t p, float* out);
/* GCN (kind 0) / SAGE-mean (kind 1) forward with an opt-in fast layer
 * transform: fast_gemm != 0 runs each GEMM with K, N <= 128 on the tcgen05
 * tensor cores (TF32; NOT bit-exact, see aes_dev_gemm_tf32).  fast_gemm == 0
 * is aes_gcn_forward / aes_sage_forward. */
AES_API int aes_gnn_forward_ex(int kind, aes_csr_t adj, const float* x, const uint64_t* dims,
                               int n_layers, const float* weights, const float* biases,
                               const uint64_t* bias_len, aes_plan_t p, int fast_gemm, float* out);
/* row_mean_normalize(a) — matrix.hpp:80-82, matrix.cpp:146-158 */
AES_API int aes_row_mean_normalize(aes_csr_t a, aes_csr_t* out);
/* argmax_rows(logits) — gnn.hpp:52, gnn.cpp:105-116 (ties -> lowest index) */
AES_API int aes_argmax_rows(const float* x, uint64_t rows, uint64_t cols, uint32_t* out);
/* evaluate(logits, labels, reference_logits, mask) — gnn.hpp:56-60,
 * gnn.cpp:118-155.  reference_logits / mask may be NULL (mask_len 0 = all
 * rows); per_class (cols entries) may be NULL.  Errors: "labels length !=
 * n_nodes", "mask length != n_nodes", "LabelOutOfRange". */
AES_API int aes_evaluate(const float* logits, uint64_t rows, uint64_t cols, const uint32_t* labels,
                         uint64_t labels_len, const float* reference_logits, const uint8_t* mask,
                         uint64_t mask_len, double* accuracy, double* agreement, uint64_t* per_class);

/* Binary files straight to HBM (formats of proj/src/io.cpp:117-220).  The
 * payload streams through pinned double buffers overlapped with the H2D
 * copies; load_ms (may be NULL) receives the wall time, like
 * load_features(path, &load_ms) (io.hpp:36-38).
 *   aes_fmat_info        header: dtype 0 = f32, 1 = u8 codes (+ x_min, x_max)
 *   aes_fmat_load_device payload into a device buffer with row pitch ld_elems
 *   aes_fmat_load_qfeat  dtype-1 file -> HBM QuantizedFeatures (codes + LUT)
 *   aes_csr_load         CSRB -> HBM CsrMatrix, validated on the GPU
 *                        ("invalid CSR payload: ..." as io.cpp:142-143) */
AES_API int aes_fmat_info(const char* path, int* dtype, uint64_t* rows, uint64_t* cols, float* x_min,
                          float* x_max);
AES_API int aes_fmat_load_device(const char* path, void* d_dst, uint64_t ld_elems, double* load_ms);
AES_API int aes_fmat_load_qfeat(const char* path, aes_qfeat_t* out, double* load_ms);
AES_API int aes_fmat_save_f32(const float* x, uint64_t rows, uint64_t cols, const char* path);
AES_API int aes_fmat_save_qfeat(aes_qfeat_t q, const char* path);
AES_API int aes_csr_load(const char* path, aes_csr_t* out, double* load_ms);
AES_API int aes_csr_save(aes_csr_t a, const char* path);

/* ======================================================================
 * Tier 2: device API (device pointers, caller's stream, no sync)
 * ====================================================================== */

/* Workspace bytes for aes_dev_sample_plan / aes_dev_fit_params over n items. */
AES_API size_t aes_dev_scan_workspace_bytes(uint64_t n_rows);

/* Sampler pass 1: per-row (chunk, cnt) and the sampled row pointer
 * srow_ptr[n+1] = exclusive scan of chunk*cnt (single-pass decoupled
 * look-back).  plan_row_ptr supplies row_nnz.  row_params (n x uint2
 * {chunk, cnt}) may be NULL.  Reference: sampling.cpp:29-118. */
AES_API int aes_dev_sample_plan(const uint64_t* plan_row_ptr, uint64_t n_rows, uint32_t width,
                                int strategy, uint64_t* srow_ptr, uint32_t* row_params,
                                void* workspace, size_t workspace_bytes, void* stream);
/* Sampler pass 2: sampled col/val in slot order: slot s + j*cnt of row i
 * <- nonzero row_ptr[i] + start_s + j (spmm.cpp:54-76).  Windows come from
 * plan_row_ptr's row lengths; bases from row_ptr (equal pointers in the
 * usual case). */
AES_API int aes_dev_sample_fill(const uint64_t* plan_row_ptr, const uint64_t* row_ptr,
                                const uint32_t* col_ind, const float* val, uint64_t n_rows,
                                uint32_t width, int strategy, const uint64_t* srow_ptr,
                                uint32_t* scol, float* sval, void* stream);

/* C[i, 0:f] = sum over k in [srow_ptr[i], srow_ptr[i+1]) ascending of
 * sval[k] * B[scol[k], 0:f], rounded as RN(acc + RN(v*b)) — bit-exact with
 * spmm.cpp:77-84.  Every row of C (0:f) is written (zeros for empty rows).
 * Vector path needs ldb, ldc % 4 == 0 and 16-B aligned B, C; the kernel
 * then also writes C columns f..round_up(f,4) (zeros when B's pad is 0).
 * `row_begin` offsets the row range (sharded drivers): rows
 * [row_begin, row_begin + n_rows) of the CSR are computed into C rows
 * [0, n_rows). */
AES_API int aes_dev_spmm_f32(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                             uint64_t n_rows, const float* b, uint64_t ldb, uint64_t f, float* c,
                             uint64_t ldc, void* stream);
/* Same, with a bound on the slots of any one row (0 = unknown).  Sampled
 * plans bound it by their width (Adaptive/Sfs/Afs); exact SpMM and FULL plans
 * do not.  (Kept for callers that know the bound; the default balanced
 * schedule handles hub rows without it, see aes_dev_spmm_set_schedule.) */
AES_API int aes_dev_spmm_f32_ex(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                                uint64_t n_rows, const float* b, uint64_t ldb, uint64_t f, float* c,
                                uint64_t ldc, uint64_t max_row_slots, void* stream);

/* Kernel-schedule override (tuning/benchmarks; 0 = default).  fp32, F <= 128:
 * 1 register-staged batches, 2..8 shared-memory cp.async rings of different
 * depth x warps-per-CTA.  int8: 21-24 dual-stream, 30-45 batch kernel ring x
 * warps (F > 128 as 128-code column tiles), 40 TMA gather, 46/48/49 wide-row
 * kernel ring x warps (128 < F <= 640; the default there), 50-57 fast-mode
 * kernels (55 column tiles, 56/57 wide-row).  Results are bit-identical for
 * every variant. */
AES_API int aes_dev_spmm_set_variant(int variant);
/* Row-group schedule of the SpMM kernels: 1 = static (warp w takes row
 * group w), 2 = heavy-first dynamic (groups with > 4096 slots first, then
 * the rest, by ticket from one counter), 3 = balanced persistent (one wave of
 * resident warps, each owning a contiguous row range with an equal share of
 * slots + rows), 0 = auto (balanced), 6 = int8 batch kernel only: static
 * 32-row groups walked grid-stride by one persistent wave (tuning).  Results
 * are bit-identical under every schedule (each row group is one warp's
 * ordered stream). */
AES_API int aes_dev_spmm_set_schedule(int schedule);

/* Int8 variant: Q is u8 codes (ldq bytes per row), lut[256] the exact
 * dequantized value of each code (aes_dev_dequant_lut).  Result is
 * bit-identical to aes_dev_spmm_f32 over dequantize(Q). */
AES_API int aes_dev_spmm_q8(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                            uint64_t n_rows, const uint8_t* q, uint64_t ldq, uint64_t f,
                            const float* lut, float* c, uint64_t ldc, void* stream);
AES_API int aes_dev_spmm_q8_ex(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                               uint64_t n_rows, const uint8_t* q, uint64_t ldq, uint64_t f,
                               const float* lut, float* c, uint64_t ldc, uint64_t max_row_slots,
                               void* stream);

/* fit_params: result[0] = x_min, result[1] = x_max (first-occurrence
 * semantics of quantize.cpp:14-19), ((uint32_t*)result)[2] = 1 when a
 * non-finite element was seen.  Deterministic two-level reduction. */
AES_API int aes_dev_fit_params(const float* x, uint64_t n, float* result, void* workspace,
                               size_t workspace_bytes, void* stream);
/* codes = quantize(x, {lo, hi, bits}) — quantize.cpp:23-51 (fp64, no
 * contraction).  Codes are u8 when bits <= 8 else u16; rows x cols with row
 * strides ldx (floats) and ldq (codes). */
AES_API int aes_dev_quantize(const float* x, uint64_t rows, uint64_t cols, uint64_t ldx, float lo,
                             float hi, uint32_t bits, void* codes, uint64_t ldq, void* stream);
/* x = dequantize(codes) — quantize.cpp:53-64 */
AES_API int aes_dev_dequantize(const void* codes, uint64_t rows, uint64_t cols, uint64_t ldq,
                               float lo, float hi, uint32_t bits, float* x, uint64_t ldx,
                               void* stream);
/* lut[q] = float(double(q) * step + double(lo)) for q < 2^bits (bits <= 8). */
AES_API int aes_dev_dequant_lut(float lo, float hi, uint32_t bits, float* lut, void* stream);

/* H = act(A @ W + bias): k-ascending, separate mul/add roundings, zero
 * entries of A skipped (gnn.cpp:11-31), bias (may be NULL) then ReLU
 * max(v, 0) when relu != 0 (gnn.cpp:41-52). */
AES_API int aes_dev_gemm_bias_act(const float* a, uint64_t m, uint64_t k, uint64_t lda,
                                  const float* w, uint64_t n, uint64_t ldw, const float* bias,
                                  int relu, float* h, uint64_t ldh, void* stream);

/* Extended layer GEMM: as aes_dev_gemm_bias_act, writing rows
 * [row_offset, row_offset + m) of the replica(s) dsts[0..n_dst) (ld ldh).
 * finite_w != 0 asserts W has no inf/NaN (check with aes_dev_all_finite), which
 * makes the reference's zero-skip result-neutral and lets the kernel drop it.
 * counters != NULL turns on the fused exchange: dsts are every rank's replica
 * (CUDA-IPC peer pointers), and each CTA, after its stores, does a
 * system-scope fence and one release-add on counters[d] for every d — a rank
 * waits for sum-over-producers aes_gemm_ctas(m_p, n) arrivals
 * (aes_dev_wait_counter) before reading its replica.  This replaces the
 * layer's all-gather (gnn.cpp:66-78 run row-sharded). */
/* One exact GCN layer, fused: h = act(SpMM(srow/scol/sval, x) w + bias) for
 * k = F_in <= 128 (k % 4 == 0), n = F_out <= 128, x / h 16-B aligned with
 * ld % 4 == 0 (gnn.cpp:66-78 for one layer: spmm_sampled -> dense_matmul ->
 * add_bias_inplace -> relu_inplace).  One persistent CTA per SM: producer
 * warps gather 128-row tiles of the aggregate into shared memory while
 * consumer warps run the ordered GEMM of the previous tile against W held in
 * shared memory; the aggregate never goes to HBM.  Bit-identical to
 * aes_dev_spmm_f32 followed by aes_dev_gemm_bias_act_ex.  finite_w = 0 keeps
 * the reference's a == 0 skip (needed only when W has inf/NaN).  Rows of the
 * plan should be bounded (sampled plans): a hub row stalls one producer warp.
 * AES_ERR_UNSUPPORTED outside that range or when h overlaps x (callers run
 * the split kernels). */
AES_API int aes_dev_gcn_layer_fused(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                                    uint64_t n_rows, const float* x, uint64_t ldx, uint64_t k, const float* w,
                                    uint64_t ldw, uint64_t n, const float* bias, int relu, int finite_w, float* h,
                                    uint64_t ldh, void* stream);
/* The same layer with its exchange fused in (the p2p layer step of
 * gnn.cpp:66-78 run row-sharded): output row r goes to dsts[d] at row
 * row_offset + r for every destination d (peer replicas mapped through CUDA
 * IPC), or only where need[d][row_offset + r] != 0 when need (halo masks, per
 * destination, NULL entries = every row) is given; every CTA then adds one
 * release arrival (system scope) to each counters[d].  Arrivals per launch:
 * aes_gcn_layer_fused_ctas(n_rows).  n_dst <= 16. */
AES_API uint64_t aes_gcn_layer_fused_ctas(uint64_t n_rows);
AES_API int aes_dev_gcn_layer_fused_bcast(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                                          uint64_t n_rows, const float* x, uint64_t ldx, uint64_t k,
                                          const float* w, uint64_t ldw, uint64_t n, const float* bias, int relu,
                                          int finite_w, float* const* dsts, unsigned long long* const* counters,
                                          const uint8_t* const* need, int n_dst, uint64_t row_offset,
                                          uint64_t ldh, void* stream);
AES_API int aes_dev_gemm_bias_act_ex(const float* a, uint64_t m, uint64_t k, uint64_t lda,
                                     const float* w, uint64_t n, uint64_t ldw, const float* bias,
                                     int relu, int finite_w, float* const* dsts,
                                     unsigned long long* const* counters, int n_dst,
                                     uint64_t row_offset, uint64_t ldh, void* stream);
/* Same with halo masks (need: one per destination, NULL entries = every
 * row): output row r (replica index) is stored to destination d only if
 * need[d][r] != 0 — the rows d's sampled slots reference (SURVEY §8f rank 1:
 * a shard needs 93 / 74 / 49 % of the remote rows at P = 2 / 4 / 8).  The
 * arrival count per CTA is unchanged. */
AES_API int aes_dev_gemm_bias_act_halo(const float* a, uint64_t m, uint64_t k, uint64_t lda,
                                       const float* w, uint64_t n, uint64_t ldw, const float* bias,
                                       int relu, int finite_w, float* const* dsts,
                                       unsigned long long* const* counters, const uint8_t* const* need,
                                       int n_dst, uint64_t row_offset, uint64_t ldh, void* stream);
/* FAST MODE (opt-in, not bit-exact): the same layer GEMM on the tcgen05
 * tensor cores (kind::tf32, TMA-fed, TMEM accumulators).  Error bound
 * |H - H_exact| <= 2^-8 * sum_k |a_ik||w_kj| per element (TF32 operands, fp32
 * accumulation).  1 <= K <= 128, N <= 128, lda % 4 == 0, A 16-B aligned;
 * wt_scratch: device buffer of aes_gemm_tf32_scratch_floats(K, N) floats. */
AES_API int aes_dev_gemm_tf32(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w,
                              uint64_t n, uint64_t ldw, const float* bias, int relu, float* h,
                              uint64_t ldh, float* wt_scratch, void* stream);
AES_API uint64_t aes_gemm_tf32_scratch_floats(uint64_t k, uint64_t n);
/* Fast-mode GEMM fused with the layer exchange: the TMA-store epilogue writes
 * every 128-row tile to rows [row_offset, ...) of each replica dsts[0..n_dst)
 * (own + CUDA-IPC peer pointers, <= 8), then each CTA adds the number of
 * tiles it stored to every counters[d] (system-scope release).  A rank waits
 * for aes_gemm_tf32_ctas(m_p) summed over all producers p. */
AES_API int aes_dev_gemm_tf32_bcast(const float* a, uint64_t m, uint64_t k, uint64_t lda,
                                    const float* w, uint64_t n, uint64_t ldw, const float* bias,
                                    int relu, float* const* dsts, unsigned long long* const* counters,
                                    int n_dst, uint64_t row_offset, uint64_t ldh, float* wt_scratch,
                                    void* stream);
AES_API uint64_t aes_gemm_tf32_ctas(uint64_t m);
/* act(A W + b) into h (as aes_dev_gemm_bias_act_ex, one destination) with
 * fit_params (proj/src/quantize.cpp:11-21) of the output fused into the
 * epilogue: one (min, max) partial per CTA into fit_partials
 * (aes_gemm_fit_partial_bytes(m, n) bytes); aes_dev_fit_merge then writes
 * result[0..2] = (x_min, x_max, non-finite flag bits) exactly as
 * aes_dev_fit_params over the m x n output would. */
AES_API int aes_dev_gemm_bias_act_fit(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w,
                                      uint64_t n, uint64_t ldw, const float* bias, int relu, int finite_w, float* h,
                                      uint64_t ldh, void* fit_partials, void* stream);
AES_API uint64_t aes_gemm_fit_partial_bytes(uint64_t m, uint64_t n);
AES_API int aes_dev_fit_merge(const void* partials, uint64_t n_partials, float* result, void* stream);
/* Number of CTAs (= arrivals per destination) the GEMM above launches. */
AES_API uint64_t aes_gemm_ctas(uint64_t m, uint64_t n);
/* Spin (one thread, ld.acquire.sys) until *counter >= target. */
AES_API int aes_dev_wait_counter(const unsigned long long* counter, unsigned long long target,
                                 void* stream);
/* Device-side barrier arrival: system-scope fence, then +1 on every
 * counters[d] (host array of device pointers, e.g. all ranks' counters). */
AES_API int aes_dev_signal_all(unsigned long long* const* counters, int n, void* stream);
/* *bad_flag = 1 if any of x[0..count) is inf/NaN (stream-ordered). */
AES_API int aes_dev_all_finite(const float* x, uint64_t count, unsigned int* bad_flag, void* stream);

/* ---- int8 FAST MODE: per-row / per-feature affine scales (affine.cu) -----
 * Opt-in beside the reference's exact global min/max path (quantize.cpp:
 * 11-64); not bit-exact, bounded instead.  codes u8 [rows, ldq];
 * params float2 (scale s, offset m) per row (ROW) or per column (FEATURE);
 * x^ = q * s + m, q = clamp(rint((x - m) / s), 0, 255).
 * Bounds: |x^ - x| <= s/2 + 2^-22 (|m| + 255 s) per element, and
 * |C - A B| <= sum_k |v_k| (s_k/2 + 2^-22 (|m_k| + 255 s_k))
 *            + (slots + 2) 2^-23 sum_k |v_k| (|m_k| + 255 s_k)
 * for the fused SpMM.  Non-finite input sets *bad_flag (stream-ordered). */
#define AES_QAFFINE_ROW 0
#define AES_QAFFINE_FEATURE 1
AES_API uint64_t aes_quantize_affine_workspace_bytes(uint64_t rows, uint64_t cols, int mode);
AES_API int aes_dev_quantize_affine(const float* x, uint64_t rows, uint64_t cols, uint64_t ldx, int mode,
                                    uint8_t* q, uint64_t ldq, float* params, unsigned int* bad_flag,
                                    void* workspace, size_t workspace_bytes, void* stream);
AES_API int aes_dev_dequantize_affine(const uint8_t* q, uint64_t rows, uint64_t cols, uint64_t ldq, int mode,
                                      const float* params, float* x, uint64_t ldx, void* stream);
/* C[r, :] = sum_k v_k * x^[scol_k, :] over the (sampled) CSR, dequantizing
 * in the gather (no table).  ldq % 4 == 0, ldc % 4 == 0, C 16-B aligned. */
/* Handle tier: quantize host x [rows, cols] in the given mode into a
 * QuantizedFeatures handle; aes_spmm_sampled_q8 and aes_dequantize then use
 * the affine decode (codes are 8-bit; x_min/x_max of aes_qfeat_info are 0).
 * aes_qfeat_affine: the handle's mode (-1 = global exact) and its params
 * (float2 per row / column) to host memory (params may be NULL). */
AES_API int aes_quantize_affine(const float* x, uint64_t rows, uint64_t cols, int mode, aes_qfeat_t* out);
AES_API int aes_qfeat_affine(aes_qfeat_t q, int* mode, float* params);
AES_API int aes_dev_spmm_q8_affine(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                                   uint64_t n_rows, const uint8_t* q, uint64_t ldq, uint64_t f, int mode,
                                   const float* params, float* c, uint64_t ldc, void* stream);

/* ---- row-sharded GCN forward over NCCL (sharded.cu) ----------------------
 * gcn_forward (proj/src/gnn.cpp:66-78) on one rank of an equal-row sharded
 * graph: per layer the shard's sampled SpMM, the ordered-fp32 GEMM + bias
 * (+ ReLU but on the last layer) into a [rows_per_rank, round4(dims[l+1])]
 * block, and an ncclAllGather of the blocks (rank order) into the other
 * replica, which holds that layer's output with row stride round4(dims[l+1])
 * (the exchange moves N * round4(fout) * 4 bytes, not N * ld * 4).
 * srow_shard: the shard's shard_rows+1 row offsets into the GLOBAL sampled
 * CSR (scol, sval); replica_a holds the layer-0 input for every row
 * ([world * rows_per_rank, ld], ld % 4 == 0, dims[l] <= ld), replica_b is the
 * ping-pong partner; *out_replica receives the one holding the logits of all
 * rows and *out_ld (may be NULL) its row stride, round4(dims[n_layers]).
 * After every all-gather ncclCommGetAsyncError is checked.  weights / biases: host arrays of n_layers device pointers (biases
 * may be NULL or hold NULL entries).  nccl_comm: the caller's ncclComm_t
 * (NCCL is looked up at run time in the process).  Bit-identical to the
 * single-GPU forward.  Stream-ordered; no host synchronisation. */
AES_API uint64_t aes_gcn_sharded_workspace_bytes(uint64_t rows_per_rank, uint64_t ld);
AES_API int aes_gcn_forward_sharded(const uint64_t* srow_shard, const uint32_t* scol, const float* sval,
                                    uint64_t shard_rows, uint64_t rows_per_rank, int n_layers, const uint64_t* dims,
                                    const float* const* weights, const float* const* biases, int finite_w,
                                    float* replica_a, float* replica_b, uint64_t ld, uint64_t max_row_slots,
                                    void* workspace, size_t workspace_bytes, void* nccl_comm, float** out_replica,
                                    uint64_t* out_ld, void* stream);

/* ---- int8 layer exchange over peer memory (exchange.cu) ------------------
 * Replaces, per hidden GCN layer, the reference composition
 * dequantize(quantize(H, fit_params(H))) (proj/src/quantize.cpp:11-64) +
 * the all-gather of H, with no host round trip:
 *   aes_dev_fit_params(own rows) -> aes_dev_publish_params -> wait (world
 *   arrivals) -> aes_dev_fold_params_lut -> aes_dev_quantize_bcast -> wait
 *   (sum over ranks of aes_quantize_bcast_ctas(rows_r) arrivals) ->
 *   aes_dev_spmm_q8_ex over the code replica with the folded LUT.
 * Stores (min, max, flag) of this rank's fit_params result (or, when
 * empty != 0, the empty-shard marker) into slot `rank` of every rank's
 * float[4*world] parameter array, then +1 on every rank's counter. */
AES_API int aes_dev_publish_params(const float* fit_result, int empty, int rank, float* const* peer_params,
                                   unsigned long long* const* peer_counters, int world, void* stream);
/* Folds the world triples in rank order with the reference's strict < / >
 * rule into out[0..1] = (x_min, x_max), out[2] = status bits (0 ok,
 * 1 NonFinite, 2 EmptyMatrix), and writes the exact dequantization table of
 * those params to lut[256] (as aes_dev_dequant_lut). */
AES_API int aes_dev_fold_params_lut(const float* params, int world, uint32_t bits, float* out, float* lut,
                                    void* stream);
/* Arrivals (per destination) aes_dev_quantize_bcast adds for `rows` rows. */
AES_API uint64_t aes_quantize_bcast_ctas(uint64_t rows);
/* quantize(x, (lohi[0], lohi[1]), bits) of this shard's rows, codes stored
 * at rows row_off.. of every dst_codes[d] (ldq % 16 == 0), then one
 * system-scope release-add per CTA on every peer_counters[d].  need (NULL, or
 * one per destination, NULL entries = every row): halo masks, row r is sent
 * to d only if need[d][r] != 0 (the rows d's sampled slots reference). */
AES_API int aes_dev_quantize_bcast(const float* x, uint64_t rows, uint64_t cols, uint64_t ldx, const float* lohi,
                                   uint32_t bits, uint8_t* const* dst_codes, uint64_t row_off, uint64_t ldq,
                                   unsigned long long* const* peer_counters, const uint8_t* const* need,
                                   int world, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AESSPMM_CUDA_H */
