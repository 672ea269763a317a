// Handle tier of the C ABI (include/aesspmm_cuda.h): the entry points the
// reference's FFI binds (proj/bindings/module.cpp:52-144), backed by HBM-
// resident objects and the sm_100a kernels.  Host buffers in, host buffers out;
// every call is synchronous on the library stream, like the reference call it
// replaces.  No CPU fallback: every arithmetic step runs in a kernel.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace aes {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int status, const std::string& msg) {
    g_err = msg;
    return status;
}
int cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + where;
    return AES_ERR_CUDA;
}

// launchers defined in other translation units
int launch_sample_fill(const uint64_t*, const uint64_t*, const uint32_t*, const float*, uint64_t, uint32_t, int,
                       const uint64_t*, uint32_t*, float*, cudaStream_t);
int launch_plan_export(const uint64_t*, uint64_t, uint32_t, int, const uint64_t*, uint32_t*, uint32_t*,
                       uint32_t*, cudaStream_t);
int launch_sampling_rate(const uint64_t*, uint64_t, uint32_t, int, double*, unsigned long long*,
                         cudaStream_t);
int launch_row_stats(const uint64_t*, uint64_t, uint64_t*, unsigned long long*, cudaStream_t);
int launch_validate(const uint64_t*, const uint32_t*, uint64_t, uint64_t, unsigned long long*, cudaStream_t);
int launch_validate_rows(const uint64_t*, const uint32_t*, uint64_t, uint64_t, unsigned long long*,
                         cudaStream_t);
int launch_gcn_normalize(const uint64_t*, const uint32_t*, uint64_t, int, const uint64_t*, float*, uint32_t*,
                         float*, cudaStream_t);
int launch_row_mean(const uint64_t*, uint64_t, float*, cudaStream_t);
int launch_argmax(const float*, uint64_t, uint64_t, uint64_t, uint32_t*, cudaStream_t);
int launch_evaluate(const uint32_t*, const uint32_t*, const uint32_t*, const uint8_t*, uint64_t, uint64_t,
                    unsigned long long*, unsigned long long*, cudaStream_t);
int launch_explicit_fill(const uint64_t*, const uint32_t*, const uint64_t*, const uint32_t*, const uint32_t*,
                         const float*, uint64_t, const uint64_t*, uint32_t*, float*, cudaStream_t);
int launch_explicit_check(const uint64_t*, const uint32_t*, const uint64_t*, const uint32_t*, uint64_t,
                          unsigned long long*, cudaStream_t);
int launch_explicit_rate(const uint64_t*, const uint32_t*, const uint64_t*, const uint32_t*, uint64_t, uint64_t,
                         unsigned char*, double*, unsigned long long*, cudaStream_t);

namespace {

// ---------------------------------------------------------------------------
// library stream + stream-ordered device buffers
// ---------------------------------------------------------------------------
cudaStream_t lib_stream() {
    // one library stream per device (handles live on the device that was
    // current when they were created; calls run on that device's stream)
    static std::once_flag once[kMaxDevices];
    static cudaStream_t streams[kMaxDevices] = {};
    const int dev = cur_device();
    std::call_once(once[dev], [dev] {
        cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
        // keep freed stream-ordered blocks cached: per-call feature/result
        // buffers (GBs at the BASELINE shapes) are then recycled, not re-mapped
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            // and never hand a block still pending on another stream to a new
            // allocation: that inserts a cross-stream wait, which serialises
            // callers pipelining aes_spmm_sampled_async over several streams
            int no = 0;
            cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &no);
            cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
        }
    });
    return streams[dev];
}

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { reset(); }
    int alloc(size_t count) {
        reset();
        n = count;
        if (count == 0) return AES_OK;
        AES_CUDA_TRY(cudaMallocAsync((void**)&p, count * sizeof(T), lib_stream()));
        return AES_OK;
    }
    void reset() {
        if (p) cudaFreeAsync(p, lib_stream());
        p = nullptr;
        n = 0;
    }
    T* release() {
        T* r = p;
        p = nullptr;
        n = 0;
        return r;
    }
};

int sync() {
    AES_CUDA_TRY(cudaStreamSynchronize(lib_stream()));
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

uint64_t round4(uint64_t x) { return (x + 3) & ~3ull; }
// u8 code rows are padded to 16 B so the int8 SpMM can gather them with
// 16-B cp.async (spmm.cu, batch kernel)
uint64_t round16(uint64_t x) { return (x + 15) & ~15ull; }

// Upload a host row-major rows x cols f32 matrix into a device buffer with
// ld = round4(cols), pad columns zeroed (the vector kernels read them).
int upload_dense(const float* h, uint64_t rows, uint64_t cols, DBuf<float>& d, uint64_t& ld) {
    ld = round4(cols ? cols : 1);
    AES_TRY(d.alloc(rows * ld));
    if (rows == 0) return AES_OK;
    cudaStream_t st = lib_stream();
    if (ld != cols) AES_CUDA_TRY(cudaMemsetAsync(d.p, 0, rows * ld * sizeof(float), st));
    return h2d_dense(h, rows, cols, d.p, ld, st);  // (pageable sources through the staging ring)
}

int download_dense(const float* d, uint64_t ld, uint64_t rows, uint64_t cols, float* h) {
    return d2h_dense(d, ld, rows, cols, h, lib_stream());
}

template <typename T>
int d2h_scalar(const T* d, T* h) {
    AES_CUDA_TRY(cudaMemcpyAsync(h, d, sizeof(T), cudaMemcpyDeviceToHost, lib_stream()));
    return sync();
}

__global__ void widen_u8_kernel(const uint8_t* __restrict__ in, uint64_t rows, uint64_t cols, uint64_t ld,
                                uint16_t* __restrict__ out) {
    const uint64_t total = rows * cols;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = e / cols, c = e - r * cols;
        out[e] = in[r * ld + c];
    }
}

// narrow u16 codes to u8 (ld), flagging any code > 255
__global__ void narrow_u16_kernel(const uint16_t* __restrict__ in, uint64_t rows, uint64_t cols, uint64_t ld,
                                  uint8_t* __restrict__ out, unsigned int* __restrict__ overflow) {
    const uint64_t total = rows * cols;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = e / cols, c = e - r * cols;
        uint16_t v = in[e];
        if (v > 255) atomicOr(overflow, 1u);
        out[r * ld + c] = (uint8_t)v;
    }
}

}  // namespace
}  // namespace aes

// ===========================================================================
// handle objects
// ===========================================================================
struct aes_csr_s {
    uint64_t n_rows = 0, n_cols = 0, nnz = 0;
    uint64_t* row_ptr = nullptr;
    uint32_t* col = nullptr;
    float* val = nullptr;
    bool owned = true;
    std::atomic<int> refs{1};
};

struct aes_plan_s {
    uint32_t width = 0;
    int strategy = 0;
    uint64_t n_rows = 0, total_slots = 0;
    aes_csr_s* src = nullptr;  // holds a reference
    uint64_t* srow_ptr = nullptr;
    uint32_t* scol = nullptr;
    float* sval = nullptr;
    // host-supplied plans (aes_plan_from_host): per-row (chunk, cnt) and starts
    bool explicit_plan = false;
    uint32_t* params = nullptr;       // uint2 per row
    uint64_t* starts_ptr = nullptr;   // n+1
    uint32_t* starts = nullptr;
    uint64_t total_starts = 0;
    // caller streams that aes_spmm_sampled_async enqueued reads of this plan
    // on, each with an event recorded after its last use: destroy makes the
    // library stream wait on them before freeing (stream-ordered lifetime)
    std::mutex use_mu;
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
    void note_use(cudaStream_t st) {
        std::lock_guard<std::mutex> lock(use_mu);
        for (auto& u : uses)
            if (u.first == st) {
                cudaEventRecord(u.second, st);
                return;
            }
        cudaEvent_t e;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            cudaStreamSynchronize(st);  // no event: make the use complete now
            return;
        }
        cudaEventRecord(e, st);
        uses.emplace_back(st, e);
    }
    void order_after_uses(cudaStream_t lib) {
        std::lock_guard<std::mutex> lock(use_mu);
        for (auto& u : uses) {
            cudaStreamWaitEvent(lib, u.second, 0);
            cudaEventDestroy(u.second);
        }
        uses.clear();
    }
};

struct aes_qfeat_s {
    uint64_t rows = 0, cols = 0, ld = 0;  // ld in codes
    float x_min = 0.f, x_max = 0.f;
    uint32_t bits = 8;
    bool u8 = true;       // codes stored as u8 (bits <= 8 and all codes <= 255)
    void* codes = nullptr;
    float* lut = nullptr;  // 256 floats when u8
    // fast mode (affine.cu): AES_QAFFINE_ROW / _FEATURE, -1 = the reference's
    // global min/max codes; params: float2 (scale, offset) per row / column
    int affine = -1;
    float* aparams = nullptr;
};

namespace {
using namespace aes;

void csr_release(aes_csr_s* a) {
    if (a && a->refs.fetch_sub(1) == 1) {
        if (a->owned) {
            cudaStream_t st = lib_stream();
            if (a->row_ptr) cudaFreeAsync(a->row_ptr, st);
            if (a->col) cudaFreeAsync(a->col, st);
            if (a->val) cudaFreeAsync(a->val, st);
        }
        delete a;
    }
}

const char* csr_error_name(int e) {
    switch (e) {
        case AES_CSR_NON_MONOTONIC: return "NonMonotonicRowPtr";
        case AES_CSR_COL_OUT_OF_RANGE: return "ColumnOutOfRange";
        case AES_CSR_UNSORTED: return "UnsortedRow";
        case AES_CSR_LENGTH_MISMATCH: return "LengthMismatch";
        case AES_CSR_NOT_SQUARE: return "NotSquare";
        default: return "ok";
    }
}

// validate_csr (matrix.cpp:28-52) with the reference's check order.
// validate_csr (matrix.cpp:28-52) with the reference's check order; the
// first violation is reported as (CsrError, row) and as the message text.
int validate_device(const aes_csr_s* a, uint64_t row_ptr_len, uint64_t nnz_len, uint64_t first_row_ptr,
                    int* err_out = nullptr, uint64_t* row_out = nullptr) {
    auto bad = [&](int e, uint64_t row, bool with_row) {
        if (err_out) *err_out = e;
        if (row_out) *row_out = row;
        std::string msg = csr_error_name(e);
        if (with_row) msg += " at row " + std::to_string(row);
        return fail(AES_ERR_CSR_INVALID, msg);
    };
    if (err_out) *err_out = AES_CSR_OK;
    if (row_out) *row_out = 0;
    if (row_ptr_len != a->n_rows + 1 || row_ptr_len == 0 || first_row_ptr != 0)
        return bad(AES_CSR_LENGTH_MISMATCH, 0, false);
    DBuf<unsigned long long> scratch;
    AES_TRY(scratch.alloc(2));
    cudaStream_t st = lib_stream();
    AES_TRY(launch_validate(a->row_ptr, a->col, a->n_rows, a->n_cols, scratch.p, st));
    unsigned long long first_bad = 0;
    AES_TRY(d2h_scalar(scratch.p, &first_bad));
    if (first_bad != ~0ull) return bad(AES_CSR_NON_MONOTONIC, first_bad, true);
    uint64_t back = 0;
    AES_TRY(d2h_scalar(a->row_ptr + a->n_rows, &back));
    if (back != nnz_len) return bad(AES_CSR_LENGTH_MISMATCH, 0, false);
    AES_TRY(launch_validate_rows(a->row_ptr, a->col, a->n_rows, a->n_cols, scratch.p + 1, st));
    unsigned long long code = 0;
    AES_TRY(d2h_scalar(scratch.p + 1, &code));
    if (code != ~0ull) return bad((int)(code & 3), code >> 2, true);
    return AES_OK;
}

// Most slots any row of a plan's sampled CSR can have (0 = unbounded: no
// plan (exact), FULL plans, host-supplied plans) — picks the ring schedule.
uint64_t plan_row_bound(const aes_plan_s* p) {
    if (!p || p->explicit_plan || p->strategy == AES_FULL) return 0;
    return p->width;
}

// spmm over a device CSR (original or sampled) with host dense operands.
int spmm_host(const uint64_t* rp, const uint32_t* col, const float* val, uint64_t n_rows, const float* b,
              uint64_t b_rows, uint64_t f, float* c, uint64_t row_bound) {
    if (n_rows == 0 || f == 0) return AES_OK;
    DBuf<float> db, dc;
    uint64_t ldb = 0;
    AES_TRY(upload_dense(b, b_rows, f, db, ldb));
    const uint64_t ldc = ldb;
    AES_TRY(dc.alloc(n_rows * ldc));
    AES_TRY(aes_dev_spmm_f32_ex(rp, col, val, n_rows, db.p, ldb, f, dc.p, ldc, row_bound, lib_stream()));
    AES_TRY(download_dense(dc.p, ldc, n_rows, f, c));
    return sync();
}

// Sampled CSR for (plan, matrix): the plan's own arrays when `a` is the
// matrix it was built on; otherwise re-filled from `a` with the plan's windows
// (spmm.cpp:44-76 fills per call from whatever matrix it is given).
int sampled_for(aes_plan_t p, aes_csr_t a, DBuf<uint32_t>& tcol, DBuf<float>& tval, const uint32_t** scol,
                const float** sval) {
    if (a == p->src) {
        *scol = p->scol;
        *sval = p->sval;
        return AES_OK;
    }
    AES_TRY(tcol.alloc(p->total_slots));
    AES_TRY(tval.alloc(p->total_slots));
    if (p->explicit_plan)
        AES_TRY(launch_explicit_fill(a->row_ptr, p->params, p->starts_ptr, p->starts, a->col, a->val, a->n_rows,
                                     p->srow_ptr, tcol.p, tval.p, lib_stream()));
    else
        AES_TRY(launch_sample_fill(p->src->row_ptr, a->row_ptr, a->col, a->val, a->n_rows, p->width, p->strategy,
                                   p->srow_ptr, tcol.p, tval.p, lib_stream()));
    *scol = tcol.p;
    *sval = tval.p;
    return AES_OK;
}

}  // namespace

// ===========================================================================
// C ABI — handle tier
// ===========================================================================
extern "C" {

const char* aes_last_error(void) { return aes::g_err.c_str(); }

const char* aes_status_name(int s) {
    switch (s) {
        case AES_OK: return "OK";
        case AES_ERR_ZERO_WIDTH: return "ZeroWidth";
        case AES_ERR_SHAPE: return "ShapeMismatch";
        case AES_ERR_PLAN_MISMATCH: return "PlanMatrixMismatch";
        case AES_ERR_EMPTY: return "EmptyMatrix";
        case AES_ERR_NONFINITE: return "NonFinite";
        case AES_ERR_QPARAMS: return "invalid QuantParams";
        case AES_ERR_BITS: return "bits must be 1..16";
        case AES_ERR_CSR_INVALID: return "InvalidCsr";
        case AES_ERR_INVALID_ARG: return "InvalidArgument";
        case AES_ERR_CUDA: return "CudaError";
        case AES_ERR_UNSUPPORTED: return "Unsupported";
        case AES_ERR_NOT_SQUARE: return "NotSquare";
        case AES_ERR_IO: return "IoError";
        default: return "Unknown";
    }
}

int aes_version(void) { return 1; }

int aes_select_strategy(uint64_t row_nnz, uint32_t width, uint32_t* chunk_len, uint32_t* sample_cnt) {
    if (width == 0) return fail(AES_ERR_ZERO_WIDTH, "ZeroWidth");
    aes::RowParams p = aes::select_strategy(row_nnz, width);
    *chunk_len = p.chunk;
    *sample_cnt = p.cnt;
    return AES_OK;
}

uint32_t aes_hash_start(uint32_t current_ind, uint64_t row_nnz, uint32_t chunk_len) {
    return aes::hash_start(current_ind, row_nnz, chunk_len);
}

// ---- CSR ------------------------------------------------------------------
int aes_csr_create(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr, uint64_t row_ptr_len,
                   const uint32_t* col_ind, const float* val, uint64_t nnz_len, aes_csr_t* out) {
    if (!out) return fail(AES_ERR_INVALID_ARG, "null out");
    *out = nullptr;
    // The reference's ctor checks sizes before anything else.
    if (row_ptr_len != n_rows + 1 || row_ptr_len == 0) return fail(AES_ERR_CSR_INVALID, "LengthMismatch");
    if (row_ptr[0] != 0) return fail(AES_ERR_CSR_INVALID, "LengthMismatch");
    auto* a = new aes_csr_s;
    a->n_rows = n_rows;
    a->n_cols = n_cols;
    a->nnz = nnz_len;
    cudaStream_t st = lib_stream();
    DBuf<uint64_t> rp;
    DBuf<uint32_t> ci;
    DBuf<float> vv;
    int s = rp.alloc(n_rows + 1);
    if (!s) s = ci.alloc(nnz_len ? nnz_len : 1);
    if (!s) s = vv.alloc(nnz_len ? nnz_len : 1);
    if (!s && cudaMemcpyAsync(rp.p, row_ptr, (n_rows + 1) * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
        s = fail(AES_ERR_CUDA, "row_ptr upload failed");
    if (!s && nnz_len) {
        if (cudaMemcpyAsync(ci.p, col_ind, nnz_len * 4, cudaMemcpyHostToDevice, st) != cudaSuccess ||
            cudaMemcpyAsync(vv.p, val, nnz_len * 4, cudaMemcpyHostToDevice, st) != cudaSuccess)
            s = fail(AES_ERR_CUDA, "csr upload failed");
    }
    a->row_ptr = rp.p;
    a->col = ci.p;
    a->val = vv.p;
    if (!s) s = validate_device(a, row_ptr_len, nnz_len, row_ptr[0]);
    if (s) {
        a->row_ptr = nullptr; a->col = nullptr; a->val = nullptr;
        delete a;
        sync();
        return s;
    }
    rp.release();
    ci.release();
    vv.release();
    *out = a;
    return AES_OK;
}

int aes_csr_wrap_device(uint64_t n_rows, uint64_t n_cols, const uint64_t* d_row_ptr, const uint32_t* d_col_ind,
                        const float* d_val, uint64_t nnz, aes_csr_t* out) {
    if (!out || !d_row_ptr) return fail(AES_ERR_INVALID_ARG, "null argument");
    auto* a = new aes_csr_s;
    a->n_rows = n_rows;
    a->n_cols = n_cols;
    a->nnz = nnz;
    a->row_ptr = const_cast<uint64_t*>(d_row_ptr);
    a->col = const_cast<uint32_t*>(d_col_ind);
    a->val = const_cast<float*>(d_val);
    a->owned = false;
    *out = a;
    return AES_OK;
}

int aes_csr_destroy(aes_csr_t a) {
    csr_release(a);
    return AES_OK;
}

int aes_csr_shape(aes_csr_t a, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz) {
    if (!a) return fail(AES_ERR_INVALID_ARG, "null csr");
    if (n_rows) *n_rows = a->n_rows;
    if (n_cols) *n_cols = a->n_cols;
    if (nnz) *nnz = a->nnz;
    return AES_OK;
}

int aes_csr_device_ptrs(aes_csr_t a, const uint64_t** row_ptr, const uint32_t** col_ind, const float** val) {
    if (!a) return fail(AES_ERR_INVALID_ARG, "null csr");
    AES_TRY(sync());  // creation is stream-ordered on the library stream
    if (row_ptr) *row_ptr = a->row_ptr;
    if (col_ind) *col_ind = a->col;
    if (val) *val = a->val;
    return AES_OK;
}

int aes_csr_download(aes_csr_t a, uint64_t* row_ptr, uint32_t* col_ind, float* val) {
    if (!a) return fail(AES_ERR_INVALID_ARG, "null csr");
    cudaStream_t st = lib_stream();
    if (row_ptr) AES_CUDA_TRY(cudaMemcpyAsync(row_ptr, a->row_ptr, (a->n_rows + 1) * 8, cudaMemcpyDeviceToHost, st));
    if (a->nnz) {
        if (col_ind) AES_CUDA_TRY(cudaMemcpyAsync(col_ind, a->col, a->nnz * 4, cudaMemcpyDeviceToHost, st));
        if (val) AES_CUDA_TRY(cudaMemcpyAsync(val, a->val, a->nnz * 4, cudaMemcpyDeviceToHost, st));
    }
    return sync();
}

int aes_csr_row_stats(aes_csr_t a, uint64_t* row_nnz, uint64_t* max_row_nnz, double* avg_degree) {
    if (!a) return fail(AES_ERR_INVALID_ARG, "null csr");
    DBuf<uint64_t> rn;
    DBuf<unsigned long long> mx;
    AES_TRY(mx.alloc(1));
    if (row_nnz) AES_TRY(rn.alloc(a->n_rows));
    AES_TRY(launch_row_stats(a->row_ptr, a->n_rows, rn.p, mx.p, lib_stream()));
    if (row_nnz && a->n_rows)
        AES_CUDA_TRY(cudaMemcpyAsync(row_nnz, rn.p, a->n_rows * 8, cudaMemcpyDeviceToHost, lib_stream()));
    unsigned long long m = 0;
    AES_TRY(d2h_scalar(mx.p, &m));
    if (max_row_nnz) *max_row_nnz = m;
    if (avg_degree) *avg_degree = a->n_rows == 0 ? 0.0 : double(a->nnz) / double(a->n_rows);
    return AES_OK;
}

int aes_gcn_normalize(aes_csr_t a, int add_self_loops, aes_csr_t* out) {
    if (!a || !out) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (a->n_rows != a->n_cols) return fail(AES_ERR_NOT_SQUARE, "NotSquare");
    cudaStream_t st = lib_stream();
    const uint64_t n = a->n_rows;
    DBuf<uint64_t> optr;
    DBuf<char> ws;
    AES_TRY(optr.alloc(n + 1));
    size_t wsb = row_scan_workspace_bytes(n);
    AES_TRY(ws.alloc(wsb));
    ScanArgs sa{a->row_ptr, a->col, n, 1, 0, add_self_loops, optr.p, nullptr};
    AES_TRY(launch_row_scan(kScanGcnNnz, sa, ws.p, wsb, st));
    uint64_t nnz = 0;
    AES_TRY(d2h_scalar(optr.p + n, &nnz));
    DBuf<uint32_t> ocol;
    DBuf<float> oval, inv;
    AES_TRY(ocol.alloc(nnz ? nnz : 1));
    AES_TRY(oval.alloc(nnz ? nnz : 1));
    AES_TRY(inv.alloc(n ? n : 1));
    AES_TRY(launch_gcn_normalize(a->row_ptr, a->col, n, add_self_loops, optr.p, inv.p, ocol.p, oval.p, st));
    AES_TRY(sync());
    auto* o = new aes_csr_s;
    o->n_rows = n;
    o->n_cols = a->n_cols;
    o->nnz = nnz;
    o->row_ptr = optr.release();
    o->col = ocol.release();
    o->val = oval.release();
    *out = o;
    return AES_OK;
}

int aes_validate_csr(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr, uint64_t row_ptr_len,
                     const uint32_t* col_ind, uint64_t nnz_len, int* error, uint64_t* row) {
    if (error) *error = AES_CSR_OK;
    if (row) *row = 0;
    if (row_ptr_len != n_rows + 1 || row_ptr_len == 0 || row_ptr[0] != 0) {
        if (error) *error = AES_CSR_LENGTH_MISMATCH;
        return fail(AES_ERR_CSR_INVALID, "LengthMismatch");
    }
    aes_csr_s tmp;
    tmp.n_rows = n_rows;
    tmp.n_cols = n_cols;
    tmp.owned = false;
    DBuf<uint64_t> rp;
    DBuf<uint32_t> ci;
    AES_TRY(rp.alloc(n_rows + 1));
    AES_TRY(ci.alloc(nnz_len ? nnz_len : 1));
    cudaStream_t st = lib_stream();
    AES_CUDA_TRY(cudaMemcpyAsync(rp.p, row_ptr, (n_rows + 1) * 8, cudaMemcpyHostToDevice, st));
    if (nnz_len) AES_CUDA_TRY(cudaMemcpyAsync(ci.p, col_ind, nnz_len * 4, cudaMemcpyHostToDevice, st));
    tmp.row_ptr = rp.p;
    tmp.col = ci.p;
    int s = validate_device(&tmp, row_ptr_len, nnz_len, row_ptr[0], error, row);
    tmp.row_ptr = nullptr;
    tmp.col = nullptr;
    return s;
}

int aes_csr_structure(uint64_t n_rows, uint64_t n_cols, const uint64_t* row_ptr, aes_csr_t* out) {
    if (!out || !row_ptr) return fail(AES_ERR_INVALID_ARG, "null argument");
    DBuf<uint64_t> rp;
    AES_TRY(rp.alloc(n_rows + 1));
    AES_CUDA_TRY(cudaMemcpyAsync(rp.p, row_ptr, (n_rows + 1) * 8, cudaMemcpyHostToDevice, lib_stream()));
    AES_TRY(sync());
    auto* a = new aes_csr_s;
    a->n_rows = n_rows;
    a->n_cols = n_cols;
    a->nnz = row_ptr[n_rows];
    a->row_ptr = rp.release();
    *out = a;
    return AES_OK;
}

int aes_fit_params(const float* x, uint64_t rows, uint64_t cols, uint32_t bits, float* x_min, float* x_max) {
    const uint64_t n = rows * cols;
    if (n == 0) return fail(AES_ERR_EMPTY, "EmptyMatrix");
    if (bits < 1 || bits > 16) return fail(AES_ERR_BITS, "bits must be 1..16");
    cudaStream_t st = lib_stream();
    DBuf<float> dx, res;
    DBuf<char> ws;
    AES_TRY(dx.alloc(n));
    AES_CUDA_TRY(cudaMemcpyAsync(dx.p, x, n * 4, cudaMemcpyHostToDevice, st));
    const size_t wsb = aes_dev_scan_workspace_bytes(1);
    AES_TRY(ws.alloc(wsb));
    AES_TRY(res.alloc(4));
    AES_TRY(aes_dev_fit_params(dx.p, n, res.p, ws.p, wsb, st));
    float r[4];
    AES_CUDA_TRY(cudaMemcpyAsync(r, res.p, sizeof(r), cudaMemcpyDeviceToHost, st));
    AES_TRY(sync());
    uint32_t flag;
    memcpy(&flag, &r[2], 4);
    if (flag) return fail(AES_ERR_NONFINITE, "NonFinite");
    *x_min = r[0];
    *x_max = r[1];
    return AES_OK;
}

// ---- plans -------------------------------------------------------------------
int aes_build_plan_set(aes_csr_t a, uint32_t width, int strategy, aes_plan_t* out) {
    if (!a || !out) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (width == 0) return fail(AES_ERR_ZERO_WIDTH, "ZeroWidth");
    if (strategy < 0 || strategy > 3) return fail(AES_ERR_INVALID_ARG, "unknown strategy");
    cudaStream_t st = lib_stream();
    const uint64_t n = a->n_rows;
    DBuf<uint64_t> srow;
    DBuf<char> ws;
    AES_TRY(srow.alloc(n + 1));
    size_t wsb = aes_dev_scan_workspace_bytes(n);
    AES_TRY(ws.alloc(wsb));
    AES_TRY(aes_dev_sample_plan(a->row_ptr, n, width, strategy, srow.p, nullptr, ws.p, wsb, st));
    uint64_t total = 0;
    AES_TRY(d2h_scalar(srow.p + n, &total));
    DBuf<uint32_t> scol;
    DBuf<float> sval;
    AES_TRY(scol.alloc(total ? total : 1));
    AES_TRY(sval.alloc(total ? total : 1));
    if (a->col)  // structure-only CSRs get the plan (row pointer) without a sampled CSR
        AES_TRY(aes_dev_sample_fill(a->row_ptr, a->row_ptr, a->col, a->val, n, width, strategy, srow.p, scol.p,
                                    sval.p, st));
    AES_TRY(sync());
    auto* p = new aes_plan_s;
    p->width = width;
    p->strategy = strategy;
    p->n_rows = n;
    p->total_slots = total;
    a->refs.fetch_add(1);
    p->src = a;
    p->srow_ptr = srow.release();
    p->scol = scol.release();
    p->sval = sval.release();
    *out = p;
    return AES_OK;
}

int aes_plan_from_host(aes_csr_t a, uint32_t width, int strategy, const uint32_t* chunk_len,
                       const uint32_t* sample_cnt, const uint64_t* starts_ptr, const uint32_t* starts,
                       aes_plan_t* out) {
    if (!a || !out || (a->n_rows && (!chunk_len || !sample_cnt || !starts_ptr)))
        return fail(AES_ERR_INVALID_ARG, "null argument");
    cudaStream_t st = lib_stream();
    const uint64_t n = a->n_rows;
    const uint64_t tot_starts = starts_ptr ? starts_ptr[n] : 0;
    if (n && starts_ptr[0] != 0) return fail(AES_ERR_INVALID_ARG, "invalid plan: starts offsets must begin at 0");
    if (tot_starts && !starts) return fail(AES_ERR_INVALID_ARG, "null argument");
    // interleave (chunk, cnt) on the host side of the copy: plain data marshaling;
    // each row must carry at least sample_cnt window starts
    std::vector<uint32_t> params(2 * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) {
        params[2 * i] = chunk_len[i];
        params[2 * i + 1] = sample_cnt[i];
        if (starts_ptr[i + 1] < starts_ptr[i] || starts_ptr[i + 1] - starts_ptr[i] < sample_cnt[i])
            return fail(AES_ERR_INVALID_ARG, "invalid plan: fewer starts than sample_cnt at row " + std::to_string(i));
    }
    DBuf<uint32_t> dpar, dst;
    DBuf<uint64_t> dsp, srow;
    DBuf<char> ws;
    AES_TRY(dpar.alloc(params.size()));
    AES_TRY(dsp.alloc(n + 1));
    AES_TRY(dst.alloc(tot_starts ? tot_starts : 1));
    AES_CUDA_TRY(cudaMemcpyAsync(dpar.p, params.data(), params.size() * 4, cudaMemcpyHostToDevice, st));
    if (starts_ptr) AES_CUDA_TRY(cudaMemcpyAsync(dsp.p, starts_ptr, (n + 1) * 8, cudaMemcpyHostToDevice, st));
    if (tot_starts) AES_CUDA_TRY(cudaMemcpyAsync(dst.p, starts, tot_starts * 4, cudaMemcpyHostToDevice, st));
    AES_TRY(srow.alloc(n + 1));
    size_t wsb = row_scan_workspace_bytes(n);
    AES_TRY(ws.alloc(wsb));
    {  // every window inside its row (the fill / mark kernels read through them)
        DBuf<unsigned long long> bad;
        AES_TRY(bad.alloc(1));
        AES_TRY(launch_explicit_check(a->row_ptr, dpar.p, dsp.p, dst.p, n, bad.p, st));
        unsigned long long bad_row = 0;
        AES_TRY(d2h_scalar(bad.p, &bad_row));
        if (bad_row != ~0ull)
            return fail(AES_ERR_INVALID_ARG,
                        "invalid plan: sample window past the end of row " + std::to_string(bad_row));
    }
    ScanArgs sa{nullptr, nullptr, n, width, strategy, 0, srow.p, dpar.p};
    AES_TRY(launch_row_scan(kScanExplicit, sa, ws.p, wsb, st));
    uint64_t total = 0;
    AES_TRY(d2h_scalar(srow.p + n, &total));
    DBuf<uint32_t> scol;
    DBuf<float> sval;
    AES_TRY(scol.alloc(total ? total : 1));
    AES_TRY(sval.alloc(total ? total : 1));
    if (a->col)  // structure-only CSRs (aes_csr_structure) carry plans for rates only
        AES_TRY(launch_explicit_fill(a->row_ptr, dpar.p, dsp.p, dst.p, a->col, a->val, n, srow.p, scol.p, sval.p,
                                     st));
    AES_TRY(sync());
    auto* p = new aes_plan_s;
    p->width = width;
    p->strategy = strategy;
    p->n_rows = n;
    p->total_slots = total;
    a->refs.fetch_add(1);
    p->src = a;
    p->srow_ptr = srow.release();
    p->scol = scol.release();
    p->sval = sval.release();
    p->explicit_plan = true;
    p->params = dpar.release();
    p->starts_ptr = dsp.release();
    p->starts = dst.release();
    p->total_starts = tot_starts;
    *out = p;
    return AES_OK;
}

int aes_plan_destroy(aes_plan_t p) {
    if (!p) return AES_OK;
    cudaStream_t st = lib_stream();
    p->order_after_uses(st);  // frees below run after every async SpMM that read the plan
    cudaFreeAsync(p->srow_ptr, st);
    cudaFreeAsync(p->scol, st);
    cudaFreeAsync(p->sval, st);
    if (p->params) cudaFreeAsync(p->params, st);
    if (p->starts_ptr) cudaFreeAsync(p->starts_ptr, st);
    if (p->starts) cudaFreeAsync(p->starts, st);
    csr_release(p->src);
    delete p;
    return AES_OK;
}

int aes_plan_info(aes_plan_t p, uint32_t* width, int* strategy, uint64_t* n_rows, uint64_t* total_slots,
                  uint64_t* total_starts) {
    if (!p) return fail(AES_ERR_INVALID_ARG, "null plan");
    if (width) *width = p->width;
    if (strategy) *strategy = p->strategy;
    if (n_rows) *n_rows = p->n_rows;
    if (total_slots) *total_slots = p->total_slots;
    if (total_starts && p->explicit_plan) {
        *total_starts = p->total_starts;
    } else if (total_starts) {
        const uint64_t n = p->n_rows;
        DBuf<uint64_t> sp;
        DBuf<char> ws;
        AES_TRY(sp.alloc(n + 1));
        size_t wsb = row_scan_workspace_bytes(n);
        AES_TRY(ws.alloc(wsb));
        ScanArgs sa{p->src->row_ptr, nullptr, n, p->width, p->strategy, 0, sp.p, nullptr};
        AES_TRY(launch_row_scan(kScanStarts, sa, ws.p, wsb, lib_stream()));
        AES_TRY(d2h_scalar(sp.p + n, total_starts));
    }
    return AES_OK;
}

int aes_plan_export(aes_plan_t p, uint32_t* chunk_len, uint32_t* sample_cnt, uint64_t* starts_ptr,
                    uint32_t* starts) {
    if (!p) return fail(AES_ERR_INVALID_ARG, "null plan");
    cudaStream_t st = lib_stream();
    const uint64_t n = p->n_rows;
    if (p->explicit_plan) {  // stored as given
        if (n) {
            DBuf<uint32_t> ch, cn;
            AES_TRY(ch.alloc(n));
            AES_TRY(cn.alloc(n));
            AES_CUDA_TRY(cudaMemcpy2DAsync(ch.p, 4, p->params, 8, 4, n, cudaMemcpyDeviceToDevice, st));
            AES_CUDA_TRY(cudaMemcpy2DAsync(cn.p, 4, p->params + 1, 8, 4, n, cudaMemcpyDeviceToDevice, st));
            if (chunk_len) AES_CUDA_TRY(cudaMemcpyAsync(chunk_len, ch.p, n * 4, cudaMemcpyDeviceToHost, st));
            if (sample_cnt) AES_CUDA_TRY(cudaMemcpyAsync(sample_cnt, cn.p, n * 4, cudaMemcpyDeviceToHost, st));
            AES_TRY(sync());
        }
        if (starts_ptr) AES_CUDA_TRY(cudaMemcpyAsync(starts_ptr, p->starts_ptr, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
        if (starts && p->total_starts)
            AES_CUDA_TRY(cudaMemcpyAsync(starts, p->starts, p->total_starts * 4, cudaMemcpyDeviceToHost, st));
        return sync();
    }
    DBuf<uint64_t> sp;
    DBuf<char> ws;
    AES_TRY(sp.alloc(n + 1));
    size_t wsb = row_scan_workspace_bytes(n);
    AES_TRY(ws.alloc(wsb));
    ScanArgs sa{p->src->row_ptr, nullptr, n, p->width, p->strategy, 0, sp.p, nullptr};
    AES_TRY(launch_row_scan(kScanStarts, sa, ws.p, wsb, st));
    uint64_t tot = 0;
    AES_TRY(d2h_scalar(sp.p + n, &tot));
    DBuf<uint32_t> dch, dcn, dst;
    AES_TRY(dch.alloc(n ? n : 1));
    AES_TRY(dcn.alloc(n ? n : 1));
    AES_TRY(dst.alloc(tot ? tot : 1));
    AES_TRY(launch_plan_export(p->src->row_ptr, n, p->width, p->strategy, sp.p, dch.p, dcn.p, dst.p, st));
    if (n) {
        if (chunk_len) AES_CUDA_TRY(cudaMemcpyAsync(chunk_len, dch.p, n * 4, cudaMemcpyDeviceToHost, st));
        if (sample_cnt) AES_CUDA_TRY(cudaMemcpyAsync(sample_cnt, dcn.p, n * 4, cudaMemcpyDeviceToHost, st));
    }
    if (starts_ptr) AES_CUDA_TRY(cudaMemcpyAsync(starts_ptr, sp.p, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
    if (starts && tot) AES_CUDA_TRY(cudaMemcpyAsync(starts, dst.p, tot * 4, cudaMemcpyDeviceToHost, st));
    return sync();
}

int aes_plan_device_ptrs(aes_plan_t p, const uint64_t** srow_ptr, const uint32_t** scol, const float** sval) {
    if (!p) return fail(AES_ERR_INVALID_ARG, "null plan");
    if (srow_ptr) *srow_ptr = p->srow_ptr;
    if (scol) *scol = p->scol;
    if (sval) *sval = p->sval;
    return AES_OK;
}

int aes_plan_download(aes_plan_t p, uint64_t* srow_ptr, uint32_t* scol, float* sval) {
    if (!p) return fail(AES_ERR_INVALID_ARG, "null plan");
    cudaStream_t st = lib_stream();
    if (srow_ptr)
        AES_CUDA_TRY(cudaMemcpyAsync(srow_ptr, p->srow_ptr, (p->n_rows + 1) * 8, cudaMemcpyDeviceToHost, st));
    if (p->total_slots) {
        if (scol) AES_CUDA_TRY(cudaMemcpyAsync(scol, p->scol, p->total_slots * 4, cudaMemcpyDeviceToHost, st));
        if (sval) AES_CUDA_TRY(cudaMemcpyAsync(sval, p->sval, p->total_slots * 4, cudaMemcpyDeviceToHost, st));
    }
    return sync();
}

int aes_sampling_rate(aes_plan_t p, aes_csr_t a, double* aggregate, double* unique_coverage, double* per_row) {
    if (!p || !a) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (p->n_rows != a->n_rows) return fail(AES_ERR_INVALID_ARG, "plan/stats row count mismatch");
    cudaStream_t st = lib_stream();
    DBuf<unsigned long long> tot;
    DBuf<double> pr;
    AES_TRY(tot.alloc(3));
    if (per_row) AES_TRY(pr.alloc(a->n_rows ? a->n_rows : 1));
    DBuf<unsigned char> seen;
    if (p->explicit_plan) {
        AES_TRY(seen.alloc(a->nnz ? a->nnz : 1));
        AES_TRY(launch_explicit_rate(a->row_ptr, p->params, p->starts_ptr, p->starts, a->n_rows, a->nnz, seen.p,
                                     pr.p, tot.p, st));
    } else {
        AES_TRY(launch_sampling_rate(a->row_ptr, a->n_rows, p->width, p->strategy, pr.p, tot.p, st));
    }
    unsigned long long t[3];
    AES_CUDA_TRY(cudaMemcpyAsync(t, tot.p, sizeof(t), cudaMemcpyDeviceToHost, st));
    if (per_row && a->n_rows)
        AES_CUDA_TRY(cudaMemcpyAsync(per_row, pr.p, a->n_rows * 8, cudaMemcpyDeviceToHost, st));
    AES_TRY(sync());
    if (aggregate) *aggregate = t[2] == 0 ? 1.0 : double(t[0]) / double(t[2]);
    if (unique_coverage) *unique_coverage = t[2] == 0 ? 1.0 : double(t[1]) / double(t[2]);
    return AES_OK;
}

// cdf_stats (bench.cpp:124-138) over host rates, and over a plan's per-row
// rates straight from the device (no per-row read-back).  Outputs hold at
// most n steps; *n_steps receives the count.
static int cdf_device(const double* d_rates, uint64_t n, double* out_rate, double* out_frac, uint64_t* n_steps) {
    cudaStream_t st = lib_stream();
    DBuf<char> ws;
    DBuf<double> dr, df;
    DBuf<uint64_t> dn;
    const size_t wsb = aes_cdf_workspace_bytes(n);
    AES_TRY(ws.alloc(wsb));
    AES_TRY(dr.alloc(n));
    AES_TRY(df.alloc(n));
    AES_TRY(dn.alloc(1));
    AES_TRY(aes_dev_cdf_stats(d_rates, n, dr.p, df.p, dn.p, ws.p, wsb, st));
    uint64_t steps = 0;
    AES_TRY(d2h_scalar(dn.p, &steps));
    AES_CUDA_TRY(cudaMemcpyAsync(out_rate, dr.p, steps * 8, cudaMemcpyDeviceToHost, st));
    AES_CUDA_TRY(cudaMemcpyAsync(out_frac, df.p, steps * 8, cudaMemcpyDeviceToHost, st));
    AES_TRY(sync());
    *n_steps = steps;
    return AES_OK;
}

int aes_cdf_stats(const double* rates, uint64_t n, double* out_rate, double* out_frac, uint64_t* n_steps) {
    if (n == 0) return fail(AES_ERR_INVALID_ARG, "rates must be nonempty");
    if (!rates || !out_rate || !out_frac || !n_steps) return fail(AES_ERR_INVALID_ARG, "null argument");
    DBuf<double> d;
    AES_TRY(d.alloc(n));
    AES_CUDA_TRY(cudaMemcpyAsync(d.p, rates, n * 8, cudaMemcpyHostToDevice, lib_stream()));
    return cdf_device(d.p, n, out_rate, out_frac, n_steps);
}

int aes_sampling_rate_cdf(aes_plan_t p, aes_csr_t a, double* out_rate, double* out_frac, uint64_t* n_steps) {
    if (!p || !a || !out_rate || !out_frac || !n_steps) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (p->n_rows != a->n_rows) return fail(AES_ERR_INVALID_ARG, "plan/stats row count mismatch");
    if (a->n_rows == 0) return fail(AES_ERR_INVALID_ARG, "rates must be nonempty");
    cudaStream_t st = lib_stream();
    DBuf<unsigned long long> tot;
    DBuf<double> pr;
    DBuf<unsigned char> seen;
    AES_TRY(tot.alloc(3));
    AES_TRY(pr.alloc(a->n_rows));
    if (p->explicit_plan) {
        AES_TRY(seen.alloc(a->nnz ? a->nnz : 1));
        AES_TRY(launch_explicit_rate(a->row_ptr, p->params, p->starts_ptr, p->starts, a->n_rows, a->nnz, seen.p,
                                     pr.p, tot.p, st));
    } else {
        AES_TRY(launch_sampling_rate(a->row_ptr, a->n_rows, p->width, p->strategy, pr.p, tot.p, st));
    }
    return cdf_device(pr.p, a->n_rows, out_rate, out_frac, n_steps);
}

// ---- SpMM ------------------------------------------------------------------------
int aes_spmm_exact(aes_csr_t a, const float* b, uint64_t b_rows, uint64_t f, float* c) {
    if (!a) return fail(AES_ERR_INVALID_ARG, "null csr");
    if (a->n_cols != b_rows) return fail(AES_ERR_SHAPE, "ShapeMismatch");
    return spmm_host(a->row_ptr, a->col, a->val, a->n_rows, b, b_rows, f, c, 0);
}

int aes_spmm_sampled(aes_csr_t a, const float* b, uint64_t b_rows, uint64_t f, aes_plan_t p, float* c,
                     uint64_t* fma_count, uint64_t* loads_a, uint64_t* loads_b) {
    if (!a || !p) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (a->n_cols != b_rows) return fail(AES_ERR_SHAPE, "ShapeMismatch");
    if (p->n_rows != a->n_rows) return fail(AES_ERR_PLAN_MISMATCH, "PlanMatrixMismatch");
    DBuf<uint32_t> tc;
    DBuf<float> tv;
    const uint32_t* scol;
    const float* sval;
    AES_TRY(sampled_for(p, a, tc, tv, &scol, &sval));
    AES_TRY(spmm_host(p->srow_ptr, scol, sval, a->n_rows, b, b_rows, f, c, plan_row_bound(p)));
    // WorkCounter semantics (spmm.cpp:95-97): fma = slots*F, loads_a = slots
    if (fma_count) *fma_count = p->total_slots * f;
    if (loads_a) *loads_a = p->total_slots;
    if (loads_b) *loads_b = p->total_slots * f;
    return AES_OK;
}

int aes_spmm_sampled_async(aes_csr_t a, const float* b, uint64_t b_rows, uint64_t f, aes_plan_t p, float* c,
                           void* stream) {
    if (!a || !p) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (a->n_cols != b_rows) return fail(AES_ERR_SHAPE, "ShapeMismatch");
    if (p->n_rows != a->n_rows) return fail(AES_ERR_PLAN_MISMATCH, "PlanMatrixMismatch");
    if (a != p->src) return fail(AES_ERR_UNSUPPORTED, "async spmm needs the plan's own matrix");
    const uint64_t n = a->n_rows;
    if (n == 0 || f == 0) return AES_OK;
    lib_stream();  // pool setup
    cudaStream_t st = stream ? as_stream(stream) : lib_stream();
    const uint64_t ld = round4(f);
    float *db = nullptr, *dc = nullptr;
    AES_CUDA_TRY(cudaMallocAsync((void**)&db, b_rows * ld * 4 + 16, st));
    AES_CUDA_TRY(cudaMallocAsync((void**)&dc, n * ld * 4 + 16, st));
    if (ld != f) AES_CUDA_TRY(cudaMemsetAsync(db, 0, b_rows * ld * 4, st));
    AES_CUDA_TRY(cudaMemcpy2DAsync(db, ld * 4, b, f * 4, f * 4, b_rows, cudaMemcpyHostToDevice, st));
    AES_TRY(aes_dev_spmm_f32_ex(p->srow_ptr, p->scol, p->sval, n, db, ld, f, dc, ld, plan_row_bound(p), st));
    AES_CUDA_TRY(cudaMemcpy2DAsync(c, f * 4, dc, ld * 4, f * 4, n, cudaMemcpyDeviceToHost, st));
    AES_CUDA_TRY(cudaFreeAsync(db, st));
    AES_CUDA_TRY(cudaFreeAsync(dc, st));
    if (st != lib_stream()) p->note_use(st);
    return AES_OK;
}

// ---- quantization -------------------------------------------------------------------
static int make_qfeat(const float* x, uint64_t rows, uint64_t cols, float lo, float hi, uint32_t bits,
                      const float* dx, aes_qfeat_t* out) {
    cudaStream_t st = lib_stream();
    auto* q = new aes_qfeat_s;
    q->rows = rows;
    q->cols = cols;
    q->x_min = lo;
    q->x_max = hi;
    q->bits = bits;
    q->u8 = bits <= 8;
    q->ld = q->u8 ? round16(cols ? cols : 1) : cols;
    const size_t esz = q->u8 ? 1 : 2;
    int s = AES_OK;
    if (cudaMallocAsync(&q->codes, rows * q->ld * esz + 16, st) != cudaSuccess) s = fail(AES_ERR_CUDA, "alloc");
    if (!s && q->ld != cols) cudaMemsetAsync(q->codes, 0, rows * q->ld * esz, st);
    if (!s) s = aes_dev_quantize(dx, rows, cols, cols, lo, hi, bits, q->codes, q->ld, st);
    if (!s && q->u8) {
        if (cudaMallocAsync((void**)&q->lut, 256 * sizeof(float), st) != cudaSuccess) s = fail(AES_ERR_CUDA, "alloc");
        if (!s) s = aes_dev_dequant_lut(lo, hi, bits, q->lut, st);
    }
    if (!s) s = sync();
    if (s) {
        aes_qfeat_destroy(q);
        return s;
    }
    (void)x;
    *out = q;
    return AES_OK;
}

int aes_quantize(const float* x, uint64_t rows, uint64_t cols, uint32_t bits, aes_qfeat_t* out) {
    if (!out) return fail(AES_ERR_INVALID_ARG, "null out");
    const uint64_t n = rows * cols;
    if (n == 0) return fail(AES_ERR_EMPTY, "EmptyMatrix");       // quantize.cpp:12
    if (bits < 1 || bits > 16) return fail(AES_ERR_BITS, "bits must be 1..16");  // :13
    cudaStream_t st = lib_stream();
    DBuf<float> dx, res;
    DBuf<char> ws;
    AES_TRY(dx.alloc(n));
    AES_CUDA_TRY(cudaMemcpyAsync(dx.p, x, n * 4, cudaMemcpyHostToDevice, st));
    const size_t wsb = aes_dev_scan_workspace_bytes(1);
    AES_TRY(ws.alloc(wsb));
    AES_TRY(res.alloc(4));
    AES_TRY(aes_dev_fit_params(dx.p, n, res.p, ws.p, wsb, st));
    float r[4];
    AES_CUDA_TRY(cudaMemcpyAsync(r, res.p, sizeof(r), cudaMemcpyDeviceToHost, st));
    AES_TRY(sync());
    uint32_t flag;
    memcpy(&flag, &r[2], 4);
    if (flag) return fail(AES_ERR_NONFINITE, "NonFinite");
    return make_qfeat(x, rows, cols, r[0], r[1], bits, dx.p, out);
}

int aes_quantize_with(const float* x, uint64_t rows, uint64_t cols, float x_min, float x_max, uint32_t bits,
                      aes_qfeat_t* out) {
    if (!out) return fail(AES_ERR_INVALID_ARG, "null out");
    if (bits < 1 || bits > 16 || !(x_min <= x_max)) return fail(AES_ERR_QPARAMS, "invalid QuantParams");
    const uint64_t n = rows * cols;
    DBuf<float> dx;
    AES_TRY(dx.alloc(n ? n : 1));
    if (n) AES_CUDA_TRY(cudaMemcpyAsync(dx.p, x, n * 4, cudaMemcpyHostToDevice, lib_stream()));
    return make_qfeat(x, rows, cols, x_min, x_max, bits, dx.p, out);
}

int aes_qfeat_from_codes(const uint16_t* codes, uint64_t rows, uint64_t cols, float x_min, float x_max,
                         uint32_t bits, aes_qfeat_t* out) {
    if (!out) return fail(AES_ERR_INVALID_ARG, "null out");
    if (bits < 1 || bits > 16) return fail(AES_ERR_QPARAMS, "invalid QuantParams");
    cudaStream_t st = lib_stream();
    const uint64_t n = rows * cols;
    DBuf<uint16_t> d16;
    AES_TRY(d16.alloc(n ? n : 1));
    if (n) AES_CUDA_TRY(cudaMemcpyAsync(d16.p, codes, n * 2, cudaMemcpyHostToDevice, st));
    auto* q = new aes_qfeat_s;
    q->rows = rows;
    q->cols = cols;
    q->x_min = x_min;
    q->x_max = x_max;
    q->bits = bits;
    q->u8 = false;
    q->ld = cols;
    int s = AES_OK;
    if (bits <= 8) {
        DBuf<unsigned int> ovf;
        uint64_t ld = round16(cols ? cols : 1);
        void* c8 = nullptr;
        s = ovf.alloc(1);
        if (!s && cudaMallocAsync(&c8, rows * ld + 16, st) != cudaSuccess) s = fail(AES_ERR_CUDA, "alloc");
        if (!s) {
            cudaMemsetAsync(c8, 0, rows * ld, st);
            cudaMemsetAsync(ovf.p, 0, 4, st);
            if (n)
                narrow_u16_kernel<<<grid_for(n, 256, num_sms() * 32), 256, 0, st>>>(d16.p, rows, cols, ld,
                                                                              (uint8_t*)c8, ovf.p);
            unsigned int o = 0;
            s = d2h_scalar(ovf.p, &o);
            if (!s && o == 0) {
                q->u8 = true;
                q->ld = ld;
                q->codes = c8;
                c8 = nullptr;
                if (cudaMallocAsync((void**)&q->lut, 1024, st) != cudaSuccess) s = fail(AES_ERR_CUDA, "alloc");
                if (!s) s = aes_dev_dequant_lut(x_min, x_max, bits, q->lut, st);
            }
        }
        if (c8) cudaFreeAsync(c8, st);
    }
    if (!s && !q->u8) q->codes = d16.release();
    if (!s) s = sync();
    if (s) {
        aes_qfeat_destroy(q);
        return s;
    }
    *out = q;
    return AES_OK;
}

// Fast mode: per-row / per-feature affine codes (affine.cu).
int aes_quantize_affine(const float* x, uint64_t rows, uint64_t cols, int mode, aes_qfeat_t* out) {
    if (!out) return fail(AES_ERR_INVALID_ARG, "null out");
    if (mode != AES_QAFFINE_ROW && mode != AES_QAFFINE_FEATURE) return fail(AES_ERR_INVALID_ARG, "unknown affine mode");
    const uint64_t n = rows * cols;
    if (n == 0) return fail(AES_ERR_EMPTY, "EmptyMatrix");
    cudaStream_t st = lib_stream();
    DBuf<float> dx;
    DBuf<char> ws;
    DBuf<unsigned int> bad;
    AES_TRY(dx.alloc(n));
    AES_CUDA_TRY(cudaMemcpyAsync(dx.p, x, n * 4, cudaMemcpyHostToDevice, st));
    const size_t wsb = aes_quantize_affine_workspace_bytes(rows, cols, mode);
    AES_TRY(ws.alloc(wsb));
    AES_TRY(bad.alloc(1));
    auto* q = new aes_qfeat_s;
    q->rows = rows;
    q->cols = cols;
    q->bits = 8;
    q->u8 = true;
    q->affine = mode;
    q->ld = round16(cols);
    int s = AES_OK;
    const uint64_t np = mode == AES_QAFFINE_ROW ? rows : cols;
    if (cudaMallocAsync(&q->codes, rows * q->ld + 16, st) != cudaSuccess ||
        cudaMallocAsync((void**)&q->aparams, np * 2 * sizeof(float), st) != cudaSuccess)
        s = fail(AES_ERR_CUDA, "alloc");
    if (!s && q->ld != cols) s = cudaMemsetAsync(q->codes, 0, rows * q->ld, st) == cudaSuccess ? AES_OK
                                                                                              : fail(AES_ERR_CUDA, "memset");
    if (!s) s = aes_dev_quantize_affine(dx.p, rows, cols, cols, mode, (uint8_t*)q->codes, q->ld, q->aparams, bad.p,
                                        ws.p, wsb, st);
    unsigned int flag = 0;
    if (!s) s = d2h_scalar(bad.p, &flag);
    if (!s && flag) s = fail(AES_ERR_NONFINITE, "NonFinite");
    if (s) {
        aes_qfeat_destroy(q);
        return s;
    }
    *out = q;
    return AES_OK;
}

int aes_qfeat_affine(aes_qfeat_t q, int* mode, float* params) {
    if (!q) return fail(AES_ERR_INVALID_ARG, "null qfeat");
    if (mode) *mode = q->affine;
    if (params && q->affine >= 0) {
        const uint64_t np = q->affine == AES_QAFFINE_ROW ? q->rows : q->cols;
        AES_CUDA_TRY(cudaMemcpyAsync(params, q->aparams, np * 8, cudaMemcpyDeviceToHost, lib_stream()));
        return sync();
    }
    return AES_OK;
}

int aes_qfeat_destroy(aes_qfeat_t q) {
    if (!q) return AES_OK;
    cudaStream_t st = lib_stream();
    if (q->codes) cudaFreeAsync(q->codes, st);
    if (q->lut) cudaFreeAsync(q->lut, st);
    if (q->aparams) cudaFreeAsync(q->aparams, st);
    delete q;
    return AES_OK;
}

int aes_qfeat_info(aes_qfeat_t q, uint64_t* rows, uint64_t* cols, float* x_min, float* x_max, uint32_t* bits) {
    if (!q) return fail(AES_ERR_INVALID_ARG, "null qfeat");
    if (rows) *rows = q->rows;
    if (cols) *cols = q->cols;
    if (x_min) *x_min = q->x_min;
    if (x_max) *x_max = q->x_max;
    if (bits) *bits = q->bits;
    return AES_OK;
}

int aes_qfeat_codes(aes_qfeat_t q, uint16_t* codes) {
    if (!q) return fail(AES_ERR_INVALID_ARG, "null qfeat");
    const uint64_t n = q->rows * q->cols;
    if (n == 0) return AES_OK;
    cudaStream_t st = lib_stream();
    if (q->u8) {
        DBuf<uint16_t> w;
        AES_TRY(w.alloc(n));
        widen_u8_kernel<<<grid_for(n, 256, num_sms() * 32), 256, 0, st>>>((const uint8_t*)q->codes, q->rows, q->cols,
                                                                    q->ld, w.p);
        AES_CUDA_TRY(cudaGetLastError());
        AES_CUDA_TRY(cudaMemcpyAsync(codes, w.p, n * 2, cudaMemcpyDeviceToHost, st));
        return sync();
    }
    AES_CUDA_TRY(cudaMemcpyAsync(codes, q->codes, n * 2, cudaMemcpyDeviceToHost, st));
    return sync();
}

static int dequant_device(aes_qfeat_t q, DBuf<float>& out, uint64_t& ld) {
    ld = round4(q->cols ? q->cols : 1);
    AES_TRY(out.alloc(q->rows * ld));
    cudaStream_t st = lib_stream();
    if (ld != q->cols) AES_CUDA_TRY(cudaMemsetAsync(out.p, 0, q->rows * ld * 4, st));
    if (q->affine >= 0)
        return aes_dev_dequantize_affine((const uint8_t*)q->codes, q->rows, q->cols, q->ld, q->affine, q->aparams,
                                         out.p, ld, st);
    return aes_dev_dequantize(q->codes, q->rows, q->cols, q->ld, q->x_min, q->x_max, q->bits, out.p, ld, st);
}

int aes_dequantize(aes_qfeat_t q, float* x) {
    if (!q) return fail(AES_ERR_INVALID_ARG, "null qfeat");
    if (q->rows * q->cols == 0) return AES_OK;
    DBuf<float> d;
    uint64_t ld;
    AES_TRY(dequant_device(q, d, ld));
    AES_TRY(download_dense(d.p, ld, q->rows, q->cols, x));
    return sync();
}

int aes_spmm_sampled_q8(aes_csr_t a, aes_qfeat_t q, aes_plan_t p, float* c) {
    if (!a || !q) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (a->n_cols != q->rows) return fail(AES_ERR_SHAPE, "ShapeMismatch");
    if (p && p->n_rows != a->n_rows) return fail(AES_ERR_PLAN_MISMATCH, "PlanMatrixMismatch");
    const uint64_t n = a->n_rows, f = q->cols;
    if (n == 0 || f == 0) return AES_OK;
    cudaStream_t st = lib_stream();
    DBuf<uint32_t> tc;
    DBuf<float> tv;
    const uint64_t* rp = a->row_ptr;
    const uint32_t* scol = a->col;
    const float* sval = a->val;
    if (p) {
        rp = p->srow_ptr;
        AES_TRY(sampled_for(p, a, tc, tv, &scol, &sval));
    }
    const uint64_t ldc = round4(f);
    DBuf<float> dc;
    AES_TRY(dc.alloc(n * ldc));
    if (q->affine >= 0) {  // fast mode: affine decode fused into the gather
        AES_TRY(aes_dev_spmm_q8_affine(rp, scol, sval, n, (const uint8_t*)q->codes, q->ld, f, q->affine, q->aparams,
                                       dc.p, ldc, st));
    } else if (q->u8) {
        AES_TRY(aes_dev_spmm_q8_ex(rp, scol, sval, n, (const uint8_t*)q->codes, q->ld, f, q->lut, dc.p, ldc,
                                   plan_row_bound(p), st));
    } else {  // 9..16-bit codes: dequantize on the GPU, then the fp32 kernel
        DBuf<float> dx;
        uint64_t ld;
        AES_TRY(dequant_device(q, dx, ld));
        AES_TRY(aes_dev_spmm_f32_ex(rp, scol, sval, n, dx.p, ld, f, dc.p, ldc, plan_row_bound(p), st));
    }
    AES_TRY(download_dense(dc.p, ldc, n, f, c));
    return sync();
}

// ---- GNN -------------------------------------------------------------------------------
int aes_dense_matmul(const float* a, uint64_t m, uint64_t k, const float* b, uint64_t n, float* c) {
    DBuf<float> da, db, dc;
    uint64_t lda, ldb;
    AES_TRY(upload_dense(a, m, k, da, lda));
    AES_TRY(upload_dense(b, k, n, db, ldb));
    const uint64_t ldc = round4(n ? n : 1);
    AES_TRY(dc.alloc(m * ldc));
    // finite B makes the reference's zero-skip result-neutral (gemm.cu): the
    // select-free kernel then runs (one scalar read-back)
    unsigned int b_bad = 1;
    if (k * n) {
        DBuf<unsigned int> bad;
        AES_TRY(bad.alloc(1));
        AES_TRY(aes_dev_all_finite(db.p, k * ldb, bad.p, lib_stream()));
        AES_TRY(d2h_scalar(bad.p, &b_bad));
    }
    float* dsts[1] = {dc.p};
    AES_TRY(aes_dev_gemm_bias_act_ex(da.p, m, k, lda, db.p, n, ldb, nullptr, 0, b_bad == 0, dsts, nullptr, 1, 0, ldc,
                                     lib_stream()));
    AES_TRY(download_dense(dc.p, ldc, m, n, c));
    return sync();
}

static int gnn_forward_impl(int kind, aes_csr_t adj, const float* x, const uint64_t* dims, int n_layers,
                            const float* weights, const float* biases, const uint64_t* bias_len, aes_plan_t p,
                            float* out, int fast_gemm = 0) {
    if (!adj || !dims) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (adj->n_cols != adj->n_rows) return fail(AES_ERR_SHAPE, "ShapeMismatch");
    if (p && p->n_rows != adj->n_rows) return fail(AES_ERR_PLAN_MISMATCH, "PlanMatrixMismatch");
    cudaStream_t st = lib_stream();
    const uint64_t n = adj->n_rows;
    DBuf<uint32_t> tc;
    DBuf<float> tv;
    const uint64_t* rp = adj->row_ptr;
    const uint32_t* scol = adj->col;
    const float* sval = adj->val;
    if (p) {
        rp = p->srow_ptr;
        AES_TRY(sampled_for(p, adj, tc, tv, &scol, &sval));
    }
    const bool sage = kind == 1;  // ModelKind::SageMean: z = concat(h, agg) (gnn.cpp:80-95)
    DBuf<float> h, agg, nxt, dw, db;
    uint64_t ldh;
    AES_TRY(upload_dense(x, n, dims[0], h, ldh));
    uint64_t woff = 0, boff = 0;
    for (int l = 0; l < n_layers; ++l) {
        const uint64_t fin = dims[l], fout = dims[l + 1];
        const uint64_t kin = sage ? 2 * fin : fin;
        if (bias_len && bias_len[l] != 0 && bias_len[l] != fout) return fail(AES_ERR_SHAPE, "ShapeMismatch");
        // agg (or [h | agg] for SAGE) with ld = round4(kin)
        const uint64_t lda = round4(kin ? kin : 1);
        AES_TRY(agg.alloc(n * lda));
        if (sage) {
            if (lda != kin) AES_CUDA_TRY(cudaMemsetAsync(agg.p, 0, n * lda * 4, st));
            if (fin)
                AES_CUDA_TRY(cudaMemcpy2DAsync(agg.p, lda * 4, h.p, ldh * 4, fin * 4, n, cudaMemcpyDeviceToDevice, st));
            // SpMM writes round4(fin) columns; aggregate into a scratch then place after h
            DBuf<float> a2;
            const uint64_t ld2 = round4(fin ? fin : 1);
            AES_TRY(a2.alloc(n * ld2));
            AES_TRY(aes_dev_spmm_f32_ex(rp, scol, sval, n, h.p, ldh, fin, a2.p, ld2, plan_row_bound(p), st));
            if (fin)
                AES_CUDA_TRY(cudaMemcpy2DAsync(agg.p + fin, lda * 4, a2.p, ld2 * 4, fin * 4, n,
                                               cudaMemcpyDeviceToDevice, st));
        } else {
            AES_TRY(aes_dev_spmm_f32_ex(rp, scol, sval, n, h.p, ldh, fin, agg.p, lda, plan_row_bound(p), st));
        }
        uint64_t ldw;
        AES_TRY(upload_dense(weights + woff, kin, fout, dw, ldw));
        const bool has_bias = bias_len ? bias_len[l] != 0 : true;
        if (has_bias) {
            AES_TRY(db.alloc(fout ? fout : 1));
            if (fout) AES_CUDA_TRY(cudaMemcpyAsync(db.p, biases + boff, fout * 4, cudaMemcpyHostToDevice, st));
        }
        const uint64_t ldo = round4(fout ? fout : 1);
        AES_TRY(nxt.alloc(n * ldo));
        if (ldo != fout) AES_CUDA_TRY(cudaMemsetAsync(nxt.p, 0, n * ldo * 4, st));
        if (fast_gemm && kin <= 128 && fout <= 128 && kin > 0) {
            // opt-in tcgen05 TF32 layer transform (not bit-exact; tc_gemm.cu)
            DBuf<float> wt;
            AES_TRY(wt.alloc(aes_gemm_tf32_scratch_floats(kin, fout)));
            AES_TRY(aes_dev_gemm_tf32(agg.p, n, kin, lda, dw.p, fout, ldw, has_bias ? db.p : nullptr,
                                      l + 1 < n_layers, nxt.p, ldo, wt.p, st));
        } else {
            // finite W makes the reference's zero-skip result-neutral (gemm.cu)
            DBuf<unsigned int> bad;
            AES_TRY(bad.alloc(1));
            AES_TRY(aes_dev_all_finite(dw.p, kin * ldw, bad.p, st));
            unsigned int w_bad = 0;
            AES_TRY(d2h_scalar(bad.p, &w_bad));
            float* dsts[1] = {nxt.p};
            AES_TRY(aes_dev_gemm_bias_act_ex(agg.p, n, kin, lda, dw.p, fout, ldw, has_bias ? db.p : nullptr,
                                             l + 1 < n_layers, w_bad == 0, dsts, nullptr, 1, 0, ldo, st));
        }
        std::swap(h.p, nxt.p);
        std::swap(h.n, nxt.n);
        ldh = ldo;
        woff += kin * fout;
        boff += has_bias ? fout : 0;
    }
    AES_TRY(download_dense(h.p, ldh, n, dims[n_layers], out));
    return sync();
}

int aes_gcn_forward(aes_csr_t adj, const float* x, const uint64_t* dims, int n_layers, const float* weights,
                    const float* biases, const uint64_t* bias_len, aes_plan_t p, float* out) {
    return gnn_forward_impl(0, adj, x, dims, n_layers, weights, biases, bias_len, p, out);
}

int aes_sage_forward(aes_csr_t adj_mean, const float* x, const uint64_t* dims, int n_layers, const float* weights,
                     const float* biases, const uint64_t* bias_len, aes_plan_t p, float* out) {
    return gnn_forward_impl(1, adj_mean, x, dims, n_layers, weights, biases, bias_len, p, out);
}

int aes_gnn_forward_ex(int kind, aes_csr_t adj, const float* x, const uint64_t* dims, int n_layers,
                       const float* weights, const float* biases, const uint64_t* bias_len, aes_plan_t p, int fast_gemm,
                       float* out) {
    return gnn_forward_impl(kind, adj, x, dims, n_layers, weights, biases, bias_len, p, out, fast_gemm);
}

int aes_row_mean_normalize(aes_csr_t a, aes_csr_t* out) {
    if (!a || !out) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (a->n_rows != a->n_cols) return fail(AES_ERR_NOT_SQUARE, "NotSquare");
    cudaStream_t st = lib_stream();
    DBuf<uint64_t> rp;
    DBuf<uint32_t> ci;
    DBuf<float> vv;
    AES_TRY(rp.alloc(a->n_rows + 1));
    AES_TRY(ci.alloc(a->nnz ? a->nnz : 1));
    AES_TRY(vv.alloc(a->nnz ? a->nnz : 1));
    AES_CUDA_TRY(cudaMemcpyAsync(rp.p, a->row_ptr, (a->n_rows + 1) * 8, cudaMemcpyDeviceToDevice, st));
    if (a->nnz) {
        AES_CUDA_TRY(cudaMemcpyAsync(ci.p, a->col, a->nnz * 4, cudaMemcpyDeviceToDevice, st));
        AES_CUDA_TRY(cudaMemcpyAsync(vv.p, a->val, a->nnz * 4, cudaMemcpyDeviceToDevice, st));
    }
    AES_TRY(launch_row_mean(rp.p, a->n_rows, vv.p, st));
    AES_TRY(sync());
    auto* o = new aes_csr_s;
    o->n_rows = a->n_rows;
    o->n_cols = a->n_cols;
    o->nnz = a->nnz;
    o->row_ptr = rp.release();
    o->col = ci.release();
    o->val = vv.release();
    *out = o;
    return AES_OK;
}

int aes_argmax_rows(const float* x, uint64_t rows, uint64_t cols, uint32_t* out) {
    if (rows == 0) return AES_OK;
    if (cols == 0) return fail(AES_ERR_INVALID_ARG, "argmax of an empty row");
    DBuf<float> dx;
    DBuf<uint32_t> dout;
    uint64_t ld;
    AES_TRY(upload_dense(x, rows, cols, dx, ld));
    AES_TRY(dout.alloc(rows));
    AES_TRY(launch_argmax(dx.p, rows, cols, ld, dout.p, lib_stream()));
    AES_CUDA_TRY(cudaMemcpyAsync(out, dout.p, rows * 4, cudaMemcpyDeviceToHost, lib_stream()));
    return sync();
}

int aes_evaluate(const float* logits, uint64_t rows, uint64_t cols, const uint32_t* labels, uint64_t labels_len,
                 const float* reference_logits, const uint8_t* mask, uint64_t mask_len, double* accuracy,
                 double* agreement, uint64_t* per_class) {
    if (labels_len != rows) return fail(AES_ERR_INVALID_ARG, "labels length != n_nodes");
    if (mask && mask_len != 0 && mask_len != rows) return fail(AES_ERR_INVALID_ARG, "mask length != n_nodes");
    if (mask_len == 0) mask = nullptr;
    cudaStream_t st = lib_stream();
    DBuf<float> dl, dr;
    DBuf<uint32_t> pred, ref, lab;
    DBuf<uint8_t> dm;
    DBuf<unsigned long long> counts, pc;
    uint64_t ld;
    AES_TRY(counts.alloc(4));
    AES_TRY(pc.alloc(cols ? cols : 1));
    AES_CUDA_TRY(cudaMemsetAsync(counts.p, 0, 32, st));
    AES_CUDA_TRY(cudaMemsetAsync(pc.p, 0, (cols ? cols : 1) * 8, st));
    if (rows) {
        if (cols == 0) return fail(AES_ERR_INVALID_ARG, "LabelOutOfRange");
        AES_TRY(upload_dense(logits, rows, cols, dl, ld));
        AES_TRY(pred.alloc(rows));
        AES_TRY(lab.alloc(rows));
        AES_TRY(launch_argmax(dl.p, rows, cols, ld, pred.p, st));
        AES_CUDA_TRY(cudaMemcpyAsync(lab.p, labels, rows * 4, cudaMemcpyHostToDevice, st));
        if (reference_logits) {
            AES_TRY(upload_dense(reference_logits, rows, cols, dr, ld));
            AES_TRY(ref.alloc(rows));
            AES_TRY(launch_argmax(dr.p, rows, cols, ld, ref.p, st));
        }
        if (mask) {
            AES_TRY(dm.alloc(rows));
            AES_CUDA_TRY(cudaMemcpyAsync(dm.p, mask, rows, cudaMemcpyHostToDevice, st));
        }
        AES_TRY(launch_evaluate(pred.p, lab.p, ref.p, dm.p, rows, cols, counts.p, pc.p, st));
    }
    unsigned long long c[4];
    AES_CUDA_TRY(cudaMemcpyAsync(c, counts.p, sizeof(c), cudaMemcpyDeviceToHost, st));
    if (per_class && cols)
        AES_CUDA_TRY(cudaMemcpyAsync(per_class, pc.p, cols * 8, cudaMemcpyDeviceToHost, st));
    AES_TRY(sync());
    if (c[3]) return fail(AES_ERR_INVALID_ARG, "LabelOutOfRange");
    if (accuracy) *accuracy = c[0] == 0 ? 0.0 : double(c[1]) / double(c[0]);
    if (agreement) *agreement = !reference_logits ? 0.0 : (c[0] == 0 ? 0.0 : double(c[2]) / double(c[0]));
    return AES_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// helpers for io.cu (same translation-unit-private allocator and stream)
// ---------------------------------------------------------------------------
namespace aes {

void* capi_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes ? bytes : 16, lib_stream()) != cudaSuccess) return nullptr;
    if (cudaStreamSynchronize(lib_stream()) != cudaSuccess) return nullptr;
    return p;
}

void capi_free(void* p) {
    if (p) cudaFreeAsync(p, lib_stream());
}

// QuantizedFeatures over device u8 codes (ownership of d_codes moves in).
int capi_make_qfeat_u8(const uint8_t* d_codes, uint64_t rows, uint64_t cols, uint64_t ld, float lo, float hi,
                       aes_qfeat_t* out) {
    auto* q = new aes_qfeat_s;
    q->rows = rows;
    q->cols = cols;
    q->ld = ld;
    q->x_min = lo;
    q->x_max = hi;
    q->bits = 8;
    q->u8 = true;
    q->codes = const_cast<uint8_t*>(d_codes);
    cudaStream_t st = lib_stream();
    int s = cudaMallocAsync((void**)&q->lut, 256 * sizeof(float), st) == cudaSuccess ? AES_OK
                                                                                    : fail(AES_ERR_CUDA, "alloc");
    if (!s) s = aes_dev_dequant_lut(lo, hi, 8, q->lut, st);
    if (!s) s = sync();
    if (s) {
        q->codes = nullptr;  // caller keeps ownership on failure
        aes_qfeat_destroy(q);
        return s;
    }
    *out = q;
    return AES_OK;
}

// CsrMatrix over device arrays (ownership moves in on success), validated.
int capi_csr_from_device(uint64_t n_rows, uint64_t n_cols, uint64_t nnz, uint64_t* rp, uint32_t* col, float* val,
                         aes_csr_t* out) {
    auto* a = new aes_csr_s;
    a->n_rows = n_rows;
    a->n_cols = n_cols;
    a->nnz = nnz;
    a->row_ptr = rp;
    a->col = col;
    a->val = val;
    uint64_t first = 0;
    int s = d2h_scalar(rp, &first);
    if (!s) s = validate_device(a, n_rows + 1, nnz, first);
    if (s) {
        a->row_ptr = nullptr;
        a->col = nullptr;
        a->val = nullptr;
        delete a;
        return s;
    }
    *out = a;
    return AES_OK;
}

int capi_qfeat_device(aes_qfeat_t q, const void** codes, uint64_t* ld, int* u8) {
    if (!q) return fail(AES_ERR_INVALID_ARG, "null qfeat");
    if (q->affine >= 0) return fail(AES_ERR_INVALID_ARG, "FMAT dtype 1 stores global-params codes only");
    *codes = q->codes;
    *ld = q->ld;
    *u8 = q->u8 ? 1 : 0;
    return AES_OK;
}

int capi_csr_device(aes_csr_t a, const uint64_t** rp, const uint32_t** col, const float** val, uint64_t* n_rows,
                    uint64_t* n_cols, uint64_t* nnz) {
    if (!a) return fail(AES_ERR_INVALID_ARG, "null csr");
    AES_TRY(sync());
    *rp = a->row_ptr;
    *col = a->col;
    *val = a->val;
    *n_rows = a->n_rows;
    *n_cols = a->n_cols;
    *nnz = a->nnz;
    return AES_OK;
}

}  // namespace aes
