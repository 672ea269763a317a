// GCN symmetric normalization D^-1/2 (A [+ I]) D^-1/2 on the GPU —
// proj/src/matrix.cpp:107-144.  Self loops are inserted at their sorted
// position when absent; deg is the post-insertion row nnz; values are
// (1/sqrtf(deg_i)) * (1/sqrtf(deg_j)) in fp32 with IEEE-rounded sqrt and
// division (__fsqrt_rn / __fdiv_rn), matching the reference's sqrtss/divss.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace aes {
namespace {

__global__ void inv_sqrt_deg_kernel(const uint64_t* __restrict__ out_ptr, uint64_t n, float* __restrict__ inv) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t deg = out_ptr[i + 1] - out_ptr[i];
        inv[i] = deg ? __fdiv_rn(1.0f, __fsqrt_rn((float)deg)) : 0.0f;
    }
}

// warp per row: copy columns with the diagonal inserted, then values.
__global__ void gcn_fill_kernel(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ col,
                                uint64_t n, int add_self_loops, const uint64_t* __restrict__ out_ptr,
                                const float* __restrict__ inv, uint32_t* __restrict__ out_col,
                                float* __restrict__ out_val) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint64_t b = row_ptr[r], e = row_ptr[r + 1];
        // first position with col >= r
        uint64_t lo = b, hi = e;
        while (lo < hi) {
            uint64_t mid = (lo + hi) >> 1;
            if (col[mid] < r) lo = mid + 1; else hi = mid;
        }
        const bool has_diag = lo < e && col[lo] == r;
        const uint64_t ins = (add_self_loops && !has_diag) ? 1 : 0;
        const uint64_t ob = out_ptr[r];
        const float inv_r = inv[r];
        for (uint64_t k = b + lane; k < e; k += 32) {
            const uint32_t c = col[k];
            const uint64_t o = ob + (k - b) + (k >= lo ? ins : 0);
            out_col[o] = c;
            out_val[o] = __fmul_rn(inv_r, inv[c]);
        }
        if (ins && lane == 0) {
            const uint64_t o = ob + (lo - b);
            out_col[o] = (uint32_t)r;
            out_val[o] = __fmul_rn(inv_r, inv_r);
        }
    }
}

}  // namespace

int launch_gcn_normalize(const uint64_t* row_ptr, const uint32_t* col, uint64_t n, int add_self_loops,
                         const uint64_t* out_ptr, float* inv_scratch, uint32_t* out_col, float* out_val,
                         cudaStream_t st) {
    if (n == 0) return AES_OK;
    inv_sqrt_deg_kernel<<<grid_for(n, 256, num_sms() * 16), 256, 0, st>>>(out_ptr, n, inv_scratch);
    gcn_fill_kernel<<<grid_for(n * 32, 256, num_sms() * 32), 256, 0, st>>>(row_ptr, col, n, add_self_loops, out_ptr,
                                                                     inv_scratch, out_col, out_val);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

namespace {

// row_mean_normalize (matrix.cpp:146-158): every value of row i becomes
// 1.0f / float(row_nnz_i); structure unchanged.
__global__ void row_mean_kernel(const uint64_t* __restrict__ row_ptr, uint64_t n, float* __restrict__ val) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += warps) {
        const uint64_t b = row_ptr[r], e = row_ptr[r + 1];
        if (b == e) continue;
        const float w = __fdiv_rn(1.0f, (float)(e - b));
        for (uint64_t k = b + lane; k < e; k += 32) val[k] = w;
    }
}

// argmax_rows (gnn.cpp:105-116): first maximum under '>' (ties -> lowest index).
__global__ void argmax_kernel(const float* __restrict__ x, uint64_t rows, uint64_t cols, uint64_t ld,
                              uint32_t* __restrict__ out) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
        const float* row = x + r * ld;
        uint32_t best = 0;
        float bv = row[0];
        for (uint64_t j = 1; j < cols; ++j) {
            const float v = row[j];
            if (v > bv) { bv = v; best = (uint32_t)j; }
        }
        out[r] = best;
    }
}

// evaluate (gnn.cpp:118-155): counts of evaluated rows, correct predictions,
// agreements with the reference argmax, and the predicted-class histogram.
__global__ void evaluate_kernel(const uint32_t* __restrict__ pred, const uint32_t* __restrict__ labels,
                                const uint32_t* __restrict__ ref, const uint8_t* __restrict__ mask, uint64_t rows,
                                uint64_t cols, unsigned long long* __restrict__ counts,
                                unsigned long long* __restrict__ per_class) {
    unsigned long long n = 0, correct = 0, agree = 0, bad = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
        bad += labels[r] >= cols;  // LabelOutOfRange is checked over all rows (gnn.cpp:125-127)
        if (mask && mask[r] == 0) continue;
        ++n;
        atomicAdd(&per_class[pred[r]], 1ull);
        correct += pred[r] == labels[r];
        if (ref) agree += pred[r] == ref[r];
    }
    for (int o = 16; o > 0; o >>= 1) {
        n += __shfl_down_sync(0xffffffffu, n, o);
        correct += __shfl_down_sync(0xffffffffu, correct, o);
        agree += __shfl_down_sync(0xffffffffu, agree, o);
        bad += __shfl_down_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&counts[0], n);
        atomicAdd(&counts[1], correct);
        atomicAdd(&counts[2], agree);
        atomicAdd(&counts[3], bad);
    }
}

}  // namespace

int launch_row_mean(const uint64_t* row_ptr, uint64_t n, float* val, cudaStream_t st) {
    if (n == 0) return AES_OK;
    row_mean_kernel<<<grid_for(n * 32, 256, num_sms() * 32), 256, 0, st>>>(row_ptr, n, val);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_argmax(const float* x, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t* out, cudaStream_t st) {
    if (rows == 0) return AES_OK;
    argmax_kernel<<<grid_for(rows, 256, num_sms() * 16), 256, 0, st>>>(x, rows, cols, ld, out);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int launch_evaluate(const uint32_t* pred, const uint32_t* labels, const uint32_t* ref, const uint8_t* mask,
                    uint64_t rows, uint64_t cols, unsigned long long* counts, unsigned long long* per_class,
                    cudaStream_t st) {
    if (rows == 0) return AES_OK;
    evaluate_kernel<<<grid_for(rows, 256, num_sms() * 16), 256, 0, st>>>(pred, labels, ref, mask, rows, cols, counts,
                                                                   per_class);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace aes
