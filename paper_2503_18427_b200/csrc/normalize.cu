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
    inv_sqrt_deg_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(out_ptr, n, inv_scratch);
    gcn_fill_kernel<<<grid_for(n * 32, 256, 148 * 32), 256, 0, st>>>(row_ptr, col, n, add_self_loops, out_ptr,
                                                                     inv_scratch, out_col, out_val);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace aes
