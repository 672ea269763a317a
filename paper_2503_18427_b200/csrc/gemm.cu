// Ordered fp32 layer GEMM + bias + ReLU epilogue for the GCN layer driver.
//
// Bit-exact with the reference dense_matmul (proj/src/gnn.cpp:11-31): every
// output element accumulates k in ascending order as acc = RN(acc + RN(a*w))
// from +0.0f, skipping a == 0 exactly as the reference does (which also keeps
// 0*inf from producing NaN).  Bias then ReLU follow gnn.cpp:41-52 with
// std::max(v, 0.0f) semantics ((v < 0) ? 0 : v, so -0.0f and NaN pass through).
// Tensor cores are deliberately not used: their reduction order and fused
// rounding cannot reproduce the reference's result bits.  (A tcgen05 TF32/BF16
// "fast mode" with a stated tolerance is listed as next work in DESIGN.md.)
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace aes {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
constexpr int kThreads = (BM / TM) * (BN / TN);  // 256

__global__ void __launch_bounds__(kThreads)
gemm_ordered_kernel(const float* __restrict__ a, uint64_t m, uint64_t k, uint64_t lda,
                    const float* __restrict__ w, uint64_t n, uint64_t ldw,
                    const float* __restrict__ bias, int relu, float* __restrict__ h, uint64_t ldh) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Ws[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const uint64_t m0 = (uint64_t)blockIdx.y * BM, n0 = (uint64_t)blockIdx.x * BN;

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    for (uint64_t k0 = 0; k0 < k; k0 += BK) {
        // A tile (BM x BK) -> As[kk][mm]; zero fill is neutral (a == 0 skipped)
#pragma unroll
        for (int e = tid; e < BM * BK; e += kThreads) {
            int mm = e / BK, kk = e % BK;
            uint64_t gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < m && gk < k) ? a[gm * lda + gk] : 0.f;
        }
#pragma unroll
        for (int e = tid; e < BK * BN; e += kThreads) {
            int kk = e / BN, nn = e % BN;
            uint64_t gk = k0 + kk, gn = n0 + nn;
            Ws[kk][nn] = (gk < k && gn < n) ? w[gk * ldw + gn] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float av[TM], wv[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = As[kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) wv[j] = Ws[kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const bool skip = av[i] == 0.f;
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    float s = __fadd_rn(acc[i][j], __fmul_rn(av[i], wv[j]));
                    acc[i][j] = skip ? acc[i][j] : s;
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        uint64_t gm = m0 + ty * TM + i;
        if (gm >= m) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            uint64_t gn = n0 + tx * TN + j;
            if (gn >= n) continue;
            float v = acc[i][j];
            if (bias) v = __fadd_rn(v, bias[gn]);
            if (relu) v = (v < 0.f) ? 0.f : v;
            h[gm * ldh + gn] = v;
        }
    }
}

}  // namespace
}  // namespace aes

extern "C" int aes_dev_gemm_bias_act(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w,
                                     uint64_t n, uint64_t ldw, const float* bias, int relu, float* h,
                                     uint64_t ldh, void* stream) {
    using namespace aes;
    if (m == 0 || n == 0) return AES_OK;
    if (lda < k || ldw < n || ldh < n) return fail(AES_ERR_INVALID_ARG, "leading dimension too small");
    dim3 grid((unsigned)((n + BN - 1) / BN), (unsigned)((m + BM - 1) / BM));
    if (grid.y > 65535u) {
        // tile rows in chunks the grid can address
        const uint64_t rows_per = (uint64_t)65535 * BM;
        for (uint64_t r0 = 0; r0 < m; r0 += rows_per) {
            uint64_t mm = m - r0 < rows_per ? m - r0 : rows_per;
            dim3 g2(grid.x, (unsigned)((mm + BM - 1) / BM));
            gemm_ordered_kernel<<<g2, kThreads, 0, as_stream(stream)>>>(a + r0 * lda, mm, k, lda, w, n, ldw,
                                                                        bias, relu, h + r0 * ldh, ldh);
        }
    } else {
        gemm_ordered_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(a, m, k, lda, w, n, ldw, bias, relu, h,
                                                                      ldh);
    }
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}
