// Scalar (global min/max) quantization for sm_100a — proj/src/quantize.cpp.
//
//  * fit_params (quantize.cpp:11-21): deterministic two-level (value, index)
//    reduction.  The reference keeps the FIRST element that attains the
//    min/max under strict '<' (so -0.0f vs +0.0f and ties resolve to the lowest
//    index); reducing (value, index) pairs with "smaller value, then smaller
//    index" reproduces the exact float it returns, sign of zero included.
//  * quantize (quantize.cpp:23-51): fp64 with __dsub_rn/__ddiv_rn/__dmul_rn/
//    __dadd_rn so ratio*levels + 2^-7 is NOT contracted into a DFMA.
//  * dequantize (quantize.cpp:53-64): float(double(q)*step + double(lo)), and
//    the 256-entry LUT of the same values that the int8 SpMM gathers through.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "minmax.cuh"
#include "quantize.cuh"

namespace aes {
namespace {

constexpr int kFitThreads = 256;
constexpr int kFitBlocks = 148 * 16;  // partials fit aes_dev_scan_workspace_bytes (2 * 148 * 8 * 32 B)

__global__ void __launch_bounds__(kFitThreads)
fit_partial_kernel(const float* __restrict__ x, uint64_t n, uint64_t chunk, MinMax* __restrict__ part) {
    const uint64_t b0 = min(n, (uint64_t)blockIdx.x * chunk);  // trailing blocks may be empty
    const uint64_t b1 = min(n, b0 + chunk);
    MinMax m{INFINITY, -INFINITY, ~0ull, ~0ull, 0u};
    if ((uintptr_t)(x + b0) % 16 == 0) {
        // float4 loads, 4 in flight per thread (chunk is a multiple of 4 here)
        const float4* x4 = reinterpret_cast<const float4*>(x + b0);
        const uint64_t n4 = (b1 - b0) / 4;
        uint64_t j = threadIdx.x;
        for (; j + 3 * kFitThreads < n4; j += 4 * kFitThreads) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(x4 + j + u * kFitThreads);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = b0 + 4 * (j + u * kFitThreads);
                fit_elem(m, v[u].x, i);
                fit_elem(m, v[u].y, i + 1);
                fit_elem(m, v[u].z, i + 2);
                fit_elem(m, v[u].w, i + 3);
            }
        }
        for (; j < n4; j += kFitThreads) {
            const float4 v = __ldcs(x4 + j);
            const uint64_t i = b0 + 4 * j;
            fit_elem(m, v.x, i);
            fit_elem(m, v.y, i + 1);
            fit_elem(m, v.z, i + 2);
            fit_elem(m, v.w, i + 3);
        }
        for (uint64_t i = b0 + 4 * n4 + threadIdx.x; i < b1; i += kFitThreads) fit_elem(m, __ldcs(x + i), i);
    } else {
        for (uint64_t i = b0 + threadIdx.x; i < b1; i += kFitThreads) fit_elem(m, __ldcs(x + i), i);
    }
    m = block_reduce<kFitThreads>(m);
    if (threadIdx.x == 0) part[blockIdx.x] = m;
}

// Level 2: one block over the partials; emit the element values themselves.
__global__ void __launch_bounds__(kFitThreads)
fit_final_kernel(const float* __restrict__ x, const MinMax* __restrict__ part, int nparts,
                 float* __restrict__ result) {
    MinMax m{INFINITY, -INFINITY, ~0ull, ~0ull, 0u};
    for (int i = threadIdx.x; i < nparts; i += kFitThreads) mm_merge(m, part[i]);
    m = block_reduce<kFitThreads>(m);
    if (threadIdx.x == 0) {
        uint32_t* flags = reinterpret_cast<uint32_t*>(result + 2);
        flags[0] = m.bad;
        result[0] = m.bad || m.ilo == ~0ull ? 0.f : x[m.ilo];
        result[1] = m.bad || m.ihi == ~0ull ? 0.f : x[m.ihi];
    }
}


// Partials that carry their values (the GEMM's fused fit epilogue): the
// same merge, the winning values written directly.
__global__ void __launch_bounds__(kFitThreads)
fit_merge_kernel(const MinMax* __restrict__ part, int nparts, float* __restrict__ result) {
    MinMax m{INFINITY, -INFINITY, ~0ull, ~0ull, 0u};
    for (int i = threadIdx.x; i < nparts; i += kFitThreads) mm_merge(m, part[i]);
    m = block_reduce<kFitThreads>(m);
    if (threadIdx.x == 0) {
        reinterpret_cast<uint32_t*>(result + 2)[0] = m.bad;
        result[0] = m.bad || m.ilo == ~0ull ? 0.f : m.lo;
        result[1] = m.bad || m.ihi == ~0ull ? 0.f : m.hi;
    }
}

// Vector form for the common contiguous case: 4 floats -> 4 codes per thread.

// Codes through the fp32 fast path with the exact fp64 fallback
// (quantize.cuh): bit-identical to the reference, off the fp64 pipe.
constexpr int kQuantBlocks = 148 * 32;
template <typename CodeT>
__global__ void __launch_bounds__(256)
quantize_fast_kernel(const float* __restrict__ x, uint64_t rows, uint64_t cols, uint64_t ldx, float lo_f,
                     float hi_f, uint32_t levels, CodeT* __restrict__ q, uint64_t ldq, int flat4) {
    const QuantParamsDev p = quant_params(lo_f, hi_f, levels);
    if (flat4) {  // contiguous rows: one float4 -> four codes
        const uint64_t n4 = rows * cols / 4;
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        auto put = [&](uint64_t e, const float4& v) {
            const uint32_t c0 = quant_code(v.x, p), c1 = quant_code(v.y, p), c2 = quant_code(v.z, p),
                           c3 = quant_code(v.w, p);
            if (sizeof(CodeT) == 1)
                __stcs(reinterpret_cast<uchar4*>(q) + e, make_uchar4(c0, c1, c2, c3));
            else
                __stcs(reinterpret_cast<ushort4*>(q) + e, make_ushort4(c0, c1, c2, c3));
        };
        uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
        for (; e + 3 * stride < n4; e += 4 * stride) {  // 4 loads in flight per thread
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldcs(x4 + e + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) put(e + u * stride, v[u]);
        }
        for (; e < n4; e += stride) put(e, __ldcs(x4 + e));
        return;
    }
    // general strides: warp per row, lane per column
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t r = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps)
        for (uint64_t c = lane; c < cols; c += 32) q[r * ldq + c] = (CodeT)quant_code(__ldcs(x + r * ldx + c), p);
}

template <typename CodeT>
__global__ void dequantize_kernel(const CodeT* __restrict__ q, uint64_t rows, uint64_t cols, uint64_t ldq,
                                  double lo, double step, float* __restrict__ x, uint64_t ldx) {
    const uint64_t total = rows * cols;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / cols, c = e - r * cols;
        const double code = (double)q[r * ldq + c];
        x[r * ldx + c] = __double2float_rn(__dadd_rn(__dmul_rn(code, step), lo));
    }
}

// u8 codes, contiguous rows: 4 codes -> one float4 through the 256-entry
// table (each CTA builds it: float(double(q) * step + lo), the same value
// per code as dequantize_kernel, quantize.cpp:53-64), grid-stride with
// 4 loads in flight per thread.
__global__ void __launch_bounds__(256)
dequantize_u8_flat_kernel(const uchar4* __restrict__ q, uint64_t n4, double lo, double step, uint32_t levels,
                          float4* __restrict__ x) {
    __shared__ float lut[256];
    const uint32_t t = threadIdx.x;
    lut[t] = t <= levels ? __double2float_rn(__dadd_rn(__dmul_rn((double)t, step), lo)) : 0.f;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    auto put = [&](uint64_t e, uchar4 c) { __stcs(x + e, make_float4(lut[c.x], lut[c.y], lut[c.z], lut[c.w])); };
    uint64_t e = blockIdx.x * (uint64_t)blockDim.x + t;
    for (; e + 3 * stride < n4; e += 4 * stride) {
        uchar4 c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = __ldcs(q + e + u * stride);
#pragma unroll
        for (int u = 0; u < 4; ++u) put(e + u * stride, c[u]);
    }
    for (; e < n4; e += stride) put(e, __ldcs(q + e));
}

__global__ void lut_kernel(double lo, double step, uint32_t levels, float* __restrict__ lut) {
    const uint32_t q = threadIdx.x;
    lut[q] = q <= levels ? __double2float_rn(__dadd_rn(__dmul_rn((double)q, step), lo)) : 0.f;
}

}  // namespace
}  // namespace aes

extern "C" {

int aes_dev_fit_params(const float* x, uint64_t n, float* result, void* workspace,
                       size_t workspace_bytes, void* stream) {
    using namespace aes;
    cudaStream_t st = as_stream(stream);
    if (n == 0) return fail(AES_ERR_EMPTY, "EmptyMatrix");
    uint64_t nbl = (n + kFitThreads - 1) / kFitThreads;
    int nb = (int)(nbl < (uint64_t)kFitBlocks ? nbl : (uint64_t)kFitBlocks);
    if (workspace_bytes < nb * sizeof(MinMax)) return fail(AES_ERR_INVALID_ARG, "fit workspace too small");
    uint64_t chunk = ((n + nb - 1) / nb + 3) & ~3ull;  // multiple of 4: float4-aligned chunks
    auto* part = static_cast<MinMax*>(workspace);
    fit_partial_kernel<<<nb, kFitThreads, 0, st>>>(x, n, chunk, part);
    fit_final_kernel<<<1, kFitThreads, 0, st>>>(x, part, nb, result);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_fit_merge(const void* partials, uint64_t n_partials, float* result, void* stream) {
    using namespace aes;
    if (!partials || !result) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (n_partials == 0) return fail(AES_ERR_EMPTY, "EmptyMatrix");
    if (n_partials >= (1ull << 31)) return fail(AES_ERR_INVALID_ARG, "too many partials");
    fit_merge_kernel<<<1, kFitThreads, 0, as_stream(stream)>>>(static_cast<const MinMax*>(partials),
                                                              (int)n_partials, result);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_quantize(const float* x, uint64_t rows, uint64_t cols, uint64_t ldx, float lo, float hi,
                     uint32_t bits, void* codes, uint64_t ldq, void* stream) {
    using namespace aes;
    cudaStream_t st = as_stream(stream);
    if (bits < 1 || bits > 16 || !(lo <= hi)) return fail(AES_ERR_QPARAMS, "invalid QuantParams");
    const uint64_t total = rows * cols;
    if (total == 0) return AES_OK;
    const int flat4 = ldx == cols && ldq == cols && total % 4 == 0 && (uintptr_t)x % 16 == 0 &&
                      (uintptr_t)codes % (bits <= 8 ? 4 : 8) == 0;
    const unsigned blocks = grid_for(flat4 ? total / 4 : rows * 32, 256, kQuantBlocks);
    if (bits <= 8)
        quantize_fast_kernel<uint8_t><<<blocks, 256, 0, st>>>(x, rows, cols, ldx, lo, hi, (1u << bits) - 1u,
                                                              static_cast<uint8_t*>(codes), ldq, flat4);
    else
        quantize_fast_kernel<uint16_t><<<blocks, 256, 0, st>>>(x, rows, cols, ldx, lo, hi, (1u << bits) - 1u,
                                                               static_cast<uint16_t*>(codes), ldq, flat4);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_dequantize(const void* codes, uint64_t rows, uint64_t cols, uint64_t ldq, float lo, float hi,
                       uint32_t bits, float* x, uint64_t ldx, void* stream) {
    using namespace aes;
    cudaStream_t st = as_stream(stream);
    if (bits < 1 || bits > 16) return fail(AES_ERR_QPARAMS, "invalid QuantParams");
    const uint64_t total = rows * cols;
    if (total == 0) return AES_OK;
    const double step = ((double)hi - (double)lo) / (double)((1u << bits) - 1u);
    const unsigned grid = grid_for(total, 256, num_sms() * 32);
    if (bits <= 8 && ldq == cols && ldx == cols && total % 4 == 0 && (uintptr_t)codes % 4 == 0 &&
        (uintptr_t)x % 16 == 0) {
        dequantize_u8_flat_kernel<<<grid_for(total / 4, 256, num_sms() * 32), 256, 0, st>>>(
            static_cast<const uchar4*>(codes), total / 4, (double)lo, step, (1u << bits) - 1u,
            reinterpret_cast<float4*>(x));
    } else if (bits <= 8)
        dequantize_kernel<uint8_t><<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(codes), rows, cols,
                                                         ldq, (double)lo, step, x, ldx);
    else
        dequantize_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(codes), rows,
                                                          cols, ldq, (double)lo, step, x, ldx);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_dequant_lut(float lo, float hi, uint32_t bits, float* lut, void* stream) {
    using namespace aes;
    if (bits < 1 || bits > 8) return fail(AES_ERR_UNSUPPORTED, "LUT needs bits <= 8");
    const uint32_t levels = (1u << bits) - 1u;
    const double step = ((double)hi - (double)lo) / (double)levels;
    lut_kernel<<<1, 256, 0, as_stream(stream)>>>((double)lo, step, levels, lut);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // extern "C"
