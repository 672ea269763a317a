// Empirical CDF of per-row sampling rates on the device: the reference's
// cdf_stats (proj/src/bench.cpp:124-138; declared proj/include/aesspmm/
// bench.hpp:58-59), the Fig. 5/6 reporting step of SURVEY §8(f) rank 4.
//
//   sort the rates ascending, then walk them: a value equal (==) to the last
//   step's value moves that step's fraction up to (i+1)/n, otherwise a new
//   step (rates[i], (i+1)/n) starts.
//
// Device form: doubles -> order-preserving u64 keys -> radix sort (CUB) ->
// tie groups by IEEE == between neighbours (so -0 and +0 merge, as in the
// reference) -> inclusive scan of group starts -> every group's FIRST value
// and LAST fraction scattered into place.  Bit-exact: fractions are one IEEE
// division double(i+1)/double(n) (__ddiv_rn), values are the sorted inputs.
// (NaN rates make the reference's std::sort undefined; here they sort to the
// ends by sign and never merge.)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace aes {
namespace {

__device__ __forceinline__ uint64_t to_key(double v) {
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double from_key(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

__global__ void cdf_keys_kernel(const double* __restrict__ rates, uint64_t n, uint64_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = to_key(rates[i]);
}

// start[i] = 1 when sorted value i opens a new step (i == 0 or v[i-1] != v[i])
__global__ void cdf_starts_kernel(const uint64_t* __restrict__ sorted, uint64_t n, uint32_t* __restrict__ start) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        start[i] = (i == 0 || !(from_key(sorted[i - 1]) == from_key(sorted[i]))) ? 1u : 0u;
}

// group[i] = inclusive scan of start (1-based step index of value i)
__global__ void cdf_scatter_kernel(const uint64_t* __restrict__ sorted, const uint32_t* __restrict__ start,
                                   const uint32_t* __restrict__ group, uint64_t n, double* __restrict__ out_rate,
                                   double* __restrict__ out_frac, uint64_t* __restrict__ n_steps) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t g = group[i] - 1;
        if (start[i]) out_rate[g] = from_key(sorted[i]);
        if (i + 1 == n || start[i + 1]) out_frac[g] = __ddiv_rn((double)(i + 1), (double)n);
        if (i + 1 == n) *n_steps = group[i];
    }
}

size_t cub_bytes(uint64_t n) {
    size_t sort_b = 0, scan_b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, sort_b, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)n);
    cub::DeviceScan::InclusiveSum(nullptr, scan_b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
    return sort_b > scan_b ? sort_b : scan_b;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace aes

extern "C" {

uint64_t aes_cdf_workspace_bytes(uint64_t n) {
    using namespace aes;
    const uint64_t m = n ? n : 1;
    return align256(8 * m) * 2 + align256(4 * m) * 2 + align256(cub_bytes(m)) + 256;
}

int aes_dev_cdf_stats(const double* rates, uint64_t n, double* out_rate, double* out_frac, uint64_t* n_steps,
                      void* workspace, size_t workspace_bytes, void* stream) {
    using namespace aes;
    if (n == 0) return fail(AES_ERR_INVALID_ARG, "rates must be nonempty");  // bench.cpp:125
    if (!rates || !out_rate || !out_frac || !n_steps || !workspace) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (n >= (1ull << 31)) return fail(AES_ERR_UNSUPPORTED, "cdf_stats: more than 2^31 rates");
    if (workspace_bytes < aes_cdf_workspace_bytes(n)) return fail(AES_ERR_INVALID_ARG, "cdf workspace too small");
    cudaStream_t st = as_stream(stream);
    char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
    uint64_t* keys = reinterpret_cast<uint64_t*>(w);
    w += align256(8 * n);
    uint64_t* sorted = reinterpret_cast<uint64_t*>(w);
    w += align256(8 * n);
    uint32_t* start = reinterpret_cast<uint32_t*>(w);
    w += align256(4 * n);
    uint32_t* group = reinterpret_cast<uint32_t*>(w);
    w += align256(4 * n);
    size_t tmp_b = cub_bytes(n);
    const unsigned grid = grid_for(n, 256, num_sms() * 16);
    cdf_keys_kernel<<<grid, 256, 0, st>>>(rates, n, keys);
    AES_CUDA_TRY(cub::DeviceRadixSort::SortKeys(w, tmp_b, keys, sorted, (int)n, 0, 64, st));
    cdf_starts_kernel<<<grid, 256, 0, st>>>(sorted, n, start);
    tmp_b = cub_bytes(n);
    AES_CUDA_TRY(cub::DeviceScan::InclusiveSum(w, tmp_b, start, group, (int)n, st));
    cdf_scatter_kernel<<<grid, 256, 0, st>>>(sorted, start, group, n, out_rate, out_frac, n_steps);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // extern "C"
