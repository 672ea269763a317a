// Shared device/host helpers for the AES-SpMM sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "aesspmm_cuda.h"

namespace aes {

// ---------------------------------------------------------------------------
// Error plumbing: thread-local message, reference exception strings.
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define AES_CUDA_TRY(expr)                                     \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return ::aes::cuda_fail(_e, #expr); \
    } while (0)

#define AES_TRY(expr)                 \
    do {                              \
        int _s = (expr);              \
        if (_s != AES_OK) return _s;  \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// Table 1 of the paper + Eq. 3, exactly as the reference evaluates them
// (proj/src/sampling.cpp:29-102).  The SAME code runs on the host (scalar API)
// and inside the sampler kernels.
// ---------------------------------------------------------------------------
struct RowParams {
    uint32_t chunk;
    uint32_t cnt;
};

__host__ __device__ __forceinline__ RowParams select_strategy(uint64_t nnz, uint32_t w) {
    if (nnz == 0) return {0u, 0u};
    if (nnz <= (uint64_t)w) return {(uint32_t)nnz, 1u};
    uint32_t c, n;
    if (nnz <= 2ull * w) {
        c = w / 4; n = 4;
    } else if (nnz <= 36ull * w) {
        c = w / 8; n = 8;
    } else if (nnz <= 54ull * w) {
        c = w / 16; n = 16;
    } else {
        c = w / 32; n = 32;
    }
    return {c < 1u ? 1u : c, n > w ? w : n};
}

__host__ __device__ __forceinline__ uint32_t hash_start(uint32_t s, uint64_t nnz, uint32_t chunk) {
    uint64_t range = nnz - (uint64_t)chunk + 1ull;
    uint64_t prod = (uint64_t)s * 1429ull;
    // Same value as the u64 modulo; avoid the 64-bit divide when it cannot matter.
    if (prod < range) return (uint32_t)prod;
    if (range <= 0xffffffffull && prod <= 0xffffffffull)
        return (uint32_t)prod % (uint32_t)range;
    return (uint32_t)(prod % range);
}

// (chunk, cnt) per strategy — sampling.cpp:68-99.
__host__ __device__ __forceinline__ RowParams row_params(uint64_t nnz, uint32_t w, int strategy) {
    if (nnz == 0) return {0u, 0u};
    switch (strategy) {
        case AES_FULL: return {(uint32_t)nnz, 1u};
        case AES_SFS: return {(uint32_t)(nnz < w ? nnz : w), 1u};
        case AES_AFS: return {1u, (uint32_t)(nnz < w ? nnz : w)};
        default: return select_strategy(nnz, w);
    }
}

// Number of entries in RowSamplePlan::starts (sampling.cpp:70-99).
__host__ __device__ __forceinline__ uint32_t row_num_starts(uint64_t nnz, uint32_t w, int strategy,
                                                            RowParams p) {
    if (nnz == 0) return 0;
    if (strategy == AES_FULL || strategy == AES_SFS) return 1;
    if (strategy == AES_AFS) return p.cnt;
    return nnz <= w ? 1u : p.cnt;
}

// starts[s] — sampling.cpp:70-99.
__host__ __device__ __forceinline__ uint32_t row_start(uint64_t nnz, uint32_t w, int strategy,
                                                       RowParams p, uint32_t s) {
    if (strategy == AES_FULL || strategy == AES_SFS) return 0;
    if (strategy == AES_AFS) return (uint32_t)((uint64_t)s * nnz / p.cnt);
    if (nnz <= w) return 0;
    return hash_start(s, nnz, p.chunk);
}

// ---------------------------------------------------------------------------
// (a0, a1) = (RN(a0 + p0), RN(a1 + p1)) as one FADD2: add.rn.f32x2 is two
// independent IEEE round-to-nearest adds.  Feed it scalar FMULs only — ptxas
// 12.9 contracts a packed mul.rn.f32x2 feeding add.rn.f32x2 into FFMA2 (one
// rounding), which would change the result bits (see spmm.cu).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void add2_rn(float& a0, float& a1, float p0, float p1) {
    unsigned long long a, p;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(p) : "f"(p0), "f"(p1));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(p));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}

// ---------------------------------------------------------------------------
// Launch geometry
// ---------------------------------------------------------------------------
// Per-device state: the library may drive several GPUs from one process, so
// SM counts, shared-memory opt-ins and occupancy are cached per device.
constexpr int kMaxDevices = 64;
inline int cur_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
    return d;
}
// SMs of the current device (148 on B200), queried once per device.
inline int num_sms() {
    static int sms[kMaxDevices] = {};
    const int d = cur_device();
    if (sms[d] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
        sms[d] = v > 0 ? v : 148;
    }
    return sms[d];
}

inline unsigned grid_for(uint64_t work, unsigned per_block, unsigned cap = 1u << 30) {
    uint64_t g = (work + per_block - 1) / per_block;
    if (g == 0) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// ---------------------------------------------------------------------------
// Internal launchers shared between translation units.
// ---------------------------------------------------------------------------
// Exclusive scan of per-row counts produced by a functor kind, writing out[n+1].
enum ScanKind : int { kScanSlots = 0, kScanStarts = 1, kScanGcnNnz = 2, kScanExplicit = 3 };
struct ScanArgs {
    const uint64_t* row_ptr;  // row lengths from here
    const uint32_t* col_ind;  // for kScanGcnNnz (diagonal probe)
    uint64_t n;
    uint32_t width;
    int strategy;
    int add_self_loops;
    uint64_t* out;           // n+1
    uint32_t* row_params;    // kScanSlots: optional output; kScanExplicit: input (uint2 per row)
};
int launch_row_scan(int kind, const ScanArgs& a, void* ws, size_t ws_bytes, cudaStream_t st);
// Dense host <-> device copies (hostio.cu): pageable host buffers go through a
// pinned staging ring with multi-threaded host copies; h2d returns once the
// host buffer may be reused, d2h once the host buffer holds the data.
int h2d_dense(const float* h, uint64_t rows, uint64_t cols, float* d, uint64_t ld, cudaStream_t st);
int d2h_dense(const float* d, uint64_t ld, uint64_t rows, uint64_t cols, float* h, cudaStream_t st);
size_t row_scan_workspace_bytes(uint64_t n);

}  // namespace aes
