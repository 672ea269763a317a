// int8 layer exchange over peer memory (fused form).
//
// A hidden GCN layer's output H_l travels between ranks as 8-bit codes with
// ONE set of global quantization params, exactly the reference composition
// dequantize(quantize(H_l, fit_params(H_l))) (proj/src/quantize.cpp:11-64,
// proj/src/gnn.cpp:66-78).  Everything stays on the device — no host fold, no
// NCCL call, no synchronisation:
//
//   1. each rank reduces its own rows with aes_dev_fit_params (first
//      occurrence, non-finite flag);
//   2. aes_dev_publish_params stores that (min, max, flag) triple into slot
//      `rank` of every rank's parameter array (NVLink P2P stores) and bumps
//      every rank's parameter counter (system-scope release);
//   3. after aes_dev_wait_counter sees all ranks, aes_dev_fold_params_lut
//      folds the triples in rank order with the reference's strict < / >
//      rule (quantize.cpp:14-19 — equal to the serial scan of the
//      concatenated rows, +-0 ties included), and builds the exact 256-entry
//      dequantization table of the folded params (quantize.cpp:53-64);
//   4. aes_dev_quantize_bcast encodes this rank's rows with the folded params
//      read from device memory (quantize.cpp:23-51 arithmetic, fp64 with
//      explicit roundings) and stores the codes straight into every rank's
//      code replica, each CTA then publishing one arrival per destination;
//   5. the next layer aggregates the replica with the fused-dequant SpMM
//      (aes_dev_spmm_q8_ex) once all code arrivals are in.
//
// Four times fewer exchange bytes than the fp32 replica broadcast.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "quantize.cuh"

namespace aes {
namespace {

constexpr int kMaxRanks = 16;
constexpr int kQuantRows = 256;     // rows per quantize CTA (one system-scope arrival each)
constexpr int kQuantThreads = 256;

struct PtrArr {
    void* p[kMaxRanks];
};

__device__ __forceinline__ void publish_release(unsigned long long* ctr) {
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
}

// One thread.  Status flag (int bits of slot 2): 0 ok, 1 non-finite, 2 empty shard.
__global__ void publish_params_kernel(const float* __restrict__ res, int empty, int rank, PtrArr params, PtrArr ctrs,
                                      int n) {
    float lo = 0.f, hi = 0.f;
    uint32_t flag = 2u;
    if (!empty) {
        lo = res[0];
        hi = res[1];
        flag = reinterpret_cast<const uint32_t*>(res)[2] ? 1u : 0u;
    }
    for (int d = 0; d < n; ++d) {
        float* slot = static_cast<float*>(params.p[d]) + 4 * rank;
        slot[0] = lo;
        slot[1] = hi;
        reinterpret_cast<uint32_t*>(slot)[2] = flag;
    }
    __threadfence_system();
    for (int d = 0; d < n; ++d) publish_release(static_cast<unsigned long long*>(ctrs.p[d]));
}

// One block of 256 threads: thread 0 folds, every thread writes one LUT entry.
// out: [lo, hi, status(int bits), 0]; status 0 ok, 1 NonFinite, 2 EmptyMatrix.
__global__ void fold_params_lut_kernel(const float* __restrict__ params, int world, uint32_t levels,
                                       float* __restrict__ out, float* __restrict__ lut) {
    __shared__ float s_lo, s_hi;
    __shared__ uint32_t s_status;
    if (threadIdx.x == 0) {
        // the params were written by peers and published with release-adds
        // the stream already acquired (aes_dev_wait_counter): plain loads
        const volatile float* pv = params;
        bool any = false, bad = false;
        float lo = 0.f, hi = 0.f;
        for (int r = 0; r < world; ++r) {
            const float rl = pv[4 * r], rh = pv[4 * r + 1];
            const uint32_t f = reinterpret_cast<const volatile uint32_t*>(pv)[4 * r + 2];
            if (f == 1u) bad = true;
            if (f != 0u) continue;
            if (!any) {
                lo = rl;
                hi = rh;
                any = true;
            } else {
                lo = rl < lo ? rl : lo;  // strict: an equal later value never replaces
                hi = rh > hi ? rh : hi;
            }
        }
        const uint32_t status = bad ? 1u : (any ? 0u : 2u);
        if (status) lo = hi = 0.f;
        s_lo = lo;
        s_hi = hi;
        s_status = status;
        out[0] = lo;
        out[1] = hi;
        reinterpret_cast<uint32_t*>(out)[2] = status;
        out[3] = 0.f;
    }
    __syncthreads();
    // the exact table of aes_dev_dequant_lut: float(double(q) * step + double(lo))
    const double dlo = (double)s_lo;
    const double step = __ddiv_rn(__dsub_rn((double)s_hi, dlo), (double)levels);
    const uint32_t q = threadIdx.x;
    lut[q] = q <= levels ? __double2float_rn(__dadd_rn(__dmul_rn((double)q, step), dlo)) : 0.f;
}

// quantize(x, params) for rows [0, rows) of this shard, codes stored into
// every destination replica at rows row_off.., then one arrival per CTA per
// destination.  lohi = fold_params_lut's params
// (device); codes through quantize.cuh's fp32 fast path with the exact fp64
// fallback.  Warp per row, lane per 4 columns (float4 loads when the rows are
// 16-B aligned).
__global__ void __launch_bounds__(kQuantThreads)
quantize_bcast_kernel(const float* __restrict__ x, uint64_t rows, uint32_t cols, uint64_t ldx,
                      const float* __restrict__ lohi, uint32_t levels, PtrArr dst, uint64_t row_off, uint64_t ldq,
                      PtrArr ctrs, PtrArr need, int n, bool vec) {
    const uint64_t r0 = (uint64_t)blockIdx.x * kQuantRows;
    const uint32_t nr = (uint32_t)min((uint64_t)kQuantRows, rows - r0);
    const QuantParamsDev p = quant_params(lohi[0], lohi[1], levels);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t c4n = (cols + 3) / 4;
    for (uint32_t rr = warp; rr < nr; rr += kQuantThreads / 32) {
        const uint64_t r = r0 + rr;
        const float* xr = x + r * ldx;
        for (uint32_t c4 = lane; c4 < c4n; c4 += 32) {
            const uint32_t c = c4 * 4;
            float v[4];
            if (vec) {
                const float4 t = __ldcs(reinterpret_cast<const float4*>(xr + c));
                v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = c + i < cols ? __ldcs(xr + c + i) : 0.f;
            }
            uint32_t packed = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (c + i < cols) packed |= quant_code(v[i], p) << (8 * i);
            for (int d = 0; d < n; ++d) {
                const uint8_t* nd = static_cast<const uint8_t*>(need.p[d]);
                if (nd && !nd[row_off + r]) continue;  // halo: d never reads this row
                uint8_t* row = static_cast<uint8_t*>(dst.p[d]) + (row_off + r) * ldq;
                if (c + 4 <= cols) {
                    *reinterpret_cast<uint32_t*>(row + c) = packed;  // ldq % 16 == 0, c % 4 == 0
                } else {
                    for (uint32_t i = 0; c + i < cols; ++i) row[c + i] = (uint8_t)(packed >> (8 * i));
                }
            }
        }
    }
    // publish: the barrier orders every thread's stores before thread 0's
    // system-scope fence (cumulativity), then one release-add per destination
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int d = 0; d < n; ++d) publish_release(static_cast<unsigned long long*>(ctrs.p[d]));
    }
}

}  // namespace
}  // namespace aes

extern "C" {

int aes_dev_publish_params(const float* fit_result, int empty, int rank, float* const* peer_params,
                           unsigned long long* const* peer_counters, int world, void* stream) {
    using namespace aes;
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
        return fail(AES_ERR_INVALID_ARG, "1..16 ranks, 0 <= rank < world");
    if (!empty && !fit_result) return fail(AES_ERR_INVALID_ARG, "null fit result");
    PtrArr p{}, c{};
    for (int d = 0; d < world; ++d) {
        p.p[d] = peer_params[d];
        c.p[d] = peer_counters[d];
    }
    publish_params_kernel<<<1, 1, 0, as_stream(stream)>>>(fit_result, empty, rank, p, c, world);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_fold_params_lut(const float* params, int world, uint32_t bits, float* out, float* lut, void* stream) {
    using namespace aes;
    if (world < 1 || world > kMaxRanks) return fail(AES_ERR_INVALID_ARG, "1..16 ranks");
    if (bits < 1 || bits > 8) return fail(AES_ERR_UNSUPPORTED, "LUT needs bits <= 8");
    if (!out || !lut) return fail(AES_ERR_INVALID_ARG, "null output");
    fold_params_lut_kernel<<<1, 256, 0, as_stream(stream)>>>(params, world, (1u << bits) - 1u, out, lut);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

uint64_t aes_quantize_bcast_ctas(uint64_t rows) { return (rows + aes::kQuantRows - 1) / aes::kQuantRows; }

int aes_dev_quantize_bcast(const float* x, uint64_t rows, uint64_t cols, uint64_t ldx, const float* lohi,
                           uint32_t bits, uint8_t* const* dst_codes, uint64_t row_off, uint64_t ldq,
                           unsigned long long* const* peer_counters, const uint8_t* const* need, int world,
                           void* stream) {
    using namespace aes;
    if (world < 1 || world > kMaxRanks) return fail(AES_ERR_INVALID_ARG, "1..16 ranks");
    if (bits < 1 || bits > 8) return fail(AES_ERR_UNSUPPORTED, "int8 exchange needs bits <= 8");
    if (ldq % 16 != 0 || ldq < cols || ldx < cols) return fail(AES_ERR_INVALID_ARG, "ldq % 16 == 0, ld >= cols");
    const uint64_t ctas = aes_quantize_bcast_ctas(rows);
    if (ctas == 0) return AES_OK;
    if (ctas >= (1ull << 31)) return fail(AES_ERR_INVALID_ARG, "too many rows");
    PtrArr dp{}, cp{}, np_{};
    for (int d = 0; d < world; ++d) {
        dp.p[d] = dst_codes[d];
        cp.p[d] = peer_counters[d];
        np_.p[d] = need ? const_cast<uint8_t*>(need[d]) : nullptr;
    }
    if (cols >= (1ull << 32)) return fail(AES_ERR_INVALID_ARG, "too many columns");
    // rows 16-B aligned and padded to whole float4s: vector loads
    const bool vec = ldx % 4 == 0 && (uintptr_t)x % 16 == 0 && ldx >= (cols + 3) / 4 * 4;
    quantize_bcast_kernel<<<(unsigned)ctas, kQuantThreads, 0, as_stream(stream)>>>(
        x, rows, (uint32_t)cols, ldx, lohi, (1u << bits) - 1u, dp, row_off, ldq, cp, np_, world, vec);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // extern "C"
