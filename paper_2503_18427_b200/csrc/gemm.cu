// Ordered fp32 layer GEMM + bias + ReLU epilogue for the GCN layer driver,
// optionally fused with the layer's exchange: the epilogue stores every output
// tile into ALL ranks' next-layer replicas over peer memory (NVLink P2P
// stores to CUDA-IPC-mapped buffers) and each CTA then publishes a
// system-scope arrival on every destination's counter — the all-gather
// disappears into the GEMM (no NCCL call, transfer overlapped tile by tile).
//
// Bit-exact with the reference dense_matmul (proj/src/gnn.cpp:11-31): every
// output element accumulates k in ascending order as acc = RN(acc + RN(a*w))
// from +0.0f, skipping a == 0 as the reference does.  When W is known to be
// finite the skip is provably result-neutral (acc is never -0 and RN(0*w) is
// +-0), so the `finite_w` form drops the select.  Bias then ReLU follow
// gnn.cpp:41-52 with std::max(v, 0.0f) semantics ((v < 0) ? 0 : v).  Tensor
// cores are not used: their reduction order and fused rounding cannot
// reproduce the reference's result bits.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"
#include "minmax.cuh"

namespace aes {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;
constexpr int kThreads = (BM / TM) * (BN / TN);  // 256
constexpr int kMaxDst = 16;

struct Bcast {
    float* dst[kMaxDst];                   // replica base pointers (own + peers)
    unsigned long long* ctr[kMaxDst];      // arrival counters (one per destination rank)
    const uint8_t* need[kMaxDst];          // halo masks: row r goes to d only if need[d][r] (null: every row)
    int n;
    uint64_t row_off;                      // this shard's first row in the replica
    MinMax* fit;                           // fused fit_params: one (min, max) partial per CTA (null: off)
    uint64_t fit_off;                      // partial index of this launch's first CTA
};

template <bool SKIP, bool BCAST, bool FIT = false, int TNV = 8>
__global__ void __launch_bounds__(kThreads, 2)
gemm_ordered_kernel(const float* __restrict__ a, uint64_t m, uint64_t k, uint64_t lda,
                    const float* __restrict__ w, uint64_t n, uint64_t ldw, const float* __restrict__ bias,
                    int relu, float* __restrict__ h, uint64_t ldh, Bcast bc) {
    // TNV = 8: 128 x 128 tiles; TNV = 4: 128 x 64 tiles for narrow outputs (n <= 64)
    constexpr int TN = TNV, BN = 16 * TNV, kRW = BK * BN / kThreads;
    // thread tx owns column quads {q * QS + 4 tx .. +3}: a half-warp's W reads
    // are 256 contiguous bytes (with 8 consecutive columns per thread they
    // were 4-way bank-conflicted: 160 M conflicts per products launch)
    constexpr int QS = BN / (TN / 4);
    __shared__ __align__(16) float As[2][BK][BM + 4];  // +4: conflict-free transposed stores
    __shared__ __align__(16) float Ws[2][BK][BN];
    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const uint64_t m0 = (uint64_t)blockIdx.y * BM, n0 = (uint64_t)blockIdx.x * BN;

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    // staging: A tile BM x BK (4 elements / thread), W tile BK x BN (4 / thread)
    float ra[4], rw[kRW];
    // interior tiles (every row, column and k of the slab in range) load
    // without bounds checks from per-thread base pointers (3.35 -> 3.09 ms
    // on the products layer GEMM: the checks were ~8 % of the issue slots)
    const bool full_mn = m0 + BM <= m && n0 + BN <= n;
    const float* pa = a + (m0 + tid / BK) * lda + tid % BK;            // element tid + 256 r: row + 32 r
    const float* pw = w + (uint64_t)(tid / BN) * ldw + n0 + tid % BN;  // k row + 2 r
    auto load_tiles = [&](uint64_t k0) {
        if (full_mn && k0 + BK <= k) {
#pragma unroll
            for (int r = 0; r < 4; ++r) ra[r] = __ldg(pa + (uint64_t)(r * kThreads / BK) * lda + k0);
#pragma unroll
            for (int r = 0; r < kRW; ++r) rw[r] = __ldg(pw + (k0 + (uint64_t)(r * kThreads / BN)) * ldw);
            return;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + r * kThreads;      // 0..1023
            const int mm = e / BK, kk = e % BK;
            const uint64_t gm = m0 + mm, gk = k0 + kk;
            ra[r] = (gm < m && gk < k) ? __ldg(a + gm * lda + gk) : 0.f;  // zero fill is neutral
        }
#pragma unroll
        for (int r = 0; r < kRW; ++r) {
            const int e = tid + r * kThreads;
            const int kw = e / BN, nn = e % BN;
            const uint64_t gkw = k0 + kw, gn = n0 + nn;
            rw[r] = (gkw < k && gn < n) ? __ldg(w + gkw * ldw + gn) : 0.f;
        }
    };
    auto store_tiles = [&](int buf) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int e = tid + r * kThreads;
            As[buf][e % BK][e / BK] = ra[r];
        }
#pragma unroll
        for (int r = 0; r < kRW; ++r) {
            const int e = tid + r * kThreads;
            Ws[buf][e / BN][e % BN] = rw[r];
        }
    };

    load_tiles(0);
    store_tiles(0);
    __syncthreads();
    int buf = 0;
    for (uint64_t k0 = 0; k0 < k; k0 += BK) {
        const bool more = k0 + BK < k;
        if (more) load_tiles(k0 + BK);  // prefetch the next K slab into registers
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * TM]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * TM + 4]);
            const float av[TM] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
            float wv[TN];
#pragma unroll
            for (int q = 0; q < TN / 4; ++q) {
                const float4 w4 = *reinterpret_cast<const float4*>(&Ws[buf][kk][q * QS + 4 * tx]);
                wv[4 * q] = w4.x;
                wv[4 * q + 1] = w4.y;
                wv[4 * q + 2] = w4.z;
                wv[4 * q + 3] = w4.w;
            }
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                // scalar FMULs, paired adds (FADD2: two independent IEEE RN
                // adds): 3 issue slots per 2 MACs instead of 4 — the kernel
                // is issue-bound (85 % issue, 70 % FMA pipe): 3.09 -> 2.86 ms
                if (SKIP) {
                    const bool skip = av[i] == 0.f;
#pragma unroll
                    for (int j = 0; j < TN; j += 2) {
                        float s0 = acc[i][j], s1 = acc[i][j + 1];
                        add2_rn(s0, s1, __fmul_rn(av[i], wv[j]), __fmul_rn(av[i], wv[j + 1]));
                        acc[i][j] = skip ? acc[i][j] : s0;
                        acc[i][j + 1] = skip ? acc[i][j + 1] : s1;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < TN; j += 2)
                        add2_rn(acc[i][j], acc[i][j + 1], __fmul_rn(av[i], wv[j]), __fmul_rn(av[i], wv[j + 1]));
                }
            }
        }
        if (more) {
            store_tiles(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }

    // epilogue: bias, ReLU, store (to every replica when broadcasting)
    // fused fit_params over the output (row-major index row * n + col, the
    // order quantize.cpp:14-19 scans): this thread meets its elements in
    // increasing index order (quads ascend), so strict compares keep first
    // occurrences
    MinMax fm{INFINITY, -INFINITY, ~0ull, ~0ull, 0u};
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const uint64_t gm = m0 + ty * TM + i;
        if (gm >= m) continue;
        float v[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const uint64_t gn = n0 + (j >> 2) * QS + 4 * tx + (j & 3);
            float x = acc[i][j];
            if (bias && gn < n) x = __fadd_rn(x, bias[gn]);
            if (relu) x = (x < 0.f) ? 0.f : x;
            v[j] = x;
            if (FIT && gn < n) fit_elem(fm, x, (bc.row_off + gm) * n + gn);
        }
        const int nd = BCAST ? bc.n : 1;
        for (int d = 0; d < nd; ++d) {
            if (BCAST && bc.need[d] && !bc.need[d][bc.row_off + gm]) continue;  // halo: d never reads this row
            float* row = BCAST ? bc.dst[d] + (bc.row_off + gm) * ldh : h + gm * ldh;
#pragma unroll
            for (int q = 0; q < TN / 4; ++q) {
                const uint64_t gq = n0 + q * QS + 4 * tx;
                if (gq + 4 <= n && ldh % 4 == 0) {
                    *reinterpret_cast<float4*>(row + gq) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2],
                                                                       v[4 * q + 3]);
                } else {
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        if (gq + r < n) row[gq + r] = v[4 * q + r];
                }
            }
        }
    }
    if (FIT) {  // one partial per CTA
        fm = block_reduce<kThreads>(fm);
        if (tid == 0) bc.fit[bc.fit_off + (uint64_t)blockIdx.y * gridDim.x + blockIdx.x] = fm;
    }
    if (BCAST) {
        // publish this CTA's tile to every destination: the barrier orders the
        // CTA's stores before thread 0's system-scope fence (cumulativity),
        // then one release-add per destination counter.
        __syncthreads();
        if (tid == 0) {
            __threadfence_system();
            for (int d = 0; d < bc.n; ++d)
                asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(bc.ctr[d]) : "memory");
        }
    }
}

// Spins with a 60 s deadline: a peer that never arrives (a crashed rank, a
// miscounted arrival) turns into a launch error instead of a hung GPU.
constexpr unsigned long long kWaitDeadlineNs = 60ull * 1000 * 1000 * 1000;

__global__ void wait_counter_kernel(const unsigned long long* ctr, unsigned long long target) {
    unsigned long long v, t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        if (v >= target) return;
        __nanosleep(64);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > kWaitDeadlineNs) {
            printf("aes_dev_wait_counter: %llu of %llu arrivals after 60 s\n", v, target);
            __trap();
        }
    }
}

// One thread: make this rank's prior work visible system-wide, then bump
// every rank's counter (a device-side cross-rank barrier arrival).
__global__ void signal_all_kernel(unsigned long long* const* ctrs, int n) {
    __threadfence_system();
    for (int d = 0; d < n; ++d) asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(ctrs[d]) : "memory");
}

struct CtrArray {
    unsigned long long* p[kMaxDst];
};
__global__ void signal_all_arr_kernel(CtrArray a, int n) {
    __threadfence_system();
    for (int d = 0; d < n; ++d) asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(a.p[d]) : "memory");
}

__global__ void all_finite_kernel(const float* __restrict__ x, uint64_t count, unsigned int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        if (!isfinite(x[i])) atomicOr(bad, 1u);
}

inline uint64_t gemm_tile_n(uint64_t n) { return n <= 64 ? 64 : 128; }

template <bool SKIP, bool BCAST, bool FIT = false>
int launch(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w, uint64_t n, uint64_t ldw,
           const float* bias, int relu, float* h, uint64_t ldh, const Bcast& bc, cudaStream_t st) {
    // narrow outputs (a GCN's last layer: 40 classes on arxiv) on 128 x 64
    // tiles: half the dead columns of a 128-wide tile
    const uint64_t bn = gemm_tile_n(n);
    const unsigned gx = (unsigned)((n + bn - 1) / bn);
    const uint64_t rows_per = (uint64_t)65535 * BM;  // grid.y limit
    for (uint64_t r0 = 0; r0 < m; r0 += rows_per) {
        const uint64_t mm = m - r0 < rows_per ? m - r0 : rows_per;
        Bcast b2 = bc;
        b2.row_off += r0;
        b2.fit_off = (r0 / BM) * gx;  // partials of the earlier row chunks
        dim3 grid(gx, (unsigned)((mm + BM - 1) / BM));
        if (bn == 64)
            gemm_ordered_kernel<SKIP, BCAST, FIT, 4><<<grid, kThreads, 0, st>>>(
                a + r0 * lda, mm, k, lda, w, n, ldw, bias, relu, h ? h + r0 * ldh : nullptr, ldh, b2);
        else
            gemm_ordered_kernel<SKIP, BCAST, FIT, 8><<<grid, kThreads, 0, st>>>(
                a + r0 * lda, mm, k, lda, w, n, ldw, bias, relu, h ? h + r0 * ldh : nullptr, ldh, b2);
    }
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace
}  // namespace aes

extern "C" {

int aes_dev_gemm_bias_act(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w, uint64_t n,
                          uint64_t ldw, const float* bias, int relu, float* h, uint64_t ldh, void* stream) {
    using namespace aes;
    if (m == 0 || n == 0) return AES_OK;
    if (lda < k || ldw < n || ldh < n) return fail(AES_ERR_INVALID_ARG, "leading dimension too small");
    Bcast bc{};
    return launch<true, false>(a, m, k, lda, w, n, ldw, bias, relu, h, ldh, bc, as_stream(stream));
}

int aes_dev_gemm_bias_act_ex(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w, uint64_t n,
                             uint64_t ldw, const float* bias, int relu, int finite_w, float* const* dsts,
                             unsigned long long* const* counters, int n_dst, uint64_t row_offset, uint64_t ldh,
                             void* stream) {
    return aes_dev_gemm_bias_act_halo(a, m, k, lda, w, n, ldw, bias, relu, finite_w, dsts, counters, nullptr, n_dst,
                                      row_offset, ldh, stream);
}

int aes_dev_gemm_bias_act_halo(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w, uint64_t n,
                               uint64_t ldw, const float* bias, int relu, int finite_w, float* const* dsts,
                               unsigned long long* const* counters, const uint8_t* const* need, int n_dst,
                               uint64_t row_offset, uint64_t ldh, void* stream) {
    using namespace aes;
    if (n_dst < 1 || n_dst > kMaxDst) return fail(AES_ERR_INVALID_ARG, "1..16 destinations");
    if (lda < k || ldw < n || ldh < n) return fail(AES_ERR_INVALID_ARG, "leading dimension too small");
    if (n == 0) return AES_OK;
    Bcast bc{};
    bc.n = n_dst;
    bc.row_off = row_offset;
    for (int d = 0; d < n_dst; ++d) {
        bc.dst[d] = dsts[d];
        bc.ctr[d] = counters ? counters[d] : nullptr;
        bc.need[d] = need ? need[d] : nullptr;
    }
    cudaStream_t st = as_stream(stream);
    const bool bcast = counters != nullptr;
    if (!bcast) {
        if (n_dst != 1) return fail(AES_ERR_INVALID_ARG, "several destinations need arrival counters");
        float* h = dsts[0] + row_offset * ldh;
        if (m == 0) return AES_OK;
        return finite_w ? launch<false, false>(a, m, k, lda, w, n, ldw, bias, relu, h, ldh, bc, st)
                        : launch<true, false>(a, m, k, lda, w, n, ldw, bias, relu, h, ldh, bc, st);
    }
    if (m == 0) return AES_OK;  // nothing to publish: arrival targets count launched CTAs only
    return finite_w ? launch<false, true>(a, m, k, lda, w, n, ldw, bias, relu, nullptr, ldh, bc, st)
                    : launch<true, true>(a, m, k, lda, w, n, ldw, bias, relu, nullptr, ldh, bc, st);
}

int aes_dev_gemm_bias_act_fit(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w, uint64_t n,
                              uint64_t ldw, const float* bias, int relu, int finite_w, float* h, uint64_t ldh,
                              void* fit_partials, void* stream) {
    using namespace aes;
    if (lda < k || ldw < n || ldh < n) return fail(AES_ERR_INVALID_ARG, "leading dimension too small");
    if (!h || !fit_partials) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (m == 0 || n == 0) return AES_OK;
    Bcast bc{};
    bc.n = 1;
    bc.fit = static_cast<MinMax*>(fit_partials);
    cudaStream_t st = as_stream(stream);
    return finite_w ? launch<false, false, true>(a, m, k, lda, w, n, ldw, bias, relu, h, ldh, bc, st)
                    : launch<true, false, true>(a, m, k, lda, w, n, ldw, bias, relu, h, ldh, bc, st);
}

uint64_t aes_gemm_fit_partial_bytes(uint64_t m, uint64_t n) { return aes_gemm_ctas(m, n) * sizeof(aes::MinMax); }

uint64_t aes_gemm_ctas(uint64_t m, uint64_t n) {
    if (m == 0 || n == 0) return 0;
    const uint64_t bn = aes::gemm_tile_n(n);
    return ((n + bn - 1) / bn) * ((m + aes::BM - 1) / aes::BM);
}

int aes_dev_wait_counter(const unsigned long long* counter, unsigned long long target, void* stream) {
    aes::wait_counter_kernel<<<1, 1, 0, aes::as_stream(stream)>>>(counter, target);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_signal_all(unsigned long long* const* counters, int n, void* stream) {
    using namespace aes;
    if (n < 1 || n > kMaxDst) return fail(AES_ERR_INVALID_ARG, "1..16 counters");
    CtrArray a{};
    for (int d = 0; d < n; ++d) a.p[d] = counters[d];
    signal_all_arr_kernel<<<1, 1, 0, as_stream(stream)>>>(a, n);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_all_finite(const float* x, uint64_t count, unsigned int* bad_flag, void* stream) {
    using namespace aes;
    cudaStream_t st = as_stream(stream);
    AES_CUDA_TRY(cudaMemsetAsync(bad_flag, 0, sizeof(unsigned int), st));
    if (count) all_finite_kernel<<<grid_for(count, 256, num_sms() * 8), 256, 0, st>>>(x, count, bad_flag);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // extern "C"
