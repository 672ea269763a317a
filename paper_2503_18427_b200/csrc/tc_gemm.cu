// Fast-mode layer GEMM on Blackwell's 5th-generation tensor cores:
//   H = act(A @ W + bias), A: M x K fp32 (the aggregated features), W: K x N.
//
// OPT-IN, NOT bit-exact: tcgen05.mma.kind::tf32 reads each fp32 operand as
// TF32 (10-bit mantissa) and accumulates in fp32 in TMEM, so results differ
// from the reference's ordered fp32 dense_matmul (proj/src/gnn.cpp:11-31) by
// at most ~2^-9 * sum_k |a_ik| |w_kj| (stated and tested in
// tests/test_gpu_tc_gemm.py).  The exact path stays gemm.cu.
//
// Structure (one persistent CTA per SM, 6 warps):
//   warp 0  TMA producer: W^T (N x K, K-major) once, then 128-row x 32-col
//           A slabs (16 KB, 128-B swizzle) into a 6-stage smem ring;
//   warp 1  MMA issuer (one elected lane): per 128-row tile, K/8 x
//           tcgen05.mma (M=128, N=N_pad, K=8) into one of two TMEM
//           accumulators; tcgen05.commit releases smem slots / signals the
//           epilogue;
//   warps 2-5 epilogue: tcgen05.ld (32 lanes x 8 columns per load) ->
//           bias + ReLU -> global (or every peer replica, see gemm.cu).
// K <= 128 and N <= 128 (the GCN hidden sizes); other shapes use gemm.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "common.cuh"

namespace aes {
namespace {

constexpr int kTileM = 128;
constexpr int kSlabK = 32;                     // fp32 elements per 128-B swizzle row
constexpr int kSlabBytes = kTileM * kSlabK * 4;  // 16 KB
constexpr int kStages = 4;
constexpr int kMaxK = 128, kMaxN = 128;
constexpr int kThreads = 6 * 32;

// Output tensor maps: one per destination replica (own + peers for the fused
// exchange) and, when fused, each destination's arrival counter.
constexpr int kMaxOut = 8;
struct OutMaps {
    CUtensorMap map[kMaxOut];
    unsigned long long* ctr[kMaxOut];
    int n;
};

struct __align__(8) Barriers {
    uint64_t full[kStages];
    uint64_t empty[kStages];
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint64_t w_full;
    uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-B swizzle: LBO = 16 B, SBO =
// 1024 B (8 rows x 128 B), version 1 (sm_100), layout type 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;            // leading byte offset (16 B units)
    d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset
    d |= (uint64_t)1 << 46;            // descriptor version (Blackwell)
    d |= (uint64_t)2 << 61;            // SWIZZLE_128B
    return d;
}

// Instruction descriptor: dense, D = F32, A = B = TF32, both K-major,
// N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t m, uint32_t n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_w,
               const __grid_constant__ OutMaps outs, uint64_t m, uint32_t k_slabs, uint32_t n, uint32_t n_pad,
               uint32_t tmem_cols, const float* __restrict__ bias, int relu) {
    extern __shared__ __align__(1024) unsigned char smem[];
    // layout: [A ring: kStages x 16 KB][W^T: k_slabs x (n_pad x 128 B)]
    //         [output staging: n_slabs x (128 rows x 128 B), 128-B swizzled][barriers]
    unsigned char* a_ring = smem;
    unsigned char* w_smem = smem + kStages * kSlabBytes;
    const uint32_t w_slab_bytes = n_pad * 128;
    const uint32_t n_slabs = (n + 31) / 32;
    unsigned char* out_smem = w_smem + k_slabs * w_slab_bytes;
    Barriers* bars = reinterpret_cast<Barriers*>(out_smem + n_slabs * kSlabBytes);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t tiles = (m + kTileM - 1) / kTileM;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tmem_full[a], 1);
            mbar_init(&bars->tmem_empty[a], 4);
        }
        mbar_init(&bars->w_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: two accumulators of n_pad fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem_base = bars->tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            // W^T once: k_slabs boxes of (32 K x n_pad rows)
            mbar_expect_tx(&bars->w_full, k_slabs * w_slab_bytes);
            for (uint32_t s = 0; s < k_slabs; ++s) tma_load_2d(w_smem + s * w_slab_bytes, &map_w, &bars->w_full, s * kSlabK, 0);
            uint32_t stage = 0, phase = 0;
            for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                for (uint32_t s = 0; s < k_slabs; ++s) {
                    mbar_wait(&bars->empty[stage], phase ^ 1);
                    mbar_expect_tx(&bars->full[stage], kSlabBytes);
                    tma_load_2d(a_ring + stage * kSlabBytes, &map_a, &bars->full[stage], s * kSlabK,
                                (int)(t * kTileM));
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc = idesc_tf32(kTileM, n_pad);
        mbar_wait(&bars->w_full, 0);
        uint32_t stage = 0, phase = 0;
        uint32_t acc = 0, acc_phase = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(&bars->tmem_empty[acc], acc_phase ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tmem_d = tmem_base + acc * n_pad;
            for (uint32_t s = 0; s < k_slabs; ++s) {
                mbar_wait(&bars->full[stage], phase);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const uint32_t a0 = smem_u32(a_ring + stage * kSlabBytes);
                    const uint32_t b0 = smem_u32(w_smem + s * w_slab_bytes);
#pragma unroll
                    for (uint32_t kk = 0; kk < kSlabK / 8; ++kk)  // 8 tf32 = 32 B per UMMA K step
                        mma_tf32(tmem_d, umma_desc_sw128(a0 + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                                 (s | kk) != 0);
                    mma_commit(&bars->empty[stage]);  // smem slot free once these MMAs retire
                }
                __syncwarp();
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) mma_commit(&bars->tmem_full[acc]);
            __syncwarp();
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    } else {
        // epilogue warps 2..5 -> TMEM lane quadrant (warp % 4) = tile rows
        // 32*quad .. +31.  TMEM -> registers -> bias/ReLU -> 128-B-swizzled
        // staging (conflict-free 16-B stores) -> TMA tensor store.
        const uint32_t quad = warp & 3;
        const bool issuer = (warp == 2 && lane == 0);
        const uint32_t r_local = quad * 32 + lane;
        uint32_t acc = 0, acc_phase = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(&bars->tmem_full[acc], acc_phase);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // the previous tile's TMA store must have finished reading staging
            if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            asm volatile("bar.sync 1, 128;" ::: "memory");
            for (uint32_t s = 0; s < n_slabs; ++s) {
                uint32_t r[32];
                tmem_ld32(tmem_base + ((quad * 32) << 16) + acc * n_pad + s * 32, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                unsigned char* slab = out_smem + s * kSlabBytes + r_local * 128;
#pragma unroll
                for (int c = 0; c < 8; ++c) {  // 16-B chunk c of this row, swizzled by row % 8
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t col = s * 32 + c * 4 + j;
                        float x = __uint_as_float(r[c * 4 + j]);
                        if (bias && col < n) x = __fadd_rn(x, bias[col]);
                        if (relu) x = (x < 0.f) ? 0.f : x;
                        v[j] = x;
                    }
                    *reinterpret_cast<float4*>(slab + ((c ^ (r_local & 7)) * 16)) = make_float4(v[0], v[1], v[2], v[3]);
                }
            }
            // TMEM accumulator can be reused as soon as it is in registers/smem
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->tmem_empty[acc]);
            // make the generic-proxy smem writes visible to the TMA (async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (issuer) {
                for (uint32_t s = 0; s < n_slabs; ++s)
                    for (int d = 0; d < outs.n; ++d)  // own replica and every peer's, over NVLink
                        tma_store_2d(&outs.map[d], out_smem + s * kSlabBytes, (int)(s * 32), (int)(t * kTileM));
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
        if (issuer) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // all tile writes complete
            if (outs.ctr[0]) {
                // publish this CTA's tiles to every destination (fused exchange):
                // async-proxy writes -> generic proxy -> system-scope release
                uint64_t mine = 0;
                for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) ++mine;
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __threadfence_system();
                for (int d = 0; d < outs.n; ++d)
                    asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(outs.ctr[d]), "l"(mine) : "memory");
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
    }
}

// W (K x N, ld ldw) -> W^T (n_pad x k_pad, K-major), zero padded.
__global__ void transpose_pad_kernel(const float* __restrict__ w, uint32_t k, uint32_t n, uint64_t ldw, float* __restrict__ wt,
                                     uint32_t n_pad, uint32_t k_pad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_pad * k_pad; i += gridDim.x * blockDim.x) {
        const uint32_t r = i / k_pad, c = i % k_pad;  // r: output column j, c: k
        wt[i] = (r < n && c < k) ? w[(uint64_t)c * ldw + r] : 0.f;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int make_map(CUtensorMap* map, const float* base, uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
             uint32_t box_outer) {
    auto fn = encode_fn();
    if (!fn) return fail(AES_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld_elems * 4};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(AES_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return AES_OK;
}

int launch_tc_gemm(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w, uint64_t n, uint64_t ldw,
                   const float* bias, int relu, float* const* dsts, unsigned long long* const* counters, int n_dst,
                   uint64_t row_offset, uint64_t ldh, float* wt_scratch, cudaStream_t st) {
    if (m == 0 || n == 0) return AES_OK;
    if (k == 0 || k > (uint64_t)kMaxK || n > (uint64_t)kMaxN)
        return fail(AES_ERR_UNSUPPORTED, "tcgen05 GEMM takes 1 <= K <= 128 and N <= 128");
    if (n_dst < 1 || n_dst > kMaxOut) return fail(AES_ERR_INVALID_ARG, "1..8 output replicas");
    if (lda % 4 || (uintptr_t)a % 16) return fail(AES_ERR_UNSUPPORTED, "A rows must be 16-B aligned");
    const uint32_t k_slabs = (uint32_t)((k + kSlabK - 1) / kSlabK);
    const uint32_t k_pad = k_slabs * kSlabK;
    const uint32_t n_pad = (uint32_t)((n + 15) / 16 * 16);  // UMMA N: multiple of 16 keeps TMEM columns aligned
    uint32_t tmem_cols = 32;
    while (tmem_cols < 2 * n_pad) tmem_cols <<= 1;
    if (!wt_scratch) return fail(AES_ERR_INVALID_ARG, "W^T scratch (n_pad * k_pad floats) required");
    transpose_pad_kernel<<<64, 256, 0, st>>>(w, (uint32_t)k, (uint32_t)n, ldw, wt_scratch, n_pad, k_pad);
    CUtensorMap map_a, map_w;
    AES_TRY(make_map(&map_a, a, k, m, lda, kSlabK, kTileM));
    AES_TRY(make_map(&map_w, wt_scratch, k_pad, n_pad, k_pad, kSlabK, n_pad));
    OutMaps outs{};
    outs.n = n_dst;
    for (int d = 0; d < n_dst; ++d) {
        float* h = dsts[d] + row_offset * ldh;
        if (ldh % 4 || (uintptr_t)h % 16) return fail(AES_ERR_UNSUPPORTED, "H rows must be 16-B aligned");
        AES_TRY(make_map(&outs.map[d], h, n, m, ldh, kSlabK, kTileM));
        outs.ctr[d] = counters ? counters[d] : nullptr;
    }
    const uint32_t n_slabs = (uint32_t)((n + 31) / 32);
    const size_t smem = (size_t)kStages * kSlabBytes + (size_t)k_slabs * n_pad * 128 + (size_t)n_slabs * kSlabBytes +
                        sizeof(Barriers) + 1024;
    static bool attr_dev[kMaxDevices] = {};
    bool& attr = attr_dev[cur_device()];
    if (!attr) {
        AES_CUDA_TRY(cudaFuncSetAttribute(
            tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
            (int)(kStages * kSlabBytes + 4 * kMaxN * 128 + 4 * kSlabBytes + sizeof(Barriers) + 1024)));
        attr = true;
    }
    const uint64_t tiles = (m + kTileM - 1) / kTileM;
    const unsigned grid = (unsigned)(tiles < (uint64_t)num_sms() ? tiles : (uint64_t)num_sms());
    tc_gemm_kernel<<<grid, kThreads, smem, st>>>(map_a, map_w, outs, m, k_slabs, (uint32_t)n, n_pad, tmem_cols, bias,
                                                 relu);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace
}  // namespace aes

extern "C" int aes_dev_gemm_tf32(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w, uint64_t n,
                                 uint64_t ldw, const float* bias, int relu, float* h, uint64_t ldh, float* wt_scratch,
                                 void* stream) {
    float* dsts[1] = {h};
    return aes::launch_tc_gemm(a, m, k, lda, w, n, ldw, bias, relu, dsts, nullptr, 1, 0, ldh, wt_scratch,
                               aes::as_stream(stream));
}

extern "C" int aes_dev_gemm_tf32_bcast(const float* a, uint64_t m, uint64_t k, uint64_t lda, const float* w,
                                       uint64_t n, uint64_t ldw, const float* bias, int relu, float* const* dsts,
                                       unsigned long long* const* counters, int n_dst, uint64_t row_offset,
                                       uint64_t ldh, float* wt_scratch, void* stream) {
    return aes::launch_tc_gemm(a, m, k, lda, w, n, ldw, bias, relu, dsts, counters, n_dst, row_offset, ldh,
                               wt_scratch, aes::as_stream(stream));
}

extern "C" uint64_t aes_gemm_tf32_ctas(uint64_t m) {
    // arrivals per destination = 128-row tiles this launch stores
    return (m + aes::kTileM - 1) / aes::kTileM;
}

extern "C" uint64_t aes_gemm_tf32_scratch_floats(uint64_t k, uint64_t n) {
    const uint64_t k_pad = (k + 31) / 32 * 32, n_pad = (n + 15) / 16 * 16;
    return k_pad * n_pad;
}
