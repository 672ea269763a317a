// int8 gather-SpMM with TMA row gathers (sm_100a `tile::gather4`).
//
// Same slot order and accumulation as the cp.async batch kernel in spmm.cu
// (bit-exact with the reference: acc = RN(acc + RN(v * d(q))) per output
// element in slot order, proj/src/spmm.cpp:77-88 over dequantize(Q),
// quantize.cpp:53-64), but the code rows reach shared memory through the
// tensor-memory accelerator: ONE elected lane issues
//     cp.async.bulk.tensor.2d...tile::gather4 [ring], [map, {x, c0, c1, c2, c3}], [mbar]
// per four slots (4 x 128 code bytes), and the warp waits on the batch's
// mbarrier.  The per-lane LDGSTS of the batch kernel (address math, 16-B
// copies, 1.8 shared-memory wavefronts per slot through the LSU data pipe,
// which ncu showed at 86 % — the limiter) disappears; the LSU is left with
// the decode reads.  Columns past F come back zero-filled (tensor-map bounds),
// so partial column tiles need no byte counts.
//
// Decodes (template DEC):
//   0  exact: 256-entry table replicated per lane, entry q at q*256 + 4*lane,
//      one PRMT builds (q << 8 | 4*lane) and one LDS reads it (bank = lane);
//      the shared offset is an ordinary array index (no assumption about
//      where the dynamic window starts)
//   1  fast mode, per-feature affine codes (affine.cu): PRMT into 2^23 + q,
//      FADD2 removes 2^23, FFMA2 accumulates v*q; C = s_j * acc + m_j * sum v
//
// Schedule: warps walk 32-row groups grid-stride (persistent CTAs: the table
// is filled once per CTA); a group's slots stream through a 16-slot ring per
// warp (4 TMA batches of 4 slots, one mbarrier each); slot metadata goes
// through cp.async two rounds ahead, row ends through shared memory.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <string>

#include "common.cuh"

namespace aes {
namespace {

constexpr int kQtC = 16;                  // ring slots per warp
constexpr int kQtB = kQtC / 4;            // 4-slot TMA batches per ring round
constexpr uint32_t kQtRingBytes = kQtC * 128;
constexpr uint32_t kQtMetaBytes = 4 * 8 * kQtC;  // 4 rounds x (C cols + C vals)
constexpr uint32_t kQtEndsBytes = 160;           // 33 row ends, padded
constexpr uint32_t kQtBarBytes = kQtB * 8;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "QT_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra QT_WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int r0,
                                            int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
__device__ __forceinline__ void cpa4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ uint32_t ldsu(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 ldsu4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void stsu(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// (a0, a1) = (RN(a0 + p0), RN(a1 + p1)): one FADD2, scalar FMULs feed it (no FFMA)
__device__ __forceinline__ void add2(float& a0, float& a1, float p0, float p1) { add2_rn(a0, a1, p0, p1); }

__device__ __forceinline__ void ffma2(float& a0, float& a1, float x, float y0, float y1) {
    unsigned long long a, y, xx;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(y0), "f"(y1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(xx), "l"(y));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}

template <int DEC>
struct QtLayout {
    static constexpr uint32_t kLut = DEC == 0 ? 256 * 256 : 0;
    __host__ __device__ static constexpr uint32_t ring(int warps) { return kLut; }
    __host__ __device__ static constexpr uint32_t meta(int warps) { return kLut + warps * kQtRingBytes; }
    __host__ __device__ static constexpr uint32_t ends(int warps) { return meta(warps) + warps * kQtMetaBytes; }
    __host__ __device__ static constexpr uint32_t bars(int warps) { return ends(warps) + warps * kQtEndsBytes; }
    __host__ __device__ static constexpr uint32_t total(int warps) { return bars(warps) + warps * kQtBarBytes; }
};

template <int DEC, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 2)
spmm_q8t_kernel(const __grid_constant__ CUtensorMap qmap, const uint64_t* __restrict__ srow,
                const uint32_t* __restrict__ scol, const float* __restrict__ sval, uint64_t n_rows, uint32_t f,
                const float* __restrict__ lut_g, const float2* __restrict__ fparams, float4* __restrict__ c,
                uint64_t ldc4, uint64_t groups) {
    typedef QtLayout<DEC> L;
    extern __shared__ __align__(1024) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ring0 = su32(smem) + L::ring(WARPS) + warp * kQtRingBytes;
    const uint32_t meta0 = su32(smem) + L::meta(WARPS) + warp * kQtMetaBytes;
    const uint32_t ends0 = su32(smem) + L::ends(WARPS) + warp * kQtEndsBytes;
    const uint32_t bar0 = su32(smem) + L::bars(WARPS) + warp * kQtBarBytes;
    if (lane == 0) {
        for (int b = 0; b < kQtB; ++b) mbar_init(bar0 + 8 * b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (DEC == 0) {
        for (int i = threadIdx.x; i < 256 * 32; i += WARPS * 32)
            reinterpret_cast<float*>(smem)[(i >> 5) * 64 + (i & 31)] = lut_g[i >> 5];
    }
    __syncthreads();

    // column tile blockIdx.y: codes 128y.., output float4 columns 32y..
    const uint32_t tile = blockIdx.y;
    const int xcrd = (int)(tile * 128);
    const uint32_t f4 = min(32u, (f + 3) / 4 - tile * 32);
    const bool st_ok = lane < f4;
    float sj[4] = {0.f, 0.f, 0.f, 0.f}, mj[4] = {0.f, 0.f, 0.f, 0.f};
    if (DEC == 1 && st_ok) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t j = (tile * 32 + lane) * 4 + u;
            if (j < f) {
                const float2 p = fparams[j];
                sj[u] = p.x;
                mj[u] = p.y;
            }
        }
    }
    const uint32_t lane4 = lane * 4;
    const uint32_t rd0 = ring0 + lane4;  // this lane's 4 codes of ring slot p at rd0 + p * 128
    uint32_t kk = 0;                      // rounds this warp has waited on (mbarrier parity)

    for (uint64_t g = (uint64_t)blockIdx.x * WARPS + warp; g < groups; g += (uint64_t)gridDim.x * WARPS) {
        const uint64_t r0 = g * 32;
        const uint32_t nr = (uint32_t)min((uint64_t)32, n_rows - r0);
        const uint64_t g0 = srow[r0];
        const uint64_t my_end = srow[r0 + 1 + min(lane, nr - 1)];
        const uint32_t total = (uint32_t)(__shfl_sync(0xffffffffu, my_end, nr - 1) - g0);
        __syncwarp();  // the previous group is done with ends / metadata
        stsu(ends0 + lane * 4, (uint32_t)(my_end - g0));
        if (lane == 0) stsu(ends0 + 128, total);

        auto issue_meta = [&](uint32_t k) {  // round k -> buffer k & 3 (lanes 0..C-1 cols, 16.. vals)
            const uint32_t i = lane & 15, s = k * kQtC + i;
            if (i < (uint32_t)kQtC && s < total) {
                const void* src = lane < 16 ? (const void*)(scol + g0 + s) : (const void*)(sval + g0 + s);
                cpa4(meta0 + (k & 3) * (8 * kQtC) + (lane >> 4) * (4 * kQtC) + i * 4, src);
            }
        };
        // TMA batch b of round k: slots k*C + 4b .. +3 (past `total`: row 0, never consumed into a row)
        auto issue = [&](int b, uint32_t k) {
            if (lane == 0) {
                const uint32_t t = k * kQtC + 4 * b;
                uint4 cc = ldsu4(meta0 + (k & 3) * (8 * kQtC) + 16 * b);
                if (t + 0 >= total) cc.x = 0;
                if (t + 1 >= total) cc.y = 0;
                if (t + 2 >= total) cc.z = 0;
                if (t + 3 >= total) cc.w = 0;
                // (no proxy fence: every lane's ring reads of this batch fed
                // arithmetic before the __syncwarp that precedes this issue)
                mbar_expect_tx(bar0 + 8 * b, 512);
                tma_gather4(ring0 + 512 * b, &qmap, bar0 + 8 * b, xcrd, (int)cc.x, (int)cc.y, (int)cc.z, (int)cc.w);
            }
        };
        const uint32_t rounds = (total + kQtC - 1) / kQtC;
        issue_meta(0);
        issue_meta(1);
        cpa_commit();
        cpa_wait_all();
        __syncwarp();
        if (rounds)
#pragma unroll
            for (int b = 0; b < kQtB; ++b) issue(b, 0);

        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, vs = 0.f;
        uint32_t row = 0;
        uint32_t row_end = ldsu(ends0);
        float4* cptr = c + r0 * ldc4 + tile * 32 + lane;  // rows are stored in order
        auto store_row = [&]() {
            if (st_ok) {
                float4 o;
                if (DEC == 0) {
                    o = make_float4(a0, a1, a2, a3);
                } else {
                    o = make_float4(fmaf(sj[0], a0, mj[0] * vs), fmaf(sj[1], a1, mj[1] * vs),
                                    fmaf(sj[2], a2, mj[2] * vs), fmaf(sj[3], a3, mj[3] * vs));
                }
                __stcs(cptr, o);
            }
            cptr += ldc4;
            a0 = a1 = a2 = a3 = vs = 0.f;
        };
        auto advance_rows = [&](uint32_t pos) {
            do {
                store_row();
                ++row;
                row_end = ldsu(ends0 + row * 4);
            } while (row < nr && row_end == pos);
        };
        if (row_end == 0) advance_rows(0);

        auto consume = [&](int p, float v) {
            const uint32_t r = ldsu(rd0 + p * 128);
            if (DEC == 0) {
                // byte offset q*256 + 4*lane: one PRMT, then LDS [off + smem base]
                const float d0 = *reinterpret_cast<const float*>(smem + __byte_perm(r, lane4, 0x7604u));
                const float d1 = *reinterpret_cast<const float*>(smem + __byte_perm(r, lane4, 0x7614u));
                const float d2 = *reinterpret_cast<const float*>(smem + __byte_perm(r, lane4, 0x7624u));
                const float d3 = *reinterpret_cast<const float*>(smem + __byte_perm(r, lane4, 0x7634u));
                add2(a0, a1, __fmul_rn(v, d0), __fmul_rn(v, d1));
                add2(a2, a3, __fmul_rn(v, d2), __fmul_rn(v, d3));
            } else {
                float q0 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7650));
                float q1 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7651));
                float q2 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7652));
                float q3 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7653));
                add2_rn(q0, q1, -8388608.f, -8388608.f);
                add2_rn(q2, q3, -8388608.f, -8388608.f);
                ffma2(a0, a1, v, q0, q1);
                ffma2(a2, a3, v, q2, q3);
                vs += v;
            }
        };

        for (uint32_t k = 0, t0 = 0; k < rounds; ++k, t0 += kQtC, ++kk) {
#pragma unroll
            for (int b = 0; b < kQtB; ++b) {
                if (b == 0) {  // metadata of round k+1 complete; round k+2's goes out
                    cpa_wait_all();
                    __syncwarp();
                    issue_meta(k + 2);
                    cpa_commit();
                }
                mbar_wait(bar0 + 8 * b, kk & 1);
                const uint4 vb = ldsu4(meta0 + (k & 3) * (8 * kQtC) + 4 * kQtC + 16 * b);
                const float vv[4] = {__uint_as_float(vb.x), __uint_as_float(vb.y), __uint_as_float(vb.z),
                                     __uint_as_float(vb.w)};
                if (row_end > t0 + 4 * b + 4) {  // no row ends in this batch
#pragma unroll
                    for (int u = 0; u < 4; ++u) consume(4 * b + u, vv[u]);
                } else {
                    const uint32_t base = t0 + 4 * b + 1;
                    uint32_t rel = row_end - base;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        consume(4 * b + u, vv[u]);
                        if (rel == (uint32_t)u) {
                            advance_rows(base + u);
                            rel = row_end - base;
                        }
                    }
                }
                __syncwarp();  // every lane is done with this batch's ring slots
                if (k + 1 < rounds) issue(b, k + 1);
            }
        }
        cpa_wait_all();
        while (row < nr) {  // (rows after the last slot)
            store_row();
            ++row;
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 qt_encode_fn() {
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

// u8 code matrix [rows, f] (row stride ldq bytes) as a 2-D tensor map with a
// 128 x 1 box: gather4 fetches four 128-B rows per instruction.  Rows are
// declared 2^31 - 1 (the device tier does not pass the feature row count;
// every gathered index comes from a validated CSR).
int make_code_map(CUtensorMap* map, const uint8_t* q, uint64_t f, uint64_t ldq) {
    auto fn = qt_encode_fn();
    if (!fn) return fail(AES_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {f, 0x7fffffffull};
    cuuint64_t strides[1] = {ldq};
    cuuint32_t box[2] = {128, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(q), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(AES_ERR_CUDA, "cuTensorMapEncodeTiled (codes) failed (" + std::to_string((int)r) + ")");
    return AES_OK;
}

template <int DEC, int WARPS>
int launch_q8t_t(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                 uint64_t ldq, uint64_t f, const float* lut, const float* fparams, float* c, uint64_t ldc,
                 cudaStream_t st) {
    typedef QtLayout<DEC> L;
    const size_t smem = L::total(WARPS);
    static int occ_dev[kMaxDevices] = {};
    int& occ = occ_dev[cur_device()];
    if (occ == 0) {
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_q8t_kernel<DEC, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        AES_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_q8t_kernel<DEC, WARPS>, WARPS * 32,
                                                                   smem));
        if (occ < 1) occ = 1;
    }
    CUtensorMap map;
    AES_TRY(make_code_map(&map, q, f, ldq));
    const uint32_t tiles = (uint32_t)((f + 127) / 128);
    const uint64_t groups = (n + 31) / 32;
    // persistent: one wave of resident CTAs per column tile (capped by the work)
    uint64_t per_tile = (uint64_t)num_sms() * occ / tiles;
    if (per_tile == 0) per_tile = 1;
    const uint64_t need = (groups + WARPS - 1) / WARPS;
    if (need < per_tile) per_tile = need;
    spmm_q8t_kernel<DEC, WARPS><<<dim3((unsigned)per_tile, tiles), WARPS * 32, smem, st>>>(
        map, srow, scol, sval, n, (uint32_t)f, lut, reinterpret_cast<const float2*>(fparams), reinterpret_cast<float4*>(c),
        ldc / 4, groups);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace

// Entry used by aes_dev_spmm_q8_ex (exact table decode) and the fast-mode
// per-feature path: codes 16-B aligned with ldq % 16 == 0, C 16-B aligned
// with ldc % 4 == 0.  fparams: per-feature (s, m), f entries (DEC 1 only).  Returns AES_ERR_UNSUPPORTED when the layout does
// not qualify (callers fall back to the cp.async kernels).
int launch_spmm_q8_tma(int dec, const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n,
                       const uint8_t* q, uint64_t ldq, uint64_t f, const float* lut, const float* fparams, float* c,
                       uint64_t ldc, cudaStream_t st) {
    if (n == 0 || f == 0) return AES_OK;
    if (ldq % 16 || (uintptr_t)q % 16 || ldc % 4 || (uintptr_t)c % 16 || ldc < ((f + 3) & ~3ull) ||
        n >= (1ull << 31) || f >= (1ull << 31))
        return AES_ERR_UNSUPPORTED;
    if (dec == 0) return launch_q8t_t<0, 16>(srow, scol, sval, n, q, ldq, f, lut, nullptr, c, ldc, st);
    return launch_q8t_t<1, 16>(srow, scol, sval, n, q, ldq, f, nullptr, fparams, c, ldc, st);
}

}  // namespace aes
