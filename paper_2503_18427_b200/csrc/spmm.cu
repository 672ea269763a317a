// Gather-SpMM over a (sampled) CSR for sm_100a, fp32 and int8-with-fused-
// dequantization.  Bit-exact with the reference accumulation
// (proj/src/spmm.cpp:77-84): each output element is owned by one lane and
// accumulated in ascending slot order as acc = RN(acc + RN(v * b)) starting
// from +0.0f — __fmul_rn/__fadd_rn keep ptxas from contracting into FFMA.
//
// Mapping (HBM-bound irregular gather, no tensor cores):
//  * wide rows (>= 32 float4 columns, e.g. F = 128): one warp owns a GROUP of
//    32 consecutive rows.  The warp loads the group's 33 row offsets with one
//    coalesced load, then streams the group's slots in batches of U slots
//    across row boundaries: slot metadata (col, val) for a batch is loaded by
//    U lanes in one coalesced request and broadcast by shuffle, the U dense-row
//    gathers (512 B each at F = 128, one LDG.128 per lane) are all issued
//    before any is consumed, and the next batch's metadata is prefetched under
//    them.  Memory-level parallelism is therefore U rows per warp regardless
//    of how short the rows are (products: 72 % of rows have <= 4 slots).
//  * narrow rows (F <= 64): sub-warp units of LPR lanes, one row each.
//  * int8: the same schedule gathers 4 codes per lane (u32) and dequantizes
//    through a 256-entry LUT replicated per shared-memory bank (lut[q][lane],
//    conflict-free) — the exact value dequantize() produces, so the result is
//    bit-identical to the fp32 kernel over dequantize(Q).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace aes {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float4 f4_zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// acc += v * b with separate IEEE roundings (FMUL then FADD).  ptxas 12.9
// fuses a packed mul.rn.f32x2 feeding add.rn.f32x2 into FFMA2 (even via
// inline PTX, in one asm block, or with -fmad=false), which would change the
// result bits; it leaves scalar FMULs feeding one FADD2 alone.  So the adds
// go out in pairs, (a0, a1) = (RN(a0 + p0), RN(a1 + p1)) as one FADD2
// (add.rn.f32x2 is two independent IEEE adds), and the products stay scalar:
// 3 instructions per 2 elements instead of 4.  tests/test_cpu_boundary.py
// greps the SASS of every SpMM / GEMM kernel for FFMA/FFMA2.
__device__ __forceinline__ void f4_axpy(float4& acc, float v, const float4& b) {
    add2_rn(acc.x, acc.y, __fmul_rn(v, b.x), __fmul_rn(v, b.y));
    add2_rn(acc.z, acc.w, __fmul_rn(v, b.z), __fmul_rn(v, b.w));
}

__device__ __forceinline__ uint32_t ld_meta_u32(const uint32_t* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_meta_f32(const float* p) { return __ldcs(p); }

// ---------------------------------------------------------------------------
// Gather "element" abstraction: fp32 rows (float4 per lane-column) or u8 code
// rows (4 codes per lane-column, dequantized through the banked LUT).
// ---------------------------------------------------------------------------
struct GatherF32 {
    const float4* __restrict__ b;
    uint64_t ld4;  // row stride in float4
    typedef float4 raw_t;
    static constexpr int kLutBytes = 0;
    __host__ void offset(uint32_t c0) { b += c0; }
    __host__ const float4* base() const { return b; }
    __device__ __forceinline__ const raw_t* src(uint32_t row, uint32_t c4) const {
        return b + (uint64_t)row * ld4 + c4;
    }
    __device__ __forceinline__ raw_t load(uint32_t row, uint32_t c4) const {
        return __ldg(b + (uint64_t)row * ld4 + c4);
    }
    __device__ __forceinline__ float4 decode(const raw_t& r, const float*) const { return r; }
};

struct GatherQ8 {
    const uint32_t* __restrict__ q;
    uint64_t ld4;  // row stride in u32 (4 codes)
    typedef uint32_t raw_t;
    static constexpr int kLutBytes = 256 * 32 * 4;
    __host__ void offset(uint32_t c0) { q += c0; }
    __host__ const uint32_t* base() const { return q; }
    __device__ __forceinline__ const raw_t* src(uint32_t row, uint32_t c4) const {
        return q + (uint64_t)row * ld4 + c4;
    }
    __device__ __forceinline__ raw_t load(uint32_t row, uint32_t c4) const {
        return __ldg(q + (uint64_t)row * ld4 + c4);
    }
    // lut is this lane's column of the banked table: lut[code * 32]
    __device__ __forceinline__ float4 decode(const raw_t& r, const float* lut) const {
        return make_float4(lut[(r & 0xffu) << 5], lut[((r >> 8) & 0xffu) << 5],
                           lut[((r >> 16) & 0xffu) << 5], lut[(r >> 24) << 5]);
    }
};

template <class G>
struct LutSmem {
    __device__ __forceinline__ static const float* setup(const float*, float*) { return nullptr; }
};
template <>
struct LutSmem<GatherQ8> {
    __device__ __forceinline__ static const float* setup(const float* lut_g, float* smem) {
        // smem[q * 32 + bank] = lut[q]
        for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) smem[i] = lut_g[i >> 5];
        __syncthreads();
        return smem + (threadIdx.x & 31);
    }
};

// ---------------------------------------------------------------------------
// Wide kernel: warp per 32-row group, flattened slot stream, U-slot batches.
// Lane handles float4 columns lane + 32*n for n < NV.
// ---------------------------------------------------------------------------
template <class G, int NV, int U>
__global__ void __launch_bounds__(kThreads)
spmm_wide_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                 const float* __restrict__ sval, uint64_t n_rows, G g, uint32_t f4, float4* __restrict__ c,
                 uint64_t ldc4, const float* __restrict__ lut_g) {
    extern __shared__ float smem_lut[];
    const float* lut = LutSmem<G>::setup(lut_g, smem_lut);

    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const uint64_t r0 = warp * 32;
    if (r0 >= n_rows) return;
    const uint32_t nr = (uint32_t)min((uint64_t)32, n_rows - r0);

    // row offsets of the group: lane l holds the END of row l (one coalesced
    // load of srow[r0+1 .. r0+32]); the group start is a broadcast load.
    const uint64_t g0 = srow[r0];
    const uint64_t my_end = srow[r0 + 1 + min(lane, nr - 1)];
    const uint64_t total = __shfl_sync(0xffffffffu, my_end, nr - 1) - g0;
    const uint32_t rel = (uint32_t)(my_end - g0);  // relative row end (group < 2^32 slots)

    float4 acc[NV];
#pragma unroll
    for (int n = 0; n < NV; ++n) acc[n] = f4_zero();

    bool colok[NV];
#pragma unroll
    for (int n = 0; n < NV; ++n) colok[n] = lane + 32u * n < f4;

    float4* crow = c + r0 * ldc4;
    uint32_t row = 0;
    uint32_t row_end = __shfl_sync(0xffffffffu, rel, 0);

    auto store_row = [&](uint32_t r) {
#pragma unroll
        for (int n = 0; n < NV; ++n)
            if (colok[n]) __stcs(crow + (uint64_t)r * ldc4 + lane + 32u * n, acc[n]);
#pragma unroll
        for (int n = 0; n < NV; ++n) acc[n] = f4_zero();
    };
    // leading empty rows
    while (row < nr && row_end == 0) {
        store_row(row);
        ++row;
        row_end = __shfl_sync(0xffffffffu, rel, min(row, nr - 1));
    }

    // metadata for the first batch
    uint32_t mc = 0;
    float mv = 0.f;
    if (lane < (uint32_t)U && lane < total) {
        mc = ld_meta_u32(scol + g0 + lane);
        mv = ld_meta_f32(sval + g0 + lane);
    }

    for (uint64_t t = 0; t < total; t += U) {
        typename G::raw_t braw[U][NV];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t cidx = __shfl_sync(0xffffffffu, mc, u);
            if (t + u < total) {
#pragma unroll
                for (int n = 0; n < NV; ++n)
                    if (colok[n]) braw[u][n] = g.load(cidx, lane + 32u * n);
            }
        }
        float vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) vv[u] = __shfl_sync(0xffffffffu, mv, u);
        // prefetch next batch's metadata under the gathers
        if (lane < (uint32_t)U && t + U + lane < total) {
            mc = ld_meta_u32(scol + g0 + t + U + lane);
            mv = ld_meta_f32(sval + g0 + t + U + lane);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (t + u < total) {
#pragma unroll
                for (int n = 0; n < NV; ++n)
                    if (colok[n]) f4_axpy(acc[n], vv[u], g.decode(braw[u][n], lut));
                const uint32_t pos = (uint32_t)(t + u + 1);
                if (pos == row_end) {
                    store_row(row);
                    ++row;
                    row_end = __shfl_sync(0xffffffffu, rel, min(row, nr - 1));
                    while (row < nr && row_end == pos) {  // empty rows
                        store_row(row);
                        ++row;
                        row_end = __shfl_sync(0xffffffffu, rel, min(row, nr - 1));
                    }
                }
            }
        }
    }
    while (row < nr) {  // trailing empty rows of a group with no slots left
        store_row(row);
        ++row;
    }
}


// ---------------------------------------------------------------------------
// Ring kernel (F <= 128 fp32 / F <= 128 int8): same warp-per-32-row-group
// slot stream, but the gathered rows land in a per-warp shared-memory ring of
// C slots through cp.async (LDGSTS), so C gathers (C x 512 B at F = 128) stay
// in flight per warp independent of the register budget.  Slot t is consumed
// after cp.async.wait_group(C-1), then slot t + C is issued into the same
// ring entry.  Slot metadata is loaded C slots at a time (lane p holds slot
// base + p) two chunks ahead of use.  Each lane only ever reads the 16 (or 4)
// bytes it copied itself, so no cross-lane barrier is needed.
// ---------------------------------------------------------------------------
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ uint32_t pin_u32(uint32_t x) {
    uint32_t y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
// (a0, a1) = (fma(x, y0, a0), fma(x, y1, a1)) as one FFMA2 — int8 FAST MODE only
__device__ __forceinline__ void fma2_rn(float& a0, float& a1, float x, float y0, float y1) {
    unsigned long long a, y, xx;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(y0), "f"(y1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(xx), "l"(y));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}
template <class T>
__device__ __forceinline__ T* pin_ptr(T* p) {
    uint64_t y;
    asm volatile("mov.b64 %0, %1;" : "=l"(y) : "l"(reinterpret_cast<uint64_t>(p)));
    return reinterpret_cast<T*>(y);
}
// Offset of the dynamic shared-memory window inside the CTA's shared window
// on sm_100a (1 KB reserved; the SASS of cvta.shared is (CgaCtaId<<24)+0x400).
constexpr uint32_t kDynSmemOffset = 0x400;
// The batch kernel relies on it; dyn_smem_offset_ok() checks it once per
// device with a probe launch (same dynamic-only shared memory layout) and the
// int8 dispatch falls back to the layout-agnostic ring kernel if a driver or
// toolkit ever places the window elsewhere — slower, never wrong.
__global__ void dyn_smem_probe_kernel(uint32_t* out) {
    extern __shared__ __align__(16) unsigned char probe_smem[];
    if (threadIdx.x == 0) *out = (uint32_t)__cvta_generic_to_shared(probe_smem) & 0xFFFFFFu;
}
bool dyn_smem_offset_ok(cudaStream_t st) {
    static int ok_dev[kMaxDevices] = {};  // 0 unknown, 1 ok, -1 not
    int& ok = ok_dev[cur_device()];
    if (ok == 0) {
        // (no probe while the caller's stream is being captured into a graph:
        // the batch kernel's own __trap() remains the guard)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return true;
        (void)cudaGetLastError();
        cudaStream_t ps = nullptr;
        uint32_t* d = nullptr;
        uint32_t h = 0;
        ok = -1;
        if (cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) == cudaSuccess) {
            if (cudaMallocAsync((void**)&d, sizeof(uint32_t), ps) == cudaSuccess) {
                dyn_smem_probe_kernel<<<1, 32, 4096, ps>>>(d);
                if (cudaMemcpyAsync(&h, d, sizeof(uint32_t), cudaMemcpyDeviceToHost, ps) == cudaSuccess &&
                    cudaStreamSynchronize(ps) == cudaSuccess && h == kDynSmemOffset)
                    ok = 1;
                cudaFreeAsync(d, ps);
                cudaStreamSynchronize(ps);
            }
            cudaStreamDestroy(ps);
        }
        (void)cudaGetLastError();
    }
    return ok == 1;
}
// LDS at (addr + kDynSmemOffset); not volatile so ptxas may schedule it
__device__ __forceinline__ float lds_lut(uint32_t addr) {
    float v;
    asm("ld.shared.f32 %0, [%1+1024];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Shared-memory helpers on 32-bit shared-window addresses (no generic->shared
// conversion per access).  Volatile so they stay ordered after cp.async.wait.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f32x4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void cp_async_sa(uint32_t sa, const void* gmem, int bytes) {
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// Ring element types: fp32 rows (float4 per lane) or u8 code rows (4 codes per
// lane, decoded through the per-bank replicated LUT at smem offset 0).
struct RingF32 {
    typedef float4 raw_t;
    static constexpr int kBytes = 16;
    static constexpr int kLutBytes = 0;
    __device__ __forceinline__ static float4 load_decode(uint32_t a, uint32_t) { return lds_f32x4(a); }
};
struct RingQ8 {
    typedef uint32_t raw_t;
    static constexpr int kBytes = 4;
    static constexpr int kLutBytes = 256 * 32 * 4;
    // lut_lane = smem address of lut[0][lane]; entry q is at lut_lane + q * 128
    __device__ __forceinline__ static float4 load_decode(uint32_t a, uint32_t lut_lane) {
        const uint32_t r = lds_u32(a);
        return make_float4(lds_f32(lut_lane + (__byte_perm(r, 0, 0x4440) << 7)),
                           lds_f32(lut_lane + (__byte_perm(r, 0, 0x4441) << 7)),
                           lds_f32(lut_lane + (__byte_perm(r, 0, 0x4442) << 7)),
                           lds_f32(lut_lane + (__byte_perm(r, 0, 0x4443) << 7)));
    }
};

// One warp, rows [rb, re) as ONE slot stream: the ring never drains at a
// row-group boundary.  Row ends (relative to the range's first slot) live in
// a 32-row window held one per lane; the next window's ends are loaded when
// the current one is entered, so crossing into it costs a register move.
// Caller guarantees srow[re] - srow[rb] < 2^31.
// SOUT: rows go to shared memory instead (the fused layer kernel): row rb + i
// of this lane at smem address sout + i * ldc4 * 16 (c unused).
template <class R, int NV, int C, bool FULL, bool SOUT = false>
__device__ __forceinline__ void ring_range(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                                           const float* __restrict__ sval,
                                           const typename R::raw_t* __restrict__ gsrc, uint32_t ld, uint32_t f4,
                                           float4* __restrict__ c, uint64_t ldc4, uint32_t ring0,
                                           uint32_t lut_lane, uint64_t rb, uint64_t re, uint32_t sout = 0) {
    typedef typename R::raw_t raw_t;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t g0 = srow[rb];
    const uint32_t total = (uint32_t)(srow[re] - g0);
    // end of row w + lane (relative to g0); rows past re read as `total`
    auto window = [&](uint64_t w) -> uint32_t {
        return (uint32_t)(srow[min(w + 1 + lane, re)] - g0);
    };
    uint32_t rel = window(rb);
    uint32_t rel_nx = window(rb + 32);
    const uint32_t* gcol = scol + g0;
    const float* gval = sval + g0;
    const char* glb = reinterpret_cast<const char*>(gsrc + lane);
    const uint32_t ld_bytes = ld * (uint32_t)sizeof(raw_t);
    bool colok[NV];
#pragma unroll
    for (int n = 0; n < NV; ++n) colok[n] = FULL || lane + 32u * n < f4;

    auto ld_col = [&](uint32_t chunk) -> uint32_t {
        const uint32_t s = chunk * C + lane;
        return (lane < (uint32_t)C && s < total) ? ld_meta_u32(gcol + s) : 0u;
    };
    auto ld_val = [&](uint32_t chunk) -> float {
        const uint32_t s = chunk * C + lane;
        return (lane < (uint32_t)C && s < total) ? ld_meta_f32(gval + s) : 0.f;
    };
    auto issue = [&](int p, uint32_t col) {
        // one IMAD.WIDE.U32: lane base + col * row_bytes
        const raw_t* src = reinterpret_cast<const raw_t*>(glb + (uint64_t)col * ld_bytes);
#pragma unroll
        for (int n = 0; n < NV; ++n)
            if (colok[n]) cp_async_sa(ring0 + (p * NV + n) * 32 * R::kBytes, src + 32 * n, R::kBytes);
    };

    {  // prologue: first C gathers in flight
        const uint32_t mc0 = ld_col(0);
#pragma unroll
        for (int p = 0; p < C; ++p) {
            const uint32_t col = __shfl_sync(0xffffffffu, mc0, p);
            if ((uint32_t)p < total) issue(p, col);
            cp_commit();
        }
    }
    uint32_t mc_is = ld_col(1), mc_nx = ld_col(2);
    float mv_cur = ld_val(0), mv_nx = ld_val(1);

    float4 acc[NV];
#pragma unroll
    for (int n = 0; n < NV; ++n) acc[n] = f4_zero();
    float4* crow = c + lane;
    uint64_t ra = rb;  // next row to store
    uint32_t wi = 0;   // its index in the window
    uint32_t row_end = __shfl_sync(0xffffffffu, rel, 0);
    auto store_row = [&]() {
#pragma unroll
        for (int n = 0; n < NV; ++n) {
            if (SOUT) {
                if (colok[n])
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                     sout + (uint32_t)(ra - rb) * (uint32_t)ldc4 * 16u + 512u * n),
                                 "f"(acc[n].x), "f"(acc[n].y), "f"(acc[n].z), "f"(acc[n].w)
                                 : "memory");
            } else if (colok[n]) {
                __stcs(crow + ra * ldc4 + 32u * n, acc[n]);
            }
            acc[n] = f4_zero();
        }
    };
    auto advance_rows = [&](uint32_t pos) {  // rows ending at slot position pos
        do {
            store_row();
            ++ra;
            if (++wi == 32) {
                wi = 0;
                rel = rel_nx;
                rel_nx = window(ra + 32);
            }
            row_end = __shfl_sync(0xffffffffu, rel, wi);
        } while (ra < re && row_end == pos);
    };
    if (row_end == 0) advance_rows(0);

    auto body = [&](int p, uint32_t t) {
        cp_wait<C - 1>();
        const float v = __shfl_sync(0xffffffffu, mv_cur, p);
#pragma unroll
        for (int n = 0; n < NV; ++n)
            if (colok[n]) f4_axpy(acc[n], v, R::load_decode(ring0 + (p * NV + n) * 32 * R::kBytes, lut_lane));
        const uint32_t col = __shfl_sync(0xffffffffu, mc_is, p);
        if (t + C < total) issue(p, col);
        cp_commit();
        if (t + 1 == row_end) advance_rows(t + 1);
    };

    uint32_t k = 0;
    for (uint32_t t0 = 0; t0 < total; t0 += C, ++k) {
        if (t0 + C <= total) {
#pragma unroll
            for (int p = 0; p < C; ++p) body(p, t0 + p);
        } else {
#pragma unroll
            for (int p = 0; p < C; ++p) {
                if (t0 + p >= total) break;
                body(p, t0 + p);
            }
        }
        mv_cur = mv_nx;
        mc_is = mc_nx;
        mv_nx = ld_val(k + 2);
        mc_nx = ld_col(k + 3);
    }
    cp_wait<0>();
    for (; ra < re; ++ra) store_row();  // trailing empty rows
}

// Rows [rb, re) in slices whose slot counts fit the stream's 32-bit offsets.
template <class R, int NV, int C, bool FULL>
__device__ __forceinline__ void ring_rows(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                                          const float* __restrict__ sval,
                                          const typename R::raw_t* __restrict__ gsrc, uint32_t ld, uint32_t f4,
                                          float4* __restrict__ c, uint64_t ldc4, uint32_t ring0, uint32_t lut_lane,
                                          uint64_t rb, uint64_t re, uint64_t hub_thr = ~0ull) {
    const uint32_t lane = threadIdx.x & 31;
    while (rb < re) {
        // next hub row (> hub_thr slots: spmm_hub_kernel stores it) in [rb, re)
        uint64_t hub = re;
        if (hub_thr != ~0ull) {
            for (uint64_t w = rb; w < re; w += 32) {
                const uint64_t r = w + lane;
                const bool big = r < re && srow[r + 1] - srow[r] > hub_thr;
                const uint32_t m = __ballot_sync(0xffffffffu, big);
                if (m) {
                    hub = w + __ffs(m) - 1;
                    break;
                }
            }
        }
        while (rb < hub) {
            uint64_t e = hub;
            if (srow[hub] - srow[rb] >= (1ull << 31)) e = min(rb + 1, hub);  // (never at the BASELINE shapes)
            ring_range<R, NV, C, FULL>(srow, scol, sval, gsrc, ld, f4, c, ldc4, ring0, lut_lane, rb, e);
            rb = e;
        }
        rb = hub < re ? hub + 1 : re;
    }
}

template <class R, int C, int NV, int WARPS>
__device__ __forceinline__ void ring_setup(const float* __restrict__ lut_g, uint32_t& ring0, uint32_t& lut_lane) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t smem0 = smem_addr(smem_raw);
    if (R::kLutBytes) {
        float* lut = reinterpret_cast<float*>(smem_raw);
        for (int i = threadIdx.x; i < 256 * 32; i += WARPS * 32) lut[i] = lut_g[i >> 5];
        __syncthreads();
    }
    lut_lane = smem0 + lane * 4;
    // ring entry (p, n) of this lane: ring0 + (p * NV + n) * 32 * kBytes
    ring0 = smem0 + R::kLutBytes + (threadIdx.x >> 5) * (C * NV * 32 * R::kBytes) + lane * R::kBytes;
}

// Static schedule: warp w of the grid owns row group w.
template <class R, int NV, int C, int WARPS, bool FULL>
__global__ void __launch_bounds__(WARPS * 32)
spmm_ring_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                 const float* __restrict__ sval, uint64_t n_rows, const typename R::raw_t* __restrict__ gsrc,
                 uint32_t ld, uint32_t f4, float4* __restrict__ c, uint64_t ldc4, const float* __restrict__ lut_g,
                 uint32_t group_rows) {
    uint32_t ring0, lut_lane;
    ring_setup<R, C, NV, WARPS>(lut_g, ring0, lut_lane);
    // a warp owns `group_rows` (<= 32) consecutive rows; fewer rows per warp
    // on small graphs keeps every SM busy
    const uint64_t r0 = ((uint64_t)blockIdx.x * WARPS + (threadIdx.x >> 5)) * group_rows;
    if (r0 >= n_rows) return;
    ring_rows<R, NV, C, FULL>(srow, scol, sval, gsrc, ld, f4, c, ldc4, ring0, lut_lane, r0,
                              min(r0 + group_rows, n_rows));
}

// Heavy-first dynamic schedule for unbounded rows (exact SpMM, FULL plans):
// a row group's slot count is unbounded there (products: rows up to 17 k
// nonzeros, 42 % of all nonzeros in rows > 2 000), and with a static
// schedule the SMs idle behind the few warps that drew the hub groups
// (ncu: 8.6 of 24 warps active on average).  A pre-pass lists the groups
// with more than kHeavySlots slots; resident warps then take tickets from one
// counter — first the heavy list, then every other group in order — so the
// long groups start early and short ones fill in behind them.  Each group is
// still one warp's ordered stream: results are unchanged.
constexpr uint32_t kHeavySlots = 4096;
constexpr int kSchedStatic = 1, kSchedDyn = 2, kSchedBal = 3;
constexpr int kSchedBalOne = 4;  // balanced, one wave (rows of unknown length: hub rows stay spread)
constexpr int kSchedAuto = 5;    // bounded rows, per-kernel choice (see the launchers)
constexpr int kSchedStaticPersist = 6;  // int8 batch kernel: persistent grid-stride 32-row groups (tuning only)
struct DynSched {
    unsigned int next;     // ticket counter
    unsigned int n_heavy;  // heavy groups listed
    unsigned int pad[2];
    unsigned int heavy[1];  // [groups]
};

__global__ void heavy_scan_kernel(const uint64_t* __restrict__ srow, uint64_t n_rows, uint32_t group_rows,
                                  uint64_t groups, DynSched* ws) {
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r0 = g * group_rows, r1 = min(r0 + group_rows, n_rows);
        if (srow[r1] - srow[r0] > kHeavySlots) ws->heavy[atomicAdd(&ws->n_heavy, 1u)] = (unsigned int)g;
    }
}

__device__ __forceinline__ bool group_is_heavy(const uint64_t* srow, uint64_t n_rows, uint32_t group_rows,
                                               uint64_t g) {
    const uint64_t r0 = g * group_rows, r1 = min(r0 + group_rows, n_rows);
    return srow[r1] - srow[r0] > kHeavySlots;
}

template <class R, int NV, int C, int WARPS, bool FULL>
__global__ void __launch_bounds__(WARPS * 32)
spmm_ring_dyn_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                     const float* __restrict__ sval, uint64_t n_rows, const typename R::raw_t* __restrict__ gsrc,
                     uint32_t ld, uint32_t f4, float4* __restrict__ c, uint64_t ldc4, const float* __restrict__ lut_g,
                     uint32_t group_rows, uint64_t groups, DynSched* ws) {
    uint32_t ring0, lut_lane;
    ring_setup<R, C, NV, WARPS>(lut_g, ring0, lut_lane);
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t n_heavy = *reinterpret_cast<volatile unsigned int*>(&ws->n_heavy);
    const uint64_t n_items = n_heavy + groups;
    uint64_t w = 0;
    if (lane == 0) w = atomicAdd(&ws->next, 1u);
    w = __shfl_sync(0xffffffffu, w, 0);
    while (w < n_items) {
        uint64_t nw = 0;  // next ticket, fetched while this group runs
        if (lane == 0) nw = atomicAdd(&ws->next, 1u);
        nw = __shfl_sync(0xffffffffu, nw, 0);
        const uint64_t g = w < n_heavy ? (uint64_t)ws->heavy[w] : w - n_heavy;
        if (w < n_heavy || !group_is_heavy(srow, n_rows, group_rows, g))
            ring_rows<R, NV, C, FULL>(srow, scol, sval, gsrc, ld, f4, c, ldc4, ring0, lut_lane, g * group_rows,
                                      min(g * group_rows + group_rows, n_rows));
        w = nw;
    }
}

// ---------------------------------------------------------------------------
// Balanced persistent schedule (the default): one wave of resident warps,
// warp w of W owns the contiguous rows whose work key
//     key(r) = (srow[r] - srow[0]) + kRowCost * r      (slots + per-row cost)
// falls in [w*K/W, (w+1)*K/W), K = key(n), and walks them in groups of <= 32
// rows.  Every warp gets the same work whatever the shard size, so there is
// no partial last wave (a row-sharded products shard at P = 8 is 2.7 waves of
// 32-row groups under the static schedule) and hub rows are balanced by
// construction (a warp holding a 17 k-slot row gets few others).  The range
// ends come from two 16-ary searches over srow, one per half-warp, 5-6
// dependent loads at kernel start.  Each group is still one warp's ordered
// stream, so results are unchanged.
// ---------------------------------------------------------------------------
constexpr uint64_t kRowCost = 1;  // a row's store + bookkeeping ~ one gathered slot

// First row r in [0, n] with key(r) >= target (key(n) >= target required),
// searched by the 16 lanes of this half-warp; every lane of the half gets it.
__device__ __forceinline__ uint64_t bal_lower_bound(const uint64_t* __restrict__ srow, uint64_t n, uint64_t s0,
                                                    uint64_t target) {
    const uint32_t lane = threadIdx.x & 31, i = lane & 15;
    const uint32_t hmask = 0xFFFFu << (lane & 16);
    uint64_t lo = 0, hi = n;  // answer in [lo, hi]
    // warp-uniform trip count (the halves may need different numbers of
    // rounds; a finished half re-probes lo == hi and stays put)
    while (__any_sync(0xffffffffu, lo < hi)) {
        const uint64_t step = (hi - lo + 16) / 16;  // ceil((hi - lo + 1) / 16)
        const uint64_t p = min(lo + (i + 1) * step - 1, hi);
        const bool ge = (srow[p] - s0) + kRowCost * p >= target;
        const uint32_t bal = (__ballot_sync(0xffffffffu, ge) & hmask) >> (lane & 16);
        const uint32_t j = __ffs(bal) - 1;  // bal != 0: probe 15 is hi
        const uint64_t pj = __shfl_sync(0xffffffffu, p, (lane & 16) + j);
        const uint64_t pm = __shfl_sync(0xffffffffu, p, (lane & 16) + (j ? j - 1 : 0));
        lo = j ? pm + 1 : lo;
        hi = pj;
    }
    return lo;
}

// Rows [rb, re) of global warp gw out of nw.
__device__ __forceinline__ void bal_range(const uint64_t* __restrict__ srow, uint64_t n_rows, uint64_t gw,
                                          uint64_t nw, uint64_t& rb, uint64_t& re) {
    const uint64_t s0 = srow[0];
    const uint64_t total = (srow[n_rows] - s0) + kRowCost * n_rows;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t k = gw + (lane >> 4);  // lower half: begin, upper half: end
    // k * total / nw without 64-bit overflow (total < 2^63 / nw in practice)
    const uint64_t target = k >= nw ? total : (uint64_t)(((unsigned __int128)total * k) / nw);
    const uint64_t r = bal_lower_bound(srow, n_rows, s0, target);
    rb = __shfl_sync(0xffffffffu, r, 0);
    re = __shfl_sync(0xffffffffu, r, 16);
}

// Hub rows (rows of unknown length: exact SpMM, FULL plans).  A row holding
// far more than a balanced warp share keeps its one warp busy long after the
// rest finish (arxiv exact: its 8.8 k-slot row took 0.8 ms on one warp while
// the whole rest of the graph needs 0.1 ms).  Order forbids splitting a row's
// slots, but not its columns: spmm_hub_kernel gives each hub row a CTA whose
// 128 lanes own one output column each and stream the row's slots through
// 128-deep per-warp cp.async rings (64 KB in flight per row, 8x a warp's),
// and the balanced kernel skips those rows.  Both kernels derive the same
// threshold from the same quantities.
constexpr uint64_t kHubMinSlots = 1024;
__device__ __forceinline__ uint64_t hub_threshold(const uint64_t* __restrict__ srow, uint64_t n_rows, uint64_t nw) {
    const uint64_t key = (srow[n_rows] - srow[0]) + kRowCost * n_rows;
    return max(kHubMinSlots, 2 * key / nw);  // more than two balanced shares
}

constexpr int kHubWarps = 4, kHubRing = 128, kHubBatch = 16, kHubRows = 256;
__global__ void __launch_bounds__(kHubWarps * 32)
spmm_hub_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                const float* __restrict__ sval, uint64_t n_rows, const float* __restrict__ b, uint64_t ldb,
                uint32_t f, float* __restrict__ c, uint64_t ldc, uint64_t bal_warps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t hubs[kHubRows];
    __shared__ uint32_t n_hubs;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t thr = hub_threshold(srow, n_rows, bal_warps);
    if (tid == 0) n_hubs = 0;
    __syncthreads();
    const uint64_t r0 = (uint64_t)blockIdx.x * kHubRows;
    for (uint32_t i = tid; i < kHubRows; i += kHubWarps * 32) {
        const uint64_t r = r0 + i;
        if (r < n_rows && srow[r + 1] - srow[r] > thr) hubs[atomicAdd(&n_hubs, 1u)] = i;
    }
    __syncthreads();
    const uint32_t nh = n_hubs;
    const uint32_t ring = smem_addr(smem_raw) + warp * (kHubRing * 128) + lane * 4;
    for (uint32_t hi = 0; hi < nh; ++hi) {
        const uint64_t h = r0 + hubs[hi];
        const uint64_t g0 = srow[h];
        const uint32_t total = (uint32_t)(srow[h + 1] - g0);  // < 2^32 (u32 plan slots)
        for (uint32_t cb = warp * 32; cb < f; cb += kHubWarps * 32) {  // column block of this warp
            const uint32_t col = cb + lane;
            // lanes past f read column f - 1 (in bounds) and store nothing
            const float* bc = b + min(col, f - 1);
            // slots are padded to whole chunks of 32: metadata past `total`
            // reads as (col 0, val 0) — a harmless in-bounds gather that is
            // never accumulated (the loop stops at total)
            auto ld_col = [&](uint32_t k) -> uint32_t {
                const uint32_t s = k * 32 + lane;
                return s < total ? ld_meta_u32(scol + g0 + s) : 0u;
            };
            auto ld_val = [&](uint32_t k) -> float {
                const uint32_t s = k * 32 + lane;
                return s < total ? ld_meta_f32(sval + g0 + s) : 0.f;
            };
            // ring entry of slot 32k + j: ring + ((k % kChunks) * 32 + j) * 128
            constexpr uint32_t kChunks = kHubRing / 32;
            auto issue_chunk_slot = [&](uint32_t base, uint32_t j, uint32_t cidx) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(base + j * 128),
                             "l"(bc + (uint64_t)cidx * ldb)
                             : "memory");
            };
            // prologue: chunks 0 .. kChunks-1 in flight, kHubBatch slots per commit group
#pragma unroll
            for (uint32_t k = 0; k < kChunks; ++k) {
                const uint32_t mc = ld_col(k);
                const uint32_t base = ring + k * 32 * 128;
#pragma unroll
                for (uint32_t j = 0; j < 32; ++j) {
                    issue_chunk_slot(base, j, __shfl_sync(0xffffffffu, mc, j));
                    if (j % kHubBatch == kHubBatch - 1) cp_commit();
                }
            }
            float acc = 0.f;
            float mv = ld_val(0);
            uint32_t mc_ahead = ld_col(kChunks);  // columns of the chunk issued while consuming chunk 0
            const uint32_t chunks = (total + 31) / 32;
            for (uint32_t k = 0; k < chunks; ++k) {
                const float mv_nx = ld_val(k + 1);
                const uint32_t mc_nx = ld_col(k + 1 + kChunks);
                const uint32_t base = ring + (k % kChunks) * 32 * 128;
                const uint32_t left = total - k * 32;  // >= 1
                if (left >= 32) {  // whole chunk: no per-slot bound checks
#pragma unroll
                    for (uint32_t j = 0; j < 32; ++j) {
                        if (j % kHubBatch == 0) cp_wait<kHubRing / kHubBatch - 1>();
                        acc = __fadd_rn(acc, __fmul_rn(__shfl_sync(0xffffffffu, mv, j), lds_f32(base + j * 128)));
                        issue_chunk_slot(base, j, __shfl_sync(0xffffffffu, mc_ahead, j));
                        if (j % kHubBatch == kHubBatch - 1) cp_commit();
                    }
                } else {  // last, partial chunk: nothing more is committed, so wait for all
                    cp_wait<0>();
#pragma unroll
                    for (uint32_t j = 0; j < 32; ++j)
                        if (j < left)
                            acc = __fadd_rn(acc, __fmul_rn(__shfl_sync(0xffffffffu, mv, j), lds_f32(base + j * 128)));
                }
                mv = mv_nx;
                mc_ahead = mc_nx;
            }
            cp_wait<0>();
            __syncwarp();
            if (col < f) c[h * ldc + col] = acc;
        }
    }
}

template <class R, int NV, int C, int WARPS, bool FULL>
__global__ void __launch_bounds__(WARPS * 32)
spmm_ring_bal_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                     const float* __restrict__ sval, uint64_t n_rows, const typename R::raw_t* __restrict__ gsrc,
                     uint32_t ld, uint32_t f4, float4* __restrict__ c, uint64_t ldc4, const float* __restrict__ lut_g,
                     int hubs) {
    uint32_t ring0, lut_lane;
    ring_setup<R, C, NV, WARPS>(lut_g, ring0, lut_lane);
    uint64_t rb, re;
    const uint64_t nw = (uint64_t)gridDim.x * WARPS;
    bal_range(srow, n_rows, (uint64_t)blockIdx.x * WARPS + (threadIdx.x >> 5), nw, rb, re);
    ring_rows<R, NV, C, FULL>(srow, scol, sval, gsrc, ld, f4, c, ldc4, ring0, lut_lane, rb, re,
                              hubs ? hub_threshold(srow, n_rows, nw) : ~0ull);
}

// ---------------------------------------------------------------------------
// Narrow kernel: LPR lanes per row (LPR in 1..16), one float4 column each.
// ---------------------------------------------------------------------------
template <class G, int LPR, int U>
__global__ void __launch_bounds__(kThreads)
spmm_narrow_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                   const float* __restrict__ sval, uint64_t n_rows, G g, uint32_t f4,
                   float4* __restrict__ c, uint64_t ldc4, const float* __restrict__ lut_g) {
    extern __shared__ float smem_lut[];
    const float* lut = LutSmem<G>::setup(lut_g, smem_lut);
    const uint64_t tid = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    const uint64_t row = tid / LPR;
    const uint32_t li = (uint32_t)(tid % LPR);
    if (row >= n_rows) return;
    const bool ok = li < f4;
    const uint64_t k0 = srow[row], k1 = srow[row + 1];
    float4 acc = f4_zero();
    for (uint64_t k = k0; k < k1; k += U) {
        uint32_t cc[U];
        float vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k + u < k1) {
                cc[u] = ld_meta_u32(scol + k + u);
                vv[u] = ld_meta_f32(sval + k + u);
            }
        }
        typename G::raw_t braw[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k + u < k1 && ok) braw[u] = g.load(cc[u], li);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k + u < k1 && ok) f4_axpy(acc, vv[u], g.decode(braw[u], lut));
    }
    if (ok) __stcs(c + row * ldc4 + li, acc);
}

// ---------------------------------------------------------------------------
// Scalar kernel for layouts the vector path cannot take (ld % 4 != 0 or
// misaligned): warp per row, lane per column, same ordering.
// ---------------------------------------------------------------------------
template <int U>
__global__ void __launch_bounds__(kThreads)
spmm_scalar_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                   const float* __restrict__ sval, uint64_t n_rows, const float* __restrict__ b,
                   uint64_t ldb, uint64_t f, float* __restrict__ c, uint64_t ldc) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = ((uint64_t)gridDim.x * kThreads) >> 5;
    for (uint64_t row = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; row < n_rows; row += warps) {
        const uint64_t k0 = srow[row], k1 = srow[row + 1];
        for (uint64_t j0 = 0; j0 < f; j0 += 32) {
            const uint64_t j = j0 + lane;
            const bool ok = j < f;
            float acc = 0.f;
            for (uint64_t k = k0; k < k1; k += U) {
                float bv[U], vv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (k + u < k1) {
                        uint32_t cc = scol[k + u];
                        vv[u] = sval[k + u];
                        if (ok) bv[u] = __ldg(b + (uint64_t)cc * ldb + j);
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (k + u < k1 && ok) acc = __fadd_rn(acc, __fmul_rn(vv[u], bv[u]));
            }
            if (ok) c[row * ldc + j] = acc;
        }
    }
}

// ---------------------------------------------------------------------------
// int8 dual-stream kernel (F <= 128 codes, ldq % 8 == 0).  The int8 SpMM is
// instruction-bound, not HBM-bound: a 128-B code row feeds 128 LUT decodes
// and 256 FP ops, so per-slot bookkeeping (wait, shuffles, issue, row-end
// test) matters.  Here each half-warp runs its own row-group stream with 8
// codes per lane (LDGSTS.64), so one warp instruction advances two slots and
// the bookkeeping is paid once per pair; the LUT is laid out with a 256-B row
// stride so PRMT(code, lane*4) yields the byte offset of lut[code][lane]
// directly (one PRMT + one LDS per code).  Same slot order and roundings as
// the fp32 kernel: bit-identical to spmm over dequantize(Q).
// ---------------------------------------------------------------------------
template <int C, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
spmm_q8_dual_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                    const float* __restrict__ sval, uint64_t n_rows, const uint2* __restrict__ q, uint32_t ld8,
                    uint32_t f8, float4* __restrict__ c, uint64_t ldc4, const float* __restrict__ lut_g,
                    uint32_t group_rows) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr uint32_t kLutBytes = 256 * 256;  // lut[q] at q*256, lane j at +4j (upper half unused)
    for (int i = threadIdx.x; i < 256 * 32; i += WARPS * 32)
        reinterpret_cast<float*>(smem_raw)[(i >> 5) * 64 + (i & 31)] = lut_g[i >> 5];
    __syncthreads();

    const uint32_t lane = threadIdx.x & 31, h = lane >> 4, hl = lane & 15;
    const uint32_t hbase = h << 4;
    const uint32_t hmask = 0xFFFFu << hbase;
    const uint32_t lane4 = lane * 4;  // byte 0 of the decode PRMT
    const uint32_t ring0 = smem_addr(smem_raw) + kLutBytes + (threadIdx.x >> 5) * (2 * C * 128) + h * (C * 128) + hl * 8;

    // this half-warp's row group
    const uint64_t gidx = ((uint64_t)blockIdx.x * WARPS + (threadIdx.x >> 5)) * 2 + h;
    const uint64_t r0 = gidx * group_rows;
    const bool active = r0 < n_rows;
    const uint32_t nr = active ? (uint32_t)min((uint64_t)group_rows, n_rows - r0) : 1;
    const uint64_t g0 = active ? srow[r0] : 0;
    const uint64_t my_end = active ? srow[r0 + 1 + min(hl, nr - 1)] : 0;
    const uint64_t end_all = __shfl_sync(0xffffffffu, my_end, hbase + nr - 1);
    const uint32_t total = active ? (uint32_t)(end_all - g0) : 0u;
    const uint32_t rel = (uint32_t)(my_end - g0);
    const uint32_t total_max = max(total, __shfl_xor_sync(0xffffffffu, total, 16));
    const uint32_t* gcol = scol + g0;
    const float* gval = sval + g0;
    const char* glb = reinterpret_cast<const char*>(q + hl);
    const uint32_t ld_bytes = ld8 * 8;
    const bool colok = hl < f8;

    auto ld_col = [&](uint32_t chunk) -> uint32_t {
        const uint32_t s = chunk * C + hl;
        return (hl < (uint32_t)C && s < total) ? ld_meta_u32(gcol + s) : 0u;
    };
    auto ld_val = [&](uint32_t chunk) -> float {
        const uint32_t s = chunk * C + hl;
        return (hl < (uint32_t)C && s < total) ? ld_meta_f32(gval + s) : 0.f;
    };
    auto issue = [&](int p, uint32_t col) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(ring0 + p * 128),
                     "l"(glb + (uint64_t)col * ld_bytes)
                     : "memory");
    };
    {
        const uint32_t mc0 = ld_col(0);
#pragma unroll
        for (int p = 0; p < C; ++p) {
            const uint32_t col = __shfl_sync(0xffffffffu, mc0, hbase + p);
            if ((uint32_t)p < total && colok) issue(p, col);
            cp_commit();
        }
    }
    uint32_t mc_is = ld_col(1), mc_nx = ld_col(2);
    float mv_cur = ld_val(0), mv_nx = ld_val(1);

    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    float4* crow = c + r0 * ldc4 + hl * 2;
    uint32_t row = 0;
    uint32_t row_end = __shfl_sync(0xffffffffu, rel, hbase);
    auto store_row = [&](uint32_t r) {
        if (colok) {  // F % 8 == 0 here: both float4 halves are in the row
            float4* dst = crow + (uint64_t)r * ldc4;
            __stcs(dst, make_float4(acc[0], acc[1], acc[2], acc[3]));
            __stcs(dst + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    };
    // half-uniform (divergent between halves): uses the half's lane mask
    auto advance_rows = [&](uint32_t pos) {
        do {
            store_row(row);
            ++row;
            row_end = __shfl_sync(hmask, rel, hbase + min(row, nr - 1));
        } while (row < nr && row_end == pos);
    };
    if (active && row_end == 0) advance_rows(0);

    auto decode_acc = [&](uint32_t r, int base, float v) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t off = __byte_perm(r, lane4, 0x6504u | (k << 4));  // (code << 8) | lane*4
            const float d = *reinterpret_cast<const float*>(smem_raw + off);
            acc[base + k] = __fadd_rn(acc[base + k], __fmul_rn(v, d));
        }
    };

    uint32_t kc = 0;
    for (uint32_t t0 = 0; t0 < total_max; t0 += C, ++kc) {
#pragma unroll
        for (int p = 0; p < C; ++p) {
            const uint32_t t = t0 + p;
            cp_wait<C - 1>();
            const float v = __shfl_sync(0xffffffffu, mv_cur, hbase + p);
            const bool live = t < total;
            if (live && colok) {
                uint2 r;
                asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(ring0 + p * 128));
                decode_acc(r.x, 0, v);
                decode_acc(r.y, 4, v);
            }
            const uint32_t col = __shfl_sync(0xffffffffu, mc_is, hbase + p);
            if (t + C < total && colok) issue(p, col);
            cp_commit();
            if (live && t + 1 == row_end) advance_rows(t + 1);
        }
        mv_cur = mv_nx;
        mc_is = mc_nx;
        mv_nx = ld_val(kc + 2);
        mc_nx = ld_col(kc + 3);
    }
    cp_wait<0>();
    if (active)
        while (row < nr) {
            store_row(row);
            ++row;
        }
}

template <int C, int WARPS>
int launch_q8_dual(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                   uint64_t ldq, uint32_t f8, float4* c, uint64_t ldc4, const float* lut, cudaStream_t st) {
    const size_t smem = 256 * 256 + (size_t)WARPS * 2 * C * 128;
    static bool attr_set_dev[kMaxDevices] = {};
    bool& attr_set = attr_set_dev[cur_device()];
    if (!attr_set) {
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_q8_dual_kernel<C, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        attr_set = true;
    }
    uint32_t gr = 16;  // row ends live in the 16 lanes of a half-warp
    while (gr > 2 && (n + gr - 1) / gr < (uint64_t)num_sms() * 128) gr >>= 1;
    const uint64_t groups = (n + gr - 1) / gr;
    const uint64_t warps = (groups + 1) / 2;
    const unsigned grid = (unsigned)((warps + WARPS - 1) / WARPS);
    spmm_q8_dual_kernel<C, WARPS><<<grid, WARPS * 32, smem, st>>>(srow, scol, sval, n,
                                                                   reinterpret_cast<const uint2*>(q),
                                                                   (uint32_t)(ldq / 8), f8, c, ldc4, lut, gr);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

// ---------------------------------------------------------------------------
// int8 batch kernel (F <= 128 codes, 16-B aligned code rows) — the default
// int8 path.  One warp, one flattened slot stream (as the fp32 ring: no
// half-warp divergence), but the gathers go out four slots per instruction:
// lane (g, j) = (lane / 8, lane % 8) copies bytes 16j..16j+15 of slot p0+g's
// code row with one 16-B LDGSTS, so the wait / commit / column shuffle /
// address arithmetic is paid once per four slots.  Consumption stays one slot
// at a time across the whole warp (lane l decodes codes 4l..4l+3), so the
// per-row accumulation order is the reference's slot order.
//
// Shared memory is one 64 KB block: the 256-entry LUT with a 256-B entry
// stride (lut[q] replicated per lane at q*256 + 4*lane, bank = lane, so
// PRMT(code, 4*lane) is the LDS offset — one PRMT + one LDS per code), and
// the per-warp gather rings in the upper 128 B of each entry ("holes"): ring
// slot p of warp w is hole w*C + p.
// ---------------------------------------------------------------------------
// DEC 0: the reference's global codes through the exact table (bit-exact);
// DEC 1: int8 FAST MODE per-feature affine codes, x^ = q s_j + m_j (affine.cu
// states the bounds): no table — PRMT places the byte in the mantissa of
// 2^23, one FADD2 per code pair removes 2^23, one FFMA2 per pair accumulates
// v q, and each stored row is s_j * acc + m_j * sum(v) (the same arithmetic
// as spmm_q8r_kernel, so the results are bit-identical to it)
template <int C, int WARPS, bool FULL, bool FASTB, int SCHED, int DEC = 0>  // SCHED: 0 static, 1 dynamic, 2 balanced
// 3 x 74 KB CTAs per SM (40 registers) for whole 128-code tiles; the partial-
// tile form (F % 128 != 0, e.g. reddit's 602) runs faster at 2 CTAs with room
// for 64 registers (reddit int8 0.64 -> 0.59 ms; products, whole tiles, loses
// 4-20 % that way)
__global__ void __launch_bounds__(WARPS * 32, WARPS >= 32 ? 1 : WARPS >= 20 ? 2 : FULL ? 3 : 2)
spmm_q8_batch_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                     const float* __restrict__ sval, uint64_t n_rows, const unsigned char* __restrict__ q,
                     uint32_t ldq, uint32_t f4, float4* __restrict__ c, uint64_t ldc4,
                     const float* __restrict__ lut_g, uint32_t group_rows, uint64_t groups, DynSched* ws,
                     const float2* __restrict__ fparams = nullptr, uint32_t fcols = 0) {
    static_assert(C % 4 == 0 && C >= 8 && C <= 16 && WARPS <= 32, "ring shape");
    // rings in the LUT's 256 holes (256-B stride) while they fit, else in
    // their own region after the row ends (128-B stride; one 32-warp CTA per
    // SM with room for 64 registers)
    constexpr bool kSep = C * WARPS > 256;
    constexpr uint32_t RS = kSep ? 128 : 256;
    constexpr int B = C / 4;  // batches per ring round
    constexpr uint32_t kEndsBytes = 144;  // 33 row ends per warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (DEC == 0) {
        for (int i = threadIdx.x; i < 256 * 32; i += WARPS * 32)
            reinterpret_cast<float*>(smem_raw)[(i >> 5) * 64 + (i & 31)] = lut_g[i >> 5];
        __syncthreads();
    }

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t smem0 = smem_addr(smem_raw);
    // LUT address of (code, lane) = smem0 + code*256 + lane*4.  The dynamic
    // window starts at a fixed offset (kDynSmemOffset) above the CTA's
    // window base (the high byte), so one PRMT builds base_hi | code<<8 |
    // lane*4 and the offset rides in the LDS immediate: no add per code.
    // A different layout would silently read wrong entries, so trap on it.
    if (DEC == 0 && (smem0 & 0xFFFFFFu) != kDynSmemOffset) __trap();
    // (pinned through asm so ptxas keeps them in registers instead of
    // re-deriving them from %tid in every slot)
    const uint32_t lane4 = pin_u32((smem0 & 0xFF000000u) | (lane * 4));
    // ring slot p of this warp: hole warp*C + p; lane reads its 4 codes at
    // rd0 + p*256 and copies its 16 B of batch slot p0 + lane/8 to wr0 + p0*256
    const uint32_t ring0 = kSep ? smem0 + 65536 + WARPS * (32 * C + kEndsBytes) + warp * (C * 128)
                                : smem0 + warp * (C * 256) + 128;
    const uint32_t rd0 = pin_u32(ring0 + lane * 4);
    const uint32_t wr0 = pin_u32(ring0 + (lane >> 3) * RS + (lane & 7) * 16);
    // slot metadata of ring round k: cols at meta0 + (k&3)*8C, vals 4C later
    const uint32_t meta0 = pin_u32(smem0 + 65536 + warp * (32 * C));
    const uint32_t mcol = pin_u32(meta0 + (lane >> 3) * 4);  // this lane's gather column, batch slot lane/8
    const uint32_t tl = pin_u32(lane >> 3);
    // column tile blockIdx.y: codes 128y.., output float4 columns 32y..
    q += (size_t)blockIdx.y * 128;
    c += (size_t)blockIdx.y * 32;
    const unsigned char* qlane = pin_ptr(q + (lane & 7) * 16);
    f4 = min(32u, f4 - blockIdx.y * 32);
    // DEC 1: (s_j, m_j) of this lane's 4 output columns of tile blockIdx.y
    float sj[4] = {0.f, 0.f, 0.f, 0.f}, mj[4] = {0.f, 0.f, 0.f, 0.f};
    if (DEC == 1) {  // (DEC 2 reads its row params per slot instead)
        const uint32_t col0 = blockIdx.y * 128 + 4 * lane;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (col0 + u < fcols) {
                const float2 pj = fparams[col0 + u];
                sj[u] = pj.x;
                mj[u] = pj.y;
            }
    }
    // the stored value of an output row (DEC 1: the affine epilogue)
    auto out4 = [&](const float4& a, float bsum) -> float4 {
        if (DEC == 0) return a;
        if (DEC == 2)
            return make_float4(__fadd_rn(a.x, bsum), __fadd_rn(a.y, bsum), __fadd_rn(a.z, bsum), __fadd_rn(a.w, bsum));
        return make_float4(fmaf(sj[0], a.x, mj[0] * bsum), fmaf(sj[1], a.y, mj[1] * bsum),
                           fmaf(sj[2], a.z, mj[2] * bsum), fmaf(sj[3], a.w, mj[3] * bsum));
    };
    uint32_t nb = 16;  // bytes this lane copies per slot
    if (!FULL) {
        const uint32_t rowb = f4 * 4, j16 = (lane & 7) * 16;
        nb = rowb > j16 ? min(16u, rowb - j16) : 0u;
    }

    const uint32_t ends0 = smem0 + 65536 + WARPS * 32 * C + warp * kEndsBytes;
    // DEC 2: the gathered rows' (s, m) pairs, 4 rounds x C slots x 8 B per warp
    const uint32_t par0 = smem0 + 65536 + WARPS * (32 * C + kEndsBytes) + (kSep ? WARPS * C * 128 : 0) +
                          warp * (32 * C);
    const float2* const rparams = fparams;

  // 32-row groups (static / dynamic schedules): one ring fill and drain per group
  auto run_group32 = [&](const uint64_t r0) {
    const uint32_t nr = (uint32_t)min((uint64_t)group_rows, n_rows - r0);
    const uint64_t g0 = srow[r0];
    const uint64_t my_end = srow[r0 + 1 + min(lane, nr - 1)];
    const uint32_t total = (uint32_t)(__shfl_sync(0xffffffffu, my_end, nr - 1) - g0);
    // row ends (relative to g0) in shared memory: ends[r] for r < nr, and
    // ends[r] = total for r >= nr, so advance_rows needs no shuffle
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + lane * 4), "r"((uint32_t)(my_end - g0)) : "memory");
    if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + 128), "r"(total) : "memory");
    __syncwarp();

    // metadata of round k -> buffer k & 3 (lanes 0..C-1: cols, 16..16+C-1: vals)
    // (lanes 0..15 stream scol, 16..31 sval: one per-lane base pointer)
    const char* const mbase = lane < 16 ? reinterpret_cast<const char*>(scol + g0 + (lane & 15))
                                        : reinterpret_cast<const char*>(sval + g0 + (lane & 15));
    const uint32_t mdst = meta0 + (lane >> 4) * (4 * C) + (lane & 15) * 4;
    auto issue_meta = [&](uint32_t k) {
        const uint32_t i = lane & 15, s = k * C + i;
        if (i < (uint32_t)C && s < total) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(mdst + (k & 3) * (8 * C)),
                         "l"(mbase + (uint64_t)(k * C) * 4)
                         : "memory");
        }
    };
    // gathers for ring positions p0..p0+3 of round k (slots k*C + p0 ..);
    // every per-lane term is pinned (qlane, mcol, tl), so the issue is one
    // compare, one LDS, one IMAD.WIDE and the LDGSTS
    auto issue = [&](int p0, uint32_t k) {
        const uint32_t t = k * C + p0 + tl;
        if (t < total && (FULL || nb != 0)) {
            const uint32_t col = lds_u32(mcol + (k & 3) * (8 * C) + p0 * 4);
            const unsigned char* src = qlane + (uint64_t)col * ldq;
            if (FULL)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(wr0 + p0 * RS), "l"(src)
                             : "memory");
            else
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(wr0 + p0 * RS), "l"(src),
                             "r"(nb)
                             : "memory");
        }
    };
    // DEC 2: (s, m) of round k's gathered rows -> params buffer k & 3 (the
    // round's columns are in shared memory by then)
    auto issue_par = [&](uint32_t k) {
        if (DEC == 2 && lane < (uint32_t)C && k * C + lane < total) {
            const uint32_t col = lds_u32(meta0 + (k & 3) * (8 * C) + lane * 4);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(par0 + (k & 3) * (8 * C) + lane * 8),
                         "l"(rparams + col)
                         : "memory");
        }
    };
    issue_meta(0);
    issue_meta(1);
    cp_commit();
    cp_wait<0>();
    __syncwarp();
    issue_par(0);
#pragma unroll
    for (int b = 0; b < B; ++b) {
        issue(4 * b, 0);
        cp_commit();
    }
    uint32_t parr = par0;  // params of the round being consumed

    float4 acc = f4_zero();
    uint32_t row = 0;
    uint32_t row_end = lds_u32(ends0);
    float4* cptr = c + r0 * ldc4 + lane;  // rows are stored in order: a running pointer
    float bs = 0.f;  // DEC 1: sum of the row's slot values
    auto store_row = [&](uint32_t) {
        if (FULL || lane < f4) __stcs(cptr, out4(acc, bs));
        cptr += ldc4;
        acc = f4_zero();
        bs = 0.f;
    };
    auto advance_rows = [&](uint32_t pos) {
        do {
            store_row(row);
            ++row;
            row_end = lds_u32(ends0 + row * 4);
        } while (row < nr && row_end == pos);
    };
    if (row_end == 0) advance_rows(0);

    auto consume = [&](int p, float v) {
        const uint32_t r = lds_u32(rd0 + p * RS);
        if (DEC != 0) {
            float q0 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7650));
            float q1 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7651));
            float q2 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7652));
            float q3 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7653));
            add2_rn(q0, q1, -8388608.0f, -8388608.0f);  // exactly q
            add2_rn(q2, q3, -8388608.0f, -8388608.0f);
            float a = v, bv = v;
            if (DEC == 2) {  // per-row codes: v s_c scales the codes, v m_c the offset
                float2 sm;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(sm.x), "=f"(sm.y) : "r"(parr + p * 8));
                bv = __fmul_rn(v, sm.y);
                a = __fmul_rn(v, sm.x);
            }
            fma2_rn(acc.x, acc.y, a, q0, q1);
            fma2_rn(acc.z, acc.w, a, q2, q3);
            bs = __fadd_rn(bs, bv);  // (no contraction: the same bits as spmm_q8r_kernel)
            return;
        }
        const float d0 = lds_lut(__byte_perm(r, lane4, 0x7604u));
        const float d1 = lds_lut(__byte_perm(r, lane4, 0x7614u));
        const float d2 = lds_lut(__byte_perm(r, lane4, 0x7624u));
        const float d3 = lds_lut(__byte_perm(r, lane4, 0x7634u));
        add2_rn(acc.x, acc.y, __fmul_rn(v, d0), __fmul_rn(v, d1));
        add2_rn(acc.z, acc.w, __fmul_rn(v, d2), __fmul_rn(v, d3));
    };

    // Every round consumes all C ring positions: positions past `total`
    // (only in the last round) accumulate garbage into acc AFTER the group's
    // last row was stored — no row ends there, so nothing of it is written.
    for (uint32_t k = 0, t0 = 0; t0 < total; t0 += C, ++k) {
        parr = par0 + (k & 3) * (8 * C);
#pragma unroll
        for (int b = 0; b < B; ++b) {
            cp_wait<B - 1>();
            __syncwarp();  // other lanes' copies of these four slots are visible
            float4 v4;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v4.x), "=f"(v4.y), "=f"(v4.z), "=f"(v4.w)
                         : "r"(meta0 + (k & 3) * (8 * C) + 4 * C + 16 * b));
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
            if (FASTB && row_end > t0 + 4 * b + 4) {  // no row ends in this batch
#pragma unroll
                for (int u = 0; u < 4; ++u) consume(4 * b + u, vv[u]);
            } else {
                const uint32_t base = t0 + 4 * b + 1;  // position after this batch's first slot
                uint32_t rel = row_end - base;           // the row ends after slot 4b + rel
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    consume(4 * b + u, vv[u]);
                    if (rel == (uint32_t)u) {
                        advance_rows(base + u);
                        rel = row_end - base;
                    }
                }
            }
            __syncwarp();  // every lane is done reading these holes
            if (b == 0) {
                issue_meta(k + 2);
                issue_par(k + 1);  // round k+1's columns landed with the wait above
            }
            issue(4 * b, k + 1);
            cp_commit();
        }
    }
    cp_wait<0>();
    while (row < nr) {
        store_row(row);
        ++row;
    }
    __syncwarp();  // the next group reuses this warp's ring, metadata and row ends
  };

  // rows [rb, re) as one slot stream (srow[re] - srow[rb] < 2^31); row ends
  // relative to the first slot in a 32-row shared-memory window
  auto run_range = [&](const uint64_t rb, const uint64_t re) {
    const uint64_t g0 = srow[rb];
    const uint32_t total = (uint32_t)(srow[re] - g0);
    const uint32_t nrows = (uint32_t)(re - rb);  // >= 1
    const uint64_t* rend = srow + rb + 1;         // end of row rb + i at rend[i]
    float4* const crow = c + rb * ldc4 + lane;
    auto window = [&](uint32_t w) -> uint32_t { return (uint32_t)(rend[min(w + lane, nrows - 1)] - g0); };
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + lane * 4), "r"(window(0)) : "memory");
    __syncwarp();

    // metadata of round k -> buffer k & 3 (lanes 0..C-1: cols, 16..16+C-1: vals)
    // (lanes 0..15 stream scol, 16..31 sval: one per-lane base pointer)
    const char* const mbase = lane < 16 ? reinterpret_cast<const char*>(scol + g0 + (lane & 15))
                                        : reinterpret_cast<const char*>(sval + g0 + (lane & 15));
    const uint32_t mdst = meta0 + (lane >> 4) * (4 * C) + (lane & 15) * 4;
    auto issue_meta = [&](uint32_t k) {
        const uint32_t i = lane & 15, s = k * C + i;
        if (i < (uint32_t)C && s < total) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(mdst + (k & 3) * (8 * C)),
                         "l"(mbase + (uint64_t)(k * C) * 4)
                         : "memory");
        }
    };
    // gathers for ring positions p0..p0+3 of round k (slots k*C + p0 ..);
    // every per-lane term is pinned (qlane, mcol, tl), so the issue is one
    // compare, one LDS, one IMAD.WIDE and the LDGSTS
    auto issue = [&](int p0, uint32_t k) {
        const uint32_t t = k * C + p0 + tl;
        if (t < total && (FULL || nb != 0)) {
            const uint32_t col = lds_u32(mcol + (k & 3) * (8 * C) + p0 * 4);
            const unsigned char* src = qlane + (uint64_t)col * ldq;
            if (FULL)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(wr0 + p0 * RS), "l"(src)
                             : "memory");
            else
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(wr0 + p0 * RS), "l"(src),
                             "r"(nb)
                             : "memory");
        }
    };
    // DEC 2: (s, m) of round k's gathered rows -> params buffer k & 3 (the
    // round's columns are in shared memory by then)
    auto issue_par = [&](uint32_t k) {
        if (DEC == 2 && lane < (uint32_t)C && k * C + lane < total) {
            const uint32_t col = lds_u32(meta0 + (k & 3) * (8 * C) + lane * 4);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(par0 + (k & 3) * (8 * C) + lane * 8),
                         "l"(rparams + col)
                         : "memory");
        }
    };
    issue_meta(0);
    issue_meta(1);
    cp_commit();
    cp_wait<0>();
    __syncwarp();
    issue_par(0);
#pragma unroll
    for (int b = 0; b < B; ++b) {
        issue(4 * b, 0);
        cp_commit();
    }
    uint32_t parr = par0;  // params of the round being consumed

    float4 acc = f4_zero();
    uint32_t ri = 0;  // next row to store (relative to rb)
    uint32_t wi = 0;  // its index in the window
    uint32_t row_end = lds_u32(ends0);
    float4* cptr = crow;  // rows are stored in order: a running pointer
    float bs = 0.f;  // DEC 1: sum of the row's slot values
    auto store_row = [&]() {
        if (FULL || lane < f4) __stcs(cptr, out4(acc, bs));
        cptr += ldc4;
        acc = f4_zero();
        bs = 0.f;
    };
    auto advance_rows = [&](uint32_t pos) {
        do {
            store_row();
            ++ri;
            if (++wi == 32) {  // enter the next window (its load latency is
                wi = 0;            // covered by the SM's other warps: issue-bound)
                const uint32_t e = window(ri);
                __syncwarp();
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + lane * 4), "r"(e) : "memory");
                __syncwarp();
            }
            row_end = lds_u32(ends0 + wi * 4);
        } while (ri < nrows && row_end == pos);
    };
    if (row_end == 0) advance_rows(0);

    auto consume = [&](int p, float v) {
        const uint32_t r = lds_u32(rd0 + p * RS);
        if (DEC != 0) {
            float q0 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7650));
            float q1 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7651));
            float q2 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7652));
            float q3 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7653));
            add2_rn(q0, q1, -8388608.0f, -8388608.0f);  // exactly q
            add2_rn(q2, q3, -8388608.0f, -8388608.0f);
            float a = v, bv = v;
            if (DEC == 2) {  // per-row codes: v s_c scales the codes, v m_c the offset
                float2 sm;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(sm.x), "=f"(sm.y) : "r"(parr + p * 8));
                bv = __fmul_rn(v, sm.y);
                a = __fmul_rn(v, sm.x);
            }
            fma2_rn(acc.x, acc.y, a, q0, q1);
            fma2_rn(acc.z, acc.w, a, q2, q3);
            bs = __fadd_rn(bs, bv);  // (no contraction: the same bits as spmm_q8r_kernel)
            return;
        }
        const float d0 = lds_lut(__byte_perm(r, lane4, 0x7604u));
        const float d1 = lds_lut(__byte_perm(r, lane4, 0x7614u));
        const float d2 = lds_lut(__byte_perm(r, lane4, 0x7624u));
        const float d3 = lds_lut(__byte_perm(r, lane4, 0x7634u));
        add2_rn(acc.x, acc.y, __fmul_rn(v, d0), __fmul_rn(v, d1));
        add2_rn(acc.z, acc.w, __fmul_rn(v, d2), __fmul_rn(v, d3));
    };

    // Every round consumes all C ring positions: positions past `total`
    // (only in the last round) accumulate garbage into acc AFTER the group's
    // last row was stored — no row ends there, so nothing of it is written.
    for (uint32_t k = 0, t0 = 0; t0 < total; t0 += C, ++k) {
        parr = par0 + (k & 3) * (8 * C);
#pragma unroll
        for (int b = 0; b < B; ++b) {
            cp_wait<B - 1>();
            __syncwarp();  // other lanes' copies of these four slots are visible
            float4 v4;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v4.x), "=f"(v4.y), "=f"(v4.z), "=f"(v4.w)
                         : "r"(meta0 + (k & 3) * (8 * C) + 4 * C + 16 * b));
            const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
            if (FASTB && row_end > t0 + 4 * b + 4) {  // no row ends in this batch
#pragma unroll
                for (int u = 0; u < 4; ++u) consume(4 * b + u, vv[u]);
            } else {
                const uint32_t base = t0 + 4 * b + 1;  // position after this batch's first slot
                uint32_t rel = row_end - base;           // the row ends after slot 4b + rel
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    consume(4 * b + u, vv[u]);
                    if (rel == (uint32_t)u) {
                        advance_rows(base + u);
                        rel = row_end - base;
                    }
                }
            }
            __syncwarp();  // every lane is done reading these holes
            if (b == 0) {
                issue_meta(k + 2);
                issue_par(k + 1);  // round k+1's columns landed with the wait above
            }
            issue(4 * b, k + 1);
            cp_commit();
        }
    }
    cp_wait<0>();
    for (; ri < nrows; ++ri) store_row();  // (only when the range has no slots)
    __syncwarp();  // the next range reuses this warp's ring, metadata and row ends
  };

    if (SCHED == 0) {  // 32-row groups, grid-stride (one group per warp unless the grid is persistent)
        for (uint64_t gi = (uint64_t)blockIdx.x * WARPS + warp; gi < groups; gi += (uint64_t)gridDim.x * WARPS)
            run_group32(gi * group_rows);
        return;
    }
    if (SCHED == 2) {  // balanced persistent: this warp's slot-balanced row range
        uint64_t rb, re;
        bal_range(srow, n_rows, (uint64_t)blockIdx.x * WARPS + warp, (uint64_t)gridDim.x * WARPS, rb, re);
        while (rb < re) {  // slices with 32-bit slot offsets (one slice at the BASELINE shapes)
            const uint64_t e = srow[re] - srow[rb] >= (1ull << 31) ? rb + 1 : re;
            run_range(rb, e);
            rb = e;
        }
        return;
    }
    // heavy-first tickets (see spmm_ring_dyn_kernel), one counter per column tile
    unsigned int* next = ws->heavy + groups + blockIdx.y;
    const uint64_t n_heavy = *reinterpret_cast<volatile unsigned int*>(&ws->n_heavy);
    const uint64_t n_items = n_heavy + groups;
    uint64_t w = 0;
    if (lane == 0) w = atomicAdd(next, 1u);
    w = __shfl_sync(0xffffffffu, w, 0);
    while (w < n_items) {
        uint64_t nw = 0;
        if (lane == 0) nw = atomicAdd(next, 1u);
        nw = __shfl_sync(0xffffffffu, nw, 0);
        const uint64_t g = w < n_heavy ? (uint64_t)ws->heavy[w] : w - n_heavy;
        if (w < n_heavy || !group_is_heavy(srow, n_rows, group_rows, g)) run_group32(g * group_rows);
        w = nw;
    }
}

// Balanced schedule: `waves` x resident CTAs, every warp one equal-work row
// range.  Measured on B200 (scripts/shard_scaling.py, products W=32):
//  * fp32 ring: one wave is 8 % slower than the static grid on the full graph
//    (1.28 vs 1.18 ms: with every warp far apart the C-row writes and the
//    metadata streams lose their locality); ~20-row ranges in successive
//    waves keep the active rows contiguous and match it (1.18 ms), while at
//    P = 8 the shards still end in whole waves (0.169 vs 0.177 ms);
//  * int8 batch kernel: one wave is best (each extra wave re-fills the 64 KB
//    LUT per CTA): 0.59 ms full graph, 0.095 vs 0.107 ms at P = 8.
// AES_SPMM_BAL_WAVES overrides the count (tuning only).
uint32_t bal_waves(uint64_t n_rows, uint64_t resident_warps, uint64_t rows_per_range) {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("AES_SPMM_BAL_WAVES");
        env = e ? atoi(e) : 0;
    }
    if (env > 0) return (uint32_t)env;
    if (rows_per_range == 0 || resident_warps == 0) return 1;
    const uint64_t w = n_rows / (resident_warps * rows_per_range);
    return (uint32_t)(w < 1 ? 1 : w > 64 ? 64 : w);
}

template <int C, int WARPS, bool FULL, bool FASTB, int DEC = 0>
int launch_q8_batch_t(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                      uint64_t ldq, uint32_t f4, float4* c, uint64_t ldc4, const float* lut, cudaStream_t st,
                      int dyn, const float2* fparams = nullptr, uint32_t fcols = 0) {
    // LUT (+ rings in its holes), slot metadata, row ends (+ separate rings)
    const size_t smem = 256 * 256 + (size_t)WARPS * (32 * C + 144) + (C * WARPS > 256 ? (size_t)WARPS * C * 128 : 0) +
                        (DEC == 2 ? (size_t)WARPS * 32 * C : 0);  // (+ the per-row params buffers)
    static int occ_dev[kMaxDevices] = {};
    int& occ = occ_dev[cur_device()];
    if (occ == 0) {
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_q8_batch_kernel<C, WARPS, FULL, FASTB, 0, DEC>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_q8_batch_kernel<C, WARPS, FULL, FASTB, 1, DEC>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AES_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &occ, spmm_q8_batch_kernel<C, WARPS, FULL, FASTB, 1, DEC>, WARPS * 32, smem));
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_q8_batch_kernel<C, WARPS, FULL, FASTB, 2, DEC>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (occ < 1) occ = 1;
    }
    // 128-code column tiles run side by side as blockIdx.y; rows per warp
    // shrink until (row groups x tiles) fills >= 64 warps per SM
    const uint32_t tiles = (f4 + 31) / 32;
    uint32_t gr = 32;
    while (gr > 2 && (n + gr - 1) / gr * tiles < (uint64_t)num_sms() * 64) gr >>= 1;
    const uint64_t groups = (n + gr - 1) / gr;
    const unsigned gx = (unsigned)((groups + WARPS - 1) / WARPS);
    // auto: the 32-row-group grid when it runs >= 4 waves (0.56 ms on the
    // full products graph, vs 0.59-0.60 balanced), the balanced wave when it
    // would end in a partial wave (row shards: P = 8 0.107 -> 0.095 ms)
    // (one 32-warp CTA per SM: balanced always — a single wave fills the
    // 64 KB table once per SM, 0.51 vs 0.59 ms static on products)
    if (dyn == kSchedAuto)
        dyn = WARPS >= 32 || gx * tiles < 4ull * num_sms() * occ ? kSchedBal : kSchedStatic;
    if (dyn == kSchedBal || dyn == kSchedBalOne) {  // one wave of resident CTAs per column tile
        // whole waves: the tiles share the resident CTA slots (rounding up
        // would leave one CTA for a second, nearly empty wave)
        const uint64_t per_wave = (uint64_t)num_sms() * occ / tiles;
        uint64_t per_tile = (per_wave ? per_wave : 1) * bal_waves(n, per_wave * WARPS, 0);
        // small graphs (pubmed: 20 k rows): at least 8 rows per warp (4 for
        // the one-CTA-per-SM form, which would otherwise leave half the SMs
        // idle), so the 64 KB LUT fill of a CTA is not paid for a handful of slots
        const uint64_t min_rows = WARPS >= 32 ? 4 : 8;
        const uint64_t cap = (n + (uint64_t)WARPS * min_rows - 1) / ((uint64_t)WARPS * min_rows);
        if (cap < per_tile) per_tile = cap ? cap : 1;
        spmm_q8_batch_kernel<C, WARPS, FULL, FASTB, 2, DEC><<<dim3((unsigned)per_tile, tiles), WARPS * 32, smem, st>>>(
            srow, scol, sval, n, q, (uint32_t)ldq, f4, c, ldc4, lut, 32, 0, nullptr, fparams, fcols);
        AES_CUDA_TRY(cudaGetLastError());
        return AES_OK;
    }
    if (dyn == kSchedDyn && groups < (1ull << 31)) {
        DynSched* ws = nullptr;
        const size_t ws_bytes = sizeof(DynSched) + (groups + tiles) * sizeof(unsigned int);
        AES_CUDA_TRY(cudaMallocAsync((void**)&ws, ws_bytes, st));
        AES_CUDA_TRY(cudaMemsetAsync(ws, 0, 16, st));
        AES_CUDA_TRY(cudaMemsetAsync(reinterpret_cast<unsigned int*>(ws->heavy) + groups, 0, tiles * 4, st));
        heavy_scan_kernel<<<grid_for(groups, 256, num_sms() * 8), 256, 0, st>>>(srow, n, gr, groups, ws);
        const uint64_t per_tile = ((uint64_t)num_sms() * occ + tiles - 1) / tiles;
        const dim3 grid((unsigned)(gx < per_tile ? gx : per_tile), tiles);
        spmm_q8_batch_kernel<C, WARPS, FULL, FASTB, 1, DEC><<<grid, WARPS * 32, smem, st>>>(
            srow, scol, sval, n, q, (uint32_t)ldq, f4, c, ldc4, lut, gr, groups, ws, fparams, fcols);
        AES_CUDA_TRY(cudaGetLastError());
        AES_CUDA_TRY(cudaFreeAsync(ws, st));
        return AES_OK;
    }
    // static: one 32-row group per warp; the hardware block scheduler balances
    // the CTAs (products 0.56 ms).  A persistent grid-stride grid fills the
    // 64 KB table once per SM slot but loses that balancing (0.61 ms), so it
    // is tuning-only (kSchedStaticPersist).
    uint64_t gs = (uint64_t)num_sms() * occ / tiles;
    if (gs == 0) gs = 1;
    const unsigned gxs = (unsigned)(dyn == kSchedStaticPersist && gx > gs ? gs : gx);
    spmm_q8_batch_kernel<C, WARPS, FULL, FASTB, 0, DEC><<<dim3(gxs, tiles), WARPS * 32, smem, st>>>(
        srow, scol, sval, n, q, (uint32_t)ldq, f4, c, ldc4, lut, gr, groups, nullptr, fparams, fcols);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

template <int C, int WARPS, bool FASTB = true, int DEC = 0>
int launch_q8_batch(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                    uint64_t ldq, uint32_t f4, float4* c, uint64_t ldc4, const float* lut, cudaStream_t st,
                    int dyn, const float2* fparams = nullptr, uint32_t fcols = 0) {
    if (f4 % 32 == 0)
        return launch_q8_batch_t<C, WARPS, true, FASTB, DEC>(srow, scol, sval, n, q, ldq, f4, c, ldc4, lut, st, dyn,
                                                             fparams, fcols);
    return launch_q8_batch_t<C, WARPS, false, FASTB, DEC>(srow, scol, sval, n, q, ldq, f4, c, ldc4, lut, st, dyn,
                                                          fparams, fcols);
}

// ---------------------------------------------------------------------------
// int8 wide-row kernel (exact global codes, 128 < F <= 128 T, 16-B aligned
// code rows).  The batch kernel runs wide rows as 128-code column tiles on
// grid.y, so every tile pays the whole per-slot bookkeeping again (metadata
// cp.async, the value LDS.128, the column LDS of each gather issue, row-end
// tests): reddit F = 602 pays it 5 times per slot, and its last tile is 70 %
// full.  Here ONE warp covers the whole code row: lane l decodes codes
// 128t + 4l .. 128t + 4l + 3 of every group t < T into accumulator t, so the
// bookkeeping is paid once per slot and only the decode (ring LDS, 4 PRMT +
// 4 LUT LDS, 4 FMUL, 2 FADD2 per group) scales with F.  Gathers: per 4-slot
// batch, T LDGSTS.128 per lane — lane (g, j) copies bytes 128t + 16j .. of
// slot p0 + g, zero-filled past the row's bytes (only group T-1 is partial).
// The LUT layout, metadata pipeline and balanced row ranges are the batch
// kernel's (SCHED 2); each output element is the same slot-order FMUL/FADD
// chain, so the results are bit-identical to it.  DEC 1 (int8 FAST MODE,
// per-feature codes) is the batch kernel's table-free decode and affine
// epilogue, (s_j, m_j) staged in shared memory once per CTA; DEC 2 (per-row codes) stages
// the gathered rows' (s, m) next to the slot metadata — again the same bits.
// ---------------------------------------------------------------------------
template <int T, int C, int WARPS, int DEC = 0>
__global__ void __launch_bounds__(WARPS * 32, 1)
spmm_q8_wide_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                    const float* __restrict__ sval, uint64_t n_rows, const unsigned char* __restrict__ q,
                    uint32_t ldq, uint32_t f4, float4* __restrict__ c, uint64_t ldc4,
                    const float* __restrict__ lut_g, const float2* __restrict__ fparams = nullptr,
                    uint32_t fcols = 0) {
    static_assert(DEC >= 0 && DEC <= 2, "wide kernel decodes: global table, per-feature or per-row affine");
    static_assert(T >= 1 && T <= 8 && C % 4 == 0 && C >= 8 && C <= 16, "wide ring shape");
    constexpr int B = C / 4;               // batches per ring round
    constexpr uint32_t RS = 128 * T;       // ring slot stride (one whole code row)
    constexpr bool kRolledEnds = true;     // batches holding a row end: rolled slot loop
    constexpr uint32_t kEndsBytes = 144;   // 33 row ends per warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (DEC == 0) {
        for (int i = threadIdx.x; i < 256 * 32; i += WARPS * 32)
            reinterpret_cast<float*>(smem_raw)[(i >> 5) * 64 + (i & 31)] = lut_g[i >> 5];
        __syncthreads();
    }

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t smem0 = smem_addr(smem_raw);
    if (DEC == 0 && (smem0 & 0xFFFFFFu) != kDynSmemOffset) __trap();  // see dyn_smem_offset_ok
    const uint32_t lane4 = pin_u32((smem0 & 0xFF000000u) | (lane * 4));
    const uint32_t meta0 = pin_u32(smem0 + 65536 + warp * (32 * C));
    const uint32_t ends0 = smem0 + 65536 + WARPS * 32 * C + warp * kEndsBytes;
    const uint32_t ring0 = smem0 + 65536 + WARPS * (32 * C + kEndsBytes) + warp * (C * RS);
    // DEC 2: the gathered rows' (s, m) pairs, 4 rounds x C slots x 8 B per warp
    const uint32_t par0 = smem0 + 65536 + WARPS * (32 * C + kEndsBytes + C * RS) + warp * (32 * C);
    // DEC 1: (s_j, m_j) of every column, staged once per CTA (zero past F)
    constexpr uint32_t kFparOff = 65536 + WARPS * (32 * C + kEndsBytes + C * RS);
    const uint32_t fpar0 = smem0 + kFparOff;
    if (DEC == 1) {
        float2* fp = reinterpret_cast<float2*>(smem_raw + kFparOff);
        for (uint32_t j = threadIdx.x; j < 128 * T; j += WARPS * 32)
            fp[j] = j < fcols ? fparams[j] : make_float2(0.f, 0.f);
        __syncthreads();
    }
    const uint32_t rd0 = pin_u32(ring0 + lane * 4);
    const uint32_t wr0 = pin_u32(ring0 + (lane >> 3) * RS + (lane & 7) * 16);
    const uint32_t mcol = pin_u32(meta0 + (lane >> 3) * 4);
    const uint32_t tl = pin_u32(lane >> 3);
    const unsigned char* qlane = pin_ptr(q + (lane & 7) * 16);
    // bytes this lane copies of group T-1 (groups < T-1 are whole)
    const uint32_t offl = 128 * (T - 1) + (lane & 7) * 16, rowb = f4 * 4;
    const uint32_t nbl = rowb > offl ? min(16u, rowb - offl) : 0u;
    const bool stl = 32 * (T - 1) + lane < f4;  // this lane stores group T-1

    uint64_t rb, re;
    bal_range(srow, n_rows, (uint64_t)blockIdx.x * WARPS + warp, (uint64_t)gridDim.x * WARPS, rb, re);
    while (rb < re) {
        // slices with 32-bit slot offsets (one slice at the BASELINE shapes)
        const uint64_t re1 = srow[re] - srow[rb] >= (1ull << 31) ? rb + 1 : re;
        const uint64_t g0 = srow[rb];
        const uint32_t total = (uint32_t)(srow[re1] - g0);
        const uint32_t nrows = (uint32_t)(re1 - rb);
        const uint64_t* rend = srow + rb + 1;  // end of row rb + i at rend[i]
        auto window = [&](uint32_t w) -> uint32_t { return (uint32_t)(rend[min(w + lane, nrows - 1)] - g0); };
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + lane * 4), "r"(window(0)) : "memory");
        __syncwarp();

        // metadata of round k -> buffer k & 3 (lanes 0..C-1: cols, 16..16+C-1: vals)
        const char* const mbase = lane < 16 ? reinterpret_cast<const char*>(scol + g0 + (lane & 15))
                                            : reinterpret_cast<const char*>(sval + g0 + (lane & 15));
        const uint32_t mdst = meta0 + (lane >> 4) * (4 * C) + (lane & 15) * 4;
        auto issue_meta = [&](uint32_t k) {
            const uint32_t i = lane & 15, s = k * C + i;
            if (i < (uint32_t)C && s < total)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(mdst + (k & 3) * (8 * C)),
                             "l"(mbase + (uint64_t)(k * C) * 4)
                             : "memory");
        };
        auto issue = [&](int p0, uint32_t k) {
            if (k * C + p0 + tl < total) {
                const uint32_t col = lds_u32(mcol + (k & 3) * (8 * C) + p0 * 4);
                const unsigned char* src = qlane + (uint64_t)col * ldq;
                const uint32_t dst = wr0 + p0 * RS;
#pragma unroll
                for (int t = 0; t < T - 1; ++t)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 128 * t),
                                 "l"(src + 128 * t)
                                 : "memory");
                if (nbl != 0)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + 128 * (T - 1)),
                                 "l"(src + 128 * (T - 1)), "r"(nbl)
                                 : "memory");
            }
        };
        // DEC 2: (s, m) of round k's gathered rows -> params buffer k & 3 (the
        // round's columns are in shared memory by then)
        auto issue_par = [&](uint32_t k) {
            if (DEC == 2 && lane < (uint32_t)C && k * C + lane < total) {
                const uint32_t col = lds_u32(meta0 + (k & 3) * (8 * C) + lane * 4);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(par0 + (k & 3) * (8 * C) + lane * 8),
                             "l"(fparams + col)
                             : "memory");
            }
        };
        issue_meta(0);
        issue_meta(1);
        cp_commit();
        cp_wait<0>();
        __syncwarp();
        issue_par(0);
#pragma unroll
        for (int b = 0; b < B; ++b) {
            issue(4 * b, 0);
            cp_commit();
        }
        uint32_t parr = par0;  // DEC 2: params of the round being consumed

        float4 acc[T];
#pragma unroll
        for (int t = 0; t < T; ++t) acc[t] = f4_zero();
        uint32_t ri = 0;  // next row to store (relative to rb)
        uint32_t wi = 0;  // its index in the window
        uint32_t row_end = lds_u32(ends0);
        float4* cptr = c + rb * ldc4 + lane;  // rows are stored in order: a running pointer
        float bs = 0.f;  // DEC 1: sum of the row's slot values
        auto out4 = [&](int t) -> float4 {
            if (DEC == 0) return acc[t];
            if (DEC == 2)
                return make_float4(__fadd_rn(acc[t].x, bs), __fadd_rn(acc[t].y, bs), __fadd_rn(acc[t].z, bs),
                                   __fadd_rn(acc[t].w, bs));
            float sj[4], mj[4];  // (s, m) of columns 128t + 4 lane .. + 3: two LDS.128
            const uint32_t pa = fpar0 + (128 * t + 4 * lane) * 8;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(sj[0]), "=f"(mj[0]), "=f"(sj[1]), "=f"(mj[1]) : "r"(pa));
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(sj[2]), "=f"(mj[2]), "=f"(sj[3]), "=f"(mj[3]) : "r"(pa + 16));
            const float4& a = acc[t];
            return make_float4(fmaf(sj[0], a.x, mj[0] * bs), fmaf(sj[1], a.y, mj[1] * bs),
                               fmaf(sj[2], a.z, mj[2] * bs), fmaf(sj[3], a.w, mj[3] * bs));
        };
        auto store_row = [&]() {
#pragma unroll
            for (int t = 0; t < T - 1; ++t) __stcs(cptr + 32 * t, out4(t));
            if (stl) __stcs(cptr + 32 * (T - 1), out4(T - 1));
            cptr += ldc4;
#pragma unroll
            for (int t = 0; t < T; ++t) acc[t] = f4_zero();
            bs = 0.f;
        };
        auto advance_rows = [&](uint32_t pos) {
            do {
                store_row();
                ++ri;
                if (++wi == 32) {  // enter the next 32-row window of row ends
                    wi = 0;
                    const uint32_t e = window(ri);
                    __syncwarp();
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + lane * 4), "r"(e) : "memory");
                    __syncwarp();
                }
                row_end = lds_u32(ends0 + wi * 4);
            } while (ri < nrows && row_end == pos);
        };
        if (row_end == 0) advance_rows(0);

        auto consume = [&](int p, float v) {
            if (DEC != 0) {
                float a = v, bv = v;
                if (DEC == 2) {  // per-row codes: v s_c scales the codes, v m_c the offset
                    float2 sm;
                    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(sm.x), "=f"(sm.y) : "r"(parr + p * 8));
                    bv = __fmul_rn(v, sm.y);
                    a = __fmul_rn(v, sm.x);
                }
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const uint32_t r = lds_u32(rd0 + p * RS + 128 * t);
                    float q0 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7650));
                    float q1 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7651));
                    float q2 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7652));
                    float q3 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7653));
                    add2_rn(q0, q1, -8388608.0f, -8388608.0f);  // exactly q
                    add2_rn(q2, q3, -8388608.0f, -8388608.0f);
                    fma2_rn(acc[t].x, acc[t].y, a, q0, q1);
                    fma2_rn(acc[t].z, acc[t].w, a, q2, q3);
                }
                bs = __fadd_rn(bs, bv);  // (no contraction: the batch kernel's bits)
                return;
            }
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const uint32_t r = lds_u32(rd0 + p * RS + 128 * t);
                const float d0 = lds_lut(__byte_perm(r, lane4, 0x7604u));
                const float d1 = lds_lut(__byte_perm(r, lane4, 0x7614u));
                const float d2 = lds_lut(__byte_perm(r, lane4, 0x7624u));
                const float d3 = lds_lut(__byte_perm(r, lane4, 0x7634u));
                add2_rn(acc[t].x, acc[t].y, __fmul_rn(v, d0), __fmul_rn(v, d1));
                add2_rn(acc[t].z, acc[t].w, __fmul_rn(v, d2), __fmul_rn(v, d3));
            }
        };

        // positions past `total` (last round only) accumulate garbage after
        // the range's last row was stored — never written
        for (uint32_t k = 0, t0 = 0; t0 < total; t0 += C, ++k) {
            parr = par0 + (k & 3) * (8 * C);
#pragma unroll
            for (int b = 0; b < B; ++b) {
                cp_wait<B - 1>();
                __syncwarp();  // other lanes' copies of these four slots are visible
                float4 v4;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v4.x), "=f"(v4.y), "=f"(v4.z), "=f"(v4.w)
                             : "r"(meta0 + (k & 3) * (8 * C) + 4 * C + 16 * b));
                const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
                if (row_end > t0 + 4 * b + 4) {  // no row ends in this batch
#pragma unroll
                    for (int u = 0; u < 4; ++u) consume(4 * b + u, vv[u]);
                } else if (kRolledEnds) {
                    // rolled: advance_rows (the per-feature epilogue above
                    // all) is inlined once per batch instead of four times,
                    // which keeps the kernel inside the instruction cache
                    const uint32_t base = t0 + 4 * b + 1;
                    uint32_t rel = row_end - base;
                    const uint32_t va = meta0 + (k & 3) * (8 * C) + 4 * C + 16 * b;
#pragma unroll 1
                    for (uint32_t u = 0; u < 4; ++u) {
                        consume(4 * b + (int)u, lds_f32(va + 4 * u));
                        if (rel == u) {
                            advance_rows(base + u);
                            rel = row_end - base;
                        }
                    }
                } else {
                    const uint32_t base = t0 + 4 * b + 1;
                    uint32_t rel = row_end - base;  // the row ends after slot 4b + rel
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        consume(4 * b + u, vv[u]);
                        if (rel == (uint32_t)u) {
                            advance_rows(base + u);
                            rel = row_end - base;
                        }
                    }
                }
                __syncwarp();  // every lane is done reading these slots
                if (b == 0) {
                    issue_meta(k + 2);
                    issue_par(k + 1);  // round k+1's columns landed with the wait above
                }
                issue(4 * b, k + 1);
                cp_commit();
            }
        }
        cp_wait<0>();
        for (; ri < nrows; ++ri) store_row();  // (only when the range has no slots)
        __syncwarp();  // the next slice reuses this warp's ring, metadata and row ends
        rb = re1;
    }
}

template <int T, int C, int WARPS, int DEC>
int launch_q8_wide_t(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                     uint64_t ldq, uint32_t f4, float4* c, uint64_t ldc4, const float* lut, cudaStream_t st,
                     const float2* fparams, uint32_t fcols) {
    const size_t smem = 256 * 256 + (size_t)WARPS * (32 * C + 144 + C * 128 * T + (DEC == 2 ? 32 * C : 0)) +
                        (DEC == 1 ? (size_t)128 * T * 8 : 0);  // (+ the staged per-feature params)
    static int occ_dev[kMaxDevices] = {};
    int& occ = occ_dev[cur_device()];
    if (occ == 0) {
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_q8_wide_kernel<T, C, WARPS, DEC>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AES_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_q8_wide_kernel<T, C, WARPS, DEC>,
                                                                   WARPS * 32, smem));
        if (occ < 1) occ = 1;
    }
    // one balanced wave (the 64 KB table filled once per CTA); small graphs
    // keep at least 8 rows per warp
    uint64_t grid = (uint64_t)num_sms() * occ;
    const uint64_t cap = (n + (uint64_t)WARPS * 8 - 1) / ((uint64_t)WARPS * 8);
    if (cap < grid) grid = cap ? cap : 1;
    spmm_q8_wide_kernel<T, C, WARPS, DEC><<<(unsigned)grid, WARPS * 32, smem, st>>>(
        srow, scol, sval, n, q, (uint32_t)ldq, f4, c, ldc4, lut, fparams, fcols);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

// F in (128, 1024] codes: T = ceil(F / 128) groups per lane
template <int C, int WARPS, int DEC = 0>
int launch_q8_wide(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                   uint64_t ldq, uint32_t f4, float4* c, uint64_t ldc4, const float* lut, cudaStream_t st,
                   const float2* fparams = nullptr, uint32_t fcols = 0) {
    switch ((f4 + 31) / 32) {
        case 1: return launch_q8_wide_t<1, C, WARPS, DEC>(srow, scol, sval, n, q, ldq, f4, c, ldc4, lut, st, fparams, fcols);
        case 2: return launch_q8_wide_t<2, C, WARPS, DEC>(srow, scol, sval, n, q, ldq, f4, c, ldc4, lut, st, fparams, fcols);
        case 3: return launch_q8_wide_t<3, C, WARPS, DEC>(srow, scol, sval, n, q, ldq, f4, c, ldc4, lut, st, fparams, fcols);
        case 4: return launch_q8_wide_t<4, C, WARPS, DEC>(srow, scol, sval, n, q, ldq, f4, c, ldc4, lut, st, fparams, fcols);
        case 5: return launch_q8_wide_t<5, C, WARPS, DEC>(srow, scol, sval, n, q, ldq, f4, c, ldc4, lut, st, fparams, fcols);
        default: return AES_ERR_UNSUPPORTED;
    }
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
int g_spmm_variant = 0;          // 0 = auto; see aes_dev_spmm_set_variant
int g_spmm_sched = 0;            // row schedule: 0 auto, kSched* otherwise
// auto: the balanced persistent schedule for every plan.  Measured on B200
// (scripts/shard_scaling.py): it matches the static one on the full products
// graph and removes the partial last wave on row shards; on unbounded rows
// (exact SpMM, FULL plans) it also replaces the heavy-first dynamic schedule
// (no pre-pass, no workspace allocation, no tickets).
int pick_schedule(uint64_t max_row_slots) {
    if (g_spmm_sched != 0) return g_spmm_sched;
    // bounded rows: per-kernel choice; unknown row lengths: one balanced wave
    // (a hub row lands in a range of its own weight, no heavy-first pre-pass)
    return max_row_slots != 0 && max_row_slots <= 256 ? kSchedAuto : kSchedBalOne;
}
// Measured on B200 (scripts/tune_spmm.py, products W=32): fp32 best with a
// 16-slot ring x 4 warps (1.18 ms); int8 with the batch kernel, 16-slot ring
// x 16 warps (0.58 ms; the generic int8 ring, variant 8, 0.89 ms).
constexpr int kDefaultVariantF32 = 2;
constexpr int kDefaultVariantQ8 = 8;

template <class G> struct RingOf;
template <> struct RingOf<GatherF32> { typedef RingF32 type; };
template <> struct RingOf<GatherQ8> { typedef RingQ8 type; };

template <class G, int NV, int C, int W, bool FULL>
int launch_ring_t(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, G g, uint32_t f4,
                  float4* c, uint64_t ldc4, const float* lut, cudaStream_t st, int dyn) {
    typedef typename RingOf<G>::type R;
    const size_t smem = (size_t)R::kLutBytes + (size_t)W * C * NV * 32 * R::kBytes;
    static int occ_dev[kMaxDevices] = {};  // per template instance and device: resident blocks per SM
    int& occ = occ_dev[cur_device()];
    if (occ == 0) {
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_ring_kernel<R, NV, C, W, FULL>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_ring_dyn_kernel<R, NV, C, W, FULL>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_ring_bal_kernel<R, NV, C, W, FULL>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AES_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_ring_bal_kernel<R, NV, C, W, FULL>,
                                                                   W * 32, smem));
        if (occ < 1) occ = 1;
    }
    if (dyn == kSchedAuto) dyn = kSchedBal;  // fp32 ring: balanced waves at every size (1.17 vs 1.18 ms full graph)
    if (dyn == kSchedBal || dyn == kSchedBalOne) {  // waves of resident CTAs, slot-balanced row ranges
        const uint64_t waves = dyn == kSchedBalOne ? 1 : bal_waves(n, (uint64_t)num_sms() * occ * W, 20);
        const uint64_t grid = waves * num_sms() * occ;
        // rows of unknown length, fp32 rows of <= 128 floats: hub rows go to
        // spmm_hub_kernel (column-split CTA per row), the balanced kernel skips them
        const int hubs = dyn == kSchedBalOne && R::kLutBytes == 0 && NV == 1;
        if (hubs) {
            static bool hub_attr_dev[kMaxDevices] = {};
            bool& hub_attr = hub_attr_dev[cur_device()];
            const size_t hub_smem = (size_t)kHubWarps * kHubRing * 128;
            if (!hub_attr) {
                AES_CUDA_TRY(cudaFuncSetAttribute(spmm_hub_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)hub_smem));
                hub_attr = true;
            }
            spmm_hub_kernel<<<(unsigned)((n + kHubRows - 1) / kHubRows), kHubWarps * 32, hub_smem, st>>>(
                srow, scol, sval, n, reinterpret_cast<const float*>(g.base()), (uint64_t)g.ld4 * 4, f4 * 4,
                reinterpret_cast<float*>(c), ldc4 * 4, grid * W);
            AES_CUDA_TRY(cudaGetLastError());
        }
        spmm_ring_bal_kernel<R, NV, C, W, FULL><<<(unsigned)grid, W * 32, smem, st>>>(
            srow, scol, sval, n, g.base(), (uint32_t)g.ld4, f4, c, ldc4, lut, hubs);
        AES_CUDA_TRY(cudaGetLastError());
        return AES_OK;
    }
    // rows per warp: 32 when the graph fills >= 8 warps per SM slot at that
    // size, otherwise shrink (power of 2, >= 2) so the grid still covers the GPU
    uint32_t gr = 32;
    while (gr > 2 && (n + gr - 1) / gr < (uint64_t)num_sms() * 64) gr >>= 1;
    const uint64_t groups = (n + gr - 1) / gr;
    const unsigned grid = (unsigned)((groups + W - 1) / W);
    if (dyn == kSchedDyn && groups < (1ull << 31)) {
        DynSched* ws = nullptr;
        AES_CUDA_TRY(cudaMallocAsync((void**)&ws, sizeof(DynSched) + groups * sizeof(unsigned int), st));
        AES_CUDA_TRY(cudaMemsetAsync(ws, 0, 16, st));
        heavy_scan_kernel<<<grid_for(groups, 256, num_sms() * 8), 256, 0, st>>>(srow, n, gr, groups, ws);
        const unsigned pgrid = (unsigned)((uint64_t)grid < (uint64_t)num_sms() * occ ? (uint64_t)grid : (uint64_t)num_sms() * occ);
        spmm_ring_dyn_kernel<R, NV, C, W, FULL><<<pgrid, W * 32, smem, st>>>(
            srow, scol, sval, n, g.base(), (uint32_t)g.ld4, f4, c, ldc4, lut, gr, groups, ws);
        AES_CUDA_TRY(cudaGetLastError());
        AES_CUDA_TRY(cudaFreeAsync(ws, st));
        return AES_OK;
    }
    spmm_ring_kernel<R, NV, C, W, FULL><<<grid, W * 32, smem, st>>>(srow, scol, sval, n, g.base(), (uint32_t)g.ld4,
                                                                    f4, c, ldc4, lut, gr);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

template <class G, int NV, int C, int W>
int launch_ring(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, G g, uint32_t f4,
                float4* c, uint64_t ldc4, const float* lut, cudaStream_t st, int dyn) {
    if (f4 == 32u * NV) return launch_ring_t<G, NV, C, W, true>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
    return launch_ring_t<G, NV, C, W, false>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
}

template <class G>
int launch_vector(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n,
                  G g, uint32_t f4, float4* c, uint64_t ldc4, const float* lut, cudaStream_t st, int dyn) {
    const size_t smem = lut ? 256 * 32 * sizeof(float) : 0;
    if (f4 <= 16) {
        uint32_t lpr = f4 <= 1 ? 1 : f4 <= 2 ? 2 : f4 <= 4 ? 4 : f4 <= 8 ? 8 : 16;
        unsigned grid = grid_for(n * lpr, kThreads);
        switch (lpr) {
            case 1: spmm_narrow_kernel<G, 1, 4><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, g, f4, c, ldc4, lut); break;
            case 2: spmm_narrow_kernel<G, 2, 4><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, g, f4, c, ldc4, lut); break;
            case 4: spmm_narrow_kernel<G, 4, 4><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, g, f4, c, ldc4, lut); break;
            case 8: spmm_narrow_kernel<G, 8, 4><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, g, f4, c, ldc4, lut); break;
            default: spmm_narrow_kernel<G, 16, 4><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, g, f4, c, ldc4, lut); break;
        }
        AES_CUDA_TRY(cudaGetLastError());
        return AES_OK;
    }
    if (f4 <= 32) {
        int v = g_spmm_variant;
        if (v == 0) v = G::kLutBytes ? kDefaultVariantQ8 : kDefaultVariantF32;
        switch (v) {
            case 2: return launch_ring<G, 1, 16, 4>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
            case 3: return launch_ring<G, 1, 16, 8>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
            case 4: return launch_ring<G, 1, 32, 4>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
            case 5: return launch_ring<G, 1, 32, 8>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
            case 6: return launch_ring<G, 1, 8, 8>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
            case 7: return launch_ring<G, 1, 32, 2>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
            case 8: return launch_ring<G, 1, 8, 16>(srow, scol, sval, n, g, f4, c, ldc4, lut, st, dyn);
            default: break;  // 1: register-staged wide kernel below
        }
    }
    if (g_spmm_variant != 1) {
        // wider rows: ring of C slots x NV float4 per lane, column tiles of 256 float4
        for (uint32_t c0 = 0; c0 < f4; c0 += 256) {
            const uint32_t tf4 = min(256u, f4 - c0);
            G gt = g;
            gt.offset(c0);
            float4* ct = c + c0;
            int rc;
            switch ((tf4 + 31) / 32) {
                case 1: rc = G::kLutBytes ? launch_ring<G, 1, 8, 16>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn)
                                      : launch_ring<G, 1, 16, 4>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn);
                    break;
                case 2: rc = launch_ring<G, 2, 8, 8>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn); break;
                case 3: rc = launch_ring<G, 3, 4, 8>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn); break;
                case 4: rc = launch_ring<G, 4, 4, 8>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn); break;
                case 5: rc = launch_ring<G, 5, 4, 4>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn); break;
                case 6: rc = launch_ring<G, 6, 4, 4>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn); break;
                case 7: rc = launch_ring<G, 7, 4, 4>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn); break;
                default: rc = launch_ring<G, 8, 4, 4>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut, st, dyn); break;
            }
            if (rc != AES_OK) return rc;
        }
        return AES_OK;
    }
    // variant 1: register-staged wide kernel, column tiles of up to 256 float4
    for (uint32_t c0 = 0; c0 < f4; c0 += 256) {
        uint32_t tf4 = min(256u, f4 - c0);
        G gt = g;
        gt.offset(c0);
        float4* ct = c + c0;
        unsigned grid = grid_for((n + 31) / 32 * 32, kThreads);
        uint32_t nv = (tf4 + 31) / 32;
        switch (nv) {
            case 1: spmm_wide_kernel<G, 1, 8><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
            case 2: spmm_wide_kernel<G, 2, 4><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
            case 3: spmm_wide_kernel<G, 3, 2><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
            case 4: spmm_wide_kernel<G, 4, 2><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
            case 5: spmm_wide_kernel<G, 5, 1><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
            case 6: spmm_wide_kernel<G, 6, 1><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
            case 7: spmm_wide_kernel<G, 7, 1><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
            default: spmm_wide_kernel<G, 8, 1><<<grid, kThreads, smem, st>>>(srow, scol, sval, n, gt, tf4, ct, ldc4, lut); break;
        }
        AES_CUDA_TRY(cudaGetLastError());
    }
    return AES_OK;
}

// ---------------------------------------------------------------------------
// Fused exact GCN layer: H = act(SpMM(A, X) W + b) in one persistent kernel
// (gnn.cpp:66-78 for one layer: spmm_sampled then dense_matmul, bias, ReLU).
//
// The SpMM is HBM-bound (gathers) and the ordered fp32 GEMM is FP32-pipe
// bound, so the split kernels leave each resource idle half of the time and
// round-trip the aggregate through HBM.  Here one CTA per SM runs both,
// warp-specialised:
//   * the CTA owns a slot-balanced contiguous row block; producer warp p
//     streams its own contiguous 1/8 of it as ONE slot stream through a
//     cp.async ring (the ring SpMM body: the ring never drains at a tile
//     boundary) and deposits every finished aggregate row into a shared-
//     memory A buffer: its rows 8i..8i+7 become rows 8p..8p+7 of GEMM tile i;
//   * 8 consumer warps run the ordered GEMM of tile i (64 rows from 8
//     producers) against W, resident in shared memory for the whole kernel,
//     and store bias + ReLU results from registers to each row's place;
//   * mbarriers pass kLayerBufs A buffers around (full: every producer
//     thread arrives, consumers wait; empty: the reverse); a producer waits
//     only for the consumers, so one slowed by a dense 8-row block has two
//     tiles of slack and never holds the other producers back.
// Bit-exact with the split path: every aggregate element is the same slot-
// order FMUL/FADD chain, every output the same k-ascending chain from +0.
// Consumer mapping: thread (tx, ty) owns tile rows 4ty..4ty+3 and columns
// {4tx..4tx+3, 64+4tx..}: the A reads broadcast, the W reads are 256
// contiguous bytes per half-warp (no bank conflicts).
// ---------------------------------------------------------------------------
constexpr int kLayerBM = 64;
constexpr int kLayerConsumers = 8, kLayerProducers = 8;
constexpr int kLayerThreads = (kLayerConsumers + kLayerProducers) * 32;  // 512
constexpr int kLayerRing = 12;  // producer ring slots (512 B each at K = 128)
constexpr int kLayerBufs = 3;   // A buffers (2 buffers + 20-slot rings: 4.49 ms vs 4.13 on products)
constexpr int kLayerPRows = kLayerBM / kLayerProducers;  // rows per producer per tile (8)

// mbarriers (shared memory): a producer waits only for the consumers, never
// for the other producers (a named barrier's bar.sync would count every
// producer thread and lock the eight streams into one pace)
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LAYER_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAYER_WAIT_%=;\n\t}" ::"r"(a), "r"(parity)
        : "memory");
}

// Row block of CTA c (slot + row balanced, bal_range) and producer p's rows in
// it: 8T consecutive rows each, T = tiles of the block.
__device__ __forceinline__ void layer_rows(const uint64_t* __restrict__ srow, uint64_t n_rows, uint64_t& c0,
                                           uint64_t& c1, uint64_t& tiles) {
    bal_range(srow, n_rows, blockIdx.x, gridDim.x, c0, c1);
    tiles = (c1 - c0 + kLayerBM - 1) / kLayerBM;
}

// One producer warp: rows [rb, re) as one ring stream; row q = r - rb goes to
// tile q / 8, A row 8p + q % 8 (smem address abase + buf * a_bytes + ...).
template <bool FULL>
__device__ __forceinline__ void layer_produce(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                                              const float* __restrict__ sval, const float4* __restrict__ gsrc,
                                              uint32_t ld, uint32_t f4, uint32_t ring0, uint64_t rb, uint64_t re,
                                              uint64_t tiles, int pw, uint32_t abase, uint32_t a_bytes,
                                              uint32_t as4, uint32_t mbar) {
    constexpr int C = kLayerRing;
    const uint32_t lane = threadIdx.x & 31;
    uint64_t tile = 0;  // tile of the next row to store
    uint32_t j = 0;     // its row within this producer's 8
    bool held = false;  // buffer of `tile` acquired
    // full[b] at mbar + 8b, empty[b] at mbar + 8(kLayerBufs + b); tile t is
    // use t / kLayerBufs of buffer t % kLayerBufs
    auto acquire = [&]() {
        if (tile >= (uint64_t)kLayerBufs)  // consumers released tile - kLayerBufs
            mbar_wait(mbar + 8 * (kLayerBufs + (uint32_t)(tile % kLayerBufs)),
                      (uint32_t)((tile / kLayerBufs - 1) & 1));
        held = true;
    };
    auto release = [&]() {
        mbar_arrive(mbar + 8 * (uint32_t)(tile % kLayerBufs));
        ++tile;
        j = 0;
        held = false;
    };
    if (rb < re) {
        const uint64_t g0 = srow[rb];
        const uint32_t total = (uint32_t)(srow[re] - g0);  // < 2^31: 1/1184 of any plan that fits in HBM
        auto window = [&](uint64_t w) -> uint32_t { return (uint32_t)(srow[min(w + 1 + lane, re)] - g0); };
        uint32_t rel = window(rb);
        uint32_t rel_nx = window(rb + 32);
        const uint32_t* gcol = scol + g0;
        const float* gval = sval + g0;
        const char* glb = reinterpret_cast<const char*>(gsrc + lane);
        const uint32_t ld_bytes = ld * 16u;
        const bool colok = FULL || lane < f4;
        auto ld_col = [&](uint32_t chunk) -> uint32_t {
            const uint32_t sidx = chunk * C + lane;
            return (lane < (uint32_t)C && sidx < total) ? ld_meta_u32(gcol + sidx) : 0u;
        };
        auto ld_val = [&](uint32_t chunk) -> float {
            const uint32_t sidx = chunk * C + lane;
            return (lane < (uint32_t)C && sidx < total) ? ld_meta_f32(gval + sidx) : 0.f;
        };
        auto issue = [&](int p, uint32_t col) {
            if (colok) cp_async_sa(ring0 + p * 512, glb + (uint64_t)col * ld_bytes, 16);
        };
        {
            const uint32_t mc0 = ld_col(0);
#pragma unroll
            for (int p = 0; p < C; ++p) {
                const uint32_t col = __shfl_sync(0xffffffffu, mc0, p);
                if ((uint32_t)p < total) issue(p, col);
                cp_commit();
            }
        }
        uint32_t mc_is = ld_col(1), mc_nx = ld_col(2);
        float mv_cur = ld_val(0), mv_nx = ld_val(1);
        float4 acc = f4_zero();
        uint64_t ra = rb;
        uint32_t wi = 0;
        uint32_t row_end = __shfl_sync(0xffffffffu, rel, 0);
        auto store_row = [&]() {
            if (!held) acquire();
            if (colok)
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 abase + (uint32_t)(tile % kLayerBufs) * a_bytes +
                                 (uint32_t)(pw * kLayerPRows + j) * as4 * 16),
                             "f"(acc.x), "f"(acc.y), "f"(acc.z), "f"(acc.w)
                             : "memory");
            acc = f4_zero();
            if (++j == kLayerPRows) release();
        };
        auto advance_rows = [&](uint32_t pos) {
            do {
                store_row();
                ++ra;
                if (++wi == 32) {
                    wi = 0;
                    rel = rel_nx;
                    rel_nx = window(ra + 32);
                }
                row_end = __shfl_sync(0xffffffffu, rel, wi);
            } while (ra < re && row_end == pos);
        };
        if (row_end == 0) advance_rows(0);
        auto body = [&](int p, uint32_t t) {
            cp_wait<C - 1>();
            const float v = __shfl_sync(0xffffffffu, mv_cur, p);
            if (colok) f4_axpy(acc, v, lds_f32x4(ring0 + p * 512));
            const uint32_t col = __shfl_sync(0xffffffffu, mc_is, p);
            if (t + C < total) issue(p, col);
            cp_commit();
            if (t + 1 == row_end) advance_rows(t + 1);
        };
        uint32_t k = 0;
        for (uint32_t t0 = 0; t0 < total; t0 += C, ++k) {
            if (t0 + C <= total) {
#pragma unroll
                for (int p = 0; p < C; ++p) body(p, t0 + p);
            } else {
#pragma unroll
                for (int p = 0; p < C; ++p) {
                    if (t0 + p >= total) break;
                    body(p, t0 + p);
                }
            }
            mv_cur = mv_nx;
            mc_is = mc_nx;
            mv_nx = ld_val(k + 2);
            mc_nx = ld_col(k + 3);
        }
        cp_wait<0>();
        while (ra < re) {  // trailing empty rows
            store_row();
            ++ra;
        }
    }
    if (j != 0 || held) release();  // a partly filled last tile
    while (tile < tiles) {  // tiles past this producer's rows: nothing to add (the
        acquire();          // wait keeps this arrival in the right phase)
        release();
    }
}

// BCAST: the layer's exchange fused in (gcn.ShardedGCN exchange="p2p"): every
// output row goes to each rank's replica (peer memory through CUDA IPC /
// NVLink) at row row_off + r, or only where need[d][row] is set (halo), and
// each CTA then publishes ONE system-scope arrival per destination after
// all its rows (aes_gcn_layer_fused_ctas(n_rows) arrivals per launch).
constexpr int kLayerMaxDst = 16;
struct LayerBcast {
    float* dst[kLayerMaxDst];
    unsigned long long* ctr[kLayerMaxDst];
    const uint8_t* need[kLayerMaxDst];
    int n;
    uint64_t row_off;
};

template <bool FULLK, bool SKIP, bool BCAST>
__global__ void __launch_bounds__(kLayerThreads, 1)
gcn_layer_fused_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                       const float* __restrict__ sval, uint64_t n_rows, const float4* __restrict__ x,
                       uint32_t ldx4, uint32_t k, const float* __restrict__ w, uint64_t ldw, uint32_t n,
                       const float* __restrict__ bias, int relu, float* __restrict__ h, uint64_t ldh,
                       LayerBcast bc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t mbar_s[2 * kLayerBufs];  // full[b], empty[b]
    const uint32_t k4 = k / 4, as4 = k4 + 1;  // A row stride in float4 (one float4 of pad)
    const uint32_t smem0 = smem_addr(smem_raw);
    const uint32_t mbar = smem_addr(mbar_s);
    float* ws = reinterpret_cast<float*>(smem_raw);  // W [k][128] (columns >= n zero)
    const uint32_t a_off = k * 128 * 4;
    const uint32_t a_bytes = kLayerBM * as4 * 16;
    const uint32_t ring_off = a_off + kLayerBufs * a_bytes;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // W resident for the whole kernel (read once per SM from L2)
    for (uint32_t i = tid; i < k * 128; i += kLayerThreads) {
        const uint32_t kk = i >> 7, jj = i & 127;
        ws[i] = jj < n ? w[(uint64_t)kk * ldw + jj] : 0.f;
    }
    if (tid < kLayerBufs) {
        mbar_init(mbar + 8 * tid, kLayerProducers * 32);                 // full: every producer thread
        mbar_init(mbar + 8 * (kLayerBufs + tid), kLayerConsumers * 32);  // empty: every consumer thread
    }
    uint64_t c0, c1, tiles;
    layer_rows(srow, n_rows, c0, c1, tiles);
    const uint64_t prow = kLayerPRows * tiles;  // rows per producer
    __syncthreads();

    if (warp >= kLayerConsumers) {
        const int pw = warp - kLayerConsumers;
        const uint64_t rb = min(c0 + (uint64_t)pw * prow, c1), re = min(rb + prow, c1);
        layer_produce<FULLK>(srow, scol, sval, x, ldx4, k4,
                             smem0 + ring_off + pw * (kLayerRing * 512) + lane * 16, rb, re, tiles, pw,
                             smem0 + a_off + lane * 16, a_bytes, as4, mbar);
        return;
    }

    // ---------------- consumers: ordered GEMM of each tile
    const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4 x 8 outputs each
    // tile row 4ty + r comes from producer (4ty + r) / 8, its row (4ty + r) % 8 of the tile
    const int pw_of = (4 * ty) / kLayerPRows, j0 = (4 * ty) % kLayerPRows;
    const uint64_t my_rb = min(c0 + (uint64_t)pw_of * prow, c1), my_re = min(my_rb + prow, c1);
    for (uint64_t i = 0; i < tiles; ++i) {
        const int buf = (int)(i % kLayerBufs);
        mbar_wait(mbar + 8 * buf, (uint32_t)((i / kLayerBufs) & 1));  // tile i's rows landed
        const float* as = reinterpret_cast<const float*>(smem_raw + a_off + buf * a_bytes);
        float acc[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) acc[r][jj] = 0.f;
        for (uint32_t k0 = 0; k0 < k; k0 += 4) {
            float4 a4[4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
                a4[r] = *reinterpret_cast<const float4*>(as + (uint32_t)(4 * ty + r) * as4 * 4 + k0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const float4 w0 = *reinterpret_cast<const float4*>(ws + (k0 + kk) * 128 + 4 * tx);
                const float4 w1 = *reinterpret_cast<const float4*>(ws + (k0 + kk) * 128 + 64 + 4 * tx);
                const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const float av = kk == 0 ? a4[r].x : kk == 1 ? a4[r].y : kk == 2 ? a4[r].z : a4[r].w;
                    // scalar FMULs, paired adds (FADD2): 3 issue slots per 2
                    // MACs (products layer 4.13 -> 3.39 ms)
                    if (SKIP) {
                        const bool skip = av == 0.f;
#pragma unroll
                        for (int jj = 0; jj < 8; jj += 2) {
                            float s0 = acc[r][jj], s1 = acc[r][jj + 1];
                            add2_rn(s0, s1, __fmul_rn(av, wv[jj]), __fmul_rn(av, wv[jj + 1]));
                            acc[r][jj] = skip ? acc[r][jj] : s0;
                            acc[r][jj + 1] = skip ? acc[r][jj + 1] : s1;
                        }
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 8; jj += 2)
                            add2_rn(acc[r][jj], acc[r][jj + 1], __fmul_rn(av, wv[jj]), __fmul_rn(av, wv[jj + 1]));
                    }
                }
            }
        }
        mbar_arrive(mbar + 8 * (kLayerBufs + buf));  // buffer buf may be refilled
        // epilogue: bias, ReLU (gnn.cpp:41-52), store to each row's place.
        // One destination (h, or a single replica without a halo mask) stores
        // directly; the pointer is formed here from the parameters, not kept
        // live across the GEMM loop (a kernel-lifetime copy cost the loop its
        // schedule: 3.38 -> 3.78 ms on the products layer)
        float* const h1 = !BCAST ? h : bc.n == 1 && !bc.need[0] ? bc.dst[0] + bc.row_off * ldh : nullptr;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const uint64_t gm = my_rb + kLayerPRows * i + j0 + r;
            if (gm >= my_re) continue;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t col0 = (half ? 64 : 0) + 4 * tx;
                if (col0 >= n) continue;
                float v[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    float xo = acc[r][4 * half + jj];
                    if (bias && col0 + jj < n) xo = __fadd_rn(xo, bias[col0 + jj]);
                    if (relu) xo = (xo < 0.f) ? 0.f : xo;
                    v[jj] = xo;
                }
                auto put = [&](float* dst) {
                    if (col0 + 4 <= n)
                        __stcs(reinterpret_cast<float4*>(dst), make_float4(v[0], v[1], v[2], v[3]));
                    else
                        for (int jj = 0; jj < 4; ++jj)
                            if (col0 + jj < n) dst[jj] = v[jj];
                };
                if (h1) {  // one destination (h, or the only replica)
                    put(h1 + gm * ldh + col0);
                    continue;
                }
                // several destinations: a rolled loop — unrolled over 16
                // destinations the kernel grew from 5.9 k to 9.4 k instructions
                // and the producer / consumer loops started missing in the
                // instruction cache (3.38 -> 3.72 ms on the products layer)
#pragma unroll 1
                for (int d = 0; d < bc.n; ++d) {
                    if (bc.need[d] && !bc.need[d][bc.row_off + gm]) continue;  // halo: d never reads it
                    put(bc.dst[d] + (bc.row_off + gm) * ldh + col0);
                }
            }
        }
    }
    if (BCAST) {
        // publish this CTA's rows to every destination: the consumer barrier
        // orders every consumer's stores before thread 0's system-scope
        // fence (cumulativity), then one release-add per destination counter
        asm volatile("bar.sync 1, %0;" ::"n"(kLayerConsumers * 32) : "memory");
        if (tid == 0) {
            __threadfence_system();
            for (int d = 0; d < bc.n; ++d)
                asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(bc.ctr[d]) : "memory");
        }
    }
}

template <bool FULLK, bool SKIP, bool BCAST = false>
int launch_layer_fused_t(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n_rows,
                         const float* x, uint64_t ldx, uint32_t k, const float* w, uint64_t ldw, uint32_t n,
                         const float* bias, int relu, float* h, uint64_t ldh, cudaStream_t st,
                         const LayerBcast& bc = LayerBcast{}) {
    const size_t smem = (size_t)k * 128 * 4 + kLayerBufs * (size_t)kLayerBM * (k / 4 + 1) * 16 +
                        (size_t)kLayerProducers * kLayerRing * 512;
    static bool attr_dev[kMaxDevices] = {};
    bool& attr = attr_dev[cur_device()];
    if (!attr) {  // opt in once for the largest k (128)
        const size_t smax = 128 * 128 * 4 + kLayerBufs * (size_t)kLayerBM * 33 * 16 +
                            (size_t)kLayerProducers * kLayerRing * 512;
        AES_CUDA_TRY(cudaFuncSetAttribute(gcn_layer_fused_kernel<FULLK, SKIP, BCAST>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax));
        attr = true;
    }
    // one CTA per SM, each a slot-balanced row block (small graphs: >= 64 rows per CTA)
    const uint64_t blocks = (n_rows + kLayerBM - 1) / kLayerBM;
    const unsigned grid = (unsigned)(blocks < (uint64_t)num_sms() ? blocks : (uint64_t)num_sms());
    gcn_layer_fused_kernel<FULLK, SKIP, BCAST><<<grid, kLayerThreads, smem, st>>>(
        srow, scol, sval, n_rows, reinterpret_cast<const float4*>(x), (uint32_t)(ldx / 4), k, w, ldw, n, bias,
        relu, h, ldh, bc);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace

int layer_fused_checks(uint64_t k, uint64_t n, const float* x, uint64_t ldx, uint64_t ldh, uint64_t ldw) {
    if (k == 0 || n == 0 || k > 128 || n > 128 || k % 4 != 0)
        return fail(AES_ERR_UNSUPPORTED, "fused layer needs 0 < k <= 128, k % 4 == 0, 0 < n <= 128");
    if (ldx % 4 != 0 || (uintptr_t)x % 16 != 0 || ldx < k || ldh < n || ldw < n)
        return fail(AES_ERR_UNSUPPORTED, "fused layer needs ldx % 4 == 0, 16-B aligned x, ldw >= n, ldh >= n");
    if (ldh % 4 != 0) return fail(AES_ERR_UNSUPPORTED, "fused layer needs ldh % 4 == 0");
    return AES_OK;
}

template <bool BCAST>
int layer_fused_dispatch(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval, uint64_t n_rows,
                                const float* x, uint64_t ldx, uint64_t k, const float* w, uint64_t ldw, uint64_t n,
                                const float* bias, int relu, int finite_w, float* h, uint64_t ldh, cudaStream_t st,
                                const LayerBcast& bc) {
    const uint32_t k32 = (uint32_t)k, n32 = (uint32_t)n;
    if (k == 128) {
        if (finite_w)
            return launch_layer_fused_t<true, false, BCAST>(srow_ptr, scol, sval, n_rows, x, ldx, k32, w, ldw, n32,
                                                            bias, relu, h, ldh, st, bc);
        return launch_layer_fused_t<true, true, BCAST>(srow_ptr, scol, sval, n_rows, x, ldx, k32, w, ldw, n32, bias,
                                                       relu, h, ldh, st, bc);
    }
    if (finite_w)
        return launch_layer_fused_t<false, false, BCAST>(srow_ptr, scol, sval, n_rows, x, ldx, k32, w, ldw, n32,
                                                         bias, relu, h, ldh, st, bc);
    return launch_layer_fused_t<false, true, BCAST>(srow_ptr, scol, sval, n_rows, x, ldx, k32, w, ldw, n32, bias,
                                                    relu, h, ldh, st, bc);
}

// int8 FAST MODE, per-feature affine codes (affine.cu dispatches here for
// 16-B aligned code rows): the batch kernel with the affine decode (DEC 1),
// one 32-warp CTA per SM on a balanced wave, no table.
int launch_q8_feature_batch(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n,
                            const uint8_t* q, uint64_t ldq, uint64_t f, const float2* params, float* c, uint64_t ldc,
                            cudaStream_t st) {
    const uint64_t f4 = (f + 3) / 4;
    if (f4 <= 16 || ldq % 16 != 0 || (uintptr_t)q % 16 != 0 || ldc % 4 != 0 || (uintptr_t)c % 16 != 0 ||
        f4 / 32 >= 65535 || f > 0xffffffffull)
        return AES_ERR_UNSUPPORTED;
    // 128 < F <= 640: one warp per whole code row, 12-slot rings (variant 56:
    // 8-slot; 55: the batch kernel's column tiles).  reddit W=32 0.440 ->
    // 0.394 ms, W=64 0.662 -> 0.532 (with the row-end batches rolled: inlined
    // at every row-end position, the per-feature epilogue had pushed the
    // kernel out of the instruction cache, 0.557 / 0.993 ms)
    if (f4 <= 160 && ((f4 > 32 && g_spmm_variant == 0) || g_spmm_variant == 56 || g_spmm_variant == 57))
        return g_spmm_variant == 56
                   ? launch_q8_wide<8, 16, 1>(srow, scol, sval, n, q, ldq, (uint32_t)f4, reinterpret_cast<float4*>(c),
                                                ldc / 4, nullptr, st, params, (uint32_t)f)
                   : launch_q8_wide<12, 16, 1>(srow, scol, sval, n, q, ldq, (uint32_t)f4, reinterpret_cast<float4*>(c),
                                                 ldc / 4, nullptr, st, params, (uint32_t)f);
    return launch_q8_batch<12, 32, true, 1>(srow, scol, sval, n, q, ldq, (uint32_t)f4, reinterpret_cast<float4*>(c),
                                            ldc / 4, nullptr, st, kSchedBal, params, (uint32_t)f);
}

// int8 FAST MODE, per-row affine codes: the batch kernel with the gathered
// rows' (s, m) staged next to the slot metadata (DEC 2).
int launch_q8_row_batch(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                        uint64_t ldq, uint64_t f, const float2* params, float* c, uint64_t ldc, cudaStream_t st) {
    const uint64_t f4 = (f + 3) / 4;
    if (f4 <= 16 || ldq % 16 != 0 || (uintptr_t)q % 16 != 0 || ldc % 4 != 0 || (uintptr_t)c % 16 != 0 ||
        f4 / 32 >= 65535 || f > 0xffffffffull)
        return AES_ERR_UNSUPPORTED;
    // 128 < F <= 640: one warp per whole code row, 12-slot rings (variant 56:
    // 8-slot; 55: the batch kernel's column tiles).  reddit W=32 0.506 ->
    // 0.327 ms, W=64 0.775 -> 0.483
    if (f4 <= 160 && ((f4 > 32 && g_spmm_variant == 0) || g_spmm_variant == 56 || g_spmm_variant == 57))
        return g_spmm_variant == 56
                   ? launch_q8_wide<8, 16, 2>(srow, scol, sval, n, q, ldq, (uint32_t)f4, reinterpret_cast<float4*>(c),
                                                ldc / 4, nullptr, st, params, (uint32_t)f)
                   : launch_q8_wide<12, 16, 2>(srow, scol, sval, n, q, ldq, (uint32_t)f4, reinterpret_cast<float4*>(c),
                                                 ldc / 4, nullptr, st, params, (uint32_t)f);
    return launch_q8_batch<12, 32, true, 2>(srow, scol, sval, n, q, ldq, (uint32_t)f4, reinterpret_cast<float4*>(c),
                                            ldc / 4, nullptr, st, kSchedBal, params, (uint32_t)f);
}

int launch_spmm_q8_tma(int dec, const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n,
                       const uint8_t* q, uint64_t ldq, uint64_t f, const float* lut, const float* fparams, float* c,
                       uint64_t ldc, cudaStream_t st);  // spmm_tma.cu
int spmm_variant() { return g_spmm_variant; }  // read by affine.cu (tuning variants 50, 51)
}  // namespace aes

extern "C" {

int aes_dev_spmm_set_variant(int variant) {
    aes::g_spmm_variant = variant;
    return AES_OK;
}

int aes_dev_spmm_set_schedule(int schedule) {
    if (schedule < 0 || schedule > 6) return aes::fail(AES_ERR_INVALID_ARG, "schedule must be 0..6");
    aes::g_spmm_sched = schedule;
    return AES_OK;
}

int aes_dev_spmm_f32(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                     uint64_t n_rows, const float* b, uint64_t ldb, uint64_t f, float* c,
                     uint64_t ldc, void* stream) {
    return aes_dev_spmm_f32_ex(srow_ptr, scol, sval, n_rows, b, ldb, f, c, ldc, 0, stream);
}

int aes_dev_spmm_f32_ex(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                        uint64_t n_rows, const float* b, uint64_t ldb, uint64_t f, float* c,
                        uint64_t ldc, uint64_t max_row_slots, void* stream) {
    using namespace aes;
    const int dyn = pick_schedule(max_row_slots);
    cudaStream_t st = as_stream(stream);
    if (n_rows == 0 || f == 0) return AES_OK;
    if (ldb < f || ldc < f) return fail(AES_ERR_INVALID_ARG, "leading dimension smaller than f");
    const uint64_t f4 = (f + 3) / 4;
    const bool vec = (ldb % 4 == 0) && (ldc % 4 == 0) && ((uintptr_t)b % 16 == 0) &&
                     ((uintptr_t)c % 16 == 0) && ldb >= f4 * 4 && ldc >= f4 * 4;
    if (vec) {
        GatherF32 g{reinterpret_cast<const float4*>(b), ldb / 4};
        return launch_vector(srow_ptr, scol, sval, n_rows, g, (uint32_t)f4,
                             reinterpret_cast<float4*>(c), ldc / 4, nullptr, st, dyn);
    }
    spmm_scalar_kernel<4><<<grid_for(n_rows * 32, kThreads, num_sms() * 64), kThreads, 0, st>>>(
        srow_ptr, scol, sval, n_rows, b, ldb, f, c, ldc);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_spmm_q8(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                    uint64_t n_rows, const uint8_t* q, uint64_t ldq, uint64_t f, const float* lut,
                    float* c, uint64_t ldc, void* stream) {
    return aes_dev_spmm_q8_ex(srow_ptr, scol, sval, n_rows, q, ldq, f, lut, c, ldc, 0, stream);
}

int aes_dev_spmm_q8_ex(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                       uint64_t n_rows, const uint8_t* q, uint64_t ldq, uint64_t f, const float* lut,
                       float* c, uint64_t ldc, uint64_t max_row_slots, void* stream) {
    using namespace aes;
    const int dyn = pick_schedule(max_row_slots);
    cudaStream_t st = as_stream(stream);
    if (n_rows == 0 || f == 0) return AES_OK;
    const uint64_t f4 = (f + 3) / 4;
    if (ldq % 4 != 0 || (uintptr_t)q % 4 != 0 || ldq < f4 * 4 || ldc % 4 != 0 ||
        (uintptr_t)c % 16 != 0 || ldc < f4 * 4 || lut == nullptr)
        return fail(AES_ERR_UNSUPPORTED,
                    "spmm_q8 needs ldq % 4 == 0, ldc % 4 == 0 and ld >= round_up(f, 4)");
    // dual-stream kernel (variants 20-24): F % 8 == 0, F <= 128, 8-B aligned
    // code rows.  Measured slower than the single-stream ring on B200
    // (1.02 vs 0.89 ms, products): the half-warp row-end divergence costs what
    // the shared bookkeeping saves, so it is opt-in only.
    const int v = g_spmm_variant;
    if (v >= 20 && v < 30 && f % 8 == 0 && f <= 128 && ldq % 8 == 0 && (uintptr_t)q % 8 == 0) {
        float4* c4 = reinterpret_cast<float4*>(c);
        const uint32_t f8 = (uint32_t)(f / 8);
        switch (v) {
            case 21: return launch_q8_dual<8, 8>(srow_ptr, scol, sval, n_rows, q, ldq, f8, c4, ldc / 4, lut, st);
            case 22: return launch_q8_dual<16, 8>(srow_ptr, scol, sval, n_rows, q, ldq, f8, c4, ldc / 4, lut, st);
            case 23: return launch_q8_dual<16, 4>(srow_ptr, scol, sval, n_rows, q, ldq, f8, c4, ldc / 4, lut, st);
            case 24: return launch_q8_dual<8, 16>(srow_ptr, scol, sval, n_rows, q, ldq, f8, c4, ldc / 4, lut, st);
            default: return launch_q8_dual<8, 8>(srow_ptr, scol, sval, n_rows, q, ldq, f8, c4, ldc / 4, lut, st);
        }
    }
    // batch kernel (variants 30-37; the default for F > 64 with 16-B aligned
    // code rows).  Wider rows run as 128-code column tiles (grid.y): every
    // tile re-reads only the 8-B slot metadata next to its 128-B gathers.
    // TMA-gather kernel (spmm_tma.cu), variant 40 only: it moves the code
    // rows off the LSU (l1tex 88 -> 72 %) but issues more instructions than it
    // saves (562 M vs 460 M per products launch, the elected-lane TMA issue
    // converts its operands to uniform registers), 0.655 vs 0.566 ms
    if (v == 40 && f4 > 16) {
        const int s = launch_spmm_q8_tma(0, srow_ptr, scol, sval, n_rows, q, ldq, f, lut, nullptr, c, ldc, st);
        if (s != AES_ERR_UNSUPPORTED) return s;
    }
    if ((v == 0 || (v >= 30 && v <= 49)) && f4 > 16 && ldq % 16 == 0 && (uintptr_t)q % 16 == 0 &&
        dyn_smem_offset_ok(st) &&
        f4 / 32 < 65535) {
        float4* c4 = reinterpret_cast<float4*>(c);
        const uint32_t f4u = (uint32_t)f4;
        // 128 < F <= 640: one warp per whole code row (spmm_q8_wide_kernel)
        // (variants 46/48/49 also take one-tile rows, 64 < F <= 128: tuning)
        if (((v == 0 && f4u > 32) || (v >= 46 && v <= 49)) && f4u <= 160) {
            int rc;
            switch (v) {
                // measured on reddit W=32: 8-slot rings x 16 warps 0.431 ms;
                // 12 x 16 0.464, 12 x 20 0.463, 16 x 12 0.567
                case 46: rc = launch_q8_wide<8, 24>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st); break;
                case 48: rc = launch_q8_wide<8, 20>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st); break;
                case 49: rc = launch_q8_wide<12, 16>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st); break;
                default: rc = launch_q8_wide<8, 16>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st); break;
            }
            if (rc != AES_ERR_UNSUPPORTED) return rc;
        }
        switch (v) {
            case 30: return launch_q8_batch<16, 16>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 31: return launch_q8_batch<8, 16>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 32: return launch_q8_batch<16, 8>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 33: return launch_q8_batch<8, 8>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 34: return launch_q8_batch<12, 16>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 35: return launch_q8_batch<16, 4>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 36: return launch_q8_batch<16, 16, false>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 37: return launch_q8_batch<12, 16, false>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 38: return launch_q8_batch<16, 32>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 39: return launch_q8_batch<12, 32>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 43: return launch_q8_batch<16, 20>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 44: return launch_q8_batch<12, 20>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            case 45: return launch_q8_batch<8, 32>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
            default:
                // whole 128-code tiles (F = 128: products, arxiv, pubmed): one
                // 32-warp CTA per SM with 64 registers and a 12-slot ring,
                // balanced wave (products 0.511 ms vs 0.585 for the 16 x 16
                // static grid); partial tiles (reddit F = 602) keep 16 x 16
                // (0.585 vs 0.600)
                if (f4u % 32 == 0)
                    return launch_q8_batch<12, 32>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
                return launch_q8_batch<16, 16>(srow_ptr, scol, sval, n_rows, q, ldq, f4u, c4, ldc / 4, lut, st, dyn);
        }
    }
    GatherQ8 g{reinterpret_cast<const uint32_t*>(q), ldq / 4};
    return launch_vector(srow_ptr, scol, sval, n_rows, g, (uint32_t)f4,
                         reinterpret_cast<float4*>(c), ldc / 4, lut, st, dyn);
}


int aes_dev_gcn_layer_fused(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval, uint64_t n_rows,
                            const float* x, uint64_t ldx, uint64_t k, const float* w, uint64_t ldw, uint64_t n,
                            const float* bias, int relu, int finite_w, float* h, uint64_t ldh, void* stream) {
    using namespace aes;
    AES_TRY(aes::layer_fused_checks(k, n, x, ldx, ldh, ldw));
    if ((uintptr_t)h % 16 != 0) return fail(AES_ERR_UNSUPPORTED, "fused layer needs a 16-B aligned h");
    // the producers gather rows of x from anywhere while the consumers write
    // h: an h overlapping x would be read after being overwritten (x extent
    // taken as n_rows rows: conservative for separate buffers)
    {
        const char *x0 = reinterpret_cast<const char*>(x), *h0 = reinterpret_cast<const char*>(h);
        const char* x1 = x0 + ldx * 4 * (n_rows ? n_rows : 1);
        const char* h1 = h0 + ldh * 4 * (n_rows ? n_rows : 1);
        if (x0 < h1 && h0 < x1) return fail(AES_ERR_UNSUPPORTED, "fused layer output must not overlap its input");
    }
    if (n_rows == 0) return AES_OK;
    return aes::layer_fused_dispatch<false>(srow_ptr, scol, sval, n_rows, x, ldx, k, w, ldw, n, bias, relu, finite_w, h,
                                       ldh, as_stream(stream), LayerBcast{});
}

uint64_t aes_gcn_layer_fused_ctas(uint64_t n_rows) {
    if (n_rows == 0) return 0;
    const uint64_t blocks = (n_rows + aes::kLayerBM - 1) / aes::kLayerBM;
    return blocks < (uint64_t)aes::num_sms() ? blocks : (uint64_t)aes::num_sms();
}

int aes_dev_gcn_layer_fused_bcast(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval,
                                  uint64_t n_rows, const float* x, uint64_t ldx, uint64_t k, const float* w,
                                  uint64_t ldw, uint64_t n, const float* bias, int relu, int finite_w,
                                  float* const* dsts, unsigned long long* const* counters,
                                  const uint8_t* const* need, int n_dst, uint64_t row_offset, uint64_t ldh,
                                  void* stream) {
    using namespace aes;
    AES_TRY(aes::layer_fused_checks(k, n, x, ldx, ldh, ldw));
    if (n_dst < 1 || n_dst > kLayerMaxDst || !dsts || !counters)
        return fail(AES_ERR_INVALID_ARG, "n_dst must be 1..16 with destination and counter arrays");
    LayerBcast bc{};
    bc.n = n_dst;
    bc.row_off = row_offset;
    for (int d = 0; d < n_dst; ++d) {
        if ((uintptr_t)dsts[d] % 16 != 0) return fail(AES_ERR_UNSUPPORTED, "fused layer needs 16-B aligned replicas");
        bc.dst[d] = dsts[d];
        bc.ctr[d] = counters[d];
        bc.need[d] = need ? need[d] : nullptr;
    }
    if (n_rows == 0) return AES_OK;
    return aes::layer_fused_dispatch<true>(srow_ptr, scol, sval, n_rows, x, ldx, k, w, ldw, n, bias, relu, finite_w,
                                      nullptr, ldh, as_stream(stream), bc);
}

}  // extern "C"
