// int8 FAST MODE (opt-in, not bit-exact): per-row or per-feature-scale affine
// quantization with the dequantization fused into the SpMM gather —
// north_star item (3).  It sits beside the reference's global min/max path
// (proj/src/quantize.cpp:11-64, reproduced bit-exactly in quant.cu/spmm.cu):
// the reference has no per-row / per-feature mode, so this one is measured
// against stated error bounds instead of bit patterns.
//
// Quantization (codes u8, 8 bits, levels 255):
//   ROW mode      params[r] = (s_r, m_r), m_r = min_j x[r,j], s_r = (max_j - m_r)/255
//   FEATURE mode  params[j] = (s_j, m_j) over the rows of column j
//   q = clamp(rint((x - m) * (255 / (max - m))), 0, 255);  x^ = q * s + m
//   A constant row / column gets s = 0 and decodes to m exactly.
//
// SpMM over the codes (no table, no shared-memory LUT):
//   ROW      C[i,:] = sum_k (v_k s_{c_k}) q_{c_k,:} + sum_k v_k m_{c_k}
//   FEATURE  C[i,j] = s_j * sum_k v_k q_{c_k,j} + m_j * sum_k v_k
// Per code: one PRMT places the byte in the mantissa of 2^23 (the float
// 2^23 + q), one packed FADD2 per two codes removes 2^23 exactly, one packed
// FFMA2 per two codes accumulates — 2 instructions per code against 3.5 for
// the exact LUT decode.
//
// Error bounds (tests/test_gpu_affine.py):
//   quantize   |x^ - x| <= s/2 + 2^-22 (|m| + 255 s)     per element
//   SpMM       |C - A B| <= sum_k |v_k| (s_k/2 + 2^-22 (|m_k| + 255 s_k))
//                           + (slots + 2) 2^-23 sum_k |v_k| (|m_k| + 255 s_k)
// (s_k, m_k: the params that apply to gathered element k).
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace aes {
namespace {

constexpr float kTwo23 = 8388608.0f;
constexpr uint32_t kTwo23Bits = 0x4B000000u;

__device__ __forceinline__ void fma2(float& a0, float& a1, float x, float y0, float y1) {
    // (a0, a1) = (fma(x, y0, a0), fma(x, y1, a1)) — one FFMA2
    unsigned long long a, y, xx;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(y0), "f"(y1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(x));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(xx), "l"(y));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
}

// the 4 codes of one u32 as exact floats
__device__ __forceinline__ void decode4(uint32_t w, float& q0, float& q1, float& q2, float& q3) {
    const float t0 = __uint_as_float(__byte_perm(w, kTwo23Bits, 0x7650));
    const float t1 = __uint_as_float(__byte_perm(w, kTwo23Bits, 0x7651));
    const float t2 = __uint_as_float(__byte_perm(w, kTwo23Bits, 0x7652));
    const float t3 = __uint_as_float(__byte_perm(w, kTwo23Bits, 0x7653));
    q0 = t0;
    q1 = t1;
    q2 = t2;
    q3 = t3;
    add2_rn(q0, q1, -kTwo23, -kTwo23);
    add2_rn(q2, q3, -kTwo23, -kTwo23);
}

__device__ __forceinline__ uint32_t quant1(float x, float m, float inv) {
    const float t = rintf((x - m) * inv);
    return (uint32_t)fminf(fmaxf(t, 0.f), 255.f);
}

// ---------------------------------------------------------------- quantize
// ROW mode: one warp per row; lane l handles codes 4l + 128i.
__global__ void __launch_bounds__(256)
quant_row_kernel(const float* __restrict__ x, uint64_t rows, uint64_t cols, uint64_t ldx,
                 uint8_t* __restrict__ q, uint64_t ldq, float2* __restrict__ params, unsigned int* __restrict__ bad) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
        const float* xr = x + r * ldx;
        float lo = INFINITY, hi = -INFINITY;
        bool finite = true;
        for (uint64_t j = lane; j < cols; j += 32) {
            const float v = __ldcs(xr + j);
            finite &= isfinite(v);
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (__any_sync(0xffffffffu, !finite)) {
            if (lane == 0) atomicExch(bad, 1u);
            continue;
        }
        const float range = hi - lo;
        const float s = range > 0.f ? range / 255.f : 0.f;
        const float inv = range > 0.f ? 255.f / range : 0.f;
        if (lane == 0) params[r] = make_float2(s, lo);
        uint8_t* qr = q + r * ldq;
        for (uint64_t j = 4 * lane; j < cols; j += 128) {
            if (j + 4 <= cols) {
                const float4 v = make_float4(xr[j], xr[j + 1], xr[j + 2], xr[j + 3]);
                const uint32_t w = quant1(v.x, lo, inv) | quant1(v.y, lo, inv) << 8 | quant1(v.z, lo, inv) << 16 |
                                   quant1(v.w, lo, inv) << 24;
                *reinterpret_cast<uint32_t*>(qr + j) = w;  // ldq % 4 == 0
            } else {
                for (uint64_t e = j; e < cols; ++e) qr[e] = (uint8_t)quant1(xr[e], lo, inv);
            }
        }
    }
}

// FEATURE mode, pass 1: per-column partial (min, max) of a block of rows.
// CTA = 256 threads = 8 row lanes x 32 column lanes; grid.x over row blocks,
// grid.y over 32-column tiles.
constexpr int kColRowsPerCta = 1024;
__global__ void __launch_bounds__(256)
col_minmax_kernel(const float* __restrict__ x, uint64_t rows, uint64_t cols, uint64_t ldx,
                  float2* __restrict__ partial, unsigned int* __restrict__ bad) {
    __shared__ float s_lo[8][32], s_hi[8][32];
    const uint32_t cl = threadIdx.x & 31, rl = threadIdx.x >> 5;
    const uint64_t j = (uint64_t)blockIdx.y * 32 + cl;
    const uint64_t r0 = (uint64_t)blockIdx.x * kColRowsPerCta;
    const uint64_t r1 = min(rows, r0 + kColRowsPerCta);
    float lo = INFINITY, hi = -INFINITY;
    bool finite = true;
    if (j < cols)
        for (uint64_t r = r0 + rl; r < r1; r += 8) {
            const float v = __ldcs(x + r * ldx + j);
            finite &= isfinite(v);
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
        }
    if (!finite) atomicExch(bad, 1u);
    s_lo[rl][cl] = lo;
    s_hi[rl][cl] = hi;
    __syncthreads();
    if (rl == 0 && j < cols) {
#pragma unroll
        for (int k = 1; k < 8; ++k) {
            lo = fminf(lo, s_lo[k][cl]);
            hi = fmaxf(hi, s_hi[k][cl]);
        }
        partial[(uint64_t)blockIdx.x * cols + j] = make_float2(lo, hi);
    }
}

// FEATURE mode, pass 2: fold the partials into (s_j, m_j)
__global__ void col_params_kernel(const float2* __restrict__ partial, uint64_t blocks, uint64_t cols,
                                  float2* __restrict__ params) {
    const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (j >= cols) return;
    float lo = INFINITY, hi = -INFINITY;
    for (uint64_t b = 0; b < blocks; ++b) {
        const float2 p = partial[b * cols + j];
        lo = fminf(lo, p.x);
        hi = fmaxf(hi, p.y);
    }
    const float range = hi - lo;
    params[j] = make_float2(range > 0.f ? range / 255.f : 0.f, lo);
}

// FEATURE mode, pass 3: element-wise codes (4 per thread)
__global__ void __launch_bounds__(256)
quant_col_kernel(const float* __restrict__ x, uint64_t rows, uint64_t cols, uint64_t ldx,
                 const float2* __restrict__ params, uint8_t* __restrict__ q, uint64_t ldq) {
    const uint64_t c4 = (cols + 3) / 4;
    const uint64_t total = rows * c4;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / c4, j0 = (e - r * c4) * 4;
        uint32_t w = 0;
        for (int u = 0; u < 4 && j0 + u < cols; ++u) {
            const float2 p = params[j0 + u];  // (s, m); 1/s == 255/range up to rounding
            w |= quant1(x[r * ldx + j0 + u], p.y, p.x > 0.f ? 1.f / p.x : 0.f) << (8 * u);
        }
        *reinterpret_cast<uint32_t*>(q + r * ldq + j0) = w;
    }
}

// x^ = q * s + m (the values the fast SpMM aggregates)
template <int MODE>
__global__ void dequant_affine_kernel(const uint8_t* __restrict__ q, uint64_t rows, uint64_t cols, uint64_t ldq,
                                      const float2* __restrict__ params, float* __restrict__ x, uint64_t ldx) {
    const uint64_t total = rows * cols;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e / cols, j = e - r * cols;
        const float2 p = params[MODE == 0 ? r : j];
        x[r * ldx + j] = fmaf((float)q[r * ldq + j], p.x, p.y);
    }
}

// ---------------------------------------------------------------- SpMM
// Warp per 32-row group, one flattened slot stream.  Lane l owns codes
// 4l..4l+3 of the 128-code column tile blockIdx.y.  Slot metadata goes
// through shared memory in batches of 32 slots as {col, a = v*s_col,
// b = v*m_col} (ROW) or {col, v, v} (FEATURE): lane l loads slot t0+l's
// (col, v) two batches ahead and its row params one batch ahead, so neither
// dependent load is on the critical path.  The last batch is padded with
// {col 0, a 0, b 0} slots (adds of +0, past every row end), so the inner
// loop has no bounds tests; U code gathers are in flight before the first
// is consumed.
struct SlotMeta {
    float a;  // ROW: v * s_col   FEATURE: v
    float b;  // ROW: v * m_col   FEATURE: v
    uint32_t col;
    uint32_t pad;
};

template <int MODE, int U, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 4)
spmm_q8a_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                const float* __restrict__ sval, uint64_t n_rows, const uint8_t* __restrict__ q, uint32_t ldq,
                uint32_t f, const float2* __restrict__ params, float* __restrict__ c, uint64_t ldc) {
    __shared__ __align__(16) SlotMeta s_meta[WARPS][64];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t r0 = ((uint64_t)blockIdx.x * WARPS + warp) * 32;
    if (r0 >= n_rows) return;
    const uint32_t nr = (uint32_t)min((uint64_t)32, n_rows - r0);
    const uint32_t col0 = blockIdx.y * 128 + 4 * lane;  // first code of this lane
    const uint32_t ne = col0 < f ? min(4u, f - col0) : 0u;  // codes this lane owns
    // lanes past the row read (and ignore) the row's last 4 bytes: in bounds
    const uint8_t* qb = q + min(col0, ldq - 4);
    float sj[4] = {0.f, 0.f, 0.f, 0.f}, mj[4] = {0.f, 0.f, 0.f, 0.f};
    if (MODE == 1)
        for (uint32_t u = 0; u < ne; ++u) {
            const float2 p = params[col0 + u];
            sj[u] = p.x;
            mj[u] = p.y;
        }
    const uint64_t g0 = srow[r0];
    const uint32_t my_end = (uint32_t)(srow[r0 + 1 + min(lane, nr - 1)] - g0);
    const uint32_t total = __shfl_sync(0xffffffffu, my_end, nr - 1);
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f, bsum = 0.f;
    uint32_t row = 0;
    uint32_t row_end = __shfl_sync(0xffffffffu, my_end, 0);
    float* cptr = c + r0 * ldc + col0;

    auto store_row = [&]() {
        float o0, o1, o2, o3;
        if (MODE == 0) {
            o0 = acc0 + bsum; o1 = acc1 + bsum; o2 = acc2 + bsum; o3 = acc3 + bsum;
        } else {
            o0 = fmaf(sj[0], acc0, mj[0] * bsum); o1 = fmaf(sj[1], acc1, mj[1] * bsum);
            o2 = fmaf(sj[2], acc2, mj[2] * bsum); o3 = fmaf(sj[3], acc3, mj[3] * bsum);
        }
        if (ne == 4) {
            __stcs(reinterpret_cast<float4*>(cptr), make_float4(o0, o1, o2, o3));  // ldc % 4 == 0
        } else {
            if (ne > 0) cptr[0] = o0;
            if (ne > 1) cptr[1] = o1;
            if (ne > 2) cptr[2] = o2;
        }
        cptr += ldc;
        acc0 = acc1 = acc2 = acc3 = bsum = 0.f;
    };
    auto advance = [&](uint32_t pos) {
        do {
            store_row();
            ++row;
            row_end = __shfl_sync(0xffffffffu, my_end, min(row, nr - 1));
        } while (row < nr && row_end == pos);
    };
    if (row_end == 0) {
        if (total == 0) {
            for (; row < nr; ++row) store_row();
            return;
        }
        advance(0);
    }

    // Metadata: a 64-entry ring per warp (two 32-slot batches).  Batch j
    // lives in half j & 1; it is staged at the start of batch j - 1, from
    // (col, v) loaded two batches ahead and row params one batch ahead.
    // Code gathers: sub-batches of U slots, sub-batch s+1's loads issued
    // before sub-batch s is consumed (U..2U gathers in flight per warp at
    // every point of the stream, across batch and row boundaries).
    auto load_cv = [&](uint32_t t0, uint32_t& cc, float& v) {
        cc = 0;
        v = 0.f;
        if (t0 + lane < total) {
            cc = __ldcs(scol + g0 + t0 + lane);
            v = __ldcs(sval + g0 + t0 + lane);
        }
    };
    auto stage = [&](uint32_t j, uint32_t cc, float v, float2 p) {
        SlotMeta m;
        m.col = cc;
        m.a = MODE == 0 ? v * p.x : v;
        m.b = MODE == 0 ? v * p.y : v;
        m.pad = 0u;
        s_meta[warp][(j & 1) * 32 + lane] = m;
    };
    uint32_t c1, c2;  // (col, v) of batches j+1 and j+2
    float v1, v2;
    float2 p1 = make_float2(0.f, 0.f);
    {
        uint32_t c0;
        float v0;
        load_cv(0, c0, v0);
        load_cv(32, c1, v1);
        load_cv(64, c2, v2);
        float2 p0 = make_float2(0.f, 0.f);
        if (MODE == 0) {
            p0 = __ldg(params + c0);
            p1 = __ldg(params + c1);
        }
        stage(0, c0, v0, p0);
    }
    __syncwarp();
    const uint32_t n_sub = (total + U - 1) / U;
    uint32_t raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
        raw[u] = __ldg(reinterpret_cast<const uint32_t*>(qb + (uint64_t)s_meta[warp][u].col * ldq));
    for (uint32_t sb = 0; sb < n_sub; ++sb) {
        const uint32_t p0 = sb * U;  // first slot of this sub-batch
        if ((p0 & 31) == 0) {
            // entering batch j = p0 / 32: stage batch j+1 (its half held
            // batch j-1, consumed — the syncwarp below orders it), rotate
            // the prefetches
            const uint32_t j = p0 >> 5;
            __syncwarp();  // every lane is done reading batch j-1's half
            stage(j + 1, c1, v1, p1);
            c1 = c2;
            v1 = v2;
            if (MODE == 0) p1 = __ldg(params + c1);
            load_cv(p0 + 96, c2, v2);
            __syncwarp();
        }
        // gathers of the next sub-batch (its metadata is staged: same or next batch)
        uint32_t nxt[U];
        const uint32_t pn = p0 + U;
#pragma unroll
        for (int u = 0; u < U; ++u)
            nxt[u] = __ldg(reinterpret_cast<const uint32_t*>(qb + (uint64_t)s_meta[warp][(pn + u) & 63].col * ldq));
        const uint32_t base = p0 + 1;  // position after slot p0
        uint32_t rel = row_end - base;  // the row ends after slot p0 + rel
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const float2 ab = *reinterpret_cast<const float2*>(&s_meta[warp][(p0 + u) & 63]);
            float q0, q1, q2, q3;
            decode4(raw[u], q0, q1, q2, q3);
            fma2(acc0, acc1, ab.x, q0, q1);
            fma2(acc2, acc3, ab.x, q2, q3);
            bsum += ab.y;
            if (rel == (uint32_t)u) {
                advance(base + u);
                rel = row_end - base;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = nxt[u];
    }
    for (; row < nr; ++row) store_row();  // (only rows after the last slot)
}

// ---------------------------------------------------------------- ring kernel
// The default fast-mode SpMM: the cp.async ring schedule of the exact int8
// batch kernel (spmm.cu) — one warp per 32-row group, one slot stream, the
// gathers four slots per 16-B LDGSTS (lane (g, j) copies bytes 16j.. of slot
// g), slot metadata two ring rounds ahead — with the table decode replaced by
// the affine one: no 64 KB table per CTA, no table reads (4 of the ~7 shared
// wavefronts per slot of the exact kernel), and 8 instead of 14 decode /
// accumulate instructions per slot.  ROW mode stages each gathered row's
// (s, m) next to the metadata, one round ahead of its use.
constexpr int kRC = 16;            // ring slots per warp
constexpr int kRB = kRC / 4;       // 4-slot batches per round
constexpr uint32_t kREnds = 160;   // 33 row ends (padded)

template <int MODE, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
spmm_q8r_kernel(const uint64_t* __restrict__ srow, const uint32_t* __restrict__ scol,
                const float* __restrict__ sval, uint64_t n_rows, const uint8_t* __restrict__ q, uint32_t ldq,
                uint32_t f, const float2* __restrict__ params, float4* __restrict__ c, uint64_t ldc4) {
    // per warp: ring kRC x 128 B | meta 4 rounds x (kRC cols + kRC vals) | row params 4 rounds x kRC x 8 B | ends
    constexpr uint32_t kRing = kRC * 128, kMeta = 4 * 8 * kRC, kPar = MODE == 0 ? 4 * 8 * kRC : 0;
    constexpr uint32_t kPerWarp = kRing + kMeta + kPar + kREnds;
    extern __shared__ __align__(16) unsigned char rsm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(rsm) + warp * kPerWarp;
    const uint32_t ring0 = base, meta0 = base + kRing, par0 = meta0 + kMeta, ends0 = par0 + kPar;
    const uint32_t tile = blockIdx.y;
    q += (size_t)tile * 128;
    const uint32_t col0 = tile * 128 + 4 * lane;
    const uint32_t f4 = min(32u, (f + 3) / 4 - tile * 32);
    const bool st_ok = lane < f4;
    uint32_t nb = 16;  // bytes this lane copies per gathered row (partial last tile)
    {
        const uint32_t rowb = min(128u, f - tile * 128), j16 = (lane & 7) * 16;
        nb = rowb > j16 ? min(16u, rowb - j16) : 0u;
    }
    float sj[4] = {0.f, 0.f, 0.f, 0.f}, mj[4] = {0.f, 0.f, 0.f, 0.f};
    if (MODE == 1)
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (col0 + u < f) {
                const float2 p = params[col0 + u];
                sj[u] = p.x;
                mj[u] = p.y;
            }
    const uint64_t r0 = ((uint64_t)blockIdx.x * WARPS + warp) * 32;
    if (r0 >= n_rows) return;
    const uint32_t nr = (uint32_t)min((uint64_t)32, n_rows - r0);
    const uint64_t g0 = srow[r0];
    const uint64_t my_end = srow[r0 + 1 + min(lane, nr - 1)];
    const uint32_t total = (uint32_t)(__shfl_sync(0xffffffffu, my_end, nr - 1) - g0);
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + lane * 4), "r"((uint32_t)(my_end - g0)) : "memory");
    if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(ends0 + 128), "r"(total) : "memory");

    // lanes 0..15 stream scol, 16..31 sval: one per-lane base pointer
    const char* const mbase = lane < 16 ? reinterpret_cast<const char*>(scol + g0 + (lane & 15))
                                        : reinterpret_cast<const char*>(sval + g0 + (lane & 15));
    const uint32_t mdst = meta0 + (lane >> 4) * (4 * kRC) + (lane & 15) * 4;
    auto issue_meta = [&](uint32_t k) {  // round k -> buffer k & 3 (lanes 0..15 cols, 16..31 vals)
        const uint32_t s = k * kRC + (lane & 15);
        if (s < total) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(mdst + (k & 3) * (8 * kRC)),
                         "l"(mbase + (uint64_t)(k * kRC) * 4)
                         : "memory");
        }
    };
    auto issue_par = [&](uint32_t k) {  // ROW: (s, m) of round k's gathered rows -> buffer k & 3
        if (MODE == 0 && lane < (uint32_t)kRC && k * kRC + lane < total) {
            uint32_t cc;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cc) : "r"(meta0 + (k & 3) * (8 * kRC) + lane * 4));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(par0 + (k & 3) * (8 * kRC) + lane * 8),
                         "l"(params + cc)
                         : "memory");
        }
    };
    const unsigned char* const qlane = q + (lane & 7) * 16;
    const uint32_t mcol = meta0 + (lane >> 3) * 4, wr0 = ring0 + (lane >> 3) * 128 + (lane & 7) * 16;
    auto issue = [&](int p0, uint32_t k) {  // gathers for ring positions p0..p0+3 of round k
        const uint32_t t = k * kRC + p0 + (lane >> 3);
        if (t < total && nb) {
            uint32_t cc;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cc) : "r"(mcol + (k & 3) * (8 * kRC) + p0 * 4));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(wr0 + p0 * 128),
                         "l"(qlane + (uint64_t)cc * ldq), "r"(nb)
                         : "memory");
        }
    };
    issue_meta(0);
    issue_meta(1);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
    issue_par(0);
#pragma unroll
    for (int b = 0; b < kRB; ++b) {
        issue(4 * b, 0);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }

    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, bs = 0.f;
    uint32_t row = 0, row_end;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(row_end) : "r"(ends0));
    float4* cptr = c + r0 * ldc4 + tile * 32 + lane;
    auto store_row = [&]() {
        if (st_ok) {
            float4 o;
            if (MODE == 0)
                o = make_float4(__fadd_rn(a0, bs), __fadd_rn(a1, bs), __fadd_rn(a2, bs), __fadd_rn(a3, bs));
            else
                o = make_float4(fmaf(sj[0], a0, mj[0] * bs), fmaf(sj[1], a1, mj[1] * bs), fmaf(sj[2], a2, mj[2] * bs),
                                fmaf(sj[3], a3, mj[3] * bs));
            __stcs(cptr, o);
        }
        cptr += ldc4;
        a0 = a1 = a2 = a3 = bs = 0.f;
    };
    auto advance_rows = [&](uint32_t pos) {
        do {
            store_row();
            ++row;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(row_end) : "r"(ends0 + row * 4));
        } while (row < nr && row_end == pos);
    };
    if (row_end == 0) advance_rows(0);
    const uint32_t rd0 = ring0 + lane * 4;
    auto consume = [&](int p, float a, float b) {
        uint32_t r;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(rd0 + p * 128));
        float q0 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7650));
        float q1 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7651));
        float q2 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7652));
        float q3 = __uint_as_float(__byte_perm(r, 0x4B000000u, 0x7653));
        add2_rn(q0, q1, -kTwo23, -kTwo23);
        add2_rn(q2, q3, -kTwo23, -kTwo23);
        fma2(a0, a1, a, q0, q1);
        fma2(a2, a3, a, q2, q3);
        bs = __fadd_rn(bs, b);
    };

    // every round consumes all kRC positions; past `total` (last round only)
    // garbage accumulates after the last row was stored and is never written
    for (uint32_t k = 0, t0 = 0; t0 < total; t0 += kRC, ++k) {
#pragma unroll
        for (int b = 0; b < kRB; ++b) {
            asm volatile("cp.async.wait_group %0;\n" ::"n"(kRB - 1) : "memory");
            __syncwarp();
            float4 v4;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v4.x), "=f"(v4.y), "=f"(v4.z), "=f"(v4.w)
                         : "r"(meta0 + (k & 3) * (8 * kRC) + 4 * kRC + 16 * b));
            float av[4] = {v4.x, v4.y, v4.z, v4.w}, bv[4] = {v4.x, v4.y, v4.z, v4.w};
            if (MODE == 0) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    float2 sm;
                    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(sm.x), "=f"(sm.y)
                                 : "r"(par0 + (k & 3) * (8 * kRC) + (4 * b + u) * 8));
                    bv[u] = __fmul_rn(av[u], sm.y);  // (no contraction into the sums: the
                    av[u] = __fmul_rn(av[u], sm.x);  // batch kernel's DEC 2 gives the same bits)
                }
            }
            if (row_end > t0 + 4 * b + 4) {  // no row ends in this batch
#pragma unroll
                for (int u = 0; u < 4; ++u) consume(4 * b + u, av[u], bv[u]);
            } else {
                const uint32_t pb = t0 + 4 * b + 1;
                uint32_t rel = row_end - pb;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    consume(4 * b + u, av[u], bv[u]);
                    if (rel == (uint32_t)u) {
                        advance_rows(pb + u);
                        rel = row_end - pb;
                    }
                }
            }
            __syncwarp();  // every lane is done reading these ring slots
            if (b == 0) {
                issue_meta(k + 2);
                issue_par(k + 1);  // round k+1's metadata landed with the wait above
            }
            issue(4 * b, k + 1);
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    while (row < nr) {
        store_row();
        ++row;
    }
}

template <int MODE, int WARPS, int MINB>
int launch_q8r_t(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                 uint64_t ldq, uint64_t f, const float2* params, float* c, uint64_t ldc, cudaStream_t st) {
    constexpr uint32_t kPerWarp = kRC * 128 + 4 * 8 * kRC + (MODE == 0 ? 4 * 8 * kRC : 0) + kREnds;
    const size_t smem = (size_t)WARPS * kPerWarp;
    static bool attr_dev[kMaxDevices] = {};
    bool& attr = attr_dev[cur_device()];
    if (!attr) {
        AES_CUDA_TRY(cudaFuncSetAttribute(spmm_q8r_kernel<MODE, WARPS, MINB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const uint64_t groups = (n + 31) / 32;
    const dim3 grid((unsigned)((groups + WARPS - 1) / WARPS), (unsigned)((f + 127) / 128));
    spmm_q8r_kernel<MODE, WARPS, MINB><<<grid, WARPS * 32, smem, st>>>(srow, scol, sval, n, q, (uint32_t)ldq,
                                                                      (uint32_t)f, params,
                                                                      reinterpret_cast<float4*>(c), ldc / 4);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

// Default 16 warps x 2 CTAs per SM with room for 64 registers (measured on
// B200: products feature 0.594 -> 0.537 ms, reddit feature 0.621 -> 0.475,
// reddit row 0.595 -> 0.522; products row 0.565 -> 0.575).  Tuning variants:
// 54 = 16 warps x 3 CTAs (40 registers), 53 = 32 warps x 1.
template <int MODE>
int launch_q8r(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
               uint64_t ldq, uint64_t f, const float2* params, float* c, uint64_t ldc, cudaStream_t st, int v) {
    if (v == 54) return launch_q8r_t<MODE, 16, 3>(srow, scol, sval, n, q, ldq, f, params, c, ldc, st);
    if (v == 53) return launch_q8r_t<MODE, 32, 1>(srow, scol, sval, n, q, ldq, f, params, c, ldc, st);
    return launch_q8r_t<MODE, 16, 2>(srow, scol, sval, n, q, ldq, f, params, c, ldc, st);
}

template <int MODE>
int launch_q8a(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
               uint64_t ldq, uint64_t f, const float2* params, float* c, uint64_t ldc, cudaStream_t st) {
    constexpr int kWarps = 8, kU = 8;
    const uint64_t groups = (n + 31) / 32;
    const dim3 grid((unsigned)((groups + kWarps - 1) / kWarps), (unsigned)((f + 127) / 128));
    spmm_q8a_kernel<MODE, kU, kWarps><<<grid, kWarps * 32, 0, st>>>(srow, scol, sval, n, q, (uint32_t)ldq,
                                                                    (uint32_t)f, params, c, ldc);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

}  // namespace

int launch_spmm_q8_tma(int dec, const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n,
                       const uint8_t* q, uint64_t ldq, uint64_t f, const float* lut, const float* fparams, float* c,
                       uint64_t ldc, cudaStream_t st);  // spmm_tma.cu
int spmm_variant();                                     // spmm.cu
int launch_q8_feature_batch(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n,
                            const uint8_t* q, uint64_t ldq, uint64_t f, const float2* params, float* c, uint64_t ldc,
                            cudaStream_t st);  // spmm.cu
int launch_q8_row_batch(const uint64_t* srow, const uint32_t* scol, const float* sval, uint64_t n, const uint8_t* q,
                        uint64_t ldq, uint64_t f, const float2* params, float* c, uint64_t ldc,
                        cudaStream_t st);  // spmm.cu
}  // namespace aes

extern "C" {

uint64_t aes_quantize_affine_workspace_bytes(uint64_t rows, uint64_t cols, int mode) {
    using namespace aes;
    if (mode != AES_QAFFINE_FEATURE) return 256;
    const uint64_t blocks = (rows + kColRowsPerCta - 1) / kColRowsPerCta;
    return 256 + (blocks ? blocks : 1) * (cols ? cols : 1) * sizeof(float2);
}

int aes_dev_quantize_affine(const float* x, uint64_t rows, uint64_t cols, uint64_t ldx, int mode, uint8_t* q,
                            uint64_t ldq, float* params, unsigned int* bad_flag, void* workspace,
                            size_t workspace_bytes, void* stream) {
    using namespace aes;
    if (mode != AES_QAFFINE_ROW && mode != AES_QAFFINE_FEATURE) return fail(AES_ERR_INVALID_ARG, "unknown affine mode");
    if (!x || !q || !params || !bad_flag) return fail(AES_ERR_INVALID_ARG, "null argument");
    if (ldq % 4 || (uintptr_t)q % 4 || ldq < ((cols + 3) & ~3ull) || ldx < cols)
        return fail(AES_ERR_UNSUPPORTED, "affine quantize needs ldq % 4 == 0 and ldq >= round_up(cols, 4)");
    if (workspace_bytes < aes_quantize_affine_workspace_bytes(rows, cols, mode) || !workspace)
        return fail(AES_ERR_INVALID_ARG, "affine quantize workspace too small");
    cudaStream_t st = as_stream(stream);
    AES_CUDA_TRY(cudaMemsetAsync(bad_flag, 0, sizeof(unsigned int), st));
    if (rows == 0 || cols == 0) return AES_OK;
    float2* p2 = reinterpret_cast<float2*>(params);
    if (mode == AES_QAFFINE_ROW) {
        quant_row_kernel<<<grid_for(rows * 32, 256, num_sms() * 16), 256, 0, st>>>(x, rows, cols, ldx, q, ldq, p2,
                                                                                   bad_flag);
    } else {
        const uint64_t blocks = (rows + kColRowsPerCta - 1) / kColRowsPerCta;
        float2* partial = reinterpret_cast<float2*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
        col_minmax_kernel<<<dim3((unsigned)blocks, (unsigned)((cols + 31) / 32)), 256, 0, st>>>(x, rows, cols, ldx,
                                                                                             partial, bad_flag);
        col_params_kernel<<<grid_for(cols, 128), 128, 0, st>>>(partial, blocks, cols, p2);
        quant_col_kernel<<<grid_for(rows * ((cols + 3) / 4), 256, num_sms() * 32), 256, 0, st>>>(x, rows, cols, ldx,
                                                                                                 p2, q, ldq);
    }
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_dequantize_affine(const uint8_t* q, uint64_t rows, uint64_t cols, uint64_t ldq, int mode,
                              const float* params, float* x, uint64_t ldx, void* stream) {
    using namespace aes;
    if (mode != AES_QAFFINE_ROW && mode != AES_QAFFINE_FEATURE) return fail(AES_ERR_INVALID_ARG, "unknown affine mode");
    cudaStream_t st = as_stream(stream);
    if (rows == 0 || cols == 0) return AES_OK;
    const float2* p2 = reinterpret_cast<const float2*>(params);
    const unsigned grid = grid_for(rows * cols, 256, num_sms() * 32);
    if (mode == AES_QAFFINE_ROW)
        dequant_affine_kernel<0><<<grid, 256, 0, st>>>(q, rows, cols, ldq, p2, x, ldx);
    else
        dequant_affine_kernel<1><<<grid, 256, 0, st>>>(q, rows, cols, ldq, p2, x, ldx);
    AES_CUDA_TRY(cudaGetLastError());
    return AES_OK;
}

int aes_dev_spmm_q8_affine(const uint64_t* srow_ptr, const uint32_t* scol, const float* sval, uint64_t n_rows,
                           const uint8_t* q, uint64_t ldq, uint64_t f, int mode, const float* params, float* c,
                           uint64_t ldc, void* stream) {
    using namespace aes;
    if (mode != AES_QAFFINE_ROW && mode != AES_QAFFINE_FEATURE) return fail(AES_ERR_INVALID_ARG, "unknown affine mode");
    if (n_rows == 0 || f == 0) return AES_OK;
    if (ldq % 4 || (uintptr_t)q % 4 || ldq < ((f + 3) & ~3ull) || ldc % 4 || (uintptr_t)c % 16 || ldc < f)
        return fail(AES_ERR_UNSUPPORTED, "affine spmm needs ldq % 4 == 0, ldc % 4 == 0, 16-B aligned C");
    if (f > 0xffffffffull || ldq > 0xffffffffull) return fail(AES_ERR_UNSUPPORTED, "F too large");
    cudaStream_t st = as_stream(stream);
    const float2* p2 = reinterpret_cast<const float2*>(params);
    const int v = spmm_variant();
    // tuning variants: 51 the TMA-gather kernel (FEATURE), 50 the register-pipelined one
    if (v == 51 && mode == AES_QAFFINE_FEATURE) {
        const int s = launch_spmm_q8_tma(1, srow_ptr, scol, sval, n_rows, q, ldq, f, nullptr, params, c, ldc, st);
        if (s != AES_ERR_UNSUPPORTED) return s;
    }
    // the batch kernel with the affine decode (spmm.cu), unless a tuning
    // variant asks for the ring kernel (52-54).  Per-row codes on one large
    // 128-code tile stay on the ring kernel: products 0.564 ms vs 0.626 for
    // the batch kernel's balanced wave (whose per-slot (s, m) read adds an
    // LDS + 2 FMUL); with several tiles or fewer rows the batch kernel wins
    // (reddit 0.496 vs 0.593, arxiv 0.034 vs 0.058, pubmed 0.017 vs 0.029)
    const bool row_ring = mode == AES_QAFFINE_ROW && f <= 128 && n_rows >= (1u << 20);
    if ((v == 0 || (v >= 55 && v <= 57)) && n_rows < (1ull << 31) && !(row_ring && v == 0)) {
        const int s = mode == AES_QAFFINE_FEATURE
                          ? launch_q8_feature_batch(srow_ptr, scol, sval, n_rows, q, ldq, f, p2, c, ldc, st)
                          : launch_q8_row_batch(srow_ptr, scol, sval, n_rows, q, ldq, f, p2, c, ldc, st);
        if (s != AES_ERR_UNSUPPORTED) return s;
    }
    // default: the cp.async ring kernel (16-B code rows, 16-B aligned C)
    if (v != 50 && ldq % 16 == 0 && (uintptr_t)q % 16 == 0 && n_rows < (1ull << 31)) {
        if (mode == AES_QAFFINE_ROW) return launch_q8r<0>(srow_ptr, scol, sval, n_rows, q, ldq, f, p2, c, ldc, st, v);
        return launch_q8r<1>(srow_ptr, scol, sval, n_rows, q, ldq, f, p2, c, ldc, st, v);
    }
    if (mode == AES_QAFFINE_ROW) return launch_q8a<0>(srow_ptr, scol, sval, n_rows, q, ldq, f, p2, c, ldc, st);
    return launch_q8a<1>(srow_ptr, scol, sval, n_rows, q, ldq, f, p2, c, ldc, st);
}

}  // extern "C"
