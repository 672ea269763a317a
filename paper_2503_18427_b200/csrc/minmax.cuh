// (value, index) min / max reduction with the reference fit_params
// semantics (proj/src/quantize.cpp:11-21): the FIRST element attaining the
// min / max under strict '<' / '>' wins, so ties (and -0.0f vs +0.0f)
// resolve to the lowest index; a non-finite element sets `bad`.  Shared by
// fit_params (quant.cu) and the layer GEMM's fused fit epilogue (gemm.cu).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace aes {

struct MinMax {
    float lo, hi;
    uint64_t ilo, ihi;
    uint32_t bad;
};

__device__ __forceinline__ void mm_merge(MinMax& a, const MinMax& b) {
    if (b.lo < a.lo || (b.lo == a.lo && b.ilo < a.ilo)) { a.lo = b.lo; a.ilo = b.ilo; }
    if (b.hi > a.hi || (b.hi == a.hi && b.ihi < a.ihi)) { a.hi = b.hi; a.ihi = b.ihi; }
    a.bad |= b.bad;
}

__device__ __forceinline__ MinMax mm_shfl(const MinMax& m, int o) {
    MinMax r;
    r.lo = __shfl_down_sync(0xffffffffu, m.lo, o);
    r.hi = __shfl_down_sync(0xffffffffu, m.hi, o);
    r.ilo = __shfl_down_sync(0xffffffffu, m.ilo, o);
    r.ihi = __shfl_down_sync(0xffffffffu, m.ihi, o);
    r.bad = __shfl_down_sync(0xffffffffu, m.bad, o);
    return r;
}

template <int THREADS>
__device__ MinMax block_reduce(MinMax m) {
    __shared__ MinMax s[THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) {
        MinMax t = mm_shfl(m, o);
        mm_merge(m, t);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) s[wid] = m;
    __syncthreads();
    if (wid == 0) {
        m = s[lane < THREADS / 32 ? lane : 0];
        for (int o = 16; o > 0; o >>= 1) {
            MinMax t = mm_shfl(m, o);
            mm_merge(m, t);
        }
    }
    return m;
}

// A thread sees its elements in increasing index order, so the strict
// compares alone keep the first occurrence (an equal later value never
// replaces); the index only matters when partial results merge.
__device__ __forceinline__ void fit_elem(MinMax& m, float v, uint64_t i) {
    if (!isfinite(v)) { m.bad = 1; return; }
    if (v < m.lo) { m.lo = v; m.ilo = i; }
    if (v > m.hi) { m.hi = v; m.ihi = i; }
}


}  // namespace aes
