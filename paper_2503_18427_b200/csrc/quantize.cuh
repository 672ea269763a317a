// Exact quantization (proj/src/quantize.cpp:23-51) with an fp32 fast path.
//
// The reference code of x is
//     q(x) = clamp(floor(t), 0, L),   t = RN(RN(RN(RN(x - lo) / range) * L) + 2^-7)
// in fp64 (range = RN(hi - lo) > 0, L = 2^bits - 1).  The fast path computes
//     e = RN32(RN32(x - lo) * s + 2^-7),   s = RN32(L / range)   (one FFMA)
// and uses floor(e) whenever e is provably on the same side of every integer
// as t.  Error bound: x - lo and L / range each carry relative error <= 2^-24
// in fp32 (a subnormal difference of two floats is exact; s cannot be
// subnormal because range <= 2 FLT_MAX), the FFMA adds <= 2^-24 |e|, and the
// fp64 chain adds <= 2^-50 |t|, so for finite e
//     |e - t| <= 3.1 * 2^-24 * max(|e|, |t|) < 2^-12  when |e| < L + 1 <= 65536
// (2^-24 * 3.1 * 65536 = 0.012 for 16 bits: the margin below scales with L).
// Hence:  |e| < L + 1 and frac(e) in (m, 1 - m)  =>  floor(e) = floor(t);
//         L + 1 <= e <= FLT_MAX  =>  t > L  =>  code L;
//         -FLT_MAX <= e <= -1    =>  t < 0  =>  code 0;
// everything else (e within m of an integer, +-inf or NaN from an fp32
// overflow, NaN input) takes the exact fp64 formula.  m = 2^-12 for bits <= 8
// (|e - t| < 4.8e-5 there) and 2^-5 for bits <= 16.  Bit-exact by
// construction; for data inside [lo, hi] the fallback is ~5e-4 of the elements
// at 8 bits.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace aes {

// The reference formula in fp64 with explicit roundings (no FMA contraction).
__device__ __forceinline__ uint32_t quant_code_exact(float x, double lo, double range, double dlev) {
    if (range == 0.0) return 0u;  // degenerate range: every code 0 (quantize.cpp:35-38)
    double qd = floor(__dadd_rn(__dmul_rn(__ddiv_rn(__dsub_rn((double)x, lo), range), dlev), 0.0078125));
    qd = qd < 0.0 ? 0.0 : qd;  // std::clamp(q, 0, levels); NaN stays NaN -> code 0
    qd = dlev < qd ? dlev : qd;
    return (uint32_t)qd;
}

struct QuantParamsDev {
    float lo_f;     // x_min
    float scale;    // RN32(L / range) (any value when range == 0)
    float top;      // L + 1
    float margin;   // m
    uint32_t levels;
    double lo, range, dlev;
};

__device__ __forceinline__ QuantParamsDev quant_params(float lo_f, float hi_f, uint32_t levels) {
    QuantParamsDev p;
    p.lo_f = lo_f;
    p.levels = levels;
    p.lo = (double)lo_f;
    p.range = __dsub_rn((double)hi_f, p.lo);
    p.dlev = (double)levels;
    p.scale = __double2float_rn(__ddiv_rn(p.dlev, p.range > 0.0 ? p.range : 1.0));
    p.top = (float)(levels + 1);
    p.margin = levels <= 255 ? 1.0f / 4096.0f : 1.0f / 32.0f;
    return p;
}

// Code of x, bit-identical to quant_code_exact (see the header comment).
__device__ __forceinline__ uint32_t quant_code(float x, const QuantParamsDev& p) {
    if (p.range == 0.0) return 0u;
    const float e = __fmaf_rn(__fsub_rn(x, p.lo_f), p.scale, 0.0078125f);
    const float fl = floorf(e);
    const float fr = __fsub_rn(e, fl);
    if (fabsf(e) < p.top && fr > p.margin && fr < 1.0f - p.margin)
        return (uint32_t)min(max((int)fl, 0), (int)p.levels);
    if (e >= p.top && e <= 3.4028235e38f) return p.levels;
    if (e <= -1.0f && e >= -3.4028235e38f) return 0u;
    return quant_code_exact(x, p.lo, p.range, p.dlev);
}

}  // namespace aes
