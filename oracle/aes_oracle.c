/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the AES-SpMM hot path.
 *
 * A plain-C restatement of the reference algorithm (arxiv 2503.18427 reference,
 * /root/reference/proj) used ONLY by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py, as the checker.  Nothing in the product path
 * links, loads or calls this file.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against the
 * reference's own golden values and against the UNMODIFIED
 * reference compiled by oracle/Makefile into oracle/_ref (when present), and
 * tests/golden/*.npz fixtures generated from that reference build.
 *
 * Arithmetic contract (compiled -O2 -ffp-contract=off, no -march): every fp32
 * product and sum is rounded separately, matching the reference build, which
 * contains no FMA instructions.
 *
 * Strategy numbering follows the reference enum order
 * (proj/include/aesspmm/sampling.hpp:14): Adaptive=0, Afs=1, Sfs=2, Full=3.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_ADAPTIVE = 0, OR_AFS = 1, OR_SFS = 2, OR_FULL = 3 };
enum { OR_OK = 0, OR_ZERO_WIDTH = 1, OR_EMPTY = 2, OR_NONFINITE = 3, OR_BAD_PARAMS = 4 };

/* Table 1 of the paper as stated in proj/src/sampling.cpp:29-54.
 * Comparisons are on integers so R == 1, 2, 36, 54 fall in the lower-ratio
 * ("<=") branch; afterwards chunk is raised to >= 1 and cnt capped at W. */
int or_select_strategy(uint64_t nnz, uint32_t w, uint32_t *chunk, uint32_t *cnt) {
    uint32_t c, n;
    if (w == 0) return OR_ZERO_WIDTH;
    if (nnz == 0) { *chunk = 0; *cnt = 0; return OR_OK; }
    if (nnz <= (uint64_t)w) { *chunk = (uint32_t)nnz; *cnt = 1; return OR_OK; }
    if (nnz <= 2ull * w)       { c = w / 4;  n = 4; }
    else if (nnz <= 36ull * w) { c = w / 8;  n = 8; }
    else if (nnz <= 54ull * w) { c = w / 16; n = 16; }
    else                       { c = w / 32; n = 32; }
    *chunk = c < 1 ? 1 : c;
    *cnt = n > w ? w : n;
    return OR_OK;
}

/* Eq. 3: start = (s * 1429) mod (nnz - chunk + 1), in 64-bit
 * (proj/src/sampling.cpp:56-60, kHashPrime at sampling.hpp:12). */
uint32_t or_hash_start(uint32_t s, uint64_t nnz, uint32_t chunk) {
    uint64_t range = nnz - (uint64_t)chunk + 1u;
    return (uint32_t)(((uint64_t)s * 1429ull) % range);
}

/* One row's plan (proj/src/sampling.cpp:62-102).  `starts` must hold
 * max(W, 1) entries; *n_starts receives how many were written. */
int or_row_plan(uint64_t nnz, uint32_t w, int strategy, uint32_t *chunk,
                uint32_t *cnt, uint32_t *starts, uint32_t *n_starts) {
    uint32_t s;
    if (w == 0) return OR_ZERO_WIDTH;
    *chunk = 0; *cnt = 0; *n_starts = 0;
    if (nnz == 0) return OR_OK;
    switch (strategy) {
    case OR_FULL:
        *chunk = (uint32_t)nnz; *cnt = 1; starts[0] = 0; *n_starts = 1;
        break;
    case OR_SFS:
        *chunk = (uint32_t)(nnz < w ? nnz : w); *cnt = 1; starts[0] = 0; *n_starts = 1;
        break;
    case OR_AFS:
        *chunk = 1;
        *cnt = (uint32_t)(nnz < w ? nnz : w);
        for (s = 0; s < *cnt; ++s) starts[s] = (uint32_t)((uint64_t)s * nnz / *cnt);
        *n_starts = *cnt;
        break;
    default: /* adaptive */
        or_select_strategy(nnz, w, chunk, cnt);
        if (nnz <= w) { starts[0] = 0; *n_starts = 1; }
        else {
            for (s = 0; s < *cnt; ++s) starts[s] = or_hash_start(s, nnz, *chunk);
            *n_starts = *cnt;
        }
        break;
    }
    return OR_OK;
}

/* (chunk, cnt) of a row under each strategy, without the starts
 * (proj/src/sampling.cpp:68-99). */
void or_row_params(uint64_t nnz, uint32_t w, int strategy, uint32_t *chunk, uint32_t *cnt) {
    *chunk = 0; *cnt = 0;
    if (nnz == 0) return;
    switch (strategy) {
    case OR_FULL: *chunk = (uint32_t)nnz; *cnt = 1; break;
    case OR_SFS:  *chunk = (uint32_t)(nnz < w ? nnz : w); *cnt = 1; break;
    case OR_AFS:  *chunk = 1; *cnt = (uint32_t)(nnz < w ? nnz : w); break;
    default:      or_select_strategy(nnz, w, chunk, cnt); break;
    }
}

/* Start offset of window s (proj/src/sampling.cpp:70-99): 0 for Full/Sfs and
 * whole Adaptive rows, floor(s*nnz/cnt) for Afs, the hash otherwise. */
uint32_t or_row_start(uint64_t nnz, uint32_t w, int strategy, uint32_t chunk,
                      uint32_t cnt, uint32_t s) {
    if (strategy == OR_FULL || strategy == OR_SFS) return 0;
    if (strategy == OR_AFS) return (uint32_t)((uint64_t)s * nnz / cnt);
    if (nnz <= w) return 0;
    return or_hash_start(s, nnz, chunk);
}

/* Sampled row pointer: srow_ptr[i+1] - srow_ptr[i] = chunk_i * cnt_i
 * (RowSamplePlan::slots, proj/include/aesspmm/sampling.hpp:33-35). */
int or_sample_count(uint64_t n, const uint64_t *row_ptr, uint32_t w, int strategy,
                    uint64_t *srow_ptr) {
    uint64_t i, acc = 0;
    uint32_t chunk, cnt;
    if (w == 0) return OR_ZERO_WIDTH;
    srow_ptr[0] = 0;
    for (i = 0; i < n; ++i) {
        or_row_params(row_ptr[i + 1] - row_ptr[i], w, strategy, &chunk, &cnt);
        acc += (uint64_t)chunk * cnt;
        srow_ptr[i + 1] = acc;
    }
    return OR_OK;
}

/* The buffer fill of proj/src/spmm.cpp:54-76 materialised as a CSR: slot
 * s + j*cnt of row i holds nonzero row_ptr[i] + starts[s] + j.  Duplicate
 * and unsorted columns (hash collisions, overlapping windows) are kept. */
int or_sample_fill(uint64_t n, const uint64_t *row_ptr, const uint32_t *col,
                   const float *val, uint32_t w, int strategy,
                   const uint64_t *srow_ptr, uint32_t *scol, float *sval) {
    uint64_t i;
    uint32_t chunk, cnt, s, j;
    if (w == 0) return OR_ZERO_WIDTH;
    for (i = 0; i < n; ++i) {
        uint64_t nnz = row_ptr[i + 1] - row_ptr[i];
        or_row_params(nnz, w, strategy, &chunk, &cnt);
        for (s = 0; s < cnt; ++s) {
            uint32_t st = or_row_start(nnz, w, strategy, chunk, cnt, s);
            for (j = 0; j < chunk; ++j) {
                uint64_t src = row_ptr[i] + st + j;
                uint64_t dst = srow_ptr[i] + s + (uint64_t)j * cnt;
                scol[dst] = col[src];
                sval[dst] = val[src];
            }
        }
    }
    return OR_OK;
}

/* C[i,:] = sum over slots k (ascending) of sval[k] * B[scol[k],:], each step
 * acc = RN(acc + RN(v*b)) from acc = +0.0f (proj/src/spmm.cpp:77-84, and
 * spmm_exact at spmm.cpp:18-36 when given the original CSR). */
void or_spmm_csr(uint64_t n, const uint64_t *srow_ptr, const uint32_t *scol,
                 const float *sval, const float *b, uint64_t ldb, uint64_t f,
                 float *c, uint64_t ldc) {
    uint64_t i, k, j;
    for (i = 0; i < n; ++i) {
        float *out = c + i * ldc;
        for (j = 0; j < f; ++j) out[j] = 0.0f;
        for (k = srow_ptr[i]; k < srow_ptr[i + 1]; ++k) {
            const float *brow = b + (uint64_t)scol[k] * ldb;
            float v = sval[k];
            for (j = 0; j < f; ++j) {
                float p = v * brow[j];
                out[j] = out[j] + p;
            }
        }
    }
}

/* fit_params (proj/src/quantize.cpp:11-21): first-occurrence min/max with
 * strict comparisons, error on empty or non-finite input. */
int or_fit_params(const float *x, uint64_t n, uint32_t bits, float *lo, float *hi) {
    uint64_t k;
    float l, h;
    if (n == 0) return OR_EMPTY;
    if (bits < 1 || bits > 16) return OR_BAD_PARAMS;
    l = x[0]; h = x[0];
    for (k = 0; k < n; ++k) {
        float v = x[k];
        if (!isfinite(v)) return OR_NONFINITE;
        if (v < l) l = v;
        if (h < v) h = v;
    }
    *lo = l; *hi = h;
    return OR_OK;
}

/* quantize (proj/src/quantize.cpp:23-51): fp64, floor(ratio*levels + 2^-7),
 * clamp to [0, levels]; a zero range yields all-zero codes. */
int or_quantize(const float *x, uint64_t n, float lo, float hi, uint32_t bits,
                uint16_t *codes) {
    uint64_t k;
    double range, levels;
    if (bits < 1 || bits > 16 || !(lo <= hi)) return OR_BAD_PARAMS;
    range = (double)hi - (double)lo;
    levels = (double)((1u << bits) - 1u);
    if (range == 0.0) { memset(codes, 0, n * sizeof(uint16_t)); return OR_OK; }
    for (k = 0; k < n; ++k) {
        double r = ((double)x[k] - (double)lo) / range;
        double t = r * levels;
        double q = floor(t + 0.0078125);
        if (q < 0.0) q = 0.0;
        if (q > levels) q = levels;
        codes[k] = (uint16_t)q;
    }
    return OR_OK;
}

/* dequantize (proj/src/quantize.cpp:53-64): float(q*step + lo) in fp64. */
void or_dequantize(const uint16_t *codes, uint64_t n, float lo, float hi,
                   uint32_t bits, float *x) {
    uint64_t k;
    double step = ((double)hi - (double)lo) / (double)((1u << bits) - 1u);
    for (k = 0; k < n; ++k) {
        double t = (double)codes[k] * step;
        x[k] = (float)(t + (double)lo);
    }
}

/* dense_matmul (proj/src/gnn.cpp:11-31): i-k-j order, k ascending, zero
 * entries of A skipped, separate mul/add roundings. */
void or_dense_matmul(const float *a, uint64_t m, uint64_t kdim, const float *b,
                     uint64_t n, float *c) {
    uint64_t i, k, j;
    for (i = 0; i < m; ++i) {
        float *out = c + i * n;
        for (j = 0; j < n; ++j) out[j] = 0.0f;
        for (k = 0; k < kdim; ++k) {
            float av = a[i * kdim + k];
            if (av == 0.0f) continue;
            for (j = 0; j < n; ++j) {
                float p = av * b[k * n + j];
                out[j] = out[j] + p;
            }
        }
    }
}

/* add_bias_inplace + relu_inplace (proj/src/gnn.cpp:41-52). */
void or_bias_act(float *c, uint64_t m, uint64_t n, const float *bias, int relu) {
    uint64_t i, j;
    for (i = 0; i < m; ++i) {
        for (j = 0; j < n; ++j) {
            float v = c[i * n + j];
            if (bias) v = v + bias[j];
            if (relu) v = v > 0.0f ? v : 0.0f;   /* std::max(v, 0.0f) */
            c[i * n + j] = v;
        }
    }
}

/* gcn_normalize (proj/src/matrix.cpp:107-144).  Pass 1 (out_col == NULL)
 * returns the output row pointer; pass 2 fills columns and values.  Self
 * loops are inserted in sorted position when absent; deg = post-insertion row
 * nnz; val = (1/sqrtf(deg_i)) * (1/sqrtf(deg_j)) in float. */
void or_gcn_normalize(uint64_t n, const uint64_t *row_ptr, const uint32_t *col,
                      int add_self_loops, uint64_t *out_ptr, uint32_t *out_col,
                      float *out_val, float *inv_sqrt_deg /* n scratch */) {
    uint64_t i, k, o = 0;
    out_ptr[0] = 0;
    for (i = 0; i < n; ++i) {
        int has_diag = 0;
        for (k = row_ptr[i]; k < row_ptr[i + 1]; ++k) has_diag |= (col[k] == i);
        {
            int ins = add_self_loops && !has_diag;
            k = row_ptr[i];
            while (k < row_ptr[i + 1] && col[k] < i) { if (out_col) out_col[o] = col[k]; ++o; ++k; }
            if (ins) { if (out_col) out_col[o] = (uint32_t)i; ++o; }
            while (k < row_ptr[i + 1]) { if (out_col) out_col[o] = col[k]; ++o; ++k; }
        }
        out_ptr[i + 1] = o;
    }
    if (!out_col) return;
    for (i = 0; i < n; ++i) {
        uint64_t deg = out_ptr[i + 1] - out_ptr[i];
        inv_sqrt_deg[i] = deg ? 1.0f / sqrtf((float)deg) : 0.0f;
    }
    for (i = 0; i < n; ++i)
        for (k = out_ptr[i]; k < out_ptr[i + 1]; ++k)
            out_val[k] = inv_sqrt_deg[i] * inv_sqrt_deg[out_col[k]];
}

/* row_mean_normalize (proj/src/matrix.cpp:146-158): val = 1/row_nnz in float. */
void or_row_mean_normalize(uint64_t n, const uint64_t *row_ptr, float *val) {
    uint64_t i, k;
    for (i = 0; i < n; ++i) {
        uint64_t nnz = row_ptr[i + 1] - row_ptr[i];
        if (nnz == 0) continue;
        {
            float w = 1.0f / (float)nnz;
            for (k = row_ptr[i]; k < row_ptr[i + 1]; ++k) val[k] = w;
        }
    }
}

/* sampling_rate (proj/src/sampling.cpp:120-152): aggregate slot rate and
 * unique coverage of sampled offsets.  `seen` is scratch of max_row_nnz bytes. */
int or_sampling_rate(uint64_t n, const uint64_t *row_ptr, uint32_t w, int strategy,
                     uint8_t *seen, double *aggregate, double *unique) {
    uint64_t i, tot_slots = 0, tot_unique = 0, tot_nnz = 0, k;
    uint32_t chunk, cnt, s, j, ns;
    if (w == 0) return OR_ZERO_WIDTH;
    for (i = 0; i < n; ++i) {
        uint64_t nnz = row_ptr[i + 1] - row_ptr[i];
        tot_nnz += nnz;
        if (nnz == 0) continue;
        or_row_params(nnz, w, strategy, &chunk, &cnt);
        tot_slots += (uint64_t)chunk * cnt;
        /* whole rows carry a single start (sampling.cpp:70-77, 90-91) */
        ns = (strategy == OR_FULL || strategy == OR_SFS ||
              (strategy == OR_ADAPTIVE && nnz <= w)) ? 1 : cnt;
        memset(seen, 0, nnz);
        for (s = 0; s < ns; ++s) {
            uint32_t st = or_row_start(nnz, w, strategy, chunk, cnt, s);
            for (j = 0; j < chunk; ++j) seen[st + j] = 1;
        }
        for (k = 0; k < nnz; ++k) tot_unique += seen[k];
    }
    *aggregate = tot_nnz == 0 ? 1.0 : (double)tot_slots / (double)tot_nnz;
    *unique = tot_nnz == 0 ? 1.0 : (double)tot_unique / (double)tot_nnz;
    return OR_OK;
}

/* cdf_stats (proj/src/bench.cpp:124-138): sort ascending, then one step per
 * run of equal (==) values: (first value of the run, (last index + 1) / n).
 * Sorts `rates` in place.  Returns the step count, or 0 for n == 0 (the
 * reference throws "rates must be nonempty"). */
static int or_cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) ? -1 : (y < x) ? 1 : 0;
}
uint64_t or_cdf_stats(double *rates, uint64_t n, double *out_rate, double *out_frac) {
    uint64_t i, steps = 0;
    if (n == 0) return 0;
    qsort(rates, n, sizeof(double), or_cmp_double);
    for (i = 0; i < n; ++i) {
        double fraction = (double)(i + 1) / (double)n;
        if (steps && out_rate[steps - 1] == rates[i]) {
            out_frac[steps - 1] = fraction;
        } else {
            out_rate[steps] = rates[i];
            out_frac[steps] = fraction;
            ++steps;
        }
    }
    return steps;
}
