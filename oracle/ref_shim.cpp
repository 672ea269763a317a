// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// A thin extern "C" driver over the UNMODIFIED reference library, compiled by
// oracle/Makefile from the sources under /root/reference/proj (outputs go to
// oracle/_ref/ only).  It exposes the reference entry points the pybind `_core`
// module does not bind (gen_synthetic, gcn_normalize, gcn_forward,
// dense_matmul) plus a kernel-only timer that mirrors the reference's own
// measurement loop (proj/src/bench.cpp:71-77: prebuilt plans, median of runs).
//
// Used by: tests/ (parity pinning), tests/golden/make_golden.py (fixtures) and
// bench.py --impl reference (the reference's CPU path timed on the host cores).

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "aesspmm/bench.hpp"
#include "aesspmm/gnn.hpp"
#include "aesspmm/io.hpp"
#include "aesspmm/matrix.hpp"
#include "aesspmm/quantize.hpp"
#include "aesspmm/sampling.hpp"
#include "aesspmm/spmm.hpp"

using namespace aes;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

CsrMatrix make_csr(std::uint64_t n_rows, std::uint64_t n_cols,
                   const std::uint64_t* row_ptr, const std::uint32_t* col,
                   const float* val) {
    CsrMatrix m(n_rows, n_cols);
    m.row_ptr.assign(row_ptr, row_ptr + n_rows + 1);
    std::uint64_t nnz = row_ptr[n_rows];
    m.col_ind.assign(col, col + nnz);
    m.val.assign(val, val + nnz);
    return m;
}

DenseMatrix make_dense(std::uint64_t r, std::uint64_t c, const float* x) {
    DenseMatrix d(r, c);
    if (r * c) std::memcpy(d.data.data(), x, r * c * sizeof(float));
    return d;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- CSR handles ---------------------------------------------------------
void* ref_csr_new(std::uint64_t n_rows, std::uint64_t n_cols,
                  const std::uint64_t* row_ptr, const std::uint32_t* col,
                  const float* val) {
    return new CsrMatrix(make_csr(n_rows, n_cols, row_ptr, col, val));
}
void ref_csr_free(void* h) { delete static_cast<CsrMatrix*>(h); }
std::uint64_t ref_csr_rows(void* h) { return static_cast<CsrMatrix*>(h)->n_rows; }
std::uint64_t ref_csr_nnz(void* h) { return static_cast<CsrMatrix*>(h)->nnz(); }
void ref_csr_copy(void* h, std::uint64_t* row_ptr, std::uint32_t* col, float* val) {
    auto* m = static_cast<CsrMatrix*>(h);
    std::copy(m->row_ptr.begin(), m->row_ptr.end(), row_ptr);
    std::copy(m->col_ind.begin(), m->col_ind.end(), col);
    std::copy(m->val.begin(), m->val.end(), val);
}

// reference gen_synthetic (proj/src/bench.cpp:161-202), power-law model
void* ref_gen_synthetic(std::uint64_t n, double alpha, std::uint32_t max_degree,
                        std::uint64_t seed) {
    void* out = nullptr;
    guard([&] {
        SyntheticParams p;
        p.model = DegreeModel::PowerLaw;
        p.alpha = alpha;
        p.max_degree = max_degree;
        p.seed = seed;
        out = new CsrMatrix(gen_synthetic(n, p));
    });
    return out;
}

// reference gcn_normalize (proj/src/matrix.cpp:130-144)
void* ref_gcn_normalize(void* h, int add_self_loops) {
    void* out = nullptr;
    guard([&] {
        out = new CsrMatrix(gcn_normalize(*static_cast<CsrMatrix*>(h), add_self_loops != 0));
    });
    return out;
}

// reference row_mean_normalize (proj/src/matrix.cpp:146-158)
void* ref_row_mean_normalize(void* h) {
    void* out = nullptr;
    guard([&] { out = new CsrMatrix(row_mean_normalize(*static_cast<CsrMatrix*>(h))); });
    return out;
}

// reference evaluate (proj/src/gnn.cpp:118-155); ref_logits / mask may be null
int ref_evaluate(const float* logits, std::uint64_t rows, std::uint64_t cols, const std::uint32_t* labels,
                 const float* ref_logits, const std::uint8_t* mask, double* acc, double* agree,
                 std::uint64_t* per_class) {
    return guard([&] {
        DenseMatrix l = make_dense(rows, cols, logits);
        std::vector<std::uint32_t> lab(labels, labels + rows);
        std::vector<std::uint8_t> m;
        if (mask) m.assign(mask, mask + rows);
        DenseMatrix r;
        if (ref_logits) r = make_dense(rows, cols, ref_logits);
        EvalResult e = evaluate(l, lab, ref_logits ? &r : nullptr, m);
        *acc = e.accuracy;
        *agree = e.agreement;
        std::copy(e.per_class.begin(), e.per_class.end(), per_class);
    });
}

// ---- binary I/O (proj/src/io.cpp) -------------------------------------------
int ref_save_csr_binary(void* h, const char* path) {
    return guard([&] { save_csr_binary(*static_cast<CsrMatrix*>(h), path); });
}
void* ref_load_csr_binary(const char* path) {
    void* out = nullptr;
    guard([&] { out = new CsrMatrix(load_csr_binary(path)); });
    return out;
}
int ref_save_fmat_f32(const float* x, std::uint64_t r, std::uint64_t c, const char* path) {
    return guard([&] { save_fmat(make_dense(r, c, x), path); });
}
int ref_save_fmat_q8(const std::uint16_t* codes, std::uint64_t r, std::uint64_t c, float lo, float hi,
                     const char* path) {
    return guard([&] {
        QuantizedFeatures q;
        q.n_rows = r;
        q.n_cols = c;
        q.codes.assign(codes, codes + r * c);
        q.params = QuantParams{lo, hi, 8};
        save_fmat(q, path);
    });
}
// dtype 0 -> x (r*c floats), dtype 1 -> codes + lo/hi
int ref_load_fmat(const char* path, int* dtype, std::uint64_t* r, std::uint64_t* c, float* lo, float* hi, float* x,
                  std::uint16_t* codes) {
    return guard([&] {
        Features f = load_features(path);
        if (std::holds_alternative<DenseMatrix>(f)) {
            const DenseMatrix& m = std::get<DenseMatrix>(f);
            *dtype = 0;
            *r = m.n_rows;
            *c = m.n_cols;
            if (x) std::copy(m.data.begin(), m.data.end(), x);
        } else {
            const QuantizedFeatures& q = std::get<QuantizedFeatures>(f);
            *dtype = 1;
            *r = q.n_rows;
            *c = q.n_cols;
            *lo = q.params.x_min;
            *hi = q.params.x_max;
            if (codes) std::copy(q.codes.begin(), q.codes.end(), codes);
        }
    });
}

// ---- sampling (proj/src/sampling.cpp) ---------------------------------------
// Flattened plan set: per-row (chunk, cnt), starts_ptr (n+1), starts.
int ref_build_plans(void* h, std::uint32_t width, int strategy,
                    std::uint32_t* chunk, std::uint32_t* cnt,
                    std::uint64_t* starts_ptr, std::uint32_t* starts,
                    std::uint64_t starts_cap) {
    return guard([&] {
        SamplePlanSet ps = build_plan_set(*static_cast<CsrMatrix*>(h), width,
                                          static_cast<Strategy>(strategy));
        std::uint64_t k = 0;
        starts_ptr[0] = 0;
        for (std::size_t i = 0; i < ps.plans.size(); ++i) {
            chunk[i] = ps.plans[i].params.chunk_len;
            cnt[i] = ps.plans[i].params.sample_cnt;
            for (std::uint32_t s : ps.plans[i].starts) {
                if (starts != nullptr && k < starts_cap) starts[k] = s;
                ++k;
            }
            starts_ptr[i + 1] = k;
        }
    });
}

int ref_sampling_rate(void* h, std::uint32_t width, int strategy, double* aggregate,
                      double* unique) {
    return guard([&] {
        const CsrMatrix& m = *static_cast<CsrMatrix*>(h);
        SamplePlanSet ps = build_plan_set(m, width, static_cast<Strategy>(strategy));
        SamplingRates r = sampling_rate(ps, row_stats(m));
        *aggregate = r.aggregate;
        *unique = r.unique_coverage;
    });
}

int ref_sampling_rate_per_row(void* h, std::uint32_t width, int strategy, double* per_row) {
    return guard([&] {
        const CsrMatrix& m = *static_cast<CsrMatrix*>(h);
        SamplePlanSet ps = build_plan_set(m, width, static_cast<Strategy>(strategy));
        SamplingRates r = sampling_rate(ps, row_stats(m));
        std::copy(r.per_row.begin(), r.per_row.end(), per_row);
    });
}

// ---- cdf_stats (proj/src/bench.cpp:124-138) ----------------------------------
int ref_cdf_stats(const double* rates, std::uint64_t n, double* out_rate, double* out_frac,
                  std::uint64_t* n_steps) {
    return guard([&] {
        auto cdf = cdf_stats(std::vector<double>(rates, rates + n));
        for (std::size_t i = 0; i < cdf.size(); ++i) {
            out_rate[i] = cdf[i].first;
            out_frac[i] = cdf[i].second;
        }
        *n_steps = cdf.size();
    });
}

// ---- SpMM (proj/src/spmm.cpp) -----------------------------------------------
int ref_spmm_sampled(void* h, const float* b, std::uint64_t b_rows, std::uint64_t f,
                     std::uint32_t width, int strategy, unsigned threads, float* c) {
    return guard([&] {
        const CsrMatrix& m = *static_cast<CsrMatrix*>(h);
        SamplePlanSet ps = build_plan_set(m, width, static_cast<Strategy>(strategy));
        DenseMatrix out = spmm_sampled(m, make_dense(b_rows, f, b), ps, threads);
        std::copy(out.data.begin(), out.data.end(), c);
    });
}

int ref_spmm_exact(void* h, const float* b, std::uint64_t b_rows, std::uint64_t f,
                   unsigned threads, float* c) {
    return guard([&] {
        const CsrMatrix& m = *static_cast<CsrMatrix*>(h);
        DenseMatrix out = spmm_exact(m, make_dense(b_rows, f, b), threads);
        std::copy(out.data.begin(), out.data.end(), c);
    });
}

// Kernel-only timing of spmm_sampled with prebuilt plans, as in
// proj/src/bench.cpp:59-77.  plan_ms is the build_plan_set time; ms[r] holds
// each of `reps` kernel times.  `c` (optional) receives the last output.
int ref_time_spmm_sampled(void* h, const float* b, std::uint64_t b_rows,
                          std::uint64_t f, std::uint32_t width, int strategy,
                          unsigned threads, int reps, double* plan_ms, double* ms,
                          float* c) {
    return guard([&] {
        using Clock = std::chrono::steady_clock;
        const CsrMatrix& m = *static_cast<CsrMatrix*>(h);
        DenseMatrix bd = make_dense(b_rows, f, b);
        auto t0 = Clock::now();
        SamplePlanSet ps = build_plan_set(m, width, static_cast<Strategy>(strategy));
        *plan_ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        DenseMatrix out;
        for (int r = 0; r < reps; ++r) {
            auto t1 = Clock::now();
            out = spmm_sampled(m, bd, ps, threads);
            ms[r] = std::chrono::duration<double, std::milli>(Clock::now() - t1).count();
        }
        if (c != nullptr) std::copy(out.data.begin(), out.data.end(), c);
    });
}

// ---- quantization (proj/src/quantize.cpp) -------------------------------------
int ref_fit_params(const float* x, std::uint64_t r, std::uint64_t c, std::uint32_t bits,
                   float* lo, float* hi) {
    return guard([&] {
        QuantParams p = fit_params(make_dense(r, c, x), bits);
        *lo = p.x_min;
        *hi = p.x_max;
    });
}

int ref_quantize(const float* x, std::uint64_t r, std::uint64_t c, float lo, float hi,
                 std::uint32_t bits, std::uint16_t* codes) {
    return guard([&] {
        QuantizedFeatures q = quantize(make_dense(r, c, x), QuantParams{lo, hi, bits});
        std::copy(q.codes.begin(), q.codes.end(), codes);
    });
}

int ref_dequantize(const std::uint16_t* codes, std::uint64_t r, std::uint64_t c,
                   float lo, float hi, std::uint32_t bits, float* x) {
    return guard([&] {
        QuantizedFeatures q;
        q.n_rows = r;
        q.n_cols = c;
        q.codes.assign(codes, codes + r * c);
        q.params = QuantParams{lo, hi, bits};
        DenseMatrix d = dequantize(q);
        std::copy(d.data.begin(), d.data.end(), x);
    });
}

// ---- GNN (proj/src/gnn.cpp) -------------------------------------------------
int ref_dense_matmul(const float* a, std::uint64_t m, std::uint64_t k, const float* b,
                     std::uint64_t n, float* c) {
    return guard([&] {
        DenseMatrix out = dense_matmul(make_dense(m, k, a), make_dense(k, n, b));
        std::copy(out.data.begin(), out.data.end(), c);
    });
}

// GCN forward: dims[0..n_layers] feature widths; weights/biases concatenated
// row-major per layer.  width==0 -> exact (plans=nullptr) path.
int ref_gnn_forward(int kind, void* h, const float* x, const std::uint64_t* dims, int n_layers,
                    const float* weights, const float* biases, std::uint32_t width,
                    int strategy, float* out) {
    return guard([&] {
        const CsrMatrix& adj = *static_cast<CsrMatrix*>(h);
        GnnModel model;
        model.kind = kind ? ModelKind::SageMean : ModelKind::Gcn;
        const std::uint64_t mult = kind ? 2 : 1;
        std::uint64_t woff = 0, boff = 0;
        for (int l = 0; l < n_layers; ++l) {
            GnnLayer layer;
            layer.weight = make_dense(mult * dims[l], dims[l + 1], weights + woff);
            layer.bias.assign(biases + boff, biases + boff + dims[l + 1]);
            woff += mult * dims[l] * dims[l + 1];
            boff += dims[l + 1];
            model.layers.push_back(std::move(layer));
        }
        DenseMatrix feats = make_dense(adj.n_rows, dims[0], x);
        DenseMatrix res;
        if (width == 0) {
            res = gnn_forward(adj, feats, model, nullptr);
        } else {
            SamplePlanSet ps = build_plan_set(adj, width, static_cast<Strategy>(strategy));
            res = gnn_forward(adj, feats, model, &ps);
        }
        std::copy(res.data.begin(), res.data.end(), out);
    });
}

int ref_gcn_forward(void* h, const float* x, const std::uint64_t* dims, int n_layers, const float* weights,
                    const float* biases, std::uint32_t width, int strategy, float* out) {
    return ref_gnn_forward(0, h, x, dims, n_layers, weights, biases, width, strategy, out);
}

}  // extern "C"
