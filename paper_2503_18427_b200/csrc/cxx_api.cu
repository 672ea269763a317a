// C++ operator API (include/aesspmm/b200.hpp) — the reference's aes:: API
// (proj/include/aesspmm/*.hpp) implemented over the C ABI.  Each call
// uploads its host operands, runs the sm_100a kernels and copies the result
// back; errors become std::invalid_argument / std::runtime_error with the
// reference's messages.  No arithmetic happens on the host.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "aesspmm/b200.hpp"
#include "aesspmm_cuda.h"

namespace aes {
namespace {

[[noreturn]] void throw_status(int s) {
    const char* msg = aes_last_error();
    if (s == AES_ERR_CUDA || s == AES_ERR_UNSUPPORTED) throw std::runtime_error(msg);
    throw std::invalid_argument(msg);
}
inline void check(int s) {
    if (s != AES_OK) throw_status(s);
}

struct Csr {
    aes_csr_t h = nullptr;
    Csr() = default;
    Csr(const Csr&) = delete;
    ~Csr() { aes_csr_destroy(h); }
};

struct Plan {
    aes_plan_t h = nullptr;
    Plan() = default;
    Plan(const Plan&) = delete;
    ~Plan() { aes_plan_destroy(h); }
};

struct QFeat {
    aes_qfeat_t h = nullptr;
    QFeat() = default;
    QFeat(const QFeat&) = delete;
    ~QFeat() { aes_qfeat_destroy(h); }
};

// FNV-1a over the host plan vectors + width + strategy.  The reference
// always executes `plans.plans`; a caller may edit them (or width/strategy)
// after build_plan_set, so the cached device plan is used only while this
// fingerprint still matches.
std::uint64_t plan_fingerprint(const SamplePlanSet& ps) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&h](std::uint64_t v) {
        for (int i = 0; i < 8; ++i, v >>= 8) h = (h ^ (v & 0xff)) * 1099511628211ull;
    };
    mix(ps.width);
    mix(static_cast<std::uint64_t>(ps.strategy));
    mix(ps.plans.size());
    for (const RowSamplePlan& p : ps.plans) {
        mix((std::uint64_t)p.params.chunk_len << 32 | p.params.sample_cnt);
        mix(p.starts.size());
        for (std::uint32_t st : p.starts) mix(st);
    }
    return h;
}

// The device plan a SamplePlanSet carries; keeps its source CSR alive.
struct DevicePlan {
    std::shared_ptr<Csr> src;
    Plan plan;
    std::uint64_t fingerprint = 0;  // of the host plans it was exported as
};

// The cached device plan of `ps`, or null when the host plans were edited.
aes_plan_t cached_plan(const SamplePlanSet& ps) {
    if (!ps.device) return nullptr;
    auto* dp = static_cast<DevicePlan*>(ps.device.get());
    return plan_fingerprint(ps) == dp->fingerprint ? dp->plan.h : nullptr;
}

std::shared_ptr<Csr> upload(const CsrMatrix& m) {
    auto c = std::make_shared<Csr>();
    check(aes_csr_create(m.n_rows, m.n_cols, m.row_ptr.data(), m.row_ptr.size(), m.col_ind.data(), m.val.data(),
                         m.col_ind.size(), &c->h));
    return c;
}

void flatten(const SamplePlanSet& ps, std::vector<std::uint32_t>& chunk, std::vector<std::uint32_t>& cnt,
             std::vector<std::uint64_t>& sp, std::vector<std::uint32_t>& starts) {
    const std::size_t n = ps.plans.size();
    chunk.resize(n);
    cnt.resize(n);
    sp.assign(n + 1, 0);
    for (std::size_t i = 0; i < n; ++i) {
        chunk[i] = ps.plans[i].params.chunk_len;
        cnt[i] = ps.plans[i].params.sample_cnt;
        sp[i + 1] = sp[i] + ps.plans[i].starts.size();
    }
    starts.resize(sp[n]);
    for (std::size_t i = 0; i < n; ++i)
        std::copy(ps.plans[i].starts.begin(), ps.plans[i].starts.end(), starts.begin() + sp[i]);
}

// A device plan usable with device matrix `a`: the one build_plan_set made
// (re-filled from `a` inside the C ABI when `a` is another upload), or one
// built from the host plan vectors.
aes_plan_t plan_for(const SamplePlanSet& ps, const Csr& a, Plan& scratch) {
    if (aes_plan_t cached = cached_plan(ps)) return cached;
    std::vector<std::uint32_t> chunk, cnt, starts;
    std::vector<std::uint64_t> sp;
    flatten(ps, chunk, cnt, sp, starts);
    check(aes_plan_from_host(a.h, ps.width, static_cast<int>(ps.strategy), chunk.data(), cnt.data(), sp.data(),
                             starts.data(), &scratch.h));
    return scratch.h;
}

DenseMatrix spmm_sampled_impl(const CsrMatrix& a, const DenseMatrix& b, const SamplePlanSet& plans,
                              WorkCounter* counter) {
    if (a.n_cols != b.n_rows) throw std::invalid_argument("ShapeMismatch");          // spmm.cpp:13
    if (plans.plans.size() != a.n_rows) throw std::invalid_argument("PlanMatrixMismatch");  // spmm.cpp:44-46
    auto da = upload(a);
    Plan scratch;
    aes_plan_t p = plan_for(plans, *da, scratch);
    DenseMatrix c(a.n_rows, b.n_cols);
    std::uint64_t fma = 0, la = 0, lb = 0;
    check(aes_spmm_sampled(da->h, b.data.data(), b.n_rows, b.n_cols, p, c.data.data(), &fma, &la, &lb));
    if (counter) *counter = WorkCounter{fma, la, lb};
    return c;
}

}  // namespace

// ---------------------------------------------------------------- matrix
std::string ValidationResult::message() const {
    switch (error) {
        case CsrError::Ok: return "ok";
        case CsrError::NonMonotonicRowPtr: return "NonMonotonicRowPtr at row " + std::to_string(row);
        case CsrError::ColumnOutOfRange: return "ColumnOutOfRange at row " + std::to_string(row);
        case CsrError::UnsortedRow: return "UnsortedRow at row " + std::to_string(row);
        case CsrError::LengthMismatch: return "LengthMismatch";
        case CsrError::NotSquare: return "NotSquare";
    }
    return "unknown";
}

ValidationResult validate_csr(const CsrMatrix& m) {
    if (m.row_ptr.empty() || m.col_ind.size() != m.val.size()) return {CsrError::LengthMismatch, 0};
    int err = 0;
    std::uint64_t row = 0;
    int s = aes_validate_csr(m.n_rows, m.n_cols, m.row_ptr.data(), m.row_ptr.size(), m.col_ind.data(),
                             m.col_ind.size(), &err, &row);
    if (s != AES_OK && s != AES_ERR_CSR_INVALID) throw_status(s);
    return {static_cast<CsrError>(err), static_cast<std::size_t>(row)};
}

RowStats row_stats(const CsrMatrix& m) {
    Csr c;
    check(aes_csr_structure(m.n_rows, m.n_cols, m.row_ptr.data(), &c.h));
    RowStats s;
    s.row_nnz.resize(m.n_rows);
    check(aes_csr_row_stats(c.h, s.row_nnz.data(), &s.max_row_nnz, &s.avg_degree));
    s.avg_degree = m.n_rows == 0 ? 0.0 : double(m.nnz()) / double(m.n_rows);
    return s;
}

CsrMatrix gcn_normalize(const CsrMatrix& a, bool add_self_loops) {
    if (a.n_rows != a.n_cols) throw std::invalid_argument("NotSquare");
    auto da = upload(a);
    Csr out;
    check(aes_gcn_normalize(da->h, add_self_loops ? 1 : 0, &out.h));
    std::uint64_t r = 0, c = 0, nnz = 0;
    check(aes_csr_shape(out.h, &r, &c, &nnz));
    CsrMatrix m(r, c);
    m.col_ind.resize(nnz);
    m.val.resize(nnz);
    check(aes_csr_download(out.h, m.row_ptr.data(), m.col_ind.data(), m.val.data()));
    return m;
}

// -------------------------------------------------------------- sampling
Strategy strategy_from_string(const std::string& s) {
    if (s == "adaptive") return Strategy::Adaptive;
    if (s == "afs") return Strategy::Afs;
    if (s == "sfs") return Strategy::Sfs;
    if (s == "full") return Strategy::Full;
    throw std::invalid_argument("unknown strategy: " + s);
}

std::string to_string(Strategy s) {
    static const char* names[] = {"adaptive", "afs", "sfs", "full"};
    int i = static_cast<int>(s);
    return (i >= 0 && i < 4) ? names[i] : "?";
}

StrategyParams select_strategy(std::uint64_t row_nnz, std::uint32_t width) {
    StrategyParams p;
    check(aes_select_strategy(row_nnz, width, &p.chunk_len, &p.sample_cnt));
    return p;
}

std::uint32_t hash_start(std::uint32_t current_ind, std::uint64_t row_nnz, std::uint32_t chunk_len) {
    return aes_hash_start(current_ind, row_nnz, chunk_len);
}

RowSamplePlan build_plan(std::uint32_t row_id, std::uint64_t row_nnz, std::uint32_t width, Strategy strategy) {
    if (width == 0) throw std::invalid_argument("ZeroWidth");
    // a one-row plan set through the same device sampler as build_plan_set
    std::vector<std::uint64_t> rp{0, row_nnz};
    Csr c;
    check(aes_csr_structure(1, 0, rp.data(), &c.h));
    Plan p;
    check(aes_build_plan_set(c.h, width, static_cast<int>(strategy), &p.h));
    std::uint64_t tot = 0;
    check(aes_plan_info(p.h, nullptr, nullptr, nullptr, nullptr, &tot));
    RowSamplePlan out;
    out.row_id = row_id;
    std::uint64_t sp[2];
    out.starts.resize(tot);
    check(aes_plan_export(p.h, &out.params.chunk_len, &out.params.sample_cnt, sp, out.starts.data()));
    return out;
}

SamplePlanSet build_plan_set(const CsrMatrix& m, std::uint32_t width, Strategy strategy) {
    if (width == 0) throw std::invalid_argument("ZeroWidth");
    auto dp = std::make_shared<DevicePlan>();
    dp->src = upload(m);
    check(aes_build_plan_set(dp->src->h, width, static_cast<int>(strategy), &dp->plan.h));
    std::uint64_t n = 0, tot = 0;
    check(aes_plan_info(dp->plan.h, nullptr, nullptr, &n, nullptr, &tot));
    std::vector<std::uint32_t> chunk(n), cnt(n), starts(tot);
    std::vector<std::uint64_t> sp(n + 1);
    check(aes_plan_export(dp->plan.h, chunk.data(), cnt.data(), sp.data(), starts.data()));
    SamplePlanSet set;
    set.width = width;
    set.strategy = strategy;
    set.plans.resize(n);
    for (std::uint64_t i = 0; i < n; ++i) {
        RowSamplePlan& p = set.plans[i];
        p.row_id = static_cast<std::uint32_t>(i);
        p.params = {chunk[i], cnt[i]};
        p.starts.assign(starts.begin() + sp[i], starts.begin() + sp[i + 1]);
    }
    dp->fingerprint = plan_fingerprint(set);
    set.device = std::static_pointer_cast<void>(dp);
    return set;
}

SamplingRates sampling_rate(const SamplePlanSet& plans, const RowStats& stats) {
    if (plans.plans.size() != stats.row_nnz.size()) throw std::invalid_argument("plan/stats row count mismatch");
    const std::size_t n = stats.row_nnz.size();
    std::vector<std::uint64_t> rp(n + 1, 0);
    for (std::size_t i = 0; i < n; ++i) rp[i + 1] = rp[i] + stats.row_nnz[i];  // offsets of the given stats
    Csr c;
    check(aes_csr_structure(n, 0, rp.data(), &c.h));
    Plan scratch;
    aes_plan_t p = cached_plan(plans);
    if (!p) {
        std::vector<std::uint32_t> chunk, cnt, starts;
        std::vector<std::uint64_t> sp;
        flatten(plans, chunk, cnt, sp, starts);
        check(aes_plan_from_host(c.h, plans.width, static_cast<int>(plans.strategy), chunk.data(), cnt.data(),
                                 sp.data(), starts.data(), &scratch.h));
        p = scratch.h;
    }
    SamplingRates r;
    r.per_row.resize(n);
    check(aes_sampling_rate(p, c.h, &r.aggregate, &r.unique_coverage, r.per_row.data()));
    return r;
}

// ----------------------------------------------------------------- bench
std::vector<std::pair<double, double>> cdf_stats(std::vector<double> rates) {
    if (rates.empty()) throw std::invalid_argument("rates must be nonempty");  // bench.cpp:125
    std::vector<double> r(rates.size()), f(rates.size());
    std::uint64_t steps = 0;
    check(aes_cdf_stats(rates.data(), rates.size(), r.data(), f.data(), &steps));
    std::vector<std::pair<double, double>> cdf(steps);
    for (std::uint64_t i = 0; i < steps; ++i) cdf[i] = {r[i], f[i]};
    return cdf;
}

// ------------------------------------------------------------------ spmm
DenseMatrix spmm_exact(const CsrMatrix& a, const DenseMatrix& b, unsigned) {
    if (a.n_cols != b.n_rows) throw std::invalid_argument("ShapeMismatch");
    auto da = upload(a);
    DenseMatrix c(a.n_rows, b.n_cols);
    check(aes_spmm_exact(da->h, b.data.data(), b.n_rows, b.n_cols, c.data.data()));
    return c;
}

DenseMatrix spmm_sampled(const CsrMatrix& a, const DenseMatrix& b, const SamplePlanSet& plans, unsigned) {
    return spmm_sampled_impl(a, b, plans, nullptr);
}

DenseMatrix spmm_sampled_instrumented(const CsrMatrix& a, const DenseMatrix& b, const SamplePlanSet& plans,
                                      WorkCounter& counter, unsigned) {
    return spmm_sampled_impl(a, b, plans, &counter);
}

WorkCounter exact_work(const CsrMatrix& a, const DenseMatrix& b) {
    WorkCounter w;
    w.fma_count = std::uint64_t(a.nnz()) * b.n_cols;
    w.loads_a = a.nnz();
    w.loads_b = w.fma_count;
    return w;
}

// -------------------------------------------------------------- quantize
QuantParams fit_params(const DenseMatrix& x, std::uint32_t bits) {
    QuantParams p;
    check(aes_fit_params(x.data.data(), x.n_rows, x.n_cols, bits, &p.x_min, &p.x_max));
    p.bits = bits;
    return p;
}

QuantizedFeatures quantize(const DenseMatrix& x, const QuantParams& p) {
    QFeat q;
    check(aes_quantize_with(x.data.data(), x.n_rows, x.n_cols, p.x_min, p.x_max, p.bits, &q.h));
    QuantizedFeatures qf;
    qf.n_rows = x.n_rows;
    qf.n_cols = x.n_cols;
    qf.params = p;
    qf.codes.resize(x.data.size());
    check(aes_qfeat_codes(q.h, qf.codes.data()));
    return qf;
}

DenseMatrix dequantize(const QuantizedFeatures& qf) {
    QFeat q;
    check(aes_qfeat_from_codes(qf.codes.data(), qf.n_rows, qf.n_cols, qf.params.x_min, qf.params.x_max,
                               qf.params.bits, &q.h));
    DenseMatrix x(qf.n_rows, qf.n_cols);
    check(aes_dequantize(q.h, x.data.data()));
    return x;
}

DenseMatrix spmm_sampled_q8(const CsrMatrix& a, const QuantizedFeatures& qf, const SamplePlanSet* plans) {
    if (a.n_cols != qf.n_rows) throw std::invalid_argument("ShapeMismatch");
    if (plans && plans->plans.size() != a.n_rows) throw std::invalid_argument("PlanMatrixMismatch");
    auto da = upload(a);
    QFeat q;
    check(aes_qfeat_from_codes(qf.codes.data(), qf.n_rows, qf.n_cols, qf.params.x_min, qf.params.x_max,
                               qf.params.bits, &q.h));
    Plan scratch;
    aes_plan_t p = plans ? plan_for(*plans, *da, scratch) : nullptr;
    DenseMatrix c(a.n_rows, qf.n_cols);
    check(aes_spmm_sampled_q8(da->h, q.h, p, c.data.data()));
    return c;
}

// ------------------------------------------------------------------- gnn
DenseMatrix dense_matmul(const DenseMatrix& a, const DenseMatrix& b, unsigned) {
    if (a.n_cols != b.n_rows) throw std::invalid_argument("ShapeMismatch");
    DenseMatrix c(a.n_rows, b.n_cols);
    check(aes_dense_matmul(a.data.data(), a.n_rows, a.n_cols, b.data.data(), b.n_cols, c.data.data()));
    return c;
}

namespace {
DenseMatrix forward_impl(bool sage, const CsrMatrix& adj, const DenseMatrix& features, const GnnModel& model,
                         const SamplePlanSet* plans) {
    if (adj.n_cols != features.n_rows) throw std::invalid_argument("ShapeMismatch");
    if (plans && plans->plans.size() != adj.n_rows) throw std::invalid_argument("PlanMatrixMismatch");
    std::vector<std::uint64_t> dims{features.n_cols}, blen;
    std::vector<float> w, bias;
    for (const GnnLayer& l : model.layers) {
        if (l.weight.n_rows != (sage ? 2 : 1) * dims.back()) throw std::invalid_argument("ShapeMismatch");
        if (!l.bias.empty() && l.bias.size() != l.weight.n_cols) throw std::invalid_argument("ShapeMismatch");
        dims.push_back(l.weight.n_cols);
        w.insert(w.end(), l.weight.data.begin(), l.weight.data.end());
        bias.insert(bias.end(), l.bias.begin(), l.bias.end());
        blen.push_back(l.bias.size());
    }
    if (model.layers.empty()) return features;
    auto da = upload(adj);
    Plan scratch;
    aes_plan_t p = plans ? plan_for(*plans, *da, scratch) : nullptr;
    DenseMatrix out(adj.n_rows, dims.back());
    auto fn = sage ? aes_sage_forward : aes_gcn_forward;
    check(fn(da->h, features.data.data(), dims.data(), static_cast<int>(model.layers.size()), w.data(),
             bias.empty() ? nullptr : bias.data(), blen.data(), p, out.data.data()));
    return out;
}
}  // namespace

DenseMatrix gcn_forward(const CsrMatrix& adj, const DenseMatrix& features, const GnnModel& model,
                        const SamplePlanSet* plans, unsigned) {
    if (model.kind != ModelKind::Gcn) throw std::invalid_argument("not a GCN model");
    return forward_impl(false, adj, features, model, plans);
}

DenseMatrix sage_forward(const CsrMatrix& adj_mean, const DenseMatrix& features, const GnnModel& model,
                         const SamplePlanSet* plans, unsigned) {
    if (model.kind != ModelKind::SageMean) throw std::invalid_argument("not a SAGE model");
    return forward_impl(true, adj_mean, features, model, plans);
}

DenseMatrix gnn_forward(const CsrMatrix& adj, const DenseMatrix& features, const GnnModel& model,
                        const SamplePlanSet* plans, unsigned n_threads) {
    return model.kind == ModelKind::Gcn ? gcn_forward(adj, features, model, plans, n_threads)
                                        : sage_forward(adj, features, model, plans, n_threads);
}

std::vector<std::uint32_t> argmax_rows(const DenseMatrix& logits) {
    std::vector<std::uint32_t> out(logits.n_rows);
    check(aes_argmax_rows(logits.data.data(), logits.n_rows, logits.n_cols, out.data()));
    return out;
}

EvalResult evaluate(const DenseMatrix& logits, const std::vector<std::uint32_t>& labels,
                    const DenseMatrix* reference_logits, const std::vector<std::uint8_t>& mask) {
    if (labels.size() != logits.n_rows) throw std::invalid_argument("labels length != n_nodes");
    if (reference_logits && reference_logits->n_rows != logits.n_rows)
        throw std::invalid_argument("reference shape mismatch");
    EvalResult r;
    r.per_class.assign(logits.n_cols, 0);
    int s = aes_evaluate(logits.data.data(), logits.n_rows, logits.n_cols, labels.data(), labels.size(),
                         reference_logits ? reference_logits->data.data() : nullptr,
                         mask.empty() ? nullptr : mask.data(), mask.size(), &r.accuracy, &r.agreement,
                         reinterpret_cast<std::uint64_t*>(r.per_class.data()));
    if (s != AES_OK) {
        if (std::string(aes_last_error()) == "LabelOutOfRange") throw std::out_of_range("LabelOutOfRange");
        throw_status(s);
    }
    return r;
}

CsrMatrix row_mean_normalize(const CsrMatrix& a) {
    if (a.n_rows != a.n_cols) throw std::invalid_argument("NotSquare");
    auto da = upload(a);
    Csr out;
    check(aes_row_mean_normalize(da->h, &out.h));
    CsrMatrix m(a.n_rows, a.n_cols);
    m.col_ind.resize(a.nnz());
    m.val.resize(a.nnz());
    check(aes_csr_download(out.h, m.row_ptr.data(), m.col_ind.data(), m.val.data()));
    return m;
}

}  // namespace aes
