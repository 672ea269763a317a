// `_core`: the reference's Python API (proj/bindings/module.cpp:52-144) with
// the same names, argument meaning and exception types, backed by the C ABI of
// libaescuda.so (include/aesspmm_cuda.h).  Objects live in HBM; numpy arrays
// are copied in and out exactly where the reference copies (module.cpp:35-48).
// The GIL is released around every device call.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "aesspmm_cuda.h"

namespace py = pybind11;

namespace {

[[noreturn]] void raise(int status) {
    std::string msg = aes_last_error();
    switch (status) {
        case AES_ERR_CUDA:
        case AES_ERR_UNSUPPORTED:
        case AES_ERR_IO:  // std::runtime_error in the reference's io.cpp
            throw std::runtime_error(msg);
        default:
            throw py::value_error(msg);  // std::invalid_argument -> ValueError
    }
}

inline void check(int s) {
    if (s != AES_OK) raise(s);
}

template <class F>
int nogil(F&& f) {
    py::gil_scoped_release rel;
    return f();
}

enum class Strategy { Adaptive = AES_ADAPTIVE, Afs = AES_AFS, Sfs = AES_SFS, Full = AES_FULL };

struct Csr {
    aes_csr_t h = nullptr;
    uint64_t n_rows = 0, n_cols = 0, nnz = 0;
    explicit Csr(aes_csr_t handle) : h(handle) { aes_csr_shape(h, &n_rows, &n_cols, &nnz); }
    ~Csr() { aes_csr_destroy(h); }
};
using CsrP = std::shared_ptr<Csr>;

struct StrategyParams {
    uint32_t chunk_len = 0, sample_cnt = 0;
};

struct RowSamplePlan {
    uint32_t row_id = 0;
    StrategyParams params;
    std::vector<uint32_t> starts;
    uint64_t slots() const { return uint64_t(params.chunk_len) * params.sample_cnt; }
};

struct PlanSet {
    aes_plan_t h = nullptr;
    CsrP src;
    uint32_t width = 0;
    Strategy strategy = Strategy::Full;
    uint64_t total_slots = 0;
    mutable std::optional<std::vector<RowSamplePlan>> plans;
    ~PlanSet() { aes_plan_destroy(h); }

    const std::vector<RowSamplePlan>& materialize() const {
        if (plans) return *plans;
        uint64_t n = 0, tot_starts = 0;
        check(aes_plan_info(h, nullptr, nullptr, &n, nullptr, &tot_starts));
        std::vector<uint32_t> chunk(n), cnt(n), starts(tot_starts);
        std::vector<uint64_t> sp(n + 1);
        check(nogil([&] { return aes_plan_export(h, chunk.data(), cnt.data(), sp.data(), starts.data()); }));
        std::vector<RowSamplePlan> out(n);
        for (uint64_t i = 0; i < n; ++i) {
            out[i].row_id = uint32_t(i);
            out[i].params = {chunk[i], cnt[i]};
            out[i].starts.assign(starts.begin() + sp[i], starts.begin() + sp[i + 1]);
        }
        plans = std::move(out);
        return *plans;
    }
};
using PlanP = std::shared_ptr<PlanSet>;

struct QuantParams {
    float x_min = 0.f, x_max = 0.f;
    uint32_t bits = 8;
};

struct QFeat {
    aes_qfeat_t h = nullptr;
    uint64_t n_rows = 0, n_cols = 0;
    QuantParams params;
    explicit QFeat(aes_qfeat_t handle) : h(handle) {
        aes_qfeat_info(h, &n_rows, &n_cols, &params.x_min, &params.x_max, &params.bits);
    }
    ~QFeat() { aes_qfeat_destroy(h); }
};
using QFeatP = std::shared_ptr<QFeat>;

using F32In = py::array_t<float, py::array::c_style | py::array::forcecast>;

F32In as_2d(F32In a) {
    if (a.ndim() != 2) throw py::value_error("expected a 2-d array");
    return a;
}

py::array_t<float> new_2d(uint64_t r, uint64_t c) {
    return py::array_t<float>({(py::ssize_t)r, (py::ssize_t)c});
}

CsrP csr_from_arrays(std::size_t n_rows, std::size_t n_cols, py::array_t<uint64_t, py::array::c_style | py::array::forcecast> row_ptr,
                     py::array_t<uint32_t, py::array::c_style | py::array::forcecast> col_ind,
                     py::array_t<float, py::array::c_style | py::array::forcecast> val) {
    // the reference copies then validates (module.cpp:17-33); sizes mismatch
    // between col_ind and val is LengthMismatch (matrix.cpp:30)
    if (col_ind.size() != val.size()) throw py::value_error("LengthMismatch");
    if (row_ptr.size() == 0) throw py::value_error("LengthMismatch");
    aes_csr_t h = nullptr;
    const uint64_t* rp = row_ptr.data();
    const uint32_t* ci = col_ind.data();
    const float* vv = val.data();
    uint64_t rpl = row_ptr.size(), nnz = col_ind.size();
    check(nogil([&] { return aes_csr_create(n_rows, n_cols, rp, rpl, ci, vv, nnz, &h); }));
    return std::make_shared<Csr>(h);
}

}  // namespace

PYBIND11_MODULE(_core, mod) {
    mod.doc() = "B200-native AES-SpMM core: CSR plans, sm_100a kernels, scalar quantization";

    py::class_<Csr, CsrP>(mod, "CsrMatrix")
        .def(py::init(&csr_from_arrays), py::arg("n_rows"), py::arg("n_cols"), py::arg("row_ptr"),
             py::arg("col_ind"), py::arg("val"))
        .def_readonly("n_rows", &Csr::n_rows)
        .def_readonly("n_cols", &Csr::n_cols)
        .def_property_readonly("nnz", [](const Csr& c) { return c.nnz; })
        .def("to_arrays",
             [](const Csr& c) {
                 py::array_t<uint64_t> rp(c.n_rows + 1);
                 py::array_t<uint32_t> ci(c.nnz);
                 py::array_t<float> vv(c.nnz);
                 uint64_t* prp = rp.mutable_data();
                 uint32_t* pci = ci.mutable_data();
                 float* pvv = vv.mutable_data();
                 check(nogil([&] { return aes_csr_download(c.h, prp, pci, pvv); }));
                 return py::make_tuple(rp, ci, vv);
             },
             "download (row_ptr, col_ind, val) from HBM")
        .def("device_ptrs",
             [](const Csr& c) {
                 const uint64_t* rp;
                 const uint32_t* ci;
                 const float* vv;
                 check(aes_csr_device_ptrs(c.h, &rp, &ci, &vv));
                 return py::make_tuple((uintptr_t)rp, (uintptr_t)ci, (uintptr_t)vv);
             });

    py::enum_<Strategy>(mod, "Strategy")
        .value("ADAPTIVE", Strategy::Adaptive)
        .value("AFS", Strategy::Afs)
        .value("SFS", Strategy::Sfs)
        .value("FULL", Strategy::Full);

    py::class_<StrategyParams>(mod, "StrategyParams")
        .def_readonly("chunk_len", &StrategyParams::chunk_len)
        .def_readonly("sample_cnt", &StrategyParams::sample_cnt)
        .def("__repr__", [](const StrategyParams& p) {
            return "StrategyParams(chunk_len=" + std::to_string(p.chunk_len) +
                   ", sample_cnt=" + std::to_string(p.sample_cnt) + ")";
        });

    py::class_<RowSamplePlan>(mod, "RowSamplePlan")
        .def_readonly("row_id", &RowSamplePlan::row_id)
        .def_readonly("params", &RowSamplePlan::params)
        .def_readonly("starts", &RowSamplePlan::starts)
        .def_property_readonly("slots", &RowSamplePlan::slots);

    py::class_<PlanSet, PlanP>(mod, "SamplePlanSet")
        .def_readonly("width", &PlanSet::width)
        .def_readonly("strategy", &PlanSet::strategy)
        .def_property_readonly("plans", [](const PlanSet& p) { return p.materialize(); })
        .def_readonly("total_slots", &PlanSet::total_slots)
        .def("sampled_csr",
             [](const PlanSet& p) {
                 py::array_t<uint64_t> sr(p.src->n_rows + 1);
                 py::array_t<uint32_t> sc(p.total_slots);
                 py::array_t<float> sv(p.total_slots);
                 uint64_t* psr = sr.mutable_data();
                 uint32_t* psc = sc.mutable_data();
                 float* psv = sv.mutable_data();
                 check(nogil([&] { return aes_plan_download(p.h, psr, psc, psv); }));
                 return py::make_tuple(sr, sc, sv);
             },
             "the sampled CSR (srow_ptr, scol, sval) in slot order, copied to host")
        .def("device_ptrs", [](const PlanSet& p) {
            const uint64_t* sr;
            const uint32_t* sc;
            const float* sv;
            check(aes_plan_device_ptrs(p.h, &sr, &sc, &sv));
            return py::make_tuple((uintptr_t)sr, (uintptr_t)sc, (uintptr_t)sv);
        });

    py::class_<QuantParams>(mod, "QuantParams")
        .def(py::init([](float lo, float hi, uint32_t bits) { return QuantParams{lo, hi, bits}; }),
             py::arg("x_min"), py::arg("x_max"), py::arg("bits") = 8)
        .def_readonly("x_min", &QuantParams::x_min)
        .def_readonly("x_max", &QuantParams::x_max)
        .def_readonly("bits", &QuantParams::bits);

    py::class_<QFeat, QFeatP>(mod, "QuantizedFeatures")
        .def_readonly("n_rows", &QFeat::n_rows)
        .def_readonly("n_cols", &QFeat::n_cols)
        .def_readonly("params", &QFeat::params)
        .def_property_readonly("codes", [](const QFeat& q) {
            py::array_t<uint16_t> a({(py::ssize_t)q.n_rows, (py::ssize_t)q.n_cols});
            uint16_t* p = a.mutable_data();
            check(nogil([&] { return aes_qfeat_codes(q.h, p); }));
            return a;
        })
        // fast mode (quantize_affine): "row" / "feature", None for the
        // reference's global min/max codes
        .def_property_readonly("affine_mode", [](const QFeat& q) -> py::object {
            int mode = -1;
            check(aes_qfeat_affine(q.h, &mode, nullptr));
            if (mode < 0) return py::none();
            return py::str(mode == AES_QAFFINE_ROW ? "row" : "feature");
        })
        .def_property_readonly("affine_params", [](const QFeat& q) -> py::object {
            int mode = -1;
            check(aes_qfeat_affine(q.h, &mode, nullptr));
            if (mode < 0) return py::none();
            const uint64_t np = mode == AES_QAFFINE_ROW ? q.n_rows : q.n_cols;
            py::array_t<float> a({(py::ssize_t)np, (py::ssize_t)2});
            float* p = a.mutable_data();
            check(nogil([&] { return aes_qfeat_affine(q.h, &mode, p); }));
            return a;
        });

    mod.def(
        "select_strategy",
        [](uint64_t row_nnz, uint32_t width) {
            StrategyParams p;
            check(aes_select_strategy(row_nnz, width, &p.chunk_len, &p.sample_cnt));
            return p;
        },
        py::arg("row_nnz"), py::arg("width"));
    mod.def(
        "hash_start",
        [](uint32_t current_ind, uint64_t row_nnz, uint32_t chunk_len) {
            if (row_nnz - uint64_t(chunk_len) + 1 == 0) throw py::value_error("hash range is zero");
            return aes_hash_start(current_ind, row_nnz, chunk_len);
        },
        py::arg("current_ind"), py::arg("row_nnz"), py::arg("chunk_len"));
    mod.def(
        "build_plan_set",
        [](CsrP m, uint32_t width, Strategy strategy) {
            aes_plan_t h = nullptr;
            check(nogil([&] { return aes_build_plan_set(m->h, width, int(strategy), &h); }));
            auto p = std::make_shared<PlanSet>();
            p->h = h;
            p->src = m;
            p->width = width;
            p->strategy = strategy;
            aes_plan_info(h, nullptr, nullptr, nullptr, &p->total_slots, nullptr);
            return p;
        },
        py::arg("matrix"), py::arg("width"), py::arg("strategy") = Strategy::Adaptive);
    mod.def(
        "sampling_rate",
        [](const PlanSet& plans, const Csr& m) {
            double agg = 0, uni = 0;
            check(nogil([&] { return aes_sampling_rate(plans.h, m.h, &agg, &uni, nullptr); }));
            return py::make_tuple(agg, uni);
        },
        py::arg("plans"), py::arg("matrix"), "aggregate (slot rate, unique coverage) of a plan set");
    mod.def(
        "sampling_rate_per_row",
        [](const PlanSet& plans, const Csr& m) {
            py::array_t<double> pr(m.n_rows);
            double* p = pr.mutable_data();
            double agg = 0, uni = 0;
            check(nogil([&] { return aes_sampling_rate(plans.h, m.h, &agg, &uni, p); }));
            return pr;
        },
        py::arg("plans"), py::arg("matrix"));
    // cdf_stats (bench.hpp:58-59, bench.cpp:124-138): [(rate, fraction), ...]
    mod.def(
        "cdf_stats",
        [](py::array_t<double, py::array::c_style | py::array::forcecast> rates) {
            const uint64_t n = (uint64_t)rates.size();
            std::vector<double> r(n ? n : 1), fr(n ? n : 1);
            uint64_t steps = 0;
            const double* pr = rates.data();
            check(nogil([&] { return aes_cdf_stats(pr, n, r.data(), fr.data(), &steps); }));
            py::list out;
            for (uint64_t i = 0; i < steps; ++i) out.append(py::make_tuple(r[i], fr[i]));
            return out;
        },
        py::arg("rates"), "empirical CDF of per-row sampling rates (sorted steps, ties merged)");
    mod.def(
        "sampling_rate_cdf",
        [](const PlanSet& plans, const Csr& m) {
            std::vector<double> r(m.n_rows ? m.n_rows : 1), fr(m.n_rows ? m.n_rows : 1);
            uint64_t steps = 0;
            check(nogil([&] { return aes_sampling_rate_cdf(plans.h, m.h, r.data(), fr.data(), &steps); }));
            py::array_t<double> ra(steps), fa(steps);
            std::copy(r.begin(), r.begin() + steps, ra.mutable_data());
            std::copy(fr.begin(), fr.begin() + steps, fa.mutable_data());
            return py::make_tuple(ra, fa);
        },
        py::arg("plans"), py::arg("matrix"), "cdf_stats of the per-row sampling rates, computed on the device");

    mod.def(
        "spmm_exact",
        [](const Csr& a, F32In b, unsigned /*n_threads*/) {
            b = as_2d(b);
            uint64_t br = b.shape(0), f = b.shape(1);
            if (a.n_cols != br) throw py::value_error("ShapeMismatch");
            auto c = new_2d(a.n_rows, f);
            float* pc = c.mutable_data();
            const float* pb = b.data();
            check(nogil([&] { return aes_spmm_exact(a.h, pb, br, f, pc); }));
            return c;
        },
        py::arg("a"), py::arg("b"), py::arg("n_threads") = 0);
    mod.def(
        "spmm_sampled",
        [](const Csr& a, F32In b, const PlanSet& p, unsigned /*n_threads*/) {
            b = as_2d(b);
            uint64_t br = b.shape(0), f = b.shape(1);
            auto c = new_2d(a.n_rows, f);
            float* pc = c.mutable_data();
            const float* pb = b.data();
            check(nogil([&] { return aes_spmm_sampled(a.h, pb, br, f, p.h, pc, nullptr, nullptr, nullptr); }));
            return c;
        },
        py::arg("a"), py::arg("b"), py::arg("plans"), py::arg("n_threads") = 0);
    mod.def(
        "spmm_sampled_instrumented",
        [](const Csr& a, F32In b, const PlanSet& p, unsigned /*n_threads*/) {
            b = as_2d(b);
            uint64_t br = b.shape(0), f = b.shape(1);
            auto c = new_2d(a.n_rows, f);
            float* pc = c.mutable_data();
            const float* pb = b.data();
            uint64_t fma = 0, la = 0, lb = 0;
            check(nogil([&] { return aes_spmm_sampled(a.h, pb, br, f, p.h, pc, &fma, &la, &lb); }));
            py::dict w;
            w["fma_count"] = fma;
            w["loads_a"] = la;
            w["loads_b"] = lb;
            return py::make_tuple(c, w);
        },
        py::arg("a"), py::arg("b"), py::arg("plans"), py::arg("n_threads") = 0);
    mod.def(
        "exact_work",
        [](const Csr& a, F32In b) {
            b = as_2d(b);
            py::dict w;
            w["fma_count"] = a.nnz * uint64_t(b.shape(1));
            w["loads_a"] = a.nnz;
            w["loads_b"] = a.nnz * uint64_t(b.shape(1));
            return w;
        },
        py::arg("a"), py::arg("b"));

    mod.def(
        "quantize",
        [](F32In x, uint32_t bits) {
            x = as_2d(x);
            aes_qfeat_t h = nullptr;
            uint64_t r = x.shape(0), c = x.shape(1);
            const float* px = x.data();
            check(nogil([&] { return aes_quantize(px, r, c, bits, &h); }));
            return std::make_shared<QFeat>(h);
        },
        py::arg("x"), py::arg("bits") = 8);
    mod.def(
        "quantize_affine",
        [](F32In x, const std::string& mode) {
            x = as_2d(x);
            int m = mode == "row" ? AES_QAFFINE_ROW : mode == "feature" ? AES_QAFFINE_FEATURE : -1;
            if (m < 0) throw py::value_error("mode must be 'row' or 'feature'");
            aes_qfeat_t h = nullptr;
            uint64_t r = x.shape(0), c = x.shape(1);
            const float* px = x.data();
            check(nogil([&] { return aes_quantize_affine(px, r, c, m, &h); }));
            return std::make_shared<QFeat>(h);
        },
        py::arg("x"), py::arg("mode") = "row",
        "FAST MODE int8 codes with per-row or per-feature (scale, offset); spmm_sampled_q8 / dequantize "
        "decode them (not bit-exact; error bounds in include/aesspmm_cuda.h)");
    mod.def(
        "quantize_with",
        [](F32In x, const QuantParams& p) {
            x = as_2d(x);
            aes_qfeat_t h = nullptr;
            uint64_t r = x.shape(0), c = x.shape(1);
            const float* px = x.data();
            check(nogil([&] { return aes_quantize_with(px, r, c, p.x_min, p.x_max, p.bits, &h); }));
            return std::make_shared<QFeat>(h);
        },
        py::arg("x"), py::arg("params"), "quantize(x, p) with explicit QuantParams (quantize.hpp:31)");
    mod.def(
        "fit_params",
        [](F32In x, uint32_t bits) {
            x = as_2d(x);
            QuantParams p;
            p.bits = bits;
            uint64_t r = x.shape(0), c = x.shape(1);
            const float* px = x.data();
            check(nogil([&] { return aes_fit_params(px, r, c, bits, &p.x_min, &p.x_max); }));
            return p;
        },
        py::arg("x"), py::arg("bits") = 8);
    mod.def(
        "quantized_from_codes",
        [](py::array_t<uint16_t, py::array::c_style | py::array::forcecast> codes, const QuantParams& p) {
            if (codes.ndim() != 2) throw py::value_error("expected a 2-d array");
            aes_qfeat_t h = nullptr;
            uint64_t r = codes.shape(0), c = codes.shape(1);
            const uint16_t* pc = codes.data();
            check(nogil([&] { return aes_qfeat_from_codes(pc, r, c, p.x_min, p.x_max, p.bits, &h); }));
            return std::make_shared<QFeat>(h);
        },
        py::arg("codes"), py::arg("params"));
    mod.def(
        "dequantize",
        [](const QFeat& q) {
            auto x = new_2d(q.n_rows, q.n_cols);
            float* px = x.mutable_data();
            check(nogil([&] { return aes_dequantize(q.h, px); }));
            return x;
        },
        py::arg("qf"));
    mod.def(
        "spmm_sampled_q8",
        [](const Csr& a, const QFeat& q, std::optional<PlanP> p) {
            auto c = new_2d(a.n_rows, q.n_cols);
            float* pc = c.mutable_data();
            aes_plan_t ph = p && *p ? (*p)->h : nullptr;
            check(nogil([&] { return aes_spmm_sampled_q8(a.h, q.h, ph, pc); }));
            return c;
        },
        py::arg("a"), py::arg("qf"), py::arg("plans") = py::none(),
        "spmm_sampled(a, dequantize(qf), plans) with dequantization fused into the int8 gather");

    mod.def(
        "dense_matmul",
        [](F32In a, F32In b, unsigned /*n_threads*/) {
            a = as_2d(a);
            b = as_2d(b);
            if (a.shape(1) != b.shape(0)) throw py::value_error("ShapeMismatch");
            uint64_t m = a.shape(0), k = a.shape(1), n = b.shape(1);
            auto c = new_2d(m, n);
            float* pc = c.mutable_data();
            const float *pa = a.data(), *pb = b.data();
            check(nogil([&] { return aes_dense_matmul(pa, m, k, pb, n, pc); }));
            return c;
        },
        py::arg("a"), py::arg("b"), py::arg("n_threads") = 0);
    mod.def(
        "gcn_normalize",
        [](const Csr& a, bool add_self_loops) {
            aes_csr_t h = nullptr;
            check(nogil([&] { return aes_gcn_normalize(a.h, add_self_loops ? 1 : 0, &h); }));
            return std::make_shared<Csr>(h);
        },
        py::arg("a"), py::arg("add_self_loops") = true);
    mod.def(
        "row_stats",
        [](const Csr& a) {
            py::array_t<uint64_t> rn(a.n_rows);
            uint64_t* p = rn.mutable_data();
            uint64_t mx = 0;
            double avg = 0;
            check(nogil([&] { return aes_csr_row_stats(a.h, p, &mx, &avg); }));
            return py::make_tuple(rn, mx, avg);
        },
        py::arg("matrix"));
    // GCN / SAGE-mean forward: weights are in_dim x out_dim (in_dim doubles for SAGE)
    auto forward = [](bool sage, const Csr& adj, F32In x, std::vector<F32In> weights, std::vector<F32In> biases,
                      std::optional<PlanP> plans, bool fast_gemm) {
        x = as_2d(x);
        if (biases.size() != weights.size()) throw py::value_error("one bias per layer (may be empty)");
        if (adj.n_cols != uint64_t(x.shape(0))) throw py::value_error("ShapeMismatch");
        std::vector<uint64_t> dims{uint64_t(x.shape(1))}, blen;
        std::vector<float> wcat, bcat;
        for (size_t l = 0; l < weights.size(); ++l) {
            F32In w = as_2d(weights[l]);
            if (uint64_t(w.shape(0)) != (sage ? 2 : 1) * dims.back()) throw py::value_error("ShapeMismatch");
            dims.push_back(w.shape(1));
            wcat.insert(wcat.end(), w.data(), w.data() + w.size());
            F32In b = biases[l];
            if (b.size() != 0 && uint64_t(b.size()) != dims.back()) throw py::value_error("ShapeMismatch");
            blen.push_back(b.size());
            bcat.insert(bcat.end(), b.data(), b.data() + b.size());
        }
        auto out = new_2d(adj.n_rows, dims.back());
        float* po = out.mutable_data();
        const float* px = x.data();
        aes_plan_t ph = plans && *plans ? (*plans)->h : nullptr;
        check(nogil([&] {
            return aes_gnn_forward_ex(sage ? 1 : 0, adj.h, px, dims.data(), int(weights.size()), wcat.data(),
                                      bcat.empty() ? nullptr : bcat.data(), blen.data(), ph, fast_gemm ? 1 : 0, po);
        }));
        return out;
    };
    mod.def(
        "gcn_forward",
        [forward](const Csr& adj, F32In x, std::vector<F32In> w, std::vector<F32In> b, std::optional<PlanP> plans,
                  unsigned, bool fast_gemm) { return forward(false, adj, x, w, b, plans, fast_gemm); },
        py::arg("adj"), py::arg("features"), py::arg("weights"), py::arg("biases"),
        py::arg("plans") = py::none(), py::arg("n_threads") = 0, py::arg("fast_gemm") = false,
        "gcn_forward (gnn.cpp:66-78): relu(spmm(adj, H) @ W + b) per layer, no ReLU after the last. "
        "fast_gemm=True: layer transforms on the tcgen05 tensor cores (TF32, not bit-exact)");
    mod.def(
        "sage_forward",
        [forward](const Csr& adj_mean, F32In x, std::vector<F32In> w, std::vector<F32In> b,
                  std::optional<PlanP> plans, unsigned, bool fast_gemm) {
            return forward(true, adj_mean, x, w, b, plans, fast_gemm);
        },
        py::arg("adj_mean"), py::arg("features"), py::arg("weights"), py::arg("biases"),
        py::arg("plans") = py::none(), py::arg("n_threads") = 0, py::arg("fast_gemm") = false,
        "sage_forward (gnn.cpp:80-95): relu(concat(H, spmm(adj_mean, H)) @ W + b) per layer");
    // ---- binary files straight to HBM (io.cpp:117-220 formats)
    mod.def(
        "load_csr_binary",
        [](const std::string& path) {
            aes_csr_t h = nullptr;
            double ms = 0;
            check(nogil([&] { return aes_csr_load(path.c_str(), &h, &ms); }));
            return std::make_shared<Csr>(h);
        },
        py::arg("path"), "CSRB file -> HBM CsrMatrix (validated on the GPU)");
    mod.def(
        "save_csr_binary",
        [](const Csr& m, const std::string& path) { check(nogil([&] { return aes_csr_save(m.h, path.c_str()); })); },
        py::arg("matrix"), py::arg("path"));
    mod.def(
        "load_features",
        [](const std::string& path) -> py::tuple {
            int dtype = 0;
            uint64_t r = 0, c = 0;
            float lo = 0, hi = 0;
            check(aes_fmat_info(path.c_str(), &dtype, &r, &c, &lo, &hi));
            double ms = 0;
            if (dtype == 1) {
                aes_qfeat_t h = nullptr;
                check(nogil([&] { return aes_fmat_load_qfeat(path.c_str(), &h, &ms); }));
                return py::make_tuple(std::make_shared<QFeat>(h), ms);
            }
            // dtype 0: f32 features as numpy (the reference returns a host DenseMatrix)
            auto out = new_2d(r, c);
            float* po = out.mutable_data();
            FILE* f = fopen(path.c_str(), "rb");
            if (!f) throw std::runtime_error("Io: cannot open for reading: " + path);
            fseek(f, 22, SEEK_SET);
            size_t got = fread(po, 4, r * c, f);
            fclose(f);
            if (got != r * c) throw std::runtime_error("TruncatedFile: " + path);
            return py::make_tuple(out, ms);
        },
        py::arg("path"), "FMAT file -> (QuantizedFeatures in HBM | float32 array, load_ms)");
    mod.def(
        "save_fmat",
        [](py::object obj, const std::string& path) {
            if (py::isinstance<QFeat>(obj)) {
                const QFeat& q = obj.cast<const QFeat&>();
                check(nogil([&] { return aes_fmat_save_qfeat(q.h, path.c_str()); }));
                return;
            }
            F32In x = as_2d(obj.cast<F32In>());
            const float* px = x.data();
            uint64_t r = x.shape(0), c = x.shape(1);
            check(nogil([&] { return aes_fmat_save_f32(px, r, c, path.c_str()); }));
        },
        py::arg("features"), py::arg("path"), "save_fmat (io.cpp:160-181): f32 array or 8-bit QuantizedFeatures");
    mod.def(
        "row_mean_normalize",
        [](const Csr& a) {
            aes_csr_t h = nullptr;
            check(nogil([&] { return aes_row_mean_normalize(a.h, &h); }));
            return std::make_shared<Csr>(h);
        },
        py::arg("a"));
    mod.def(
        "argmax_rows",
        [](F32In logits) {
            logits = as_2d(logits);
            uint64_t r = logits.shape(0), c = logits.shape(1);
            py::array_t<uint32_t> out(r);
            uint32_t* po = out.mutable_data();
            const float* px = logits.data();
            check(nogil([&] { return aes_argmax_rows(px, r, c, po); }));
            return out;
        },
        py::arg("logits"));
    mod.def(
        "evaluate",
        [](F32In logits, py::array_t<uint32_t, py::array::c_style | py::array::forcecast> labels,
           std::optional<F32In> reference_logits, std::optional<py::array_t<uint8_t, py::array::c_style |
                                                                             py::array::forcecast>> mask) {
            logits = as_2d(logits);
            uint64_t r = logits.shape(0), c = logits.shape(1);
            const float* ref = nullptr;
            F32In refa;
            if (reference_logits) {
                refa = as_2d(*reference_logits);
                if (uint64_t(refa.shape(0)) != r) throw py::value_error("reference shape mismatch");
                ref = refa.data();
            }
            const uint8_t* pm = mask ? mask->data() : nullptr;
            uint64_t ml = mask ? mask->size() : 0;
            double acc = 0, agree = 0;
            std::vector<uint64_t> per_class(c);
            const float* pl = logits.data();
            const uint32_t* lab = labels.data();
            uint64_t nl = labels.size();
            check(nogil([&] {
                return aes_evaluate(pl, r, c, lab, nl, ref, pm, ml, &acc, &agree, per_class.data());
            }));
            py::dict d;
            d["accuracy"] = acc;
            d["agreement"] = agree;
            d["per_class"] = per_class;
            return d;
        },
        py::arg("logits"), py::arg("labels"), py::arg("reference_logits") = py::none(), py::arg("mask") = py::none(),
        "evaluate (gnn.cpp:118-155): accuracy vs labels, argmax agreement vs reference logits");
}
