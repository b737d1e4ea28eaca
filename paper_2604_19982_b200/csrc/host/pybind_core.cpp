// Python module paper_2604_19982_b200._core — drop-in for the reference's trijoin._core join
// surface (proj/python/bindings.cpp:101-121, :215-229): same `join` signature, defaults,
// GIL release, (records, stats_json) result and ValueError on invalid specs. Extra entry
// points expose in-memory datasets, a device-resident join handle for benchmarking, the
// GPU primitives and the benchmark index replicator.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <chrono>
#include <csignal>
#include <cstdlib>
#include <execinfo.h>
#include <unistd.h>
#include <cstring>
#include <bit>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "packed.hpp"
#include "replicate.hpp"
#include "trijoin/engine.hpp"

namespace py = pybind11;
using namespace trijoin;

namespace {

using DatasetPtr = std::shared_ptr<const PreparedDataset>;

JoinSpec make_spec(const std::string& type, double tau, uint32_t k, uint64_t filter_chunk, uint64_t refine_chunk,
                   const std::vector<uint32_t>& lods, bool pipeline, uint32_t workers, uint64_t seed, bool exact) {
    JoinSpec spec;
    if (type == "within") spec.type = JoinType::Within;
    else if (type == "intersect") spec.type = JoinType::Intersect;
    else if (type == "knn") spec.type = JoinType::Knn;
    else throw std::invalid_argument("type must be within, intersect, or knn, got: " + type);
    spec.tau = tau;
    spec.k = k;
    spec.filter_chunk = filter_chunk;
    spec.refine_chunk = refine_chunk;
    spec.lods = lods;
    spec.pipeline = pipeline;
    spec.workers = workers;
    spec.seed = seed;
    spec.exact = exact;
    validate(spec);
    return spec;
}

// (records, stats_json) as the reference's _core.join returns them (python/bindings.cpp:101-121);
// built with the CPython API directly (one shared str per stage name).
py::tuple pack_output(const JoinOutput& out) {
    // hundreds of thousands of fresh tuples would trigger repeated cyclic-GC passes over
    // the whole interpreter heap; the records hold no cycles, so collection is paused
    struct GcPause {
        int was = PyGC_Disable();
        ~GcPause() {
            if (was) PyGC_Enable();
        }
    } gc_pause;
    const size_t n = out.records.size();
    py::list records(n);
    std::map<int16_t, py::str> names;
    // shared immutable objects: one int per object id, one float when ub == lb (bitwise)
    std::vector<py::object> ints;
    auto int_of = [&](uint32_t v) -> PyObject* {
        if (v >= ints.size()) ints.resize(std::max<size_t>(v + 1, ints.size() * 2));
        if (!ints[v]) ints[v] = py::reinterpret_steal<py::object>(PyLong_FromUnsignedLong(v));
        PyObject* o = ints[v].ptr();
        Py_INCREF(o);
        return o;
    };
    // +0.0 (every confirmed intersection record's bounds) as one shared float
    const py::object zero = py::reinterpret_steal<py::object>(PyFloat_FromDouble(0.0));
    auto float_of = [&](double v) -> PyObject* {
        if (std::bit_cast<uint64_t>(v) == 0) {
            Py_INCREF(zero.ptr());
            return zero.ptr();
        }
        PyObject* o = PyFloat_FromDouble(v);
        if (!o) throw py::error_already_set();
        return o;
    };
    int16_t last_stage = 0;
    PyObject* last_name = nullptr;
    for (size_t i = 0; i < n; ++i) {
        const JoinResultRecord& r = out.records[i];
        if (!last_name || r.decided_at != last_stage) {
            auto it = names.find(r.decided_at);
            if (it == names.end()) it = names.emplace(r.decided_at, py::str(stage_name(r.decided_at))).first;
            last_stage = r.decided_at;
            last_name = it->second.ptr();
        }
        PyObject* t = PyTuple_New(6);
        if (!t) throw py::error_already_set();
        PyTuple_SET_ITEM(t, 0, int_of(r.r));
        PyTuple_SET_ITEM(t, 1, int_of(r.s));
        PyObject* lb = float_of(r.lb);
        PyTuple_SET_ITEM(t, 2, lb);
        if (std::memcmp(&r.lb, &r.ub, sizeof(double)) == 0) {
            Py_INCREF(lb);
            PyTuple_SET_ITEM(t, 3, lb);
        } else {
            PyTuple_SET_ITEM(t, 3, float_of(r.ub));
        }
        PyObject* nm = last_name;
        Py_INCREF(nm);
        PyTuple_SET_ITEM(t, 4, nm);
        PyTuple_SET_ITEM(t, 5, int_of(r.rank));
        PyList_SET_ITEM(records.ptr(), static_cast<Py_ssize_t>(i), t);
    }
    return py::make_tuple(records, out.stats.to_json());
}

// Packed-form caches of the Python Dataset objects (immutable once loaded): keyed by the
// dataset's address, validated by a weak reference (a freed dataset's entry is dropped).
detail::JoinCache* dataset_cache(const std::shared_ptr<PreparedDataset>& ds) {
    static std::mutex mu;
    // never destroyed (pinned host buffers must not be released after the CUDA runtime's teardown)
    static auto& caches = *new std::map<const PreparedDataset*,
                                        std::pair<std::weak_ptr<PreparedDataset>, std::unique_ptr<detail::JoinCache>>>;
    std::lock_guard<std::mutex> lk(mu);
    for (auto it = caches.begin(); it != caches.end();)
        it = it->second.first.expired() ? caches.erase(it) : std::next(it);
    auto& e = caches[ds.get()];
    if (!e.second || e.first.lock() != ds) e = {ds, std::make_unique<detail::JoinCache>()};
    return e.second.get();
}

// Records as a numpy structured array: r u4, s u4, lb f8, ub f8, stage i2, rank u4.
py::object records_array(const JoinOutput& out) {
    struct Rec {
        uint32_t r, s;
        double lb, ub;
        int16_t stage, pad;
        uint32_t rank;
    };
    static_assert(sizeof(Rec) == 32);
    py::list names, formats, offsets;
    for (auto [n, f, o] : {std::tuple{"r", "<u4", 0}, {"s", "<u4", 4}, {"lb", "<f8", 8}, {"ub", "<f8", 16},
                           {"stage", "<i2", 24}, {"rank", "<u4", 28}}) {
        names.append(n);
        formats.append(f);
        offsets.append(o);
    }
    py::dict spec;
    spec["names"] = names;
    spec["formats"] = formats;
    spec["offsets"] = offsets;
    spec["itemsize"] = 32;
    const py::dtype dt = py::reinterpret_borrow<py::dtype>(py::module_::import("numpy").attr("dtype")(spec));
    if (dt.itemsize() != static_cast<py::ssize_t>(sizeof(Rec))) throw std::runtime_error("record dtype is not 32 bytes");
    py::array a(dt, std::vector<py::ssize_t>{static_cast<py::ssize_t>(out.records.size())});
    Rec* w = static_cast<Rec*>(a.mutable_data());
    for (size_t i = 0; i < out.records.size(); ++i) {
        const JoinResultRecord& x = out.records[i];
        w[i] = {x.r, x.s, x.lb, x.ub, x.decided_at, 0, x.rank};
    }
    return a;
}

py::tuple join_paths(const std::string& r_path, const std::string& s_path, const JoinSpec& spec,
                     bool oracle = false) {
    JoinOutput out;
    {
        py::gil_scoped_release release;
        ThreadPool pool(spec.workers);
        const PreparedDataset R = load_index(r_path);
        PreparedDataset s_store;
        const PreparedDataset* S = &R;
        if (!s_path.empty() && s_path != r_path) {
            s_store = load_index(s_path);
            S = &s_store;
        }
        out = oracle ? run_oracle(R, *S, spec, pool) : run_join(R, *S, spec, pool);
    }
    return pack_output(out);
}

// A device-resident (R, S) pair on one GPU: packed and uploaded once, joined many times.
class Resident {
public:
    // shard_count > 1: only the queries of shard shard_index (blocks of `block` queries dealt
    // round-robin) are packed and uploaded; S is uploaded whole.
    Resident(DatasetPtr R, DatasetPtr S, int device, unsigned workers, uint32_t shard_index, uint32_t shard_count,
             uint32_t block, bool compact)
        : R_(std::move(R)), S_(std::move(S)) {
        py::gil_scoped_release release;
        ctx_ = detail::device_context(device);
        ThreadPool pool(workers);
        std::vector<uint32_t> ids;
        const bool sharded = shard_count > 1;
        if (sharded) {
            if (shard_index >= shard_count || block == 0) throw std::invalid_argument("Resident: bad shard");
            const size_t nr = R_->objects.size();
            for (size_t b0 = size_t{shard_index} * block; b0 < nr; b0 += size_t{shard_count} * block)
                for (size_t r = b0; r < std::min(nr, b0 + block); ++r) ids.push_back(static_cast<uint32_t>(r));
        }
        n_queries_ = sharded ? ids.size() : R_->objects.size();
        const bool two = sharded || S_.get() != R_.get();
        if (compact) { // compact-resident (TJ_DATASET_COMPACT): the streamed form, kept in HBM
            auto upload = [&](const PreparedDataset& D, const std::vector<uint32_t>* sel, detail::DatasetHandle& h) {
                auto hd = sel ? detail::pack_header(D, *sel, pool) : detail::pack_header(D, pool);
                detail::check(tj_dataset_begin_ex(ctx_, &hd->view, hd->vb_ptrs.data(), hd->fb_ptrs.data(),
                                                  TJ_DATASET_COMPACT, &h.p),
                              ctx_);
                for (size_t li = 0; li < D.lod_schedule.size(); ++li) {
                    auto lv = detail::pack_level(D, *hd, li, pool);
                    detail::check(tj_dataset_put_level(h.p, static_cast<uint32_t>(li), &lv->view), ctx_);
                    detail::check(tj_dataset_sync(h.p), ctx_); // lv's pinned buffers are reused next
                }
                bytes_ += tj_dataset_device_bytes(h.p);
            };
            upload(*R_, sharded ? &ids : nullptr, dr_);
            if (two) upload(*S_, nullptr, ds_);
            return;
        }
        auto pr = detail::pack_dataset(*R_, pool, sharded ? &ids : nullptr);
        detail::check(tj_dataset_upload(ctx_, &pr->view, &dr_.p), ctx_);
        bytes_ = pr->bytes();
        if (two) {
            auto ps = detail::pack_dataset(*S_, pool);
            detail::check(tj_dataset_upload(ctx_, &ps->view, &ds_.p), ctx_);
            bytes_ += ps->bytes();
        }
    }
    uint64_t device_bytes() const { return bytes_; }
    uint64_t n_queries() const { return n_queries_; }

    py::dict run(const std::string& type, double tau, uint32_t k, const std::vector<uint32_t>& lods,
                 uint64_t refine_chunk, uint32_t flags, uint32_t shard_index, uint32_t shard_count,
                 bool want_arrays) {
        JoinSpec spec = make_spec(type, tau, k, 4194304, refine_chunk, lods, true, 0, 0, false);
        tj_join_spec c{};
        c.type = spec.type == JoinType::Within ? TJ_WITHIN : spec.type == JoinType::Intersect ? TJ_INTERSECT : TJ_KNN;
        c.tau = spec.tau;
        c.k = spec.k;
        c.filter_chunk = spec.filter_chunk;
        c.refine_chunk = spec.refine_chunk;
        c.n_lods = static_cast<uint32_t>(spec.lods.size());
        c.lods = spec.lods.data();
        c.pipeline = 1;
        c.flags = flags;
        c.shard_index = shard_index;
        c.shard_count = shard_count;
        c.shard_block = 1024;
        detail::ResultHandle res;
        {
            py::gil_scoped_release release;
            detail::check(tj_join(ctx_, dr_.p, ds_.p ? ds_.p : dr_.p, &c, nullptr, &res.r), ctx_);
        }
        const tj_join_result& r = res.r;
        py::dict d;
        d["n_cands"] = r.n_cands;
        uint64_t undecided_after_mbb = 0, confirmed = 0;
        for (uint64_t op = 0; op < r.n_cands; ++op) {
            confirmed += r.status[op] == TJ_CONFIRMED;
            undecided_after_mbb += r.decided_at[op] != TJ_STAGE_MBB;
        }
        d["confirmed"] = confirmed;
        d["voxel_pairs_in"] = undecided_after_mbb; // = stats stages["voxel"].pairs_in
        d["vp_generated"] = r.vp_generated;
        d["vp_pruned"] = r.vp_pruned;
        d["mbb_ms"] = r.mbb_ms;
        d["voxel_ms"] = r.voxel_ms;
        d["refine_ms"] = r.refine_ms;
        d["total_ms"] = r.total_ms;
        d["decision_mode"] = r.decision_mode;
        py::list levels;
        for (uint32_t i = 0; i < r.n_levels_run; ++i) {
            py::dict l;
            l["level"] = r.level[i];
            l["vps"] = r.level_vps[i];
            l["facet_pairs"] = r.level_facet_pairs[i];
            l["evaluated"] = r.level_pairs_evaluated[i];
            l["tested"] = r.level_pairs_tested[i];
            l["screened"] = r.level_pairs_screened[i];
            l["verified"] = r.level_pairs_verified[i];
            l["vps_skipped"] = r.level_vps_skipped[i];
            l["facets_dropped"] = r.level_facets_dropped[i];
            l["ms"] = r.level_ms[i];
            l["kernel_ms"] = r.level_kernel_ms[i];
            l["screen_ms"] = r.level_screen_ms[i];
            levels.append(l);
        }
        d["levels"] = levels;
        if (want_arrays) {
            const size_t n = r.n_cands;
            d["pair_r"] = py::array_t<uint32_t>(n, r.pair_r);
            d["pair_s"] = py::array_t<uint32_t>(n, r.pair_s);
            d["lb"] = py::array_t<double>(n, r.lb);
            d["ub"] = py::array_t<double>(n, r.ub);
            d["status"] = py::array_t<uint8_t>(n, r.status);
            d["decided_at"] = py::array_t<int16_t>(n, r.decided_at);
        }
        return d;
    }

private:
    DatasetPtr R_, S_;
    uint64_t n_queries_ = 0;
    tj_ctx* ctx_ = nullptr;
    detail::DatasetHandle dr_, ds_;
    uint64_t bytes_ = 0;
};

} // namespace

// $TRIJOIN_BACKTRACE=1: print a native backtrace on SIGSEGV / SIGABRT (diagnostics).
void crash_handler(int sig) {
    void* frames[64];
    const int n = backtrace(frames, 64);
    const char msg[] = "trijoin: fatal signal, native backtrace:\n";
    (void)!write(2, msg, sizeof(msg) - 1);
    backtrace_symbols_fd(frames, n, 2);
    std::signal(sig, SIG_DFL);
    std::raise(sig);
}

PYBIND11_MODULE(_core, m) {
    if (const char* e = std::getenv("TRIJOIN_BACKTRACE"); e && *e == '1') {
        std::signal(SIGSEGV, crash_handler);
        std::signal(SIGABRT, crash_handler);
    }
    m.doc() = "B200-native filter-and-refine spatial joins over triangulated polyhedra (trijoin drop-in)";

    py::register_exception<EngineError>(m, "EngineError", PyExc_RuntimeError);
    py::register_exception<IndexError>(m, "IndexError", PyExc_RuntimeError);

    m.def(
        "join",
        [](const std::string& r, const std::string& s, const std::string& type, double tau, uint32_t k,
           uint64_t filter_chunk, uint64_t refine_chunk, const std::vector<uint32_t>& lods, bool pipeline,
           uint32_t workers, uint64_t seed, bool exact) {
            return join_paths(r, s, make_spec(type, tau, k, filter_chunk, refine_chunk, lods, pipeline, workers, seed, exact));
        },
        py::arg("r"), py::arg("s") = "", py::arg("type") = "within", py::arg("tau") = 0.0, py::arg("k") = 1,
        py::arg("filter_chunk") = 4194304, py::arg("refine_chunk") = 500000,
        py::arg("lods") = std::vector<uint32_t>{20, 40, 60, 80, 100}, py::arg("pipeline") = true,
        py::arg("workers") = 0, py::arg("seed") = 0, py::arg("exact") = false,
        "Returns (records, stats_json). Each record is (r, s, lb, ub, stage, rank); rank is 0 except for knn. "
        "s defaults to a self-join on r.");

    m.def(
        "oracle",
        [](const std::string& r, const std::string& s, const std::string& type, double tau, uint32_t k,
           uint32_t workers, uint64_t seed) {
            return join_paths(r, s, make_spec(type, tau, k, 4194304, 500000, {20, 40, 60, 80, 100}, true, workers,
                                              seed, false),
                              true);
        },
        py::arg("r"), py::arg("s") = "", py::arg("type") = "within", py::arg("tau") = 0.0, py::arg("k") = 1,
        py::arg("workers") = 0, py::arg("seed") = 0,
        "Exhaustive exact join over the level-100 geometry on the GPU (reference _core.oracle). "
        "Returns (records, stats_json).");

    m.def(
        "oracle_datasets",
        [](const PreparedDataset& R, const PreparedDataset& S, const std::string& type, double tau, uint32_t k) {
            JoinOutput out;
            {
                py::gil_scoped_release release;
                ThreadPool pool(1);
                out = run_oracle(R, S, make_spec(type, tau, k, 4194304, 500000, {20, 40, 60, 80, 100}, true, 1, 0,
                                                 false),
                                 pool);
            }
            return pack_output(out);
        },
        py::arg("r"), py::arg("s"), py::arg("type") = "within", py::arg("tau") = 0.0, py::arg("k") = 1,
        "run_oracle on loaded datasets (s may be r: self-join). Returns (records, stats_json).");

    py::class_<PreparedDataset, std::shared_ptr<PreparedDataset>>(m, "Dataset")
        .def_property_readonly("n_objects", [](const PreparedDataset& d) { return d.objects.size(); })
        .def_property_readonly("lod_schedule", [](const PreparedDataset& d) { return d.lod_schedule; })
        .def("mbbs",
             [](const PreparedDataset& d) {
                 py::array_t<double> a(std::vector<py::ssize_t>{static_cast<py::ssize_t>(d.objects.size()), 6});
                 double* w = a.mutable_data();
                 for (size_t o = 0; o < d.objects.size(); ++o) {
                     const Aabb& b = d.objects[o].mbb;
                     const double v[6] = {b.min.x, b.min.y, b.min.z, b.max.x, b.max.y, b.max.z};
                     std::memcpy(w + 6 * o, v, sizeof(v));
                 }
                 return a;
             })
        .def("facet_count", [](const PreparedDataset& d, size_t level_index) {
            uint64_t n = 0;
            for (const auto& o : d.objects) n += o.ladder.levels.at(level_index).mesh.facets.size();
            return n;
        });

    m.def(
        "load_dataset",
        [](const std::string& path) {
            py::gil_scoped_release release;
            return std::make_shared<PreparedDataset>(load_index(path));
        },
        py::arg("path"));

    m.def(
        "pack_timing",
        [](std::shared_ptr<PreparedDataset> R, unsigned workers) {
            // host-side cost of the streamed upload's packing (diagnostics for bench.py)
            using Clock = std::chrono::steady_clock;
            py::dict d;
            py::gil_scoped_release release;
            ThreadPool pool(workers);
            auto t0 = Clock::now();
            auto h = detail::pack_header(*R, pool);
            double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
            std::vector<double> lv;
            for (size_t li = 0; li < R->lod_schedule.size(); ++li) {
                t0 = Clock::now();
                auto p = detail::pack_level(*R, *h, li, pool);
                lv.push_back(std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
            }
            py::gil_scoped_acquire acquire;
            d["header_ms"] = ms;
            d["level_ms"] = lv;
            d["workers"] = pool.size();
            return d;
        },
        py::arg("R"), py::arg("workers") = 0u);

    m.def(
        "save_dataset",
        [](std::shared_ptr<PreparedDataset> ds, const std::string& path) {
            py::gil_scoped_release release;
            save_index(*ds, path);
        },
        py::arg("dataset"), py::arg("path"));

    m.def(
        "join_datasets",
        [](std::shared_ptr<PreparedDataset> R, std::shared_ptr<PreparedDataset> S, const std::string& type, double tau,
           uint32_t k, uint64_t filter_chunk, uint64_t refine_chunk, const std::vector<uint32_t>& lods, bool pipeline,
           uint32_t workers, bool exact, const std::string& records) {
            const JoinSpec spec = make_spec(type, tau, k, filter_chunk, refine_chunk, lods, pipeline, workers, 0, exact);
            JoinOutput out;
            {
                py::gil_scoped_release release;
                ThreadPool pool(workers);
                // the datasets' packed streamed form is kept with them: later joins only copy
                detail::JoinCache* rc = dataset_cache(R);
                detail::JoinCache* sc = S && S != R ? dataset_cache(S) : rc;
                out = detail::run_join_cached(*R, S ? *S : *R, spec, pool, nullptr, rc, sc);
            }
            if (records == "array") return py::tuple(py::make_tuple(records_array(out), out.stats.to_json()));
            if (records != "list") throw std::invalid_argument("records must be 'list' or 'array'");
            return pack_output(out);
        },
        py::arg("R"), py::arg("S") = nullptr, py::arg("type") = "within", py::arg("tau") = 0.0, py::arg("k") = 1,
        py::arg("filter_chunk") = 4194304, py::arg("refine_chunk") = 500000,
        py::arg("lods") = std::vector<uint32_t>{20, 40, 60, 80, 100}, py::arg("pipeline") = true,
        py::arg("workers") = 0, py::arg("exact") = false, py::arg("records") = "list",
        "run_join on in-memory datasets (host buffers in, records out): packs (once per dataset; the packed "
        "form is kept with the dataset), uploads, joins, copies back. records='array' returns the records as "
        "a numpy structured array (r, s, lb, ub, stage code, rank) instead of a list of tuples.");

    py::class_<Resident>(m, "Resident")
        .def(py::init([](std::shared_ptr<PreparedDataset> R, std::shared_ptr<PreparedDataset> S, int device,
                         unsigned workers, uint32_t shard_index, uint32_t shard_count, uint32_t block, bool compact) {
                 return new Resident(R, S ? S : R, device, workers, shard_index, shard_count, block, compact);
             }),
             py::arg("R"), py::arg("S") = nullptr, py::arg("device") = 0, py::arg("workers") = 0,
             py::arg("shard_index") = 0u, py::arg("shard_count") = 1u, py::arg("block") = 1024u,
             py::arg("compact") = false)
        .def_property_readonly("device_bytes", &Resident::device_bytes)
        .def_property_readonly("n_queries", &Resident::n_queries)
        .def("run", &Resident::run, py::arg("type") = "within", py::arg("tau") = 0.0, py::arg("k") = 1,
             py::arg("lods") = std::vector<uint32_t>{20, 40, 60, 80, 100}, py::arg("refine_chunk") = 500000,
             py::arg("flags") = 0u, py::arg("shard_index") = 0u, py::arg("shard_count") = 1u,
             py::arg("arrays") = false);

    m.def(
        "replicate_index",
        [](std::shared_ptr<PreparedDataset> tmpl, const std::string& out_path, const std::vector<uint32_t>& ids,
           const std::vector<std::array<double, 3>>& shifts) {
            std::vector<Point3> sh;
            sh.reserve(shifts.size());
            for (const auto& s : shifts) sh.push_back({s[0], s[1], s[2]});
            py::gil_scoped_release release;
            return replicate_index(*tmpl, out_path, ids, sh);
        },
        py::arg("template"), py::arg("out_path"), py::arg("template_ids"), py::arg("shifts"));

    m.def(
        "replicate_dataset",
        [](std::shared_ptr<PreparedDataset> tmpl, py::array_t<uint32_t, py::array::c_style | py::array::forcecast> ids,
           py::array_t<double, py::array::c_style | py::array::forcecast> shifts, unsigned workers) {
            if (shifts.ndim() != 2 || shifts.shape(1) != 3 || ids.ndim() != 1 || shifts.shape(0) != ids.shape(0))
                throw std::invalid_argument("replicate_dataset: ids (n,) and shifts (n, 3) expected");
            const size_t n = ids.shape(0);
            std::span<const uint32_t> id_span(ids.data(), n);
            std::span<const Point3> sh(reinterpret_cast<const Point3*>(shifts.data()), n);
            py::gil_scoped_release release;
            ThreadPool pool(workers);
            return std::make_shared<PreparedDataset>(replicate_dataset(*tmpl, id_span, sh, pool));
        },
        py::arg("template"), py::arg("template_ids"), py::arg("shifts"), py::arg("workers") = 0u,
        "In-memory translated copies of template objects (the benchmark inputs without index files).");

    m.def(
        "tri_tri_distance",
        [](py::array_t<double, py::array::c_style | py::array::forcecast> a,
           py::array_t<double, py::array::c_style | py::array::forcecast> b) {
            if (a.ndim() != 2 || a.shape(1) != 9 || b.ndim() != 2 || b.shape(1) != 9 || a.shape(0) != b.shape(0))
                throw std::invalid_argument("tri_tri_distance: expected two (n, 9) arrays");
            const size_t n = a.shape(0);
            py::array_t<double> out(n);
            tri_tri_distance_batch({reinterpret_cast<const Triangle*>(a.data()), n},
                                   {reinterpret_cast<const Triangle*>(b.data()), n}, {out.mutable_data(), n});
            return out;
        },
        py::arg("a"), py::arg("b"));

    m.def("device_count", [] { return tj_device_count(); });
    m.def("kernel_launches", [] { return tj_kernel_launches(); });
}
