// 3DPJ1 index container (reference format: src/index_io.cpp:109-234; little-endian,
// length-prefixed objects). Reading locates every object's byte range first, then decodes
// the objects on all host cores (the reference decodes serially from a string copy).
#include <algorithm>
#include <atomic>
#include <bit>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <thread>

#include "replicate.hpp"
#include "trijoin/index.hpp"

static_assert(std::endian::native == std::endian::little, "3DPJ1 is little-endian");

namespace trijoin {

namespace {

constexpr char kMagic[5] = {'3', 'D', 'P', 'J', '1'};
constexpr uint32_t kVersion = 1;

class Writer {
public:
    explicit Writer(std::string& out) : out_(out) {}
    template <class T>
    void raw(const T& v) {
        out_.append(reinterpret_cast<const char*>(&v), sizeof(T));
    }
    void pt(const Point3& p) {
        raw(p.x);
        raw(p.y);
        raw(p.z);
    }
    void box(const Aabb& b) {
        pt(b.min);
        pt(b.max);
    }

private:
    std::string& out_;
};

class Cursor {
public:
    Cursor(std::string_view d, size_t pos, std::string where) : d_(d), pos_(pos), where_(std::move(where)) {}
    void require(uint64_t n) const {
        if (n > d_.size() || pos_ > d_.size() - n) throw IndexError("truncated index: " + where_);
    }
    template <class T>
    T get() {
        require(sizeof(T));
        T v;
        std::memcpy(&v, d_.data() + pos_, sizeof(T));
        pos_ += sizeof(T);
        return v;
    }
    Point3 pt() {
        const double x = get<double>(), y = get<double>(), z = get<double>();
        return {x, y, z};
    }
    Aabb box() {
        Aabb b;
        b.min = pt();
        b.max = pt();
        return b;
    }
    template <class T>
    void array(T* dst, uint64_t n) {
        if (n > (d_.size() - std::min(pos_, d_.size())) / sizeof(T)) throw IndexError("truncated index: " + where_);
        std::memcpy(dst, d_.data() + pos_, n * sizeof(T));
        pos_ += n * sizeof(T);
    }
    void where(std::string w) { where_ = std::move(w); }
    size_t pos() const { return pos_; }

private:
    std::string_view d_;
    size_t pos_;
    std::string where_;
};

void decode_object(std::string_view bytes, size_t begin, size_t end, uint64_t index, uint32_t n_lods,
                   const std::vector<int>& schedule, PreparedObject& obj) {
    const std::string tag = "object " + std::to_string(index);
    Cursor c(bytes.substr(0, end), begin, tag);
    obj.id = c.get<uint32_t>();
    obj.mbb = c.box();
    obj.anchor = c.pt();
    const uint32_t n_levels = c.get<uint32_t>();
    if (n_levels != n_lods) throw IndexError("corrupt index: " + tag + " level count mismatch");
    obj.ladder.levels.resize(n_levels);
    for (uint32_t li = 0; li < n_levels; ++li) {
        LodMesh& lod = obj.ladder.levels[li];
        c.where(tag + " level " + std::to_string(schedule[li]) + " mesh");
        lod.level = static_cast<int>(c.get<uint32_t>());
        lod.clamped = c.get<uint8_t>() != 0;
        const uint64_t nv = c.get<uint64_t>();
        c.require(nv * 24);
        lod.mesh.vertices.resize(nv);
        c.array(reinterpret_cast<double*>(lod.mesh.vertices.data()), nv * 3);
        const uint64_t nf = c.get<uint64_t>();
        c.require(nf * 12);
        lod.mesh.facets.resize(nf);
        c.array(reinterpret_cast<uint32_t*>(lod.mesh.facets.data()), nf * 3);
        for (const auto& f : lod.mesh.facets)
            if (f[0] >= nv || f[1] >= nv || f[2] >= nv)
                throw IndexError("corrupt index: facet index out of range in " + tag);
        c.where(tag + " level " + std::to_string(lod.level) + " bounds");
        c.require(nf * 16);
        lod.hd.resize(nf);
        lod.ph.resize(nf);
        c.array(lod.hd.data(), nf);
        c.array(lod.ph.data(), nf);
        c.where(tag + " level " + std::to_string(lod.level) + " ancestors");
        const uint64_t no = c.get<uint64_t>();
        c.require(no * 4);
        lod.ancestor_of_original.resize(no);
        c.array(lod.ancestor_of_original.data(), no);
        for (uint32_t a : lod.ancestor_of_original)
            if (a >= nf) throw IndexError("corrupt index: ancestor out of range in " + tag);
    }
    c.where(tag + " voxels");
    VoxelSet& vs = obj.voxels;
    const uint32_t nvox = c.get<uint32_t>();
    vs.reassigned = c.get<uint32_t>();
    vs.boxes.resize(nvox);
    vs.anchors.resize(nvox);
    for (uint32_t v = 0; v < nvox; ++v) {
        vs.boxes[v] = c.box();
        vs.anchors[v] = c.pt();
    }
    vs.facets_per_level.assign(n_levels, {});
    for (uint32_t li = 0; li < n_levels; ++li) {
        c.where(tag + " voxel facets, level " + std::to_string(schedule[li]));
        vs.facets_per_level[li].resize(nvox);
        for (uint32_t v = 0; v < nvox; ++v) {
            const uint64_t n = c.get<uint64_t>();
            c.require(n * 4);
            auto& ids = vs.facets_per_level[li][v];
            ids.resize(n);
            c.array(ids.data(), n);
        }
    }
    if (c.pos() != end) throw IndexError("corrupt index: " + tag + " section length mismatch");
}

} // namespace

void serialize_object(const PreparedObject& obj, std::string& body) {
    {
        Writer b(body);
        b.raw(obj.id);
        b.box(obj.mbb);
        b.pt(obj.anchor);
        b.raw(static_cast<uint32_t>(obj.ladder.levels.size()));
        for (const LodMesh& lod : obj.ladder.levels) {
            b.raw(static_cast<uint32_t>(lod.level));
            b.raw(static_cast<uint8_t>(lod.clamped ? 1 : 0));
            b.raw(static_cast<uint64_t>(lod.mesh.vertices.size()));
            for (const Point3& v : lod.mesh.vertices) b.pt(v);
            b.raw(static_cast<uint64_t>(lod.mesh.facets.size()));
            for (const auto& f : lod.mesh.facets) {
                b.raw(f[0]);
                b.raw(f[1]);
                b.raw(f[2]);
            }
            for (double v : lod.hd) b.raw(v);
            for (double v : lod.ph) b.raw(v);
            b.raw(static_cast<uint64_t>(lod.ancestor_of_original.size()));
            for (uint32_t a : lod.ancestor_of_original) b.raw(a);
        }
        const VoxelSet& vs = obj.voxels;
        b.raw(vs.voxel_count());
        b.raw(vs.reassigned);
        for (uint32_t v = 0; v < vs.voxel_count(); ++v) {
            b.box(vs.boxes[v]);
            b.pt(vs.anchors[v]);
        }
        for (const auto& level : vs.facets_per_level)
            for (const auto& ids : level) {
                b.raw(static_cast<uint64_t>(ids.size()));
                for (uint32_t f : ids) b.raw(f);
            }
    }
}

std::string serialize_index(const PreparedDataset& ds) {
    std::string out;
    Writer w(out);
    out.append(kMagic, sizeof(kMagic));
    w.raw(kVersion);
    w.raw(static_cast<uint32_t>(ds.lod_schedule.size()));
    for (int l : ds.lod_schedule) w.raw(static_cast<uint32_t>(l));
    w.raw(static_cast<uint64_t>(ds.objects.size()));
    std::string body;
    for (const PreparedObject& obj : ds.objects) {
        body.clear();
        serialize_object(obj, body);
        w.raw(static_cast<uint64_t>(body.size()));
        out += body;
    }
    return out;
}

PreparedDataset deserialize_index(std::string_view bytes) {
    if (bytes.size() < sizeof(kMagic)) throw IndexError("truncated index: header");
    if (std::memcmp(bytes.data(), kMagic, sizeof(kMagic)) != 0)
        throw IndexError("not a spatial join index (bad magic)");
    Cursor c(bytes, sizeof(kMagic), "header");
    const uint32_t version = c.get<uint32_t>();
    if (version != kVersion)
        throw IndexError("unsupported index version " + std::to_string(version) + " (expected 1)");
    PreparedDataset ds;
    const uint32_t n_lods = c.get<uint32_t>();
    c.require(uint64_t(n_lods) * 4);
    ds.lod_schedule.resize(n_lods);
    for (uint32_t i = 0; i < n_lods; ++i) ds.lod_schedule[i] = static_cast<int>(c.get<uint32_t>());
    const uint64_t n_objects = c.get<uint64_t>();

    // Pass 1: object byte ranges from the length prefixes.
    std::vector<std::pair<size_t, size_t>> ranges;
    ranges.reserve(std::min<uint64_t>(n_objects, bytes.size() / 8 + 1));
    for (uint64_t oi = 0; oi < n_objects; ++oi) {
        c.where("object " + std::to_string(oi) + " header");
        const uint64_t len = c.get<uint64_t>();
        c.require(len);
        const size_t b = c.pos();
        ranges.emplace_back(b, b + len);
        c = Cursor(bytes, b + len, "object " + std::to_string(oi));
    }
    if (c.pos() != bytes.size()) throw IndexError("corrupt index: trailing bytes after last object");

    // Pass 2: decode objects in parallel.
    ds.objects.resize(n_objects);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nthreads = static_cast<unsigned>(std::min<uint64_t>(hw, std::max<uint64_t>(1, n_objects / 64)));
    std::atomic<uint64_t> next{0};
    std::exception_ptr first_error;
    uint64_t first_error_obj = UINT64_MAX;
    std::mutex mu;
    auto work = [&] {
        for (;;) {
            const uint64_t oi = next.fetch_add(1);
            if (oi >= n_objects) return;
            try {
                decode_object(bytes, ranges[oi].first, ranges[oi].second, oi, n_lods, ds.lod_schedule, ds.objects[oi]);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (oi < first_error_obj) {
                    first_error_obj = oi;
                    first_error = std::current_exception();
                }
            }
        }
    };
    if (nthreads <= 1) {
        work();
    } else {
        std::vector<std::thread> ts;
        for (unsigned t = 0; t < nthreads; ++t) ts.emplace_back(work);
        for (auto& t : ts) t.join();
    }
    if (first_error) std::rethrow_exception(first_error);
    return ds;
}

void save_index(const PreparedDataset& ds, const std::string& path) {
    const std::string bytes = serialize_index(ds);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw IndexError("cannot open " + path + " for writing");
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw IndexError("failed writing " + path);
}

PreparedDataset load_index(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw IndexError("cannot open " + path);
    std::string bytes;
    if (std::fseek(f, 0, SEEK_END) == 0) {
        const long n = std::ftell(f);
        if (n > 0) {
            bytes.resize(static_cast<size_t>(n));
            std::fseek(f, 0, SEEK_SET);
            const size_t got = std::fread(bytes.data(), 1, bytes.size(), f);
            bytes.resize(got);
        }
    }
    std::fclose(f);
    return deserialize_index(bytes);
}

} // namespace trijoin
