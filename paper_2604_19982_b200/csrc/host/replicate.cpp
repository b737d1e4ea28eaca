// Index replicator (SURVEY.md §8d "Index replicator (for B-E)"): writes a 3DPJ1 index whose
// objects are translated copies of preprocessed template objects. Full preprocessing of
// the benchmark configurations would take CPU-hours; translated copies keep the real
// per-object LOD ladders, voxelisations and Hausdorff paddings. MBBs, voxel boxes and
// anchors are translated with the vertices (x -> fl(x + shift), monotone, so a translated
// min/max equals the min/max of the translated vertices). Non-zero hd/ph are padded by a
// few ulps of the coordinate magnitude so the bounds stay conservative after rounding;
// level-100 paddings stay exactly 0. Both the GPU engine and the reference CPU engine
// consume the same file, so parity is unaffected.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "replicate.hpp"

namespace trijoin {

namespace {

void shift_point(Point3& p, const Point3& s) {
    p.x += s.x;
    p.y += s.y;
    p.z += s.z;
}

} // namespace

PreparedObject replicated_object(const PreparedObject& src, const Point3& s, uint32_t id) {
    PreparedObject obj = src;
    obj.id = id;
    shift_point(obj.mbb.min, s);
    shift_point(obj.mbb.max, s);
    shift_point(obj.anchor, s);
    const double mag = std::max({std::fabs(obj.mbb.min.x), std::fabs(obj.mbb.min.y), std::fabs(obj.mbb.min.z),
                                 std::fabs(obj.mbb.max.x), std::fabs(obj.mbb.max.y), std::fabs(obj.mbb.max.z)});
    const double pad = std::ldexp(mag, -50); // ~4.4 ulp of the largest coordinate
    for (LodMesh& lod : obj.ladder.levels) {
        for (Point3& v : lod.mesh.vertices) shift_point(v, s);
        for (double& h : lod.hd)
            if (h != 0.0) h += pad;
        for (double& h : lod.ph)
            if (h != 0.0) h += pad;
    }
    for (Aabb& b : obj.voxels.boxes) {
        shift_point(b.min, s);
        shift_point(b.max, s);
    }
    for (Point3& a : obj.voxels.anchors) shift_point(a, s);
    return obj;
}

PreparedDataset replicate_dataset(const PreparedDataset& tmpl, std::span<const uint32_t> template_ids,
                                  std::span<const Point3> shifts, ThreadPool& pool) {
    if (template_ids.size() != shifts.size()) throw std::invalid_argument("replicate_dataset: size mismatch");
    for (uint32_t t : template_ids)
        if (t >= tmpl.objects.size()) throw std::invalid_argument("replicate_dataset: template id out of range");
    PreparedDataset out;
    out.lod_schedule = tmpl.lod_schedule;
    out.objects.resize(template_ids.size());
    pool.parallel_jobs(template_ids.size(), [&](size_t i) {
        out.objects[i] = replicated_object(tmpl.objects[template_ids[i]], shifts[i], static_cast<uint32_t>(i));
    });
    return out;
}

uint64_t replicate_index(const PreparedDataset& tmpl, const std::string& out_path,
                         std::span<const uint32_t> template_ids, std::span<const Point3> shifts) {
    if (template_ids.size() != shifts.size()) throw std::invalid_argument("replicate_index: size mismatch");
    for (uint32_t t : template_ids)
        if (t >= tmpl.objects.size()) throw std::invalid_argument("replicate_index: template id out of range");
    std::FILE* f = std::fopen(out_path.c_str(), "wb");
    if (!f) throw IndexError("cannot open " + out_path + " for writing");
    // header
    PreparedDataset header;
    header.lod_schedule = tmpl.lod_schedule;
    std::string head = serialize_index(header); // magic, version, lods, count = 0
    const uint64_t count = template_ids.size();
    std::memcpy(head.data() + head.size() - 8, &count, 8);
    uint64_t bytes = std::fwrite(head.data(), 1, head.size(), f);
    std::string body;
    for (size_t i = 0; i < template_ids.size(); ++i) {
        const PreparedObject obj = replicated_object(tmpl.objects[template_ids[i]], shifts[i], static_cast<uint32_t>(i));
        body.clear();
        serialize_object(obj, body);
        const uint64_t len = body.size();
        bytes += std::fwrite(&len, 1, 8, f);
        bytes += std::fwrite(body.data(), 1, body.size(), f);
    }
    if (std::fclose(f) != 0) throw IndexError("failed writing " + out_path);
    return bytes;
}

} // namespace trijoin
