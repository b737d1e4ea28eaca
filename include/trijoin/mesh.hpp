// trijoin mesh types — drop-in for the reference's proj/include/trijoin/mesh.hpp (types
// only: OFF parsing and LOD-ladder construction are offline preprocessing, out of scope).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "trijoin/geom.hpp"

namespace trijoin {

struct Mesh {
    std::vector<Point3> vertices;
    std::vector<std::array<uint32_t, 3>> facets;

    bool operator==(const Mesh&) const = default;

    Triangle triangle(size_t f) const {
        const auto& t = facets[f];
        return {vertices[t[0]], vertices[t[1]], vertices[t[2]]};
    }
    Aabb bounds() const {
        Aabb b = Aabb::empty();
        for (const Point3& v : vertices) b.expand(v);
        return b;
    }
};

// One level of detail: `level` is the percentage of the original facet count; hd / ph are
// the per-facet Hausdorff paddings of Eq. 1 / Eq. 2 (0 at level 100).
struct LodMesh {
    int level = 100;
    Mesh mesh;
    std::vector<double> hd;
    std::vector<double> ph;
    std::vector<uint32_t> ancestor_of_original;
    bool clamped = false;
};

struct LodLadder {
    std::vector<LodMesh> levels; // coarse -> fine; back() is level 100
};

} // namespace trijoin
