// trijoin mesh types — drop-in for the reference's proj/include/trijoin/mesh.hpp. The
// Hausdorff paddings (hd / ph) run on the GPU (csrc/preprocess.cu); OFF
// parsing and the edge-collapse simplifier of build_lod_ladder stay offline CPU tools.
#pragma once

#include <array>
#include <cstdint>
#include <span>
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

// Reference include/trijoin/mesh.hpp:65-73 (src/hausdorff.cpp:11-33, src/simplify.cpp:256-267),
// bitwise equal to the reference, computed on the GPU (tj_facet_hd_batch / tj_facet_ph_batch).
// (2/3) * longest_edge / grid_level: host arithmetic.
double hd_covering_radius(const Triangle& f_prime, int grid_level);
double compute_facet_hd(const Triangle& f_prime, const Mesh& original, int grid_level = 8);
double compute_facet_ph(uint32_t f_prime_id, const LodMesh& lod, const Mesh& original);

// Batched forms (one GPU pass): hd of every facet of `lod` against `original`; and the hd / ph
// fill of every level but the last of a ladder, as build_lod_ladder does after simplification
// (reference src/simplify.cpp:229-252; level 100 keeps hd = ph = 0).
std::vector<double> compute_facet_hd(const Mesh& lod, const Mesh& original, int grid_level = 8);
void fill_ladder_paddings(LodLadder& ladder, const Mesh& original, int hd_grid = 8);
// Many ladders at once (one launch per kernel for the whole set).
void fill_ladder_paddings(std::span<LodLadder* const> ladders, std::span<const Mesh* const> originals,
                          int hd_grid = 8);

} // namespace trijoin
