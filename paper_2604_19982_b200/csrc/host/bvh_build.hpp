// Host construction of the reference's triangle BVH (src/bvh.cpp:19-80, TriBvh) for the GPU
// point-to-mesh queries of csrc/preprocess.cu. Restated, not transcribed: each node splits its
// range at (n / 2) under the (centroid on the longest box axis, facet id) total order of
// src/bvh.cpp:66-75 — the reference's nth_element yields the same two *sets*, so node boxes,
// leaf sets and the tree shape are identical (only the order inside a leaf may differ, which a
// minimum over the leaf ignores). Nodes are numbered in preorder like the reference's.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

namespace tjx::bvh {

constexpr uint32_t kLeafSize = 4;  // src/bvh.cpp:9

struct BvhNode {
    double lo[3], hi[3];
    uint32_t left, count, right, pad; // internal: children; leaf: first triangle (leaf order), count
};

// ---------------------------------------------------------------- host: tree construction
struct HostBvh {
    std::vector<BvhNode> nodes;
    std::vector<uint32_t> order; // leaf order -> facet id
};

struct TriSoup {
    const double* v;       // mesh vertices (3 per vertex)
    const uint32_t* f;     // mesh-local vertex ids (3 per facet)
    double coord(uint32_t t, int k, int d) const { return v[3 * (size_t)f[3 * (size_t)t + k] + d]; }
};

inline void build_node(HostBvh& h, const TriSoup& s, const std::vector<double>& cen, size_t begin, size_t end) {
    const uint32_t index = (uint32_t)h.nodes.size();
    h.nodes.emplace_back();
    BvhNode box{};
    for (int d = 0; d < 3; ++d) {
        box.lo[d] = INFINITY;
        box.hi[d] = -INFINITY;
    }
    for (size_t i = begin; i < end; ++i)
        for (int k = 0; k < 3; ++k)
            for (int d = 0; d < 3; ++d) { // Aabb::expand: std::min / std::max
                const double c = s.coord(h.order[i], k, d);
                box.lo[d] = c < box.lo[d] ? c : box.lo[d];
                box.hi[d] = box.hi[d] < c ? c : box.hi[d];
            }
    if (end - begin <= kLeafSize) {
        box.left = (uint32_t)begin;
        box.count = (uint32_t)(end - begin);
        h.nodes[index] = box;
        return;
    }
    const double ex = box.hi[0] - box.lo[0], ey = box.hi[1] - box.lo[1], ez = box.hi[2] - box.lo[2];
    int axis = 0;
    if (ey > ex) axis = 1;
    if (ez > (axis == 0 ? ex : ey)) axis = 2;
    const size_t mid = begin + (end - begin) / 2;
    // the set of the first (end - begin) / 2 elements under the (centroid, id) total order: any
    // selection under a total order yields the same set as the reference's nth_element
    std::nth_element(h.order.begin() + begin, h.order.begin() + mid, h.order.begin() + end, [&](uint32_t a, uint32_t b) {
        const double ca = cen[3 * (size_t)a + axis], cb = cen[3 * (size_t)b + axis];
        if (ca != cb) return ca < cb;
        return a < b;
    });
    h.nodes[index] = box;
    build_node(h, s, cen, begin, mid);
    const uint32_t r = (uint32_t)h.nodes.size();
    build_node(h, s, cen, mid, end);
    h.nodes[index].left = index + 1; // preorder: the left child follows its parent
    h.nodes[index].right = r;
    h.nodes[index].count = 0;
}

inline HostBvh build_bvh(const TriSoup& s, uint32_t nf) {
    HostBvh h;
    h.order.resize(nf);
    std::iota(h.order.begin(), h.order.end(), 0u);
    if (!nf) return h;
    std::vector<double> cen(3 * (size_t)nf);
    for (uint32_t t = 0; t < nf; ++t)
        for (int d = 0; d < 3; ++d) // Triangle::centroid: (v0 + v1 + v2) * (1 / 3)
            cen[3 * (size_t)t + d] = ((s.coord(t, 0, d) + s.coord(t, 1, d)) + s.coord(t, 2, d)) * (1.0 / 3.0);
    h.nodes.reserve(2 * (size_t)nf / kLeafSize + 2);
    build_node(h, s, cen, 0, nf);
    return h;
}

} // namespace tjx::bvh
