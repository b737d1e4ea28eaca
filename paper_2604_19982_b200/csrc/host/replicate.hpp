// Benchmark input tooling: translated-copy index writer (see replicate.cpp).
#pragma once

#include <cstring>
#include <span>
#include <string>

#include "trijoin/index.hpp"
#include "trijoin/parcore.hpp"

namespace trijoin {

// Appends one object's 3DPJ1 body (reference src/index_io.cpp:117-146 layout) to `body`.
void serialize_object(const PreparedObject& obj, std::string& body);

// A template object translated by s (MBB, anchors, voxel boxes and vertices; non-zero hd / ph
// padded by a few ulps of the coordinate magnitude), renumbered to id.
PreparedObject replicated_object(const PreparedObject& src, const Point3& s, uint32_t id);

// The same translated copies in memory (no index file): object i = template_ids[i] shifted.
PreparedDataset replicate_dataset(const PreparedDataset& tmpl, std::span<const uint32_t> template_ids,
                                  std::span<const Point3> shifts, ThreadPool& pool);

// Object i of the output = template_ids[i] translated by shifts[i]; returns bytes written.
uint64_t replicate_index(const PreparedDataset& tmpl, const std::string& out_path,
                         std::span<const uint32_t> template_ids, std::span<const Point3> shifts);

} // namespace trijoin
