// Benchmark input tooling: translated-copy index writer (see replicate.cpp).
#pragma once

#include <cstring>
#include <span>
#include <string>

#include "trijoin/index.hpp"

namespace trijoin {

// Appends one object's 3DPJ1 body (reference src/index_io.cpp:117-146 layout) to `body`.
void serialize_object(const PreparedObject& obj, std::string& body);

// Object i of the output = template_ids[i] translated by shifts[i]; returns bytes written.
uint64_t replicate_index(const PreparedDataset& tmpl, const std::string& out_path,
                         std::span<const uint32_t> template_ids, std::span<const Point3> shifts);

} // namespace trijoin
