// TEST INFRASTRUCTURE (force-included into the reference's proj/tests/acceptance.cpp by
// `make -C tests/cpp acceptance`). The drop-in headers (include/trijoin/) declare the join
// path only; the reference's offline preprocessing tools the harness uses to build its
// datasets are linked from the reference build's own objects, declared here with the
// reference's signatures (proj/include/trijoin/index.hpp:63-65, mesh.hpp:58).
#pragma once
#include <vector>

#include "trijoin/index.hpp"
#include "trijoin/mesh.hpp"
#include "trijoin/parcore.hpp"

namespace trijoin {
PreparedDataset preprocess_dataset(const std::vector<Mesh>& meshes, const PreprocessParams& params, ThreadPool& pool);
LodLadder build_lod_ladder(const Mesh& mesh, const std::vector<int>& levels, int hd_grid = 8);
} // namespace trijoin
