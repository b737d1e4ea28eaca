"""Generate the benchmark template indexes (run in the build container only).

TEST/BENCH INPUT TOOLING. Uses the reference's own generator and preprocessor
(`trijoin.generate` / `trijoin.preprocess` from the oracle/_ref build of
/root/reference/proj, proj/src/dataset.cpp:122-226, proj/src/voxelize.cpp:206-215) to
preprocess T copies of each builtin shape with the parameters of SURVEY.md §8(d):
lods=[20,60,100], voxel_ratio=0.02, hd_grid=8, seed=1. Each copy gets its own object id
and therefore its own k-means voxelisation seed. bench.py replicates these templates to
the full configuration sizes with `replicate_index` (translated copies), so the GPU box
needs neither /root/reference nor hours of preprocessing.

    python benchdata/make_templates.py      # writes benchdata/*.idx
"""
import os
import shutil
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "oracle", "_ref"))
import trijoin  # noqa: E402  (the reference module)

TEMPLATES = {
    # name: (shape, facets, scale, copies)
    "sphere300_s035": ("sphere", 300, 0.35, 16),   # nuclei (configs B, C, D)
    "sphere1000_s035": ("sphere", 1000, 0.35, 8),  # nuclei, config A
    "tube1000_s3": ("tube", 1000, 3.0, 8),         # vessels (configs A, C)
    "mixed20k": ("mixed", 20000, 1.0, 4),          # scanned-surface meshes, config E
}


def main():
    tmp = tempfile.mkdtemp()
    try:
        for name, (shape, facets, scale, copies) in TEMPLATES.items():
            d = os.path.join(tmp, name)
            trijoin.generate(d, shape=shape, facets=facets, scale=scale, count=copies, seed=1,
                             scatter_within=(0.0, 0.0, 0.0, 1000.0, 1000.0, 1000.0))
            out = os.path.join(HERE, name + ".idx")
            n = trijoin.preprocess(d, out, voxel_ratio=0.02, lods=[20, 60, 100], seed=1, hd_grid=8, workers=0)
            print(name, n, "objects", os.path.getsize(out), "bytes")
    finally:
        shutil.rmtree(tmp)


if __name__ == "__main__":
    main()
