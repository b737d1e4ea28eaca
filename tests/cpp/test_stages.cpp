// Stage-level C++ API of the drop-in, checked the way the reference's own doctest suites
// check it (proj/tests/test_filter.cpp, test_refine.cpp, test_knn.cpp, test_index.cpp,
// test_engine.cpp), plus the equivalence of the staged pipeline with run_join. Every
// stage runs on the GPU (csrc/stages.cu); run_join's own parity with the reference is
// established by tests/test_gpu_join.py. Usage: test_stages <golden dir>; exit 0 = pass.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <set>
#include <string>

#include "trijoin/engine.hpp"
#include "trijoin/knn.hpp"
#include "trijoin/refine.hpp"

using namespace trijoin;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                                    \
    do {                                                                            \
        ++g_checks;                                                                 \
        if (!(c)) {                                                                 \
            ++g_fail;                                                               \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);       \
        }                                                                           \
    } while (0)
#define REQUIRE(c)                                                                  \
    do {                                                                            \
        ++g_checks;                                                                 \
        if (!(c)) {                                                                 \
            std::fprintf(stderr, "FAIL (fatal) %s:%d: %s\n", __FILE__, __LINE__, #c); \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

namespace {

std::string G;
PreparedDataset load(const char* name) { return load_index(G + "/" + name); }

struct SplitMix {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double in(double a, double b) { return a + (b - a) * ((next() >> 11) * 0x1.0p-53); }
};

double box_gap(const Aabb& a, const Aabb& b) {
    const double gx = std::max({0.0, a.min.x - b.max.x, b.min.x - a.max.x});
    const double gy = std::max({0.0, a.min.y - b.max.y, b.min.y - a.max.y});
    const double gz = std::max({0.0, a.min.z - b.max.z, b.min.z - a.max.z});
    return std::sqrt(gx * gx + gy * gy + gz * gz);
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, 8) == 0; }

bool same_cands(const CandidateSet& a, const CandidateSet& b) {
    if (a.size() != b.size() || a.r2op_offsets != b.r2op_offsets || a.num_confirmed != b.num_confirmed) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (a.pairs[i] != b.pairs[i] || a.status[i] != b.status[i] || a.decided_at[i] != b.decided_at[i] ||
            !same_bits(a.intervals[i].lb, b.intervals[i].lb) || !same_bits(a.intervals[i].ub, b.intervals[i].ub))
            return false;
    return true;
}

// ---- test_index.cpp:150-180: STR tree shape and containment
void rtree_structure() {
    std::vector<PreparedObject> objs(1600);
    SplitMix rng{77};
    for (uint32_t i = 0; i < objs.size(); ++i) {
        objs[i].id = i;
        const Point3 c{rng.in(-50, 50), rng.in(-50, 50), rng.in(-50, 50)};
        objs[i].mbb = {c - Point3{1, 1, 1}, c + Point3{1, 1, 1}};
    }
    const RTree tree = build_rtree(objs);
    CHECK(tree.node_levels == 3); // 1600 -> 100 leaves -> 7 -> root
    std::vector<uint32_t> e = tree.entries;
    std::sort(e.begin(), e.end());
    REQUIRE(e.size() == objs.size());
    for (uint32_t i = 0; i < e.size(); ++i) CHECK(e[i] == i);
    for (const RTree::Node& n : tree.nodes) {
        if (n.leaf) {
            for (uint32_t x = n.first; x < n.first + n.count; ++x) {
                const Aabb& m = objs[tree.entries[x]].mbb;
                CHECK(box_gap(n.box, m) == 0.0 && n.box.min.x <= m.min.x && n.box.max.x >= m.max.x);
            }
        } else {
            for (uint32_t c = n.first; c < n.first + n.count; ++c)
                CHECK(n.box.min.x <= tree.nodes[c].box.min.x && n.box.max.y >= tree.nodes[c].box.max.y &&
                      n.box.max.z >= tree.nodes[c].box.max.z);
        }
    }
    CHECK(build_rtree(std::span<const PreparedObject>{}).empty());
}

// ---- test_filter.cpp:40-76: mbb_filter_within keeps exactly the box-reachable pairs
void mbb_within_exact(const PreparedDataset& ds) {
    ThreadPool pool(2);
    const RTree tree = build_rtree(ds.objects);
    for (double tau : {0.0, 0.6, 2.0, 50.0}) {
        CandidateSet c = mbb_filter_within(ds, ds, tree, tau, pool);
        std::map<std::pair<uint32_t, uint32_t>, size_t> at;
        for (size_t i = 0; i < c.size(); ++i) at[c.pairs[i]] = i;
        for (uint32_t r = 0; r < ds.objects.size(); ++r)
            for (uint32_t s = 0; s < ds.objects.size(); ++s) {
                const double gap = mindist_aabb(ds.objects[r].mbb, ds.objects[s].mbb);
                CHECK(at.count({r, s}) == (gap <= tau ? 1u : 0u));
                if (gap <= tau) {
                    const Interval& iv = c.intervals[at[{r, s}]];
                    CHECK(iv.lb >= gap && iv.lb <= iv.ub);
                    CHECK(iv.ub <= distance(ds.objects[r].anchor, ds.objects[s].anchor) + 1e-12);
                }
            }
        CHECK(c.r2op_offsets.size() == ds.objects.size() + 1);
        for (uint32_t r = 0; r < ds.objects.size(); ++r)
            for (uint64_t op = c.r2op_offsets[r]; op < c.r2op_offsets[r + 1]; ++op) CHECK(c.pairs[op].first == r);
        for (size_t i = 0; i < c.size(); ++i) {
            if (c.status[i] == PairStatus::Confirmed)
                CHECK(c.intervals[i].ub <= tau && c.decided_at[i] == stage::kMbb);
            else
                CHECK(c.status[i] == PairStatus::Undecided);
        }
    }
}

// ---- SURVEY §8a row a3 (closed form of the reference's best-first search): candidates(r)
// = {s : mindist <= u_k(r)}, u_k(r) the k-th smallest anchor distance over S
void mbb_knn_closed_form(const PreparedDataset& ds) {
    ThreadPool pool(2);
    const RTree tree = build_rtree(ds.objects);
    for (uint32_t k : {1u, 3u, 5u}) {
        const CandidateSet c = mbb_filter_knn(ds, ds, tree, k, pool);
        for (uint32_t r = 0; r < ds.objects.size(); ++r) {
            std::vector<double> ad;
            for (const auto& o : ds.objects) ad.push_back(distance(ds.objects[r].anchor, o.anchor));
            std::nth_element(ad.begin(), ad.begin() + (k - 1), ad.end());
            const double uk = ad[k - 1];
            std::set<uint32_t> want, got;
            for (uint32_t s = 0; s < ds.objects.size(); ++s)
                if (mindist_aabb(ds.objects[r].mbb, ds.objects[s].mbb) <= uk) want.insert(s);
            for (uint64_t op = c.r2op_offsets[r]; op < c.r2op_offsets[r + 1]; ++op) {
                got.insert(c.pairs[op].second);
                CHECK(c.status[op] == PairStatus::Undecided);
            }
            CHECK(got == want);
            CHECK(got.size() >= k);
        }
    }
}

// ---- test_filter.cpp:166-205: chunked_filter results are invariant to budget and pipeline;
// per-chunk bounds + compaction reproduce them
void chunk_invariance(const PreparedDataset& ds) {
    ThreadPool pool(2);
    const RTree tree = build_rtree(ds.objects);
    const CandidateSet base = mbb_filter_within(ds, ds, tree, 2.5, pool);
    CandidateSet ref = base;
    FilterStats rs;
    const VoxelPairList rl = chunked_filter(ref, ds, ds, UINT64_MAX, 2.5, false, pool, &rs);
    for (uint64_t budget : {1ull, 64ull, 4194304ull})
        for (bool pipe : {false, true}) {
            CandidateSet c = base;
            FilterStats st;
            const VoxelPairList l = chunked_filter(c, ds, ds, budget, 2.5, pipe, pool, &st);
            CHECK(same_cands(c, ref));
            CHECK(l.op_offsets == rl.op_offsets && l.vpairs == rl.vpairs);
            CHECK(st.vp_generated == rs.vp_generated && st.vp_pruned == rs.vp_pruned);
            if (budget == 1) CHECK(st.chunks == base.undecided_count());
        }
    CHECK(rs.vp_generated >= rs.vp_pruned);
    // one chunk of all undecided ops through the per-chunk stages
    CandidateSet c = base;
    FilterChunk ch;
    ch.vp_offsets.push_back(0);
    for (uint32_t op = 0; op < c.size(); ++op)
        if (c.status[op] == PairStatus::Undecided) {
            ch.ops.push_back(op);
            ch.vp_offsets.push_back(ch.total_vp() + voxel_pair_count(c, op, ds, ds));
        }
    const ChunkBounds b = voxel_pair_bounds(ch, c, ds, ds, pool);
    for (size_t ci = 0; ci < ch.ops.size(); ++ci) { // op minima of the materialised bounds
        double mlb = INFINITY, mub = INFINITY;
        for (uint64_t t = ch.vp_offsets[ci]; t < ch.vp_offsets[ci + 1]; ++t) {
            mlb = std::min(mlb, b.vp_lb[t]);
            mub = std::min(mub, b.vp_ub[t]);
        }
        CHECK(same_bits(mlb, b.op_lb[ci]) && same_bits(mub, b.op_ub[ci]));
    }
    prune_within(c, 2.5, stage::kVoxel, ch.ops);
    const auto surv = voxel_pair_compact(ch, b, c, ds, ds, pool);
    CHECK(same_cands(c, ref));
    CHECK(surv.size() == rl.vpairs.size());
    for (size_t i = 0; i < surv.size() && i < rl.vpairs.size(); ++i) {
        const auto [op, vr, vs] = surv[i];
        CHECK(rl.vpairs[i] == std::make_pair(vr, vs));
        CHECK(i >= rl.op_offsets[op] && i < rl.op_offsets[op + 1]);
    }
    // test_filter.cpp:207-239: a pruned voxel pair's lb is its box gap, above the op's ub
    int pruned_seen = 0;
    JoinTrace tr;
    tr.on_vp_pruned = [&](uint32_t op, uint32_t vr, uint32_t vs, double lb_v, double ub_o) {
        const auto [r, s] = base.pairs[op];
        CHECK(same_bits(lb_v, mindist_aabb(ds.objects[r].voxels.boxes[vr], ds.objects[s].voxels.boxes[vs])));
        CHECK(lb_v > ub_o);
        ++pruned_seen;
    };
    CandidateSet c2 = base;
    FilterStats st2;
    chunked_filter(c2, ds, ds, 4194304, 2.5, true, pool, &st2, &tr);
    CHECK((uint64_t)pruned_seen == st2.vp_pruned);
}

JoinOutput staged_join(const PreparedDataset& R, const PreparedDataset& S, const JoinSpec& spec) {
    // run_join's stage sequence (reference src/engine.cpp:122-237) through the stage API
    ThreadPool pool(2);
    const RTree tree = build_rtree(S.objects);
    const bool knn = spec.type == JoinType::Knn;
    const double tau = spec.type == JoinType::Intersect ? 0.0 : spec.tau;
    CandidateSet c = knn ? mbb_filter_knn(R, S, tree, spec.k, pool) : mbb_filter_within(R, S, tree, tau, pool);
    KnnState st;
    if (knn) {
        st = make_knn_state(c, spec.k);
        knn_prune_to_fixpoint(st, c, stage::kMbb, pool);
    }
    const VoxelPairList vl =
        chunked_filter(c, R, S, spec.filter_chunk, knn ? std::nullopt : std::optional<double>(tau), true, pool);
    if (knn) knn_prune_to_fixpoint(st, c, stage::kVoxel, pool);
    RefineConfig cfg;
    cfg.lods = spec.lods;
    cfg.chunk = spec.refine_chunk;
    if (knn)
        knn_resolve(st, c, vl, R, S, cfg, pool);
    else
        refine_loop(c, vl, R, S, cfg, tau, nullptr, pool);
    JoinOutput out;
    if (!knn) {
        for (uint32_t op = 0; op < c.size(); ++op)
            if (c.status[op] == PairStatus::Confirmed)
                out.records.push_back({c.pairs[op].first, c.pairs[op].second, c.intervals[op].lb, c.intervals[op].ub,
                                       c.decided_at[op], 0});
    } else {
        for (uint32_t r = 0; r + 1 < c.r2op_offsets.size(); ++r) {
            std::vector<uint32_t> conf;
            for (uint64_t op = c.r2op_offsets[r]; op < c.r2op_offsets[r + 1]; ++op)
                if (c.status[op] == PairStatus::Confirmed) conf.push_back((uint32_t)op);
            std::sort(conf.begin(), conf.end(), [&](uint32_t a, uint32_t b) {
                if (c.intervals[a].ub != c.intervals[b].ub) return c.intervals[a].ub < c.intervals[b].ub;
                if (c.intervals[a].lb != c.intervals[b].lb) return c.intervals[a].lb < c.intervals[b].lb;
                return c.pairs[a].second < c.pairs[b].second;
            });
            uint32_t rank = 0;
            for (uint32_t op : conf)
                out.records.push_back({r, c.pairs[op].second, c.intervals[op].lb, c.intervals[op].ub,
                                       c.decided_at[op], ++rank});
        }
    }
    return out;
}

// ---- the staged pipeline equals run_join (records bit-identical; test_engine.cpp:105-178)
void staged_equals_run_join(const PreparedDataset& R, const PreparedDataset& S, JoinSpec spec) {
    ThreadPool pool(2);
    spec.lods = {20, 60, 100};
    const JoinOutput a = run_join(R, S, spec, pool);
    const JoinOutput b = staged_join(R, S, spec);
    CHECK(format_records(a.records, spec.type == JoinType::Knn) == format_records(b.records, spec.type == JoinType::Knn));
}

// ---- StageResidency (extension): chained stage calls on device copies pinned once give the
// same records as the per-call uploads (and as run_join); scopes nest and share datasets
void staged_with_residency(const PreparedDataset& R, const PreparedDataset& S, JoinSpec spec) {
    spec.lods = {20, 60, 100};
    const JoinOutput a = staged_join(R, S, spec);
    StageResidency outer(R, S);
    {
        StageResidency inner(R, R); // nested, sharing R
        const JoinOutput b = staged_join(R, S, spec);
        CHECK(format_records(a.records, spec.type == JoinType::Knn) == format_records(b.records, spec.type == JoinType::Knn));
    }
    const JoinOutput c = staged_join(R, S, spec);
    CHECK(format_records(a.records, spec.type == JoinType::Knn) == format_records(c.records, spec.type == JoinType::Knn));
}

// ---- test_refine.cpp:183-218: refine_loop results independent of chunk and pipeline
void refine_chunk_invariance(const PreparedDataset& ds) {
    ThreadPool pool(2);
    const RTree tree = build_rtree(ds.objects);
    CandidateSet c0 = mbb_filter_within(ds, ds, tree, 1.3, pool);
    const VoxelPairList vl = chunked_filter(c0, ds, ds, 4194304, 1.3, true, pool);
    CandidateSet ref;
    for (uint64_t chunk : {1ull, 100ull, 500000ull})
        for (bool pipe : {true, false}) {
            CandidateSet c = c0;
            RefineConfig cfg;
            cfg.lods = {20, 60, 100};
            cfg.chunk = chunk;
            cfg.pipeline = pipe;
            RefineStats stats;
            refine_loop(c, vl, ds, ds, cfg, 1.3, nullptr, pool, &stats);
            CHECK(c.undecided_count() == 0);
            CHECK(stats.levels.size() >= 1 && stats.levels.front().level == 20);
            if (ref.size() == 0) ref = c;
            CHECK(same_cands(c, ref));
        }
    // exactly one of tau / knn (src/refine.cpp:264-265)
    bool threw = false;
    try {
        CandidateSet c = c0;
        RefineConfig cfg;
        refine_loop(c, vl, ds, ds, cfg, std::nullopt, nullptr, pool);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
}

// ---- test_knn.cpp: the strict snapshot rules
CandidateSet single_query(const std::vector<Interval>& iv) {
    CandidateSet c;
    for (uint32_t s = 0; s < iv.size(); ++s) c.pairs.emplace_back(0, s);
    c.intervals = iv;
    c.status.assign(iv.size(), PairStatus::Undecided);
    c.decided_at.assign(iv.size(), stage::kNone);
    c.r2op_offsets = {0, iv.size()};
    c.num_confirmed = {0};
    return c;
}

void knn_rules() {
    ThreadPool pool(2);
    { // test_knn.cpp:85-101
        CandidateSet c = single_query({{5, 9}, {6, 10}, {8, 12}, {1, 4}});
        KnnState st = make_knn_state(c, 2);
        const auto d = knn_prune_round(st, c, pool);
        REQUIRE(d.size() == 1);
        CHECK(d[0].op == 3 && d[0].status == PairStatus::Confirmed);
        knn_apply_deltas(st, c, d, stage::kMbb);
        CHECK(st.num_confirmed[0] == 1);
        knn_prune_to_fixpoint(st, c, stage::kMbb, pool);
        CHECK(c.status[0] == PairStatus::Undecided && c.status[1] == PairStatus::Undecided &&
              c.status[2] == PairStatus::Undecided);
    }
    { // :103-115
        CandidateSet c = single_query({{1, 2}, {3, 4}});
        KnnState st = make_knn_state(c, 1);
        CHECK(knn_prune_to_fixpoint(st, c, 55, pool) == 2);
        CHECK(c.status[0] == PairStatus::Confirmed && c.status[1] == PairStatus::Removed);
        CHECK(c.decided_at[0] == 55 && c.decided_at[1] == 55 && c.num_confirmed[0] == 1);
    }
    { // :117-123
        CandidateSet c = single_query({{1, 2}, {3, 4}, {5, 6}});
        KnnState st = make_knn_state(c, 9);
        knn_prune_to_fixpoint(st, c, stage::kMbb, pool);
        for (auto s : c.status) CHECK(s == PairStatus::Confirmed);
    }
    { // finalize fills by (lb, s) and removes the rest
        CandidateSet c = single_query({{2, 2}, {1, 1}, {1, 1}, {3, 3}});
        KnnState st = make_knn_state(c, 2);
        knn_finalize(st, c);
        CHECK(c.status[1] == PairStatus::Confirmed && c.status[2] == PairStatus::Confirmed);
        CHECK(c.status[0] == PairStatus::Removed && c.status[3] == PairStatus::Removed);
        CHECK(c.decided_at[0] == 100 && st.num_confirmed[0] == 2 && c.num_confirmed[0] == 2);
    }
    { // random multi-query sets against a sequential restatement of the round rule
        SplitMix rng{2024};
        CandidateSet c;
        c.r2op_offsets.push_back(0);
        for (uint32_t r = 0; r < 40; ++r) {
            for (uint32_t s = 0; s < 12; ++s) {
                const double d = rng.in(0, 10), lo = d - rng.in(0, 2), hi = d + rng.in(0, 2);
                c.pairs.emplace_back(r, s);
                c.intervals.push_back({std::max(0.0, lo), hi});
            }
            c.r2op_offsets.push_back(c.pairs.size());
        }
        c.status.assign(c.pairs.size(), PairStatus::Undecided);
        c.decided_at.assign(c.pairs.size(), stage::kNone);
        c.num_confirmed.assign(40, 0);
        for (uint32_t k : {1u, 3u}) {
            CandidateSet a = c, b = c;
            KnnState st = make_knn_state(a, k);
            knn_prune_to_fixpoint(st, a, 7, pool);
            // sequential mirror (test_knn.cpp:48-78)
            std::vector<uint32_t> conf(40, 0);
            for (bool changed = true; changed;) {
                changed = false;
                std::vector<std::pair<uint32_t, PairStatus>> ds;
                for (uint32_t r = 0; r < 40; ++r) {
                    std::vector<uint32_t> u;
                    for (uint64_t op = b.r2op_offsets[r]; op < b.r2op_offsets[r + 1]; ++op)
                        if (b.status[op] == PairStatus::Undecided) u.push_back((uint32_t)op);
                    const uint32_t kl = k - conf[r];
                    for (uint32_t m : u) {
                        size_t far = 0, close = 0;
                        for (uint32_t n : u) {
                            if (n == m) continue;
                            far += b.intervals[n].lb > b.intervals[m].ub;
                            close += b.intervals[n].ub < b.intervals[m].lb;
                        }
                        if ((u.size() - 1) - far < kl) ds.emplace_back(m, PairStatus::Confirmed);
                        else if (close >= kl) ds.emplace_back(m, PairStatus::Removed);
                    }
                }
                for (auto [op, s] : ds) {
                    b.status[op] = s;
                    if (s == PairStatus::Confirmed) ++conf[b.pairs[op].first];
                    changed = true;
                }
            }
            CHECK(a.status == b.status);
            CHECK(st.num_confirmed == conf);
        }
    }
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: test_stages <golden dir>\n");
        return 2;
    }
    G = argv[1];
    rtree_structure();
    knn_rules();
    const PreparedDataset m12 = load("mini12_s31.idx"), m14 = load("mini14_s53.idx"), m10 = load("mini10_s61.idx");
    mbb_within_exact(m12);
    mbb_knn_closed_form(m14);
    chunk_invariance(m10);
    refine_chunk_invariance(m10);
    const PreparedDataset nuc = load("nuclei60.idx"), ves = load("vessels8.idx"), m18 = load("mini18_s21.idx");
    for (double tau : {0.0, 0.4, 1.6, 3.0}) {
        JoinSpec s;
        s.type = JoinType::Within;
        s.tau = tau;
        staged_equals_run_join(m18, m18, s);
    }
    for (uint32_t k : {1u, 3u}) {
        JoinSpec s;
        s.type = JoinType::Knn;
        s.k = k;
        staged_equals_run_join(m14, m14, s);
        staged_equals_run_join(nuc, ves, s);
        staged_with_residency(nuc, ves, s);
    }
    {
        JoinSpec s;
        s.type = JoinType::Within;
        s.tau = 0.5;
        s.filter_chunk = 64;
        staged_equals_run_join(nuc, ves, s);
        s.type = JoinType::Intersect;
        s.tau = 0.0;
        staged_equals_run_join(nuc, ves, s);
        staged_with_residency(nuc, ves, s);
    }
    std::printf("test_stages: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
