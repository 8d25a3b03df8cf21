// shim_test.cpp -- the C++ drop-in (include/srm/b200/engine.hpp) driven with the
// reference's own types, compared against the reference's own functions where the two
// are defined to agree (RSA, reorder_by_locality, shape_any_collision) and checked
// against the engine-level cases of test_engine.cpp where they are not (generate).
// Built by `make shimtest` (needs /root/reference headers at build time only); run by
// tests/test_gpu_shim.py on a GPU.
#include <cmath>
#include <cstdio>
#include <numbers>
#include <stdexcept>
#include <string>
#include <vector>

#include "srm/b200/engine.hpp"
#include "srm/descriptors.hpp"
#include "srm/engine.hpp"
#include "srm/recipes.hpp"
#include "srm/rsa.hpp"

using namespace srm;

static int failures = 0, checks = 0;
#define CHECK(cond)                                                       \
    do {                                                                  \
        ++checks;                                                         \
        if (!(cond)) {                                                    \
            ++failures;                                                   \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                 \
    } while (0)

template <int N>
static std::size_t violations(const std::vector<Particle<N>>& ps, const PeriodicBox<N>& box, double rel_tol) {
    std::size_t bad = 0;
    for (std::size_t i = 0; i < ps.size(); ++i)
        for (std::size_t j = i + 1; j < ps.size(); ++j) {
            Vec<N> d = ps[i].pos - ps[j].pos;
            for (int a = 0; a < N; ++a) d[a] -= box.length(a) * std::nearbyint(d[a] / box.length(a));
            if (d.norm() < (ps[i].radius + ps[j].radius) * (1.0 - rel_tol)) ++bad;
        }
    return bad;
}

static Snapshot<DiskShape> disk_start(std::size_t n, double f0, std::uint64_t seed) {
    Snapshot<DiskShape> snap;
    snap.box = PeriodicBox2::unit();
    const double r = std::sqrt(f0 / (static_cast<double>(n) * std::numbers::pi));
    Rng rng(seed);
    snap.particles = srm::rsa_place<2>(n, r, snap.box, kRsaDefaultAttempts, rng);
    snap.refresh_volume_fraction();
    return snap;
}

int main() {
    // rsa_place: bit-identical to the reference for a fresh Rng(seed)
    {
        const auto box = PeriodicBox3::unit();
        std::vector<double> radii(3000, 0.02);
        Rng rng(77);
        const auto ref = srm::rsa_place<3>(radii, box, kRsaDefaultAttempts, rng);
        const auto mine = srm::b200::rsa_place<3>(radii, box, kRsaDefaultAttempts, 77);
        bool same = ref.size() == mine.size();
        for (std::size_t i = 0; same && i < ref.size(); ++i)
            same = ref[i].id == mine[i].id && ref[i].pos == mine[i].pos && ref[i].radius == mine[i].radius;
        CHECK(same);
    }
    // srm_generate: test_engine.cpp:144-159 on the device
    {
        auto snap = disk_start(100, 0.1, 42);
        SrmParams p;
        p.c_w = 0.05;
        p.c_m = 0.01;
        p.n_k = 8;
        p.n_l = 8;
        p.f_target = 0.5;
        p.seed = 7;
        std::int64_t calls = 0;
        const auto res = srm::b200::srm_generate<DiskShape>(snap, p, [&](const ProgressRecord& r) {
            ++calls;
            CHECK(r.iteration == calls);
        });
        CHECK(res.status == GenerateStatus::Converged);
        CHECK(res.snapshot.volume_fraction >= 0.5 * (1.0 - 1e-12));
        CHECK(res.snapshot.volume_fraction <= 0.5 * (1.0 + 1e-9));
        CHECK(violations<2>(res.snapshot.particles, snap.box, 1e-12) == 0);
        CHECK(res.snapshot.iteration_count == calls);
        CHECK(res.snapshot.seed == 7);
    }
    // generate in 3d (test_engine.cpp:161-178)
    {
        Snapshot<BallShape> snap;
        snap.box = PeriodicBox3::unit();
        const double r = std::cbrt(0.05 * 3.0 / (100 * 4.0 * std::numbers::pi));
        Rng rng(11);
        snap.particles = srm::rsa_place<3>(100, r, snap.box, kRsaDefaultAttempts, rng);
        snap.refresh_volume_fraction();
        SrmParams p;
        p.c_w = 0.05;
        p.c_m = 0.02;
        p.f_target = 0.3;
        p.seed = 3;
        const auto res = srm::b200::srm_generate<BallShape>(snap, p);
        CHECK(res.status == GenerateStatus::Converged);
        CHECK(violations<3>(res.snapshot.particles, snap.box, 1e-12) == 0);
    }
    // iteration budget and validation (test_engine.cpp:206-273)
    {
        auto snap = disk_start(100, 0.1, 12);
        SrmParams p;
        p.c_w = 0.001;
        p.c_m = 0.01;
        p.max_iterations = 5;
        const auto res = srm::b200::srm_generate<DiskShape>(snap, p);
        CHECK(res.status == GenerateStatus::IterationLimitExceeded);
        CHECK(res.snapshot.iteration_count == 5);
        SrmParams bad;
        bad.c_w = 0.26;
        bool threw = false;
        try {
            srm::b200::srm_generate<DiskShape>(snap, bad);
        } catch (const ValidationError&) {
            threw = true;
        }
        CHECK(threw);
    }
    // reorder_by_locality and shape_any_collision equal the reference's
    {
        const auto box = PeriodicBox2::unit();
        auto snap = disk_start(2000, 0.3, 5);
        CellGrid<2> grid(box, 0.03);
        grid.build(snap.particles);
        auto a = snap.particles, b = snap.particles;
        const auto ra = srm::reorder_by_locality<DiskShape>(a, grid);
        const auto rb = srm::b200::reorder_by_locality<DiskShape>(b, grid);
        CHECK(ra == rb);
        bool same = true;
        for (std::size_t i = 0; i < a.size(); ++i) same = same && a[i].pos == b[i].pos && a[i].id == b[i].id;
        CHECK(same);
        CHECK(srm::b200::shape_any_collision<DiskShape>(snap.particles, grid) ==
              srm::shape_any_collision<DiskShape>(snap.particles, grid));
        auto over = snap.particles;
        over[1].pos = over[0].pos;
        grid.build(over);
        CHECK(srm::b200::shape_any_collision<DiskShape>(over, grid));
        CHECK(srm::shape_any_collision<DiskShape>(over, grid));
    }
    // migrate keeps validity; relax with zero step is the identity
    {
        auto snap = disk_start(300, 0.3, 21);
        const double max_r = max_bounding_radius<DiskShape>(snap.particles);
        CellGrid<2> grid(snap.box, 2.5 * max_r + 0.01, max_r, 0.01);
        Rng rng(2);
        const auto acc = srm::b200::migrate<DiskShape>(snap.particles, grid, 0.01, 0.0, 8, rng);
        std::size_t moved = 0;
        for (auto v : acc) moved += v;
        CHECK(moved > 0);
        CHECK(violations<2>(snap.particles, snap.box, 0.0) == 0);
        auto before = snap.particles;
        srm::b200::relax_sweeps<DiskShape>(snap.particles, snap.box, 0.0, 0.0, 4, 3, rng);
        bool same = true;
        for (std::size_t i = 0; i < before.size(); ++i) same = same && before[i].pos == snap.particles[i].pos;
        CHECK(same);
    }
    // nearest_neighbor_distances on the device: bit-identical to the reference's
    {
        auto snap = disk_start(500, 0.35, 31);
        const auto mine = srm::b200::nearest_neighbor_distances(snap);
        const auto ref = srm::nearest_neighbor_distances(snap);
        CHECK(mine.size() == ref.size());
        bool same = mine.size() == ref.size();
        for (std::size_t i = 0; same && i < ref.size(); ++i) same = mine[i] == ref[i];
        CHECK(same);
    }
    // local_nematic_order on the device: the reference's neighbour counts, values to rounding
    {
        const PeriodicBox3 box = PeriodicBox3::cube(8.0);
        Rng rng(17);
        const auto snap = srm::rsa_platelets(600, 1.0, 20.0, box, 100000, rng);
        const auto ref = srm::local_nematic_order(snap, 1.5);
        const auto mine = srm::b200::local_nematic_order(snap, 1.5);
        bool same = ref.value.size() == mine.value.size();
        for (std::size_t i = 0; same && i < ref.value.size(); ++i) {
            same = ref.neighbor_count[i] == mine.neighbor_count[i];
            if (ref.neighbor_count[i] > 0)
                same = same && std::fabs(ref.value[i] - mine.value[i]) <= 1e-12 * std::fabs(ref.value[i]);
            else
                same = same && std::isnan(mine.value[i]);
        }
        CHECK(same);
        bool threw = false;
        try {
            srm::b200::local_nematic_order(snap, 0.0);
        } catch (const ValidationError&) {
            threw = true;
        }
        CHECK(threw);
    }
    // platelets (SpherodiskShape): rsa_platelets bit-identical to the reference's for
    // Rng(seed); srm_generate to a target fraction, no overlap by the reference's own test
    {
        const PeriodicBox3 box = PeriodicBox3::cube(6.0);
        Rng rng(5);
        const auto ref = srm::rsa_platelets(120, 1.0, 20.0, box, 10000, rng);
        const auto mine = srm::b200::rsa_platelets(120, 1.0, 20.0, box, 10000, 5);
        bool same = ref.particles.size() == mine.particles.size();
        for (std::size_t i = 0; same && i < ref.particles.size(); ++i)
            same = ref.particles[i].pos == mine.particles[i].pos && ref.particles[i].normal == mine.particles[i].normal;
        CHECK(same);
        SrmParams p;
        p.c_w = 0.01;
        p.c_m = 0.05;
        p.c_r = 0.05;
        p.n_k = 10;
        p.n_l = 10;
        p.f_target = 1.2 * mine.volume_fraction;
        p.seed = 9;
        const auto res = srm::b200::srm_generate(mine, p);
        CHECK(res.status == GenerateStatus::Converged);
        CHECK(res.snapshot.volume_fraction >= p.f_target * (1.0 - 1e-12));
        const double max_r = max_bounding_radius<SpherodiskShape>(res.snapshot.particles);
        CellGrid<3> grid(box, 2.5 * max_r);
        build_shape_grid<SpherodiskShape>(grid, res.snapshot.particles);
        CHECK(!srm::shape_any_collision<SpherodiskShape>(std::span<const Spherodisk>(res.snapshot.particles), grid));
        CHECK(!srm::b200::shape_any_collision<SpherodiskShape>(res.snapshot.particles, grid));
        // migrate and relax_sweeps on platelets keep the state valid (reference test) and
        // keep unit normals
        auto ps = res.snapshot.particles;
        CellGrid<3> g2(box, 2.5 * max_r + 0.05, max_r, 0.05);
        Rng rng2(3);
        const auto acc = srm::b200::migrate<SpherodiskShape>(ps, g2, 0.05, 0.05, 10, rng2);
        std::size_t moved = 0;
        for (auto v : acc) moved += v;
        CHECK(moved > 0);
        srm::b200::relax_sweeps<SpherodiskShape>(ps, box, 0.05, 0.05, 10, 2, rng2);
        build_shape_grid<SpherodiskShape>(grid, ps);
        CHECK(!srm::shape_any_collision<SpherodiskShape>(std::span<const Spherodisk>(ps), grid));
        bool unit = true;
        for (const auto& q : ps) unit = unit && std::fabs(q.normal.norm() - 1.0) < 1e-12;
        CHECK(unit);
    }
    // a progress sink that throws: srm_generate rethrows the sink's own exception after the
    // run (engine.hpp:251-254 propagates it); the cached context stays usable
    {
        auto snap = disk_start(100, 0.1, 31);
        SrmParams p;
        p.c_w = 0.05;
        p.c_m = 0.01;
        p.f_target = 0.4;
        int seen = 0;
        bool threw = false;
        try {
            srm::b200::srm_generate<DiskShape>(snap, p, [&](const ProgressRecord& r) {
                ++seen;
                if (r.iteration == 3) throw std::runtime_error("sink stop");
            });
        } catch (const std::runtime_error& e) {
            threw = std::string(e.what()) == "sink stop";
        }
        CHECK(threw);
        CHECK(seen == 3);
        const auto again = srm::b200::srm_generate<DiskShape>(snap, p);
        CHECK(again.status == GenerateStatus::Converged);
    }
    // fine-grained drop-ins in a loop reuse one cached device context per thread
    {
        auto snap = disk_start(400, 0.3, 32);
        Rng rng(5);
        for (int k = 0; k < 50; ++k)
            srm::b200::relax_sweeps<DiskShape>(snap.particles, snap.box, 0.002, 0.0, 4, 1, rng);
        CHECK(violations<2>(snap.particles, snap.box, 0.0) == 0);
    }
    std::printf("shim_test: %d/%d checks passed\n", checks - failures, checks);
    return failures == 0 ? 0 : 1;
}
