// ref_harness.cpp -- extern "C" bindings over the UNMODIFIED reference headers
// (/root/reference/proj/core/include, compiled where they lie; nothing is copied).
// TEST INFRASTRUCTURE ONLY: built into oracle/_ref/libsrm_ref.so by oracle/Makefile
// with the reference's Release flags (-O3 -DNDEBUG, no -march).  Used to pin the
// oracle restatement, to generate golden fixtures, as the end-to-end statistical
// oracle (srm_generate itself), and as the CPU baseline in bench.py.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "srm/cell_grid.hpp"
#include "srm/descriptors.hpp"
#include "srm/engine.hpp"
#include "srm/geometry.hpp"
#include "srm/random.hpp"
#include "srm/recipes.hpp"
#include "srm/rsa.hpp"
#include "srm/shape.hpp"
#include "srm/snapshot_io.hpp"
#include "srm/spherodisk.hpp"

using namespace srm;

namespace {

template <int N>
PeriodicBox<N> make_box(const double* L) {
    std::array<double, N> l;
    for (int a = 0; a < N; ++a) l[a] = L[a];
    return PeriodicBox<N>(l);
}

template <int N>
std::vector<Particle<N>> make_particles(int64_t n, const double* pos, const double* r,
                                        const int32_t* id) {
    std::vector<Particle<N>> ps(static_cast<std::size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        ps[i].id = id ? id[i] : static_cast<int>(i);
        for (int a = 0; a < N; ++a) ps[i].pos[a] = pos[i * N + a];
        ps[i].radius = r ? r[i] : 0.0;
    }
    return ps;
}

template <int N>
void store_particles(const std::vector<Particle<N>>& ps, double* pos, double* r, int32_t* id) {
    for (std::size_t i = 0; i < ps.size(); ++i) {
        if (id) id[i] = ps[i].id;
        for (int a = 0; a < N; ++a) pos[i * N + a] = ps[i].pos[a];
        if (r) r[i] = ps[i].radius;
    }
}

template <int N>
double bench_rounds_impl(const double* L, int64_t n, const double* pos, const double* r,
                         const int32_t* id, double c_m, int n_l, int rounds, uint64_t seed,
                         int threads, int64_t* accepted_total) {
    const auto box = make_box<N>(L);
    const auto start = make_particles<N>(n, pos, r, id);
    std::atomic<int64_t> acc{0};
    auto worker = [&](int t) {
        auto P = start;
        Rng rng(mix_seed(seed, 10000 + static_cast<std::uint64_t>(t)));
        const double max_r = max_bounding_radius<SphereShape<N>>(P);
        // srm_generate's grid (engine.hpp:220-221) at fixed size (factor 1)
        CellGrid<N> grid(box, 2.5 * max_r + c_m, max_r, c_m);
        int64_t local = 0;
        for (int k = 0; k < rounds; ++k) {
            build_shape_grid<SphereShape<N>>(grid, P);
            const auto a = migrate<SphereShape<N>>(P, grid, c_m, 0.0, n_l, rng);
            for (auto v : a) local += v;
            volatile bool any = shape_any_collision<SphereShape<N>>(P, grid);
            (void)any;
        }
        acc += local;
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (threads <= 1) {
        worker(0);
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(worker, t);
        for (auto& th : pool) th.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (accepted_total) *accepted_total = acc.load();
    return std::chrono::duration<double>(t1 - t0).count();
}

}  // namespace

extern "C" {

uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

void ref_rng_uniforms(uint64_t seed, int64_t n, double* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.uniform();
}

void ref_rng_raw(uint64_t seed, int64_t n, uint64_t* out) {
    Rng rng(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = rng.raw();
}

void ref_wrap(int dim, const double* L, double* p) {
    if (dim == 2) {
        Vec2 v{{p[0], p[1]}};
        v = make_box<2>(L).wrap(v);
        p[0] = v[0]; p[1] = v[1];
    } else {
        Vec3 v{{p[0], p[1], p[2]}};
        v = make_box<3>(L).wrap(v);
        p[0] = v[0]; p[1] = v[1]; p[2] = v[2];
    }
}

double ref_min_image_dist2(int dim, const double* L, const double* a, const double* b) {
    if (dim == 2) return make_box<2>(L).min_image_dist2(Vec2{{a[0], a[1]}}, Vec2{{b[0], b[1]}});
    return make_box<3>(L).min_image_dist2(Vec3{{a[0], a[1], a[2]}}, Vec3{{b[0], b[1], b[2]}});
}

// returns 0 ok, 1 invalid_argument (safety bound or non-positive size)
int ref_grid_dims(int dim, const double* L, double cell_size, double max_radius, double slack,
                  int checked, int32_t* dims, double* edge) {
    try {
        if (dim == 2) {
            const auto box = make_box<2>(L);
            CellGrid<2> g = checked ? CellGrid<2>(box, cell_size, max_radius, slack)
                                    : CellGrid<2>(box, cell_size);
            for (int a = 0; a < 2; ++a) { dims[a] = g.dims()[a]; edge[a] = L[a] / g.dims()[a]; }
        } else {
            const auto box = make_box<3>(L);
            CellGrid<3> g = checked ? CellGrid<3>(box, cell_size, max_radius, slack)
                                    : CellGrid<3>(box, cell_size);
            for (int a = 0; a < 3; ++a) { dims[a] = g.dims()[a]; edge[a] = L[a] / g.dims()[a]; }
        }
    } catch (const std::invalid_argument&) {
        return 1;
    }
    return 0;
}

void ref_cell_keys(int dim, const double* L, double cell_size, int64_t n, const double* pos,
                   uint64_t* keys, int32_t* coords) {
    if (dim == 2) {
        const auto box = make_box<2>(L);
        CellGrid<2> g(box, cell_size);
        for (int64_t i = 0; i < n; ++i) {
            const Vec2 p{{pos[2 * i], pos[2 * i + 1]}};
            keys[i] = g.cell_of(p);
            if (coords) { auto c = g.cell_coords(p); coords[2 * i] = c[0]; coords[2 * i + 1] = c[1]; }
        }
    } else {
        const auto box = make_box<3>(L);
        CellGrid<3> g(box, cell_size);
        for (int64_t i = 0; i < n; ++i) {
            const Vec3 p{{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}};
            keys[i] = g.cell_of(p);
            if (coords) {
                auto c = g.cell_coords(p);
                for (int a = 0; a < 3; ++a) coords[3 * i + a] = c[a];
            }
        }
    }
}

// reorder_by_locality on (pos, r, id) in place; remap[old] = new
void ref_reorder(int dim, const double* L, double cell_size, int64_t n, double* pos, double* r,
                 int32_t* id, int32_t* remap) {
    auto run = [&](auto tag) {
        constexpr int N = decltype(tag)::value;
        const auto box = make_box<N>(L);
        CellGrid<N> g(box, cell_size);
        auto ps = make_particles<N>(n, pos, r, id);
        g.build(ps);
        auto m = reorder_by_locality<SphereShape<N>>(ps, g);
        store_particles<N>(ps, pos, r, id);
        for (int64_t i = 0; i < n; ++i) remap[i] = m[i];
    };
    if (dim == 2) run(std::integral_constant<int, 2>{});
    else run(std::integral_constant<int, 3>{});
}

// per-particle check_particle_collision against a grid of the given cell size;
// returns check_any_collision
int ref_collisions(int dim, const double* L, double cell_size, int64_t n, const double* pos,
                   const double* r, const int32_t* id, uint8_t* per_particle) {
    auto run = [&](auto tag) -> int {
        constexpr int N = decltype(tag)::value;
        const auto box = make_box<N>(L);
        CellGrid<N> g(box, cell_size);
        auto ps = make_particles<N>(n, pos, r, id);
        g.build(ps);
        if (per_particle)
            for (int64_t i = 0; i < n; ++i)
                per_particle[i] = check_particle_collision<N>(ps[i], ps, g) ? 1 : 0;
        return shape_any_collision<SphereShape<N>>(ps, g) ? 1 : 0;
    };
    if (dim == 2) return run(std::integral_constant<int, 2>{});
    return run(std::integral_constant<int, 3>{});
}

// rsa_place; returns 0 ok, 1 ValidationError, 2 PlacementFailure (placed_out set)
int ref_rsa_place(int dim, const double* L, int64_t n, const double* radii, int64_t max_attempts,
                  uint64_t seed, double* pos_out, int32_t* id_out, int64_t* placed_out) {
    auto run = [&](auto tag) -> int {
        constexpr int N = decltype(tag)::value;
        const auto box = make_box<N>(L);
        Rng rng(seed);
        std::vector<double> rad(radii, radii + n);
        try {
            auto ps = rsa_place<N>(rad, box, static_cast<std::size_t>(max_attempts), rng);
            store_particles<N>(ps, pos_out, nullptr, id_out);
            if (placed_out) *placed_out = n;
        } catch (const PlacementFailure& e) {
            if (placed_out) *placed_out = static_cast<int64_t>(e.placed_count);
            return 2;
        } catch (const ValidationError&) {
            return 1;
        }
        return 0;
    };
    if (dim == 2) return run(std::integral_constant<int, 2>{});
    return run(std::integral_constant<int, 3>{});
}

// srm_generate on disks/spheres; state in/out.  returns 0 converged, 1 iteration
// limit, 2 ValidationError
int ref_generate(int dim, const double* L, int64_t n, double* pos, double* r, int32_t* id,
                 double c_w, double c_m, int n_k, int n_l, double f_target,
                 int64_t max_iterations, uint64_t seed, int reorder_period,
                 int64_t* iterations_out, double* f_out, int64_t* accepted_out) {
    auto run = [&](auto tag) -> int {
        constexpr int N = decltype(tag)::value;
        Snapshot<SphereShape<N>> snap;
        snap.box = make_box<N>(L);
        snap.particles = make_particles<N>(n, pos, r, id);
        snap.refresh_volume_fraction();
        SrmParams p;
        p.c_w = c_w; p.c_m = c_m; p.n_k = n_k; p.n_l = n_l; p.f_target = f_target;
        p.max_iterations = max_iterations; p.seed = seed; p.reorder_period = reorder_period;
        int64_t acc = 0;
        try {
            auto res = srm_generate<SphereShape<N>>(snap, p, [&](const ProgressRecord& rec) {
                if (rec.accepted) ++acc;
            });
            store_particles<N>(res.snapshot.particles, pos, r, id);
            if (iterations_out) *iterations_out = res.snapshot.iteration_count;
            if (f_out) *f_out = res.snapshot.volume_fraction;
            if (accepted_out) *accepted_out = acc;
            return res.status == GenerateStatus::Converged ? 0 : 1;
        } catch (const ValidationError&) {
            return 2;
        }
    };
    if (dim == 2) return run(std::integral_constant<int, 2>{});
    return run(std::integral_constant<int, 3>{});
}

// reference migrate (engine.hpp:89-107) with Rng(seed) over a grid sized like
// srm_generate's; pos in/out, accepted flags out
void ref_migrate(int dim, const double* L, int64_t n, double* pos, const double* r,
                 const int32_t* id, double cell_size, double c_m, int n_l, uint64_t seed,
                 uint8_t* accepted) {
    auto run = [&](auto tag) {
        constexpr int N = decltype(tag)::value;
        const auto box = make_box<N>(L);
        auto ps = make_particles<N>(n, pos, r, id);
        CellGrid<N> g(box, cell_size);
        build_shape_grid<SphereShape<N>>(g, ps);
        Rng rng(seed);
        auto a = migrate<SphereShape<N>>(ps, g, c_m, 0.0, n_l, rng);
        store_particles<N>(ps, pos, nullptr, nullptr);
        for (int64_t i = 0; i < n; ++i) accepted[i] = a[i];
    };
    if (dim == 2) run(std::integral_constant<int, 2>{});
    else run(std::integral_constant<int, 3>{});
}

void ref_nnd(int dim, const double* L, int64_t n, const double* pos, double* out) {
    if (dim == 2) {
        std::vector<Vec2> c(n);
        for (int64_t i = 0; i < n; ++i) c[i] = Vec2{{pos[2 * i], pos[2 * i + 1]}};
        auto d = nearest_neighbor_distances<2>(c, make_box<2>(L));
        std::memcpy(out, d.data(), sizeof(double) * n);
    } else {
        std::vector<Vec3> c(n);
        for (int64_t i = 0; i < n; ++i) c[i] = Vec3{{pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}};
        auto d = nearest_neighbor_distances<3>(c, make_box<3>(L));
        std::memcpy(out, d.data(), sizeof(double) * n);
    }
}

void ref_histogram(int64_t n, const double* values, int bins, double lo, double hi,
                   int64_t* counts) {
    auto h = histogram(std::span<const double>(values, n), bins, lo, hi);
    for (int b = 0; b < bins; ++b) counts[b] = h.counts[b];
}

// CPU baseline: `threads` independent replicas (srmgen --ensemble semantics) each
// running `rounds` SRM rounds (build_shape_grid -> migrate -> shape_any_collision)
// at fixed size.  Returns wall seconds.
double ref_bench_rounds(int dim, const double* L, int64_t n, const double* pos, const double* r,
                        const int32_t* id, double c_m, int n_l, int rounds, uint64_t seed,
                        int threads, int64_t* accepted_total) {
    if (dim == 2) return bench_rounds_impl<2>(L, n, pos, r, id, c_m, n_l, rounds, seed, threads,
                                              accepted_total);
    return bench_rounds_impl<3>(L, n, pos, r, id, c_m, n_l, rounds, seed, threads,
                                accepted_total);
}


// ---- platelets (spherodisk.hpp, spherodisk.cpp, recipes.cpp:107-148) ------------------
static Spherodisk make_pl(const double* p, const double* nrm, double D, double t, int id = 0) {
    Spherodisk q;
    q.id = id;
    for (int a = 0; a < 3; ++a) {
        q.pos[a] = p[a];
        q.normal[a] = nrm[a];
    }
    q.diameter = D;
    q.thickness = t;
    return q;
}

int ref_pl_overlap(const double* L, const double* pa, const double* na, double Da, double ta, const double* pb,
                   const double* nb, double Db, double tb) {
    return SpherodiskShape::overlap(make_pl(pa, na, Da, ta), make_pl(pb, nb, Db, tb), make_box<3>(L)) ? 1 : 0;
}

int ref_pl_disks_within(const double* c1, const double* n1, double r1, const double* c2, const double* n2, double r2,
                        double threshold) {
    auto v = [](const double* x) { return Vec3{{x[0], x[1], x[2]}}; };
    return disks_within(v(c1), v(n1), r1, v(c2), v(n2), r2, threshold) ? 1 : 0;
}

double ref_pl_disk_distance(const double* c1, const double* n1, double r1, const double* c2, const double* n2,
                            double r2) {
    auto v = [](const double* x) { return Vec3{{x[0], x[1], x[2]}}; };
    return disk_disk_distance(v(c1), v(n1), r1, v(c2), v(n2), r2);
}

double ref_pl_measure(double D, double t) {
    Spherodisk q;
    q.diameter = D;
    q.thickness = t;
    return spherodisk_measure(q);
}

void ref_pl_rotate(const double* v, const double* axis, double angle, double* out) {
    const Vec3 r = rotate_about_axis(Vec3{{v[0], v[1], v[2]}}, Vec3{{axis[0], axis[1], axis[2]}}, angle);
    for (int a = 0; a < 3; ++a) out[a] = r[a];
}

static void store_pl(const std::vector<Spherodisk>& ps, double* pos, double* nrm, double* D, double* t, int32_t* id) {
    for (size_t i = 0; i < ps.size(); ++i) {
        for (int a = 0; a < 3; ++a) {
            if (pos) pos[3 * i + a] = ps[i].pos[a];
            if (nrm) nrm[3 * i + a] = ps[i].normal[a];
        }
        if (D) D[i] = ps[i].diameter;
        if (t) t[i] = ps[i].thickness;
        if (id) id[i] = ps[i].id;
    }
}

// rsa_platelets with Rng(seed); 0 ok, 1 placement failure, 2 invalid
int ref_rsa_platelets(int64_t n, double diameter, double aspect, const double* L, int64_t max_attempts, uint64_t seed,
                      double* pos, double* nrm, int32_t* id) {
    try {
        Rng rng(seed);
        auto snap = rsa_platelets(n, diameter, aspect, make_box<3>(L), static_cast<std::size_t>(max_attempts), rng);
        store_pl(snap.particles, pos, nrm, nullptr, nullptr, id);
        return 0;
    } catch (const PlacementFailure&) {
        return 1;
    } catch (const ValidationError&) {
        return 2;
    }
}

// srm_generate<SpherodiskShape> (engine.hpp:176-260); state in/out
int ref_generate_platelets(const double* L, int64_t n, double* pos, double* nrm, double* D, double* t, int32_t* id,
                           double c_w, double c_m, double c_r, int n_k, int n_l, double f_target, int64_t max_iterations,
                           uint64_t seed, int reorder_period, int64_t* iterations_out, double* f_out) {
    PlateletSnapshot snap;
    snap.box = make_box<3>(L);
    snap.particles.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) snap.particles[i] = make_pl(pos + 3 * i, nrm + 3 * i, D[i], t[i], id[i]);
    snap.refresh_volume_fraction();
    SrmParams p;
    p.c_w = c_w; p.c_m = c_m; p.c_r = c_r; p.n_k = n_k; p.n_l = n_l; p.f_target = f_target;
    p.max_iterations = max_iterations; p.seed = seed; p.reorder_period = reorder_period;
    try {
        auto res = srm_generate<SpherodiskShape>(snap, p);
        store_pl(res.snapshot.particles, pos, nrm, D, t, id);
        if (iterations_out) *iterations_out = res.snapshot.iteration_count;
        if (f_out) *f_out = res.snapshot.volume_fraction;
        return res.status == GenerateStatus::Converged ? 0 : 1;
    } catch (const ValidationError&) {
        return 2;
    }
}

// descriptors.hpp:182-209 local_nematic_order; 0 ok, 2 invalid cutoff
int ref_local_nematic_order(const double* L, int64_t n, const double* pos, const double* nrm, const double* D,
                            const double* t, double cutoff, double* value, int32_t* count) {
    PlateletSnapshot snap;
    snap.box = make_box<3>(L);
    snap.particles.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i)
        snap.particles[i] = make_pl(pos + 3 * i, nrm + 3 * i, D[i], t[i], static_cast<int32_t>(i));
    try {
        const auto o = local_nematic_order(snap, cutoff);
        for (int64_t i = 0; i < n; ++i) {
            value[i] = o.value[i];
            count[i] = o.neighbor_count[i];
        }
        return 0;
    } catch (const ValidationError&) {
        return 2;
    }
}

// CPU baseline for platelets: `threads` replicas x `rounds` SRM rounds at fixed size
// (build_shape_grid -> migrate -> shape_any_collision with SpherodiskShape).  Wall s.
double ref_pl_bench_rounds(const double* L, int64_t n, const double* pos, const double* nrm, const double* D,
                           const double* t, const int32_t* id, double c_m, double c_r, int n_l, int rounds,
                           uint64_t seed, int threads, int64_t* accepted_total) {
    std::vector<Spherodisk> start(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) start[i] = make_pl(pos + 3 * i, nrm + 3 * i, D[i], t[i], id[i]);
    const auto box = make_box<3>(L);
    std::atomic<int64_t> acc{0};
    auto worker = [&](int th) {
        auto P = start;
        Rng rng(mix_seed(seed, 10000 + static_cast<std::uint64_t>(th)));
        const double max_r = max_bounding_radius<SpherodiskShape>(P);
        CellGrid<3> grid(box, 2.5 * max_r + c_m, max_r, c_m);
        int64_t local = 0;
        for (int k = 0; k < rounds; ++k) {
            build_shape_grid<SpherodiskShape>(grid, P);
            const auto a = migrate<SpherodiskShape>(P, grid, c_m, c_r, n_l, rng);
            for (auto v : a) local += v;
            volatile bool any = shape_any_collision<SpherodiskShape>(std::span<const Spherodisk>(P), grid);
            (void)any;
        }
        acc += local;
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (threads <= 1) {
        worker(0);
    } else {
        std::vector<std::thread> pool;
        for (int th = 0; th < threads; ++th) pool.emplace_back(worker, th);
        for (auto& th : pool) th.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (accepted_total) *accepted_total = acc.load();
    return std::chrono::duration<double>(t1 - t0).count();
}

// snapshot_io.cpp snapshot_to_binary / snapshot_to_text of a state (spheres/disks: pos, r;
// platelets (shape 1): pos, nrm, D, t); returns the byte count, copies up to cap bytes
static void fill_meta(SrmParams& p, const double* pd, const int64_t* pi) {
    p.c_w = pd[0]; p.c_m = pd[1]; p.c_r = pd[2]; p.f_target = pd[3];
    p.n_k = static_cast<int>(pi[0]); p.n_l = static_cast<int>(pi[1]); p.max_iterations = pi[2];
    p.seed = static_cast<std::uint64_t>(pi[3]); p.reorder_period = static_cast<int>(pi[4]);
}

int64_t ref_snapshot_bytes(int dim, int shape, const double* L, int64_t n, const double* pos, const double* r,
                           const double* nrm, const double* D, const double* t, const int32_t* id, double f,
                           int64_t iterations, uint64_t seed, const double* pd, const int64_t* pi, int binary,
                           char* out, int64_t cap) {
    std::string bytes;
    if (shape == 1) {
        PlateletSnapshot s;
        s.box = make_box<3>(L);
        s.particles.resize(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) s.particles[i] = make_pl(pos + 3 * i, nrm + 3 * i, D[i], t[i], id[i]);
        s.volume_fraction = f; s.iteration_count = iterations; s.seed = seed;
        fill_meta(s.params, pd, pi);
        bytes = binary ? snapshot_to_binary(s) : snapshot_to_text(s);
    } else if (dim == 2) {
        DiskSnapshot s;
        s.box = make_box<2>(L);
        s.particles = make_particles<2>(n, pos, r, id);
        s.volume_fraction = f; s.iteration_count = iterations; s.seed = seed;
        fill_meta(s.params, pd, pi);
        bytes = binary ? snapshot_to_binary(s) : snapshot_to_text(s);
    } else {
        SphereSnapshot s;
        s.box = make_box<3>(L);
        s.particles = make_particles<3>(n, pos, r, id);
        s.volume_fraction = f; s.iteration_count = iterations; s.seed = seed;
        fill_meta(s.params, pd, pi);
        bytes = binary ? snapshot_to_binary(s) : snapshot_to_text(s);
    }
    if (out) std::memcpy(out, bytes.data(), std::min<size_t>(bytes.size(), static_cast<size_t>(cap)));
    return static_cast<int64_t>(bytes.size());
}

// shape_any_collision<SpherodiskShape> over a grid of cell size cs
int ref_pl_any_collision(const double* L, double cs, int64_t n, const double* pos, const double* nrm, const double* D,
                         const double* t, const int32_t* id) {
    std::vector<Spherodisk> ps(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) ps[i] = make_pl(pos + 3 * i, nrm + 3 * i, D[i], t[i], id[i]);
    const auto box = make_box<3>(L);
    CellGrid<3> g(box, cs);
    build_shape_grid<SpherodiskShape>(g, ps);
    return shape_any_collision<SpherodiskShape>(std::span<const Spherodisk>(ps), g) ? 1 : 0;
}

}  // extern "C"
