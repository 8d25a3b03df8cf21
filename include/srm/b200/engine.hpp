// srm/b200/engine.hpp -- header-only C++ drop-in for the reference's SRM engine API,
// running on a B200 through libsrm_b200.so (C ABI: include/srm_b200.h).
//
// The functions keep the signatures of /root/reference/proj/core/include/srm/engine.hpp
// and shape.hpp, on the reference's own types, so switching a caller is a namespace
// change:  srm::srm_generate<S>(...)  ->  srm::b200::srm_generate<S>(...).
//
//   srm_generate        engine.hpp:176-260
//   migrate             engine.hpp:89-107   (Rng& -> one rng.raw() draw as the Philox key)
//   relax_sweeps/shake  engine.hpp:112-130  (idem)
//   swell_all           engine.hpp:134-138
//   reorder_by_locality engine.hpp:144-166
//   shape_any_collision shape.hpp:75-81
//   rsa_place           rsa.hpp:21-61       (seeded form; bit-identical to Rng(seed))
//   rsa_platelets       recipes.cpp:107-148 (seeded form; bit-identical to Rng(seed))
//   nearest_neighbor_distances  descriptors.hpp:96-115 (exact, on the device)
//   local_nematic_order         descriptors.hpp:182-209 (platelets; counts exact, values to 1e-12)
//
// Differences the caller can observe:
//   * migrate is the coloured Gauss-Seidel sweep: the reference's
//     per-particle rule in (colour class, cell, slot) order with Philox trials keyed by
//     (key, slot, attempt, round, iteration), so trajectories differ from the
//     storage-order mt19937_64 sweep (statistically equal, tests/test_gpu_e2e.py);
//   * errors: ValidationError / PlacementFailure / std::invalid_argument as in the
//     reference; device failures throw srm::b200::DeviceError.
// Disks, spheres and thin platelets (SphereShape<2>, SphereShape<3>, SpherodiskShape).
#pragma once

#include <algorithm>
#include <limits>
#include <cstddef>
#include <cstdint>
#include <exception>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "srm/cell_grid.hpp"
#include "srm/engine.hpp"
#include "srm/errors.hpp"
#include "srm/geometry.hpp"
#include "srm/random.hpp"
#include "srm/descriptors.hpp"
#include "srm/recipes.hpp"
#include "srm/rsa.hpp"
#include "srm/spherodisk.hpp"
#include "srm/shape.hpp"
#include "srm_b200.h"

namespace srm::b200 {

struct DeviceError : srm::Error {
    using srm::Error::Error;
};

template <typename S>
inline constexpr bool is_sphere_shape_v = std::is_same_v<S, SphereShape<S::dim>>;
template <typename S>
inline constexpr bool is_supported_shape_v = is_sphere_shape_v<S> || std::is_same_v<S, SpherodiskShape>;

namespace detail {

inline void check(int st, const srm_b200_ctx* c, bool invalid_argument = false) {
    if (st == SRM_B200_OK || st == SRM_B200_ITERATION_LIMIT) return;
    const std::string msg = c ? srm_b200_last_error(c) : srm_b200_create_error();
    if (st == SRM_B200_INVALID) {
        if (invalid_argument) throw std::invalid_argument(msg);
        throw ValidationError(msg);
    }
    throw DeviceError("srm_b200 status " + std::to_string(st) + ": " + msg);
}

// Device contexts cached per host thread, keyed by (dimension, shape kind, box, device):
// a caller looping on the fine-grained drop-ins (migrate / relax_sweeps / ... inside a
// recipe loop, recipes.cpp:218-241) reuses one context -- its device buffers, CUDA
// stream and cached generate graph -- instead of allocating a fresh one per call.  A
// context grows (is recreated) when a call needs more capacity.  A context in use by an
// enclosing call on the same thread (a progress sink calling back into the shim) is not
// shared: that call gets a private one.
class ContextCache {
  public:
    struct Lease {
        srm_b200_ctx* ctx = nullptr;
        bool* busy = nullptr;  // cached entry: released on destruction; private: destroyed
    };
    ~ContextCache() {
        for (auto& e : entries_) srm_b200_destroy(e.ctx);
    }
    Lease acquire(int dim, int kind, const double* L, int64_t capacity, int device) {
        for (auto& e : entries_) {
            if (e.dim != dim || e.kind != kind || e.device != device || e.L[0] != L[0] || e.L[1] != L[1] ||
                e.L[2] != L[2])
                continue;
            if (*e.busy) break;  // re-entrant use: a private context below
            if (e.cap < capacity) {
                srm_b200_destroy(e.ctx);
                e.ctx = nullptr;
                check(srm_b200_create(dim, kind, L, capacity, device, &e.ctx), nullptr);
                e.cap = capacity;
            }
            *e.busy = true;
            return Lease{e.ctx, e.busy.get()};
        }
        srm_b200_ctx* c = nullptr;
        check(srm_b200_create(dim, kind, L, capacity, device, &c), nullptr);
        const bool shared = std::none_of(entries_.begin(), entries_.end(), [&](const Entry& e) {
            return e.dim == dim && e.kind == kind && e.device == device && e.L[0] == L[0] && e.L[1] == L[1] &&
                   e.L[2] == L[2];
        });
        if (!shared) return Lease{c, nullptr};
        entries_.push_back(Entry{dim, kind, device, {L[0], L[1], L[2]}, capacity, c, std::make_unique<bool>(true)});
        return Lease{c, entries_.back().busy.get()};
    }
    static ContextCache& local() {
        thread_local ContextCache cache;
        return cache;
    }

  private:
    struct Entry {
        int dim, kind, device;
        double L[3];
        int64_t cap;
        srm_b200_ctx* ctx;
        std::unique_ptr<bool> busy;
    };
    std::vector<Entry> entries_;
};

// One device context (from the per-thread cache) holding a copy of the particles of shape S
template <typename S>
class Device {
    static constexpr int N = S::dim;
    static constexpr bool kPlatelet = std::is_same_v<S, SpherodiskShape>;

  public:
    Device(const PeriodicBox<N>& box, std::size_t capacity, int device = 0) {
        double L[3] = {1.0, 1.0, 1.0};
        for (int a = 0; a < N; ++a) L[a] = box.length(a);
        lease_ = ContextCache::local().acquire(N, kPlatelet ? SRM_B200_PLATELET : SRM_B200_SPHERE, L,
                                               static_cast<int64_t>(capacity < 1 ? 1 : capacity), device);
        ctx_ = lease_.ctx;
    }
    ~Device() {
        if (lease_.busy) *lease_.busy = false;
        else srm_b200_destroy(ctx_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    srm_b200_ctx* get() const { return ctx_; }

    void upload(std::span<const typename S::ParticleT> ps) {
        if constexpr (kPlatelet) {  // Spherodisk (spherodisk.hpp:16-22) as SoA
            const std::size_t n = ps.size();
            std::vector<double> pos(3 * n), nrm(3 * n), D(n), t(n);
            std::vector<int32_t> id(n);
            for (std::size_t i = 0; i < n; ++i) {
                for (int a = 0; a < 3; ++a) {
                    pos[3 * i + a] = ps[i].pos[a];
                    nrm[3 * i + a] = ps[i].normal[a];
                }
                D[i] = ps[i].diameter;
                t[i] = ps[i].thickness;
                id[i] = ps[i].id;
            }
            check(srm_b200_upload_platelets(ctx_, static_cast<int64_t>(n), pos.data(), nrm.data(), D.data(), t.data(),
                                            id.data()),
                  ctx_);
        } else {  // Particle<N> is {int id; Vec<N> pos; double radius} (geometry.hpp:139-144)
            check(srm_b200_upload_records(ctx_, static_cast<int64_t>(ps.size()), ps.data(), sizeof(Particle<N>),
                                          offsetof(Particle<N>, id), offsetof(Particle<N>, pos),
                                          offsetof(Particle<N>, radius)),
                  ctx_);
        }
    }
    void download(std::vector<typename S::ParticleT>& ps) {
        if constexpr (kPlatelet) {
            const std::size_t n = ps.size();
            std::vector<double> pos(3 * n), nrm(3 * n), D(n), t(n);
            std::vector<int32_t> id(n);
            check(srm_b200_download_platelets(ctx_, pos.data(), nrm.data(), D.data(), t.data(), id.data()), ctx_);
            for (std::size_t i = 0; i < n; ++i) {
                for (int a = 0; a < 3; ++a) {
                    ps[i].pos[a] = pos[3 * i + a];
                    ps[i].normal[a] = nrm[3 * i + a];
                }
                ps[i].diameter = D[i];
                ps[i].thickness = t[i];
                ps[i].id = id[i];
            }
        } else {
            check(srm_b200_download_records(ctx_, ps.data(), sizeof(Particle<N>), offsetof(Particle<N>, id),
                                            offsetof(Particle<N>, pos), offsetof(Particle<N>, radius)),
                  ctx_);
        }
    }

  private:
    ContextCache::Lease lease_{};
    srm_b200_ctx* ctx_ = nullptr;
};

inline srm_b200_params to_c(const SrmParams& p) {
    srm_b200_params c{};
    c.c_w = p.c_w;
    c.c_m = p.c_m;
    c.c_r = p.c_r;
    c.n_k = p.n_k;
    c.n_l = p.n_l;
    c.f_target = p.f_target;
    c.max_iterations = p.max_iterations;
    c.seed = p.seed;
    c.reorder_period = p.reorder_period;
    return c;
}

// The sink runs on the calling thread while the device loop runs (records arrive live).
// An exception it throws must not cross the C ABI: it is kept, later records are not
// delivered, and srm_generate rethrows it after the run, as the reference's call would
// have propagated it (engine.hpp:251-254).
struct SinkCall {
    const ProgressSink* sink;
    std::exception_ptr error;
};

inline void progress_trampoline(const srm_b200_progress_record* rec, void* user) {
    auto* call = static_cast<SinkCall*>(user);
    if (call->error) return;
    try {
        (*call->sink)(ProgressRecord{rec->iteration, rec->volume_fraction, rec->accepted != 0, rec->elapsed_seconds});
    } catch (...) {
        call->error = std::current_exception();
    }
}

}  // namespace detail

// engine.hpp:176-260
template <ShapeModel S>
GenerateResult<S> srm_generate(const Snapshot<S>& initial, const SrmParams& params,
                               const ProgressSink& progress = {}) {
    static_assert(is_supported_shape_v<S>, "srm::b200 supports disks, spheres and platelets");
    constexpr int N = S::dim;
    GenerateResult<S> result;
    result.snapshot = initial;
    Snapshot<S>& snap = result.snapshot;
    snap.params = params;
    snap.seed = params.seed;
    detail::Device<S> dev(initial.box, initial.particles.size());
    dev.upload(initial.particles);
    const srm_b200_params cp = detail::to_c(params);
    srm_b200_generate_out out{};
    detail::SinkCall call{&progress, nullptr};
    const int st = srm_b200_generate(dev.get(), &cp, initial.iteration_count,
                                     progress ? &detail::progress_trampoline : nullptr, &call, &out);
    if (call.error) std::rethrow_exception(call.error);
    detail::check(st, dev.get());
    dev.download(snap.particles);
    snap.volume_fraction = out.volume_fraction;
    snap.iteration_count = out.iteration_count;
    result.status = st == SRM_B200_ITERATION_LIMIT ? GenerateStatus::IterationLimitExceeded
                                                   : GenerateStatus::Converged;
    return result;
}

// engine.hpp:89-107: one migration sweep against `grid` (its cell size), the coloured
// Gauss-Seidel round of DESIGN.md §3.1 keyed by one draw of rng.  Returns the accepted flags.
template <ShapeModel S>
std::vector<std::uint8_t> migrate(std::vector<typename S::ParticleT>& particles, const CellGrid<S::dim>& grid,
                                  double c_m, double c_r, int n_l, Rng& rng) {
    static_assert(is_supported_shape_v<S>, "srm::b200 supports disks, spheres and platelets");
    constexpr int N = S::dim;
    std::vector<std::uint8_t> acc(particles.size(), 0);
    if (particles.empty()) return acc;
    const std::uint64_t key = rng.raw();
    detail::Device<S> dev(grid.box(), particles.size());
    dev.upload(particles);
    srm_b200_round_stats st{};
    detail::check(srm_b200_set_rotation(dev.get(), c_r), dev.get(), true);
    detail::check(srm_b200_round(dev.get(), grid.cell_size(), c_m, n_l, key, 0, 0, 0, acc.data(), &st), dev.get(),
                  true);
    dev.download(particles);
    for (auto& a : acc) a = a != 255 ? 1 : 0;
    return acc;
}

// engine.hpp:112-122
template <ShapeModel S>
void relax_sweeps(std::vector<typename S::ParticleT>& particles, const PeriodicBox<S::dim>& box, double c_m,
                  double c_r, int n_l, int sweeps, Rng& rng) {
    static_assert(is_supported_shape_v<S>, "srm::b200 supports disks, spheres and platelets");
    if (particles.empty() || sweeps < 1) return;
    const std::uint64_t key = rng.raw();
    detail::Device<S> dev(box, particles.size());
    dev.upload(particles);
    detail::check(srm_b200_relax_sweeps(dev.get(), c_m, c_r, n_l, sweeps, key), dev.get(), true);
    dev.download(particles);
}

// engine.hpp:126-130
template <ShapeModel S>
void shake(std::vector<typename S::ParticleT>& particles, const PeriodicBox<S::dim>& box, const SrmParams& params,
           Rng& rng) {
    relax_sweeps<S>(particles, box, params.c_m, params.c_r, params.n_l, params.n_k, rng);
}

// engine.hpp:134-138 (on the device; radius *= 1 + c_w)
template <ShapeModel S>
void swell_all(std::vector<typename S::ParticleT>& particles, double c_w) {
    static_assert(is_supported_shape_v<S>, "srm::b200 supports disks, spheres and platelets");
    if (particles.empty()) return;
    detail::Device<S> dev(PeriodicBox<S::dim>::unit(), particles.size());
    dev.upload(particles);
    detail::check(srm_b200_swell_all(dev.get(), c_w), dev.get());
    dev.download(particles);
}

// engine.hpp:144-166
template <ShapeModel S>
std::vector<int> reorder_by_locality(std::vector<typename S::ParticleT>& particles, const CellGrid<S::dim>& grid) {
    static_assert(is_supported_shape_v<S>, "srm::b200 supports disks, spheres and platelets");
    std::vector<int> remap(particles.size());
    if (particles.empty()) return remap;
    detail::Device<S> dev(grid.box(), particles.size());
    dev.upload(particles);
    detail::check(srm_b200_reorder_by_locality(dev.get(), grid.cell_size(), remap.data()), dev.get(), true);
    dev.download(particles);
    return remap;
}

// shape.hpp:75-81 (the device counts overlapping pairs; any collision <=> count > 0)
template <ShapeModel S>
bool shape_any_collision(std::span<const typename S::ParticleT> particles, const CellGrid<S::dim>& grid) {
    static_assert(is_supported_shape_v<S>, "srm::b200 supports disks, spheres and platelets");
    if (particles.empty()) return false;
    detail::Device<S> dev(grid.box(), particles.size());
    dev.upload(particles);
    srm_b200_round_stats st{};
    detail::check(srm_b200_overlap_stats(dev.get(), grid.cell_size(), &st), dev.get(), true);
    return st.overlap_pairs > 0;
}

// rsa.hpp:21-61 with Rng(seed): bit-identical to srm::rsa_place for a fresh Rng(seed)
template <int N>
std::vector<Particle<N>> rsa_place(std::span<const double> radii, const PeriodicBox<N>& box,
                                   std::size_t max_attempts_per_particle, std::uint64_t seed) {
    double L[3] = {1.0, 1.0, 1.0};
    for (int a = 0; a < N; ++a) L[a] = box.length(a);
    std::vector<double> pos(radii.size() * N);
    std::vector<int32_t> ids(radii.size());
    int64_t placed = 0;
    const int st = srm_b200_rsa_place(N, L, static_cast<int64_t>(radii.size()), radii.data(),
                                      static_cast<int64_t>(max_attempts_per_particle), seed, pos.data(), ids.data(),
                                      &placed);
    if (st == SRM_B200_PLACEMENT_FAILURE)
        throw PlacementFailure("rsa_place: exceeded " + std::to_string(max_attempts_per_particle) +
                                   " attempts after placing " + std::to_string(placed) +
                                   " particles; initial volume fraction too high",
                               static_cast<std::size_t>(placed), max_attempts_per_particle);
    if (st == SRM_B200_INVALID) throw ValidationError("rsa_place: invalid radii or box");
    std::vector<Particle<N>> out(radii.size());
    for (std::size_t i = 0; i < radii.size(); ++i) {
        out[i].id = ids[i];
        for (int a = 0; a < N; ++a) out[i].pos[a] = pos[i * N + a];
        out[i].radius = radii[i];
    }
    return out;
}

// recipes.cpp:107-148 with Rng(seed): bit-identical to srm::rsa_platelets for a fresh Rng(seed)
inline PlateletSnapshot rsa_platelets(std::int64_t n, double diameter, double aspect_ratio, const PeriodicBox3& box,
                                      std::size_t max_attempts_per_particle, std::uint64_t seed) {
    double L[3] = {box.length(0), box.length(1), box.length(2)};
    const std::size_t m = n > 0 ? static_cast<std::size_t>(n) : 0;
    std::vector<double> pos(3 * m), nrm(3 * m);
    std::vector<int32_t> ids(m);
    int64_t placed = 0;
    const int st = srm_b200_rsa_platelets(n, diameter, aspect_ratio, L, static_cast<int64_t>(max_attempts_per_particle),
                                          seed, pos.data(), nrm.data(), ids.data(), &placed);
    if (st == SRM_B200_PLACEMENT_FAILURE)
        throw PlacementFailure("rsa_platelets: exceeded attempt budget", static_cast<std::size_t>(placed),
                               max_attempts_per_particle);
    if (st == SRM_B200_INVALID) throw ValidationError("rsa_platelets: invalid size, aspect ratio or box");
    PlateletSnapshot snap;
    snap.box = box;
    snap.particles.resize(m);
    for (std::size_t i = 0; i < m; ++i) {
        auto& q = snap.particles[i];
        q.id = ids[i];
        for (int a = 0; a < 3; ++a) {
            q.pos[a] = pos[3 * i + a];
            q.normal[a] = nrm[3 * i + a];
        }
        q.diameter = diameter;
        q.thickness = diameter / aspect_ratio;
    }
    snap.refresh_volume_fraction();
    return snap;
}

// descriptors.hpp:96-115 on the device: exact (the minimum over all other centres)
template <ShapeModel S>
std::vector<double> nearest_neighbor_distances(const Snapshot<S>& snap) {
    static_assert(is_sphere_shape_v<S>, "nearest_neighbor_distances: disks and spheres");
    if (snap.particles.size() < 2) throw ValidationError("nearest_neighbor_distances: need at least 2 particles");
    detail::Device<S> dev(snap.box, snap.particles.size());
    dev.upload(snap.particles);
    std::vector<double> out(snap.particles.size());
    detail::check(srm_b200_nnd_histogram(dev.get(), 0, 0.0, 0.0, nullptr, nullptr, nullptr, out.data()), dev.get());
    return out;
}

// descriptors.hpp:182-209 on the device: per platelet the mean |n_i . n_j| over the
// platelets whose centre lies within `cutoff` (NaN when none) and their number.  The
// counts are the reference's; the values agree to rounding (the sum over neighbours runs
// in another cell order).
inline NematicOrder local_nematic_order(const Snapshot<SpherodiskShape>& snap, double cutoff) {
    if (!(cutoff > 0.0)) throw ValidationError("local_nematic_order: cutoff must be positive");
    NematicOrder out;
    const std::size_t n = snap.particles.size();
    out.value.assign(n, std::numeric_limits<double>::quiet_NaN());
    out.neighbor_count.assign(n, 0);
    if (n == 0) return out;
    detail::Device<SpherodiskShape> dev(snap.box, n);
    dev.upload(snap.particles);
    std::vector<int32_t> cnt(n);
    detail::check(srm_b200_platelet_order(dev.get(), cutoff, out.value.data(), cnt.data(), nullptr, nullptr, nullptr),
                  dev.get());
    for (std::size_t i = 0; i < n; ++i) out.neighbor_count[i] = cnt[i];
    return out;
}

}  // namespace srm::b200
