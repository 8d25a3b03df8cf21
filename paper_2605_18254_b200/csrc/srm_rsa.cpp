// srm_rsa.cpp -- host-side initial-state generators: rsa_place (rsa.hpp:21-69) and
// rsa_platelets (recipes.cpp:107-148).
//
// Random sequential adsorption is sequential by definition (each acceptance changes
// the next candidate's test), so it stays on the host, as input generation whose time
// is excluded from the metric.  It consumes std::mt19937_64 exactly as the reference's
// Rng does (random.hpp:16-61), and its accept test is the reference predicate
// (strictly non-touching, rsa.hpp:19-20, cell_grid.hpp:197-207), so the output is bit-identical to
// srm::rsa_place for the same seed (pinned in tests/test_rsa.py).  The neighbour search
// is its own flat cell list; any complete search yields the same decisions.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/srm_b200.h"
#include "srm_platelet.cuh"

namespace {

struct RsaGrid {
    int dim;
    int n[3] = {1, 1, 1};
    double edge[3] = {1, 1, 1};
    std::vector<int32_t> head, next;

    int coord(int a, double p) const {
        int i = static_cast<int>(std::floor(p / edge[a]));
        i %= n[a];
        if (i < 0) i += n[a];
        return i;
    }
};

inline double min_image_dist2(int dim, const double* L, const double* a, const double* b) {
    double s = 0.0;
    for (int k = 0; k < dim; ++k) {
        double d = a[k] - b[k];
        const double half = 0.5 * L[k];
        if (d > half) d -= L[k];
        if (d < -half) d += L[k];
        s += d * d;
    }
    return s;
}

}  // namespace

extern "C" {

uint64_t srm_b200_mix_seed(uint64_t seed, uint64_t stream) {
    // random.hpp:84-89 splitmix64 step
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

int srm_b200_rsa_place(int dim, const double* L, int64_t count, const double* radii, int64_t max_attempts,
                       uint64_t seed, double* pos_out, int32_t* id_out, int64_t* placed_out) {
    if (placed_out) *placed_out = 0;
    if (dim != 2 && dim != 3) return SRM_B200_INVALID;
    if (count < 1) return SRM_B200_INVALID;  // rsa.hpp:22 need at least one particle
    double max_r = radii[0];
    for (int64_t i = 1; i < count; ++i) max_r = std::max(max_r, radii[i]);
    double min_len = L[0];
    for (int a = 1; a < dim; ++a) min_len = std::min(min_len, L[a]);
    for (int64_t i = 0; i < count; ++i)
        if (!(radii[i] > 0.0)) return SRM_B200_INVALID;      // rsa.hpp:26-27
    if (!(max_r < min_len / 4.0)) return SRM_B200_INVALID;  // rsa.hpp:28-29

    RsaGrid g;
    g.dim = dim;
    int64_t ncells = 1;
    for (int a = 0; a < dim; ++a) {
        int k = static_cast<int>(std::floor(L[a] / (2.0 * max_r)));
        k = std::max(1, std::min(k, 1 << 12));
        g.n[a] = k;
        g.edge[a] = L[a] / k;
        ncells *= k;
    }
    g.head.assign(static_cast<size_t>(ncells), -1);
    g.next.assign(static_cast<size_t>(count), -1);

    std::mt19937_64 gen(seed);
    auto uniform = [&]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };

    double cand[3];
    for (int64_t i = 0; i < count; ++i) {
        const double ri = radii[i];
        bool accepted = false;
        for (int64_t attempt = 0; attempt < max_attempts; ++attempt) {
            for (int a = 0; a < dim; ++a) cand[a] = uniform() * L[a];  // random.hpp:56-61
            for (int a = 0; a < dim; ++a) {                             // geometry.hpp:107-114
                if (cand[a] < 0.0) cand[a] += L[a];
                if (cand[a] >= L[a]) cand[a] -= L[a];
            }
            int c[3] = {0, 0, 0};
            for (int a = 0; a < dim; ++a) c[a] = g.coord(a, cand[a]);
            bool hit = false;
            int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
            for (int a = 0; a < dim; ++a) {
                if (g.n[a] <= 3) { lo[a] = 0; hi[a] = g.n[a] - 1; }
                else { lo[a] = c[a] - 1; hi[a] = c[a] + 1; }
            }
            for (int zz = lo[2]; zz <= hi[2] && !hit; ++zz) {
                int z = dim == 3 ? ((zz % g.n[2]) + g.n[2]) % g.n[2] : 0;
                for (int yy = lo[1]; yy <= hi[1] && !hit; ++yy) {
                    int y = ((yy % g.n[1]) + g.n[1]) % g.n[1];
                    for (int xx = lo[0]; xx <= hi[0] && !hit; ++xx) {
                        int x = ((xx % g.n[0]) + g.n[0]) % g.n[0];
                        const int64_t cell = (static_cast<int64_t>(z) * g.n[1] + y) * g.n[0] + x;
                        for (int32_t j = g.head[cell]; j >= 0; j = g.next[j]) {
                            const double rr = ri + radii[j];
                            if (min_image_dist2(dim, L, cand, pos_out + static_cast<int64_t>(j) * dim) <= rr * rr) {
                                hit = true;
                                break;
                            }
                        }
                    }
                }
            }
            if (!hit) {
                accepted = true;
                break;
            }
        }
        if (!accepted) {
            if (placed_out) *placed_out = i;
            return SRM_B200_PLACEMENT_FAILURE;
        }
        for (int a = 0; a < dim; ++a) pos_out[i * dim + a] = cand[a];
        if (id_out) id_out[i] = static_cast<int32_t>(i);
        int c[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) c[a] = g.coord(a, cand[a]);
        const int64_t cell = (static_cast<int64_t>(c[2]) * g.n[1] + c[1]) * g.n[0] + c[0];
        g.next[i] = g.head[cell];
        g.head[cell] = static_cast<int32_t>(i);
    }
    if (placed_out) *placed_out = count;
    return SRM_B200_OK;
}


// Clustered random sequential adsorption (BASELINE.json configs[2]: the clustered,
// non-equilibrium start of the polydisperse config; the reference has no generator
// for it, so this is builder-defined).  Cluster centres: the first n_clusters * dim
// uniforms of Rng(seed) (random_point, random.hpp:56-61); particle i belongs to cluster
// i mod n_clusters and its candidates are wrap(centre + sigma * gaussian per axis)
// (Rng::gaussian, Box-Muller with a cached spare, random.hpp:30-52), accepted when
// strictly non-touching every placed particle (the rsa_place predicate).
int srm_b200_rsa_clustered(int dim, const double* L, int64_t count, const double* radii, int64_t n_clusters,
                           double sigma, int64_t max_attempts, uint64_t seed, double* pos_out, int32_t* id_out,
                           int64_t* placed_out) {
    if (placed_out) *placed_out = 0;
    if (dim != 2 && dim != 3) return SRM_B200_INVALID;
    if (count < 1 || n_clusters < 1 || !(sigma >= 0.0)) return SRM_B200_INVALID;
    double max_r = radii[0];
    for (int64_t i = 1; i < count; ++i) max_r = std::max(max_r, radii[i]);
    double min_len = L[0];
    for (int a = 1; a < dim; ++a) min_len = std::min(min_len, L[a]);
    for (int64_t i = 0; i < count; ++i)
        if (!(radii[i] > 0.0)) return SRM_B200_INVALID;
    if (!(max_r < min_len / 4.0)) return SRM_B200_INVALID;

    RsaGrid g;
    g.dim = dim;
    int64_t ncells = 1;
    for (int a = 0; a < dim; ++a) {
        int k = static_cast<int>(std::floor(L[a] / (2.0 * max_r)));
        k = std::max(1, std::min(k, 1 << 12));
        g.n[a] = k;
        g.edge[a] = L[a] / k;
        ncells *= k;
    }
    g.head.assign(static_cast<size_t>(ncells), -1);
    g.next.assign(static_cast<size_t>(count), -1);

    std::mt19937_64 gen(seed);
    auto uniform = [&]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
    bool have_spare = false;
    double spare = 0.0;
    auto gaussian = [&]() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 == 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = r * std::sin(a);
        have_spare = true;
        return r * std::cos(a);
    };
    std::vector<double> centre(static_cast<size_t>(n_clusters) * dim);
    for (int64_t k = 0; k < n_clusters; ++k)
        for (int a = 0; a < dim; ++a) centre[k * dim + a] = uniform() * L[a];

    double cand[3];
    for (int64_t i = 0; i < count; ++i) {
        const double ri = radii[i];
        const double* c0 = &centre[(i % n_clusters) * dim];
        bool accepted = false;
        for (int64_t attempt = 0; attempt < max_attempts; ++attempt) {
            for (int a = 0; a < dim; ++a) {
                double p = c0[a] + sigma * gaussian();
                p = std::fmod(p, L[a]);  // far tails: back into [0, L)
                if (p < 0.0) p += L[a];
                if (p >= L[a]) p -= L[a];
                cand[a] = p;
            }
            int c[3] = {0, 0, 0};
            for (int a = 0; a < dim; ++a) c[a] = g.coord(a, cand[a]);
            bool hit = false;
            for (int dz = (dim == 3 ? -1 : 0); dz <= (dim == 3 ? 1 : 0) && !hit; ++dz) {
                if (dim == 3 && g.n[2] < 3 && dz != 0 && (dz == 1 || g.n[2] == 1)) continue;
                const int z = dim == 3 ? ((c[2] + dz) % g.n[2] + g.n[2]) % g.n[2] : 0;
                for (int dy = -1; dy <= 1 && !hit; ++dy) {
                    if (g.n[1] < 3 && dy != 0 && (dy == 1 || g.n[1] == 1)) continue;
                    const int y = ((c[1] + dy) % g.n[1] + g.n[1]) % g.n[1];
                    for (int dx = -1; dx <= 1 && !hit; ++dx) {
                        if (g.n[0] < 3 && dx != 0 && (dx == 1 || g.n[0] == 1)) continue;
                        const int x = ((c[0] + dx) % g.n[0] + g.n[0]) % g.n[0];
                        const int64_t cell = (static_cast<int64_t>(z) * g.n[1] + y) * g.n[0] + x;
                        for (int32_t j = g.head[cell]; j >= 0; j = g.next[j]) {
                            const double rr = ri + radii[j];
                            if (min_image_dist2(dim, L, cand, pos_out + static_cast<int64_t>(j) * dim) <= rr * rr) {
                                hit = true;
                                break;
                            }
                        }
                    }
                }
            }
            if (!hit) {
                accepted = true;
                break;
            }
        }
        if (!accepted) {
            if (placed_out) *placed_out = i;
            return SRM_B200_PLACEMENT_FAILURE;
        }
        for (int a = 0; a < dim; ++a) pos_out[i * dim + a] = cand[a];
        if (id_out) id_out[i] = static_cast<int32_t>(i);
        int c[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) c[a] = g.coord(a, cand[a]);
        const int64_t cell = (static_cast<int64_t>(c[2]) * g.n[1] + c[1]) * g.n[0] + c[0];
        g.next[i] = g.head[cell];
        g.head[cell] = static_cast<int32_t>(i);
    }
    if (placed_out) *placed_out = count;
    return SRM_B200_OK;
}

int srm_b200_rsa_platelets(int64_t count, double diameter, double aspect_ratio, const double* L, int64_t max_attempts,
                           uint64_t seed, double* pos_out, double* normal_out, int32_t* id_out, int64_t* placed_out) {
    using namespace srmb::pl;
    if (placed_out) *placed_out = 0;
    if (count < 1) return SRM_B200_INVALID;                  // recipes.cpp:109
    if (!(aspect_ratio > 1.0)) return SRM_B200_INVALID;      // recipes.cpp:110-111
    const double thickness = diameter / aspect_ratio;
    const double bound = 0.5 * (diameter + thickness);
    double min_len = L[0];
    for (int a = 1; a < 3; ++a) min_len = std::min(min_len, L[a]);
    if (!(bound < min_len / 4.0)) return SRM_B200_INVALID;   // recipes.cpp:116-117

    // Rng (random.hpp:16-52): mt19937_64, 53-bit uniforms, Box-Muller with a cached spare
    std::mt19937_64 gen(seed);
    auto uniform = [&]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
    bool have_spare = false;
    double spare = 0.0;
    auto gaussian = [&]() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 == 0.0) u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * 3.141592653589793238462643383279502884 * u2;
        spare = r * std::sin(a);
        have_spare = true;
        return r * std::cos(a);
    };
    SeedTable tab;  // spherodisk.cpp:60-66 rim seeds
    for (int k = 0; k < kSeeds; ++k) {
        const double a = 2.0 * 3.141592653589793238462643383279502884 * k / kSeeds;
        tab.c[k] = std::cos(a);
        tab.s[k] = std::sin(a);
    }

    RsaGrid g;  // any complete neighbour search decides like CellGrid(box, 2.5 bound)
    g.dim = 3;
    int64_t ncells = 1;
    for (int a = 0; a < 3; ++a) {
        int k = static_cast<int>(std::floor(L[a] / (2.0 * bound)));
        k = std::max(1, std::min(k, 1 << 10));
        g.n[a] = k;
        g.edge[a] = L[a] / k;
        ncells *= k;
    }
    g.head.assign(static_cast<size_t>(ncells), -1);
    g.next.assign(static_cast<size_t>(count), -1);

    double cand[3];
    V3 cn{0.0, 0.0, 0.0};
    for (int64_t i = 0; i < count; ++i) {
        bool accepted = false;
        for (int64_t attempt = 0; attempt < max_attempts; ++attempt) {
            for (int a = 0; a < 3; ++a) cand[a] = uniform() * L[a];  // random.hpp:56-61 random_point
            for (int a = 0; a < 3; ++a) {
                if (cand[a] < 0.0) cand[a] += L[a];
                if (cand[a] >= L[a]) cand[a] -= L[a];
            }
            for (;;) {  // random.hpp:70-76 random_unit_vector<3>
                const V3 gv{gaussian(), gaussian(), gaussian()};
                const double n2 = dot(gv, gv);
                if (n2 > 1e-24) {
                    cn = mul(gv, 1.0 / std::sqrt(n2));
                    break;
                }
            }
            int c[3];
            for (int a = 0; a < 3; ++a) c[a] = g.coord(a, cand[a]);
            bool hit = false;
            for (int dz = -1; dz <= 1 && !hit; ++dz) {
                if (g.n[2] < 3 && dz != 0 && (g.n[2] == 1 || dz == 1)) continue;
                const int z = ((c[2] + dz) % g.n[2] + g.n[2]) % g.n[2];
                for (int dy = -1; dy <= 1 && !hit; ++dy) {
                    if (g.n[1] < 3 && dy != 0 && (g.n[1] == 1 || dy == 1)) continue;
                    const int y = ((c[1] + dy) % g.n[1] + g.n[1]) % g.n[1];
                    for (int dx = -1; dx <= 1 && !hit; ++dx) {
                        if (g.n[0] < 3 && dx != 0 && (g.n[0] == 1 || dx == 1)) continue;
                        const int x = ((c[0] + dx) % g.n[0] + g.n[0]) % g.n[0];
                        const int64_t cell = (static_cast<int64_t>(z) * g.n[1] + y) * g.n[0] + x;
                        for (int32_t j = g.head[cell]; j >= 0 && !hit; j = g.next[j]) {
                            // shape_collides (shape.hpp:64-73): overlap(candidate, placed)
                            const double* pj = pos_out + 3 * static_cast<int64_t>(j);
                            V3 d;
                            double dd[3];
                            for (int a = 0; a < 3; ++a) {
                                double v = pj[a] - cand[a];
                                const double half = 0.5 * L[a];
                                if (v > half) v -= L[a];
                                if (v < -half) v += L[a];
                                dd[a] = v;
                            }
                            d = V3{dd[0], dd[1], dd[2]};
                            const double* nj = normal_out + 3 * static_cast<int64_t>(j);
                            hit = spherodisk_overlap(d, cn, diameter, thickness, V3{nj[0], nj[1], nj[2]}, diameter,
                                                     thickness, tab);
                        }
                    }
                }
            }
            if (!hit) {
                accepted = true;
                break;
            }
        }
        if (!accepted) {
            if (placed_out) *placed_out = i;
            return SRM_B200_PLACEMENT_FAILURE;
        }
        for (int a = 0; a < 3; ++a) pos_out[3 * i + a] = cand[a];
        normal_out[3 * i] = cn.x;
        normal_out[3 * i + 1] = cn.y;
        normal_out[3 * i + 2] = cn.z;
        if (id_out) id_out[i] = static_cast<int32_t>(i);
        int c[3];
        for (int a = 0; a < 3; ++a) c[a] = g.coord(a, cand[a]);
        const int64_t cell = (static_cast<int64_t>(c[2]) * g.n[1] + c[1]) * g.n[0] + c[0];
        g.next[i] = g.head[cell];
        g.head[cell] = static_cast<int32_t>(i);
    }
    if (placed_out) *placed_out = count;
    return SRM_B200_OK;
}

}  // extern "C"
