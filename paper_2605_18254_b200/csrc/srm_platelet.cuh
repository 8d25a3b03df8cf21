// srm_platelet.cuh -- thin circular platelets (spherodisks) on the B200 path: the
// overlap test, the rigid-body move and the measure of the reference's SpherodiskShape
// (spherodisk.hpp:16-99, spherodisk.cpp:14-112), host and device from one source.
//
// Every expression keeps the reference's operation order (Vec ops component-wise,
// dot = ((0 + a0 b0) + a1 b1) + a2 b2, no FMA contraction: --fmad=false on the device,
// -ffp-contract=off on the host), so decisions are bit-identical to the reference on
// the same inputs.  The only transcendentals of the reference's test -- cos/sin of the
// 32 rim seed angles 2 pi k / 32 of the slow-convergence fallback, and cos/sin of the
// fixed rotation angle c_r of a move -- are evaluated once on the host (glibc, as the
// reference) and handed to the device as tables.
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define SRM_HD __host__ __device__ __forceinline__
#else
#define SRM_HD inline
#endif

namespace srmb {
namespace pl {

struct V3 {
    double x, y, z;
};

SRM_HD V3 add(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
SRM_HD V3 sub(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
SRM_HD V3 mul(V3 a, double s) { return V3{a.x * s, a.y * s, a.z * s}; }
SRM_HD double dot(V3 a, V3 b) {
    double s = 0.0;
    s += a.x * b.x;
    s += a.y * b.y;
    s += a.z * b.z;
    return s;
}
SRM_HD double norm(V3 a) { return sqrt(dot(a, a)); }
SRM_HD V3 cross(V3 a, V3 b) { return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

constexpr int kSeeds = 32;  // rim seeds of the fallback (spherodisk.cpp:60-66)

// cos/sin of 2 pi k / 32, k < 32, as the reference evaluates them (host libm)
struct SeedTable {
    double c[kSeeds], s[kSeeds];
};

// spherodisk.cpp:14-21 closest point of the closed disk (c, n, r) to p
SRM_HD V3 closest_on_disk(V3 c, V3 n, double r, V3 p) {
    const V3 w = sub(p, c);
    V3 in_plane = sub(w, mul(n, dot(w, n)));
    const double d2 = dot(in_plane, in_plane);
    if (d2 > r * r) in_plane = mul(in_plane, r / sqrt(d2));
    return add(c, in_plane);
}

// spherodisk.cpp:29-40 alternating projections from p2 on disk 2; stops when the
// (non-increasing) distance stalls below tol.  Returns the last distance.
SRM_HD double alternate(V3 c1, V3 n1, double r1, V3 c2, V3 n2, double r2, V3 p2, double tol, int max_iter,
                        bool* converged) {
    double prev = static_cast<double>(INFINITY);
    for (int it = 0; it < max_iter; ++it) {
        const V3 p1 = closest_on_disk(c1, n1, r1, p2);
        p2 = closest_on_disk(c2, n2, r2, p1);
        const double d = norm(sub(p1, p2));
        if (prev - d <= tol) {
            *converged = true;
            return d;
        }
        prev = d;
    }
    *converged = false;
    return prev;
}

SRM_HD double max3(double a, double b, double c) {
    // std::max({a, b, c}): the first of the largest
    double m = a;
    if (m < b) m = b;
    if (m < c) m = c;
    return m;
}

// spherodisk.cpp:70-112 disks_within, in two stages so that a team of lanes can run the
// rim seeds of the fallback side by side (the result is the OR over the seeds, so the
// order they run in does not change it).  disks_within_pre: the separation proofs and
// the projections with early accept; kDwFalse / kDwTrue decide, kDwSeeds sends the pair
// to the fallback, rim_seed_within(k) = seed k of it.
enum { kDwFalse = 0, kDwTrue = 1, kDwSeeds = 2 };

SRM_HD double disks_tol(double r1, double r2) { return 1e-12 * max3(r1, r2, 1e-30); }

SRM_HD int disks_within_pre(V3 c1, V3 n1, double r1, V3 c2, V3 n2, double r2, double threshold) {
    const V3 d = sub(c2, c1);
    if (norm(d) - r1 - r2 > threshold) return kDwFalse;
    const double ndot = dot(n1, n2);
    const double t = 1.0 - ndot * ndot;
    const double sin_tilt = sqrt(t > 0.0 ? t : 0.0);
    if (fabs(dot(n1, d)) - r2 * sin_tilt > threshold) return kDwFalse;
    if (fabs(dot(n2, d)) - r1 * sin_tilt > threshold) return kDwFalse;

    const double tol = disks_tol(r1, r2);
    V3 p2 = closest_on_disk(c2, n2, r2, c1);
    double prev = static_cast<double>(INFINITY);
    for (int it = 0; it < 200; ++it) {
        const V3 p1 = closest_on_disk(c1, n1, r1, p2);
        p2 = closest_on_disk(c2, n2, r2, p1);
        const double dist = norm(sub(p1, p2));
        if (dist <= threshold) return kDwTrue;
        if (prev - dist <= tol) return kDwFalse;  // converged above the threshold
        prev = dist;
    }
    return kDwSeeds;
}

SRM_HD bool rim_seed_within(V3 c1, V3 n1, double r1, V3 c2, V3 n2, double r2, double threshold, const SeedTable& tab,
                            int k) {
    V3 u = fabs(n2.x) < 0.9 ? V3{1.0, 0.0, 0.0} : V3{0.0, 1.0, 0.0};
    u = sub(u, mul(n2, dot(u, n2)));
    u = mul(u, 1.0 / norm(u));
    const V3 v = cross(n2, u);
    const V3 seed = add(c2, mul(add(mul(u, tab.c[k]), mul(v, tab.s[k])), r2));
    bool conv;
    return alternate(c1, n1, r1, c2, n2, r2, seed, disks_tol(r1, r2), 64, &conv) <= threshold;
}

SRM_HD bool disks_within(V3 c1, V3 n1, double r1, V3 c2, V3 n2, double r2, double threshold, const SeedTable& tab) {
    const int st = disks_within_pre(c1, n1, r1, c2, n2, r2, threshold);
    if (st != kDwSeeds) return st == kDwTrue;
    for (int k = 0; k < kSeeds; ++k)
        if (rim_seed_within(c1, n1, r1, c2, n2, r2, threshold, tab, k)) return true;
    return false;
}

// spherodisk.hpp:25 and 62-68: platelets a, b (centres pa, pb already wrapped;
// d = min_image(pb - pa)) overlap when the medial disks are within the sweep radii
SRM_HD bool spherodisk_overlap(V3 d, V3 na, double Da, double ta, V3 nb, double Db, double tb, const SeedTable& tab) {
    const double cull = 0.5 * (Da + Db + ta + tb);
    if (dot(d, d) > cull * cull) return false;
    return disks_within(V3{0.0, 0.0, 0.0}, na, 0.5 * (Da - ta), d, nb, 0.5 * (Db - tb), 0.5 * (ta + tb), tab);
}

// spherodisk_overlap's first stage (disks_within_pre of the same medial disks)
SRM_HD int spherodisk_overlap_pre(V3 d, V3 na, double Da, double ta, V3 nb, double Db, double tb) {
    const double cull = 0.5 * (Da + Db + ta + tb);
    if (dot(d, d) > cull * cull) return kDwFalse;
    return disks_within_pre(V3{0.0, 0.0, 0.0}, na, 0.5 * (Da - ta), d, nb, 0.5 * (Db - tb), 0.5 * (ta + tb));
}

// spherodisk.hpp:29-34 swept-solid volume
SRM_HD double spherodisk_measure(double D, double t) {
    constexpr double pi = 3.141592653589793238462643383279502884;
    const double a = 0.5 * (D - t);
    const double s = 0.5 * t;
    return 2.0 * pi * a * a * s + pi * pi * a * s * s + (4.0 / 3.0) * pi * s * s * s;
}

// spherodisk.hpp:49-53 Rodrigues rotation with cos/sin of the angle given
SRM_HD V3 rotate_about_axis(V3 v, V3 axis, double c, double s) {
    return add(add(mul(v, c), mul(cross(axis, v), s)), mul(axis, dot(axis, v) * (1.0 - c)));
}

// spherodisk.hpp:85-91 the rotated normal, renormalised
SRM_HD V3 rotate_normal(V3 n, V3 axis, double c, double s) {
    const V3 r = rotate_about_axis(n, axis, c, s);
    return mul(r, 1.0 / norm(r));
}

}  // namespace pl
}  // namespace srmb
