// srm_device.cuh -- device-side primitives of the B200 SRM hot loop.
//
// Everything here is compiled with --fmad=false: each double operation is one IEEE
// correctly rounded operation in the order written, matching the reference's
// non-contracted x86-64 build (no -march, so no FMA) operation for operation.
#pragma once

#include <cstdint>

// Checked build (-DSRM_B200_CHECKED, tools/build_variant.sh): index bounds of the hot
// kernels, a message and a trap on the first violation.  compute-sanitizer is closed on
// the GPU pool this was developed on (profiles/r11_sanitizer_refused.log); the GPU parity
// tests run once under this build instead (profiles/r16_checked_build.log).
#ifdef SRM_B200_CHECKED
#include <cstdio>
#define SRM_CHK(cond, code)                                                                           \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("SRM_CHK %d failed at %s:%d (block %d thread %d)\n", code, __FILE__, __LINE__,     \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                      \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define SRM_CHK(cond, code) ((void)0)
#endif

namespace srmb {

constexpr uint8_t kNotAccepted = 255;

struct Box {
    double L[3];
    double half[3];  // 0.5 * L, as geometry.hpp:120 computes it
};

// geometry.hpp:107-114 PeriodicBox::wrap -- two sequential conditional shifts.
__host__ __device__ __forceinline__ double wrap1(double p, double L) {
    if (p < 0.0) p += L;
    if (p >= L) p -= L;
    return p;
}

// geometry.hpp:117-125 single-shift min_image along one axis.
__host__ __device__ __forceinline__ double min_image1(double d, double L, double half) {
    if (d > half) d -= L;
    if (d < -half) d += L;
    return d;
}

// geometry.hpp:127-129 + 44-49: s = 0; s += dx*dx; s += dy*dy; (s += dz*dz)
template <int D>
__host__ __device__ __forceinline__ double dist2(const Box& b, const double* a, const double* c) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double d = min_image1(a[k] - c[k], b.L[k], b.half[k]);
        s += d * d;
    }
    return s;
}

// shape.hpp:34-37 SphereShape::overlap -- contact counts as overlap.
template <int D>
__host__ __device__ __forceinline__ bool sphere_overlap(const Box& b, const double* a, double ra,
                                                        const double* c, double rc) {
    const double rr = ra + rc;
    return dist2<D>(b, a, c) <= rr * rr;
}

// ---------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  Pinned against curand_Philox4x32_10 and the
// Random123 known-answer vectors in tests/test_oracle_pins.py.
struct U4 {
    uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Counter layout:
//   key = (lo32(seed), hi32(seed))
//   ctr = (slot, attempt, (round_id & 0xFFFFFF) | stream << 24 | draw << 25, iteration)
struct RngKey {
    uint32_t k0, k1;
    uint32_t round_id;   // already masked to 24 bits
    uint32_t iteration;  // low 32 bits of the global iteration count
};

// Unit vector with only +,-,*,/,sqrt (bit-identical to oracle/srm_oracle.c):
//   3D Marsaglia (1972); 2D normalised point in the unit disk.
// one rejection draw: the point (x1, x2) of draw `draw` and its squared norm s
__device__ __forceinline__ double draw_point(const RngKey& key, uint32_t slot, uint32_t attempt, uint32_t stream,
                                             uint32_t draw, double* x1, double* x2) {
    const U4 o = philox4x32_10(U4{slot, attempt, key.round_id | (stream << 24) | (draw << 25), key.iteration},
                               key.k0, key.k1);
    const uint64_t a = ((static_cast<uint64_t>(o.x) << 32) | o.y) >> 11;
    const uint64_t b = ((static_cast<uint64_t>(o.z) << 32) | o.w) >> 11;
    *x1 = __dsub_rn(__dmul_rn(__ull2double_rn(a), 0x1p-52), 1.0);
    *x2 = __dsub_rn(__dmul_rn(__ull2double_rn(b), 0x1p-52), 1.0);
    return __dadd_rn(__dmul_rn(*x1, *x1), __dmul_rn(*x2, *x2));
}

template <int D>
__device__ __forceinline__ bool draw_ok(double s) {
    return D == 3 ? s < 1.0 : (s < 1.0 && s > 1e-24);
}

template <int D>
__device__ __forceinline__ void point_to_unit(double x1, double x2, double s, double* u) {
    if constexpr (D == 3) {
        const double q = __dmul_rn(2.0, __dsqrt_rn(__dsub_rn(1.0, s)));
        u[0] = __dmul_rn(x1, q);
        u[1] = __dmul_rn(x2, q);
        u[2] = __dsub_rn(1.0, __dmul_rn(2.0, s));
    } else {
        const double inv = __ddiv_rn(1.0, __dsqrt_rn(s));
        u[0] = __dmul_rn(x1, inv);
        u[1] = __dmul_rn(x2, inv);
    }
}

// The first accepted of draws 0, 1, 2, ... (< 64).  SRM_DRAW_PAIRS: draws 0 and 1 are
// computed together (no divergence for the ~21% of 3D trials whose first draw is
// rejected, at the price of a second Philox call for the other 79%).
#ifndef SRM_DRAW_PAIRS
#define SRM_DRAW_PAIRS 0
#endif
template <int D>
__device__ __forceinline__ void unit_vector(const RngKey& key, uint32_t slot, uint32_t attempt,
                                            uint32_t stream, double* u) {
    if (!SRM_DRAW_PAIRS) {
        for (uint32_t draw = 0; draw < 64; ++draw) {
            double x1, x2;
            const double s = draw_point(key, slot, attempt, stream, draw, &x1, &x2);
            if (draw_ok<D>(s)) {
                point_to_unit<D>(x1, x2, s, u);
                return;
            }
        }
        u[0] = 1.0;
#pragma unroll
        for (int k = 1; k < D; ++k) u[k] = 0.0;
        return;
    }
    double a1, a2, b1, b2;
    const double sa = draw_point(key, slot, attempt, stream, 0, &a1, &a2);
    const double sb = draw_point(key, slot, attempt, stream, 1, &b1, &b2);
    if (draw_ok<D>(sa)) {
        point_to_unit<D>(a1, a2, sa, u);
        return;
    }
    if (draw_ok<D>(sb)) {
        point_to_unit<D>(b1, b2, sb, u);
        return;
    }
    for (uint32_t draw = 2; draw < 64; ++draw) {
        const double s = draw_point(key, slot, attempt, stream, draw, &a1, &a2);
        if (draw_ok<D>(s)) {
            point_to_unit<D>(a1, a2, s, u);
            return;
        }
    }
    u[0] = 1.0;
#pragma unroll
    for (int k = 1; k < D; ++k) u[k] = 0.0;
}

// shape.hpp:39-44 propose_move: wrap(p + c_m * u) (component-wise u*c_m then x+step)
template <int D>
__device__ __forceinline__ void propose(const Box& b, const double* x, double c_m,
                                        const RngKey& key, uint32_t slot, uint32_t attempt,
                                        double* out) {
    double u[D];
    unit_vector<D>(key, slot, attempt, 0, u);
#pragma unroll
    for (int k = 0; k < D; ++k) out[k] = wrap1(__dadd_rn(x[k], __dmul_rn(u[k], c_m)), b.L[k]);
}

}  // namespace srmb
