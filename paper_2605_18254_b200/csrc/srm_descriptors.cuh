// srm_descriptors.cuh -- the end-to-end parity statistics on the device (SURVEY.md §8f
// row 3): nearest-neighbour distances (descriptors.hpp:28-115), the reference's
// fixed-range histogram (descriptors.hpp:251-277) and radial pair-distance counts (the
// RDF of the parity tests; the reference has none).  All three run on the
// context's sorted cell grid (any cell size: the answers do not depend on it) and are
// exact: the NND is sqrt of the minimum squared min-image distance over all other
// centres, which is what the reference's ring search returns; the pair counts bin every
// unordered pair once, with numpy.histogram's edge rule (tests/stats_util.py).
#pragma once

#include "srm_kernels.cuh"

namespace srmb {

// Cells at Chebyshev distance exactly r from cell c, as contiguous sorted ranges (x runs
// per (y, z) row).  Requires 2 r + 1 <= dims on every axis (no cell visited twice).
template <int D, typename F>
__device__ __forceinline__ void for_ring_ranges(const GridParams& g, const cell_t* __restrict__ cs, const int* c, int r,
                                                F&& f) {
    const int dx = g.dims[0], dy = g.dims[1], dz = D == 3 ? g.dims[2] : 1;
    const int rz = D == 3 ? r : 0;
    for (int oz = -rz; oz <= rz; ++oz) {
        int z = c[2] + oz;
        z = z < 0 ? z + dz : (z >= dz ? z - dz : z);
        for (int oy = -r; oy <= r; ++oy) {
            int y = c[1] + oy;
            y = y < 0 ? y + dy : (y >= dy ? y - dy : y);
            const int64_t row = (static_cast<int64_t>(z) * dy + y) * dx;
            const bool shell = (D == 3 && (oz == -r || oz == r)) || oy == -r || oy == r;
            auto xrun = [&](int xl, int xr) {  // unwrapped [xl, xr]
                if (xl < 0 && xr >= 0) {
                    f(cs[row + xl + dx], cs[row + dx]);
                    f(cs[row], cs[row + xr + 1]);
                } else if (xr >= dx && xl < dx) {
                    f(cs[row + xl], cs[row + dx]);
                    f(cs[row], cs[row + xr - dx + 1]);
                } else {
                    const int a = xl < 0 ? xl + dx : (xl >= dx ? xl - dx : xl);
                    f(cs[row + a], cs[row + a + (xr - xl) + 1]);
                }
            };
            if (shell) {
                xrun(c[0] - r, c[0] + r);
            } else {
                xrun(c[0] - r, c[0] - r);
                if (r > 0) xrun(c[0] + r, c[0] + r);
            }
        }
    }
}

// NND of sorted particle q, out[slot] = sqrt(min over j != q of min_image_dist2).  Rings
// r = 0, 1, ... until the best squared distance is below (r edge_min)^2 (every unvisited
// cell is at least r cells away along some axis: descriptors.hpp:68-73); a grid too small
// for the next ring falls back to all particles.
// nn_align (platelets, optional): |n_q . n_j| of the nearest neighbour j found (the first
// at the minimum distance in scan order), by slot -- the nearest-neighbour alignment of
// the platelet parity summaries.
template <int D>
__global__ void __launch_bounds__(256) k_nnd(int64_t n, State S, Box box, const GridParams* __restrict__ gp,
                                             const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                             double* __restrict__ out, double* __restrict__ nn_align = nullptr) {
    const GridParams& g = *gp;
    double emin = g.edge[0];
    for (int a = 1; a < D; ++a) emin = g.edge[a] < emin ? g.edge[a] : emin;
    int dmin = g.dims[0];
    for (int a = 1; a < D; ++a) dmin = g.dims[a] < dmin ? g.dims[a] : dmin;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        double x[D];
        rec_pos<D>(S.rec[q], x);
        int c[3];
        decode_key<D>(g, skey[q], c);
        double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
        int64_t arg = -1;
        auto scan = [&](int64_t b, int64_t e) {
            for (int64_t j = b; j < e; ++j) {
                if (j == q) continue;
                double y[D];
                rec_pos<D>(S.rec[j], y);
                const double d2 = dist2<D>(box, x, y);
                if (d2 < best) {
                    best = d2;
                    arg = j;
                }
            }
        };
        bool done = false;
        for (int r = 0; !done; ++r) {
            if (2 * r + 1 > dmin) {  // the ring would alias through the periodic wrap: all
                best = __longlong_as_double(0x7ff0000000000000LL);
                scan(0, n);
                break;
            }
            for_ring_ranges<D>(g, cs, c, r, scan);
            const double bound = static_cast<double>(r) * emin;
            done = best < bound * bound;
        }
        out[S.slot[q]] = sqrt(best);
        if (nn_align) {
            double a = __longlong_as_double(0x7ff8000000000000LL);  // NaN: no neighbour
            if (arg >= 0) {
                const double4 u = S.aux[q], w = S.aux[arg];
                a = fabs(u.x * w.x + u.y * w.y + u.z * w.z);
            }
            nn_align[S.slot[q]] = a;
        }
    }
}

// descriptors.hpp:182-209 local_nematic_order: per platelet the mean |n_i . n_j| over the
// platelets whose centre lies within `cutoff` (NaN when none) and their number, by slot.
// The grid's cells are at least `cutoff` wide, so the one-cell stencil `s` holds them all.
__global__ void __launch_bounds__(256) k_local_nematic(int64_t n, State S, Box box, const GridParams* __restrict__ gp,
                                                       const cell_t* __restrict__ cs,
                                                       const uint32_t* __restrict__ skey, const int32_t* s,
                                                       double cutoff, double* __restrict__ value,
                                                       int32_t* __restrict__ count) {
    const GridParams& g = *gp;
    const double cut2 = cutoff * cutoff;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        double x[3];
        rec_pos<3>(S.rec[q], x);
        const double4 u = S.aux[q];
        double acc = 0.0;
        int cnt = 0;
        for_near_ranges<3>(g, cs, skey[q], s, [&](int64_t b0, int64_t e0) {
            for (int64_t j = b0; j < e0; ++j) {
                if (j == q) continue;
                double y[3];
                rec_pos<3>(S.rec[j], y);
                if (dist2<3>(box, x, y) <= cut2) {
                    const double4 w = S.aux[j];
                    acc += fabs(u.x * w.x + u.y * w.y + u.z * w.z);
                    ++cnt;
                }
            }
        });
        const int32_t sl = S.slot[q];
        count[sl] = cnt;
        value[sl] = cnt > 0 ? acc / cnt : __longlong_as_double(0x7ff8000000000000LL);
    }
}

// Sum of n (x) n over the platelets (xx, yy, zz, xy, xz, yz) in a fixed order: per-block
// partials, finished on the host -- the Q tensor of the nematic order parameter S2.
__global__ void __launch_bounds__(256) k_q_tensor(int64_t n, const double4* __restrict__ aux,
                                                  double* __restrict__ part) {
    __shared__ double ss[6][256];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = b0 + chunk < n ? b0 + chunk : n;
    double a[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t i = b0 + threadIdx.x; i < b1; i += 256) {
        const double4 u = aux[i];
        a[0] += u.x * u.x;
        a[1] += u.y * u.y;
        a[2] += u.z * u.z;
        a[3] += u.x * u.y;
        a[4] += u.x * u.z;
        a[5] += u.y * u.z;
    }
    for (int k = 0; k < 6; ++k) ss[k][threadIdx.x] = a[k];
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (static_cast<int>(threadIdx.x) < w)
            for (int k = 0; k < 6; ++k) ss[k][threadIdx.x] += ss[k][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = ss[threadIdx.x][0];
}

// descriptors.hpp:254-277 histogram over [lo, hi] (top edge inclusive, non-finite values
// ignored): counts[bins], then total and in_range.
__global__ void k_histogram(int64_t n, const double* __restrict__ v, int bins, double lo, double hi,
                            unsigned long long* __restrict__ counts, unsigned long long* __restrict__ tot) {
    const double width = (hi - lo) / bins;
    unsigned long long total = 0, inr = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = v[i];
        if (!isfinite(x)) continue;
        ++total;
        if (x < lo || x > hi) continue;
        int64_t b = static_cast<int64_t>((x - lo) / width);
        if (b >= bins) b = bins - 1;
        atomicAdd(&counts[b], 1ull);
        ++inr;
    }
    atomicAdd(&tot[0], total);
    atomicAdd(&tot[1], inr);
}

// Unordered pair distances |x_i - x_j| (min image, ((dx^2 + dy^2) + dz^2)) binned like
// numpy.histogram on the edges e[0..bins] (uniform: index from the scaled offset, then
// corrected against the edges; the last bin includes e[bins]).  Each pair counted once,
// by the lower sorted index; stencil half width s = the cells within e[bins].
template <int D>
__global__ void __launch_bounds__(256) k_pair_counts(int64_t n, State S, Box box, const GridParams* __restrict__ gp,
                                                     const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                                     const double* __restrict__ edges, int bins, const int32_t* s,
                                                     unsigned long long* __restrict__ counts) {
    extern __shared__ unsigned long long hcount[];
    for (int b = threadIdx.x; b < bins; b += blockDim.x) hcount[b] = 0;
    __syncthreads();
    const GridParams& g = *gp;
    const double lo = edges[0], hi = edges[bins];
    const double norm = bins / (hi - lo);
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        double x[D];
        rec_pos<D>(S.rec[q], x);
        for_near_ranges<D>(g, cs, skey[q], s, [&](int64_t b0, int64_t e0) {
            for (int64_t j = b0 > q + 1 ? b0 : q + 1; j < e0; ++j) {
                double y[D];
                rec_pos<D>(S.rec[j], y);
                const double r = sqrt(dist2<D>(box, x, y));
                if (!(r >= lo && r <= hi)) continue;
                int k = static_cast<int>((r - lo) * norm);
                if (k >= bins) k = bins - 1;
                if (r < edges[k]) --k;
                else if (k < bins - 1 && r >= edges[k + 1]) ++k;
                atomicAdd(&hcount[k], 1ull);
            }
        });
    }
    __syncthreads();
    for (int b = threadIdx.x; b < bins; b += blockDim.x)
        if (hcount[b]) atomicAdd(&counts[b], hcount[b]);
}

}  // namespace srmb
