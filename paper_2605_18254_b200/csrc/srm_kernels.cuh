// srm_kernels.cuh -- CUDA kernels of the B200 SRM round (sm_100a).
//
// One SRM round (engine.hpp:227-234: build_shape_grid -> migrate -> shape_any_collision)
// is, on the device:
//   grid rebuild   k_keys -> k_scan_* -> k_scatter -> k_cellsort -> k_gather
//   near lists     k_near_lists (round-start neighbours within the trial reach)
//   migrate        k_sweep_cells, one launch per (superblock colour, colour class)
//   reduction      k_stats_sweep (overlap pairs, max penetration over the non-movers)
// All kernels read the grid / round parameters from device memory so that the same
// launches can be replayed from a CUDA graph.  DESIGN.md §2-§4 has the data layout
// and the roofline of each kernel.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>

#include "srm_device.cuh"

namespace srmb {

constexpr int kScanTile = 4096;  // cells per scan tile (1024 threads x 4)

struct GridParams {
    int32_t dims[3];
    double edge[3];
    int64_t ncells;
    int32_t near_s[3];  // near-search half width per axis; -1 = every cell on the axis
    double extra;       // near cutoff: (ri + rj + extra) * (1 + 1e-9) + 1e-300
    double rmax;        // largest radius of the state the grid indexes
    int32_t col_m[3];   // colouring modulus per axis
    int32_t col_n[3];   // colours per axis
    int32_t ncls;       // colour classes = col_n[0] * col_n[1] * col_n[2]
    int64_t cls_cells;  // largest number of cells in one class
    // fp32 prefilter (near_candidates): margin above the fp32 rounding of coordinates
    float margin_f, extra_f, rmax_f;
    float L_f[3], half_f[3], edge_f[3];
    int32_t nsb[3];     // superblocks per axis (even, or 1), DESIGN.md §3.1
};

struct RoundParams {
    double c_m;
    int32_t n_l;
    RngKey key;
};

// Per-particle SoA record set.  x[a] for a < D.
struct State {
    double* x[3];
    double* r;
    int32_t* id;
    int32_t* slot;
    float4* xf;  // sorted fp32 copy (x, y, z, r) for prefilters; only in the sorted state S
    double4* lv; // live record (x, y, z, r) during the sweep, one 32-byte sector; only in S
};

struct StatsDev {
    unsigned long long overlap_pairs;
    unsigned long long pen_bits;  // max penetration as the bits of a non-negative double
    unsigned long long candidate_pairs;
    unsigned long long active_count;  // non-movers: particles that kept their round-start position
};

__device__ __forceinline__ double near_cut(double ri, double rj, double extra) {
    const double c = __dadd_rn(__dmul_rn(__dadd_rn(__dadd_rn(ri, rj), extra), 1.0 + 1e-9), 1e-300);
    return __dmul_rn(c, c);
}

// ---------------------------------------------------------------------------------
// Grid: cell_grid.hpp:319-336 cell_coords + flat_index, bit for bit.
template <int D>
__device__ __forceinline__ uint32_t cell_of(const GridParams& g, const double* p) {
    uint64_t idx = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
        int i = static_cast<int>(floor(__ddiv_rn(p[a], g.edge[a])));
        i %= g.dims[a];
        if (i < 0) i += g.dims[a];
        idx = idx * static_cast<uint64_t>(g.dims[a]) + static_cast<uint64_t>(i);
    }
    return static_cast<uint32_t>(idx);
}

template <int D>
__global__ void k_keys(int64_t n, State T, const GridParams* __restrict__ gp,
                       uint32_t* __restrict__ key, uint32_t* __restrict__ count) {
    const GridParams g = *gp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double p[D];
#pragma unroll
        for (int a = 0; a < D; ++a) p[a] = T.x[a][i];
        const uint32_t k = cell_of<D>(g, p);
        key[i] = k;
        atomicAdd(&count[k], 1u);
    }
}

// ---- exclusive scan of count[ncells] -> cell_start[ncells+1] (3 passes) ----------
__global__ void k_scan_tiles(const uint32_t* __restrict__ count, const GridParams* __restrict__ gp,
                             uint64_t* __restrict__ partial) {
    const int64_t ncells = gp->ncells;
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint64_t s = 0;
    if (base < ncells) {
#pragma unroll
        for (int k = 0; k < kScanTile / 1024; ++k) {
            const int64_t c = base + (int64_t)k * 1024 + threadIdx.x;
            if (c < ncells) s += count[c];
        }
    }
    // block reduce
    __shared__ uint64_t red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint64_t v = red[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) partial[blockIdx.x] = v;
    }
}

// single block: exclusive scan of the tile sums, in chunks of 1024
__global__ void k_scan_partials(uint64_t* __restrict__ partial, int64_t ntiles_cap,
                                const GridParams* __restrict__ gp, int64_t* __restrict__ cell_start) {
    const int64_t ncells = gp->ncells;
    const int64_t ntiles = (ncells + kScanTile - 1) / kScanTile;
    (void)ntiles_cap;
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t carry_s;
    if (threadIdx.x == 0) carry_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t b0 = 0; b0 < ntiles; b0 += 1024) {
        const int64_t t = b0 + threadIdx.x;
        const uint64_t v = t < ntiles ? partial[t] : 0;
        uint64_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const uint64_t w = warp_tot[lane];
            uint64_t wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t u = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += u;
            }
            warp_tot[lane] = wi - w;
        }
        __syncthreads();
        const uint64_t carry = carry_s;
        const uint64_t excl = carry + warp_tot[wid] + incl - v;
        if (t < ntiles) partial[t] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry_s = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) cell_start[ncells] = (int64_t)carry_s;
}

__global__ void k_scan_down(const uint32_t* __restrict__ count, const uint64_t* __restrict__ partial,
                            const GridParams* __restrict__ gp, int64_t* __restrict__ cell_start) {
    const int64_t ncells = gp->ncells;
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    if (base >= ncells) return;
    __shared__ uint64_t warp_tot[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // thread t owns cells base + 4t .. base + 4t + 3 (contiguous)
    uint32_t v[4];
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t c = base + 4 * (int64_t)threadIdx.x + k;
        v[k] = c < ncells ? count[c] : 0u;
        s += v[k];
    }
    uint64_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint64_t w = warp_tot[lane];
        uint64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t u = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += u;
        }
        warp_tot[lane] = wi - w;
    }
    __syncthreads();
    uint64_t run = partial[blockIdx.x] + warp_tot[wid] + incl - s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t c = base + 4 * (int64_t)threadIdx.x + k;
        if (c < ncells) cell_start[c] = (int64_t)run;
        run += v[k];
    }
}

// atomic scatter into cell ranges; count[] returns to zero for the next histogram
__global__ void k_scatter(int64_t n, const uint32_t* __restrict__ key,
                          const int64_t* __restrict__ cell_start, uint32_t* __restrict__ count,
                          int32_t* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key[i];
        const uint32_t r = atomicSub(&count[k], 1u) - 1u;
        perm[cell_start[k] + r] = static_cast<int32_t>(i);
    }
}

// deterministic within-cell order: ascending slot (== engine.hpp:151-163 stability
// when slot is the storage index)
__global__ void k_cellsort(const GridParams* __restrict__ gp, const int64_t* __restrict__ cell_start,
                           const int32_t* __restrict__ slot, int32_t* __restrict__ perm) {
    const int64_t ncells = gp->ncells;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncells;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = cell_start[c], e = cell_start[c + 1];
        if (e - b < 2) continue;
        for (int64_t q = b + 1; q < e; ++q) {
            const int32_t v = perm[q];
            const int32_t sv = slot[v];
            int64_t k = q - 1;
            while (k >= b && slot[perm[k]] > sv) {
                perm[k + 1] = perm[k];
                --k;
            }
            perm[k + 1] = v;
        }
    }
}

template <int D>
__global__ void k_gather(int64_t n, const int32_t* __restrict__ perm, const uint32_t* __restrict__ key,
                         State T, State S, uint32_t* __restrict__ skey) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t src = perm[q];
        float f[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int a = 0; a < D; ++a) {
            const double v = T.x[a][src];
            S.x[a][q] = v;
            f[a] = static_cast<float>(v);
        }
        const double rr = T.r[src];
        S.r[q] = rr;
        f[3] = static_cast<float>(rr);
        if (S.xf) S.xf[q] = make_float4(f[0], f[1], f[2], f[3]);
        if (S.lv) S.lv[q] = make_double4(S.x[0][q], D > 1 ? S.x[1][q] : 0.0, D > 2 ? S.x[2][q] : 0.0, rr);
        S.id[q] = T.id[src];
        S.slot[q] = T.slot[src];
        skey[q] = key[src];
    }
}

// ---------------------------------------------------------------------------------
// Stencil walk over the sorted cell ranges around cell `k`: half width g.near_s[a]
// (or the whole axis), x-runs merged into contiguous particle ranges.
template <int D, typename F>
__device__ __forceinline__ void for_near_ranges(const GridParams& g, const int64_t* __restrict__ cs,
                                                uint32_t k, const int32_t* s, F&& f) {
    const int dx = g.dims[0], dy = g.dims[1], dz = D == 3 ? g.dims[2] : 1;
    const int cx = static_cast<int>(k % static_cast<uint32_t>(dx));
    const uint32_t rest = k / static_cast<uint32_t>(dx);
    const int cy = static_cast<int>(rest % static_cast<uint32_t>(dy));
    const int cz = D == 3 ? static_cast<int>(rest / static_cast<uint32_t>(dy)) : 0;
    const bool fy = s[1] < 0, fz = D == 3 ? s[2] < 0 : true;
    const int ylo = fy ? 0 : cy - s[1], yhi = fy ? dy - 1 : cy + s[1];
    const int zlo = D == 3 ? (fz ? 0 : cz - s[2]) : 0, zhi = D == 3 ? (fz ? dz - 1 : cz + s[2]) : 0;
    for (int zz = zlo; zz <= zhi; ++zz) {
        int z = zz;
        if (z < 0) z += dz;
        if (z >= dz) z -= dz;
        for (int yy = ylo; yy <= yhi; ++yy) {
            int y = yy;
            if (y < 0) y += dy;
            if (y >= dy) y -= dy;
            const int64_t row = ((int64_t)z * dy + y) * dx;
            if (s[0] < 0) {
                f(cs[row], cs[row + dx]);
            } else {
                const int lo = cx - s[0], hi = cx + s[0];
                if (lo < 0) {
                    f(cs[row + lo + dx], cs[row + dx]);
                    f(cs[row], cs[row + hi + 1]);
                } else if (hi >= dx) {
                    f(cs[row + lo], cs[row + dx]);
                    f(cs[row], cs[row + hi - dx + 1]);
                } else {
                    f(cs[row + lo], cs[row + hi + 1]);
                }
            }
        }
    }
}

template <int D>
__device__ __forceinline__ void load_pos(const State& S, int64_t i, double* p) {
#pragma unroll
    for (int a = 0; a < D; ++a) p[a] = S.x[a][i];
}

// ---------------------------------------------------------------------------------
// Migrate: coloured Gauss-Seidel sweep.
//
// The reference's migrate (engine.hpp:89-107) visits particles in storage order; each
// gets <= n_l trials from its pre-sweep position and keeps the first one that clears the
// LIVE positions of all others.  Here the visiting order is (superblock colour,
// superblock, colour class, cell, slot): cells are coloured so that two cells of one
// class are farther apart than any trial can reach (GridParams::col_*), and superblocks
// of one colour are a whole superblock apart (GridParams::nsb), hence one superblock
// colour is one launch with a CTA per superblock and a thread per cell of a class,
// particles of a cell sequentially in slot order; the result is identical to the
// sequential sweep in that order (oracle/srm_oracle.c orc_sweep_round).
//
// Live positions: S.lv[j] holds (x, r) of j -- its round-start position, overwritten by
// its accepted trial when j moves; one 32-byte sector per neighbour read.

constexpr int kNearLocal = 16;  // near candidates kept per particle; more -> rescan per trial

// Near candidates of sorted particle q: every j whose round-start distance is within
// ri + rj + 2 c_m (every j a trial of q can touch while j sits within c_m of its start).
// fp32 prefilter on the sorted float4 copy with an absolute margin above its rounding
// error, so the set is a superset of the exact fp64 near set; the stencil rows and the
// x cells of each row are pruned by the chord of the (inflated) cutoff sphere.
template <int D, typename F>
__device__ __forceinline__ void near_candidates(const GridParams& g, const int64_t* __restrict__ cs,
                                                const float4* __restrict__ xf, int64_t q, uint32_t key, F&& visit) {
    const float4 me = xf[q];
    const int dx = g.dims[0], dy = g.dims[1], dz = D == 3 ? g.dims[2] : 1;
    const int cx = static_cast<int>(key % static_cast<uint32_t>(dx));
    const uint32_t rest = key / static_cast<uint32_t>(dx);
    const int cy = static_cast<int>(rest % static_cast<uint32_t>(dy));
    const int cz = D == 3 ? static_cast<int>(rest / static_cast<uint32_t>(dy)) : 0;
    const float cutm = __fadd_rn(__fadd_rn(__fadd_rn(me.w, g.rmax_f), g.extra_f), __fmul_rn(2.f, g.margin_f));
    const float cut2 = __fmul_rn(__fmul_rn(cutm, cutm), 1.00001f);
    const float base = __fadd_rn(__fadd_rn(me.w, g.extra_f), g.margin_f);  // + r_j
    // y / z rows: unwrapped range [c - s, c + s], or every row when the stencil covers the axis
    const int sy = g.near_s[1], sz = D == 3 ? g.near_s[2] : 0;
    const int ylo = sy < 0 ? 0 : cy - sy, yhi = sy < 0 ? dy - 1 : cy + sy;
    const int zlo = D == 3 ? (sz < 0 ? 0 : cz - sz) : 0, zhi = D == 3 ? (sz < 0 ? dz - 1 : cz + sz) : 0;
    for (int zz = zlo; zz <= zhi; ++zz) {
        float dzd = 0.f;
        if (D == 3 && sz >= 0) {
            const float zb = zz * g.edge_f[2];
            dzd = fmaxf(0.f, fmaxf(zb - me.z, me.z - (zb + g.edge_f[2])));
        }
        const int z = zz < 0 ? zz + dz : (zz >= dz ? zz - dz : zz);
        for (int yy = ylo; yy <= yhi; ++yy) {
            float dyd = 0.f;
            if (sy >= 0) {
                const float yb = yy * g.edge_f[1];
                dyd = fmaxf(0.f, fmaxf(yb - me.y, me.y - (yb + g.edge_f[1])));
            }
            const float dyz2 = __fmaf_rn(dyd, dyd, __fmul_rn(dzd, dzd));
            if (dyz2 > cut2) continue;
            const int y = yy < 0 ? yy + dy : (yy >= dy ? yy - dy : yy);
            const int64_t row = (static_cast<int64_t>(z) * dy + y) * dx;
            auto run = [&](int64_t b, int64_t e) {
                for (int64_t j = b; j < e; ++j) {
                    const float4 c = xf[j];
                    float ex = c.x - me.x, ey = c.y - me.y, ez = D == 3 ? c.z - me.z : 0.f;
                    if (ex > g.half_f[0]) ex -= g.L_f[0]; else if (ex < -g.half_f[0]) ex += g.L_f[0];
                    if (ey > g.half_f[1]) ey -= g.L_f[1]; else if (ey < -g.half_f[1]) ey += g.L_f[1];
                    if (D == 3) { if (ez > g.half_f[2]) ez -= g.L_f[2]; else if (ez < -g.half_f[2]) ez += g.L_f[2]; }
                    const float d2 = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
                    const float lim = __fadd_rn(base, c.w);
                    if (d2 > __fmul_rn(__fmul_rn(lim, lim), 1.00001f) || j == q) continue;
                    visit(j);
                }
            };
            const int sx = g.near_s[0];
            if (sx < 0) {
                run(cs[row], cs[row + dx]);
                continue;
            }
            const float xh = __fadd_rn(__fsqrt_rn(__fsub_rn(cut2, dyz2)), g.margin_f);
            const int xl = max(cx - sx, static_cast<int>(floorf(__fdiv_rn(__fsub_rn(me.x, xh), g.edge_f[0]))));
            const int xr = min(cx + sx, static_cast<int>(ceilf(__fdiv_rn(__fadd_rn(me.x, xh), g.edge_f[0]))) - 1);
            if (xl > xr) continue;
            if (xl < 0) {
                run(cs[row + xl + dx], cs[row + dx]);
                run(cs[row], cs[row + xr + 1]);
            } else if (xr >= dx) {
                run(cs[row + xl], cs[row + dx]);
                run(cs[row], cs[row + xr - dx + 1]);
            } else {
                run(cs[row + xl], cs[row + xr + 1]);
            }
        }
    }
}

constexpr uint8_t kNearOverflow = 255;

// Near lists of every particle, one parallel pass before the sweep: nbr[q*kNearLocal..]
// and nbr_cnt[q] (kNearOverflow: more than kNearLocal, the sweep rescans the grid).
template <int D>
__global__ void __launch_bounds__(256) k_near_lists(int64_t n, State S, const GridParams* __restrict__ gp,
                                                    const int64_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                                    int32_t* __restrict__ nbr, uint8_t* __restrict__ nbr_cnt) {
    const GridParams& g = *gp;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        int32_t* my = nbr + q * kNearLocal;
        int nn = 0;
        const int32_t idq = S.id[q];
        near_candidates<D>(g, cs, S.xf, q, skey[q], [&](int64_t j) {
            if (S.id[j] == idq) return;  // shape.hpp:544 self-exclusion by id
            if (nn < kNearLocal) my[nn] = static_cast<int32_t>(j);
            ++nn;
        });
        nbr_cnt[q] = nn > kNearLocal ? kNearOverflow : static_cast<uint8_t>(nn);
    }
}

template <int D>
__device__ __forceinline__ void sweep_particle(int64_t q, const State& S, const State& T, const Box& box,
                                               const GridParams& g, const RoundParams& rp,
                                               const int64_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                               const int32_t* __restrict__ nbr, const uint8_t* __restrict__ nbr_cnt,
                                               uint8_t* __restrict__ acc, int32_t* __restrict__ active,
                                               StatsDev* stats) {
    const int nn = nbr_cnt[q];
    double xi[D];
    load_pos<D>(S, q, xi);
    const double ri = S.r[q];
    const int32_t sl = S.slot[q];
    double p[D];
    int accepted = -1;
    if (nn != kNearOverflow) {
        // the near list once (64 B, four 16-byte loads); per trial every record load is
        // issued before any test (no early exit), kBatch at a time, so a trial costs one
        // memory latency per batch instead of one per neighbour
        constexpr int kBatch = 4;
        int32_t nb[kNearLocal];
        const int4* nb4 = reinterpret_cast<const int4*>(nbr + q * kNearLocal);
#pragma unroll
        for (int c = 0; c < kNearLocal / 4; ++c) {
            int4 v = make_int4(0, 0, 0, 0);
            if (4 * c < nn) v = nb4[c];
            nb[4 * c] = v.x; nb[4 * c + 1] = v.y; nb[4 * c + 2] = v.z; nb[4 * c + 3] = v.w;
        }
        for (int l = 0; l < rp.n_l && accepted < 0; ++l) {
            propose<D>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), p);
            bool hit = false;
#pragma unroll
            for (int t0 = 0; t0 < kNearLocal; t0 += kBatch) {
                if (t0 < nn) {
                    double4 v[kBatch];
#pragma unroll
                    for (int u = 0; u < kBatch; ++u)
                        if (t0 + u < nn) v[u] = S.lv[nb[t0 + u]];
#pragma unroll
                    for (int u = 0; u < kBatch; ++u) {
                        if (t0 + u < nn) {
                            const double xl[3] = {v[u].x, v[u].y, v[u].z};
                            hit |= sphere_overlap<D>(box, p, ri, xl, v[u].w);
                        }
                    }
                }
            }
            if (!hit) accepted = l;
        }
    } else {  // crowded neighbourhood: rescan (same candidate set, id filter as the list)
        const int32_t idq = S.id[q];
        for (int l = 0; l < rp.n_l && accepted < 0; ++l) {
            propose<D>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), p);
            bool ok = true;
            near_candidates<D>(g, cs, S.xf, q, skey[q], [&](int64_t j) {
                if (!ok || S.id[j] == idq) return;
                const double4 v = S.lv[j];
                const double xl[3] = {v.x, v.y, v.z};
                if (sphere_overlap<D>(box, p, ri, xl, v.w)) ok = false;
            });
            if (ok) accepted = l;
        }
    }
    if (accepted >= 0) S.lv[q] = make_double4(p[0], D > 1 ? p[1] : 0.0, D > 2 ? p[D > 2 ? 2 : 0] : 0.0, ri);
#pragma unroll
    for (int a = 0; a < D; ++a) T.x[a][q] = accepted >= 0 ? p[a] : xi[a];
    T.r[q] = ri;
    T.id[q] = S.id[q];
    T.slot[q] = sl;
    acc[q] = accepted >= 0 ? static_cast<uint8_t>(accepted) : kNotAccepted;
    if (accepted < 0) active[atomicAdd(&stats->active_count, 1ull)] = static_cast<int32_t>(q);
}

// colour class of a cell
__device__ __forceinline__ int colour1(int x, int m, int n) {
    const int body = m * (n / m);
    return x < body ? x % m : m + (x - body);
}

#ifndef SRM_SWEEP_THREADS
#define SRM_SWEEP_THREADS 128
#endif
constexpr int kSweepThreads = SRM_SWEEP_THREADS;

// Cells of colour class cls in the superblock (lo, hi) form a lattice per axis:
// first + stride * i, i < cnt (colour1 inverted on [lo, hi)).
__device__ __forceinline__ void class_lattice(const GridParams& g, int cls, const int* lo, const int* hi, int* first,
                                              int* stride, int* cnt) {
    int rem = cls;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int m = g.col_m[a], n = g.dims[a];
        const int cv = rem % g.col_n[a];
        rem /= g.col_n[a];
        const int body = m * (n / m);
        if (cv < m) {
            const int f = lo[a] + ((cv - lo[a] % m) + m) % m;
            const int b = min(hi[a], body);
            first[a] = f;
            stride[a] = m;
            cnt[a] = f < b ? (b - f + m - 1) / m : 0;
        } else {
            const int x = body + (cv - m);
            first[a] = x;
            stride[a] = 1;
            cnt[a] = (x >= lo[a] && x < hi[a]) ? 1 : 0;
        }
    }
}

// Superblock sb of colour sbc: along axis a its block index is colour bit + 2 * j_a
// (every block when the axis is not split); block k covers [ceil(k n / nsb), ceil((k+1) n / nsb)),
// i.e. x lies in block floor(x nsb / n) (oracle/srm_oracle.c orc_superblocks).
__device__ __forceinline__ void superblock_range(const GridParams& g, int sbc, int64_t sb, int* lo, int* hi) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int nsb = g.nsb[a], n = g.dims[a];
        int k = 0;
        if (nsb >= 2) {
            const int per = nsb / 2;
            k = ((sbc >> a) & 1) + 2 * static_cast<int>(sb % per);
            sb /= per;
        }
        lo[a] = static_cast<int>((static_cast<int64_t>(k) * n + nsb - 1) / nsb);
        hi[a] = static_cast<int>((static_cast<int64_t>(k + 1) * n + nsb - 1) / nsb);
    }
}

// One step of the sweep: colour class cls of the superblocks of colour sbc.  A thread
// per cell (blockIdx.y = superblock), the particles of a cell in slot order.  Cells of
// one class are farther apart than any trial can reach and superblocks of one colour a
// whole superblock apart, so all threads of the launch are independent and the launch
// sequence (sbc, cls) reproduces the sequential sweep of orc_sweep_round bit for bit.
template <int D>
__global__ void __launch_bounds__(kSweepThreads) k_sweep_cells(int sbc, int cls, State S, State T, Box box,
                                                               const GridParams* __restrict__ gp,
                                                               const RoundParams* __restrict__ rpp,
                                                               const int64_t* __restrict__ cs,
                                                               const uint32_t* __restrict__ skey,
                                                               const int32_t* __restrict__ nbr,
                                                               const uint8_t* __restrict__ nbr_cnt,
                                                               uint8_t* __restrict__ acc, int32_t* __restrict__ active,
                                                               StatsDev* stats) {
    const GridParams& g = *gp;
    if (cls >= g.ncls) return;
    int lo[3], hi[3], first[3], stride[3], cnt[3];
    superblock_range(g, sbc, blockIdx.y, lo, hi);
    class_lattice(g, cls, lo, hi, first, stride, cnt);
    const int cxy = cnt[0] * cnt[1];
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= static_cast<int64_t>(cxy) * cnt[2]) return;
    const int iz = static_cast<int>(t / cxy), r2 = static_cast<int>(t - static_cast<int64_t>(iz) * cxy);
    const int iy = r2 / cnt[0], ix = r2 - iy * cnt[0];
    const int64_t cell = (static_cast<int64_t>(first[2] + stride[2] * iz) * g.dims[1] + first[1] + stride[1] * iy) *
                             g.dims[0] +
                         first[0] + stride[0] * ix;
    const RoundParams rp = *rpp;
    const int64_t e = cs[cell + 1];
    for (int64_t q = cs[cell]; q < e; ++q)
        sweep_particle<D>(q, S, T, box, g, rp, cs, skey, nbr, nbr_cnt, acc, active, stats);
}

// Overlap reduction after the sweep.  A particle that accepted a trial cleared every
// live position at its turn and every later mover cleared it, so only pairs of
// particles that kept their round-start positions can overlap; those
// are exactly the particles on the non-mover list.
template <int D>
__global__ void __launch_bounds__(256) k_stats_sweep(State S, Box box, const GridParams* __restrict__ gp,
                                                     const int64_t* __restrict__ cs,
                                                     const uint32_t* __restrict__ skey,
                                                     const uint8_t* __restrict__ acc,
                                                     const int32_t* __restrict__ active, StatsDev* stats) {
    const int64_t m = static_cast<int64_t>(stats->active_count);
    const GridParams& g = *gp;
    unsigned long long pairs = 0;
    double pen = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = active[k];
        double xi[D];
        load_pos<D>(S, i, xi);
        const double ri = S.r[i];
        const int32_t idi = S.id[i];
        for_near_ranges<D>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
            for (int64_t j = b; j < e; ++j) {
                if (j <= i || acc[j] != kNotAccepted || S.id[j] == idi) continue;
                double xj[D];
                load_pos<D>(S, j, xj);
                const double rr = ri + S.r[j];
                const double d2 = dist2<D>(box, xi, xj);
                if (d2 <= rr * rr) {
                    ++pairs;
                    const double pe = rr - sqrt(d2);
                    pen = pe > pen ? pe : pen;
                }
            }
        });
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pairs += __shfl_down_sync(0xffffffffu, pairs, o);
        const double t = __shfl_down_sync(0xffffffffu, pen, o);
        pen = t > pen ? t : pen;
    }
    if ((threadIdx.x & 31) == 0) {
        if (pairs) atomicAdd(&stats->overlap_pairs, pairs);
        if (pen > 0.0) atomicMax(&stats->pen_bits, (unsigned long long)__double_as_longlong(pen));
    }
}

// Ordered candidate pairs of the reference's 3^d scan (cell_grid.hpp:394-414), from the
// cell offsets only (parity statistic, not on the timed path).
template <int D>
__global__ void __launch_bounds__(256) k_candidates(int64_t n, const GridParams* __restrict__ gp,
                                                    const int64_t* __restrict__ cs,
                                                    const uint32_t* __restrict__ skey, StatsDev* stats) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long cand = 0;
    if (i < n) {
        const GridParams& g = *gp;
        const int32_t s1[3] = {g.dims[0] <= 3 ? -1 : 1, g.dims[1] <= 3 ? -1 : 1, g.dims[2] <= 3 ? -1 : 1};
        for_near_ranges<D>(g, cs, skey[i], s1, [&](int64_t b, int64_t e) { cand += (unsigned long long)(e - b); });
        cand -= 1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cand += __shfl_down_sync(0xffffffffu, cand, o);
    if ((threadIdx.x & 31) == 0 && cand) atomicAdd(&stats->candidate_pairs, cand);
}

// Overlap statistics of a state with no migration (srm_b200_overlap_stats): every pair
// within ri + rj via the near stencil (extra = 0).
template <int D>
__global__ void __launch_bounds__(256) k_overlap_full(int64_t n, State S, Box box,
                                                      const GridParams* __restrict__ gp,
                                                      const int64_t* __restrict__ cs,
                                                      const uint32_t* __restrict__ skey,
                                                      int with_candidates, StatsDev* stats) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long pairs = 0, cand = 0;
    double pen = 0.0;
    if (i < n) {
        const GridParams& g = *gp;
        double xi[D];
        load_pos<D>(S, i, xi);
        const double ri = S.r[i];
        const int32_t idi = S.id[i];
        for_near_ranges<D>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
            for (int64_t j = b; j < e; ++j) {
                if (j <= i || S.id[j] == idi) continue;
                double xj[D];
                load_pos<D>(S, j, xj);
                const double rr = ri + S.r[j];
                const double d2 = dist2<D>(box, xi, xj);
                if (d2 <= rr * rr) {
                    ++pairs;
                    const double pe = rr - sqrt(d2);
                    pen = pe > pen ? pe : pen;
                }
            }
        });
        if (with_candidates) {
            const int32_t s1[3] = {g.dims[0] <= 3 ? -1 : 1, g.dims[1] <= 3 ? -1 : 1,
                                   g.dims[2] <= 3 ? -1 : 1};
            for_near_ranges<D>(g, cs, skey[i], s1, [&](int64_t b, int64_t e) { cand += (unsigned long long)(e - b); });
            cand -= 1;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pairs += __shfl_down_sync(0xffffffffu, pairs, o);
        cand += __shfl_down_sync(0xffffffffu, cand, o);
        const double t = __shfl_down_sync(0xffffffffu, pen, o);
        pen = t > pen ? t : pen;
    }
    if ((threadIdx.x & 31) == 0) {
        if (pairs) atomicAdd(&stats->overlap_pairs, pairs);
        if (cand) atomicAdd(&stats->candidate_pairs, cand);
        if (pen > 0.0) atomicMax(&stats->pen_bits, (unsigned long long)__double_as_longlong(pen));
    }
}

// ---------------------------------------------------------------------------------
// Small utility kernels.
__global__ void k_set_grid(GridParams* gp, GridParams v) { *gp = v; }
__global__ void k_set_round(RoundParams* rp, RoundParams v) { *rp = v; }

template <int D>
__global__ void k_unpack_records(int64_t n, const char* __restrict__ rec, int64_t stride,
                                 int64_t off_id, int64_t off_pos, int64_t off_r, State T) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const char* b = rec + i * stride;
        T.id[i] = *reinterpret_cast<const int32_t*>(b + off_id);
#pragma unroll
        for (int a = 0; a < D; ++a) T.x[a][i] = *reinterpret_cast<const double*>(b + off_pos + 8 * a);
        T.r[i] = *reinterpret_cast<const double*>(b + off_r);
        T.slot[i] = static_cast<int32_t>(i);
    }
}

template <int D>
__global__ void k_pack_records(int64_t n, State T, char* __restrict__ rec, int64_t stride,
                               int64_t off_id, int64_t off_pos, int64_t off_r) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        char* b = rec + (int64_t)T.slot[i] * stride;
        *reinterpret_cast<int32_t*>(b + off_id) = T.id[i];
#pragma unroll
        for (int a = 0; a < D; ++a) *reinterpret_cast<double*>(b + off_pos + 8 * a) = T.x[a][i];
        *reinterpret_cast<double*>(b + off_r) = T.r[i];
    }
}

// interleaved host layout <-> SoA, scattered back to slot order
template <int D>
__global__ void k_unpack_soa(int64_t n, const double* __restrict__ pos, const double* __restrict__ r,
                             const int32_t* __restrict__ id, State T) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < D; ++a) T.x[a][i] = pos[i * D + a];
        T.r[i] = r[i];
        T.id[i] = id ? id[i] : static_cast<int32_t>(i);
        T.slot[i] = static_cast<int32_t>(i);
    }
}

template <int D>
__global__ void k_pack_soa(int64_t n, State T, double* __restrict__ pos, double* __restrict__ r,
                           int32_t* __restrict__ id) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = T.slot[i];
#pragma unroll
        for (int a = 0; a < D; ++a) pos[s * D + a] = T.x[a][i];
        r[s] = T.r[i];
        id[s] = T.id[i];
    }
}

__global__ void k_scale_radius(int64_t n, double* __restrict__ r, double factor) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        r[i] = r[i] * factor;  // engine.hpp:520 p.radius *= factor
}

template <int D>
__global__ void k_copy_state(int64_t n, State A, State B) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < D; ++a) B.x[a][i] = A.x[a][i];
        B.r[i] = A.r[i];
        B.id[i] = A.id[i];
        B.slot[i] = A.slot[i];
    }
}

// reorder_by_locality: sorted order becomes storage order; ids = slots
__global__ void k_assign_slots(int64_t n, State S, int32_t* __restrict__ remap_old_to_new,
                               const int32_t* __restrict__ old_slot) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        if (remap_old_to_new) remap_old_to_new[old_slot[q]] = static_cast<int32_t>(q);
        S.slot[q] = static_cast<int32_t>(q);
        S.id[q] = static_cast<int32_t>(q);
    }
}

// sorted -> slot order helpers for parity outputs
__global__ void k_keys_by_slot(int64_t n, const int32_t* __restrict__ slot,
                               const uint32_t* __restrict__ skey, uint32_t* __restrict__ out) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        out[slot[q]] = skey[q];
}

__global__ void k_acc_by_slot(int64_t n, const int32_t* __restrict__ slot,
                              const uint8_t* __restrict__ acc, uint8_t* __restrict__ out) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        out[slot[q]] = acc[q];
}

// ---- deterministic reductions: fixed 1184-block partition, fixed trees -------------
constexpr int kRedBlocks = 1184;  // 148 SMs x 8
template <int D>
__device__ __forceinline__ double particle_measure(double r) {
    constexpr double pi = 3.141592653589793238462643383279502884;
    if (D == 2) return pi * r * r;                    // geometry.hpp:149-151
    return (4.0 / 3.0) * pi * r * r * r;              // geometry.hpp:153-155
}

template <int D>
__global__ void __launch_bounds__(256) k_reduce_partials(int64_t n, const double* __restrict__ r,
                                                         double* __restrict__ part_sum,
                                                         double* __restrict__ part_max) {
    __shared__ double ss[256], sm[256];
    const int64_t chunk = (n + kRedBlocks - 1) / kRedBlocks;
    const int64_t b0 = blockIdx.x * chunk;
    const int64_t b1 = b0 + chunk < n ? b0 + chunk : n;
    double s = 0.0, m = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += 256) {
        const double v = r[i];
        s = s + particle_measure<D>(v);
        m = v > m ? v : m;
    }
    ss[threadIdx.x] = s;
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            ss[threadIdx.x] = ss[threadIdx.x] + ss[threadIdx.x + w];
            sm[threadIdx.x] = sm[threadIdx.x + w] > sm[threadIdx.x] ? sm[threadIdx.x + w] : sm[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part_sum[blockIdx.x] = ss[0];
        part_max[blockIdx.x] = sm[0];
    }
}

__global__ void __launch_bounds__(256) k_reduce_final(const double* __restrict__ part_sum,
                                                      const double* __restrict__ part_max,
                                                      double* __restrict__ out /* [sum, max] */) {
    __shared__ double ss[256], sm[256];
    double s = 0.0, m = 0.0;
    for (int i = threadIdx.x; i < kRedBlocks; i += 256) {
        s = s + part_sum[i];
        m = part_max[i] > m ? part_max[i] : m;
    }
    ss[threadIdx.x] = s;
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            ss[threadIdx.x] = ss[threadIdx.x] + ss[threadIdx.x + w];
            sm[threadIdx.x] = sm[threadIdx.x + w] > sm[threadIdx.x] ? sm[threadIdx.x + w] : sm[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = ss[0];
        out[1] = sm[0];
    }
}

}  // namespace srmb
