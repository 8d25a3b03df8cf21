// srm_kernels.cuh -- CUDA kernels of the B200 SRM round (sm_100a).
//
// One SRM round (engine.hpp:227-234: build_shape_grid -> migrate -> shape_any_collision)
// is, on the device:
//   grid rebuild   k_keys -> k_scan_lookback -> k_scatter -> k_cellsort -> k_gather
//   near lists     k_near_tiles / k_near_lists (round-start neighbours within the trial reach)
//   migrate        k_sweep_warpq, one launch per colour class (warp queues)
//   reduction      k_stats_sweep (overlap pairs, max penetration over the non-movers)
// All kernels read the grid / round parameters from device memory so that the same
// launches can be replayed from a CUDA graph.  DESIGN.md §2-§4 has the data layout
// and the roofline of each kernel.
#pragma once

#include <cooperative_groups.h>

#include <cstdint>

#include "srm_device.cuh"
#include "srm_platelet.cuh"

namespace srmb {

// cell offsets into the sorted state: 32-bit (a context holds at most 2^31 - 1 particles)
using cell_t = int32_t;


// Division by a grid constant d >= 1 as a multiply-high (Granlund & Montgomery 1994,
// 33-bit multiplier): q = (umulhi(n, m) + n) >> l, exact for every 32-bit n.
struct FastDiv {
    uint32_t d, m, l;
};

__host__ __device__ inline uint32_t fdiv(uint32_t n, const FastDiv& f) {
#ifdef __CUDA_ARCH__
    const uint64_t hi = __umulhi(n, f.m);
#else
    const uint64_t hi = (static_cast<uint64_t>(n) * f.m) >> 32;
#endif
    return static_cast<uint32_t>((hi + n) >> f.l);
}

__host__ __device__ inline FastDiv make_fastdiv(uint32_t d) {
    uint32_t l = 0;
    while ((uint64_t{1} << l) < d) ++l;
    const uint64_t m = ((uint64_t{1} << 32) * ((uint64_t{1} << l) - d)) / d + 1;
    return FastDiv{d, static_cast<uint32_t>(m), l};
}

struct GridParams {
    int32_t dims[3];
    double edge[3];
    double inv_edge[3];  // 1 / edge (cell_of's quotient estimate)
    int64_t n_state;     // particles of the state the grid indexes (checked builds: index bounds)
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
    int32_t near_kind;   // near lists: 0 / 3 shared-memory bricks (sparse / crowded), 2 global memory
    int32_t ntiles;      // bricks of k_near_tiles (near_kind 0)
    FastDiv fd_dims[3];  // division by dims[a]
    FastDiv fd_m[3];     // division by col_m[a]
    int32_t col_body[3]; // col_m * floor(dims / col_m): cells coloured x mod m
    // wavefront sweep (k_sweep_wave): 1 = the whole sweep is one launch of
    // row tasks in wave order; lag_y / lag_z = wave-time offsets per y / z colour step
    int32_t wave, wave_lag_y, wave_lag_z, wave_pmax;
    // dependency resolution (srm_resolve.cuh) instead of class launches:
    // sparse 3D sphere grids on the shared-memory bricks
    int32_t resolve;
};

// cell coordinates of a flat key (x fastest, cell_grid.hpp:73-79)
template <int D>
__device__ __forceinline__ void decode_key(const GridParams& g, uint32_t key, int* c) {
    const uint32_t r1 = fdiv(key, g.fd_dims[0]);
    c[0] = static_cast<int>(key - r1 * static_cast<uint32_t>(g.dims[0]));
    if (D == 3) {
        const uint32_t r2 = fdiv(r1, g.fd_dims[1]);
        c[1] = static_cast<int>(r1 - r2 * static_cast<uint32_t>(g.dims[1]));
        c[2] = static_cast<int>(r2);
    } else {
        c[1] = static_cast<int>(r1);
        c[2] = 0;
    }
}

// CellGrid ctor (cell_grid.hpp:31-52) + the near-search stencil, the colouring
// and the near-list kernel choice for a state whose largest radius is
// max_r_state and whose trial moves have length c_m.  The colouring expression is the
// oracle's orc_colouring.  Host and device (the device-resident generate loop) share it.
// Returns 0, or 1 (cell_size <= 0), 2 (more than 2^32 cells).
#ifndef SRM_TILE_X
#define SRM_TILE_X 16
#endif
#ifndef SRM_TILE_Y
#define SRM_TILE_Y 8
#endif
#ifndef SRM_TILE_Z
#define SRM_TILE_Z 4
#endif
constexpr int kTX = SRM_TILE_X, kTY = SRM_TILE_Y, kTZ = SRM_TILE_Z;  // tiles::k_near_tiles brick (cells)
constexpr int kCTX = 4, kCTY = 4, kCTZ = 4, kCTileCap = 4096;         // ctiles::k_near_tiles (crowded)
constexpr double kCrowded = 1.8;  // mean particles per cell above which the crowded bricks are used
#ifndef SRM_WAVE_LY
#define SRM_WAVE_LY 64  // wave-time lag per y colour step (rows of one layer)
#endif
#ifndef SRM_WAVE_LZ
#define SRM_WAVE_LZ 64  // extra wave-time lag per z colour step (beyond the minimum)
#endif
#ifndef SRM_SWEEP_THREADS
#define SRM_SWEEP_THREADS 64
#endif
#ifndef SRM_TRIAL_TEAM
#define SRM_TRIAL_TEAM 16
#endif
// a class with at most this many cells runs as one wave of 16-lane teams (k_sweep_trials)
constexpr int64_t kSmallClassCells = 148LL * 8 * SRM_SWEEP_THREADS / SRM_TRIAL_TEAM;
constexpr int kWaveMaxP = 8192;  // wave times per sweep (k_wave_order's histogram)
constexpr int kWaveMaxDeps = 32; // dependency rows polled by one warp (a lane each)
constexpr int kWaveMaxRow = 2048; // cells per row (the row's done-bitmap in shared memory)
__host__ __device__ inline int grid_params(double cell_size, double max_r_state, double c_m, const Box& box, int dim,
                                           int near_mode, GridParams* out, int64_t n = 0, int wave_mode = 1) {
    const double extra = 2.0 * c_m;
    if (!(cell_size > 0.0)) return 1;
    GridParams g{};
    g.ncells = 1;
    for (int a = 0; a < 3; ++a) {
        if (a >= dim) {
            g.dims[a] = 1;
            g.edge[a] = 1.0;
            g.inv_edge[a] = 1.0;
            g.near_s[a] = -1;
            continue;
        }
        const double L = box.L[a];
        const double fl = floor(L / cell_size);
        if (!(fl < 4294967296.0)) return 2;
        int nn = static_cast<int>(fl);
        if (nn < 3) nn = 3;
        g.dims[a] = nn;
        g.edge[a] = L / nn;
        g.inv_edge[a] = 1.0 / g.edge[a];
        g.ncells *= nn;
        if (g.ncells > 4294967295LL) return 2;
    }
    g.extra = extra;
    g.rmax = max_r_state;
    g.n_state = n;
    const double cut = ((max_r_state + max_r_state + extra) * (1.0 + 1e-9) + 1e-300) * (1.0 + 1e-9);
    for (int a = 0; a < dim; ++a) {
        int64_t s = 1;
        while (static_cast<double>(s) * g.edge[a] < cut && 2 * s + 1 < g.dims[a]) ++s;
        g.near_s[a] = (2 * s + 1 >= g.dims[a]) ? -1 : static_cast<int32_t>(s);
    }
    // colouring: two cells of one class are more than any trial's reach apart
    const double cutc = ((max_r_state + max_r_state + 3.0 * c_m) * (1.0 + 1e-9) + 1e-300) * (1.0 + 1e-9);
    g.ncls = 1;
    g.cls_cells = 1;
    for (int a = 0; a < 3; ++a) {
        if (a >= dim) {
            g.col_m[a] = 1;
            g.col_n[a] = 1;
            continue;
        }
        int64_t s = 1;
        while (static_cast<double>(s) * g.edge[a] < cutc && 2 * s + 1 < g.dims[a]) ++s;
        if (2 * s + 1 >= g.dims[a]) {
            g.col_m[a] = g.dims[a];
            g.col_n[a] = g.dims[a];
        } else {
            g.col_m[a] = static_cast<int32_t>(s + 1);
            g.col_n[a] = g.col_m[a] + g.dims[a] % g.col_m[a];
        }
        g.ncls *= g.col_n[a];
        g.cls_cells *= (g.dims[a] + g.col_m[a] - 1) / g.col_m[a];
    }
    for (int a = 0; a < 3; ++a) {
        g.fd_dims[a] = make_fastdiv(static_cast<uint32_t>(g.dims[a]));
        g.fd_m[a] = make_fastdiv(static_cast<uint32_t>(g.col_m[a]));
        g.col_body[a] = g.col_m[a] * (g.dims[a] / g.col_m[a]);
    }
    // fp32 prefilter: coordinates live in [0, L); 8 ulp of the largest box length
    // bounds the rounding of any coordinate difference and of the radii sums
    double lmax = 0.0;
    for (int a = 0; a < dim; ++a) lmax = lmax > box.L[a] ? lmax : box.L[a];
    const double ulp = 5.9604644775390625e-08;  // 2^-24
    g.margin_f = static_cast<float>(8.0 * ulp * lmax + 4.0 * ulp * (2.0 * max_r_state + extra));
    g.extra_f = static_cast<float>(extra);
    g.rmax_f = static_cast<float>(max_r_state);
    for (int a = 0; a < 3; ++a) {
        g.L_f[a] = static_cast<float>(box.L[a]);
        g.half_f[a] = 0.5f * g.L_f[a];
        g.edge_f[a] = static_cast<float>(g.edge[a]);
    }
    // near lists: 0 the 16 x 8 x 4 bricks, 3 the crowded 4 x 4 x 4 bricks (mean occupancy
    // above kCrowded), 2 the per-particle global path
    const bool one = dim == 3 && near_mode == 0 && g.near_s[0] == 1 && g.near_s[1] == 1 && g.near_s[2] == 1;
    const bool crowded = static_cast<double>(n) > kCrowded * static_cast<double>(g.ncells);
    const bool tiles = one && !crowded && g.dims[0] >= kTX + 2 && g.dims[1] >= kTY + 2 && g.dims[2] >= kTZ + 2;
    const bool ctiles = one && crowded && g.dims[0] >= kCTX + 2 && g.dims[1] >= kCTY + 2 && g.dims[2] >= kCTZ + 2;
    g.near_kind = tiles ? 0 : (ctiles ? 3 : 2);
    // wavefront sweep: rows of cells (x) are tasks; a row waits for the rows within the
    // near reach (y, z) whose (z colour, y colour) is lower -- the class order of every
    // pair that can interact.  Needs a finite reach on y and z (at most
    // kWaveMaxDeps dependency rows) and is meant for sparse grids (crowded ones take the
    // team sweep).
    {
        const int sy = g.near_s[1], sz = dim == 3 ? g.near_s[2] : 0;
        const bool finite = g.near_s[0] >= 0 && g.dims[0] <= kWaveMaxRow && sy >= 0 && sz >= 0 &&
                            (2 * sy + 1) * (2 * sz + 1) <= kWaveMaxDeps;
        // wave_mode: bit 0 on; bits 8-15 / 16-23 override lag_y / the extra z lag (tuning)
        const int ly = (wave_mode >> 8) & 0xff, lz = (wave_mode >> 16) & 0xff;
        g.wave_lag_y = ly ? ly : SRM_WAVE_LY;
        g.wave_lag_z = (dim == 3 ? sz : 0) + 1 + g.wave_lag_y * (g.col_n[1] - 1) + (ly || lz ? lz : SRM_WAVE_LZ);
        g.wave_pmax = g.dims[2] - 1 + g.wave_lag_z * (g.col_n[2] - 1) + g.wave_lag_y * (g.col_n[1] - 1);
        g.wave = (wave_mode & 1) && finite && !crowded && g.wave_pmax < kWaveMaxP ? 1 : 0;
    }
    // (wave_mode bit 1: allowed; bit 2: also on small grids, which otherwise take the trial teams)
    g.resolve = (wave_mode & 2) && g.near_kind == 0 && g.ncls <= 255 &&
                        ((wave_mode & 4) || g.ncells / g.ncls > kSmallClassCells)
                    ? 1 : 0;
    g.ntiles = tiles ? ((g.dims[0] + kTX - 1) / kTX) * ((g.dims[1] + kTY - 1) / kTY) * ((g.dims[2] + kTZ - 1) / kTZ)
                     : (ctiles ? ((g.dims[0] + kCTX - 1) / kCTX) * ((g.dims[1] + kCTY - 1) / kCTY) *
                                     ((g.dims[2] + kCTZ - 1) / kCTZ)
                               : 0);
    *out = g;
    return 0;
}

struct RoundParams {
    double c_m;
    int32_t n_l;
    int32_t write_acc;  // also record the accepted trial per particle (parity outputs)
    RngKey key;
    double cos_r, sin_r;  // platelets: cos/sin of the rotation angle c_r (host libm)
};

// Per-particle state: one 32-byte record (x, y, z, r) per particle (z = 0 in 2D) -- a
// single sector per gather / neighbour read -- plus the reference id and storage slot.
struct State {
    double4* rec;   // (x, y, z, r) -- platelets: (x, y, z, diameter)
    int32_t* id;
    int32_t* slot;
    float4* xf;     // sorted fp32 copy (x, y, z, bounding radius) for the near-list screen; only in S
    double4* aux;   // platelets only: (nx, ny, nz, thickness); null for disks/spheres
};

// rim-seed cos/sin table of the platelet overlap fallback (set from the host, glibc)
__constant__ pl::SeedTable c_seed_table;

__device__ __forceinline__ double bounding_radius(const double4 r, const double4* aux, int64_t i) {
    return aux ? 0.5 * (r.w + aux[i].w) : r.w;  // shape.hpp:91-96 / spherodisk.hpp:94-96
}

template <int D>
__device__ __forceinline__ void rec_pos(const double4 v, double* p) {
    p[0] = v.x;
    if (D > 1) p[D > 1 ? 1 : 0] = v.y;
    if (D > 2) p[D > 2 ? 2 : 0] = v.z;
}

struct StatsDev {
    unsigned long long overlap_pairs;
    unsigned long long pen_bits;  // max penetration as the bits of a non-negative double
    unsigned long long candidate_pairs;
    unsigned long long active_count;  // non-movers: particles that kept their round-start position
    unsigned long long pool_top;      // near-list overflow pool: entries taken this round
    unsigned long long wave_waits;    // k_sweep_wave: dependency rows found unfinished (diagnostic)
    unsigned long long wave_polls;    // k_sweep_wave: polls of unfinished dependency rows (diagnostic)
    unsigned long long pair_tests;    // platelets: ordered pair tests (spherodisk_overlap) of the sweep + reduction
    unsigned long long pend[48];      // dependency resolution: pend[p] = particles still pending after pass p
    unsigned long long rev_count;     // half-stencil bricks: reverse entries (j, i) of the round
    unsigned long long ovf_count;     // ... and rows that outgrew their 7 entries (rebuilt from the full stencil)
};

// Overflow pool of the near lists: a row whose list does not fit (n > kNearCap) keeps
// its n entries at pool[row[1] ...] (row[1] = -1: the pool was full, the sweep rescans
// the stencil).  Taken with an atomic bump on StatsDev::pool_top, zeroed every round.
struct NearPool {
    int32_t* e;
    int64_t cap;
};

__device__ __forceinline__ double near_cut(double ri, double rj, double extra) {
    const double c = __dadd_rn(__dmul_rn(__dadd_rn(__dadd_rn(ri, rj), extra), 1.0 + 1e-9), 1e-300);
    return __dmul_rn(c, c);
}

// ---------------------------------------------------------------------------------
// Grid: cell_grid.hpp:62-81 cell_coords + flat_index, bit for bit.
template <int D>
__device__ __forceinline__ uint32_t cell_of(const GridParams& g, const double* p) {
    uint64_t idx = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
        // floor(p / edge) of the correctly rounded quotient, as the reference computes it.
        // The product with 1 / edge is within 3e-16 (relative) of that quotient, so when it
        // is farther than 1e-9 (1 + |t|) from an integer the two floors agree and the
        // division (some 40 instructions) is skipped; otherwise the quotient proper.
        const double t = __dmul_rn(p[a], g.inv_edge[a]);
        const double fl = floor(t), fr = t - fl, eps = 1e-9 * (1.0 + fabs(t));
        int i;
        if (fr > eps && 1.0 - fr > eps && fabs(t) < 1e9) i = static_cast<int>(fl);
        else i = static_cast<int>(floor(__ddiv_rn(p[a], g.edge[a])));
        if (i < 0 || i >= g.dims[a]) {  // (wrapped positions: only i == dims, by rounding)
            i %= g.dims[a];
            if (i < 0) i += g.dims[a];
        }
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
        rec_pos<D>(T.rec[i], p);
        const uint32_t k = cell_of<D>(g, p);
        SRM_CHK(static_cast<int64_t>(k) < g.ncells, 401);
        key[i] = k;
        atomicAdd(&count[k], 1u);
    }
}

// Single-pass exclusive scan of count[ncells] -> cell_start[ncells + 1] with decoupled
// look-back (Merrill & Garland 2016): a block per tile of kLbTile cells, tile ids in
// launch order from a counter (so a tile only waits on tiles that are running or done);
// each tile publishes its aggregate, then its inclusive prefix, as one 64-bit word
// (2-bit state | 62-bit value) in status[1 + tile].  status[0] is the tile counter.
// status[] must be zero on entry (one memset per scan).
constexpr int kLbThreads = 256, kLbPer = 16, kLbTile = kLbThreads * kLbPer;
constexpr unsigned long long kLbAgg = 1ull << 62, kLbPrefix = 2ull << 62, kLbMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kLbThreads) k_scan_lookback(const uint32_t* __restrict__ count,
                                                              const GridParams* __restrict__ gp,
                                                              unsigned long long* __restrict__ status,
                                                              cell_t* __restrict__ cell_start) {
    __shared__ unsigned tile_s;
    __shared__ unsigned long long warp_tot[kLbThreads / 32];
    __shared__ unsigned long long excl_s;
    const int64_t ncells = gp->ncells;
    const int64_t ntiles = (ncells + kLbTile - 1) / kLbTile;
    if (threadIdx.x == 0) tile_s = atomicAdd(reinterpret_cast<unsigned*>(status), 1u);
    __syncthreads();
    const int64_t tile = tile_s;
    if (tile >= ntiles) return;
    const int64_t base = tile * kLbTile + static_cast<int64_t>(threadIdx.x) * kLbPer;
    uint32_t v[kLbPer];
    if (base + kLbPer <= ncells) {
#pragma unroll
        for (int k = 0; k < kLbPer; k += 4) {
            const uint4 q = *reinterpret_cast<const uint4*>(count + base + k);
            v[k] = q.x;
            v[k + 1] = q.y;
            v[k + 2] = q.z;
            v[k + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kLbPer; ++k) v[k] = base + k < ncells ? count[base + k] : 0u;
    }
    unsigned long long t = 0;
#pragma unroll
    for (int k = 0; k < kLbPer; ++k) t += v[k];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {  // warp 0: publish the aggregate, look back 32 tiles at a time
        unsigned long long total = 0;
#pragma unroll
        for (int w = 0; w < kLbThreads / 32; ++w) {
            const unsigned long long x = warp_tot[w];
            __syncwarp();
            if (lane == 0) warp_tot[w] = total;
            total += x;
        }
        volatile unsigned long long* st = status + 1;
        unsigned long long excl = 0;
        if (tile == 0) {
            if (lane == 0) st[0] = kLbPrefix | total;
        } else {
            if (lane == 0) st[tile] = kLbAgg | total;
            int64_t j0 = tile - 1;  // window [j0 - 31, j0], lane l reads tile j0 - l
            for (;;) {
                const int64_t j = j0 - lane;
                unsigned long long w = kLbPrefix;  // (before tile 0: an empty prefix)
                if (j >= 0) {
                    do {
                        w = st[j];
                    } while ((w & ~kLbMask) == 0);
                }
                const unsigned pm = __ballot_sync(0xffffffffu, (w & ~kLbMask) == kLbPrefix);
                const int stop = pm ? __ffs(pm) - 1 : 32;  // the nearest prefix in the window
                unsigned long long v = lane <= stop && j >= 0 ? (w & kLbMask) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                excl += __shfl_sync(0xffffffffu, v, 0);
                if (pm) break;
                j0 -= 32;
            }
            if (lane == 0) st[tile] = kLbPrefix | (excl + total);
        }
        if (lane == 0) {
            excl_s = excl;
            if (tile == ntiles - 1) cell_start[ncells] = static_cast<cell_t>(excl + total);
        }
    }
    __syncthreads();
    unsigned long long run = excl_s + warp_tot[wid] + incl - t;
    if (base + kLbPer <= ncells) {
#pragma unroll
        for (int k = 0; k < kLbPer; k += 2) {
            int2 o;
            o.x = static_cast<int>(run);
            run += v[k];
            o.y = static_cast<int>(run);
            run += v[k + 1];
            *reinterpret_cast<int2*>(cell_start + base + k) = o;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kLbPer; ++k) {
            if (base + k < ncells) cell_start[base + k] = static_cast<cell_t>(run);
            run += v[k];
        }
    }
}

// atomic scatter into cell ranges (count[] returns to zero for the next histogram); the
// entry carries the sort key of the within-cell order with it: slot << 32 | source index
__global__ void k_scatter(int64_t n, const uint32_t* __restrict__ key, const int32_t* __restrict__ slot,
                          const cell_t* __restrict__ cell_start, uint32_t* __restrict__ count,
                          unsigned long long* __restrict__ perm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key[i];
        const uint32_t r = atomicSub(&count[k], 1u) - 1u;
        SRM_CHK(cell_start[k] + static_cast<int64_t>(r) >= 0 && cell_start[k] + static_cast<int64_t>(r) < n, 403);
        perm[cell_start[k] + r] = (static_cast<unsigned long long>(static_cast<uint32_t>(slot[i])) << 32) |
                                  static_cast<uint32_t>(i);
    }
}

// deterministic within-cell order: ascending slot (== engine.hpp:151-163 stability when
// slot is the storage index); the entries hold their slots, so the insertion sort makes
// no dependent loads
__global__ void k_cellsort(const GridParams* __restrict__ gp, const cell_t* __restrict__ cell_start,
                           unsigned long long* __restrict__ perm) {
    const int64_t ncells = gp->ncells;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncells;
         c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = cell_start[c], e = cell_start[c + 1];
        const int64_t cnt = e - b;
        if (cnt < 2) continue;
        if (cnt <= 4) {  // the usual cell: loads in flight together, sorted in registers
            unsigned long long v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = k < cnt ? perm[b + k] : ~0ull;
#pragma unroll
            for (int a = 1; a < 4; ++a)
#pragma unroll
                for (int k = a; k > 0; --k)
                    if (v[k] < v[k - 1]) {
                        const unsigned long long t = v[k];
                        v[k] = v[k - 1];
                        v[k - 1] = t;
                    }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < cnt) perm[b + k] = v[k];
            continue;
        }
        for (int64_t q = b + 1; q < e; ++q) {
            const unsigned long long v = perm[q];
            int64_t k = q - 1;
            unsigned long long w;
            while (k >= b && (w = perm[k]) > v) {
                perm[k + 1] = w;
                --k;
            }
            perm[k + 1] = v;
        }
    }
}

template <int D>
__global__ void k_gather(int64_t n, const unsigned long long* __restrict__ perm, const uint32_t* __restrict__ key,
                         State T, State S, uint32_t* __restrict__ skey) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t src = static_cast<int32_t>(perm[q] & 0xffffffffull);
        SRM_CHK(src >= 0 && src < n, 402);
        const double4 v = T.rec[src];
        S.rec[q] = v;
        double rb = v.w;
        if (T.aux) {
            const double4 a = T.aux[src];
            S.aux[q] = a;
            rb = 0.5 * (v.w + a.w);
        }
        if (S.xf)
            S.xf[q] = make_float4(static_cast<float>(v.x), static_cast<float>(v.y), static_cast<float>(v.z),
                                  static_cast<float>(rb));
        S.id[q] = T.id[src];
        S.slot[q] = T.slot[src];
        skey[q] = key[src];
    }
}

// ---------------------------------------------------------------------------------
// Stencil walk over the sorted cell ranges around cell `k`: half width g.near_s[a]
// (or the whole axis), x-runs merged into contiguous particle ranges.
template <int D, typename F>
__device__ __forceinline__ void for_near_ranges(const GridParams& g, const cell_t* __restrict__ cs,
                                                uint32_t k, const int32_t* s, F&& f) {
    const int dx = g.dims[0], dy = g.dims[1], dz = D == 3 ? g.dims[2] : 1;
    int cc_[3];
    decode_key<D>(g, k, cc_);
    const int cx = cc_[0], cy = cc_[1], cz = cc_[2];
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
    rec_pos<D>(S.rec[i], p);
}

// ---------------------------------------------------------------------------------
// Migrate: coloured Gauss-Seidel sweep.
//
// The reference's migrate (engine.hpp:89-107) visits particles in storage order; each
// gets <= n_l trials from its pre-sweep position and keeps the first one that clears the
// LIVE positions of all others.  Here the visiting order is (colour class, cell, slot):
// cells are coloured so that two cells of one class are farther apart than any trial
// can reach (GridParams::col_*), hence the rank-r particles of the cells of one class
// are independent: one launch per (class, rank), a thread per particle, and the result
// is identical to the sequential sweep in that order (oracle/srm_oracle.c
// orc_sweep_round).
//
// Live positions: S.rec[j] holds (x, r) of j -- its round-start position, overwritten by
// its accepted trial when j moves; one 32-byte sector per neighbour read.

// Near list row of a particle: kNearRow int32 = one 32-byte sector, [0] = n = number of
// near neighbours (round-start distance within ri + rj + 2 c_m, fp32 screen with a
// margin: a superset of the exact near set), entries [1, 1 + n) = their sorted indices.
// n > kNearCap means overflow: the sweep rescans the stencil.  At the bench window the
// mean list length is below one, so one sector holds a row.
constexpr int kNearRow = 8;
constexpr int kNearCap = kNearRow - 1;

// append j to a register-held list (no dynamically indexed local arrays)
struct NearList {
    int n = 0;
    int32_t e[kNearCap];
    __device__ __forceinline__ void add(int32_t j) {
#pragma unroll
        for (int s = 0; s < kNearCap; ++s)
            if (n == s) e[s] = j;
        ++n;
    }
    __device__ __forceinline__ void store(int32_t* row) const {
        int4* r = reinterpret_cast<int4*>(row);
        r[0] = make_int4(n, e[0], e[1], e[2]);
        r[1] = make_int4(e[3], e[4], e[5], e[6]);
    }
};

// Near candidates of sorted particle q: every j whose round-start distance is within
// ri + rj + 2 c_m (every j a trial of q can touch while j sits within c_m of its start).
// fp32 prefilter on the sorted float4 copy with an absolute margin above its rounding
// error, so the set is a superset of the exact fp64 near set; the stencil rows and the
// x cells of each row are pruned by the chord of the (inflated) cutoff sphere.
template <int D, typename F>
__device__ __forceinline__ void near_candidates(const GridParams& g, const cell_t* __restrict__ cs,
                                                const float4* __restrict__ xf, int64_t q, uint32_t key, F&& visit,
                                                int j0 = 0, int js = 1) {
    const float4 me = xf[q];
    const int dx = g.dims[0], dy = g.dims[1], dz = D == 3 ? g.dims[2] : 1;
    int cc_[3];
    decode_key<D>(g, key, cc_);
    const int cx = cc_[0], cy = cc_[1], cz = cc_[2];
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
            auto run = [&](int64_t b, int64_t e) {  // (a team lane takes every js-th candidate from j0)
                for (int64_t j = b + j0; j < e; j += js) {
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

// colour class of a cell
__device__ __forceinline__ int colour1(const GridParams& g, int a, int x) {
    const int m = g.col_m[a];
    if (x >= g.col_body[a]) return m + (x - g.col_body[a]);
    return x - static_cast<int>(fdiv(static_cast<uint32_t>(x), g.fd_m[a])) * m;
}

template <int D>
__device__ __forceinline__ int class_of_key(const GridParams& g, uint32_t key) {
    int cc_[3];
    decode_key<D>(g, key, cc_);
    const int cx = cc_[0], cy = cc_[1], cz = cc_[2];
    int k = colour1(g, 0, cx);
    k += g.col_n[0] * colour1(g, 1, cy);
    if (D == 3) k += g.col_n[0] * g.col_n[1] * colour1(g, 2, cz);
    return k;
}

// Near list of sorted particle q over its full stencil from global memory (grids that
// k_near_tiles does not cover, and its crowded bricks).
// A list longer than the row goes to the overflow pool (a second scan writes it there).
template <int D>
__device__ __forceinline__ void near_full_particle(int64_t q, const State& S, const GridParams& g,
                                                   const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                                   int32_t* __restrict__ nbr, NearPool pool, StatsDev* stats) {
    NearList nl;
    const int32_t idq = S.id[q];
    near_candidates<D>(g, cs, S.xf, q, skey[q], [&](int64_t j) {
        if (S.id[j] == idq) return;  // shape.hpp:70 self-exclusion by id
        nl.add(static_cast<int32_t>(j));
    });
    if (nl.n > kNearCap) {
        const int64_t off = static_cast<int64_t>(atomicAdd(&stats->pool_top, static_cast<unsigned long long>(nl.n)));
        if (off + nl.n <= pool.cap) {
            int32_t* dst = pool.e + off;
            int k = 0;
            near_candidates<D>(g, cs, S.xf, q, skey[q], [&](int64_t j) {
                if (S.id[j] == idq) return;
                dst[k++] = static_cast<int32_t>(j);
            });
            nl.e[0] = static_cast<int32_t>(off);
        } else {
            nl.e[0] = -1;
        }
    }
    nl.store(nbr + q * kNearRow);
}

template <int D>
__global__ void __launch_bounds__(256) k_near_lists(int64_t n, State S, const GridParams* __restrict__ gp,
                                                    const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                                    int32_t* __restrict__ nbr, NearPool pool, StatsDev* stats) {
    const GridParams& g = *gp;
    if (g.near_kind != 2) return;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        near_full_particle<D>(q, S, g, cs, skey, nbr, pool, stats);
}

// staged slot -> sorted index of one row of halo cells (k_near_tiles)
struct RowMap {
    int64_t sa, sb, sc;  // sorted index - slot in the runs [.., ka), [ka, kc), [kc, ..)
    int32_t ka, kc;
    float sy, sz;        // periodic image shift of the row
};

#ifndef SRM_TILE_THREADS
#define SRM_TILE_THREADS 256
#endif
#ifndef SRM_TILE_CAP
#define SRM_TILE_CAP 2048
#endif
// near-list screen variants (tuning): 0 = a store per candidate, 1 = a hit
// bitmask per 16 slot pairs; rows of the 3x3 stencil unrolled SRM_NEAR_ROWUNROLL times;
// SRM_NEAR_MONO: a constant cutoff in bricks whose radii are all equal
#ifndef SRM_NEAR_SCREEN
#define SRM_NEAR_SCREEN 0  // the sparse bricks (2: a record per pair of slots -- fewer instructions, measured slower)
#endif
#ifndef SRM_NEAR_HALF
#define SRM_NEAR_HALF 0  // 1: the sparse bricks screen half the stencil (each pair once) and a merge kernel
                         // completes the rows -- bit-exact, measured slower (0.91 + 0.11 + 0.02 ms against 0.72 ms
                         // at cfg 4: the branchy row loop and 3.5e6 row atomics cost more than the 37% fewer
                         // candidates save; profiles/r15_near_analysis.md)
#endif
#if SRM_NEAR_HALF && SRM_NEAR_SCREEN != 0
#error "the half stencil records hits with the store-per-candidate screen"
#endif
#ifndef SRM_CNEAR_SCREEN
#define SRM_CNEAR_SCREEN 0  // the crowded bricks (most lists overflow: they need the hit count)
#endif
#ifndef SRM_NEAR_ROWUNROLL
#define SRM_NEAR_ROWUNROLL 9
#endif
#ifndef SRM_NEAR_MONO
#define SRM_NEAR_MONO 0
#endif
constexpr int kNearRowUnroll = SRM_NEAR_ROWUNROLL;
#ifndef SRM_RTILE_MINB
#define SRM_RTILE_MINB 3  // CTAs per SM of the fused brick kernel (85 registers)
#endif
#include "srm_resolve.cuh"
static_assert(kResolveMaxPasses + 2 <= 48, "StatsDev::pend");
#define NT_FUSED 0
#define NT_SCREEN SRM_NEAR_SCREEN
#define NT_HALF SRM_NEAR_HALF
namespace tiles {  // sparse grids (~1-2 particles per cell): 16 x 8 x 4 bricks
#define NT_X SRM_TILE_X
#define NT_Y SRM_TILE_Y
#define NT_Z SRM_TILE_Z
#define NT_CAP SRM_TILE_CAP
#define NT_THREADS SRM_TILE_THREADS
#define NT_MINB 4
#define NT_KIND 0
#include "srm_near_tiles.cuh"
#undef NT_X
#undef NT_Y
#undef NT_Z
#undef NT_CAP
#undef NT_THREADS
#undef NT_MINB
#undef NT_KIND
}  // namespace tiles
#undef NT_HALF
#define NT_HALF 0
#undef NT_SCREEN
#define NT_SCREEN SRM_CNEAR_SCREEN
namespace ctiles {  // crowded grids: 4 x 4 x 4 bricks, 4096 staged particles
#define NT_X kCTX
#define NT_Y kCTY
#define NT_Z kCTZ
#define NT_CAP kCTileCap
#define NT_THREADS 256
#define NT_MINB 2
#define NT_KIND 3
#include "srm_near_tiles.cuh"
#undef NT_X
#undef NT_Y
#undef NT_Z
#undef NT_CAP
#undef NT_THREADS
#undef NT_MINB
#undef NT_KIND
}  // namespace ctiles
#undef NT_FUSED
#undef NT_SCREEN
#define NT_FUSED 1
#define NT_SCREEN 0  // (hits recorded by the store-per-candidate screen: they carry the stencil row)
namespace rtiles {  // the sparse bricks fused with pass 0 of the dependency resolution
#define NT_X SRM_TILE_X
#define NT_Y SRM_TILE_Y
#define NT_Z SRM_TILE_Z
#define NT_CAP SRM_TILE_CAP
#define NT_THREADS SRM_TILE_THREADS
#define NT_MINB SRM_RTILE_MINB
#define NT_KIND 0
#include "srm_near_tiles.cuh"
#undef NT_X
#undef NT_Y
#undef NT_Z
#undef NT_CAP
#undef NT_THREADS
#undef NT_MINB
#undef NT_KIND
}  // namespace rtiles
#undef NT_FUSED
#undef NT_SCREEN
#undef NT_HALF

// Half-stencil bricks: the reverse entries (j, i) -- "i, found from i's side, is a near
// neighbour of j" -- appended to j's row.  Rows in the pool (n > kNearCap) hold their full
// stencil already; a row that outgrows its entries goes to the overflow list once and is
// rebuilt from the full stencil by k_near_rebuild.  (The order of a row's entries is free:
// every entry is tested, the decisions are ANDs.)
__global__ void __launch_bounds__(256) k_near_merge(const GridParams* __restrict__ gp, const int2* __restrict__ rev,
                                                    int64_t rev_cap, int32_t* __restrict__ nbr,
                                                    int32_t* __restrict__ ovf, StatsDev* stats) {
    if (gp->near_kind != 0 || gp->resolve) return;
    const int64_t m = min(static_cast<int64_t>(stats->rev_count), rev_cap);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        const int2 e = rev[t];
        int32_t* row = nbr + static_cast<int64_t>(e.x) * kNearRow;
        if (*reinterpret_cast<volatile int32_t*>(row) > kNearCap) continue;
        const int pos = atomicAdd(row, 1);
        if (pos < kNearCap) row[1 + pos] = e.y;
        else if (pos == kNearCap) ovf[atomicAdd(&stats->ovf_count, 1ull)] = e.x;
    }
}

__global__ void __launch_bounds__(128) k_near_rebuild(State S, const GridParams* __restrict__ gp,
                                                      const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                                      int32_t* __restrict__ nbr, NearPool pool,
                                                      const int32_t* __restrict__ ovf, StatsDev* stats) {
    if (gp->near_kind != 0 || gp->resolve) return;
    const int64_t m = static_cast<int64_t>(stats->ovf_count);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        near_full_particle<3>(ovf[t], S, *gp, cs, skey, nbr, pool, stats);
}

#ifndef SRM_SWEEP_THREADS
#define SRM_SWEEP_THREADS 64
#endif
#ifndef SRM_PREFETCH
#define SRM_PREFETCH 3  // neighbour records loaded before the proposal is computed (1..3)
#endif
#ifndef SRM_SERPENTINE
#define SRM_SERPENTINE 1
#endif
#ifndef SRM_SWEEP_MINB
#define SRM_SWEEP_MINB 10
#endif
constexpr int kSweepThreads = SRM_SWEEP_THREADS;


// Crowded neighbourhood (overflowed near list): test trial p of q against every
// candidate of its stencil (same candidates, id filter).
template <bool kLive>
__device__ __forceinline__ double4 ld_rec(const double4* p) {
    if (kLive) {  // two 16-byte L2-only loads of one 32-byte sector
        const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
        return make_double4(a.x, a.y, b.x, b.y);
    }
    return *p;
}

template <int D, bool kLive = false>
__device__ __forceinline__ bool trial_clear_rescan(int64_t q, const double* p, double ri, const State& S, const Box& box,
                                                const GridParams& g, const cell_t* __restrict__ cs,
                                                const uint32_t* __restrict__ skey) {
    const int32_t idq = S.id[q];
    bool ok = true;
    near_candidates<D>(g, cs, S.xf, q, skey[q], [&](int64_t j) {
        if (!ok || S.id[j] == idq) return;
        const double4 v = ld_rec<kLive>(S.rec + j);
        const double xl[3] = {v.x, v.y, v.z};
        if (sphere_overlap<D>(box, p, ri, xl, v.w)) ok = false;
    });
    return ok;
}

// One trial of particle q (slot sl, round-start position xi, radius ri): propose trial l
// and test it against the live positions of q's near list (or, for an overflowed list,
// of every candidate of its stencil).  Returns true when the trial is clear (p = trial).
// kLive: neighbours' records may be rewritten by other warps of the same launch
// (k_sweep_wave), so they are read from L2 (ld.global.cg), never from a stale L1 line.
template <int D, bool kLive = false>
__device__ __forceinline__ bool trial_clear(int64_t q, int32_t sl, int l, const double* xi, double ri,
                                           const State& S, const Box& box, const GridParams& g,
                                           const RoundParams& rp, const cell_t* __restrict__ cs,
                                           const uint32_t* __restrict__ skey, const int32_t* __restrict__ nbr,
                                           const int32_t* __restrict__ pool, double* p) {
    // the row and the first three neighbours' live records are loaded before the
    // proposal is computed, so the Philox arithmetic runs while they are in flight (the
    // neighbours cannot move during q's visit: they belong to other classes, or to q's
    // cell and were visited by this lane before q)
    const int32_t* row = nbr + q * kNearRow;
    const int4 h0 = *reinterpret_cast<const int4*>(row);  // (n, e0, e1, e2)
    const int nn = h0.x;
    SRM_CHK(q >= 0 && q < g.n_state && nn >= 0, 201);
    SRM_CHK(nn > kNearCap || ((nn < 1 || (h0.y >= 0 && h0.y < g.n_state)) && (nn < 2 || (h0.z >= 0 && h0.z < g.n_state)) &&
                              (nn < 3 || (h0.w >= 0 && h0.w < g.n_state))), 202);
    double4 v[SRM_PREFETCH];
    if (nn <= kNearCap) {
        if (nn > 0) v[0] = ld_rec<kLive>(S.rec + h0.y);
        if (SRM_PREFETCH > 1 && nn > 1) v[SRM_PREFETCH > 1 ? 1 : 0] = ld_rec<kLive>(S.rec + h0.z);
        if (SRM_PREFETCH > 2 && nn > 2) v[SRM_PREFETCH > 2 ? 2 : 0] = ld_rec<kLive>(S.rec + h0.w);
    }
    propose<D>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), p);
    if (nn <= kNearCap) {
#pragma unroll
        for (int u = 0; u < SRM_PREFETCH; ++u) {
            if (u < nn) {
                const double xl[3] = {v[u].x, v[u].y, v[u].z};
                if (sphere_overlap<D>(box, p, ri, xl, v[u].w)) return false;
            }
        }
        for (int t = SRM_PREFETCH; t < nn; ++t) {  // the rest of the row (rare at the bench window)
            SRM_CHK(row[1 + t] >= 0 && row[1 + t] < g.n_state, 203);
            const double4 w = ld_rec<kLive>(S.rec + row[1 + t]);
            const double xl[3] = {w.x, w.y, w.z};
            if (sphere_overlap<D>(box, p, ri, xl, w.w)) return false;
        }
        return true;
    }
    if (h0.y >= 0) {  // the list is in the overflow pool
        const int32_t* e = pool + h0.y;
        for (int t = 0; t < nn; ++t) {
            SRM_CHK(e[t] >= 0 && e[t] < g.n_state, 204);
            const double4 w = ld_rec<kLive>(S.rec + e[t]);
            const double xl[3] = {w.x, w.y, w.z};
            if (sphere_overlap<D>(box, p, ri, xl, w.w)) return false;
        }
        return true;
    }
    return trial_clear_rescan<D, kLive>(q, p, ri, S, box, g, cs, skey);
}

// The cells of colour class cls form a lattice per axis: first + stride * i, i < cnt
// (colour1 inverted: a body colour v < m is x = v + m i, a remainder colour one cell).
__device__ __forceinline__ void class_lattice(const GridParams& g, int cls, int* first, int* stride, int* cnt) {
    int rem = cls;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int m = g.col_m[a];
        const int v = rem % g.col_n[a];
        rem /= g.col_n[a];
        if (v < m) {
            first[a] = v;
            stride[a] = m;
            cnt[a] = g.col_body[a] / m;
        } else {
            first[a] = g.col_body[a] + (v - m);
            stride[a] = 1;
            cnt[a] = 1;
        }
    }
}

// The class sweep with a queue per warp: each lane holds one item (particle, next trial,
// its cell's end) and every round runs one trial per item.  A lane whose particle is
// done takes the next particle of its cell (slot order) or, when the cell is finished,
// claims the next non-empty cell of the warp's share of the class lattice from a
// 32-cell window in shared memory (free lanes rank themselves with a ballot; items never
// move between lanes).  The window's cell ranges are loaded one window ahead so that the
// cell_start loads overlap the trials in flight.  No barriers and no work lists: warps
// progress independently.  Per cell the visiting order and the trials are those of the
// sequential sweep (orc_sweep_round).
template <int D>
__global__ void __launch_bounds__(kSweepThreads, SRM_SWEEP_MINB) k_sweep_warpq(int cls_arg, const int* __restrict__ cls_dev,
                                                                               State S, Box box,
                                                                               const GridParams* __restrict__ gp,
                                                                               const RoundParams* __restrict__ rpp,
                                                                               const cell_t* __restrict__ cs,
                                                                               const uint32_t* __restrict__ skey,
                                                                               const int32_t* __restrict__ nbr,
                                                                               const int32_t* __restrict__ pool,
                                                                               uint8_t* __restrict__ acc,
                                                                               int32_t* __restrict__ active,
                                                                               StatsDev* stats) {
    __shared__ int2 win_s[kSweepThreads];  // per warp: 32 (begin, end) cell ranges
    const int cls = cls_dev ? *cls_dev : cls_arg;  // (device-resident loop: from the controller)
    const GridParams& g = *gp;
    if (cls >= g.ncls) return;
    const RoundParams rp = *rpp;
    const int lane = threadIdx.x & 31;
    int2* win = win_s + (threadIdx.x & ~31);
    const unsigned lt = (1u << lane) - 1u;
    // the class lattice (constants of the launch) lives in shared memory, not registers
    __shared__ int lat_s[9];
    __shared__ FastDiv fd_s[2];
    if (threadIdx.x == 0) {
        class_lattice(g, cls, lat_s, lat_s + 3, lat_s + 6);
        fd_s[0] = make_fastdiv(static_cast<uint32_t>(lat_s[6]));
        fd_s[1] = make_fastdiv(static_cast<uint32_t>(lat_s[6] * lat_s[7]));
    }
    __syncthreads();
    const uint32_t cells = static_cast<uint32_t>(lat_s[6]) * lat_s[7] * lat_s[8];
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t next = static_cast<uint32_t>(static_cast<uint64_t>(cells) * w / nwarps);  // [next, stop)
    const uint32_t stop = static_cast<uint32_t>(static_cast<uint64_t>(cells) * (w + 1) / nwarps);
    // odd classes walk the share backwards: they start where the previous class launch
    // ended, whose records are still in L2 (the order of independent cells is free)
    const uint32_t flip = (SRM_SERPENTINE && (cls & 1)) ? next + stop - 1 : 0;
    // raw window entry of this lane (the lattice cell next + lane), loaded ahead
    int32_t rb = 0, re = 0;
    auto load_raw = [&]() {
        uint32_t t = next + lane;
        rb = 0;
        re = 0;
        if (t < stop) {
            if (flip) t = flip - t;
            const int cx = lat_s[6];
            const uint32_t iz = fdiv(t, fd_s[1]);
            const uint32_t r2 = t - iz * static_cast<uint32_t>(cx * lat_s[7]);
            const uint32_t iy = fdiv(r2, fd_s[0]), ix = r2 - iy * static_cast<uint32_t>(cx);
            const int64_t cell = (static_cast<int64_t>(lat_s[2] + lat_s[5] * static_cast<int>(iz)) * g.dims[1] + lat_s[1] +
                                  lat_s[4] * static_cast<int>(iy)) * g.dims[0] + lat_s[0] + lat_s[3] * static_cast<int>(ix);
            rb = static_cast<int32_t>(cs[cell]);
            re = static_cast<int32_t>(cs[cell + 1]);
        }
        next = stop - next < 32u ? stop : next + 32u;
    };
    bool have_raw = next < stop;
    if (have_raw) load_raw();
    int wn = 0, wofs = 0;  // window entries [wofs, wn) not yet claimed
    bool valid = false;
    int32_t iq = 0, il = 0, isl = 0, iend = 0;
    for (;;) {
        // free lanes claim cells (warp-uniform loop)
        for (;;) {
            const unsigned fm = __ballot_sync(0xffffffffu, !valid);
            if (fm == 0) break;
            if (wofs == wn) {
                if (!have_raw) break;
                // publish the raw window: the non-empty ranges, in lattice order
                const bool ne = rb < re;
                const unsigned gm = __ballot_sync(0xffffffffu, ne);
                __syncwarp();
                if (ne) win[__popc(gm & lt)] = make_int2(rb, re);
                __syncwarp();
                wn = __popc(gm);
                wofs = 0;
                have_raw = next < stop;
                if (have_raw) load_raw();  // the next window, in flight behind the trials
                continue;
            }
            const int rank = __popc(fm & lt);
            const int avail = wn - wofs;
            if (!valid && rank < avail) {
                const int2 c = win[wofs + rank];
                iq = c.x;
                iend = c.y;
                il = 0;
                isl = S.slot[iq];
                valid = true;
            }
            const int nf = __popc(fm);
            wofs += nf < avail ? nf : avail;
        }
        if (__ballot_sync(0xffffffffu, valid) == 0) break;
        if (valid) {
            const double4 me = S.rec[iq];  // round-start record (the particle has not moved)
            double xi[D], p[D];
            rec_pos<D>(me, xi);
            const bool clear = trial_clear<D>(iq, isl, il, xi, me.w, S, box, g, rp, cs, skey, nbr, pool, p);
            bool done = true;
            if (clear) {
                S.rec[iq] = make_double4(p[0], D > 1 ? p[D > 1 ? 1 : 0] : 0.0, D > 2 ? p[D > 2 ? 2 : 0] : 0.0, me.w);
                if (rp.write_acc) acc[iq] = static_cast<uint8_t>(il);
            } else if (il + 1 < rp.n_l) {
                ++il;
                done = false;
            } else {
                if (rp.write_acc) acc[iq] = kNotAccepted;
                active[atomicAdd(&stats->active_count, 1ull)] = iq;
            }
            if (done) {
                if (iq + 1 < iend) {  // the next particle of the cell
                    iq += 1;
                    il = 0;
                    isl = S.slot[iq];
                } else {
                    valid = false;
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// Wavefront sweep: the whole coloured Gauss-Seidel sweep in ONE
// persistent launch.  A task is a row of cells (all x at one (y, z)).  The result of the
// sequential class order (orc_sweep_round) depends only on the relative order of
// particles that can interact, which sit in cells within the near reach g.near_s of each
// other; two such rows have different (z colour, y colour) unless they are the same row,
// and the class order runs them in increasing (cz, cy).  So a row may run once the rows
// within reach with a lower (cz, cy) are done, and in any order otherwise; inside a row,
// a cell may run once the cells within reach along x with a lower x colour are done.
// Rows are handed out by a ticket counter in increasing wave time
//     P(y, z) = z + lag_z * cz(z) + lag_y * cy(y),
// which puts every dependency of a row at a strictly smaller P: between rows within reach
// z changes by at most the reach, lag_z exceeds the reach plus lag_y's whole range, and
// across the periodic seam the lower colour is always the cell near z = 0 (colour 0 at
// x = 0, the remainder colours highest).  A warp therefore only ever waits for rows held
// by running or finished warps: no deadlock and no residency assumption.  The lags keep a
// row's dependencies several wave steps behind it (waits are rare), and the wave keeps the
// rows being swept -- their records, near-list rows and their neighbours' records --
// within a band of layers that stays in L2, instead of streaming the whole domain once
// per colour class as the class launches do.
struct WaveCtl {
    unsigned ticket;  // next task
    unsigned epoch;   // sweep number: a row is done in this sweep when done[row] == epoch
};

__device__ __forceinline__ int wave_time(const GridParams& g, int y, int z) {
    return z + g.wave_lag_z * colour1(g, 2, z) + g.wave_lag_y * colour1(g, 1, y);
}

// rows sorted by wave time (a counting sort; rows of equal time are independent, so their
// order is free), the ticket counter reset, the sweep epoch advanced.  One CTA.
constexpr int kWaveOrderThreads = 1024;
__global__ void __launch_bounds__(kWaveOrderThreads) k_wave_order(const GridParams* __restrict__ gp, WaveCtl* wc,
                                                                  int32_t* __restrict__ order) {
    __shared__ int hist[kWaveMaxP];
    __shared__ int wsum[kWaveOrderThreads / 32];
    const GridParams& g = *gp;
    if (!g.wave) return;
    const int ny = g.dims[1], nrows = g.dims[1] * g.dims[2], np = g.wave_pmax + 1;
    for (int p = threadIdx.x; p < np; p += blockDim.x) hist[p] = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) atomicAdd(&hist[wave_time(g, r % ny, r / ny)], 1);
    __syncthreads();
    // exclusive scan of hist[0, np): a contiguous chunk per thread
    const int per = (np + blockDim.x - 1) / blockDim.x, b = threadIdx.x * per, e = min(np, b + per);
    int local = 0;
    for (int p = b; p < e; ++p) local += hist[p];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < wid; ++w) base += wsum[w];
    int run = base + incl - local;
    for (int p = b; p < e; ++p) {
        const int c = hist[p];
        hist[p] = run;
        run += c;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < nrows; r += blockDim.x) order[atomicAdd(&hist[wave_time(g, r % ny, r / ny)], 1)] = r;
    if (threadIdx.x == 0) {
        wc->ticket = 0;
        wc->epoch += 1;
    }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int D>
__global__ void __launch_bounds__(kSweepThreads, SRM_SWEEP_MINB) k_sweep_wave(State S, Box box,
                                                                              const GridParams* __restrict__ gp,
                                                                              const RoundParams* __restrict__ rpp,
                                                                              const cell_t* __restrict__ cs,
                                                                              const uint32_t* __restrict__ skey,
                                                                              const int32_t* __restrict__ nbr,
                                                                              const int32_t* __restrict__ pool,
                                                                              uint8_t* __restrict__ acc,
                                                                              int32_t* __restrict__ active,
                                                                              StatsDev* stats, WaveCtl* wc,
                                                                              const int32_t* __restrict__ order,
                                                                              unsigned* __restrict__ done) {
    constexpr int kWarps = kSweepThreads / 32, kWords = kWaveMaxRow / 32;
    __shared__ int2 win_s[kSweepThreads];             // per warp: 32 (begin, end) cell ranges
    __shared__ int winx_s[kSweepThreads];             // ... and their x
    __shared__ unsigned bits_s[kWarps][kWords];       // per warp: cells of the row already swept
    const GridParams& g = *gp;
    if (!g.wave) return;
    const RoundParams rp = *rpp;
    const unsigned epoch = *reinterpret_cast<volatile unsigned*>(&wc->epoch);
    const int lane = threadIdx.x & 31;
    int2* win = win_s + (threadIdx.x & ~31);
    int* winx = winx_s + (threadIdx.x & ~31);
    unsigned* bits = bits_s[threadIdx.x >> 5];
    const unsigned lt = (1u << lane) - 1u;
    const int dxc = g.dims[0], dyc = g.dims[1], dzc = g.dims[2];
    const unsigned nrows = static_cast<unsigned>(dyc) * static_cast<unsigned>(dzc);
    const int sx = g.near_s[0], sy = g.near_s[1], sz = D == 3 ? g.near_s[2] : 0;
    const int wy = 2 * sy + 1, ndep = wy * (2 * sz + 1);
    const int m = g.col_m[0], nbody = g.col_body[0] / m;  // x colours: body v < m has nbody cells
    const uint32_t ncl = static_cast<uint32_t>(dxc);
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(&wc->ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nrows) break;
        const int row = __ldcg(order + t);
        const int y = row % dyc, z = row / dyc;
        for (int w = lane; w < kWords; w += 32) bits[w] = 0u;
        // wait for the rows within reach with a lower (z colour, y colour): a lane each
        if (lane < ndep) {
            int yy = y + lane % wy - sy, zz = z + lane / wy - sz;
            yy = yy < 0 ? yy + dyc : (yy >= dyc ? yy - dyc : yy);
            zz = zz < 0 ? zz + dzc : (zz >= dzc ? zz - dzc : zz);
            const int cz = colour1(g, 2, z), czz = colour1(g, 2, zz);
            const bool lower = czz < cz || (czz == cz && colour1(g, 1, yy) < colour1(g, 1, y));
            if (lower) {
                const unsigned* f = done + (static_cast<int64_t>(zz) * dyc + yy);
                if (ld_relaxed(f) != epoch) {
                    unsigned polls = 1, ns = 64;
                    while (ld_relaxed(f) != epoch) {
                        __nanosleep(ns);
                        ns = ns < 1024 ? 2 * ns : ns;
                        ++polls;
                    }
                    atomicAdd(&stats->wave_waits, 1ull);
                    atomicAdd(&stats->wave_polls, static_cast<unsigned long long>(polls));
                }
                // acquire: the dependency's records (read from L2 below) after its release
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
        __syncwarp();
        const int64_t rowcell = static_cast<int64_t>(row) * dxc;
        // x of the c-th cell in claim order (colour by colour); the cell may start when the
        // cells within reach along x with a lower colour are done (bits)
        auto cell_x = [&](uint32_t c) -> int {
            const uint32_t body = static_cast<uint32_t>(m * nbody);
            if (c >= body) return g.col_body[0] + static_cast<int>(c - body);
            const uint32_t v = c / static_cast<uint32_t>(nbody), i = c - v * static_cast<uint32_t>(nbody);
            return static_cast<int>(v) + m * static_cast<int>(i);
        };
        auto ready = [&](int x) -> bool {
            const int cx = colour1(g, 0, x);
            for (int d = -sx; d <= sx; ++d) {
                if (d == 0) continue;
                int xx = x + d;
                xx = xx < 0 ? xx + dxc : (xx >= dxc ? xx - dxc : xx);
                if (colour1(g, 0, xx) < cx && !((bits[xx >> 5] >> (xx & 31)) & 1u)) return false;
            }
            return true;
        };
        uint32_t next = 0;
        int32_t rb = 0, re = 0, rx = 0;
        auto load_raw = [&]() {
            const uint32_t c = next + lane;
            rb = 0;
            re = 0;
            rx = -1;
            if (c < ncl) {
                rx = cell_x(c);
                const int64_t cell = rowcell + rx;
                rb = static_cast<int32_t>(cs[cell]);
                re = static_cast<int32_t>(cs[cell + 1]);
            }
            next = ncl - next < 32u ? ncl : next + 32u;
        };
        __syncwarp();
        bool have_raw = true;
        load_raw();
        int wn = 0, wofs = 0;
        bool valid = false, started = false;
        int32_t iq = 0, il = 0, isl = 0, iend = 0, ix = 0;
        for (;;) {
            for (;;) {  // free lanes claim cells (warp-uniform loop)
                const unsigned fm = __ballot_sync(0xffffffffu, !valid);
                if (fm == 0) break;
                if (wofs == wn) {
                    if (!have_raw) break;
                    const bool ne = rb < re;
                    if (rx >= 0 && !ne) atomicOr(&bits[rx >> 5], 1u << (rx & 31));  // empty: done
                    const unsigned gm = __ballot_sync(0xffffffffu, ne);
                    __syncwarp();  // every lane is done reading the previous window
                    if (ne) {
                        win[__popc(gm & lt)] = make_int2(rb, re);
                        winx[__popc(gm & lt)] = rx;
                    }
                    __syncwarp();
                    wn = __popc(gm);
                    wofs = 0;
                    have_raw = next < ncl;
                    if (have_raw) load_raw();
                    continue;
                }
                const int rank = __popc(fm & lt);
                const int avail = wn - wofs;
                if (!valid && rank < avail) {
                    const int2 c = win[wofs + rank];
                    iq = c.x;
                    iend = c.y;
                    ix = winx[wofs + rank];
                    il = 0;
                    valid = true;
                    started = false;
                }
                const int nf = __popc(fm);
                wofs += nf < avail ? nf : avail;
            }
            if (__ballot_sync(0xffffffffu, valid) == 0) break;
            if (valid && !started && ready(ix)) {
                started = true;
                isl = S.slot[iq];
            }
            bool cell_done = false;
            if (valid && started) {
                const double4 me = S.rec[iq];  // own record: only this lane writes it
                double xi[D], p[D];
                rec_pos<D>(me, xi);
                const bool clear = trial_clear<D, true>(iq, isl, il, xi, me.w, S, box, g, rp, cs, skey, nbr, pool, p);
                bool fin = true;
                if (clear) {
                    S.rec[iq] = make_double4(p[0], D > 1 ? p[D > 1 ? 1 : 0] : 0.0, D > 2 ? p[D > 2 ? 2 : 0] : 0.0, me.w);
                    if (rp.write_acc) acc[iq] = static_cast<uint8_t>(il);
                } else if (il + 1 < rp.n_l) {
                    ++il;
                    fin = false;
                } else {
                    if (rp.write_acc) acc[iq] = kNotAccepted;
                    active[atomicAdd(&stats->active_count, 1ull)] = iq;
                }
                if (fin) {
                    if (iq + 1 < iend) {
                        iq += 1;
                        il = 0;
                        isl = S.slot[iq];
                    } else {
                        valid = false;
                        cell_done = true;
                    }
                }
            }
            if (cell_done) atomicOr(&bits[ix >> 5], 1u << (ix & 31));
            __syncwarp();  // the cell's moves visible to the warp before a dependent cell starts
        }
        // publish the row: every lane's stores are ordered before lane 0's release by the
        // warp barrier (bar.warp.sync orders memory among its threads)
        __syncwarp();
        if (lane == 0) st_release(done + row, epoch);
    }
}

// The class sweep of crowded sphere grids (the ctiles near kind: several particles per
// cell, long near lists in the overflow pool): a team of kSphTeam lanes per cell.  A
// class then holds few cells of long chains (cfg 3's clusters: ~14 particles per cell),
// so a lane per cell leaves most of the GPU idle; here the team's lanes split the
// candidates of each trial and vote with a ballot.  Every lane computes the same
// proposal, and "no candidate overlaps" does not depend on who tests what, so the
// decisions are those of the sequential sweep (orc_sweep_round), like k_sweep_warpq's.
#ifndef SRM_SPH_TEAM
#define SRM_SPH_TEAM 16
#endif
#ifndef SRM_SPH_TEAM_ON
#define SRM_SPH_TEAM_ON 1
#endif
constexpr int kSphTeam = SRM_SPH_TEAM;
static_assert(kSphTeam >= 2 && kSphTeam <= 32 && (kSphTeam & (kSphTeam - 1)) == 0, "team: a power of two");

__global__ void __launch_bounds__(kSweepThreads, 8) k_sweep_team(int cls_arg, const int* __restrict__ cls_dev, State S,
                                                              Box box, const GridParams* __restrict__ gp,
                                                              const RoundParams* __restrict__ rpp,
                                                              const cell_t* __restrict__ cs,
                                                              const uint32_t* __restrict__ skey,
                                                              const int32_t* __restrict__ nbr,
                                                              const int32_t* __restrict__ pool,
                                                              uint8_t* __restrict__ acc, int32_t* __restrict__ active,
                                                              StatsDev* stats) {
    const int cls = cls_dev ? *cls_dev : cls_arg;
    const GridParams& g = *gp;
    if (cls >= g.ncls) return;
    const RoundParams rp = *rpp;
    const int lane = threadIdx.x & 31, tl = lane & (kSphTeam - 1);
    const unsigned tm = (kSphTeam == 32 ? 0xffffffffu : ((1u << (kSphTeam & 31)) - 1u)) << (lane & ~(kSphTeam - 1));
    int first[3], stride[3], cnt[3];
    class_lattice(g, cls, first, stride, cnt);
    const uint32_t cells = static_cast<uint32_t>(cnt[0]) * cnt[1] * cnt[2];
    const uint32_t nteams = (gridDim.x * blockDim.x) / kSphTeam;
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / kSphTeam;
    const int cx = cnt[0], cxy = cnt[0] * cnt[1];
    for (uint32_t t = team; t < cells; t += nteams) {
        const int iz = static_cast<int>(t / cxy), r2 = static_cast<int>(t - static_cast<uint32_t>(iz) * cxy);
        const int iy = r2 / cx, ix = r2 - iy * cx;
        const int64_t cell = (static_cast<int64_t>(first[2] + stride[2] * iz) * g.dims[1] + first[1] + stride[1] * iy) *
                                 g.dims[0] + first[0] + stride[0] * ix;
        const int64_t b = cs[cell], e = cs[cell + 1];
        for (int64_t q = b; q < e; ++q) {
            const double4 me = S.rec[q];
            const int32_t sl = S.slot[q], idq = S.id[q];
            const int32_t* row = nbr + q * kNearRow;
            const int nn = row[0];
            const int32_t* list = nn <= kNearCap ? row + 1 : (row[1] >= 0 ? pool + row[1] : nullptr);
            const double xi[3] = {me.x, me.y, me.z};
            int accepted = -1;
            double p[3];
            for (int l = 0; l < rp.n_l; ++l) {
                propose<3>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), p);
                bool hit = false;
                if (list) {
                    for (int k = tl; k < nn && !hit; k += kSphTeam) {
                        const double4 w = S.rec[list[k]];
                        const double xl[3] = {w.x, w.y, w.z};
                        hit = sphere_overlap<3>(box, p, me.w, xl, w.w);
                    }
                } else {  // overflowed list, pool full: the stencil, split over the team
                    near_candidates<3>(
                        g, cs, S.xf, q, skey[q],
                        [&](int64_t j) {
                            if (hit || S.id[j] == idq) return;
                            const double4 w = S.rec[j];
                            const double xl[3] = {w.x, w.y, w.z};
                            hit = sphere_overlap<3>(box, p, me.w, xl, w.w);
                        },
                        tl, kSphTeam);
                }
                if ((__ballot_sync(tm, hit) & tm) == 0u) {
                    accepted = l;
                    break;
                }
            }
            if (tl == 0) {
                if (accepted >= 0) {
                    S.rec[q] = make_double4(p[0], p[1], p[2], me.w);
                    if (rp.write_acc) acc[q] = static_cast<uint8_t>(accepted);
                } else {
                    if (rp.write_acc) acc[q] = kNotAccepted;
                    active[atomicAdd(&stats->active_count, 1ull)] = static_cast<int32_t>(q);
                }
            }
            __syncwarp(tm);  // the move is visible to the team before the cell's next particle
        }
    }
}

// The class sweep of small grids (a lane per cell would leave most of the GPU idle:
// cfg 1's 10^4 disks hold ~1000 cells per class): a team of kTrialTeam lanes per cell,
// a trial per lane.  A particle's trials are independent draws (Philox keyed by slot and
// trial index) tested against the same live neighbours, so the team runs trials l0 ..
// l0 + kTrialTeam - 1 at once and the lowest clear one is the sequential sweep's choice
// (orc_sweep_round); its lane writes the move.  At dense windows most trials fail, so
// the chain per particle shrinks from ~n_l trials to ~1.
#ifndef SRM_TRIAL_TEAM
#define SRM_TRIAL_TEAM 16
#endif
#ifndef SRM_TRIAL_TEAM_ON
#define SRM_TRIAL_TEAM_ON 1
#endif
constexpr int kTrialTeam = SRM_TRIAL_TEAM;
static_assert(kTrialTeam >= 2 && kTrialTeam <= 32 && (kTrialTeam & (kTrialTeam - 1)) == 0, "team: a power of two");

template <int D>
__global__ void __launch_bounds__(kSweepThreads, 8) k_sweep_trials(int cls_arg, const int* __restrict__ cls_dev, State S,
                                                                   Box box, const GridParams* __restrict__ gp,
                                                                   const RoundParams* __restrict__ rpp,
                                                                   const cell_t* __restrict__ cs,
                                                                   const uint32_t* __restrict__ skey,
                                                                   const int32_t* __restrict__ nbr,
                                                                   const int32_t* __restrict__ pool,
                                                                   uint8_t* __restrict__ acc, int32_t* __restrict__ active,
                                                                   StatsDev* stats) {
    const int cls = cls_dev ? *cls_dev : cls_arg;
    const GridParams& g = *gp;
    if (cls >= g.ncls) return;
    const RoundParams rp = *rpp;
    const int lane = threadIdx.x & 31, tl = lane & (kTrialTeam - 1), t0 = lane & ~(kTrialTeam - 1);
    const unsigned tm = (kTrialTeam == 32 ? 0xffffffffu : ((1u << (kTrialTeam & 31)) - 1u)) << t0;
    int first[3], stride[3], cnt[3];
    class_lattice(g, cls, first, stride, cnt);
    const uint32_t cells = static_cast<uint32_t>(cnt[0]) * cnt[1] * cnt[2];
    const uint32_t nteams = (gridDim.x * blockDim.x) / kTrialTeam;
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / kTrialTeam;
    const int cx = cnt[0], cxy = cnt[0] * cnt[1];
    for (uint32_t t = team; t < cells; t += nteams) {
        const int iz = static_cast<int>(t / cxy), r2 = static_cast<int>(t - static_cast<uint32_t>(iz) * cxy);
        const int iy = r2 / cx, ix = r2 - iy * cx;
        const int64_t cell = (static_cast<int64_t>(first[2] + stride[2] * iz) * g.dims[1] + first[1] + stride[1] * iy) *
                                 g.dims[0] + first[0] + stride[0] * ix;
        const int64_t b = cs[cell], e = cs[cell + 1];
        for (int64_t q = b; q < e; ++q) {
            const double4 me = S.rec[q];
            const int32_t sl = S.slot[q];
            double xi[D], p[D];
            rec_pos<D>(me, xi);
            bool done = false;
            for (int l0 = 0; l0 < rp.n_l && !done; l0 += kTrialTeam) {
                const int l = l0 + tl;
                const bool clear = l < rp.n_l &&
                                   trial_clear<D>(q, sl, l, xi, me.w, S, box, g, rp, cs, skey, nbr, pool, p);
                const unsigned cm = __ballot_sync(tm, clear) & tm;
                if (cm) {
                    done = true;
                    if (lane == __ffs(cm) - 1) {  // the lowest clear trial
                        S.rec[q] = make_double4(p[0], D > 1 ? p[D > 1 ? 1 : 0] : 0.0, D > 2 ? p[D > 2 ? 2 : 0] : 0.0, me.w);
                        if (rp.write_acc) acc[q] = static_cast<uint8_t>(l);
                    }
                }
            }
            if (!done && tl == 0) {
                if (rp.write_acc) acc[q] = kNotAccepted;
                active[atomicAdd(&stats->active_count, 1ull)] = static_cast<int32_t>(q);
            }
            __syncwarp(tm);  // the move is visible to the team before the cell's next particle
        }
    }
}

// The platelet class sweep with a team of kPlTeam lanes per particle.  The exact
// disk-disk test (spherodisk.cpp) dominates a platelet trial and a class holds few cells
// (27 classes of ~1700 cells at cfg 5), so one lane per cell leaves the GPU idle: here a
// team walks its share of the class's cells in order, and for each trial the team's
// lanes split q's candidates (the near list, or the rescanned stencil) and vote with a
// ballot.  Every lane computes the same proposal, and "no candidate overlaps" does not
// depend on who tests what, so the decisions are those of the sequential sweep, the
// oracle's orc_pl_sweep_round.
#ifndef SRM_PL_TEAM
#define SRM_PL_TEAM 32
#endif
constexpr int kPlTeam = SRM_PL_TEAM;
// resident CTAs per SM the team kernel is compiled for (4: 210 registers, no spills;
// without a bound ptxas caps it at 128 registers and spills)
#ifndef SRM_PL_MINB
#define SRM_PL_MINB 4
#endif

__global__ void __launch_bounds__(kSweepThreads, SRM_PL_MINB) k_sweep_pl_team(int cls_arg, const int* __restrict__ cls_dev, State S,
                                                                 Box box, const GridParams* __restrict__ gp,
                                                                 const RoundParams* __restrict__ rpp,
                                                                 const cell_t* __restrict__ cs,
                                                                 const uint32_t* __restrict__ skey,
                                                                 const int32_t* __restrict__ nbr,
                                                                 const int32_t* __restrict__ pool,
                                                                 uint8_t* __restrict__ acc, int32_t* __restrict__ active,
                                                                 StatsDev* stats) {
    const int cls = cls_dev ? *cls_dev : cls_arg;
    const GridParams& g = *gp;
    if (cls >= g.ncls) return;
    const RoundParams rp = *rpp;
    unsigned long long tests = 0;  // pair tests of this lane (StatsDev::pair_tests)
    const int lane = threadIdx.x & 31, tl = lane & (kPlTeam - 1);
    const unsigned tm = ((1u << kPlTeam) - 1u) << (lane & ~(kPlTeam - 1));
    int first[3], stride[3], cnt[3];
    class_lattice(g, cls, first, stride, cnt);
    const uint32_t cells = static_cast<uint32_t>(cnt[0]) * cnt[1] * cnt[2];
    const uint32_t nteams = (gridDim.x * blockDim.x) / kPlTeam;
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / kPlTeam;
    // cells strided over the teams: with fewer cells than teams the busy teams are the
    // first ones, packed into the first CTAs, so they are resident together
    const int cx = cnt[0], cxy = cnt[0] * cnt[1];
    for (uint32_t t = team; t < cells; t += nteams) {
        const int iz = static_cast<int>(t / cxy), r2 = static_cast<int>(t - static_cast<uint32_t>(iz) * cxy);
        const int iy = r2 / cx, ix = r2 - iy * cx;
        const int64_t cell = (static_cast<int64_t>(first[2] + stride[2] * iz) * g.dims[1] + first[1] + stride[1] * iy) *
                                 g.dims[0] + first[0] + stride[0] * ix;
        const int64_t b = cs[cell], e = cs[cell + 1];
        for (int64_t q = b; q < e; ++q) {
            const double4 me = S.rec[q], ni = S.aux[q];
            const int32_t sl = S.slot[q], idq = S.id[q];
            const int32_t* row = nbr + q * kNearRow;
            const int nn = row[0];
            const double xi[3] = {me.x, me.y, me.z};
            int accepted = -1;
            double p[3];
            pl::V3 pn{0.0, 0.0, 0.0};
            for (int l = 0; l < rp.n_l; ++l) {
                propose<3>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), p);
                double ax[3];
                unit_vector<3>(rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), 1, ax);
                pn = pl::rotate_normal(pl::V3{ni.x, ni.y, ni.z}, pl::V3{ax[0], ax[1], ax[2]}, rp.cos_r, rp.sin_r);
                bool hit = false;
                auto cand = [&](int64_t j, pl::V3& d, pl::V3& nb, double4& v, double4& a) {
                    v = S.rec[j];
                    a = S.aux[j];
                    d = pl::V3{min_image1(v.x - p[0], box.L[0], box.half[0]),
                               min_image1(v.y - p[1], box.L[1], box.half[1]),
                               min_image1(v.z - p[2], box.L[2], box.half[2])};
                    nb = pl::V3{a.x, a.y, a.z};
                };
                auto test = [&](int64_t j) {
                    pl::V3 d, nb;
                    double4 v, a;
                    cand(j, d, nb, v, a);
                    return pl::spherodisk_overlap(d, pn, me.w, ni.w, nb, v.w, a.w, c_seed_table);
                };
                if (nn <= kNearCap || row[1] >= 0) {
                    // the list (in the row, or in the overflow pool), a candidate per lane per
                    // pass; a pair the projections leave undecided (disks_within's rim-seed
                    // fallback, 32 x 64 projections) is resolved by the whole team, a seed per
                    // lane, unless another candidate of the pass already overlaps
                    const int32_t* e = nn <= kNearCap ? row + 1 : pool + row[1];
                    const double r1 = 0.5 * (me.w - ni.w);
                    for (int base = 0; base < nn; base += kPlTeam) {
                        const int k = base + tl;
                        pl::V3 d{0.0, 0.0, 0.0}, nb{0.0, 0.0, 1.0};
                        double r2 = 0.0, th = 0.0;
                        int st = pl::kDwFalse;
                        if (k < nn) {
                            double4 v, a;
                            cand(e[k], d, nb, v, a);
                            st = pl::spherodisk_overlap_pre(d, pn, me.w, ni.w, nb, v.w, a.w);
                            ++tests;
                            r2 = 0.5 * (v.w - a.w);
                            th = 0.5 * (ni.w + a.w);
                        }
                        hit = (__ballot_sync(tm, st == pl::kDwTrue) & tm) != 0u;
                        unsigned pend = __ballot_sync(tm, st == pl::kDwSeeds) & tm;
                        while (pend && !hit) {
                            const int src = __ffs(pend) - 1;
                            pend &= pend - 1u;
                            const pl::V3 sd{__shfl_sync(tm, d.x, src), __shfl_sync(tm, d.y, src),
                                            __shfl_sync(tm, d.z, src)};
                            const pl::V3 sn{__shfl_sync(tm, nb.x, src), __shfl_sync(tm, nb.y, src),
                                            __shfl_sync(tm, nb.z, src)};
                            const double sr2 = __shfl_sync(tm, r2, src), sth = __shfl_sync(tm, th, src);
                            bool h = false;
                            for (int sk = tl; sk < pl::kSeeds && !h; sk += kPlTeam)
                                h = pl::rim_seed_within(pl::V3{0.0, 0.0, 0.0}, pn, r1, sd, sn, sr2, sth, c_seed_table, sk);
                            hit = (__ballot_sync(tm, h) & tm) != 0u;
                        }
                        if (hit) break;
                    }
                } else {  // crowded neighbourhood, pool full: the stencil, split over the team
                    near_candidates<3>(
                        g, cs, S.xf, q, skey[q],
                        [&](int64_t j) {
                            if (!hit && S.id[j] != idq) {
                                hit = test(j);
                                ++tests;
                            }
                        },
                        tl, kPlTeam);
                }
                if ((__ballot_sync(tm, hit) & tm) == 0u) {
                    accepted = l;
                    break;
                }
            }
            if (tl == 0) {
                if (accepted >= 0) {
                    S.rec[q] = make_double4(p[0], p[1], p[2], me.w);
                    S.aux[q] = make_double4(pn.x, pn.y, pn.z, ni.w);
                    if (rp.write_acc) acc[q] = static_cast<uint8_t>(accepted);
                } else {
                    if (rp.write_acc) acc[q] = kNotAccepted;
                    active[atomicAdd(&stats->active_count, 1ull)] = static_cast<int32_t>(q);
                }
            }
            __syncwarp(tm);  // the move is visible to the team before the cell's next particle
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tests += __shfl_down_sync(0xffffffffu, tests, o);
    if (lane == 0 && tests) atomicAdd(&stats->pair_tests, tests);
}

// ---------------------------------------------------------------------------------
// Device-resident srm_generate (engine.hpp:176-260): a controller kept in device memory
// drives a CUDA graph of conditional nodes; every decision the host loop takes between
// rounds (swell factor and clamp, grid of the iteration, success, shake, commit, volume
// fraction, reorder cadence, iteration budget) is taken here, so a whole run is one
// graph launch with no host round-trip.  A "step" is one round: a growth round on the
// working state W (a copy of P, swollen), or a shake round (W = P), see GenCtl::phase.
struct GenProgress {
    int64_t iteration;
    double volume_fraction;
    int32_t accepted;
    int32_t rounds;
    uint64_t t_ns;  // globaltimer at the end of the iteration
};

struct GenCtl {
    // inputs
    double f_target, stop, c_w, c_m, box_measure;
    int64_t max_iter, it0;
    int64_t n;  // particles (the near-list kernel choice depends on the occupancy)
    int32_t n_k, n_l, reorder_period, dim, near_mode, wave_mode;
    uint64_t seed;
    double cos_r, sin_r;  // platelet rotation angle (host libm)
    // state
    double f, max_r, factor, cs;
    int64_t done, accepted, rounds, shakes;
    int32_t phase;  // 0 new iteration, 1 growth rounds, 2 shake rounds, 3 finished
    int32_t k;      // round index in the phase
    int32_t reorder_since;
    int32_t status;  // 0 ok, 1 iteration budget exhausted, 2 invalid grid (CellGrid safety bound)
    int32_t cls;     // colour class of the running sweep launch
    int32_t iter_done;  // an iteration ended in this step (progress record)
    int32_t success;
    int32_t rounds_this;
    int32_t do_copy, do_scale;  // this step starts with W <- P (and W *= factor)
    uint64_t t0;
    GridParams g_iter;  // the grid of the current iteration (growth rounds and reorder)
    // live progress (engine.hpp:251-254): a ring in pinned, host-mapped memory.  The
    // device publishes iteration records as they end; the host thread consumes them while
    // the graph runs and reports its position back.  recs == nullptr: no progress sink.
    GenProgress* recs;
    int64_t recs_cap;
    int64_t* pub;   // records published (device -> host); pub[2] = the run's start time
    int64_t* cons;  // records consumed (host -> device)
};

__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Start of a step: phase logic before the round; writes the grid and round parameters.
__global__ void k_gen_step(GenCtl* c, GridParams* gp, RoundParams* rp, StatsDev* stats, Box box,
                           cudaGraphConditionalHandle h_active) {
    bool active = true, copy = false, scale = false;
    c->iter_done = 0;
    if (c->phase == 0) {  // a new iteration (engine.hpp:205-224)
        c->done += 1;
        double factor = 1.0 + c->c_w;
        const double N = static_cast<double>(c->dim);
        if (c->f * pow(factor, N) > c->f_target) factor = pow(c->f_target / c->f, 1.0 / N);
        c->factor = factor;
        c->cs = 2.5 * c->max_r + c->c_m;
        GridParams g{};
        if (c->cs < 2.0 * (c->max_r * factor) + c->c_m ||
            grid_params(c->cs, c->max_r * factor, c->c_m, box, c->dim, c->near_mode, &g, c->n, c->wave_mode) != 0) {
            c->status = 2;
            c->phase = 3;
            active = false;
        } else {
            c->g_iter = g;
            *gp = g;
            c->phase = 1;
            c->k = 0;
            c->rounds_this = 0;
            copy = true;
            scale = true;
        }
    } else if (c->phase == 2 && c->k == 0) {  // shake on P with the pre-swell grid (engine.hpp:244-249)
        GridParams g{};
        grid_params(c->cs, c->max_r, c->c_m, box, c->dim, c->near_mode, &g, c->n, c->wave_mode);
        *gp = g;
        copy = true;
    }
    if (active) {
        RoundParams v{};
        v.c_m = c->c_m;
        v.n_l = c->n_l;
        v.write_acc = 0;
        v.key.k0 = static_cast<uint32_t>(c->seed);
        v.key.k1 = static_cast<uint32_t>(c->seed >> 32);
        v.key.round_id = static_cast<uint32_t>(c->phase == 1 ? c->k : c->n_k + c->k) & 0xFFFFFFu;
        v.key.iteration = static_cast<uint32_t>(c->it0 + c->done);
        v.cos_r = c->cos_r;
        v.sin_r = c->sin_r;
        *rp = v;
        *stats = StatsDev{0, 0, 0, 0};
    }
    c->do_copy = copy ? 1 : 0;
    c->do_scale = scale ? 1 : 0;
    cudaGraphSetConditional(h_active, active ? 1u : 0u);
}

__global__ void k_gen_flags(const GenCtl* c, cudaGraphConditionalHandle h_copy, cudaGraphConditionalHandle h_scale) {
    cudaGraphSetConditional(h_copy, c->do_copy ? 1u : 0u);
    cudaGraphSetConditional(h_scale, c->do_scale ? 1u : 0u);
}

__global__ void k_gen_t0(GenCtl* c) {
    c->t0 = global_ns();
    if (c->pub) *reinterpret_cast<volatile int64_t*>(c->pub + 2) = static_cast<int64_t>(c->t0);
}

// wave_on: the graph swept this round with k_sweep_wave already when the grid allows it
__global__ void k_gen_cls_begin(GenCtl* c, const GridParams* __restrict__ gp, cudaGraphConditionalHandle h_cls,
                                int wave_on) {
    c->cls = 0;
    cudaGraphSetConditional(h_cls, gp->ncls > 0 && !(wave_on && gp->wave) && !gp->resolve ? 1u : 0u);
}

__global__ void k_gen_cls_next(GenCtl* c, const GridParams* __restrict__ gp, cudaGraphConditionalHandle h_cls) {
    c->cls += 1;
    cudaGraphSetConditional(h_cls, c->cls < gp->ncls ? 1u : 0u);
}

// After the round: success / shake / commit decisions (engine.hpp:227-249).
__global__ void k_gen_after(GenCtl* c, const StatsDev* __restrict__ stats, cudaGraphConditionalHandle h_commit,
                            cudaGraphConditionalHandle h_f, cudaGraphConditionalHandle h_reorder) {
    bool commit = false, newf = false, reorder = false;
    c->rounds_this += 1;
    if (c->phase == 1) {
        c->rounds += 1;
        c->k += 1;
        if (stats->overlap_pairs == 0) {  // accepted: P <- W, f, reorder cadence
            commit = true;
            newf = true;
            c->success = 1;
            c->accepted += 1;
            // (max_r: the committed state's bounding radius, recomputed by k_gen_f)
            if (c->reorder_period > 0 && ++c->reorder_since >= c->reorder_period) {
                c->reorder_since = 0;
                reorder = true;
            }
            c->phase = 0;
            c->iter_done = 1;
        } else if (c->k >= c->n_k) {  // failed: shake
            c->phase = 2;
            c->k = 0;
            c->rounds_this = 0;
        }
    } else if (c->phase == 2) {
        c->shakes += 1;
        c->k += 1;
        if (c->k >= c->n_k) {
            commit = true;  // the shaken W back into P
            c->success = 0;
            c->phase = 0;
            c->iter_done = 1;
        }
    }
    cudaGraphSetConditional(h_commit, commit ? 1u : 0u);
    cudaGraphSetConditional(h_f, newf ? 1u : 0u);
    cudaGraphSetConditional(h_reorder, reorder ? 1u : 0u);
}

// volume fraction and max bounding radius of the committed state (shape.hpp:83-96),
// recomputed as the host loop does: for platelets 0.5 (D + t) of the swollen D and t is
// not always max_r * factor to the last ulp
__global__ void k_gen_f(GenCtl* c, const double* __restrict__ red_out) {
    c->f = red_out[0] / c->box_measure;
    c->max_r = red_out[1];
}

__global__ void k_gen_grid_iter(const GenCtl* c, GridParams* gp) { *gp = c->g_iter; }

// End of a step: progress record, loop condition (engine.hpp:202-211).
__global__ void k_gen_end(GenCtl* c, cudaGraphConditionalHandle h_run) {
    if (c->iter_done) {
        GenProgress r;
        r.iteration = c->it0 + c->done;
        r.volume_fraction = c->f;
        r.accepted = c->success;
        r.rounds = c->rounds_this;
        r.t_ns = global_ns();
        if (c->recs) {
            const int64_t idx = c->done - 1;
            // a full ring waits for the host (it polls while the graph runs)
            while (idx - *reinterpret_cast<volatile int64_t*>(c->cons) >= c->recs_cap) __nanosleep(1000);
            c->recs[idx % c->recs_cap] = r;
            __threadfence_system();
            *reinterpret_cast<volatile int64_t*>(c->pub) = idx + 1;
        }
    }
    if (c->phase == 0) {
        if (!(c->f < c->stop)) c->phase = 3;
        else if (c->done >= c->max_iter) {
            c->status = 1;
            c->phase = 3;
        }
    }
    cudaGraphSetConditional(h_run, c->phase != 3 ? 1u : 0u);
}

__global__ void k_scale_radius_ctl(int64_t n, double4* __restrict__ rec, double4* __restrict__ aux,
                                   const GenCtl* __restrict__ c) {
    const double factor = c->factor;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rec[i].w = rec[i].w * factor;  // engine.hpp:224 / shape.hpp:46 p.radius *= factor
        if (aux) aux[i].w = aux[i].w * factor;
    }
}

// Overlap reduction after the sweep.  A particle that accepted a trial cleared every
// live position at its turn and every later mover cleared it, so only pairs of
// particles that kept their round-start positions can overlap; those
// are exactly the particles on the non-mover list.
template <int D>
__global__ void __launch_bounds__(256) k_stats_sweep(State S, Box box, const GridParams* __restrict__ gp,
                                                     const cell_t* __restrict__ cs,
                                                     const uint32_t* __restrict__ skey,
                                                     const uint8_t* __restrict__ acc,
                                                     const int32_t* __restrict__ active, StatsDev* stats,
                                                     const double4* rec_alt = nullptr) {
    const int64_t m = static_cast<int64_t>(stats->active_count);
    const GridParams& g = *gp;
    // (graph runs: a round swept by the dependency resolution left its records in rec_alt)
    if (rec_alt && g.resolve) S.rec = const_cast<double4*>(rec_alt);
    unsigned long long pairs = 0;
    double pen = 0.0;
    // the pair test of non-mover i against j > i (movers never overlap anything,
    // DESIGN.md §3.3)
    auto pair = [&](int64_t i, const double* xi, double ri, int32_t idi, int64_t j) {
        if (j <= i || S.id[j] == idi) return;
        double xj[D];
        const double4 vj = S.rec[j];
        rec_pos<D>(vj, xj);
        const double rr = ri + vj.w;
        const double d2 = dist2<D>(box, xi, xj);
        if (d2 <= rr * rr) {
            ++pairs;
            const double pe = rr - sqrt(d2);
            pen = pe > pen ? pe : pen;
        }
    };
    const int sy = g.near_s[1], sz = D == 3 ? g.near_s[2] : 0;
    const int rows = (2 * sy + 1) * (2 * sz + 1);
    if (g.near_s[0] >= 0 && sy >= 0 && sz >= 0 && rows <= 32) {
        // a warp per non-mover, a lane per (y, z) row of its stencil: the rows' loads are
        // independent, so one item costs two memory latencies instead of 2 x rows
        const int lane = threadIdx.x & 31;
        const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
        const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
        const int dx = g.dims[0], dy = g.dims[1], dz = D == 3 ? g.dims[2] : 1, sx = g.near_s[0];
        for (int64_t k = warp; k < m; k += nwarps) {
            if (lane >= rows) continue;
            const int64_t i = active[k];
            double xi[D];
            const double4 vi = S.rec[i];
            rec_pos<D>(vi, xi);
            const int32_t idi = S.id[i];
            int c[3];
            decode_key<D>(g, skey[i], c);
            int y = c[1] + lane % (2 * sy + 1) - sy, z = D == 3 ? c[2] + lane / (2 * sy + 1) - sz : 0;
            y = y < 0 ? y + dy : (y >= dy ? y - dy : y);
            z = z < 0 ? z + dz : (z >= dz ? z - dz : z);
            const int64_t row = (static_cast<int64_t>(z) * dy + y) * dx;
            const int lo = c[0] - sx, hi = c[0] + sx;
            auto run = [&](int64_t b, int64_t e) {
                for (int64_t j = b; j < e; ++j) pair(i, xi, vi.w, idi, j);
            };
            if (lo < 0) {
                run(cs[row + lo + dx], cs[row + dx]);
                run(cs[row], cs[row + hi + 1]);
            } else if (hi >= dx) {
                run(cs[row + lo], cs[row + dx]);
                run(cs[row], cs[row + hi - dx + 1]);
            } else {
                run(cs[row + lo], cs[row + hi + 1]);
            }
        }
    } else {  // wide stencils: a thread per non-mover
        for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
            const int64_t i = active[k];
            double xi[D];
            const double4 vi = S.rec[i];
            rec_pos<D>(vi, xi);
            const int32_t idi = S.id[i];
            for_near_ranges<D>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
                for (int64_t j = b; j < e; ++j) pair(i, xi, vi.w, idi, j);
            });
        }
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

// Ordered candidate pairs of the reference's 3^d scan (cell_grid.hpp:137-157), from the
// cell offsets only (parity statistic, not on the timed path).
template <int D>
__global__ void __launch_bounds__(256) k_candidates(int64_t n, const GridParams* __restrict__ gp,
                                                    const cell_t* __restrict__ cs,
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
                                                      const cell_t* __restrict__ cs,
                                                      const uint32_t* __restrict__ skey,
                                                      int with_candidates, StatsDev* stats) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long pairs = 0, cand = 0;
    double pen = 0.0;
    if (i < n) {
        const GridParams& g = *gp;
        double xi[D];
        const double4 vi = S.rec[i];
        rec_pos<D>(vi, xi);
        const double ri = vi.w;
        const int32_t idi = S.id[i];
        for_near_ranges<D>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
            for (int64_t j = b; j < e; ++j) {
                if (j <= i || S.id[j] == idi) continue;
                double xj[D];
                const double4 vj = S.rec[j];
                rec_pos<D>(vj, xj);
                const double rr = ri + vj.w;
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

// Overlap statistics of a platelet state: unordered pairs {i, j > i} with overlap(i, j)
// or overlap(j, i) -- shape_any_collision tests every ordered pair, and the platelet
// test is not symmetric in its arguments (spherodisk.cpp), so the non-mover shortcut
// of the spheres does not apply.  Penetration is not defined for platelets (0).  A warp
// per particle i, a candidate j per lane (the stencil's contiguous ranges, 32 at a
// time); a pair the projections leave undecided in a direction goes to the rim-seed
// fallback run by the whole warp, a seed per lane.  The count is an OR per pair, so it
// does not depend on who decides what.
constexpr int kOverlapPlThreads = 128;
__global__ void __launch_bounds__(kOverlapPlThreads, 3) k_overlap_pl(int64_t n, State S, Box box,
                                                                  const GridParams* __restrict__ gp,
                                                                  const cell_t* __restrict__ cs,
                                                                  const uint32_t* __restrict__ skey, StatsDev* stats) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;  // whole warps
    unsigned long long pairs = 0, tests = 0;
    const GridParams& g = *gp;
    const double4 vi = S.rec[i], ai = S.aux[i];
    const int32_t idi = S.id[i];
    const pl::V3 ni{ai.x, ai.y, ai.z};
    const pl::V3 o{0.0, 0.0, 0.0};
    for_near_ranges<3>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
        for (int64_t base = b; base < e; base += 32) {
            const int64_t j = base + lane;
            // sa, sb: the stage of overlap(i, j) and overlap(j, i); kDwFalse for no pair
            int sa = pl::kDwFalse, sb = pl::kDwFalse;
            pl::V3 dij = o, dji = o, nj{0.0, 0.0, 1.0};
            double Dj = 0.0, tj = 0.0;
            if (j < e && j > i && S.id[j] != idi) {
                const double4 vj = S.rec[j], aj = S.aux[j];
                dij = pl::V3{min_image1(vj.x - vi.x, box.L[0], box.half[0]),
                             min_image1(vj.y - vi.y, box.L[1], box.half[1]),
                             min_image1(vj.z - vi.z, box.L[2], box.half[2])};
                dji = pl::V3{min_image1(vi.x - vj.x, box.L[0], box.half[0]),
                             min_image1(vi.y - vj.y, box.L[1], box.half[1]),
                             min_image1(vi.z - vj.z, box.L[2], box.half[2])};
                nj = pl::V3{aj.x, aj.y, aj.z};
                Dj = vj.w;
                tj = aj.w;
                sa = pl::spherodisk_overlap_pre(dij, ni, vi.w, ai.w, nj, Dj, tj);
                ++tests;
                if (sa != pl::kDwTrue) {
                    sb = pl::spherodisk_overlap_pre(dji, nj, Dj, tj, ni, vi.w, ai.w);
                    ++tests;
                }
            }
            const bool hit = sa == pl::kDwTrue || sb == pl::kDwTrue;
            pairs += hit ? 1 : 0;
            unsigned pend = __ballot_sync(0xffffffffu, !hit && (sa == pl::kDwSeeds || sb == pl::kDwSeeds));
            while (pend) {
                const int src = __ffs(pend) - 1;
                pend &= pend - 1u;
                const int qa = __shfl_sync(0xffffffffu, sa, src), qb = __shfl_sync(0xffffffffu, sb, src);
                const pl::V3 nq{__shfl_sync(0xffffffffu, nj.x, src), __shfl_sync(0xffffffffu, nj.y, src),
                                __shfl_sync(0xffffffffu, nj.z, src)};
                const double Dq = __shfl_sync(0xffffffffu, Dj, src), tq = __shfl_sync(0xffffffffu, tj, src);
                bool found = false;
                if (qa == pl::kDwSeeds) {  // overlap(i, j): disks (0, ni) and (dij, nj)
                    const pl::V3 d{__shfl_sync(0xffffffffu, dij.x, src), __shfl_sync(0xffffffffu, dij.y, src),
                                   __shfl_sync(0xffffffffu, dij.z, src)};
                    const bool h = pl::rim_seed_within(o, ni, 0.5 * (vi.w - ai.w), d, nq, 0.5 * (Dq - tq),
                                                       0.5 * (ai.w + tq), c_seed_table, lane);
                    found = __ballot_sync(0xffffffffu, h) != 0u;
                }
                if (!found && qb == pl::kDwSeeds) {  // overlap(j, i): disks (0, nj) and (dji, ni)
                    const pl::V3 d{__shfl_sync(0xffffffffu, dji.x, src), __shfl_sync(0xffffffffu, dji.y, src),
                                   __shfl_sync(0xffffffffu, dji.z, src)};
                    const bool h = pl::rim_seed_within(o, nq, 0.5 * (Dq - tq), d, ni, 0.5 * (vi.w - ai.w),
                                                       0.5 * (tq + ai.w), c_seed_table, lane);
                    found = __ballot_sync(0xffffffffu, h) != 0u;
                }
                if (found && lane == src) ++pairs;
            }
        }
    });
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        pairs += __shfl_down_sync(0xffffffffu, pairs, off);
        tests += __shfl_down_sync(0xffffffffu, tests, off);
    }
    if (lane == 0 && pairs) atomicAdd(&stats->overlap_pairs, pairs);
    if (lane == 0 && tests) atomicAdd(&stats->pair_tests, tests);
}

// platelet records (host layout) <-> device state, scattered back to slot order
__global__ void k_unpack_pl(int64_t n, const double* __restrict__ pos, const double* __restrict__ nrm,
                            const double* __restrict__ dia, const double* __restrict__ thk,
                            const int32_t* __restrict__ id, State T) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T.rec[i] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], dia[i]);
        T.aux[i] = make_double4(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2], thk[i]);
        T.id[i] = id ? id[i] : static_cast<int32_t>(i);
        T.slot[i] = static_cast<int32_t>(i);
    }
}

__global__ void k_pack_pl(int64_t n, State T, double* __restrict__ pos, double* __restrict__ nrm,
                          double* __restrict__ dia, double* __restrict__ thk, int32_t* __restrict__ id) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = T.slot[i];
        const double4 v = T.rec[i], a = T.aux[i];
        pos[3 * s] = v.x; pos[3 * s + 1] = v.y; pos[3 * s + 2] = v.z;
        nrm[3 * s] = a.x; nrm[3 * s + 1] = a.y; nrm[3 * s + 2] = a.z;
        dia[s] = v.w;
        thk[s] = a.w;
        id[s] = T.id[i];
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
        double p[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < D; ++a) p[a] = *reinterpret_cast<const double*>(b + off_pos + 8 * a);
        T.rec[i] = make_double4(p[0], p[1], p[2], *reinterpret_cast<const double*>(b + off_r));
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
        const double4 v = T.rec[i];
        const double p[3] = {v.x, v.y, v.z};
#pragma unroll
        for (int a = 0; a < D; ++a) *reinterpret_cast<double*>(b + off_pos + 8 * a) = p[a];
        *reinterpret_cast<double*>(b + off_r) = v.w;
    }
}

// interleaved host layout <-> SoA, scattered back to slot order
template <int D>
__global__ void k_unpack_soa(int64_t n, const double* __restrict__ pos, const double* __restrict__ r,
                             const int32_t* __restrict__ id, State T) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double p[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int a = 0; a < D; ++a) p[a] = pos[i * D + a];
        T.rec[i] = make_double4(p[0], p[1], p[2], r[i]);
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
        const double4 v = T.rec[i];
        const double p[3] = {v.x, v.y, v.z};
#pragma unroll
        for (int a = 0; a < D; ++a) pos[s * D + a] = p[a];
        r[s] = v.w;
        id[s] = T.id[i];
    }
}

__global__ void k_scale_radius(int64_t n, double4* __restrict__ rec, double4* __restrict__ aux, double factor) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        rec[i].w = rec[i].w * factor;              // engine.hpp:224 / shape.hpp:46 p.radius *= factor
        if (aux) aux[i].w = aux[i].w * factor;     // spherodisk.hpp:88-91 diameter, thickness
    }
}

template <int D>
__global__ void k_copy_state(int64_t n, State A, State B, const GridParams* sel_gp = nullptr,
                             const double4* rec_alt = nullptr) {
    if (sel_gp && sel_gp->resolve) A.rec = const_cast<double4*>(rec_alt);  // (graph runs, as k_stats_sweep)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        B.rec[i] = A.rec[i];
        if (A.aux) B.aux[i] = A.aux[i];
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
__global__ void __launch_bounds__(256) k_reduce_partials(int64_t n, const double4* __restrict__ rec,
                                                         double* __restrict__ part_sum,
                                                         double* __restrict__ part_max,
                                                         const double4* __restrict__ aux = nullptr) {
    __shared__ double ss[256], sm[256];
    const int64_t chunk = (n + kRedBlocks - 1) / kRedBlocks;
    const int64_t b0 = blockIdx.x * chunk;
    const int64_t b1 = b0 + chunk < n ? b0 + chunk : n;
    double s = 0.0, m = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += 256) {
        const double v = rec[i].w;
        if (aux) {  // platelets: swept volume, bounding radius (spherodisk.hpp:29-34, 94-96)
            const double t = aux[i].w;
            s = s + pl::spherodisk_measure(v, t);
            const double b = 0.5 * (v + t);
            m = b > m ? b : m;
        } else {
            s = s + particle_measure<D>(v);
            m = v > m ? v : m;
        }
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
