// srm_kernels.cuh -- CUDA kernels of the B200 SRM round (sm_100a).
//
// One SRM round (engine.hpp:227-234: build_shape_grid -> migrate -> shape_any_collision)
// is, on the device:
//   grid rebuild   k_keys -> k_scan_* -> k_scatter -> k_cellsort -> k_gather
//   migrate        k_phase0 (fused near-list build + attempt 0) -> k_phase (attempts >= 1)
//   reduction      k_stats  (overlap pairs, max penetration, movers, candidate pairs)
// All kernels read the grid / round parameters from device memory so that the same
// launches can be replayed from a CUDA graph.  DESIGN.md §2-§4 has the data layout
// and the roofline of each kernel.
#pragma once

#include <cstdint>

#include "srm_device.cuh"

namespace srmb {

constexpr int kNbrCap = 32;  // near-list capacity per particle; overflow -> full rescan
constexpr uint8_t kOverflow = 255;
constexpr int kScanTile = 4096;  // cells per scan tile (1024 threads x 4)

struct GridParams {
    int32_t dims[3];
    double edge[3];
    int64_t ncells;
    int32_t near_s[3];  // near-search half width per axis; -1 = every cell on the axis
    double extra;       // near cutoff: (ri + rj + extra) * (1 + 1e-9) + 1e-300
    double rmax;        // largest radius of the state the grid indexes
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
};

struct StatsDev {
    unsigned long long overlap_pairs;
    unsigned long long pen_bits;  // max penetration as the bits of a non-negative double
    unsigned long long candidate_pairs;
    unsigned long long nonmovers;     // particles that kept their round-start position
    unsigned long long active_count;  // length of the attempt-0 reject list
    unsigned long long fallback_tiles;  // phase-0 tiles that overflowed shared memory
    unsigned long long rejected[256];  // rejected after phase l (early exit of later phases)
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
#pragma unroll
        for (int a = 0; a < D; ++a) S.x[a][q] = T.x[a][src];
        S.r[q] = T.r[src];
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

// Rejected particles of attempt 0 are appended to the active list (warp-aggregated).
__device__ __forceinline__ void push_active(bool rejected, int64_t i, int32_t* __restrict__ active,
                                            StatsDev* stats) {
    const unsigned full = __activemask();
    const unsigned m = __ballot_sync(full, rejected);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(&stats->active_count, (unsigned long long)__popc(m));
    base = __shfl_sync(full, base, leader);
    if (rejected) active[base + __popc(m & ((1u << lane) - 1u))] = static_cast<int32_t>(i);
}

// Migrate attempt 0 fused with the near-list build for one particle, straight from
// global memory (the fallback of the tiled kernel).  S = sorted round-start state
// (read only), T = output state (sorted order): T.x = new positions, T.r/id/slot copied.
template <int D>
__device__ __forceinline__ bool phase0_global(int64_t i, const State& S, const State& T, const Box& box,
                                              const GridParams& g, const RoundParams& rp,
                                              const int64_t* __restrict__ cs,
                                              const uint32_t* __restrict__ skey,
                                              uint8_t* __restrict__ acc, int32_t* __restrict__ nbr,
                                              uint8_t* __restrict__ nbr_cnt) {
    double xi[D], p[D];
    load_pos<D>(S, i, xi);
    const double ri = S.r[i];
    const int32_t idi = S.id[i];
    const int32_t sloti = S.slot[i];
    propose<D>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sloti), 0u, p);
    bool ok = true;
    int nn = 0;
    bool overflow = false;
    int32_t* my = nbr + i * kNbrCap;
    for_near_ranges<D>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
        for (int64_t j = b; j < e; ++j) {
            if (j == i) continue;
            double xj[D];
            load_pos<D>(S, j, xj);
            const double rj = S.r[j];
            if (dist2<D>(box, xi, xj) > near_cut(ri, rj, g.extra)) continue;
            if (nn < kNbrCap) my[nn++] = static_cast<int32_t>(j);
            else overflow = true;
            if (!ok || S.id[j] == idi) continue;
            if (sphere_overlap<D>(box, p, ri, xj, rj)) { ok = false; continue; }
            double pj[D];
            propose<D>(box, xj, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[j]), 0u, pj);
            if (sphere_overlap<D>(box, p, ri, pj, rj)) ok = false;
        }
    });
#pragma unroll
    for (int a = 0; a < D; ++a) T.x[a][i] = ok ? p[a] : xi[a];
    T.r[i] = ri;
    T.id[i] = idi;
    T.slot[i] = sloti;
    acc[i] = ok ? 0 : kNotAccepted;
    nbr_cnt[i] = overflow ? kOverflow : static_cast<uint8_t>(nn);
    return !ok;
}

template <int D>
__global__ void __launch_bounds__(256) k_phase0(int64_t n, State S, State T, Box box,
                                                const GridParams* __restrict__ gp,
                                                const RoundParams* __restrict__ rpp,
                                                const int64_t* __restrict__ cs,
                                                const uint32_t* __restrict__ skey,
                                                uint8_t* __restrict__ acc, int32_t* __restrict__ nbr,
                                                uint8_t* __restrict__ nbr_cnt, int32_t* __restrict__ active,
                                                StatsDev* stats) {
    const GridParams g = *gp;
    const RoundParams rp = *rpp;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool rejected = false;
    if (i < n) rejected = phase0_global<D>(i, S, T, box, g, rp, cs, skey, acc, nbr, nbr_cnt);
    push_active(rejected, i, active, stats);
}


// Migrate attempt l >= 1 for the still-active particles, over the
// list of attempt-0 rejects (grid-stride; the list length is read on the device).
template <int D>
__global__ void __launch_bounds__(256) k_phase_list(int l, State S, State T, Box box,
                                                    const GridParams* __restrict__ gp,
                                                    const RoundParams* __restrict__ rpp,
                                                    const int64_t* __restrict__ cs,
                                                    const uint32_t* __restrict__ skey,
                                                    uint8_t* __restrict__ acc,
                                                    const int32_t* __restrict__ nbr,
                                                    const uint8_t* __restrict__ nbr_cnt,
                                                    const int32_t* __restrict__ active, StatsDev* stats) {
    if (l >= rpp->n_l) return;
    const int64_t m = static_cast<int64_t>(stats->active_count);
    if ((l == 1 ? static_cast<unsigned long long>(m) : stats->rejected[l - 1]) == 0) return;
    const GridParams& g = *gp;
    const RoundParams rp = *rpp;
    unsigned long long rej = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = active[k];
        if (acc[i] != kNotAccepted) continue;
        double xi[D], p[D];
        load_pos<D>(S, i, xi);
        const double ri = S.r[i];
        const int32_t idi = S.id[i];
        propose<D>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[i]), static_cast<uint32_t>(l), p);
        bool ok = true;
        auto test = [&](int64_t j) {
            if (!ok || S.id[j] == idi) return;
            const double rj = S.r[j];
            const uint8_t aj = acc[j];
            double xj[D];
            if (aj >= static_cast<uint8_t>(l)) {  // still active in this phase (or accepting now)
                load_pos<D>(S, j, xj);
                if (sphere_overlap<D>(box, p, ri, xj, rj)) { ok = false; return; }
                double pj[D];
                propose<D>(box, xj, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[j]),
                           static_cast<uint32_t>(l), pj);
                if (sphere_overlap<D>(box, p, ri, pj, rj)) ok = false;
            } else {  // accepted in an earlier phase: its final position
                load_pos<D>(T, j, xj);
                if (sphere_overlap<D>(box, p, ri, xj, rj)) ok = false;
            }
        };
        const uint8_t cnt = nbr_cnt[i];
        if (cnt != kOverflow) {
            const int32_t* my = nbr + i * kNbrCap;
            for (int t = 0; t < cnt && ok; ++t) test(my[t]);
        } else {
            for_near_ranges<D>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
                for (int64_t j = b; j < e && ok; ++j) {
                    if (j == i) continue;
                    double xj[D];
                    load_pos<D>(S, j, xj);
                    if (dist2<D>(box, xi, xj) > near_cut(ri, S.r[j], g.extra)) continue;
                    test(j);
                }
            });
        }
        if (ok) {
#pragma unroll
            for (int a = 0; a < D; ++a) T.x[a][i] = p[a];
            acc[i] = static_cast<uint8_t>(l);
        } else {
            ++rej;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rej += __shfl_down_sync(0xffffffffu, rej, o);
    if ((threadIdx.x & 31) == 0 && rej) atomicAdd(&stats->rejected[l], rej);
}

// Overlap reduction after the round.  Only pairs of non-movers can overlap (DESIGN.md
// §3.3) and every non-mover is on the attempt-0 reject list, so the reduction walks
// that list: each non-mover scans its near list for later non-movers.
template <int D>
__global__ void __launch_bounds__(256) k_stats_list(State S, Box box, const GridParams* __restrict__ gp,
                                                    const int64_t* __restrict__ cs,
                                                    const uint32_t* __restrict__ skey,
                                                    const uint8_t* __restrict__ acc,
                                                    const int32_t* __restrict__ nbr,
                                                    const uint8_t* __restrict__ nbr_cnt,
                                                    const int32_t* __restrict__ active, StatsDev* stats) {
    const int64_t m = static_cast<int64_t>(stats->active_count);
    const GridParams& g = *gp;
    unsigned long long pairs = 0, stay = 0;
    double pen = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = active[k];
        if (acc[i] != kNotAccepted) continue;
        ++stay;
        double xi[D];
        load_pos<D>(S, i, xi);
        const double ri = S.r[i];
        const int32_t idi = S.id[i];
        auto test = [&](int64_t j) {
            if (j <= i || acc[j] != kNotAccepted || S.id[j] == idi) return;
            double xj[D];
            load_pos<D>(S, j, xj);
            const double rr = ri + S.r[j];
            const double d2 = dist2<D>(box, xi, xj);
            if (d2 <= rr * rr) {
                ++pairs;
                const double pe = rr - sqrt(d2);
                pen = pe > pen ? pe : pen;
            }
        };
        const uint8_t c = nbr_cnt[i];
        if (c != kOverflow) {
            const int32_t* my = nbr + i * kNbrCap;
            for (int t = 0; t < c; ++t) test(my[t]);
        } else {
            for_near_ranges<D>(g, cs, skey[i], g.near_s, [&](int64_t b, int64_t e) {
                for (int64_t j = b; j < e; ++j) test(j);
            });
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        pairs += __shfl_down_sync(0xffffffffu, pairs, o);
        stay += __shfl_down_sync(0xffffffffu, stay, o);
        const double t = __shfl_down_sync(0xffffffffu, pen, o);
        pen = t > pen ? t : pen;
    }
    if ((threadIdx.x & 31) == 0) {
        if (pairs) atomicAdd(&stats->overlap_pairs, pairs);
        if (stay) atomicAdd(&stats->nonmovers, stay);
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
