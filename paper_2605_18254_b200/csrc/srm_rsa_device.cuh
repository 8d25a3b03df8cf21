// srm_rsa_device.cuh -- random sequential adsorption on the device (
// DESIGN.md §3.5).  The reference's rsa_place (rsa.hpp:21-61) is sequential: particle i
// draws uniform candidates until one is strictly non-touching every particle placed
// before it.  Here every unplaced particle draws its candidate of round r at once (a
// Philox counter (i, r), so a candidate is a pure function of (seed, i, r)), and a
// candidate is accepted iff it clears every particle placed in earlier rounds and no
// accepted lower-index candidate of round r overlaps it -- exactly the sequential RSA
// that visits the unplaced particles of each round in index order (oracle/srm_oracle.c
// orc_rsa_rounds), so each placed particle is uniform on the space left free before it.
//   k_rsa_propose  candidates of the unplaced particles (written over their records)
//   (grid build)   all n records, placed and candidates, sorted by cell
//   k_rsa_check    per candidate: clears the placed? its lower-index overlapping candidates
//   k_rsa_resolve  (repeated) accept iff no conflict accepted, once all are decided
//   k_rsa_commit   accepted -> placed
#pragma once

#include "srm_kernels.cuh"

namespace srmb {

constexpr int kRsaConf = 8;  // lower-index overlapping candidates kept per candidate

__device__ __forceinline__ void rsa_candidate(int dim, const Box& box, uint32_t k0, uint32_t k1, uint32_t i, uint32_t r,
                                              double* out) {
    const U4 a = philox4x32_10(U4{i, r, 0xFFFFFFFFu, 0u}, k0, k1);
    const U4 b = philox4x32_10(U4{i, r, 0xFFFFFFFFu, 1u}, k0, k1);
    const uint64_t w[3] = {((static_cast<uint64_t>(a.x) << 32) | a.y) >> 11,
                           ((static_cast<uint64_t>(a.z) << 32) | a.w) >> 11,
                           ((static_cast<uint64_t>(b.x) << 32) | b.y) >> 11};
    for (int d = 0; d < dim; ++d)
        out[d] = wrap1(__dmul_rn(__dmul_rn(__ull2double_rn(w[d]), 0x1p-53), box.L[d]), box.L[d]);
}

// record i = (candidate, r_i) for every unplaced particle (storage order: id = slot = i)
__global__ void k_rsa_propose(int64_t n, int dim, double4* __restrict__ rec, const uint8_t* __restrict__ placed,
                              Box box, uint32_t k0, uint32_t k1, uint32_t round) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (placed[i]) continue;
        double c[3] = {0.0, 0.0, 0.0};
        rsa_candidate(dim, box, k0, k1, static_cast<uint32_t>(i), round, c);
        rec[i] = make_double4(c[0], c[1], c[2], rec[i].w);
    }
}

// state[i]: 0 undecided, 1 accepted, 2 rejected; conf[i] = the lower-index candidates
// that overlap candidate i (nconf[i] > kRsaConf: overflow, reported to the host)
template <int D>
__global__ void __launch_bounds__(256) k_rsa_check(int64_t n, State S, Box box, const GridParams* __restrict__ gp,
                                                   const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                                   const uint8_t* __restrict__ placed, int8_t* __restrict__ state,
                                                   int32_t* __restrict__ conf, int32_t* __restrict__ nconf,
                                                   int64_t* __restrict__ where) {
    const GridParams& g = *gp;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = S.id[q];
        if (placed[i]) continue;
        where[i] = q;
        double x[D];
        const double4 v = S.rec[q];
        rec_pos<D>(v, x);
        bool clear = true;
        int nc = 0;
        for_near_ranges<D>(g, cs, skey[q], g.near_s, [&](int64_t b, int64_t e) {
            for (int64_t j = b; j < e && clear; ++j) {
                if (j == q) continue;
                double y[D];
                const double4 w = S.rec[j];
                rec_pos<D>(w, y);
                const double rr = v.w + w.w;
                if (dist2<D>(box, x, y) > rr * rr) continue;  // rsa.hpp: strictly non-touching
                const int32_t k = S.id[j];
                if (placed[k]) {
                    clear = false;
                } else if (k < i) {
                    if (nc < kRsaConf) conf[static_cast<int64_t>(i) * kRsaConf + nc] = k;
                    ++nc;
                }
            }
        });
        state[i] = clear ? 0 : 2;
        nconf[i] = clear ? nc : 0;
    }
}

// one sweep of the resolution: a candidate is accepted once every conflicting candidate
// is rejected, rejected as soon as one is accepted (a candidate with more than kRsaConf
// conflicts rescans its stencil for them)
template <int D>
__global__ void k_rsa_resolve(int64_t n, const uint8_t* __restrict__ placed, int8_t* __restrict__ state,
                              const int32_t* __restrict__ conf, const int32_t* __restrict__ nconf,
                              int* __restrict__ undecided, State S, Box box, const GridParams* __restrict__ gp,
                              const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                              const int64_t* __restrict__ where) {
    int left = 0;
    const volatile int8_t* vs = state;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (placed[i] || state[i] != 0) continue;
        const int nc = nconf[i];
        bool all_rejected = true, any_accepted = false;
        if (nc <= kRsaConf) {
            for (int t = 0; t < nc; ++t) {
                const int8_t st = vs[conf[i * kRsaConf + t]];
                any_accepted = any_accepted || st == 1;
                all_rejected = all_rejected && st == 2;
            }
        } else {  // the sorted position of i, its stencil, its lower-index overlapping candidates
            const int64_t q = where[i];
            double x[D];
            const double4 v = S.rec[q];
            rec_pos<D>(v, x);
            for_near_ranges<D>(*gp, cs, skey[q], gp->near_s, [&](int64_t b, int64_t e) {
                for (int64_t j = b; j < e; ++j) {
                    const int32_t k = S.id[j];
                    if (j == q || k >= i || placed[k]) continue;
                    double y[D];
                    const double4 w = S.rec[j];
                    rec_pos<D>(w, y);
                    const double rr = v.w + w.w;
                    if (dist2<D>(box, x, y) > rr * rr) continue;
                    const int8_t st = vs[k];
                    any_accepted = any_accepted || st == 1;
                    all_rejected = all_rejected && st == 2;
                }
            });
        }
        if (any_accepted) state[i] = 2;
        else if (all_rejected) state[i] = 1;
        else ++left;
    }
    if (left) atomicAdd(undecided, left);
}

__global__ void k_rsa_commit(int64_t n, uint8_t* __restrict__ placed, const int8_t* __restrict__ state,
                             unsigned long long* __restrict__ count) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (!placed[i] && state[i] == 1) {
            placed[i] = 1;
            ++c;
        }
    }
    if (c) atomicAdd(count, c);
}

// ---- platelets (rsa_platelets, recipes.cpp:107-148) ---------------------------------
// The same rounds with candidate = (centre, normal): the centre as for spheres, the normal
// the unit vector of (slot i, attempt r, stream 1) under the key (seed, round_id 0xFFFFFF,
// iteration 0xFFFFFFFF) -- counters no sweep uses.  A candidate is placed iff the
// reference's test overlap(candidate, p) (shape.hpp:64-73, candidate first; asymmetric)
// is false for every platelet p placed before it in (round, index) order (oracle
// orc_rsa_pl_rounds).  Records: rec = (centre, D), aux = (normal, t).
__device__ __forceinline__ RngKey rsa_pl_key(uint32_t k0, uint32_t k1) { return RngKey{k0, k1, 0xFFFFFFu, 0xFFFFFFFFu}; }

__global__ void k_rsa_pl_propose(int64_t n, double4* __restrict__ rec, double4* __restrict__ aux,
                                 const uint8_t* __restrict__ placed, Box box, uint32_t k0, uint32_t k1,
                                 uint32_t round) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (placed[i]) continue;
        double c[3], u[3];
        rsa_candidate(3, box, k0, k1, static_cast<uint32_t>(i), round, c);
        unit_vector<3>(rsa_pl_key(k0, k1), static_cast<uint32_t>(i), round, 1, u);
        rec[i] = make_double4(c[0], c[1], c[2], rec[i].w);
        aux[i] = make_double4(u[0], u[1], u[2], aux[i].w);
    }
}

// overlap(candidate at sorted q, platelet at sorted j) with the candidate first
__device__ __forceinline__ bool rsa_pl_hits(const State& S, const Box& box, int64_t q, int64_t j) {
    const double4 v = S.rec[q], a = S.aux[q], w = S.rec[j], b = S.aux[j];
    const pl::V3 d{min_image1(w.x - v.x, box.L[0], box.half[0]), min_image1(w.y - v.y, box.L[1], box.half[1]),
                   min_image1(w.z - v.z, box.L[2], box.half[2])};
    return pl::spherodisk_overlap(d, pl::V3{a.x, a.y, a.z}, v.w, a.w, pl::V3{b.x, b.y, b.z}, w.w, b.w, c_seed_table);
}

__global__ void __launch_bounds__(256) k_rsa_pl_check(int64_t n, State S, Box box, const GridParams* __restrict__ gp,
                                                      const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                                      const uint8_t* __restrict__ placed, int8_t* __restrict__ state,
                                                      int32_t* __restrict__ conf, int32_t* __restrict__ nconf,
                                                      int64_t* __restrict__ where) {
    const GridParams& g = *gp;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t i = S.id[q];
        if (placed[i]) continue;
        where[i] = q;
        bool clear = true;
        int nc = 0;
        for_near_ranges<3>(g, cs, skey[q], g.near_s, [&](int64_t b, int64_t e) {
            for (int64_t j = b; j < e && clear; ++j) {
                if (j == q) continue;
                const int32_t k = S.id[j];
                if (!placed[k] && k > i) continue;  // later candidates of the round do not matter to i
                if (!rsa_pl_hits(S, box, q, j)) continue;
                if (placed[k]) {
                    clear = false;
                } else {
                    if (nc < kRsaConf) conf[static_cast<int64_t>(i) * kRsaConf + nc] = k;
                    ++nc;
                }
            }
        });
        state[i] = clear ? 0 : 2;
        nconf[i] = clear ? nc : 0;
    }
}

__global__ void k_rsa_pl_resolve(int64_t n, const uint8_t* __restrict__ placed, int8_t* __restrict__ state,
                                 const int32_t* __restrict__ conf, const int32_t* __restrict__ nconf,
                                 int* __restrict__ undecided, State S, Box box, const GridParams* __restrict__ gp,
                                 const cell_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                                 const int64_t* __restrict__ where) {
    int left = 0;
    const volatile int8_t* vs = state;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (placed[i] || state[i] != 0) continue;
        const int nc = nconf[i];
        bool all_rejected = true, any_accepted = false;
        if (nc <= kRsaConf) {
            for (int t = 0; t < nc; ++t) {
                const int8_t st = vs[conf[i * kRsaConf + t]];
                any_accepted = any_accepted || st == 1;
                all_rejected = all_rejected && st == 2;
            }
        } else {  // more conflicts than kept: rescan the stencil for them
            const int64_t q = where[i];
            for_near_ranges<3>(*gp, cs, skey[q], gp->near_s, [&](int64_t b, int64_t e) {
                for (int64_t j = b; j < e; ++j) {
                    const int32_t k = S.id[j];
                    if (j == q || k >= i || placed[k]) continue;
                    if (!rsa_pl_hits(S, box, q, j)) continue;
                    const int8_t st = vs[k];
                    any_accepted = any_accepted || st == 1;
                    all_rejected = all_rejected && st == 2;
                }
            });
        }
        if (any_accepted) state[i] = 2;
        else if (all_rejected) state[i] = 1;
        else ++left;
    }
    if (left) atomicAdd(undecided, left);
}

}  // namespace srmb
