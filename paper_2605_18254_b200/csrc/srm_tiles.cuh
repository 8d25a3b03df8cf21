// srm_tiles.cuh -- attempt 0 of the parallel migrate as a shared-memory brick kernel.
//
// One CTA owns a brick of Bx x By x Bz cells of the round's grid.  It stages the brick
// plus a halo of s cells per side (s = near-search half width) into shared memory:
// the staged cells are (By+2s)(Bz+2s) contiguous x-runs of the cell-sorted SoA, so the
// copy is a set of coalesced row segments (one thread per staged particle).  Brick
// particles then compute their attempt-0 proposal once (Philox + unit vector + wrap)
// and scan their neighbourhood from shared memory:
//   1. the per-particle stencil is pruned: x cells and y/z rows whose box lies beyond
//      the largest possible cutoff are skipped (fp32, margin-protected);
//   2. an fp32 prefilter on brick-relative coordinates (no min-image inside a brick)
//      selects near candidates -- a superset of the fp64 near set, which is all the
//      near list needs;
//   3. the attempt decision uses fp32 "definitely clear" pre-tests and the exact fp64
//      reference predicate (shape.hpp:508-511) whenever the fp32 test cannot exclude
//      contact.  Halo neighbours' proposals are computed lazily, only for near pairs.
// All fp32 tests carry an absolute margin larger than their rounding error, so every
// decision equals phase0_global's (and the oracle's) bit for bit.  A brick whose staged
// count exceeds the shared-memory capacity falls back to phase0_global.
#pragma once

#include "srm_kernels.cuh"

namespace srmb {

constexpr int kTileThreads = 256;
constexpr int kMaxRows = 256;
constexpr int kTileSmemMax = 150 * 1024;  // dynamic shared memory per brick CTA, upper bound

struct AxisTile {
    int32_t full;   // the brick spans the whole axis (one brick along it), cells in global order
    int32_t all;    // the near stencil covers every cell along the axis
    int32_t B;      // brick width in cells (dims when full)
    int32_t ntile;  // bricks along the axis
    int32_t s;      // near half width (when !all)
};

struct TileParams {
    AxisTile ax[3];
    int64_t ntiles;
    int32_t capS;        // staged particles per brick (shared-memory capacity)
    int32_t capC;        // brick (centre) particles per brick
    int32_t nst_max[3];  // staged cells per axis, upper bound
    float margin;        // absolute fp32 margin (covers the rounding of brick coordinates)
    float extra_f;       // near-cut extra (2 c_m) in fp32
    float rmax_f;        // largest radius (stencil pruning)
    float edge_f[3];
    int32_t enabled;
    int32_t bricks_only;  // every axis in brick mode: the pair-parallel, min-image-free path
    int32_t smem_bytes;
    int32_t maxseg;       // stencil rows per particle (pair kernel segments)
};

__device__ __forceinline__ int block_excl_scan_int(int v, int* total) {
    __shared__ int warp_sum[kTileThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int w = lane < kTileThreads / 32 ? warp_sum[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < kTileThreads / 32) warp_sum[lane] = wi - w;
        if (lane == kTileThreads / 32 - 1) *total = wi;
    }
    __syncthreads();
    const int r = warp_sum[wid] + incl - v;
    __syncthreads();
    return r;
}

// largest j in [0, n) with a[j] <= v (a non-decreasing, a[0] <= v)
__device__ __forceinline__ int upper_index(const int* a, int n, int v) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a[mid] <= v) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// fp32 squared distance of two brick-frame points; min-image on whole-axis bricks
template <int D, bool BR>
__device__ __forceinline__ float d2_rel(const float4& a, const float4& b, const bool* mi, const float* Lf,
                                        const float* Hf) {
    float dx = b.x - a.x, dy = b.y - a.y, dz = D == 3 ? b.z - a.z : 0.f;
    if (!BR) {
        if (mi[0]) { if (dx > Hf[0]) dx -= Lf[0]; else if (dx < -Hf[0]) dx += Lf[0]; }
        if (mi[1]) { if (dy > Hf[1]) dy -= Lf[1]; else if (dy < -Hf[1]) dy += Lf[1]; }
        if (D == 3 && mi[2]) { if (dz > Hf[2]) dz -= Lf[2]; else if (dz < -Hf[2]) dz += Lf[2]; }
    }
    return __fmaf_rn(dx, dx, __fmaf_rn(dy, dy, __fmul_rn(dz, dz)));
}

// "definitely farther than lim" with the relative slack of the fp32 rounding
__device__ __forceinline__ bool clear_f(float d2, float lim) { return d2 > __fmul_rn(__fmul_rn(lim, lim), 1.00001f); }
// "definitely within lim" (lim already reduced by the absolute margin)
__device__ __forceinline__ bool inside_f(float d2, float lim) {
    return lim > 0.f && d2 < __fmul_rn(__fmul_rn(lim, lim), 0.99999f);
}

template <int D>
__device__ __forceinline__ float4 rel_of_proposal(const float4& rel_x0, const double* x0, const double* p,
                                                  const Box& box) {
    float v[3] = {rel_x0.x, rel_x0.y, rel_x0.z};
#pragma unroll
    for (int a = 0; a < D; ++a)
        v[a] = __fadd_rn(v[a], static_cast<float>(min_image1(p[a] - x0[a], box.L[a], box.half[a])));
    return make_float4(v[0], v[1], v[2], rel_x0.w);
}

template <int D, bool BR>
__global__ void __launch_bounds__(kTileThreads, 3)
    k_phase0_tiled(State S, State T, Box box, const GridParams* __restrict__ gp,
                   const TileParams* __restrict__ tpp, const RoundParams* __restrict__ rpp,
                   const int64_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                   uint8_t* __restrict__ acc, int32_t* __restrict__ nbr, uint8_t* __restrict__ nbr_cnt,
                   int32_t* __restrict__ active, StatsDev* stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_rowbase[kMaxRows + 1];
    __shared__ int s_lenA[kMaxRows];
    __shared__ int s_kA[kMaxRows];
    __shared__ int s_A0[kMaxRows];
    __shared__ long long s_gA[kMaxRows], s_gB[kMaxRows], s_rc0[kMaxRows];
    __shared__ signed char s_shA[kMaxRows], s_shB[kMaxRows], s_shY[kMaxRows], s_shZ[kMaxRows];
    __shared__ int s_cpre[kMaxRows + 1];
    __shared__ int s_crow[kMaxRows];
    __shared__ int s_total;

    const GridParams& g = *gp;
    const TileParams& tp = *tpp;
    const RoundParams rp = *rpp;
    const int capS = tp.capS, capC = tp.capC;
    float4* srel = reinterpret_cast<float4*>(smem_raw);
    float4* spf = srel + capS;
    double* sx0 = reinterpret_cast<double*>(spf + capC);
    double* sr = sx0 + D * capS;
    double* sp = sr + capS;
    int* sid = reinterpret_cast<int*>(sp + D * capC);
    int* sgi = sid + capS;
    int* sslot = sgi + capS;
    int* coff = sslot + capS;
    const int X1 = tp.nst_max[0] + 1;
    const int dimsv[3] = {g.dims[0], g.dims[1], D == 3 ? g.dims[2] : 1};
    const int dx = dimsv[0], dy = dimsv[1];
    const float Lf[3] = {static_cast<float>(box.L[0]), static_cast<float>(box.L[1]), static_cast<float>(box.L[2])};
    const float Hf[3] = {0.5f * Lf[0], 0.5f * Lf[1], 0.5f * Lf[2]};
    const bool mi[3] = {tp.ax[0].full != 0, tp.ax[1].full != 0, tp.ax[2].full != 0};
    const float margin = tp.margin, extra_f = tp.extra_f;

    for (int64_t t = blockIdx.x; t < tp.ntiles; t += gridDim.x) {
        int tc[3];
        {
            int64_t rest = t;
            tc[0] = static_cast<int>(rest % tp.ax[0].ntile);
            rest /= tp.ax[0].ntile;
            tc[1] = static_cast<int>(rest % tp.ax[1].ntile);
            tc[2] = static_cast<int>(rest / tp.ax[1].ntile);
        }
        int o[3], Be[3], nst[3], c0[3];
        double origin[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const AxisTile& A = tp.ax[a];
            if (A.full) {
                o[a] = 0; Be[a] = dimsv[a]; nst[a] = dimsv[a]; c0[a] = 0; origin[a] = 0.0;
            } else {
                o[a] = tc[a] * A.B;
                Be[a] = min(A.B, dimsv[a] - o[a]);
                nst[a] = Be[a] + 2 * A.s;
                c0[a] = A.s;
                origin[a] = static_cast<double>(o[a]) * g.edge[a];
            }
        }
        const int nrows = nst[1] * nst[2];

        // ---- 1. staged rows: global row, x chunks, periodic shifts -------------------
        int tot = 0;
        if (threadIdx.x < nrows) {
            const int r = threadIdx.x;
            const int iy = r % nst[1], iz = r / nst[1];
            int gy = tp.ax[1].full ? iy : o[1] - tp.ax[1].s + iy;
            int gz = tp.ax[2].full ? iz : o[2] - tp.ax[2].s + iz;
            // unwrapped cell u < 0 is global cell u + dims: its positions sit one box
            // length above the brick, so they are shifted by -L (and u >= dims by +L)
            signed char shy = 0, shz = 0;
            if (gy < 0) { gy += dy; shy = -1; } else if (gy >= dy) { gy -= dy; shy = 1; }
            if (gz < 0) { gz += dimsv[2]; shz = -1; } else if (gz >= dimsv[2]) { gz -= dimsv[2]; shz = 1; }
            const long long rc0 = (static_cast<long long>(gz) * dy + gy) * dx;
            int A0, A1, B1 = 0, kA;
            signed char shA = 0, shB = 0;
            if (tp.ax[0].full) {
                A0 = 0; A1 = dx; kA = dx;
            } else {
                const int u0 = o[0] - tp.ax[0].s, u1 = u0 + nst[0];
                if (u0 < 0) { A0 = u0 + dx; A1 = dx; shA = -1; B1 = u1; }
                else if (u1 > dx) { A0 = u0; A1 = dx; B1 = u1 - dx; shB = 1; }
                else { A0 = u0; A1 = u1; }
                kA = A1 - A0;
            }
            const long long gA = cs[rc0 + A0];
            const int lenA = static_cast<int>(cs[rc0 + A1] - gA);
            const long long gB = cs[rc0];
            const int lenB = B1 > 0 ? static_cast<int>(cs[rc0 + B1] - gB) : 0;
            tot = lenA + lenB;
            s_lenA[r] = lenA; s_kA[r] = kA; s_A0[r] = A0;
            s_gA[r] = gA; s_gB[r] = gB; s_rc0[r] = rc0;
            s_shA[r] = shA; s_shB[r] = shB; s_shY[r] = shy; s_shZ[r] = shz;
        }
        const int rb = block_excl_scan_int(tot, &s_total);
        if (threadIdx.x < nrows) s_rowbase[threadIdx.x] = rb;
        if (threadIdx.x == nrows - 1) s_rowbase[nrows] = rb + tot;
        const int total = s_total;
        __syncthreads();  // s_rowbase[] complete before any thread reads it

        // ---- 2. local cell offsets (rows x (nst_x + 1)) ----------------------------------
        if (total <= capS) {
            for (int idx = threadIdx.x; idx < nrows * (nst[0] + 1); idx += blockDim.x) {
                const int r = idx / (nst[0] + 1), k = idx % (nst[0] + 1);
                int off;
                if (k == nst[0]) off = s_rowbase[r + 1] - s_rowbase[r];
                else if (k < s_kA[r]) off = static_cast<int>(cs[s_rc0[r] + s_A0[r] + k] - s_gA[r]);
                else off = s_lenA[r] + static_cast<int>(cs[s_rc0[r] + (k - s_kA[r])] - s_gB[r]);
                coff[r * X1 + k] = s_rowbase[r] + off;
            }
        }
        __syncthreads();

        // ---- 3. brick rows and their particle counts ---------------------------------------
        const int ncr = Be[1] * Be[2];
        int ccount = 0;
        if (total <= capS && threadIdx.x < ncr) {
            const int c = threadIdx.x;
            const int r = (c0[2] + c / Be[1]) * nst[1] + (c0[1] + c % Be[1]);
            s_crow[c] = r;
            ccount = coff[r * X1 + c0[0] + Be[0]] - coff[r * X1 + c0[0]];
        }
        const int cpre = block_excl_scan_int(ccount, &s_total);
        if (threadIdx.x < ncr) s_cpre[threadIdx.x] = cpre;
        if (threadIdx.x == ncr - 1) s_cpre[ncr] = cpre + ccount;
        const int nc = s_total;

        if (total > capS || nc > capC) {
            // ---- fallback: brick particles straight from global memory ---------------
            if (threadIdx.x == 0) atomicAdd(&stats->fallback_tiles, 1ull);
            for (int c = 0; c < Be[1] * Be[2]; ++c) {
                const int gy = o[1] + c % Be[1], gz = o[2] + c / Be[1];
                const long long rc0 = (static_cast<long long>(gz) * dy + gy) * dx;
                const long long b = cs[rc0 + o[0]], e = cs[rc0 + o[0] + Be[0]];
                for (long long i = b + threadIdx.x; i < e; i += blockDim.x) {
                    const bool rej = phase0_global<D>(i, S, T, box, g, rp, cs, skey, acc, nbr, nbr_cnt);
                    if (rej) {
                        const unsigned long long pos = atomicAdd(&stats->active_count, 1ull);
                        active[pos] = static_cast<int32_t>(i);
                    }
                }
            }
            __syncthreads();
            continue;
        }

        // ---- 4. stage every particle of the brick + halo (thread per particle) ---------------
        for (int q = threadIdx.x; q < total; q += blockDim.x) {
            const int r = upper_index(s_rowbase, nrows, q);
            const int e = q - s_rowbase[r];
            const int lenA = s_lenA[r];
            const long long gsrc = e < lenA ? s_gA[r] + e : s_gB[r] + (e - lenA);
            double x0[D];
            load_pos<D>(S, gsrc, x0);
            const double sh[3] = {(e < lenA ? s_shA[r] : s_shB[r]) * box.L[0], s_shY[r] * box.L[1],
                                  s_shZ[r] * box.L[2]};
            float rel[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int a = 0; a < D; ++a) {
                sx0[a * capS + q] = x0[a];
                rel[a] = static_cast<float>(x0[a] + sh[a] - origin[a]);
            }
            const double rr = S.r[gsrc];
            sr[q] = rr;
            srel[q] = make_float4(rel[0], rel[1], rel[2], static_cast<float>(rr));
            sid[q] = S.id[gsrc];
            sgi[q] = static_cast<int>(gsrc);
            sslot[q] = S.slot[gsrc];
        }
        __syncthreads();

        // ---- 5. attempt-0 proposals of the brick particles (once each) --------------------
        for (int c = threadIdx.x; c < nc; c += blockDim.x) {
            const int j = upper_index(s_cpre, ncr, c);
            const int q = coff[s_crow[j] * X1 + c0[0]] + (c - s_cpre[j]);
            double x0[D], p[D];
#pragma unroll
            for (int a = 0; a < D; ++a) x0[a] = sx0[a * capS + q];
            propose<D>(box, x0, rp.c_m, rp.key, static_cast<uint32_t>(sslot[q]), 0u, p);
#pragma unroll
            for (int a = 0; a < D; ++a) sp[a * capC + c] = p[a];
            spf[c] = rel_of_proposal<D>(srel[q], x0, p, box);
        }
        __syncthreads();

        // ---- 6. attempt 0 for the brick particles ----------------------------------------
        for (int cb = 0; cb < nc; cb += blockDim.x) {
            const int c = cb + threadIdx.x;
            bool rejected = false;
            int gi = -1;
            if (c < nc) {
                const int jrow = upper_index(s_cpre, ncr, c);
                const int r = s_crow[jrow];
                const int q = coff[r * X1 + c0[0]] + (c - s_cpre[jrow]);
                gi = sgi[q];
                const int iy = r % nst[1], iz = r / nst[1];
                const int cx = static_cast<int>(skey[gi] % static_cast<uint32_t>(dx));
                const int kx = tp.ax[0].full ? cx : cx - (o[0] - tp.ax[0].s);
                const float4 me = srel[q];
                const float4 mp = spf[c];
                bool ok = true, overflow = false;
                int nn = 0;
                int32_t* my = nbr + static_cast<int64_t>(gi) * kNbrCap;
                const float lim_near = __fadd_rn(__fadd_rn(me.w, extra_f), margin);  // + rj
                const float lim_ov = __fadd_rn(me.w, margin);                        // + rj

                // one staged candidate q2; c2base >= 0 marks a brick row (c2 = c2base + q2)
                auto visit = [&](int q2, int c2base, int qlo, int qhi) {
                    const float4 cq = srel[q2];
                    if (clear_f(d2_rel<D, BR>(me, cq, mi, Lf, Hf), __fadd_rn(lim_near, cq.w))) return;
                    if (q2 == q) return;
                    if (nn < kNbrCap) my[nn++] = sgi[q2];
                    else overflow = true;
                    if (!ok || sid[q2] == sid[q]) return;
                    const float lov = __fadd_rn(lim_ov, cq.w);
                    // p_i against x0_j
                    if (!clear_f(d2_rel<D, BR>(mp, cq, mi, Lf, Hf), lov)) {
                        double pi[D], xj[D];
#pragma unroll
                        for (int a = 0; a < D; ++a) { pi[a] = sp[a * capC + c]; xj[a] = sx0[a * capS + q2]; }
                        if (sphere_overlap<D>(box, pi, sr[q], xj, sr[q2])) { ok = false; return; }
                    }
                    // p_i against p_j (brick particle: stored; halo: computed here)
                    const bool brick = c2base >= 0 && q2 >= qlo && q2 < qhi;
                    double pj[D], xj[D];
                    float4 pf;
                    if (brick) {
                        pf = spf[c2base + q2];
                    } else {
#pragma unroll
                        for (int a = 0; a < D; ++a) xj[a] = sx0[a * capS + q2];
                        propose<D>(box, xj, rp.c_m, rp.key, static_cast<uint32_t>(sslot[q2]), 0u, pj);
                        pf = rel_of_proposal<D>(cq, xj, pj, box);
                    }
                    if (clear_f(d2_rel<D, BR>(mp, pf, mi, Lf, Hf), lov)) return;
                    if (brick) {
#pragma unroll
                        for (int a = 0; a < D; ++a) pj[a] = sp[a * capC + c2base + q2];
                    }
                    double pi[D];
#pragma unroll
                    for (int a = 0; a < D; ++a) pi[a] = sp[a * capC + c];
                    if (sphere_overlap<D>(box, pi, sr[q], pj, sr[q2])) ok = false;
                };
                // brick-row bookkeeping of staged row r2: q-range of its brick cells and c base
                auto brick_row = [&](int r2, int& qlo, int& qhi) -> int {
                    const int iy2 = r2 % nst[1], iz2 = r2 / nst[1];
                    const int jy = iy2 - c0[1], jz = iz2 - c0[2];
                    if (jy < 0 || jy >= Be[1] || jz < 0 || jz >= Be[2]) return -1;
                    const int jj = jz * Be[1] + jy;
                    qlo = coff[r2 * X1 + c0[0]];
                    qhi = coff[r2 * X1 + c0[0] + Be[0]];
                    return s_cpre[jj] - qlo;
                };

                if (BR) {
                    // pruned stencil: cells/rows whose box is beyond the largest cutoff
                    const float cutm = __fadd_rn(__fadd_rn(__fadd_rn(me.w, tp.rmax_f), extra_f), __fmul_rn(2.f, margin));
                    auto lohi = [&](float v, int kc, int s, float e, int& lo, int& hi) {
                        lo = max(kc - s, static_cast<int>(floorf(__fdiv_rn(__fsub_rn(v, cutm), e))) + s);
                        hi = min(kc + s, static_cast<int>(ceilf(__fdiv_rn(__fadd_rn(v, cutm), e))) - 1 + s);
                    };
                    int xlo, xhi, ylo, yhi, zlo = 0, zhi = 0;
                    lohi(me.x, kx, tp.ax[0].s, tp.edge_f[0], xlo, xhi);
                    lohi(me.y, iy, tp.ax[1].s, tp.edge_f[1], ylo, yhi);
                    if (D == 3) lohi(me.z, iz, tp.ax[2].s, tp.edge_f[2], zlo, zhi);
                    const float cut2 = __fmul_rn(__fmul_rn(cutm, cutm), 1.00001f);
                    for (int iz2 = zlo; iz2 <= zhi; ++iz2) {
                        float dzd = 0.f;
                        if (D == 3) {
                            const float zb = (iz2 - tp.ax[2].s) * tp.edge_f[2];
                            dzd = fmaxf(0.f, fmaxf(zb - me.z, me.z - (zb + tp.edge_f[2])));
                        }
                        for (int iy2 = ylo; iy2 <= yhi; ++iy2) {
                            const float yb = (iy2 - tp.ax[1].s) * tp.edge_f[1];
                            const float dyd = fmaxf(0.f, fmaxf(yb - me.y, me.y - (yb + tp.edge_f[1])));
                            if (__fmaf_rn(dyd, dyd, __fmul_rn(dzd, dzd)) > cut2) continue;
                            const int r2 = iz2 * nst[1] + iy2;
                            int qlo = 0, qhi = 0;
                            const int c2b = brick_row(r2, qlo, qhi);
                            const int b = coff[r2 * X1 + xlo], e = coff[r2 * X1 + xhi + 1];
                            for (int q2 = b; q2 < e; ++q2) visit(q2, c2b, qlo, qhi);
                        }
                    }
                } else {
                    auto scan_range = [&](int r2, int b, int e) {
                        int qlo = 0, qhi = 0;
                        const int c2b = brick_row(r2, qlo, qhi);
                        for (int q2 = b; q2 < e; ++q2) visit(q2, c2b, qlo, qhi);
                    };
                    auto scan_row = [&](int r2) {
                        const int bse = r2 * X1;
                        const AxisTile& A = tp.ax[0];
                        if (A.all) {
                            scan_range(r2, coff[bse], coff[bse + nst[0]]);
                        } else if (A.full) {
                            const int lo2 = kx - A.s, hi2 = kx + A.s;
                            if (lo2 < 0) {
                                scan_range(r2, coff[bse + lo2 + dx], coff[bse + dx]);
                                scan_range(r2, coff[bse], coff[bse + hi2 + 1]);
                            } else if (hi2 >= dx) {
                                scan_range(r2, coff[bse + lo2], coff[bse + dx]);
                                scan_range(r2, coff[bse], coff[bse + hi2 - dx + 1]);
                            } else {
                                scan_range(r2, coff[bse + lo2], coff[bse + hi2 + 1]);
                            }
                        } else {
                            scan_range(r2, coff[bse + kx - A.s], coff[bse + kx + A.s + 1]);
                        }
                    };
                    auto axis_rows = [&](int axis, int ic, int n_st, int* list) -> int {
                        const AxisTile& A = tp.ax[axis];
                        int m = 0;
                        if (A.all) {
                            for (int k = 0; k < n_st; ++k) list[m++] = k;
                        } else if (A.full) {
                            for (int d = -A.s; d <= A.s; ++d) {
                                int k = ic + d;
                                if (k < 0) k += dimsv[axis];
                                if (k >= dimsv[axis]) k -= dimsv[axis];
                                list[m++] = k;
                            }
                        } else {
                            for (int d = -A.s; d <= A.s; ++d) list[m++] = ic + d;
                        }
                        return m;
                    };
                    int ylist[16], zlist[16];
                    const int ny = axis_rows(1, iy, nst[1], ylist);
                    const int nz = D == 3 ? axis_rows(2, iz, nst[2], zlist) : 1;
                    if (D == 2) zlist[0] = 0;
                    for (int zz = 0; zz < nz; ++zz)
                        for (int yy = 0; yy < ny; ++yy) scan_row(zlist[zz] * nst[1] + ylist[yy]);
                }

                double pi[D], xi[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    pi[a] = sp[a * capC + c];
                    xi[a] = sx0[a * capS + q];
                }
#pragma unroll
                for (int a = 0; a < D; ++a) T.x[a][gi] = ok ? pi[a] : xi[a];
                T.r[gi] = sr[q];
                T.id[gi] = sid[q];
                T.slot[gi] = sslot[q];
                acc[gi] = ok ? 0 : kNotAccepted;
                nbr_cnt[gi] = overflow ? kOverflow : static_cast<uint8_t>(nn);
                rejected = !ok;
            }
            push_active(rejected, gi, active, stats);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------
// Pair-parallel brick kernel (every axis in brick mode).  Same staging as above, but
// the neighbourhood scan is flattened: each brick particle's pruned stencil becomes a
// list of contiguous shared-memory segments, a block-wide prefix over the candidate
// counts numbers all (particle, candidate) pairs of the brick, and threads take
// uniform chunks of kPairChunk consecutive pairs.  Per-particle results (near list,
// conflict flag) merge through shared-memory atomics; near-list order is irrelevant to
// every consumer (later attempts and the reduction AND / count over it).  Proposals of
// all staged particles are computed in one uniform pass; the exact fp64 tests (close
// calls only) reload positions from global memory and recompute the proposal.
constexpr int kPairChunk = 8;
constexpr int kNbrBuf = 16;  // near candidates buffered per brick particle (more -> overflow)

template <int D>
__device__ __forceinline__ void proposal_of(const State& S, int64_t gi, const Box& box, const RoundParams& rp,
                                            double* p) {
    double x0[D];
    load_pos<D>(S, gi, x0);
    propose<D>(box, x0, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[gi]), 0u, p);
}

template <int D>
__global__ void __launch_bounds__(kTileThreads, 3)
    k_phase0_pairs(State S, State T, Box box, const GridParams* __restrict__ gp,
                   const TileParams* __restrict__ tpp, const RoundParams* __restrict__ rpp,
                   const int64_t* __restrict__ cs, const uint32_t* __restrict__ skey,
                   uint8_t* __restrict__ acc, int32_t* __restrict__ nbr, uint8_t* __restrict__ nbr_cnt,
                   int32_t* __restrict__ active, StatsDev* stats) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_rowbase[kMaxRows + 1];
    __shared__ int s_lenA[kMaxRows];
    __shared__ int s_kA[kMaxRows];
    __shared__ int s_A0[kMaxRows];
    __shared__ int s_gA[kMaxRows], s_gB[kMaxRows];
    __shared__ unsigned s_rc0[kMaxRows];  // row cell index (< 2^32 cells)
    __shared__ signed char s_shA[kMaxRows], s_shB[kMaxRows], s_shY[kMaxRows], s_shZ[kMaxRows];
    __shared__ int s_cpre[kMaxRows + 1];
    __shared__ int s_crow[kMaxRows];
    __shared__ int s_total;

    const GridParams& g = *gp;
    const TileParams& tp = *tpp;
    const RoundParams rp = *rpp;
    const int capS = tp.capS, capC = tp.capC, MS = tp.maxseg;
    const int X1 = tp.nst_max[0] + 1;
    const int rows_max = tp.nst_max[1] * tp.nst_max[2];
    float4* srel = reinterpret_cast<float4*>(smem_raw);
    float4* sprel = srel + capS;
    double* sp = reinterpret_cast<double*>(sprel + capS);  // D * capC, brick particles only
    int* sid = reinterpret_cast<int*>(sp + D * capC);
    int* sgi = sid + capS;
    int* coff = sgi + capS;
    short2* srng = reinterpret_cast<short2*>(coff + rows_max * X1);          // MS ranges per thread
    short* wbuf = reinterpret_cast<short*>(srng + kTileThreads * MS);       // kNbrCap per thread
    (void)MS;

    const int dimsv[3] = {g.dims[0], g.dims[1], D == 3 ? g.dims[2] : 1};
    const int dx = dimsv[0], dy = dimsv[1];
    const float margin = tp.margin, extra_f = tp.extra_f;

    for (int64_t t = blockIdx.x; t < tp.ntiles; t += gridDim.x) {
        int tc[3];
        {
            int64_t rest = t;
            tc[0] = static_cast<int>(rest % tp.ax[0].ntile);
            rest /= tp.ax[0].ntile;
            tc[1] = static_cast<int>(rest % tp.ax[1].ntile);
            tc[2] = static_cast<int>(rest / tp.ax[1].ntile);
        }
        int o[3], Be[3], nst[3], sw[3];
        double origin[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const AxisTile& A = tp.ax[a];
            if (a >= D) {
                o[a] = 0; Be[a] = 1; nst[a] = 1; sw[a] = 0; origin[a] = 0.0;
            } else {
                o[a] = tc[a] * A.B;
                Be[a] = min(A.B, dimsv[a] - o[a]);
                sw[a] = A.s;
                nst[a] = Be[a] + 2 * A.s;
                origin[a] = static_cast<double>(o[a]) * g.edge[a];
            }
        }
        const int nrows = nst[1] * nst[2];

        // ---- A. staged rows ----------------------------------------------------------------
        int tot = 0;
        if (threadIdx.x < nrows) {
            const int r = threadIdx.x;
            const int iy = r % nst[1], iz = r / nst[1];
            int gy = o[1] - sw[1] + iy;
            int gz = o[2] - sw[2] + iz;
            signed char shy = 0, shz = 0;  // u < 0 -> -L, u >= dims -> +L (see k_phase0_tiled)
            if (gy < 0) { gy += dy; shy = -1; } else if (gy >= dy) { gy -= dy; shy = 1; }
            if (gz < 0) { gz += dimsv[2]; shz = -1; } else if (gz >= dimsv[2]) { gz -= dimsv[2]; shz = 1; }
            const long long rc0 = (static_cast<long long>(gz) * dy + gy) * dx;
            int A0, A1, B1 = 0;
            signed char shA = 0, shB = 0;
            const int u0 = o[0] - sw[0], u1 = u0 + nst[0];
            if (u0 < 0) { A0 = u0 + dx; A1 = dx; shA = -1; B1 = u1; }
            else if (u1 > dx) { A0 = u0; A1 = dx; B1 = u1 - dx; shB = 1; }
            else { A0 = u0; A1 = u1; }
            const long long gA = cs[rc0 + A0];
            const int lenA = static_cast<int>(cs[rc0 + A1] - gA);
            const long long gB = cs[rc0];
            const int lenB = B1 > 0 ? static_cast<int>(cs[rc0 + B1] - gB) : 0;
            tot = lenA + lenB;
            s_lenA[r] = lenA; s_kA[r] = A1 - A0; s_A0[r] = A0;
            s_gA[r] = static_cast<int>(gA); s_gB[r] = static_cast<int>(gB); s_rc0[r] = static_cast<unsigned>(rc0);
            s_shA[r] = shA; s_shB[r] = shB; s_shY[r] = shy; s_shZ[r] = shz;
        }
        const int rb = block_excl_scan_int(tot, &s_total);
        if (threadIdx.x < nrows) s_rowbase[threadIdx.x] = rb;
        if (threadIdx.x == nrows - 1) s_rowbase[nrows] = rb + tot;
        const int total = s_total;
        __syncthreads();

        // ---- B. local cell offsets -----------------------------------------------------------
        if (total <= capS) {
            for (int idx = threadIdx.x; idx < nrows * (nst[0] + 1); idx += blockDim.x) {
                const int r = idx / (nst[0] + 1), k = idx % (nst[0] + 1);
                int off;
                if (k == nst[0]) off = s_rowbase[r + 1] - s_rowbase[r];
                else if (k < s_kA[r]) off = static_cast<int>(cs[static_cast<long long>(s_rc0[r]) + s_A0[r] + k] - s_gA[r]);
                else off = s_lenA[r] + static_cast<int>(cs[static_cast<long long>(s_rc0[r]) + (k - s_kA[r])] - s_gB[r]);
                coff[r * X1 + k] = s_rowbase[r] + off;
            }
        }
        __syncthreads();

        // ---- C. brick rows and their particle counts -------------------------------------------
        const int ncr = Be[1] * Be[2];
        int ccount = 0;
        if (total <= capS && threadIdx.x < ncr) {
            const int c = threadIdx.x;
            const int r = (sw[2] + c / Be[1]) * nst[1] + (sw[1] + c % Be[1]);
            s_crow[c] = r;
            ccount = coff[r * X1 + sw[0] + Be[0]] - coff[r * X1 + sw[0]];
        }
        const int cpre = block_excl_scan_int(ccount, &s_total);
        if (threadIdx.x < ncr) s_cpre[threadIdx.x] = cpre;
        if (threadIdx.x == ncr - 1) s_cpre[ncr] = cpre + ccount;
        const int nc = s_total;

        if (total > capS || nc > capC) {
            if (threadIdx.x == 0) atomicAdd(&stats->fallback_tiles, 1ull);
            for (int c = 0; c < ncr; ++c) {
                const int gy = o[1] + c % Be[1], gz = o[2] + c / Be[1];
                const long long rc0 = (static_cast<long long>(gz) * dy + gy) * dx;
                const long long b = cs[rc0 + o[0]], e = cs[rc0 + o[0] + Be[0]];
                for (long long i = b + threadIdx.x; i < e; i += blockDim.x) {
                    const bool rej = phase0_global<D>(i, S, T, box, g, rp, cs, skey, acc, nbr, nbr_cnt);
                    if (rej) {
                        const unsigned long long pos = atomicAdd(&stats->active_count, 1ull);
                        active[pos] = static_cast<int32_t>(i);
                    }
                }
            }
            __syncthreads();
            continue;
        }
        __syncthreads();

        // ---- D. stage every particle + its attempt-0 proposal (uniform pass) ---------------------
        for (int q = threadIdx.x; q < total; q += blockDim.x) {
            const int r = upper_index(s_rowbase, nrows, q);
            const int e = q - s_rowbase[r];
            const int lenA = s_lenA[r];
            const long long gsrc = e < lenA ? s_gA[r] + e : s_gB[r] + (e - lenA);
            double x0[D], p[D];
            load_pos<D>(S, gsrc, x0);
            const double sh[3] = {(e < lenA ? s_shA[r] : s_shB[r]) * box.L[0], s_shY[r] * box.L[1],
                                  s_shZ[r] * box.L[2]};
            float rel[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int a = 0; a < D; ++a) rel[a] = static_cast<float>(x0[a] + sh[a] - origin[a]);
            const float4 rq = make_float4(rel[0], rel[1], rel[2], static_cast<float>(S.r[gsrc]));
            srel[q] = rq;
            sid[q] = S.id[gsrc];
            sgi[q] = static_cast<int>(gsrc);
            propose<D>(box, x0, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[gsrc]), 0u, p);
            sprel[q] = rel_of_proposal<D>(rq, x0, p, box);
            // brick particle: keep its fp64 proposal, indexed by brick order c
            const int iy = r % nst[1], iz = r / nst[1];
            const int jy = iy - sw[1], jz = iz - sw[2];
            if (jy >= 0 && jy < Be[1] && jz >= 0 && jz < Be[2]) {
                const int qlo = coff[r * X1 + sw[0]], qhi = coff[r * X1 + sw[0] + Be[0]];
                if (q >= qlo && q < qhi) {
                    const int c = s_cpre[jz * Be[1] + jy] + (q - qlo);
#pragma unroll
                    for (int a = 0; a < D; ++a) sp[a * capC + c] = p[a];
                }
            }
        }
        __syncthreads();

        // ---- E. attempt 0: thread per brick particle over its pruned candidate ranges ------------
        // The candidate loop only runs the fp32 near prefilter and queues near candidates
        // in a per-thread shared buffer; the conflict tests run afterwards in a second,
        // short loop, so the near-pair work does not diverge inside the candidate loop.
        for (int cb = 0; cb < nc; cb += kTileThreads) {
            const int c = cb + threadIdx.x;
            short* wb = wbuf + threadIdx.x * kNbrBuf;
            bool rejected = false;
            int gi = -1;
            if (c < nc) {
                const int jrow = upper_index(s_cpre, ncr, c);
                const int r = s_crow[jrow];
                const int q = coff[r * X1 + sw[0]] + (c - s_cpre[jrow]);
                const float4 me = srel[q];
                gi = sgi[q];
                const int iy = r % nst[1], iz = r / nst[1];
                const int kx = static_cast<int>(skey[gi] % static_cast<uint32_t>(dx)) - (o[0] - sw[0]);
                const float cutm = __fadd_rn(__fadd_rn(__fadd_rn(me.w, tp.rmax_f), extra_f), __fmul_rn(2.f, margin));
                auto lohi = [&](float v, int kc, int s, float e, int& lo, int& hi) {
                    lo = max(kc - s, static_cast<int>(floorf(__fdiv_rn(__fsub_rn(v, cutm), e))) + s);
                    hi = min(kc + s, static_cast<int>(ceilf(__fdiv_rn(__fadd_rn(v, cutm), e))) - 1 + s);
                };
                int xlo, xhi, ylo, yhi, zlo = 0, zhi = 0;
                lohi(me.x, kx, sw[0], tp.edge_f[0], xlo, xhi);
                lohi(me.y, iy, sw[1], tp.edge_f[1], ylo, yhi);
                if (D == 3) lohi(me.z, iz, sw[2], tp.edge_f[2], zlo, zhi);
                const float cut2 = __fmul_rn(__fmul_rn(cutm, cutm), 1.00001f);
                const float lim0 = __fadd_rn(__fadd_rn(me.w, extra_f), margin);  // + r_j
                int nn = 0;
                bool conflict = false;
                const int idq = sid[q];
                const float4 mp = sprel[q];
                // conflict tests of brick particle c against staged candidate q2
                auto test = [&](int q2) {
                    if (sid[q2] == idq) return;
                    const float4 cq = srel[q2];
                    const float lov = __fadd_rn(__fadd_rn(me.w, cq.w), margin);
                    const float lin = __fsub_rn(__fsub_rn(__fadd_rn(me.w, cq.w), margin), margin);
                    const float dx2 = d2_rel<D, true>(mp, cq, nullptr, nullptr, nullptr);
                    const float dp2 = d2_rel<D, true>(mp, sprel[q2], nullptr, nullptr, nullptr);
                    bool cf = inside_f(dx2, lin) || inside_f(dp2, lin);
                    const bool band_x = !cf && !clear_f(dx2, lov);
                    const bool band_p = !cf && !clear_f(dp2, lov);
                    if (band_x || band_p) {  // rounding band around contact: exact fp64
                        double pi[D], xj[D];
                        proposal_of<D>(S, gi, box, rp, pi);
                        const int64_t gj = sgi[q2];
                        const double ri = S.r[gi], rj = S.r[gj];
                        load_pos<D>(S, gj, xj);
                        if (band_x && sphere_overlap<D>(box, pi, ri, xj, rj)) cf = true;
                        if (!cf && band_p) {
                            double pj[D];
                            propose<D>(box, xj, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[gj]), 0u, pj);
                            if (sphere_overlap<D>(box, pi, ri, pj, rj)) cf = true;
                        }
                    }
                    conflict = conflict || cf;
                };
                // pruned stencil -> contiguous candidate ranges; each row's x range is cut to
                // the chord of the (margin-inflated) cutoff sphere at the row's distance
                short2* rg = srng + threadIdx.x * MS;
                int nr = 0;
                for (int iz2 = zlo; iz2 <= zhi; ++iz2) {
                    float dzd = 0.f;
                    if (D == 3) {
                        const float zb = (iz2 - sw[2]) * tp.edge_f[2];
                        dzd = fmaxf(0.f, fmaxf(zb - me.z, me.z - (zb + tp.edge_f[2])));
                    }
                    for (int iy2 = ylo; iy2 <= yhi; ++iy2) {
                        const float yb = (iy2 - sw[1]) * tp.edge_f[1];
                        const float dyd = fmaxf(0.f, fmaxf(yb - me.y, me.y - (yb + tp.edge_f[1])));
                        const float dyz2 = __fmaf_rn(dyd, dyd, __fmul_rn(dzd, dzd));
                        if (dyz2 > cut2) continue;
                        const float xh = __fadd_rn(__fsqrt_rn(__fsub_rn(cut2, dyz2)), margin);
                        const int xl = max(xlo, static_cast<int>(floorf(__fdiv_rn(__fsub_rn(me.x, xh), tp.edge_f[0]))) + sw[0]);
                        const int xr = min(xhi, static_cast<int>(ceilf(__fdiv_rn(__fadd_rn(me.x, xh), tp.edge_f[0]))) - 1 + sw[0]);
                        const int* rowoff = coff + (iz2 * nst[1] + iy2) * X1;
                        const int b = rowoff[xl], e = rowoff[xr + 1];
                        if (e > b) rg[nr++] = make_short2(static_cast<short>(b), static_cast<short>(e));
                    }
                }
                // one flat loop over every candidate of every range
                if (nr > 0) {
                    int k = 0;
                    short2 cur = rg[0];
                    int q2 = cur.x, e = cur.y;
                    while (true) {
                        const float4 cq = srel[q2];
                        if (!clear_f(d2_rel<D, true>(me, cq, nullptr, nullptr, nullptr), __fadd_rn(lim0, cq.w)) &&
                            q2 != q) {
                            if (nn < kNbrBuf) wb[nn] = static_cast<short>(q2);
                            else test(q2);  // buffer full (rare): test inline
                            ++nn;
                        }
                        if (++q2 == e) {
                            if (++k == nr) break;
                            cur = rg[k];
                            q2 = cur.x;
                            e = cur.y;
                        }
                    }
                }
                const int nb = min(nn, kNbrBuf);
                for (int k = 0; k < nb; ++k) test(wb[k]);
                const bool ok = !conflict;
#pragma unroll
                for (int a = 0; a < D; ++a) T.x[a][gi] = ok ? sp[a * capC + c] : S.x[a][gi];
                T.r[gi] = S.r[gi];
                T.id[gi] = idq;
                T.slot[gi] = S.slot[gi];
                acc[gi] = ok ? 0 : kNotAccepted;
                // more near candidates than the buffer holds: the list is marked overflowed
                // and later attempts rescan the grid for this particle
                nbr_cnt[gi] = nn > kNbrBuf ? kOverflow : static_cast<uint8_t>(nn);
                // only rejected particles need their near list (later attempts, reduction)
                if (!ok && nn <= kNbrBuf) {
                    int32_t* my = nbr + static_cast<int64_t>(gi) * kNbrCap;
                    for (int k = 0; k < nn; ++k) my[k] = sgi[wb[k]];
                }
                rejected = !ok;
            }
            push_active(rejected, gi, active, stats);
        }
        __syncthreads();
    }
}

__global__ void k_set_tiles(TileParams* tp, TileParams v) { *tp = v; }

}  // namespace srmb
