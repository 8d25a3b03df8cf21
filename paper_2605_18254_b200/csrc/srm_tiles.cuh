// srm_tiles.cuh -- attempt 0 of the parallel migrate as a shared-memory brick kernel.
//
// One CTA owns a brick of Bx x By x Bz cells of the round's grid.  It stages the brick
// plus a halo of s cells per side (s = near-search half width) into shared memory:
// the staged cells are (By+2s)(Bz+2s) contiguous x-runs of the cell-sorted SoA, so the
// copy is a set of coalesced row segments.  While staging, every staged particle's
// attempt-0 proposal (Philox + unit vector + wrap) is computed once.  Then each thread
// takes one brick particle and scans its neighbourhood from shared memory:
//   1. fp32 prefilter on tile-relative coordinates (no min-image inside a brick), with
//      an absolute margin that covers the fp32 rounding, so it can only pass MORE pairs;
//   2. the exact fp64 near test decides near-list membership;
//   3. the exact reference predicate (shape.hpp:508-511) on x0_j and p_j decides the
//      attempt.
// Decisions are therefore identical to phase0_global's (and the oracle's).  A brick
// whose staged count exceeds the shared-memory capacity falls back to phase0_global.
#pragma once

#include "srm_kernels.cuh"

namespace srmb {

constexpr int kTileThreads = 256;
constexpr int kMaxRows = 256;
constexpr int kTileSmemMax = 160 * 1024;  // dynamic shared memory per brick CTA, upper bound

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
    int32_t cap;         // staged particles per brick (shared-memory capacity)
    int32_t nst_max[3];  // staged cells per axis, upper bound
    float margin;        // absolute fp32 prefilter margin
    float extra_f;       // near-cut extra (2 c_m) in fp32
    int32_t enabled;
    int32_t smem_bytes;
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

template <int D>
__global__ void __launch_bounds__(kTileThreads, 2)
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

    const GridParams g = *gp;
    const TileParams tp = *tpp;
    const RoundParams rp = *rpp;
    const int cap = tp.cap;
    double* sx0 = reinterpret_cast<double*>(smem_raw);
    double* sr = sx0 + D * cap;
    double* sp = sr + cap;
    float4* srel = reinterpret_cast<float4*>(sp + D * cap);
    int* sid = reinterpret_cast<int*>(srel + cap);
    int* sgi = sid + cap;
    int* coff = sgi + cap;
    const int X1 = tp.nst_max[0] + 1;
    const int dimsv[3] = {g.dims[0], g.dims[1], D == 3 ? g.dims[2] : 1};
    const int dx = dimsv[0], dy = dimsv[1];
    const float Lf[3] = {static_cast<float>(box.L[0]), static_cast<float>(box.L[1]), static_cast<float>(box.L[2])};
    const float Hf[3] = {0.5f * Lf[0], 0.5f * Lf[1], 0.5f * Lf[2]};

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

        // ---- 1. staged rows: global row, x chunks, shifts ----------------------------
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
        __syncthreads();
        const int total = s_total;

        if (total > cap) {
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

        // ---- 2. local cell offsets -------------------------------------------------------
        for (int idx = threadIdx.x; idx < nrows * (nst[0] + 1); idx += blockDim.x) {
            const int r = idx / (nst[0] + 1), k = idx % (nst[0] + 1);
            int off;
            if (k == nst[0]) off = s_rowbase[r + 1] - s_rowbase[r];
            else if (k < s_kA[r]) off = static_cast<int>(cs[s_rc0[r] + s_A0[r] + k] - s_gA[r]);
            else off = s_lenA[r] + static_cast<int>(cs[s_rc0[r] + (k - s_kA[r])] - s_gB[r]);
            coff[r * X1 + k] = s_rowbase[r] + off;
        }

        // ---- 3. stage particles + their attempt-0 proposals (warp per row) ----------------
        {
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            for (int r = wid; r < nrows; r += kTileThreads / 32) {
                const int base = s_rowbase[r], len = s_rowbase[r + 1] - base, lenA = s_lenA[r];
                const double shy = s_shY[r] * box.L[1], shz = s_shZ[r] * box.L[2];
                for (int e = lane; e < len; e += 32) {
                    const long long gsrc = e < lenA ? s_gA[r] + e : s_gB[r] + (e - lenA);
                    const int q = base + e;
                    double x0[D];
                    load_pos<D>(S, gsrc, x0);
                    const double shx = (e < lenA ? s_shA[r] : s_shB[r]) * box.L[0];
                    const double sh[3] = {shx, shy, shz};
                    float rel[3] = {0.f, 0.f, 0.f};
#pragma unroll
                    for (int a = 0; a < D; ++a) {
                        sx0[a * cap + q] = x0[a];
                        rel[a] = static_cast<float>(x0[a] + sh[a] - origin[a]);
                    }
                    const double rr = S.r[gsrc];
                    sr[q] = rr;
                    srel[q] = make_float4(rel[0], rel[1], rel[2], static_cast<float>(rr));
                    sid[q] = S.id[gsrc];
                    sgi[q] = static_cast<int>(gsrc);
                    double p[D];
                    propose<D>(box, x0, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[gsrc]), 0u, p);
#pragma unroll
                    for (int a = 0; a < D; ++a) sp[a * cap + q] = p[a];
                }
            }
        }

        // ---- 4. brick rows and their particle counts ---------------------------------------
        const int ncr = Be[1] * Be[2];
        int ccount = 0;
        __syncthreads();
        if (threadIdx.x < ncr) {
            const int c = threadIdx.x;
            const int r = (c0[2] + c / Be[1]) * nst[1] + (c0[1] + c % Be[1]);
            s_crow[c] = r;
            ccount = coff[r * X1 + c0[0] + Be[0]] - coff[r * X1 + c0[0]];
        }
        const int cpre = block_excl_scan_int(ccount, &s_total);
        if (threadIdx.x < ncr) s_cpre[threadIdx.x] = cpre;
        __syncthreads();
        const int nc = s_total;
        if (threadIdx.x == 0) s_cpre[ncr] = nc;
        __syncthreads();

        // ---- 5. attempt 0 for the brick particles ----------------------------------------
        const bool mi[3] = {tp.ax[0].full != 0, tp.ax[1].full != 0, tp.ax[2].full != 0};
        for (int cbase = 0; cbase < nc; cbase += blockDim.x) {
            const int c = cbase + threadIdx.x;
            bool rejected = false;
            int gi = -1;
            if (c < nc) {
                int lo = 0, hi = ncr - 1;  // largest j with s_cpre[j] <= c
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_cpre[mid] <= c) lo = mid; else hi = mid - 1;
                }
                const int r = s_crow[lo];
                const int q = coff[r * X1 + c0[0]] + (c - s_cpre[lo]);
                gi = sgi[q];
                const int iy = r % nst[1], iz = r / nst[1];
                const int cx = static_cast<int>(skey[gi] % static_cast<uint32_t>(dx));
                const int kx = tp.ax[0].full ? cx : cx - (o[0] - tp.ax[0].s);
                double xi[D], pi[D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    xi[a] = sx0[a * cap + q];
                    pi[a] = sp[a * cap + q];
                }
                const double ri = sr[q];
                const int idi = sid[q];
                const float4 me = srel[q];
                bool ok = true, overflow = false;
                int nn = 0;
                int32_t* my = nbr + static_cast<int64_t>(gi) * kNbrCap;

                auto scan_range = [&](int b, int e) {
                    for (int q2 = b; q2 < e; ++q2) {
                        if (q2 == q) continue;
                        const float4 cq = srel[q2];
                        float ddx = cq.x - me.x, ddy = cq.y - me.y, ddz = D == 3 ? cq.z - me.z : 0.f;
                        if (mi[0]) { if (ddx > Hf[0]) ddx -= Lf[0]; else if (ddx < -Hf[0]) ddx += Lf[0]; }
                        if (mi[1]) { if (ddy > Hf[1]) ddy -= Lf[1]; else if (ddy < -Hf[1]) ddy += Lf[1]; }
                        if (D == 3 && mi[2]) { if (ddz > Hf[2]) ddz -= Lf[2]; else if (ddz < -Hf[2]) ddz += Lf[2]; }
                        const float d2f = __fmaf_rn(ddx, ddx, __fmaf_rn(ddy, ddy, __fmul_rn(ddz, ddz)));
                        const float lim = __fadd_rn(__fadd_rn(__fadd_rn(me.w, cq.w), tp.extra_f), tp.margin);
                        if (d2f > __fmul_rn(__fmul_rn(lim, lim), 1.00001f)) continue;
                        double xj[D];
#pragma unroll
                        for (int a = 0; a < D; ++a) xj[a] = sx0[a * cap + q2];
                        const double rj = sr[q2];
                        if (dist2<D>(box, xi, xj) > near_cut(ri, rj, g.extra)) continue;
                        if (nn < kNbrCap) my[nn++] = sgi[q2];
                        else overflow = true;
                        if (!ok || sid[q2] == idi) continue;
                        if (sphere_overlap<D>(box, pi, ri, xj, rj)) { ok = false; continue; }
                        double pj[D];
#pragma unroll
                        for (int a = 0; a < D; ++a) pj[a] = sp[a * cap + q2];
                        if (sphere_overlap<D>(box, pi, ri, pj, rj)) ok = false;
                    }
                };
                auto scan_row = [&](int r2) {
                    const int bse = r2 * X1;
                    const AxisTile& A = tp.ax[0];
                    if (A.all) {
                        scan_range(coff[bse], coff[bse + nst[0]]);
                    } else if (A.full) {
                        const int lo2 = kx - A.s, hi2 = kx + A.s;
                        if (lo2 < 0) {
                            scan_range(coff[bse + lo2 + dx], coff[bse + dx]);
                            scan_range(coff[bse], coff[bse + hi2 + 1]);
                        } else if (hi2 >= dx) {
                            scan_range(coff[bse + lo2], coff[bse + dx]);
                            scan_range(coff[bse], coff[bse + hi2 - dx + 1]);
                        } else {
                            scan_range(coff[bse + lo2], coff[bse + hi2 + 1]);
                        }
                    } else {
                        scan_range(coff[bse + kx - A.s], coff[bse + kx + A.s + 1]);
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

#pragma unroll
                for (int a = 0; a < D; ++a) T.x[a][gi] = ok ? pi[a] : xi[a];
                T.r[gi] = ri;
                T.id[gi] = idi;
                T.slot[gi] = S.slot[gi];
                acc[gi] = ok ? 0 : kNotAccepted;
                nbr_cnt[gi] = overflow ? kOverflow : static_cast<uint8_t>(nn);
                rejected = !ok;
            }
            push_active(rejected, gi, active, stats);
        }
        __syncthreads();
    }
}

__global__ void k_set_tiles(TileParams* tp, TileParams v) { *tp = v; }

}  // namespace srmb
