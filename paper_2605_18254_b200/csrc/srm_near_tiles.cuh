// srm_near_tiles.cuh -- the shared-memory near-list brick kernel, included once per brick
// shape (srm_kernels.cuh: namespace tiles = the sparse grids' 16 x 8 x 4 bricks, namespace
// ctiles = 4 x 4 x 4 bricks with a large staging capacity for crowded grids: polydisperse
// and platelet states of 2-12 particles per cell).  Parameters: NT_X, NT_Y, NT_Z (brick
// cells), NT_CAP (staged particles), NT_THREADS, NT_MINB (CTAs per SM), NT_KIND
// (GridParams::near_kind that selects it).  No include guard: included twice.

// Near lists through shared memory (3D, a one-cell stencil on every axis).  A CTA takes a
// brick of kTX x kTY x kTZ cells and stages the fp32 records, sorted indices and ids of
// the brick and its full one-cell halo (the particles of a row of halo cells are one to
// three contiguous runs of the sorted state: the periodic images at x = -1 and x >= dims),
// shifted by +-L on the way in so that pair distances are plain differences.  Every interior particle is then screened against the nine contiguous
// shared-memory ranges of its 3x3x3 stencil and writes its own row (one sector, no
// atomics).  Same screen as near_candidates (cutoff, margin, factor), so the lists hold
// the same pairs as k_near_lists.  A brick whose halo holds more than kTileCap particles
// takes near_full_particle.
#undef NT_TAG
#if NT_FUSED
#define NT_TAG(row9) ((row9) << 12)  // the stencil row of a hit, beside its staged slot
#else
#define NT_TAG(row9) 0
#endif
constexpr int kTX = NT_X, kTY = NT_Y, kTZ = NT_Z;  // brick (cells)
constexpr int kHX = kTX + 2, kHY = kTY + 2, kHZ = kTZ + 2;
constexpr int kHCells = kHX * kHY * kHZ;
constexpr int kHRows = kHY * kHZ;
constexpr int kTileCap = NT_CAP;  // staged particles
constexpr int kTileThreads = NT_THREADS;
constexpr int kCellsPerThread = (kHCells + kTileThreads - 1) / kTileThreads;
// per-thread hit buffer (uint16 entries): screens 0 / 1 keep kNearCap + 1 hit slots; screen 2
// keeps kPairCap + 1 pair records and, behind them, the kNearCap hit slots it resolves them to
constexpr int kPairCap = 8;
constexpr int kHitRows = NT_SCREEN == 2 ? kPairCap + 1 + kNearCap : kNearCap + 1;
constexpr size_t kTileSmem = kTileCap * (16 + 4) + (kHCells + 1) * 4 +
                             (kHCells * 4 > kTileThreads * kHitRows * 2 ? kHCells * 4 : kTileThreads * kHitRows * 2);
static_assert(NT_SCREEN != 2 || kTileCap <= 4096, "pair records: 11 bits of pair index + the stencil row");
static_assert(kTileCap <= 65536, "16-bit hit slots");
static_assert(kHRows <= kTileThreads && kHRows <= 64, "a thread per halo row; 6-step row search");
static_assert(kTY * kTZ <= 32 && kTX <= 16, "one warp scans the interior rows; 4-step cell search");

__global__ void __launch_bounds__(kTileThreads, NT_MINB) k_near_tiles(State S, const GridParams* __restrict__ gp,
                                                             const cell_t* __restrict__ cs,
                                                             const uint32_t* __restrict__ skey,
                                                             int32_t* __restrict__ nbr, NearPool pool,
                                                             StatsDev* stats
#if NT_HALF
                                                             , int2* __restrict__ rev, int64_t rev_cap,
                                                             int32_t* __restrict__ ovf
#endif
#if NT_FUSED
                                                             , Box box, const RoundParams* __restrict__ rpp,
                                                             double4* __restrict__ rec_new,
                                                             uint8_t* __restrict__ dflag, uint8_t* __restrict__ acc
#endif
                                                             ) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // shifted fp32 records of staged slots 2p, 2p + 1, interleaved for f32x2 arithmetic:
    // pxy[p] = (x0, x1, y0, y1), pzw[p] = (z0, z1, w0, w1)
    float4* pxy = reinterpret_cast<float4*>(smem_raw);             // [kTileCap / 2]
    float4* pzw = pxy + kTileCap / 2;                               // [kTileCap / 2]
    int32_t* pj = reinterpret_cast<int32_t*>(pzw + kTileCap / 2);  // [kTileCap] sorted index of a slot
    int32_t* hoff = pj + kTileCap;                                  // [kHCells + 1] staged offset of a cell
    int32_t* hsrc = hoff + kHCells + 1;                             // [kHCells] first sorted index of a cell
    uint16_t* lst = reinterpret_cast<uint16_t*>(hsrc);              // [kNearCap + 1][kTileThreads] hit slots
                                                                    // (aliases hsrc: used after the staging)
#if NT_HALF
    // half stencil: an interior particle screens the cells AFTER its own in
    // (z, y, x) order, the later slots of its cell, and whatever part of the stencil lies in
    // the brick's halo; a hit on another interior particle j is j's hit on i as well and goes
    // to the reverse list (j, i), merged into j's row by k_near_merge
    constexpr int kRevCap = 320;
    __shared__ int2 s_rev[kRevCap];
    __shared__ int s_nrev;
    __shared__ unsigned long long s_revbase;
    if (threadIdx.x == 0) s_nrev = 0;
#endif
    __shared__ int wsum[kTileThreads / 32];
    __shared__ int rowoff[kTY * kTZ + 1];
    __shared__ RowMap rmap[kHRows];
    const GridParams& g = *gp;
    if (g.near_kind != NT_KIND || static_cast<int>(blockIdx.x) >= g.ntiles) return;  // (graph launches: upper bounds)
#if NT_FUSED
    if (!g.resolve) return;
    __shared__ uint8_t hcls[kHCells];  // colour class of a halo cell (the sweep order between cells)
    __shared__ RoundParams rp;
    if (threadIdx.x == 0) rp = *rpp;
    static_assert(kTileCap <= 4096, "hit slots carry the stencil row in bits 12-15");
#else
    if (NT_KIND == 0 && g.resolve) return;  // the fused variant (rtiles) has this grid
#endif
    const int dx = g.dims[0], dy = g.dims[1], dz = g.dims[2];
    const int ntx = (dx + kTX - 1) / kTX, nty = (dy + kTY - 1) / kTY;
    const int tx = blockIdx.x % ntx, ty = (blockIdx.x / ntx) % nty, tz = blockIdx.x / (ntx * nty);
    const int x0 = tx * kTX, y0 = ty * kTY, z0 = tz * kTZ;
    const int wx = min(kTX, dx - x0), wy = min(kTY, dy - y0), wz = min(kTZ, dz - z0);  // interior extent
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // 1. counts of the halo cells (cells outside the halo of a partial brick: 0); a
    //    thread owns kCellsPerThread consecutive cells
    int cnts[kCellsPerThread];
    int local = 0;
#pragma unroll
    for (int k = 0; k < kCellsPerThread; ++k) {
        const int hc = threadIdx.x * kCellsPerThread + k;
        int c = 0;
        if (hc < kHCells) {
            const int hx = hc % kHX, hy = (hc / kHX) % kHY, hz = hc / (kHX * kHY);
            if (hx <= wx + 1 && hy <= wy + 1 && hz <= wz + 1) {
                int X = x0 - 1 + hx, Y = y0 - 1 + hy, Z = z0 - 1 + hz;
                X = X < 0 ? X + dx : (X >= dx ? X - dx : X);
                Y = Y < 0 ? Y + dy : (Y >= dy ? Y - dy : Y);
                Z = Z < 0 ? Z + dz : (Z >= dz ? Z - dz : Z);
                const int64_t cell = (static_cast<int64_t>(Z) * dy + Y) * dx + X;
                const int64_t b = cs[cell];
                c = static_cast<int>(cs[cell + 1] - b);
                hsrc[hc] = static_cast<int32_t>(b);
#if NT_FUSED
                hcls[hc] = static_cast<uint8_t>(colour1(g, 0, X) + g.col_n[0] * (colour1(g, 1, Y) + g.col_n[1] * colour1(g, 2, Z)));
#endif
            }
        }
        cnts[k] = c;
        local += c;
    }
    // 2. exclusive scan over the halo cells
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int wbase = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kTileThreads / 32; ++w) {
        if (w < wid) wbase += wsum[w];
        total += wsum[w];
    }
    {
        int off = wbase + incl - local;
#pragma unroll
        for (int k = 0; k < kCellsPerThread; ++k) {
            const int hc = threadIdx.x * kCellsPerThread + k;
            if (hc < kHCells) hoff[hc] = off;
            off += cnts[k];
        }
        if (threadIdx.x == 0) hoff[kHCells] = total;
    }
    __syncthreads();
    if (total > kTileCap) {  // crowded brick: the per-particle path over global memory
        for (int r = 0; r < wy * wz; ++r) {
            const int Y = y0 + r % wy, Z = z0 + r / wy;
            const int64_t row = (static_cast<int64_t>(Z) * dy + Y) * dx;
            const int64_t b = cs[row + x0], e = cs[row + x0 + wx];
            for (int64_t q = b + threadIdx.x; q < e; q += blockDim.x) {
                near_full_particle<3>(q, S, g, cs, skey, nbr, pool, stats);
#if NT_FUSED
                {  // pending, with its first trial drawn (the row carries no precedence mask)
                    const double4 me = S.rec[q];
                    const double xi[3] = {me.x, me.y, me.z};
                    double p[3];
                    propose<3>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[q]), 0u, p);
                    rec_new[q] = make_double4(p[0], p[1], p[2], me.w);
                    dflag[q] = kUndecided;
                }
#endif
            }
        }
        return;
    }
    // 3. stage the halo.  Along x a row of halo cells holds up to three runs of
    //    consecutive sorted indices: [0, xa) the image of the last column (shift -L),
    //    [xa, xc) the body, [xc, kHX) the image of the first columns (+L).  A table per
    //    row (a thread per row) maps a staged slot to its sorted index; then every thread
    //    copies a strided set of slots, all loads in flight before any store.
    if (threadIdx.x < kHRows) {
        const int r = threadIdx.x, hy = r % kHY, hz = r / kHY;
        const int xa = x0 == 0 ? 1 : 0, xc = min(kHX, dx - x0 + 1);
        const int h0 = r * kHX;
        RowMap m;
        m.ka = hoff[h0 + xa];
        m.kc = hoff[h0 + xc];
        const bool used = hy <= wy + 1 && hz <= wz + 1;
        m.sa = used && xa ? hsrc[h0] - hoff[h0] : 0;
        m.sb = used && xa < kHX ? hsrc[h0 + xa] - m.ka : 0;
        m.sc = used && xc < kHX ? hsrc[h0 + xc] - m.kc : 0;
        const int Y = y0 - 1 + hy, Z = z0 - 1 + hz;
        m.sy = Y < 0 ? -g.L_f[1] : (Y >= dy ? g.L_f[1] : 0.f);
        m.sz = Z < 0 ? -g.L_f[2] : (Z >= dz ? g.L_f[2] : 0.f);
        rmap[r] = m;
    }
    __syncthreads();
    bool same_r = true;  // every staged radius equals the grid's largest: monodisperse brick
    for (int k0 = 0; k0 < total; k0 += 4 * kTileThreads) {
        float4 v[4];
        int32_t src[4];
        float sxf[4], syf[4], szf[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + threadIdx.x + u * kTileThreads;
            if (k < total) {
                int r = 0;  // the last row whose first slot is <= k
#pragma unroll
                for (int step = 32; step > 0; step >>= 1)
                    if (r + step < kHRows && hoff[(r + step) * kHX] <= k) r += step;
                const RowMap& m = rmap[r];
                src[u] = static_cast<int32_t>(k + (k < m.ka ? m.sa : (k < m.kc ? m.sb : m.sc)));
                SRM_CHK(src[u] >= 0 && src[u] < g.n_state, 101);
                sxf[u] = k < m.ka ? -g.L_f[0] : (k < m.kc ? 0.f : g.L_f[0]);
                syf[u] = m.sy;
                szf[u] = m.sz;
                v[u] = S.xf[src[u]];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = k0 + threadIdx.x + u * kTileThreads;
            if (k < total) {
                float* a = reinterpret_cast<float*>(pxy + (k >> 1)) + (k & 1);
                float* b = reinterpret_cast<float*>(pzw + (k >> 1)) + (k & 1);
                a[0] = __fadd_rn(v[u].x, sxf[u]);
                a[2] = __fadd_rn(v[u].y, syf[u]);
                b[0] = __fadd_rn(v[u].z, szf[u]);
                b[2] = v[u].w;
                pj[k] = src[u];
                same_r = same_r && v[u].w == g.rmax_f;
            }
        }
    }
    // interior rows (hy in [1, wy], hz in [1, wz]) hold contiguous particles
    if (wid == 0) {
        const int nr = wy * wz;  // <= 32
        int c = 0;
        if (lane < nr) {
            const int h0 = ((1 + lane / wy) * kHY + 1 + lane % wy) * kHX + 1;
            c = hoff[h0 + wx] - hoff[h0];
        }
        int in = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, in, o);
            if (lane >= o) in += t;
        }
        if (lane < nr) rowoff[lane] = in - c;
        if (lane == nr - 1) rowoff[nr] = in;
    }
    const bool mono = __syncthreads_and(same_r) != 0;
    // 4. screen every interior particle against its 3x3x3 stencil in shared memory
    const int nr = wy * wz;
    const int nint = rowoff[nr];
    for (int f = threadIdx.x; f < nint; f += blockDim.x) {
        int r = 0;  // the last interior row whose offset is <= f
#pragma unroll
        for (int step = 16; step > 0; step >>= 1)
            if (r + step < nr && rowoff[r + step] <= f) r += step;
        const int rb = ((1 + r / wy) * kHY + 1 + r % wy) * kHX;
        const int i = hoff[rb + 1] + (f - rowoff[r]);
        int hx = 1;  // the cell of i in its row: the last x with hoff <= i
#pragma unroll
        for (int step = 8; step > 0; step >>= 1)
            if (hx + step <= wx && hoff[rb + hx + step] <= i) hx += step;
        const int hc = rb + hx;
        SRM_CHK(i >= 0 && i < total && hc > kHX * kHY && hc < kHCells - kHX * kHY, 102);
        const float mx = reinterpret_cast<const float*>(pxy + (i >> 1))[i & 1];
        const float my = reinterpret_cast<const float*>(pxy + (i >> 1))[2 + (i & 1)];
        const float mz = reinterpret_cast<const float*>(pzw + (i >> 1))[i & 1];
        const float mw = reinterpret_cast<const float*>(pzw + (i >> 1))[2 + (i & 1)];
        const int32_t qi = pj[i];
        const float base = __fadd_rn(__fadd_rn(mw, g.extra_f), g.margin_f);  // + r_j
        const float2 nmx = make_float2(-mx, -mx), nmy = make_float2(-my, -my), nmz = make_float2(-mz, -mz);
        const float2 base2 = make_float2(base, base), fac2 = make_float2(1.00001f, 1.00001f);
        const float limm = __fadd_rn(g.rmax_f, base);  // (monodisperse bricks: r_j = rmax)
        const float l2m = __fmul_rn(__fmul_rn(limm, limm), 1.00001f);
        uint16_t* ql = lst + threadIdx.x;
        int nn = 0;
#if NT_SCREEN == 0 || NT_SCREEN == 2
        // hits are rare per lane but common per warp: record the hit slots branch-free (a
        // store to the current list slot every test, the count advances on a hit; slot
        // kNearCap absorbs the overflow), resolve them after the scan
        int at = 0;
#else
        // the screen of a range sets a bit per hit in a register mask (16 slot pairs per
        // mask); the few hits are recorded after each chunk
        auto record = [&](int k) {
            if (nn < kNearCap) ql[nn * kTileThreads] = static_cast<uint16_t>(k);
            ++nn;
        };
#endif
#if NT_HALF
        {
            const int hy = 1 + r % wy, hz = 1 + r / wy;
            // slots [kb, ke) two at a time; hits carry the stencil row beside the slot
            auto scan = [&](int kb, int ke, int tag) {
                const int kbt = kb + tag, ket = ke + tag, it = i + tag;
                int kt = (kb & ~1) + tag;
                for (int p = kb >> 1; 2 * p < ke; ++p, kt += 2) {
                    const float4 A = pxy[p], B = pzw[p];
                    const float2 ex = __fadd2_rn(make_float2(A.x, A.y), nmx);
                    const float2 ey = __fadd2_rn(make_float2(A.z, A.w), nmy);
                    const float2 ez = __fadd2_rn(make_float2(B.x, B.y), nmz);
                    const float2 d2 = __ffma2_rn(ex, ex, __ffma2_rn(ey, ey, __fmul2_rn(ez, ez)));
                    const float2 lim = __fadd2_rn(make_float2(B.z, B.w), base2);
                    const float2 l2 = __fmul2_rn(__fmul2_rn(lim, lim), fac2);
                    ql[at * kTileThreads] = static_cast<uint16_t>(kt);
                    nn += (d2.x <= l2.x && kt >= kbt && kt != it) ? 1 : 0;
                    at = min(nn, kNearCap);
                    ql[at * kTileThreads] = static_cast<uint16_t>(kt + 1);
                    nn += (d2.y <= l2.y && kt + 1 < ket && kt + 1 != it) ? 1 : 0;
                    at = min(nn, kNearCap);
                }
            };
#pragma unroll 1
            for (int row9 = 0; row9 < 9; ++row9) {
                const int ddy = row9 % 3 - 1, ddz = row9 / 3 - 1;
                const int c = hc + ddy * kHX + ddz * kHX * kHY;
                const int tag = row9 << 12;
                SRM_CHK(c >= 1 && c + 2 <= kHCells, 103);
                if (row9 > 4) {  // a row after this one: all three cells
                    scan(hoff[c - 1], hoff[c + 2], tag);
                } else if (row9 == 4) {  // the particle's row: the later slots of its cell and
                                         // the next cell; the previous cell when it is halo
                    scan(i + 1, hoff[c + 2], tag);
                    if (hx == 1) scan(hoff[c - 1], hoff[c], tag);
                } else if (hy + ddy < 1 || hy + ddy > wy || hz + ddz < 1) {  // a halo row before this one
                    scan(hoff[c - 1], hoff[c + 2], tag);
                } else {  // an interior row before this one: its halo cells only
                    if (hx == 1) scan(hoff[c - 1], hoff[c], tag);
                    if (hx == wx) scan(hoff[c + 1], hoff[c + 2], tag);
                }
            }
            const int32_t idi = S.id[qi];
            // a hit (slot k of stencil row r9) -> sorted index, or -1 for the same id; an
            // interior particle after this one in scan order learns of the pair from here
            auto push_rev = [&](int32_t j) {
                const int at_ = atomicAdd(&s_nrev, 1);
                if (at_ < kRevCap) {
                    s_rev[at_] = make_int2(j, qi);
                } else {  // (buffer full: straight to the global list)
                    const unsigned long long gpos = atomicAdd(&stats->rev_count, 1ull);
                    if (static_cast<int64_t>(gpos) < rev_cap) rev[gpos] = make_int2(j, qi);
                    else ovf[atomicAdd(&stats->ovf_count, 1ull)] = j;  // (list full: j's row is rebuilt)
                }
            };
            auto symmetric = [&](int k, int r9) {
                const int ddy = r9 % 3 - 1, ddz = r9 / 3 - 1;
                const int c = hc + ddy * kHX + ddz * kHX * kHY;
                const int hxj = hx - 1 + (k >= hoff[c] ? 1 : 0) + (k >= hoff[c + 1] ? 1 : 0);
                const bool after = r9 > 4 || (r9 == 4 && k > i);
                return after && hxj >= 1 && hxj <= wx && hy + ddy >= 1 && hy + ddy <= wy && hz + ddz >= 1 &&
                       hz + ddz <= wz;
            };
            if (nn <= kNearCap) {
                int32_t e[kNearCap];
                int m = 0;
#pragma unroll
                for (int t = 0; t < kNearCap; ++t) {
                    if (t < nn) {
                        const int tk = ql[t * kTileThreads];
                        const int k = tk & 0xfff, r9 = tk >> 12;
                        SRM_CHK(k < total && r9 < 9, 106);
                        const int32_t j = pj[k];
                        if (S.id[j] != idi) {
#pragma unroll
                            for (int u = 0; u < kNearCap; ++u)
                                if (u == m) e[u] = j;
                            ++m;
                            if (symmetric(k, r9)) push_rev(j);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kNearCap; ++u)
                    if (u >= m) e[u] = 0;
                int4* rowp = reinterpret_cast<int4*>(nbr + static_cast<int64_t>(qi) * kNearRow);
                rowp[0] = make_int4(m, e[0], e[1], e[2]);
                rowp[1] = make_int4(e[3], e[4], e[5], e[6]);
                continue;
            }
            // more hits than the row holds already: the full stencil into the overflow pool
            // (as the full-stencil kernel does: count, reserve, fill -- the same predicate
            // both times), and the reverse entries of the pairs this particle owns
            int cnt = 0;
            int32_t* dst = nullptr;
            int64_t off = 0;
#pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {
                int m = 0;
#pragma unroll 1
                for (int r9 = 0; r9 < 9; ++r9) {
                    const int c = hc + (r9 % 3 - 1) * kHX + (r9 / 3 - 1) * kHX * kHY;
                    const int kb = hoff[c - 1], ke = hoff[c + 2];
                    for (int k = kb; k < ke; ++k) {
                        const float* a = reinterpret_cast<const float*>(pxy + (k >> 1)) + (k & 1);
                        const float* b = reinterpret_cast<const float*>(pzw + (k >> 1)) + (k & 1);
                        const float ex = __fadd_rn(a[0], -mx), ey = __fadd_rn(a[2], -my), ez = __fadd_rn(b[0], -mz);
                        const float d2 = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
                        const float lim = __fadd_rn(b[2], base);
                        if (d2 <= __fmul_rn(__fmul_rn(lim, lim), 1.00001f) && k != i) {
                            const int32_t j = pj[k];
                            if (S.id[j] != idi) {
                                if (pass == 1) {
                                    if (dst && m < cnt) dst[m] = j;
                                    if (symmetric(k, r9)) push_rev(j);
                                }
                                ++m;
                            }
                        }
                    }
                }
                if (pass == 0) {
                    cnt = m;
                    off = static_cast<int64_t>(atomicAdd(&stats->pool_top, static_cast<unsigned long long>(cnt)));
                    dst = off + cnt <= pool.cap ? pool.e + off : nullptr;
                }
            }
            int4* rowp = reinterpret_cast<int4*>(nbr + static_cast<int64_t>(qi) * kNearRow);
            if (!dst) {  // pool full: the sweep rescans the stencil
                rowp[0] = make_int4(cnt, -1, 0, 0);
                rowp[1] = make_int4(0, 0, 0, 0);
            } else if (cnt > kNearCap) {
                rowp[0] = make_int4(cnt, static_cast<int32_t>(off), 0, 0);
                rowp[1] = make_int4(0, 0, 0, 0);
            } else {  // same-id images removed: the list fits the row after all
                int32_t e2[kNearCap];
#pragma unroll
                for (int t = 0; t < kNearCap; ++t) e2[t] = t < cnt ? dst[t] : 0;
                rowp[0] = make_int4(cnt, e2[0], e2[1], e2[2]);
                rowp[1] = make_int4(e2[3], e2[4], e2[5], e2[6]);
            }
            continue;
        }
#endif
#pragma unroll kNearRowUnroll
        for (int row9 = 0; row9 < 9; ++row9) {
            const int ddy = row9 % 3 - 1, ddz = row9 / 3 - 1;
            const int c = hc + ddy * kHX + ddz * kHX * kHY;
            const int kb = hoff[c - 1], ke = hoff[c + 2];
            SRM_CHK(c >= 1 && c + 2 <= kHCells && kb >= 0 && kb <= ke && ke <= total, 103);
#if NT_SCREEN == 0
            // slots [kb, ke) two at a time (pairs 2p, 2p + 1; the ends masked)
            for (int p = kb >> 1; 2 * p < ke; ++p) {
                const float4 A = pxy[p], B = pzw[p];
                const float2 ex = __fadd2_rn(make_float2(A.x, A.y), nmx);
                const float2 ey = __fadd2_rn(make_float2(A.z, A.w), nmy);
                const float2 ez = __fadd2_rn(make_float2(B.x, B.y), nmz);
                const float2 d2 = __ffma2_rn(ex, ex, __ffma2_rn(ey, ey, __fmul2_rn(ez, ez)));
                float2 l2;
                if (SRM_NEAR_MONO && mono) {
                    l2 = make_float2(l2m, l2m);
                } else {
                    const float2 lim = __fadd2_rn(make_float2(B.z, B.w), base2);
                    l2 = __fmul2_rn(__fmul2_rn(lim, lim), fac2);
                }
                const int k0 = 2 * p;
                ql[at * kTileThreads] = static_cast<uint16_t>(k0 + NT_TAG(row9));
                nn += (d2.x <= l2.x && k0 >= kb && k0 != i) ? 1 : 0;
                at = min(nn, kNearCap);
                ql[at * kTileThreads] = static_cast<uint16_t>(k0 + 1 + NT_TAG(row9));
                nn += (d2.y <= l2.y && k0 + 1 < ke && k0 + 1 != i) ? 1 : 0;
                at = min(nn, kNearCap);
            }
#elif NT_SCREEN == 2
            // slots [kb, ke) two at a time; ONE record per pair with a hit in either slot
            // (pair index + stencil row).  The ends of the range, the particle itself and
            // the slots proper are sorted out after the scan, from the few recorded pairs.
            if (mono) {
                for (int p = kb >> 1; 2 * p < ke; ++p) {
                    const float4 A = pxy[p];
                    const float2 Bz = *reinterpret_cast<const float2*>(pzw + p);
                    const float2 ex = __fadd2_rn(make_float2(A.x, A.y), nmx);
                    const float2 ey = __fadd2_rn(make_float2(A.z, A.w), nmy);
                    const float2 ez = __fadd2_rn(Bz, nmz);
                    const float2 d2 = __ffma2_rn(ex, ex, __ffma2_rn(ey, ey, __fmul2_rn(ez, ez)));
                    ql[at * kTileThreads] = static_cast<uint16_t>(p + (row9 << 11));
                    nn += (d2.x <= l2m || d2.y <= l2m) ? 1 : 0;
                    at = min(nn, kPairCap);
                }
            } else {
                for (int p = kb >> 1; 2 * p < ke; ++p) {
                    const float4 A = pxy[p], B = pzw[p];
                    const float2 ex = __fadd2_rn(make_float2(A.x, A.y), nmx);
                    const float2 ey = __fadd2_rn(make_float2(A.z, A.w), nmy);
                    const float2 ez = __fadd2_rn(make_float2(B.x, B.y), nmz);
                    const float2 d2 = __ffma2_rn(ex, ex, __ffma2_rn(ey, ey, __fmul2_rn(ez, ez)));
                    const float2 lim = __fadd2_rn(make_float2(B.z, B.w), base2);
                    const float2 l2 = __fmul2_rn(__fmul2_rn(lim, lim), fac2);
                    ql[at * kTileThreads] = static_cast<uint16_t>(p + (row9 << 11));
                    nn += (d2.x <= l2.x || d2.y <= l2.y) ? 1 : 0;
                    at = min(nn, kPairCap);
                }
            }
#else
            // slots [kb, ke) two at a time (pairs 2p, 2p + 1), 16 pairs per mask
            for (int pb = kb >> 1; 2 * pb < ke; pb += 16) {
                const int pe = min((ke + 1) >> 1, pb + 16);
                unsigned hits = 0u, bit = 1u;
                if (SRM_NEAR_MONO && mono) {  // the same cutoff for every candidate (bit for bit)
#pragma unroll 2
                    for (int p = pb; p < pe; ++p) {
                        const float4 A = pxy[p];
                        const float2 Bz = *reinterpret_cast<const float2*>(pzw + p);
                        const float2 ex = __fadd2_rn(make_float2(A.x, A.y), nmx);
                        const float2 ey = __fadd2_rn(make_float2(A.z, A.w), nmy);
                        const float2 ez = __fadd2_rn(Bz, nmz);
                        const float2 d2 = __ffma2_rn(ex, ex, __ffma2_rn(ey, ey, __fmul2_rn(ez, ez)));
                        if (d2.x <= l2m) hits |= bit;
                        if (d2.y <= l2m) hits |= bit << 1;
                        bit <<= 2;
                    }
                } else {
#pragma unroll 2
                    for (int p = pb; p < pe; ++p) {
                        const float4 A = pxy[p], B = pzw[p];
                        const float2 ex = __fadd2_rn(make_float2(A.x, A.y), nmx);
                        const float2 ey = __fadd2_rn(make_float2(A.z, A.w), nmy);
                        const float2 ez = __fadd2_rn(make_float2(B.x, B.y), nmz);
                        const float2 d2 = __ffma2_rn(ex, ex, __ffma2_rn(ey, ey, __fmul2_rn(ez, ez)));
                        const float2 lim = __fadd2_rn(make_float2(B.z, B.w), base2);
                        const float2 l2 = __fmul2_rn(__fmul2_rn(lim, lim), fac2);
                        if (d2.x <= l2.x) hits |= bit;
                        if (d2.y <= l2.y) hits |= bit << 1;
                        bit <<= 2;
                    }
                }
                if (hits) {  // the slots of the hits: in [kb, ke), not i itself
                    const int k0 = 2 * pb;
                    if (kb > k0) hits &= ~1u;
                    const int top = ke - k0;  // slots k0 + top ... are past the range
                    if (top < 32) hits &= (1u << top) - 1u;
                    if (i >= k0 && i < k0 + 32) hits &= ~(1u << (i - k0));
                    while (hits) {
                        record(k0 + __ffs(hits) - 1);
                        hits &= hits - 1u;
                    }
                }
            }
#endif
        }
#if NT_SCREEN == 2
        {
            // the recorded pairs -> hit slots (the same fp32 predicate per slot, now with the
            // range ends and the particle itself excluded), kept behind the pair records
            const int npairs = nn;
            uint16_t* qh = ql + (kPairCap + 1) * kTileThreads;
            nn = 0;
            auto slot_hit = [&](int k) {
                const float* a = reinterpret_cast<const float*>(pxy + (k >> 1)) + (k & 1);
                const float* b = reinterpret_cast<const float*>(pzw + (k >> 1)) + (k & 1);
                const float ex = __fadd_rn(a[0], -mx), ey = __fadd_rn(a[2], -my), ez = __fadd_rn(b[0], -mz);
                const float d2 = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
                const float lim = __fadd_rn(b[2], base);
                return d2 <= __fmul_rn(__fmul_rn(lim, lim), 1.00001f);
            };
            if (npairs <= kPairCap) {
#pragma unroll 1
                for (int t = 0; t < npairs; ++t) {
                    const int tg = ql[t * kTileThreads];
                    const int P = tg & 0x7ff, r9 = tg >> 11;
                    const int c = hc + (r9 % 3 - 1) * kHX + (r9 / 3 - 1) * kHX * kHY;
                    const int kb = hoff[c - 1], ke = hoff[c + 2];
#pragma unroll
                    for (int sub = 0; sub < 2; ++sub) {
                        const int k = 2 * P + sub;
                        if (k >= kb && k < ke && k != i && slot_hit(k)) {
                            if (nn < kNearCap) qh[nn * kTileThreads] = static_cast<uint16_t>(k);
                            ++nn;
                        }
                    }
                }
            } else {  // more pairs than records (rare on these grids): count the hits exactly
#pragma unroll 1
                for (int row9 = 0; row9 < 9; ++row9) {
                    const int c = hc + (row9 % 3 - 1) * kHX + (row9 / 3 - 1) * kHX * kHY;
                    const int kb = hoff[c - 1], ke = hoff[c + 2];
                    for (int k = kb; k < ke; ++k)
                        if (k != i && slot_hit(k)) ++nn;
                }
                // (more than kPairCap pairs always hold more than kNearCap hits: only the
                //  particle's own pair is recorded without one -- the slots next to a range
                //  end sit two cells away along x; the overflow branch copes either way)
                if (nn <= kNearCap) nn = kNearCap + 1;
            }
            ql = qh;  // the resolution below reads hit slots
        }
#endif
        // resolve: sorted indices, and shape.hpp:70 self-exclusion by id
        int32_t e[kNearCap];
        int m = 0;
#if NT_FUSED
        // the first trial T1 (a pure function of slot, round and iteration) becomes the
        // tentative record of the new state
        const double4 me64 = S.rec[qi];
        double t1[3];
        {
            const double xi[3] = {me64.x, me64.y, me64.z};
            propose<3>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(S.slot[qi]), 0u, t1);
        }
        rec_new[qi] = make_double4(t1[0], t1[1], t1[2], me64.w);
        if (nn > kNearCap) dflag[qi] = kUndecided;
        if (nn <= kNearCap) {
            const int32_t idi = S.id[qi];
            const int mycls = hcls[hc];
            unsigned pmask = 0;  // bit t: entry t precedes this particle in (class, cell, slot)
#pragma unroll
            for (int t = 0; t < kNearCap; ++t) {
                if (t < nn) {
                    const int tk = ql[t * kTileThreads];
                    const int k = tk & 0xfff, r9 = tk >> 12;
                    SRM_CHK(k < total && r9 < 9, 106);
                    const int c = hc + (r9 % 3 - 1) * kHX + (r9 / 3 - 1) * kHX * kHY;
                    const int hcj = c - 1 + (k >= hoff[c] ? 1 : 0) + (k >= hoff[c + 1] ? 1 : 0);
                    const int32_t j = pj[k];
                    if (S.id[j] != idi) {
                        const bool pre = hcls[hcj] < mycls || (hcj == hc && k < i);
#pragma unroll
                        for (int u = 0; u < kNearCap; ++u)
                            if (u == m) e[u] = j;
                        pmask |= (pre ? 1u : 0u) << m;
                        ++m;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kNearCap; ++u)
                if (u >= m) e[u] = 0;
            bool decided = false;
            if (pmask == 0) {  // every near neighbour is visited later: it sits at its round-start record
                decided = true;
#pragma unroll
                for (int u = 0; u < kNearCap; ++u) {
                    if (u < m) {
                        const double4 v = S.rec[e[u]];
                        const double xl[3] = {v.x, v.y, v.z};
                        if (sphere_overlap<3>(box, t1, me64.w, xl, v.w)) decided = false;
                    }
                }
            }
            dflag[qi] = decided ? static_cast<uint8_t>(0) : kUndecided;
            if (decided) {
                if (rp.write_acc) acc[qi] = 0;
                continue;
            }
            int4* rowp = reinterpret_cast<int4*>(nbr + static_cast<int64_t>(qi) * kNearRow);
            rowp[0] = make_int4(m | static_cast<int>(pmask << 8) | kRowMask, e[0], e[1], e[2]);
            rowp[1] = make_int4(e[3], e[4], e[5], e[6]);
            continue;
        }
        if (false) {  // (longer lists: the overflow branch below)
#else
        if (nn <= kNearCap) {
#endif
            const int32_t idi = S.id[qi];
#pragma unroll
            for (int t = 0; t < kNearCap; ++t) {
                e[t] = 0;
                if (t < nn) {
                    SRM_CHK(ql[t * kTileThreads] < total, 104);
                    const int32_t j = pj[ql[t * kTileThreads]];
                    SRM_CHK(j >= 0 && j < g.n_state, 105);
                    if (S.id[j] != idi) e[t] = j;
                    else e[t] = -1;
                }
            }
#pragma unroll
            for (int t = 0; t < kNearCap; ++t) {  // compact out the (rare) same-id entries
                if (t < nn && e[t] >= 0) {
#pragma unroll
                    for (int u = 0; u < kNearCap; ++u)
                        if (u == m) e[u] = e[t];
                    ++m;
                }
            }
        } else {  // a longer list (crowded grids: most particles): nn entries from the
                  // overflow pool, filled by a second, scalar pass over the staged stencil
                  // (the same fp32 screen, so the same pairs as near_full_particle)
            const int32_t idi = S.id[qi];
            int64_t off = static_cast<int64_t>(atomicAdd(&stats->pool_top, static_cast<unsigned long long>(nn)));
            int4* row = reinterpret_cast<int4*>(nbr + static_cast<int64_t>(qi) * kNearRow);
            if (off + nn > pool.cap) {  // pool full: the sweep rescans the stencil
                row[0] = make_int4(nn, -1, 0, 0);
                row[1] = make_int4(0, 0, 0, 0);
                continue;
            }
            int32_t* dst = pool.e + off;
#pragma unroll 1
            for (int ddz = -1; ddz <= 1; ++ddz) {
#pragma unroll 1
                for (int ddy = -1; ddy <= 1; ++ddy) {
                    const int c = hc + ddy * kHX + ddz * kHX * kHY;
                    const int kb = hoff[c - 1], ke = hoff[c + 2];
                    for (int k = kb; k < ke; ++k) {
                        const float* a = reinterpret_cast<const float*>(pxy + (k >> 1)) + (k & 1);
                        const float* b = reinterpret_cast<const float*>(pzw + (k >> 1)) + (k & 1);
                        const float ex = __fadd_rn(a[0], -mx), ey = __fadd_rn(a[2], -my), ez = __fadd_rn(b[0], -mz);
                        const float d2 = __fmaf_rn(ex, ex, __fmaf_rn(ey, ey, __fmul_rn(ez, ez)));
                        const float lim = __fadd_rn(b[2], base);
                        const float l2 = __fmul_rn(__fmul_rn(lim, lim), 1.00001f);
                        if (d2 <= l2 && k != i) {
                            const int32_t j = pj[k];
                            if (S.id[j] != idi) {
#if NT_FUSED
                                // (bit 31: the entry precedes this particle in the sweep order)
                                const int hcj = c - 1 + (k >= hoff[c] ? 1 : 0) + (k >= hoff[c + 1] ? 1 : 0);
                                const bool pre = hcls[hcj] < hcls[hc] || (hcj == hc && k < i);
                                if (m < nn) dst[m] = pre ? (j | static_cast<int32_t>(0x80000000u)) : j;
#else
                                if (m < nn) dst[m] = j;  // never past the entries reserved above
#endif
                                ++m;
                            }
                        }
                    }
                }
            }
            if (m > nn) {  // the passes disagree (cannot happen with equal predicates): rescan
                row[0] = make_int4(m, -1, 0, 0);
                row[1] = make_int4(0, 0, 0, 0);
            } else if (m > kNearCap) {
                row[0] = make_int4(m | (NT_FUSED ? kRowPool : 0), static_cast<int32_t>(off), 0, 0);
                row[1] = make_int4(0, 0, 0, 0);
            } else {  // same-id images removed: the list fits the row after all
                int32_t e2[kNearCap];
                unsigned pm = 0;
#pragma unroll
                for (int t = 0; t < kNearCap; ++t) {
                    e2[t] = t < m ? dst[t] : 0;
                    if (NT_FUSED && e2[t] < 0) {
                        pm |= 1u << t;
                        e2[t] &= 0x7fffffff;
                    }
                }
                row[0] = make_int4(m | (NT_FUSED ? static_cast<int>(pm << 8) | kRowMask : 0), e2[0], e2[1], e2[2]);
                row[1] = make_int4(e2[3], e2[4], e2[5], e2[6]);
            }
            continue;
        }
        int4* row = reinterpret_cast<int4*>(nbr + static_cast<int64_t>(qi) * kNearRow);
        row[0] = make_int4(m, e[0], e[1], e[2]);
        row[1] = make_int4(e[3], e[4], e[5], e[6]);
    }
#if NT_HALF
    // the brick's reverse entries leave with one atomic
    __syncthreads();
    const int nrev = min(s_nrev, kRevCap);
    if (threadIdx.x == 0 && nrev) s_revbase = atomicAdd(&stats->rev_count, static_cast<unsigned long long>(nrev));
    __syncthreads();
    for (int t = threadIdx.x; t < nrev; t += blockDim.x) {
        const int64_t gpos = static_cast<int64_t>(s_revbase) + t;
        if (gpos < rev_cap) rev[gpos] = s_rev[t];
        else ovf[atomicAdd(&stats->ovf_count, 1ull)] = s_rev[t].x;
    }
#endif
}

