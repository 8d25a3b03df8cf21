// srm_resolve.cuh -- the migrate step of sparse 3D sphere grids by dependency resolution
// (DESIGN.md §3.7).  Included by srm_kernels.cuh after the sweep primitives.
//
// The coloured Gauss-Seidel sweep visits particles in the order pi = (colour class, cell,
// slot) and tests each trial against the LIVE positions of the particle's near list (the
// j within r_i + r_j + 2 c_m of it at the start of the round: nothing else can touch a
// trial).  So the outcome of particle i is a function of
//   * the FINAL positions of its near neighbours that precede it in pi, and
//   * the round-start positions of those that follow it,
// and of nothing else.  The class launches realise pi with one launch per class over the
// whole domain; here every particle is decided as soon as its preceding near neighbours
// are, whatever their class:
//   pass 0  rtiles::k_near_tiles (srm_near_tiles.cuh, NT_FUSED): the near-list brick kernel
//           also draws every particle's first trial T1 (Philox, a pure function of slot,
//           round and iteration), marks which list entries precede the particle, and
//           decides the particles without a preceding entry whose T1 clears their
//           neighbours' round-start positions.  Everything else becomes pending: the row
//           (list + precedence mask) is written, the record of the new state holds T1.
//   pass p  k_resolve_pass: a pending particle whose preceding neighbours were all decided
//           in earlier passes runs its trials (T1 first, then trials 1 .. n_l - 1) against
//           the final records of those and the round-start records of the others.
// The result is the sequential sweep's, bit for bit (same trials, same positions tested,
// decisions are ANDs of exact fp64 predicates): tests compare it with orc_sweep_round.
//
// State: rec_old = S.rec (round-start records, never written), rec_new (the round's
// result), dflag[q] = the pass that decided q (kUndecided: pending).  A reader at pass p
// uses rec_new[j] only if dflag[j] < p, i.e. j was decided by an earlier launch, so no
// load ever races a store of the same launch.

constexpr uint8_t kUndecided = 255;
constexpr int kResolveMaxPasses = 40;          // general passes (launches) per round, at most
constexpr int kResolveThreads = 256;
#ifndef SRM_RESOLVE_MINB
#define SRM_RESOLVE_MINB 4  // CTAs per SM of k_resolve_pass (64 registers)
#endif
constexpr int kResolveMaxCtas = 148 * SRM_RESOLVE_MINB;  // CTAs (list segments) of a pass: all resident
constexpr int kResolveSoloItems = 512;         // a list this short is finished by one CTA
constexpr int32_t kRowMask = 1 << 30;          // row[0] bit: bits 8-14 hold the precedence mask
constexpr int32_t kRowPool = 1 << 29;          // row[0] bit: the list is in the pool, precedence in bit 31 of each entry

// a record that an earlier launch wrote: read from L2 (never from a stale L1 line)
__device__ __forceinline__ double4 ldcg_rec(const double4* p) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// does near entry j precede q in pi?  (rows without a stored mask: overflowed lists)
template <int D>
__device__ __forceinline__ bool precedes(const GridParams& g, const uint32_t* __restrict__ skey, int32_t j,
                                         int32_t q, uint32_t keyq, int clsq) {
    const uint32_t kj = skey[j];
    if (kj == keyq) return j < q;  // same cell: slot order = sorted order
    return class_of_key<D>(g, kj) < clsq;
}

// The rare rows without a precedence mask (overflowed lists in the pool, a stencil rescan
// when the pool was full, rows written by near_full_particle): precedence from the cell
// keys.  Returns -1 (a preceding neighbour is undecided), the accepted trial (p = its
// position), or n_l (every trial rejected).  Kept out of line: the common path stays lean.
template <int D>
__device__ __noinline__ int resolve_overflow(int32_t q, int pass, int4 h0, const double* xi, double ri, int32_t sl,
                                             const State& S, const double4* __restrict__ rec_new,
                                             const uint8_t* __restrict__ dflag, const Box& box, const GridParams& g,
                                             const RoundParams& rp, const cell_t* __restrict__ cs,
                                             const uint32_t* __restrict__ skey, const int32_t* __restrict__ nbr,
                                             const int32_t* __restrict__ pool, double* p) {
    const int nn = h0.x;
    const uint32_t keyq = skey[q];
    const int clsq = class_of_key<D>(g, keyq);
    const int32_t idq = S.id[q];
    bool ready = true;
    auto live = [&](int32_t j, double4* out) {  // live record of j, or "not ready"
        if (precedes<D>(g, skey, j, q, keyq, clsq)) {
            if (__ldcg(dflag + j) >= pass) {
                ready = false;
                return;
            }
            *out = ldcg_rec(rec_new + j);
        } else {
            *out = S.rec[j];
        }
    };
    auto each = [&](auto&& f) {
        if (nn <= kNearCap) {  // (a row written without a mask, e.g. by near_full_particle)
            const int32_t* e = nbr + static_cast<int64_t>(q) * kNearRow + 1;
            for (int t = 0; t < nn; ++t) f(e[t]);
        } else if (h0.y >= 0) {
            const int32_t* e = pool + h0.y;
            for (int t = 0; t < nn; ++t) f(e[t]);
        } else {
            near_candidates<D>(g, cs, S.xf, q, keyq, [&](int64_t j) {
                if (S.id[j] != idq) f(static_cast<int32_t>(j));
            });
        }
    };
    // readiness, and the live records of the list (they cannot change while q is visited:
    // preceding neighbours are final, following ones count with their round-start records);
    // the first kLocal are kept for the trials
    constexpr int kLocal = 24;
    double4 w[kLocal];
    int cnt = 0;
    each([&](int32_t j) {
        if (!ready) return;
        double4 v;
        live(j, &v);
        if (cnt < kLocal) w[cnt] = v;
        ++cnt;
    });
    if (!ready) return -1;
    int l = 0;
    for (;;) {
        bool clear = true;
        if (cnt <= kLocal) {
            for (int t = 0; t < cnt && clear; ++t) {
                const double xl[3] = {w[t].x, w[t].y, w[t].z};
                if (sphere_overlap<D>(box, p, ri, xl, w[t].w)) clear = false;
            }
        } else {
            each([&](int32_t j) {
                if (!clear) return;
                double4 v;
                live(j, &v);
                const double xl[3] = {v.x, v.y, v.z};
                if (sphere_overlap<D>(box, p, ri, xl, v.w)) clear = false;
            });
        }
        if (clear) return l;
        if (++l >= rp.n_l) return l;
        propose<D>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), p);
    }
}

// the decision of q is final: its record, accept flag and (for a non-mover) list entry
template <int D>
__device__ __forceinline__ void resolve_commit(int32_t q, int l, bool clear, const double* p, const double4 me,
                                               double4* __restrict__ rec_new, const RoundParams& rp,
                                               uint8_t* __restrict__ acc, int32_t* __restrict__ active,
                                               StatsDev* stats) {
    if (clear) {
        if (l > 0) rec_new[q] = make_double4(p[0], D > 1 ? p[D > 1 ? 1 : 0] : 0.0, D > 2 ? p[D > 2 ? 2 : 0] : 0.0, me.w);
        if (rp.write_acc) acc[q] = static_cast<uint8_t>(l);
    } else {  // every trial rejected: the particle keeps its round-start position
        rec_new[q] = me;
        if (rp.write_acc) acc[q] = kNotAccepted;
        active[atomicAdd(&stats->active_count, 1ull)] = q;
    }
}

// rows without a precedence mask, start to finish.  Returns 0 (blocked) or 1 (decided).
template <int D>
__device__ __noinline__ int resolve_slow(int32_t q, int pass, int4 h0, const State& S, double4* __restrict__ rec_new,
                                         const uint8_t* __restrict__ dflag, const Box& box, const GridParams& g,
                                         const RoundParams& rp, const cell_t* __restrict__ cs,
                                         const uint32_t* __restrict__ skey, const int32_t* __restrict__ nbr,
                                         const int32_t* __restrict__ pool, uint8_t* __restrict__ acc,
                                         int32_t* __restrict__ active, StatsDev* stats) {
    const double4 me = S.rec[q], t1 = rec_new[q];
    double xi[D], p[D];
    rec_pos<D>(me, xi);
    rec_pos<D>(t1, p);
    const int l = resolve_overflow<D>(q, pass, h0, xi, me.w, S.slot[q], S, rec_new, dflag, box, g, rp, cs, skey, nbr, pool, p);
    if (l < 0) return 0;
    resolve_commit<D>(q, l, l < rp.n_l, p, me, rec_new, rp, acc, active, stats);
    return 1;
}

// Phase A of a pass, one pending particle q: are the preceding neighbours decided, and
// does the first trial T1 (rec_new[q], drawn by pass 0) clear the live records of the near
// list?  Returns 0 (a preceding neighbour is undecided: q stays pending), 1 (decided: T1
// accepted, the record is already in place) or 2 (ready, T1 rejected: trials 1 .. follow
// in resolve_retry).  No Philox here: the lanes of a warp stay together.
template <int D>
__device__ __forceinline__ int resolve_try(int32_t q, int pass, const State& S, double4* __restrict__ rec_new,
                                           const uint8_t* __restrict__ dflag, const Box& box, const GridParams& g,
                                           const RoundParams& rp, const cell_t* __restrict__ cs,
                                           const uint32_t* __restrict__ skey, const int32_t* __restrict__ nbr,
                                           const int32_t* __restrict__ pool, uint8_t* __restrict__ acc,
                                           int32_t* __restrict__ active, StatsDev* stats) {
    SRM_CHK(q >= 0 && q < g.n_state, 301);
    const int4* row = reinterpret_cast<const int4*>(nbr + static_cast<int64_t>(q) * kNearRow);
    const int4 h0 = row[0];
    if (h0.x & kRowPool) {  // a longer list in the pool; bit 31 of an entry: it precedes q
        const int nn = h0.x & 0xffffff;
        const int32_t* ent = pool + h0.y;
        const double4 t1 = rec_new[q];
        double p[D];
        rec_pos<D>(t1, p);
        unsigned worst = 0;
        bool clear = true;
        for (int t0 = 0; t0 < nn; t0 += 4) {  // four entries' flags and records in flight
            int32_t e[4];
            uint8_t fl[4];
            double4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = t0 + u < nn ? ent[t0 + u] : 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                fl[u] = 0;
                if (t0 + u < nn) {
                    const int32_t j = e[u] & 0x7fffffff;
                    SRM_CHK(j < g.n_state, 302);
                    if (e[u] < 0) fl[u] = __ldcg(dflag + j);
                    v[u] = e[u] < 0 ? ldcg_rec(rec_new + j) : S.rec[j];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (t0 + u < nn) {
                    worst = max(worst, static_cast<unsigned>(fl[u]));
                    const double xl[3] = {v[u].x, v[u].y, v[u].z};
                    if (sphere_overlap<D>(box, p, t1.w, xl, v[u].w)) clear = false;
                }
            }
            if (worst >= static_cast<unsigned>(pass)) return 0;
        }
        if (!clear) return 2;
        if (rp.write_acc) acc[q] = 0;
        return 1;
    }
    if (!(h0.x & kRowMask))  // a row written without precedence (pool full: rescan; near_full_particle): rare
        return resolve_slow<D>(q, pass, h0, S, rec_new, dflag, box, g, rp, cs, skey, nbr, pool, acc, active, stats);
    const int4 h1 = row[1];
    const double4 t1 = rec_new[q];  // (T1, radius)
    const int nn = h0.x & 0xff;
    const unsigned mask = (static_cast<unsigned>(h0.x) >> 8) & 0x7fu;
    const int32_t e[kNearCap] = {h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
    for (int t = 0; t < kNearCap; ++t) SRM_CHK(t >= nn || (e[t] >= 0 && e[t] < g.n_state), 303);
    SRM_CHK(nn <= kNearCap, 304);
    auto live = [&](int t, int32_t j) {  // final record of a preceding neighbour, round-start record of a following one
        return ((mask >> t) & 1u) ? ldcg_rec(rec_new + j) : S.rec[j];
    };
    constexpr int kPre = 3;  // records loaded together with the flags; the rest (rare) one by one
    unsigned worst = 0;      // the latest pass that decided a preceding neighbour (kUndecided: none yet)
    double4 v[kPre];
#pragma unroll
    for (int t = 0; t < kNearCap; ++t)
        if (t < nn && ((mask >> t) & 1u)) worst = max(worst, static_cast<unsigned>(__ldcg(dflag + e[t])));
#pragma unroll
    for (int t = 0; t < kPre; ++t)
        if (t < nn) v[t] = live(t, e[t]);
    if (worst >= static_cast<unsigned>(pass)) return 0;
    double p[D];
    rec_pos<D>(t1, p);
    bool clear = true;
#pragma unroll
    for (int t = 0; t < kPre; ++t) {
        if (t < nn) {
            const double xl[3] = {v[t].x, v[t].y, v[t].z};
            if (sphere_overlap<D>(box, p, t1.w, xl, v[t].w)) clear = false;
        }
    }
    const int32_t* ent = nbr + static_cast<int64_t>(q) * kNearRow + 1;
    for (int t = kPre; t < nn && clear; ++t) {
        const double4 w = live(t, ent[t]);
        const double xl[3] = {w.x, w.y, w.z};
        if (sphere_overlap<D>(box, p, t1.w, xl, w.w)) clear = false;
    }
    if (!clear) return 2;
    if (rp.write_acc) acc[q] = 0;
    return 1;
}

// Phase B: trials 1 .. n_l - 1 of a ready particle whose T1 was rejected.  The live records
// of its list are loaded once (they cannot change: preceding neighbours are final, the
// following ones count with their round-start records).
template <int D>
__device__ __forceinline__ void resolve_retry(int32_t q, const State& S, double4* __restrict__ rec_new, const Box& box,
                                              const RoundParams& rp, const int32_t* __restrict__ nbr,
                                              const int32_t* __restrict__ pool,
                                              uint8_t* __restrict__ acc, int32_t* __restrict__ active,
                                              StatsDev* stats) {
    const int32_t* rowi = nbr + static_cast<int64_t>(q) * kNearRow;
    const int h = rowi[0];
    const bool pooled = (h & kRowPool) != 0;
    const int nn = pooled ? (h & 0xffffff) : (h & 0xff);
    const unsigned mask = (static_cast<unsigned>(h) >> 8) & 0x7fu;
    const int32_t* ent = pooled ? pool + rowi[1] : rowi + 1;
    const double4 me = S.rec[q];
    const int32_t sl = S.slot[q];
    auto live = [&](int t) {
        const int32_t e = ent[t];
        const bool pre = pooled ? e < 0 : ((mask >> t) & 1u) != 0;
        const int32_t j = e & 0x7fffffff;
        return pre ? ldcg_rec(rec_new + j) : S.rec[j];
    };
    constexpr int kLocal = 16;  // live records kept for the trials (longer lists reload the rest)
    double4 v[kLocal];
    for (int t = 0; t < nn && t < kLocal; ++t) v[t] = live(t);
    double xi[D], p[D];
    rec_pos<D>(me, xi);
    bool clear = false;
    int l = 1;
    for (; l < rp.n_l; ++l) {
        propose<D>(box, xi, rp.c_m, rp.key, static_cast<uint32_t>(sl), static_cast<uint32_t>(l), p);
        clear = true;
        for (int t = 0; t < nn && clear; ++t) {
            const double4 w = t < kLocal ? v[t] : live(t);
            const double xl[3] = {w.x, w.y, w.z};
            if (sphere_overlap<D>(box, p, me.w, xl, w.w)) clear = false;
        }
        if (clear) break;
    }
    resolve_commit<D>(q, l, clear, p, me, rec_new, rp, acc, active, stats);
}

// Pass p >= 1.  The particle indices are split into gridDim.x contiguous ranges of
// `span` (a multiple of kResolveThreads), one per CTA, for the whole round: pass 1 walks
// its range and takes the pending particles (dflag == kUndecided: pass 0 keeps no list);
// the particles still blocked go to the CTA's own segment of the pending list
// (list[b * span ...], count in seg_cnt), which the same CTA walks in the next pass.  No
// list position is ever reserved with an atomic; the total (pend[pass], a fire-and-forget
// reduction) only tells the next launch when the rest is short enough for CTA 0 to finish
// alone.  A CTA takes kResolveThreads entries at a time, a thread each: phase A for all;
// blocked and retry entries collect in shared memory and leave a full CTA at a time
// (phase B, the Philox work, runs in full warps).  `finish` (the last launch of a round):
// CTA 0 finishes a list of any length, so the round always completes.
template <int D>
__global__ void __launch_bounds__(kResolveThreads, SRM_RESOLVE_MINB) k_resolve_pass(int pass, int finish, int64_t n, int64_t span,
                                                                   State S, double4* __restrict__ rec_new,
                                                                   uint8_t* __restrict__ dflag, Box box,
                                                                   const GridParams* __restrict__ gp,
                                                                   const RoundParams* __restrict__ rpp,
                                                                   const cell_t* __restrict__ cs,
                                                                   const uint32_t* __restrict__ skey,
                                                                   const int32_t* __restrict__ nbr,
                                                                   const int32_t* __restrict__ pool,
                                                                   uint8_t* __restrict__ acc,
                                                                   int32_t* __restrict__ active,
                                                                   int32_t* __restrict__ list_a,
                                                                   int32_t* __restrict__ list_b,
                                                                   int32_t* __restrict__ seg_cnt, StatsDev* stats) {
    const GridParams& g = *gp;
    if (!g.resolve) return;
    __shared__ RoundParams rp;
    __shared__ int32_t s_keep[2 * kResolveThreads], s_retry[2 * kResolveThreads];
    __shared__ int s_nkeep, s_nretry, s_flush, s_doretry;
    if (threadIdx.x == 0) {
        rp = *rpp;
        s_nkeep = 0;
        s_nretry = 0;
    }
    const int G = static_cast<int>(gridDim.x);
    const int32_t* in = (pass & 1) ? list_a : list_b;   // pass 1 ignores it
    int32_t* out = (pass & 1) ? list_b : list_a;
    const int32_t* cnt_in = seg_cnt + ((pass & 1) ? 0 : G);
    int32_t* cnt_out = seg_cnt + ((pass & 1) ? G : 0);
    const int64_t total = pass == 1 ? n : static_cast<int64_t>(stats->pend[pass - 1]);
    const bool solo = pass > 1 && (finish || total <= kResolveSoloItems);
    if (total == 0 || (solo && blockIdx.x != 0)) return;
    __syncthreads();
    if (!solo) {
        const int64_t seg = static_cast<int64_t>(blockIdx.x) * span;
        const int64_t count = pass == 1 ? max(static_cast<int64_t>(0), min(span, n - seg)) : cnt_in[blockIdx.x];
        int32_t* mine = out + seg;  // this CTA's segment of the next list
        int kept = 0;               // entries written to it (block-uniform)
        for (int64_t base = 0; base < count; base += kResolveThreads) {
            const int64_t t = base + threadIdx.x;
            int32_t q = -1;
            if (t < count) {
                if (pass == 1) q = dflag[seg + t] == kUndecided ? static_cast<int32_t>(seg + t) : -1;
                else q = in[seg + t];
            }
            if (q >= 0) {
                const int st = resolve_try<D>(q, pass, S, rec_new, dflag, box, g, rp, cs, skey, nbr, pool, acc, active, stats);
                if (st == 0) s_keep[atomicAdd(&s_nkeep, 1)] = q;
                else if (st == 2) s_retry[atomicAdd(&s_nretry, 1)] = q;
                else dflag[q] = static_cast<uint8_t>(pass);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                s_flush = s_nkeep >= kResolveThreads;
                s_doretry = s_nretry >= kResolveThreads;
                if (s_flush) s_nkeep -= kResolveThreads;
                if (s_doretry) s_nretry -= kResolveThreads;
            }
            __syncthreads();
            if (s_flush) {
                SRM_CHK(kept + static_cast<int>(threadIdx.x) < span, 305);
                mine[kept + threadIdx.x] = s_keep[s_nkeep + threadIdx.x];
                kept += kResolveThreads;
            }
            if (s_doretry) {
                const int32_t r = s_retry[s_nretry + threadIdx.x];
                resolve_retry<D>(r, S, rec_new, box, rp, nbr, pool, acc, active, stats);
                dflag[r] = static_cast<uint8_t>(pass);
            }
            __syncthreads();
        }
        // what is left in the buffers
        const int nk = s_nkeep, nr = s_nretry;
        SRM_CHK(kept + nk <= span && nk <= 2 * kResolveThreads && nr <= 2 * kResolveThreads, 306);
        if (static_cast<int>(threadIdx.x) < nk) mine[kept + threadIdx.x] = s_keep[threadIdx.x];
        if (threadIdx.x == 0) {
            cnt_out[blockIdx.x] = kept + nk;
            if (kept + nk) atomicAdd(&stats->pend[pass], static_cast<unsigned long long>(kept + nk));
        }
        if (static_cast<int>(threadIdx.x) < nr) {
            const int32_t r = s_retry[threadIdx.x];
            resolve_retry<D>(r, S, rec_new, box, rp, nbr, pool, acc, active, stats);
            dflag[r] = static_cast<uint8_t>(pass);
        }
        return;
    }
    // one CTA finishes: the segments' entries are gathered into one list (the other buffer
    // is free: nobody else writes in this launch), then iterations of (decide what is ready;
    // barrier; publish the flags and compact the rest in place).  Flags become visible only
    // after the barrier, so an iteration never reads a record written in the same iteration.
    __shared__ int64_t s_m;
    __shared__ int s_w[kResolveThreads / 32];
    int32_t* cur = out;
    __shared__ int s_off[kResolveMaxCtas + 1];  // first position of a segment's entries in the gathered list
    if (threadIdx.x == 0) {
        int at = 0;
        for (int b = 0; b < G; ++b) {
            s_off[b] = at;
            at += cnt_in[b];
        }
        s_off[G] = at;
        s_m = at;
    }
    __syncthreads();
    for (int b = 0; b < G; ++b) {
        const int c = s_off[b + 1] - s_off[b];
        for (int k = threadIdx.x; k < c; k += kResolveThreads) cur[s_off[b] + k] = in[static_cast<int64_t>(b) * span + k];
    }
    __syncthreads();
    int64_t m = s_m;
    while (m > 0) {
        __syncthreads();
        if (threadIdx.x == 0) s_m = 0;
        for (int64_t b = 0; b < m; b += kResolveThreads) {
            const int64_t t = b + threadIdx.x;
            if (t < m) {
                const int32_t q = cur[t];
                // (every flag other than kUndecided was published before the iteration's barrier)
                int st = resolve_try<D>(q, kUndecided, S, rec_new, dflag, box, g, rp, cs, skey, nbr, pool, acc, active, stats);
                if (st == 2) {
                    resolve_retry<D>(q, S, rec_new, box, rp, nbr, pool, acc, active, stats);
                    st = 1;
                }
                if (st == 1) cur[t] = ~q;  // decided: its flag is published after the barrier
            }
        }
        __threadfence();
        __syncthreads();
        // publish flags, compact the blocked entries to the front (order is irrelevant)
        for (int64_t b = 0; b < m; b += kResolveThreads) {
            const int64_t t = b + threadIdx.x;
            int32_t q = 0;
            bool keep = false;
            if (t < m) {
                q = cur[t];
                if (q < 0) dflag[~q] = static_cast<uint8_t>(pass);
                else keep = true;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            if (lane == 0) s_w[wid] = __popc(bal);
            __syncthreads();  // (also: every entry of the slice was read above)
            int before = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kResolveThreads / 32; ++w) {
                if (w < wid) before += s_w[w];
                tot += s_w[w];
            }
            const int64_t dst = s_m + before + __popc(bal & ((1u << lane) - 1u));
            if (keep) cur[dst] = q;  // dst <= t, and the entries up to the slice's end were read already
            __syncthreads();
            if (threadIdx.x == 0) s_m += tot;
            __syncthreads();
        }
        __threadfence();
        __syncthreads();
        m = s_m;
    }
}
