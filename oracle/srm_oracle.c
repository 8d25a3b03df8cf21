/*
 * srm_oracle.c -- CPU restatement of the SRM hot loop.  TEST INFRASTRUCTURE ONLY:
 * the product never loads this file's library.  See srm_oracle.h for scope and
 * DESIGN.md §3 for the parallel round semantics restated here.
 *
 * Compile with -ffp-contract=off -fno-fast-math: every double operation below is a
 * single correctly rounded IEEE operation in the order written, which is the order
 * of the reference's expressions cited next to each function.
 */
#include "srm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------ */
/* geometry.hpp:107-114  PeriodicBox::wrap -- two sequential conditional shifts.   */
void orc_wrap(int dim, const double* L, double* p) {
    for (int a = 0; a < dim; ++a) {
        if (p[a] < 0.0) p[a] += L[a];
        if (p[a] >= L[a]) p[a] -= L[a];
    }
}

/* geometry.hpp:117-129  min_image (single conditional shift per axis) + ordered
 * norm2 (geometry.hpp:44-49: s = 0; s += v0*v0; s += v1*v1; ...).                 */
double orc_min_image_dist2(int dim, const double* L, const double* a, const double* b) {
    double s = 0.0;
    for (int k = 0; k < dim; ++k) {
        double d = a[k] - b[k];
        const double half = 0.5 * L[k];
        if (d > half) d -= L[k];
        if (d < -half) d += L[k];
        s += d * d;
    }
    return s;
}

/* shape.hpp:34-37 SphereShape::overlap: contact counts as overlap. */
static int sphere_overlap(int dim, const double* L, const double* a, double ra, const double* b,
                          double rb) {
    const double rr = ra + rb;
    return orc_min_image_dist2(dim, L, a, b) <= rr * rr;
}

/* ------------------------------------------------------------------------------ */
/* cell_grid.hpp:40-52 CellGrid(box, cell_size): n = max(3, (int)floor(L/cs)),
 * edge = L/n.                                                                      */
int orc_grid_dims(int dim, const double* L, double cell_size, int32_t* dims, double* edge) {
    if (!(cell_size > 0.0)) return -1;
    for (int a = 0; a < dim; ++a) {
        int n = (int)floor(L[a] / cell_size);
        if (n < 3) n = 3;
        dims[a] = n;
        edge[a] = L[a] / n;
    }
    return 0;
}

/* cell_grid.hpp:62-71: i = (int)floor(p/edge); i %= n; if (i < 0) i += n. */
void orc_cell_coords(int dim, const int32_t* dims, const double* edge, const double* p,
                     int32_t* c) {
    for (int a = 0; a < dim; ++a) {
        int i = (int)floor(p[a] / edge[a]);
        i %= dims[a];
        if (i < 0) i += dims[a];
        c[a] = i;
    }
}

/* cell_grid.hpp:74-79 row-major, x fastest. */
uint64_t orc_cell_of(int dim, const int32_t* dims, const double* edge, const double* p) {
    int32_t c[3];
    orc_cell_coords(dim, dims, edge, p, c);
    uint64_t idx = 0;
    for (int a = dim - 1; a >= 0; --a) idx = idx * (uint64_t)dims[a] + (uint64_t)c[a];
    return idx;
}

void orc_keys(int dim, const int32_t* dims, const double* edge, int64_t n, const double* pos,
              uint32_t* keys) {
    for (int64_t i = 0; i < n; ++i) keys[i] = (uint32_t)orc_cell_of(dim, dims, edge, pos + i * dim);
}

/* engine.hpp:151-163: counting sort by cell, stable in storage order.  Here the
 * tie-break is the slot (= storage index in the reference), so the result equals
 * reorder_by_locality's permutation whenever slot[i] == i.                          */
void orc_sort_by_cell(int64_t n, const uint32_t* keys, const int32_t* slot, int64_t ncells,
                      int32_t* order, int64_t* cell_start) {
    memset(cell_start, 0, sizeof(int64_t) * (size_t)(ncells + 1));
    for (int64_t i = 0; i < n; ++i) ++cell_start[keys[i] + 1];
    for (int64_t c = 0; c < ncells; ++c) cell_start[c + 1] += cell_start[c];
    /* process sources in ascending slot order so the counting sort's stability
       yields (key, slot) order */
    int32_t* by_slot = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int64_t* cursor = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncells > 0 ? ncells : 1));
    /* slots are a permutation of 0..n-1 in every use; fall back to an insertion
       order by slot value otherwise */
    int perm_ok = 1;
    for (int64_t i = 0; i < n; ++i) by_slot[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (slot[i] < 0 || slot[i] >= n || by_slot[slot[i]] != -1) { perm_ok = 0; break; }
        by_slot[slot[i]] = (int32_t)i;
    }
    if (!perm_ok) {
        for (int64_t i = 0; i < n; ++i) by_slot[i] = (int32_t)i;
        /* stable insertion sort of indices by slot value */
        for (int64_t i = 1; i < n; ++i) {
            int32_t v = by_slot[i];
            int64_t k = i - 1;
            while (k >= 0 && slot[by_slot[k]] > slot[v]) { by_slot[k + 1] = by_slot[k]; --k; }
            by_slot[k + 1] = v;
        }
    }
    for (int64_t c = 0; c < ncells; ++c) cursor[c] = cell_start[c];
    for (int64_t q = 0; q < n; ++q) {
        const int32_t src = by_slot[q];
        order[cursor[keys[src]]++] = src;
    }
    free(by_slot);
    free(cursor);
}

/* ------------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as
 * 1, 2, 3", SC'11): 10 rounds of two 32x32->64 multiplies with the published
 * multipliers and Weyl key increments.                                             */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n1 = lo1;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        const uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Counter layout:
 *   key  = (lo32(seed), hi32(seed))
 *   ctr  = (slot, attempt, (round_id & 0xFFFFFF) | stream << 24 | draw << 25, iteration)
 * Unit vectors use only +,-,*,/,sqrt so CPU and GPU agree bit for bit:
 *   3D: Marsaglia (1972) -- (x1,x2) uniform in the unit disk, s = x1^2+x2^2 < 1,
 *       u = (2 x1 sqrt(1-s), 2 x2 sqrt(1-s), 1 - 2 s)
 *   2D: (x1,x2) uniform in the unit disk (1e-24 < s < 1), u = (x1,x2) * (1/sqrt(s))
 *       (the reference normalises the same way: random.hpp:68-73, g * (1/sqrt(n2)))
 * A draw takes one Philox block: two 53-bit uniforms on [-1,1).  After 64 rejected
 * draws (probability < 1e-42) the direction falls back to +x.                       */
void orc_unit_vector(int dim, uint64_t seed, uint32_t slot, uint32_t attempt, uint32_t stream,
                     uint32_t round_id, uint32_t iteration, double* u) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (uint32_t draw = 0; draw < 64; ++draw) {
        const uint32_t ctr[4] = {slot, attempt,
                                 (round_id & 0xFFFFFFu) | (stream << 24) | (draw << 25),
                                 iteration};
        uint32_t o[4];
        orc_philox4x32_10(ctr, key, o);
        const uint64_t a = (((uint64_t)o[0] << 32) | o[1]) >> 11;
        const uint64_t b = (((uint64_t)o[2] << 32) | o[3]) >> 11;
        const double x1 = (double)a * 0x1p-52 - 1.0;
        const double x2 = (double)b * 0x1p-52 - 1.0;
        const double t1 = x1 * x1;
        const double t2 = x2 * x2;
        const double s = t1 + t2;
        if (dim == 3) {
            if (s < 1.0) {
                const double q = 2.0 * sqrt(1.0 - s);
                u[0] = x1 * q;
                u[1] = x2 * q;
                u[2] = 1.0 - 2.0 * s;
                return;
            }
        } else {
            if (s < 1.0 && s > 1e-24) {
                const double inv = 1.0 / sqrt(s);
                u[0] = x1 * inv;
                u[1] = x2 * inv;
                return;
            }
        }
    }
    u[0] = 1.0;
    u[1] = 0.0;
    if (dim == 3) u[2] = 0.0;
}

/* shape.hpp:39-44 SphereShape::propose_move: wrap(p + c_m * u), where
 * Vec operator*(double, Vec) multiplies each component (geometry.hpp:29-33) and
 * operator+ adds component-wise (geometry.hpp:21-24).                             */
void orc_propose(int dim, const double* L, const double* x, double c_m, uint64_t seed,
                 uint32_t slot, uint32_t attempt, uint32_t round_id, uint32_t iteration,
                 double* out) {
    double u[3];
    orc_unit_vector(dim, seed, slot, attempt, 0, round_id, iteration, u);
    for (int a = 0; a < dim; ++a) {
        const double step = u[a] * c_m;
        out[a] = x[a] + step;
    }
    orc_wrap(dim, L, out);
}

/* ------------------------------------------------------------------------------ */
/* Independent pair search (not the reference's grid): a uniform bin grid whose bin
 * edge is >= cutoff; emits, for every i, all j != i whose min-image distance to i is
 * <= cut_ij (a superset filter; callers apply the exact predicate).                  */
typedef struct {
    int64_t* start; /* n+1 */
    int32_t* nbr;
} orc_csr;

static void csr_free(orc_csr* c) { free(c->start); free(c->nbr); }

static void build_pairs(int dim, const double* L, int64_t n, const double* x, const double* r,
                        double extra, int brute, orc_csr* out) {
    /* cut_ij = (r_i + r_j + extra) * (1 + 1e-9) + 1e-300 */
    double maxr = 0.0;
    for (int64_t i = 0; i < n; ++i) if (r[i] > maxr) maxr = r[i];
    const double cut_max = (2.0 * maxr + extra) * (1.0 + 1e-9) + 1e-300;
    int64_t cap = 16 * n + 16;
    int64_t cnt = 0;
    out->start = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
    out->nbr = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
#define ORC_PUSH(jj)                                                                     \
    do {                                                                                 \
        if (cnt == cap) { cap *= 2; out->nbr = (int32_t*)realloc(out->nbr, sizeof(int32_t) * (size_t)cap); } \
        out->nbr[cnt++] = (int32_t)(jj);                                                 \
    } while (0)
    if (brute || n < 64) {
        for (int64_t i = 0; i < n; ++i) {
            out->start[i] = cnt;
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                const double c = (r[i] + r[j] + extra) * (1.0 + 1e-9) + 1e-300;
                if (orc_min_image_dist2(dim, L, x + i * dim, x + j * dim) <= c * c) ORC_PUSH(j);
            }
        }
        out->start[n] = cnt;
        return;
    }
    int32_t nb[3] = {1, 1, 1};
    double be[3] = {1, 1, 1};
    int64_t nbins = 1;
    for (int a = 0; a < dim; ++a) {
        int64_t k = (int64_t)(L[a] / cut_max);
        if (k < 1) k = 1;
        if (k > 4096) k = 4096;
        nb[a] = (int32_t)k;
        be[a] = L[a] / (double)k;
        nbins *= k;
    }
    int64_t* bstart = (int64_t*)calloc((size_t)(nbins + 1), sizeof(int64_t));
    int64_t* bin = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int32_t* items = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)nbins);
    for (int64_t i = 0; i < n; ++i) {
        int64_t idx = 0;
        for (int a = dim - 1; a >= 0; --a) {
            int64_t c = (int64_t)floor(x[i * dim + a] / be[a]);
            c %= nb[a];
            if (c < 0) c += nb[a];
            idx = idx * nb[a] + c;
        }
        bin[i] = idx;
        ++bstart[idx + 1];
    }
    for (int64_t b = 0; b < nbins; ++b) bstart[b + 1] += bstart[b];
    for (int64_t b = 0; b < nbins; ++b) cur[b] = bstart[b];
    for (int64_t i = 0; i < n; ++i) items[cur[bin[i]]++] = (int32_t)i;
    for (int64_t i = 0; i < n; ++i) {
        out->start[i] = cnt;
        int64_t c[3] = {0, 0, 0};
        int64_t rem = bin[i];
        for (int a = 0; a < dim; ++a) { c[a] = rem % nb[a]; rem /= nb[a]; }
        int lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            if (a >= dim) { lo[a] = 0; hi[a] = 0; continue; }
            if (nb[a] <= 3) { lo[a] = 0; hi[a] = nb[a] - 1; }
            else { lo[a] = -1; hi[a] = 1; }
        }
        for (int dz = lo[2]; dz <= hi[2]; ++dz)
            for (int dy = lo[1]; dy <= hi[1]; ++dy)
                for (int dx = lo[0]; dx <= hi[0]; ++dx) {
                    int64_t m[3];
                    const int d[3] = {dx, dy, dz};
                    for (int a = 0; a < dim; ++a) {
                        if (nb[a] <= 3) m[a] = d[a];
                        else { m[a] = c[a] + d[a]; if (m[a] < 0) m[a] += nb[a]; if (m[a] >= nb[a]) m[a] -= nb[a]; }
                    }
                    int64_t idx = 0;
                    for (int a = dim - 1; a >= 0; --a) idx = idx * nb[a] + m[a];
                    for (int64_t t = bstart[idx]; t < bstart[idx + 1]; ++t) {
                        const int32_t j = items[t];
                        if (j == i) continue;
                        const double cj = (r[i] + r[j] + extra) * (1.0 + 1e-9) + 1e-300;
                        if (orc_min_image_dist2(dim, L, x + i * dim, x + (int64_t)j * dim) <= cj * cj)
                            ORC_PUSH(j);
                    }
                }
    }
    out->start[n] = cnt;
#undef ORC_PUSH
    free(bstart); free(bin); free(items); free(cur);
}

/* ------------------------------------------------------------------------------ */
/* Colouring of the round grid.  Per axis: s = smallest s >= 1 with
 * s * edge >= cutc, cutc = (2 maxR + 3 c_m)(1+1e-9)^2 + ..., the reach of any trial
 * against any (possibly moving) neighbour; "all" when 2s+1 >= dims (every coordinate its
 * own colour), else modulus m = s+1 with the tail cells (dims mod m) each its own
 * colour.  Two cells of one class are then farther apart than any interaction.      */
void orc_colouring(int dim, const int32_t* dims, const double* edge, double maxr, double c_m,
                   int32_t* m_out, int32_t* ncol_out) {
    const double cutc = ((maxr + maxr + 3.0 * c_m) * (1.0 + 1e-9) + 1e-300) * (1.0 + 1e-9);
    for (int a = 0; a < 3; ++a) {
        if (a >= dim) { m_out[a] = 1; ncol_out[a] = 1; continue; }
        int64_t s = 1;
        while ((double)s * edge[a] < cutc && 2 * s + 1 < dims[a]) ++s;
        if (2 * s + 1 >= dims[a]) { m_out[a] = dims[a]; ncol_out[a] = dims[a]; }
        else { m_out[a] = (int32_t)(s + 1); ncol_out[a] = (int32_t)(s + 1) + dims[a] % (int32_t)(s + 1); }
    }
}

static int colour1(int x, int m, int n) {
    const int body = m * (n / m);
    return x < body ? x % m : m + (x - body);
}

/* One SRM round's migrate as a coloured Gauss-Seidel sweep: the
 * reference's migrate (engine.hpp:89-107) -- per particle <= n_l trials from its
 * pre-sweep position, each tested against the LIVE positions of all other particles
 * (shape.hpp:64-73, trial first), first clear trial kept, otherwise an exact revert --
 * in the order (cell class, cell, slot) of the round grid of cell size `cell_size`
 * instead of storage order.  Cells of one class never interact, so the GPU runs them
 * concurrently and equals this sequential sweep bit for bit.  Trials draw Philox
 * (orc_propose) instead of mt19937_64.  brute != 0: all-pairs candidate search.      */
void orc_sweep_round(int dim, const double* L, int64_t n, const double* x0, const double* r,
                     const int32_t* id, const int32_t* slot, double cell_size, double c_m, int n_l,
                     uint64_t seed, uint32_t round_id, uint32_t iteration, double* xnew,
                     uint8_t* acc, int brute) {
    int32_t dims[3] = {1, 1, 1};
    double edge[3] = {1.0, 1.0, 1.0};
    orc_grid_dims(dim, L, cell_size, dims, edge);
    const double maxr = orc_max_radius(n, r);
    int32_t m[3], ncol[3];
    orc_colouring(dim, dims, edge, maxr, c_m, m, ncol);
    /* candidates: j whose round-start distance is within ri + rj + 2 c_m (a superset of
       every j a trial of i can touch while j sits within c_m of its start) */
    orc_csr nb;
    build_pairs(dim, L, n, x0, r, 2.0 * c_m, brute, &nb);
    int64_t ncells = 1;
    for (int a = 0; a < dim; ++a) ncells *= dims[a];
    uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n + 1));
    orc_keys(dim, dims, edge, n, x0, keys);
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int64_t* cstart = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncells + 1));
    orc_sort_by_cell(n, keys, slot, ncells, order, cstart);
    /* class of every particle, then a stable pass per class in (cell, slot) order */
    int32_t* cls = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int64_t nclass = (int64_t)ncol[0] * ncol[1] * ncol[2];
    for (int64_t i = 0; i < n; ++i) {
        int32_t c[3];
        orc_cell_coords(dim, dims, edge, x0 + i * dim, c);
        int64_t k = 0;
        for (int a = dim - 1; a >= 0; --a) k = k * ncol[a] + colour1(c[a], m[a], dims[a]);
        cls[i] = (int32_t)k;
    }
    memcpy(xnew, x0, sizeof(double) * (size_t)(n * dim));
    for (int64_t i = 0; i < n; ++i) acc[i] = ORC_NOT_ACCEPTED;
    double p[3];
    /* order: (cell class, cell, slot) */
    for (int64_t k = 0; k < nclass; ++k) {
        for (int64_t q = 0; q < n; ++q) { /* q walks the (cell, slot) order */
            const int64_t i = order[q];
            if (cls[i] != k) continue;
            for (int l = 0; l < n_l; ++l) {
                orc_propose(dim, L, x0 + i * dim, c_m, seed, (uint32_t)slot[i], (uint32_t)l, round_id,
                            iteration, p);
                int ok = 1;
                for (int64_t t = nb.start[i]; t < nb.start[i + 1] && ok; ++t) {
                    const int64_t j = nb.nbr[t];
                    if (id[j] == id[i]) continue;
                    if (sphere_overlap(dim, L, p, r[i], xnew + j * dim, r[j])) ok = 0;
                }
                if (ok) {
                    memcpy(xnew + i * dim, p, sizeof(double) * (size_t)dim);
                    acc[i] = (uint8_t)l;
                    break;
                }
            }
        }
    }
    free(keys); free(order); free(cstart); free(cls);
    csr_free(&nb);
}

/* Global overlap statistics over all pairs of a state (the counting form of
 * cell_grid.hpp:209-215 / shape.hpp:75-81: count > 0 <=> any collision).        */
void orc_overlap_stats(int dim, const double* L, int64_t n, const double* x, const double* r,
                       const int32_t* id, orc_round_stats* out) {
    orc_csr nb;
    build_pairs(dim, L, n, x, r, 0.0, 0, &nb);
    int64_t pairs = 0;
    double pen = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t t = nb.start[i]; t < nb.start[i + 1]; ++t) {
            const int64_t j = nb.nbr[t];
            if (j <= i || id[j] == id[i]) continue;
            const double rr = r[i] + r[j];
            const double d2 = orc_min_image_dist2(dim, L, x + i * dim, x + j * dim);
            if (d2 <= rr * rr) {
                ++pairs;
                const double p = rr - sqrt(d2);
                if (p > pen) pen = p;
            }
        }
    }
    out->overlap_pairs = pairs;
    out->max_penetration = pen;
    out->candidate_pairs = 0;
    out->movers = 0;
    csr_free(&nb);
}

/* Ordered candidate pairs visited by a 3^d neighbourhood scan (cell_grid.hpp:137-157
 * with dims >= 3, so the offset cells are distinct), self excluded.                  */
int64_t orc_candidate_pairs(int dim, const int32_t* dims, int64_t n, const uint32_t* keys) {
    int64_t ncells = 1;
    for (int a = 0; a < dim; ++a) ncells *= dims[a];
    int64_t* cnt = (int64_t*)calloc((size_t)ncells, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) ++cnt[keys[i]];
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t rem = keys[i];
        int c[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) { c[a] = (int)(rem % dims[a]); rem /= dims[a]; }
        const int zlo = dim == 3 ? -1 : 0, zhi = dim == 3 ? 1 : 0;
        for (int dz = zlo; dz <= zhi; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int d[3] = {dx, dy, dz};
                    int64_t idx = 0;
                    for (int a = dim - 1; a >= 0; --a) {
                        int m = c[a] + d[a];
                        if (m < 0) m += dims[a];
                        if (m >= dims[a]) m -= dims[a];
                        idx = idx * dims[a] + m;
                    }
                    total += cnt[idx];
                }
        total -= 1;
    }
    free(cnt);
    return total;
}

double orc_max_radius(int64_t n, const double* r) {
    double m = 0.0; /* shape.hpp:91-96 starts from 0.0 */
    for (int64_t i = 0; i < n; ++i) m = r[i] > m ? r[i] : m;
    return m;
}

/* geometry.hpp:149-164: pi r^2 or (4/3) pi r^3, summed in storage order, / measure */
double orc_volume_fraction_seq(int dim, const double* L, int64_t n, const double* r) {
    const double pi = 3.141592653589793238462643383279502884;
    double sum = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (dim == 2) sum += pi * r[i] * r[i];
        else sum += (4.0 / 3.0) * pi * r[i] * r[i] * r[i];
    }
    double m = 1.0;
    for (int a = 0; a < dim; ++a) m *= L[a];
    return sum / m;
}

/* ==================================================================================
 * Thin circular platelets (spherodisks): the reference's SpherodiskShape restated
 * (spherodisk.hpp:16-99, spherodisk.cpp:14-112).  Vectors are double[3]; every
 * expression keeps the reference's operation order.                                  */
typedef struct { double v[3]; } pv3;

/* geometry.hpp:117-125 minimum image of one coordinate difference */
static double orc_min_image(double d, double L) {
    const double half = 0.5 * L;
    if (d > half) d -= L;
    if (d < -half) d += L;
    return d;
}

static pv3 pv(double x, double y, double z) { pv3 r; r.v[0] = x; r.v[1] = y; r.v[2] = z; return r; }
static pv3 pv_add(pv3 a, pv3 b) { for (int i = 0; i < 3; ++i) a.v[i] += b.v[i]; return a; }
static pv3 pv_sub(pv3 a, pv3 b) { for (int i = 0; i < 3; ++i) a.v[i] -= b.v[i]; return a; }
static pv3 pv_mul(pv3 a, double s) { for (int i = 0; i < 3; ++i) a.v[i] *= s; return a; }
static double pv_dot(pv3 a, pv3 b) { double s = 0.0; for (int i = 0; i < 3; ++i) s += a.v[i] * b.v[i]; return s; }
static double pv_norm(pv3 a) { return sqrt(pv_dot(a, a)); }
static pv3 pv_cross(pv3 a, pv3 b) {
    return pv(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2], a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}

/* spherodisk.cpp:14-21 */
static pv3 pl_closest(pv3 c, pv3 n, double r, pv3 p) {
    const pv3 w = pv_sub(p, c);
    pv3 in_plane = pv_sub(w, pv_mul(n, pv_dot(w, n)));
    const double d2 = pv_dot(in_plane, in_plane);
    if (d2 > r * r) in_plane = pv_mul(in_plane, r / sqrt(d2));
    return pv_add(c, in_plane);
}

/* spherodisk.cpp:29-40 */
static double pl_alternate(pv3 c1, pv3 n1, double r1, pv3 c2, pv3 n2, double r2, pv3 p2, double tol, int max_iter) {
    double prev = INFINITY;
    for (int it = 0; it < max_iter; ++it) {
        const pv3 p1 = pl_closest(c1, n1, r1, p2);
        p2 = pl_closest(c2, n2, r2, p1);
        const double d = pv_norm(pv_sub(p1, p2));
        if (prev - d <= tol) return d;
        prev = d;
    }
    return prev;
}

static double pl_max3(double a, double b, double c) {
    double m = a;
    if (m < b) m = b;
    if (m < c) m = c;
    return m;
}

/* spherodisk.cpp:70-112 */
static int pl_disks_within(pv3 c1, pv3 n1, double r1, pv3 c2, pv3 n2, double r2, double threshold) {
    const pv3 d = pv_sub(c2, c1);
    if (pv_norm(d) - r1 - r2 > threshold) return 0;
    const double ndot = pv_dot(n1, n2);
    const double t = 1.0 - ndot * ndot;
    const double sin_tilt = sqrt(0.0 < t ? t : 0.0);
    if (fabs(pv_dot(n1, d)) - r2 * sin_tilt > threshold) return 0;
    if (fabs(pv_dot(n2, d)) - r1 * sin_tilt > threshold) return 0;
    const double tol = 1e-12 * pl_max3(r1, r2, 1e-30);
    pv3 p2 = pl_closest(c2, n2, r2, c1);
    double prev = INFINITY;
    int converged = 0;
    for (int it = 0; it < 200; ++it) {
        const pv3 p1 = pl_closest(c1, n1, r1, p2);
        p2 = pl_closest(c2, n2, r2, p1);
        const double dist = pv_norm(pv_sub(p1, p2));
        if (dist <= threshold) return 1;
        if (prev - dist <= tol) { converged = 1; break; }
        prev = dist;
    }
    if (converged) return 0;
    pv3 u = fabs(n2.v[0]) < 0.9 ? pv(1.0, 0.0, 0.0) : pv(0.0, 1.0, 0.0);
    u = pv_sub(u, pv_mul(n2, pv_dot(u, n2)));
    u = pv_mul(u, 1.0 / pv_norm(u));
    const pv3 v = pv_cross(n2, u);
    const double pi = 3.141592653589793238462643383279502884;
    for (int k = 0; k < 32; ++k) {
        const double a = 2.0 * pi * k / 32;
        const pv3 seed = pv_add(c2, pv_mul(pv_add(pv_mul(u, cos(a)), pv_mul(v, sin(a))), r2));
        if (pl_alternate(c1, n1, r1, c2, n2, r2, seed, tol, 64) <= threshold) return 1;
    }
    return 0;
}

/* spherodisk.hpp:62-68 with the minimum image of geometry.hpp:117-125 */
int orc_pl_overlap(const double* L, const double* pa, const double* na, double Da, double ta,
                   const double* pb, const double* nb, double Db, double tb) {
    pv3 d;
    for (int k = 0; k < 3; ++k) d.v[k] = orc_min_image(pb[k] - pa[k], L[k]);
    const double cull = 0.5 * (Da + Db + ta + tb);
    if (pv_dot(d, d) > cull * cull) return 0;
    return pl_disks_within(pv(0.0, 0.0, 0.0), pv(na[0], na[1], na[2]), 0.5 * (Da - ta), d, pv(nb[0], nb[1], nb[2]),
                           0.5 * (Db - tb), 0.5 * (ta + tb));
}

double orc_pl_disks_within(const double* c1, const double* n1, double r1, const double* c2, const double* n2, double r2,
                           double threshold) {
    return pl_disks_within(pv(c1[0], c1[1], c1[2]), pv(n1[0], n1[1], n1[2]), r1, pv(c2[0], c2[1], c2[2]),
                           pv(n2[0], n2[1], n2[2]), r2, threshold);
}

/* spherodisk.hpp:29-34 */
double orc_pl_measure(double D, double t) {
    const double pi = 3.141592653589793238462643383279502884;
    const double a = 0.5 * (D - t);
    const double s = 0.5 * t;
    return 2.0 * pi * a * a * s + pi * pi * a * s * s + (4.0 / 3.0) * pi * s * s * s;
}

/* spherodisk.hpp:84-91 propose_move with Philox draws: translation = unit vector of
 * stream 0 (as spheres), rotation axis = unit vector of stream 1, angle c_r (cos/sin
 * given), normal renormalised. */
void orc_pl_propose(const double* L, const double* x, const double* nrm, double c_m, double cos_r, double sin_r,
                    uint64_t seed, uint32_t slot, uint32_t attempt, uint32_t round_id, uint32_t iteration,
                    double* pout, double* nout) {
    orc_propose(3, L, x, c_m, seed, slot, attempt, round_id, iteration, pout);
    double ax[3];
    orc_unit_vector(3, seed, slot, attempt, 1, round_id, iteration, ax);
    const pv3 axis = pv(ax[0], ax[1], ax[2]), v = pv(nrm[0], nrm[1], nrm[2]);
    const pv3 r = pv_add(pv_add(pv_mul(v, cos_r), pv_mul(pv_cross(axis, v), sin_r)),
                         pv_mul(axis, pv_dot(axis, v) * (1.0 - cos_r)));
    const pv3 nn = pv_mul(r, 1.0 / pv_norm(r));
    for (int k = 0; k < 3; ++k) nout[k] = nn.v[k];
}

/* One platelet round: the sphere sweep's visiting order (class, cell, slot) on the
 * grid of cell size cell_size with bounding radii rb = (D + t) / 2 (shape.hpp:91-96),
 * each trial tested as overlap(trial, other) (shape.hpp:64-73, trial first). */
void orc_pl_sweep_round(const double* L, int64_t n, const double* x0, const double* n0, const double* D,
                        const double* t, const int32_t* id, const int32_t* slot, double cell_size, double c_m,
                        double cos_r, double sin_r, int n_l, uint64_t seed, uint32_t round_id, uint32_t iteration,
                        double* xnew, double* nnew, uint8_t* acc) {
    const int dim = 3;
    double* rb = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; ++i) rb[i] = 0.5 * (D[i] + t[i]);
    int32_t dims[3] = {1, 1, 1};
    double edge[3] = {1.0, 1.0, 1.0};
    orc_grid_dims(dim, L, cell_size, dims, edge);
    const double maxr = orc_max_radius(n, rb);
    int32_t m[3], ncol[3];
    orc_colouring(dim, dims, edge, maxr, c_m, m, ncol);
    orc_csr nb;
    build_pairs(dim, L, n, x0, rb, 2.0 * c_m, 0, &nb);
    int64_t ncells = 1;
    for (int a = 0; a < dim; ++a) ncells *= dims[a];
    uint32_t* keys = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n + 1));
    orc_keys(dim, dims, edge, n, x0, keys);
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int64_t* cstart = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ncells + 1));
    orc_sort_by_cell(n, keys, slot, ncells, order, cstart);
    int32_t* cls = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    const int64_t nclass = (int64_t)ncol[0] * ncol[1] * ncol[2];
    for (int64_t i = 0; i < n; ++i) {
        int32_t c[3];
        orc_cell_coords(dim, dims, edge, x0 + i * dim, c);
        int64_t k = 0;
        for (int a = dim - 1; a >= 0; --a) k = k * ncol[a] + colour1(c[a], m[a], dims[a]);
        cls[i] = (int32_t)k;
    }
    memcpy(xnew, x0, sizeof(double) * (size_t)(n * 3));
    memcpy(nnew, n0, sizeof(double) * (size_t)(n * 3));
    for (int64_t i = 0; i < n; ++i) acc[i] = ORC_NOT_ACCEPTED;
    double p[3], q[3];
    for (int64_t k = 0; k < nclass; ++k) {
        for (int64_t qq = 0; qq < n; ++qq) {
            const int64_t i = order[qq];
            if (cls[i] != k) continue;
            for (int l = 0; l < n_l; ++l) {
                orc_pl_propose(L, x0 + i * 3, n0 + i * 3, c_m, cos_r, sin_r, seed, (uint32_t)slot[i], (uint32_t)l,
                               round_id, iteration, p, q);
                int ok = 1;
                for (int64_t tt = nb.start[i]; tt < nb.start[i + 1] && ok; ++tt) {
                    const int64_t j = nb.nbr[tt];
                    if (id[j] == id[i]) continue;
                    if (orc_pl_overlap(L, p, q, D[i], t[i], xnew + j * 3, nnew + j * 3, D[j], t[j])) ok = 0;
                }
                if (ok) {
                    memcpy(xnew + i * 3, p, sizeof(double) * 3);
                    memcpy(nnew + i * 3, q, sizeof(double) * 3);
                    acc[i] = (uint8_t)l;
                    break;
                }
            }
        }
    }
    free(rb); free(keys); free(order); free(cstart); free(cls);
    csr_free(&nb);
}

/* Any-collision in counting form for platelets: unordered pairs {i, j} with
 * overlap(i, j) or overlap(j, i) (shape_any_collision tests every ordered pair). */
int64_t orc_pl_overlap_pairs(const double* L, int64_t n, const double* x, const double* nrm, const double* D,
                             const double* t, const int32_t* id) {
    double* rb = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; ++i) rb[i] = 0.5 * (D[i] + t[i]);
    orc_csr nb;
    build_pairs(3, L, n, x, rb, 0.0, 0, &nb);
    int64_t pairs = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t tt = nb.start[i]; tt < nb.start[i + 1]; ++tt) {
            const int64_t j = nb.nbr[tt];
            if (j <= i || id[j] == id[i]) continue;
            if (orc_pl_overlap(L, x + i * 3, nrm + i * 3, D[i], t[i], x + j * 3, nrm + j * 3, D[j], t[j]) ||
                orc_pl_overlap(L, x + j * 3, nrm + j * 3, D[j], t[j], x + i * 3, nrm + i * 3, D[i], t[i]))
                ++pairs;
        }
    free(rb);
    csr_free(&nb);
    return pairs;
}

/* ---- parallel RSA ------------------------------------------------------------------- */
/* DESIGN.md §3.5.  The sequential restatement of the device's rounds: within a round the
 * device accepts a candidate iff it clears the particles placed before the round and no
 * lower-index candidate of the round that was itself accepted overlaps it -- which is
 * exactly this loop in ascending index. */
void orc_rsa_candidate(int dim, const double* L, uint64_t seed, uint32_t i, uint32_t r, double* out) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o0[4], o1[4];
    const uint32_t c0[4] = {i, r, 0xFFFFFFFFu, 0u}, c1[4] = {i, r, 0xFFFFFFFFu, 1u};
    orc_philox4x32_10(c0, key, o0);
    orc_philox4x32_10(c1, key, o1);
    const uint64_t w[3] = {(((uint64_t)o0[0] << 32) | o0[1]) >> 11, (((uint64_t)o0[2] << 32) | o0[3]) >> 11,
                           (((uint64_t)o1[0] << 32) | o1[1]) >> 11};
    for (int a = 0; a < dim; ++a) {
        double p = (double)w[a] * 0x1p-53 * L[a];
        if (p < 0.0) p += L[a];
        if (p >= L[a]) p -= L[a];
        out[a] = p;
    }
}

int64_t orc_rsa_rounds(int dim, const double* L, int64_t n, const double* radii, uint64_t seed, int64_t max_rounds,
                       double* pos, uint8_t* placed, int64_t* rounds_out) {
    int64_t count = 0, r = 0;
    int64_t* list = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) placed[i] = 0;
    for (r = 0; r < max_rounds && count < n; ++r) {
        for (int64_t i = 0; i < n; ++i) {
            if (placed[i]) continue;
            double c[3] = {0.0, 0.0, 0.0};
            orc_rsa_candidate(dim, L, seed, (uint32_t)i, (uint32_t)r, c);
            int hit = 0;
            for (int64_t k = 0; k < count && !hit; ++k) {
                const int64_t j = list[k];
                const double rr = radii[i] + radii[j];
                hit = orc_min_image_dist2(dim, L, c, pos + j * dim) <= rr * rr;
            }
            if (!hit) {
                for (int a = 0; a < dim; ++a) pos[i * dim + a] = c[a];
                placed[i] = 1;
                list[count++] = i;
            }
        }
    }
    free(list);
    if (rounds_out) *rounds_out = r;
    return count;
}

/* Platelet RSA in rounds (the device's srm_b200_rsa_platelets_device; recipes.cpp:107-148
 * restated the same way as orc_rsa_rounds): in round r every unplaced platelet i draws a
 * centre (orc_rsa_candidate) and a normal (unit vector of slot i, attempt r, stream 1 with
 * round_id 0xFFFFFF and iteration 0xFFFFFFFF) and is placed iff the reference's test
 * overlap(candidate, p) (shape.hpp:64-73, candidate first) is false for every platelet p
 * placed before it in (round, index) order.  All platelets share diameter D and
 * thickness t = D / aspect (recipes.cpp:116-117). */
int64_t orc_rsa_pl_rounds(const double* L, int64_t n, double D, double t, uint64_t seed, int64_t max_rounds,
                          double* pos, double* nrm, uint8_t* placed, int64_t* rounds_out) {
    int64_t count = 0, r = 0;
    int64_t* list = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) placed[i] = 0;
    for (r = 0; r < max_rounds && count < n; ++r) {
        for (int64_t i = 0; i < n; ++i) {
            if (placed[i]) continue;
            double c[3], u[3];
            orc_rsa_candidate(3, L, seed, (uint32_t)i, (uint32_t)r, c);
            orc_unit_vector(3, seed, (uint32_t)i, (uint32_t)r, 1, 0xFFFFFFu, 0xFFFFFFFFu, u);
            int hit = 0;
            for (int64_t k = 0; k < count && !hit; ++k) {
                const int64_t j = list[k];
                hit = orc_pl_overlap(L, c, u, D, t, pos + 3 * j, nrm + 3 * j, D, t);
            }
            if (!hit) {
                for (int a = 0; a < 3; ++a) {
                    pos[3 * i + a] = c[a];
                    nrm[3 * i + a] = u[a];
                }
                placed[i] = 1;
                list[count++] = i;
            }
        }
    }
    free(list);
    if (rounds_out) *rounds_out = r;
    return count;
}
