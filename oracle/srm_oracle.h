/*
 * srm_oracle.h -- CPU restatement of the SRM hot loop (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity oracle for the B200 path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it, and only as the checker.  The product
 * (paper_2605_18254_b200/) never links, loads or calls anything in oracle/.
 *
 * It restates, in plain C99 compiled with -ffp-contract=off (no FMA contraction, so
 * every operation rounds exactly like the reference's plain `-O3` C++ build):
 *   - periodic geometry        (reference proj/core/include/srm/geometry.hpp:107-129)
 *   - cell grid dims / keys    (cell_grid.hpp:40-81)
 *   - stable sort by cell      (engine.hpp:144-166, reorder_by_locality)
 *   - overlap predicates       (shape.hpp:34-37, cell_grid.hpp:194-215)
 *   - Philox4x32-10            (Salmon et al. SC'11; checked against curand's
 *                               curand_Philox4x32_10 and the Random123 KAT vectors)
 *   - the migrate round the GPU implements: the reference's sequential Gauss-Seidel
 *     migrate (engine.hpp:89-107) in a colour-class order with Philox trials instead of
 *     storage order with one mt19937_64 stream, see DESIGN.md §3.
 *
 * Parity status: the grid/key/sort/overlap functions are PINNED against the reference
 * itself (oracle/_ref, built from /root/reference sources) and the reference's own
 * known-answer test cases (tests/test_oracle_pins.py).  The sweep keeps the
 * reference's per-particle algorithm; only the visiting order and the random stream
 * differ, so it is pinned to the reference through its primitives (same propose_move
 * arithmetic, same overlap predicate) and end to end statistically.
 */
#ifndef SRM_ORACLE_H
#define SRM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_NOT_ACCEPTED 255u

/* ---- geometry (geometry.hpp) ---------------------------------------------- */
void orc_wrap(int dim, const double* L, double* p);
double orc_min_image_dist2(int dim, const double* L, const double* a, const double* b);

/* ---- grid (cell_grid.hpp) -------------------------------------------------- */
/* returns 0 on success, -1 if cell_size <= 0 (cell_grid.hpp:41) */
int orc_grid_dims(int dim, const double* L, double cell_size, int32_t* dims, double* edge);
void orc_cell_coords(int dim, const int32_t* dims, const double* edge, const double* p,
                     int32_t* c);
uint64_t orc_cell_of(int dim, const int32_t* dims, const double* edge, const double* p);
void orc_keys(int dim, const int32_t* dims, const double* edge, int64_t n, const double* pos,
              uint32_t* keys);
/* order[q] = source index of the q-th particle sorted by (key, slot); cell_start has
 * ncells+1 entries. Equivalent to engine.hpp:144-166 when slot == storage index. */
void orc_sort_by_cell(int64_t n, const uint32_t* keys, const int32_t* slot, int64_t ncells,
                      int32_t* order, int64_t* cell_start);

/* ---- RNG --------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void orc_unit_vector(int dim, uint64_t seed, uint32_t slot, uint32_t attempt, uint32_t stream,
                     uint32_t round_id, uint32_t iteration, double* u);
void orc_propose(int dim, const double* L, const double* x, double c_m, uint64_t seed,
                 uint32_t slot, uint32_t attempt, uint32_t round_id, uint32_t iteration,
                 double* out);

/* ---- round ------------------------------------------------------------------- */
typedef struct {
    int64_t overlap_pairs;   /* unordered pairs with min_image_dist2 <= (ri+rj)^2 */
    double max_penetration;  /* max (ri+rj - dist) over those pairs, 0 if none      */
    int64_t candidate_pairs; /* ordered (i, j != i) with cell(j) in 3^d stencil of cell(i) */
    int64_t movers;          /* particles that accepted a trial this round          */
} orc_round_stats;

/* Colouring of the round grid: per-axis modulus m and colour count. */
void orc_colouring(int dim, const int32_t* dims, const double* edge, double maxr, double c_m,
                   int32_t* m_out, int32_t* ncol_out);


/* One SRM round's migrate for disks/spheres as the coloured Gauss-Seidel sweep of
 * DESIGN.md §3.1 on the round grid of cell size `cell_size`:
 *   x0[n*dim] round-start positions, r[n], id[n], slot[n] (Philox stream and in-cell
 *   order); xnew[n*dim] out, acc[n] out (attempt of acceptance or 255).
 * brute != 0 forces the O(n^2) all-pairs candidate search. */
void orc_sweep_round(int dim, const double* L, int64_t n, const double* x0, const double* r,
                     const int32_t* id, const int32_t* slot, double cell_size, double c_m, int n_l,
                     uint64_t seed, uint32_t round_id, uint32_t iteration, double* xnew,
                     uint8_t* acc, int brute);

/* Global overlap statistics of a state (all pairs, cell-list accelerated). */
void orc_overlap_stats(int dim, const double* L, int64_t n, const double* x, const double* r,
                       const int32_t* id, orc_round_stats* out);

/* candidate pair count for the given grid (integer, exact) */
int64_t orc_candidate_pairs(int dim, const int32_t* dims, int64_t n, const uint32_t* keys);

/* ---- platelets (spherodisk.hpp:16-99, spherodisk.cpp:14-112) ---------------------- */
/* SpherodiskShape::overlap(a, b) on the periodic box L (argument order matters) */
int orc_pl_overlap(const double* L, const double* pa, const double* na, double Da, double ta,
                   const double* pb, const double* nb, double Db, double tb);
/* disks_within (returns 0/1) */
double orc_pl_disks_within(const double* c1, const double* n1, double r1, const double* c2, const double* n2,
                           double r2, double threshold);
double orc_pl_measure(double D, double t);
void orc_pl_propose(const double* L, const double* x, const double* nrm, double c_m, double cos_r, double sin_r,
                    uint64_t seed, uint32_t slot, uint32_t attempt, uint32_t round_id, uint32_t iteration,
                    double* pout, double* nout);
void orc_pl_sweep_round(const double* L, int64_t n, const double* x0, const double* n0, const double* D,
                        const double* t, const int32_t* id, const int32_t* slot, double cell_size, double c_m,
                        double cos_r, double sin_r, int n_l, uint64_t seed, uint32_t round_id, uint32_t iteration,
                        double* xnew, double* nnew, uint8_t* acc);
int64_t orc_pl_overlap_pairs(const double* L, int64_t n, const double* x, const double* nrm, const double* D,
                             const double* t, const int32_t* id);

/* ---- parallel RSA (the device initial-state generator) ------------ */
/* Candidate of particle i in RSA round r: uniforms from Philox4x32-10 with key = seed and
 * counters (i, r, 0xFFFFFFFF, 0) and (i, r, 0xFFFFFFFF, 1), 53 bits each, times L, wrapped
 * (random_point, random.hpp:56-61, with Philox instead of mt19937_64). */
void orc_rsa_candidate(int dim, const double* L, uint64_t seed, uint32_t i, uint32_t r, double* out);
/* Rounds r = 0, 1, ...: every unplaced particle draws its round-r candidate; in ascending
 * index, a candidate is accepted iff it is strictly non-touching every particle placed in
 * an earlier round or earlier in this round (rsa.hpp:45-55's predicate).  Stops when all
 * are placed or after max_rounds.  pos[i] = particle i's position (placed ones); returns
 * the number placed. */
int64_t orc_rsa_rounds(int dim, const double* L, int64_t n, const double* radii, uint64_t seed, int64_t max_rounds,
                       double* pos, uint8_t* placed, int64_t* rounds_out);
int64_t orc_rsa_pl_rounds(const double* L, int64_t n, double D, double t, uint64_t seed, int64_t max_rounds,
                          double* pos, double* nrm, uint8_t* placed, int64_t* rounds_out);

/* ---- reductions ---------------------------------------------------------------- */
double orc_max_radius(int64_t n, const double* r);
/* volume fraction with the reference's sequential summation order (shape.hpp:83-89) */
double orc_volume_fraction_seq(int dim, const double* L, int64_t n, const double* r);

#ifdef __cplusplus
}
#endif
#endif
