/*
 * srm_b200.h -- C ABI of the B200-native SRM hot loop (libsrm_b200.so).
 *
 * Plain pointers and sizes only; no C++ types, no exceptions cross this boundary.
 * Every call is synchronous at the API boundary (it returns after the device work it
 * enqueued has finished) except where noted.  One context = one CUDA stream = one
 * device-resident particle state; contexts are independent, so independent runs may
 * proceed concurrently on separate host threads (reference: srmgen --ensemble,
 * tools/srmgen.cpp:119-143).
 *
 * Each entry point names the reference interface it replaces (paths relative to
 * /root/reference/proj/core/include/srm/).  The C++ drop-in shim over this ABI is
 * include/srm/b200/engine.hpp; the Python mirror is paper_2605_18254_b200/__init__.py.
 *
 * Host-side layouts:
 *   pos      double[n*dim], particle-major (x0,y0,[z0],x1,...) == Vec<N>::v
 *   radius   double[n]
 *   id       int32[n]          (Particle<N>::id, geometry.hpp:139-144)
 *   records  any array of structs holding id/pos/radius at given byte offsets, e.g.
 *            std::vector<srm::Particle<N>> (id @0, pos @8, radius @8+8N; stride 32/40)
 * The device keeps its own SoA copy, physically sorted by cell.
 */
#ifndef SRM_B200_H
#define SRM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct srm_b200_ctx srm_b200_ctx;

/* Status codes; the C++ shim maps them back onto errors.hpp:10-43. */
typedef enum {
    SRM_B200_OK = 0,
    SRM_B200_ITERATION_LIMIT = 1, /* GenerateStatus::IterationLimitExceeded (engine.hpp:67) */
    SRM_B200_INVALID = 2,         /* ValidationError / std::invalid_argument                */
    SRM_B200_CUDA_ERROR = 3,      /* device failure (no reference counterpart)              */
    SRM_B200_PLACEMENT_FAILURE = 4, /* PlacementFailure (errors.hpp:15-23)                  */
    SRM_B200_NO_DEVICE = 5,       /* no CUDA device: the product has no CPU fallback         */
    SRM_B200_IO_ERROR = 6         /* IoError (errors.hpp): snapshot file I/O or format       */
} srm_b200_status;

typedef enum {
    SRM_B200_SPHERE = 0,  /* Disk (dim 2) / Ball (dim 3), shape.hpp:29-53 */
    SRM_B200_PLATELET = 1 /* thin circular platelet, SpherodiskShape (spherodisk.hpp:72-99), dim 3 */
} srm_b200_shape;

/* engine.hpp:22-32 SrmParams, field for field. */
typedef struct {
    double c_w;
    double c_m;
    double c_r;
    int32_t n_k;
    int32_t n_l;
    double f_target;
    int64_t max_iterations;
    uint64_t seed;
    int32_t reorder_period;
} srm_b200_params;

/* engine.hpp:75-80 ProgressRecord */
typedef struct {
    int64_t iteration;
    double volume_fraction;
    int32_t accepted;
    double elapsed_seconds;
    int32_t rounds; /* rounds run in this iteration (growth rounds, or n_k shake sweeps) */
} srm_b200_progress_record;

/* engine.hpp:82 ProgressSink */
typedef void (*srm_b200_progress_fn)(const srm_b200_progress_record* rec, void* user);

/* Result of srm_b200_generate (engine.hpp:67-73 GenerateResult + Snapshot metadata). */
typedef struct {
    int32_t status;            /* SRM_B200_OK or SRM_B200_ITERATION_LIMIT */
    double volume_fraction;    /* Snapshot::volume_fraction                */
    int64_t iteration_count;   /* Snapshot::iteration_count (accumulated)  */
    int64_t accepted_iterations;
    int64_t rounds;            /* growth rounds run (each = rebuild+migrate+check) */
    int64_t shake_rounds;      /* shake sweeps run (rebuild+migrate)              */
} srm_b200_generate_out;

/* Per-round statistics, the counting form of shape_any_collision (shape.hpp:75-81). */
typedef struct {
    int64_t overlap_pairs;   /* unordered overlapping pairs; > 0 <=> any collision   */
    double max_penetration;  /* max (ri + rj - dist) over overlapping pairs          */
    int64_t candidate_pairs; /* ordered pairs visited by the 3^d scan (-1: not computed) */
    int64_t movers;          /* particles that accepted a trial                     */
} srm_b200_round_stats;

/* ---- context ------------------------------------------------------------------ */
/* box_lengths[dim]: PeriodicBox<N> ctor (geometry.hpp:68-74; throws on <= 0 -> INVALID).
 * capacity: maximum particle count.  device: CUDA ordinal. */
int srm_b200_create(int dim, int shape_kind, const double* box_lengths, int64_t capacity,
                    int device, srm_b200_ctx** out);
void srm_b200_destroy(srm_b200_ctx* ctx);
/* message of the last failing call on this context ("" if none) */
const char* srm_b200_last_error(const srm_b200_ctx* ctx);
/* message of the last srm_b200_create failure (thread-local) */
const char* srm_b200_create_error(void);

/* ---- state transfer (Snapshot::particles in / out) ----------------------------- */
int srm_b200_upload(srm_b200_ctx* ctx, int64_t n, const double* pos, const double* radius,
                    const int32_t* id);
int srm_b200_download(srm_b200_ctx* ctx, double* pos, double* radius, int32_t* id);
/* platelet contexts (SRM_B200_PLATELET): centre[3n], unit normal[3n], diameter[n],
 * thickness[n] (Spherodisk, spherodisk.hpp:16-22) */
int srm_b200_upload_platelets(srm_b200_ctx* ctx, int64_t n, const double* pos, const double* normal,
                              const double* diameter, const double* thickness, const int32_t* id);
int srm_b200_download_platelets(srm_b200_ctx* ctx, double* pos, double* normal, double* diameter,
                                double* thickness, int32_t* id);
/* rotation angle c_r of platelet moves for srm_b200_round / srm_b200_rounds (SrmParams::c_r;
 * srm_b200_generate and srm_b200_relax_sweeps take it from their own arguments) */
int srm_b200_set_rotation(srm_b200_ctx* ctx, double c_r);

/* array-of-structs variants: one cudaMemcpy of the raw records + an unpack kernel */
int srm_b200_upload_records(srm_b200_ctx* ctx, int64_t n, const void* records, int64_t stride,
                            int64_t off_id, int64_t off_pos, int64_t off_radius);
int srm_b200_download_records(srm_b200_ctx* ctx, void* records, int64_t stride, int64_t off_id,
                              int64_t off_pos, int64_t off_radius);
int64_t srm_b200_count(const srm_b200_ctx* ctx);

/* ---- the drop-in entry points ---------------------------------------------------- */
/* engine.hpp:176-260 srm_generate<S>(initial, params, progress) on the uploaded state;
 * iteration_count_in = initial.iteration_count.  The final state stays on the device
 * (download it).  progress may be NULL. */
int srm_b200_generate(srm_b200_ctx* ctx, const srm_b200_params* params,
                      int64_t iteration_count_in, srm_b200_progress_fn progress, void* user,
                      srm_b200_generate_out* out);

/* srm_b200_generate's loop: device_loop != 0 (default) runs the whole run as one CUDA
 * graph whose controller kernels take every per-iteration decision on the device (no
 * host round-trip per iteration; progress records are delivered after the run);
 * device_loop == 0 drives the same kernels from the host, reading the round statistics
 * after every round (progress delivered live).  Both follow engine.hpp:176-260. */
int srm_b200_set_generate_mode(srm_b200_ctx* ctx, int device_loop);

/* engine.hpp:112-122 relax_sweeps (and shake, engine.hpp:126-130, with sweeps = n_k):
 * `sweeps` x (rebuild grid sized 2.5*maxR + c_m, migrate).  The Rng& of the reference
 * signature becomes a 64-bit Philox key (the shim draws it with rng.raw()). */
int srm_b200_relax_sweeps(srm_b200_ctx* ctx, double c_m, double c_r, int n_l, int sweeps,
                          uint64_t key);

/* engine.hpp:134-138 swell_all: radius *= (1 + c_w) */
int srm_b200_swell_all(srm_b200_ctx* ctx, double c_w);

/* engine.hpp:144-166 reorder_by_locality against a grid of cell size `cell_size`
 * (CellGrid(box, cell_size), cell_grid.hpp:40-52): stable sort by cell, ids and
 * storage order reassigned to slots.  remap_out[old] = new (may be NULL). */
int srm_b200_reorder_by_locality(srm_b200_ctx* ctx, double cell_size, int32_t* remap_out);

/* shape.hpp:91-96 max_bounding_radius; shape.hpp:83-89 shape_volume_fraction
 * (fixed-order device tree sum; equals the sequential sum to ~1e-15 relative) */
int srm_b200_max_bounding_radius(srm_b200_ctx* ctx, double* out);
int srm_b200_volume_fraction(srm_b200_ctx* ctx, double* out);

/* ---- stage entry points (parity tests, benchmarks) --------------------------------- */
/* CellGrid ctor (cell_grid.hpp:31-52): dims/edges for a cell size; safety-checked
 * when max_radius >= 0 (cell_size >= 2*max_radius + slack else INVALID). */
int srm_b200_grid_dims(srm_b200_ctx* ctx, double cell_size, double max_radius, double slack,
                       int32_t* dims_out, double* edge_out, int64_t* ncells_out);

/* Device grid rebuild (cell_grid.hpp:62-108 + engine.hpp:144-166): per-particle keys,
 * stable sort by (key, slot), cell offsets.  Outputs (any may be NULL):
 *   keys_out[n]    keys in the CURRENT host (slot) order: keys_out[s] = cell_of(particle s)
 *   order_out[n]   slots in sorted order (== reorder_by_locality's inverse remap)
 *   cell_start_out[ncells+1]
 * Also leaves the device state physically sorted. */
int srm_b200_grid_build(srm_b200_ctx* ctx, double cell_size, uint32_t* keys_out,
                        int32_t* order_out, int64_t* cell_start_out);

/* shape_any_collision (shape.hpp:75-81) in counting form, against a grid of cell
 * size cell_size (candidate_pairs counts its 3^d scan). */
int srm_b200_overlap_stats(srm_b200_ctx* ctx, double cell_size, srm_b200_round_stats* out);

/* One SRM round (engine.hpp:227-234 body): rebuild the grid of cell size `cell_size`,
 * run the parallel migrate with Philox key/round/iteration, and reduce
 * the overlap statistics.  accepted_out[n] (slot order, may be NULL): phase of
 * acceptance or 255.  with_candidates: also count candidate_pairs. */
int srm_b200_round(srm_b200_ctx* ctx, double cell_size, double c_m, int n_l, uint64_t key,
                   uint32_t round_id, uint32_t iteration, int with_candidates,
                   uint8_t* accepted_out, srm_b200_round_stats* out);

/* `rounds` back-to-back rounds at fixed size, device resident, statistics of the last
 * one; round_id = first_round + k.  Benchmark/e2e entry point. */
int srm_b200_rounds(srm_b200_ctx* ctx, double cell_size, double c_m, int n_l, uint64_t key,
                    uint32_t first_round, uint32_t iteration, int rounds,
                    srm_b200_round_stats* last);

/* ---- snapshots: the reference's file format (snapshot_io.cpp) ------- */
/* the Snapshot fields a file carries besides the particles (snapshot_io.cpp:128-148) */
typedef struct {
    double volume_fraction;
    int64_t iteration_count;
    uint64_t seed;
    srm_b200_params params;
} srm_b200_snapshot_meta;
/* dimension, shape kind and box of a context */
int srm_b200_describe(const srm_b200_ctx* ctx, int* dim, int* shape_kind, double* box_lengths);
/* snapshot_io.cpp:170-191 snapshot_to_binary (binary != 0) or :150-167 snapshot_to_text of
 * host arrays (spheres/disks: pos, radius; platelets: pos, normal, diameter, thickness),
 * byte-identical to the reference's.  out == NULL: *len_inout = the size needed. */
int srm_b200_snapshot_encode(int dim, int shape_kind, const double* box_lengths, int64_t n,
                             const double* pos, const double* radius, const double* normal,
                             const double* diameter, const double* thickness, const int32_t* id,
                             const srm_b200_snapshot_meta* meta, int binary, char* out,
                             int64_t* len_inout);
/* save_snapshot (snapshot_io.cpp:421-426): the context's state, written atomically */
int srm_b200_save_snapshot(srm_b200_ctx* ctx, const char* path, const srm_b200_snapshot_meta* meta,
                           int binary);
/* load_snapshot (snapshot_io.cpp:414-420), binary or text: the header (dim, shape kind,
 * count, box, meta) ... */
int srm_b200_snapshot_info(const char* path, int* dim, int* shape_kind, int64_t* count,
                           double* box_lengths, srm_b200_snapshot_meta* meta);
/* ... and the particles into a context of the same shape and box (count <= capacity) */
int srm_b200_load_snapshot(srm_b200_ctx* ctx, const char* path);
/* message of the last SRM_B200_IO_ERROR (thread-local) */
const char* srm_b200_io_error(void);

/* ---- parity statistics on the device ---------------------------- */
/* descriptors.hpp:96-115 nearest_neighbor_distances of the context's state (exact: the
 * minimum over all other centres, as the reference's ring search) and, when counts_out is
 * given, descriptors.hpp:254-277 histogram(nnd, bins, lo, hi) (counts[bins], total,
 * in_range).  nnd_out (nullable): n distances in download order.  Any shape (platelets:
 * centre distances). */
int srm_b200_nnd_histogram(srm_b200_ctx* ctx, int bins, double lo, double hi, int64_t* counts_out,
                           int64_t* total_out, int64_t* in_range_out, double* nnd_out);
/* Unordered centre-pair distances (min image) binned on edges[0..bins] with
 * numpy.histogram's rule (last bin closed): the RDF counts of the parity tests
 * (tests/stats_util.py rdf_counts; the reference has no RDF). */
int srm_b200_pair_counts(srm_b200_ctx* ctx, const double* edges, int bins, int64_t* counts_out);
/* Platelet statistics on the device (platelet contexts; every output nullable, per-platelet
 * outputs in download order):
 *   value_out / count_out  descriptors.hpp:182-209 local_nematic_order(snapshot, cutoff):
 *                          mean |n_i . n_j| over the platelets whose centre lies within
 *                          cutoff (NaN when none) and their number; skipped when cutoff <= 0
 *                          and both are null, ValidationError's code when asked with cutoff <= 0
 *   nnd_out / nn_align_out centre nearest-neighbour distance and |n . n'| of that neighbour
 *   q_out[6]               sum over platelets of n (x) n: xx, yy, zz, xy, xz, yz (the Q tensor
 *                          of the nematic order parameter S2 = largest eigenvalue of
 *                          (3 q / n - 1) / 2), summed in a fixed order */
int srm_b200_platelet_order(srm_b200_ctx* ctx, double cutoff, double* value_out, int32_t* count_out, double* nnd_out,
                            double* nn_align_out, double* q_out);

/* ---- initial states (rsa.hpp:21-69) ------------------------------------------------ */
/* rsa_place with Rng(seed) (std::mt19937_64): bit-identical to the reference for the
 * same seed.  Host code (input generation; excluded from the metric).
 * Returns OK / INVALID / PLACEMENT_FAILURE (placed_out = particles placed). */
int srm_b200_rsa_place(int dim, const double* box_lengths, int64_t n, const double* radii,
                       int64_t max_attempts, uint64_t seed, double* pos_out, int32_t* id_out,
                       int64_t* placed_out);
/* recipes.cpp:107-148 rsa_platelets with Rng(seed): n platelets of one diameter and
 * aspect ratio (diameter / thickness) in the box; bit-identical to the reference.
 * Returns OK / INVALID / PLACEMENT_FAILURE (placed_out = platelets placed). */
int srm_b200_rsa_platelets(int64_t n, double diameter, double aspect_ratio, const double* box_lengths,
                           int64_t max_attempts, uint64_t seed, double* pos_out, double* normal_out,
                           int32_t* id_out, int64_t* placed_out);
/* Clustered RSA (BASELINE.json configs[2] start; builder-defined, no reference
 * counterpart): cluster centres uniform, particle i in cluster i mod n_clusters, candidates
 * wrap(centre + sigma * gaussian), strictly non-touching as rsa_place.  Rng(seed) =
 * std::mt19937_64 with the reference's uniform / Box-Muller gaussian (random.hpp:16-61).
 * Returns OK / INVALID / PLACEMENT_FAILURE (placed_out = particles placed). */
int srm_b200_rsa_clustered(int dim, const double* box_lengths, int64_t n, const double* radii,
                           int64_t n_clusters, double sigma, int64_t max_attempts, uint64_t seed,
                           double* pos_out, int32_t* id_out, int64_t* placed_out);
/* Random sequential adsorption on the device: rounds in which every
 * unplaced particle draws a Philox candidate (seed, index, round), accepted iff strictly
 * non-touching (rsa.hpp's predicate) every particle placed earlier and every accepted
 * lower-index candidate of the round -- the sequential RSA that visits each round's
 * unplaced particles in index order (oracle orc_rsa_rounds, bit for bit).  The state
 * (id = index) is left in the context.  OK, or PLACEMENT_FAILURE after max_rounds
 * (placed_out / rounds_out report), INVALID. */
int srm_b200_rsa_device(srm_b200_ctx* ctx, int64_t n, const double* radii, uint64_t seed, int64_t max_rounds,
                        int64_t* placed_out, int64_t* rounds_out);
/* rsa_platelets (recipes.cpp:107-148) on the device: the same rounds with candidate =
 * (Philox centre, Philox unit normal), placed iff the reference's overlap(candidate, p)
 * (candidate first) is false for every platelet placed before it in (round, index) order
 * (oracle orc_rsa_pl_rounds, bit for bit).  Diameter D, thickness D / aspect_ratio for all;
 * the state (id = index) is left in the platelet context.  OK, PLACEMENT_FAILURE after
 * max_rounds (placed_out / rounds_out report), INVALID (recipes.cpp:109-117 checks). */
int srm_b200_rsa_platelets_device(srm_b200_ctx* ctx, int64_t n, double diameter, double aspect_ratio, uint64_t seed,
                                  int64_t max_rounds, int64_t* placed_out, int64_t* rounds_out);
/* random.hpp:84-89 mix_seed */
uint64_t srm_b200_mix_seed(uint64_t seed, uint64_t stream);

/* ---- instrumentation ---------------------------------------------------------------- */
/* Kernel launches issued by this context since creation (or the last reset). */
int64_t srm_b200_launch_count(const srm_b200_ctx* ctx);
void srm_b200_reset_launch_count(srm_b200_ctx* ctx);
/* CUDA graphs the device-resident srm_b200_generate captured and instantiated on this
 * context (a later call reuses the cached graph while its buffers and bounds are unchanged). */
int64_t srm_b200_graph_builds(const srm_b200_ctx* ctx);
/* CUDA-event timing of kernel families on the context stream.  enable != 0 starts
 * recording; srm_b200_timing_get fills ms[SRM_B200_NPHASE] with accumulated device
 * milliseconds and calls[SRM_B200_NPHASE] with the number of timed launches. */
#define SRM_B200_NPHASE 4 /* 0 grid rebuild, 1 sweep (migrate), 2 near lists, 3 reduction */
int srm_b200_timing_enable(srm_b200_ctx* ctx, int enable);
int srm_b200_timing_get(srm_b200_ctx* ctx, double* ms, int64_t* calls);
/* device sync + last-error check */
int srm_b200_sync(srm_b200_ctx* ctx);
/* CUDA-event stopwatch on the context stream: op 0 records the start event, op 1
 * records the stop event, waits for it and writes the elapsed device milliseconds. */
int srm_b200_stopwatch(srm_b200_ctx* ctx, int op, double* ms);
/* Diagnostics of the last round whose statistics were read: info[0] non-movers,
 * [1] colour classes of the sweep, [2] largest cells per class, [3] near-search half
 * width (x), [4] colouring modulus (x), [5] cells of the grid, [6] / [7] wavefront sweep
 * dependency rows found unfinished / polls spent on them (0 without the wavefront sweep),
 * [8] platelets: ordered pair tests (spherodisk_overlap) of the round's sweep and reduction.
 * info must hold 9 entries. */
int srm_b200_last_round_info(srm_b200_ctx* ctx, int64_t* info);

/* ---- self tests of the device primitives (no reference counterpart) ------------------ */
/* the hand-written device Philox4x32-10 next to CUDA's curand_Philox4x32_10 */
int srm_b200_selftest_philox(int64_t n, const uint32_t* ctr, const uint32_t* key,
                             uint32_t* out_mine, uint32_t* out_curand);
/* device unit vectors for bit-exact comparison with the oracle */
int srm_b200_selftest_unit_vectors(int dim, uint64_t seed, int64_t n, const uint32_t* slot,
                                   const uint32_t* attempt, uint32_t stream, uint32_t round_id,
                                   uint32_t iteration, double* out);

#ifdef __cplusplus
}
#endif
#endif
