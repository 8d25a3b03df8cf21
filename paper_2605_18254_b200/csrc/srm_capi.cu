// srm_capi.cu -- context, C ABI and the SRM control loop of libsrm_b200.so.
//
// See include/srm_b200.h for the contract of every entry point and the reference
// interface it replaces.  Device data layout: DESIGN.md §2.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <exception>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/srm_b200.h"
#include "srm_descriptors.cuh"
#include "srm_rsa_device.cuh"
#include "srm_kernels.cuh"

using namespace srmb;



namespace {

thread_local std::string g_create_error;

struct CudaError {
    std::string msg;
};
struct Invalid {
    std::string msg;
};

#define SRM_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw CudaError{std::string(#call) + ": " + cudaGetErrorString(e_)};           \
    } while (0)

constexpr int kMaxPhases = 254;  // acc[] encodes the phase of acceptance in a byte

int blocks_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 2147483647) b = 2147483647;
    return static_cast<int>(b);
}

template <typename T>
T* dalloc(int64_t count) {
    void* p = nullptr;
    if (count < 1) count = 1;
    SRM_CUDA(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(count)));
    return static_cast<T*>(p);
}

template <typename T>
struct DevBuf {  // device scratch of one call
    T* p = nullptr;
    explicit DevBuf(int64_t count) { p = dalloc<T>(count > 0 ? count : 1); }
    ~DevBuf() { cudaFree(p); }
};

}  // namespace

struct srm_b200_ctx {
    int dim = 3;
    int shape = 0;
    double c_r = 0.0;  // rotation angle of platelet moves (srm_b200_set_rotation / params.c_r)
    int device = 0;
    Box box{};
    int64_t cap = 0;
    int64_t n = 0;
    cudaStream_t stream = nullptr;
    std::string err;

    State P{}, Q{}, S{};
    uint32_t* key = nullptr;
    uint32_t* skey = nullptr;
    int32_t* perm = nullptr;             // scratch (remap, accept flags by slot)
    unsigned long long* perm64 = nullptr;  // grid build: slot << 32 | source index, cell-sorted
    int32_t* active = nullptr;  // non-mover list of the current round
    int32_t* nbr = nullptr;     // near-list rows (kNearRow int32 per particle)
    NearPool pool{nullptr, 0};  // near-list overflow pool
    int queue_ctas = 148 * 8;  // resident CTAs of k_sweep_warpq (set in init)
    std::vector<int64_t> cls_cells_h;  // cells before each colour class (launch sizes)
    // near-list kernel choice (SRM_B200_NEAR): 0 the shared-memory bricks where they apply
    // (GridParams::near_kind), otherwise the per-particle full stencil
    int near_mode = std::getenv("SRM_B200_NEAR") ? std::atoi(std::getenv("SRM_B200_NEAR")) : 0;
    // wavefront sweep (k_sweep_wave) where the grid allows it; SRM_B200_WAVE=0: class launches
    // (tuning: SRM_B200_WAVE=1:ly:lz sets the wave lags, GridParams::wave_lag_*)
    int wave_mode = [] {
        const char* v = std::getenv("SRM_B200_WAVE");
        if (!v) return 1;  // (the grid marks where the wave can run; wave_default picks it)
        int on = 1, ly = 0, lz = 0;
        std::sscanf(v, "%d:%d:%d", &on, &ly, &lz);
        return (on ? 1 : 0) | (std::min(std::max(ly, 0), 255) << 8) | (std::min(std::max(lz, 0), 255) << 16);
    }() | resolve_bits();
    // dependency resolution (srm_resolve.cuh) on sparse 3D sphere grids: SRM_B200_RESOLVE=1,
    // or SRM_B200_SWEEP=resolve (also on small grids, which otherwise take the trial teams)
    static int resolve_bits() {
        const char* f = std::getenv("SRM_B200_SWEEP");
        const char* w = std::getenv("SRM_B200_WAVE");
        const char* r = std::getenv("SRM_B200_RESOLVE");
        if (f && *f) return std::string(f) == "resolve" ? 6 : 0;
        if (w && std::atoi(w) != 0) return 0;
        return r && std::atoi(r) != 0 ? 2 : 0;  // opt-in: measured slower than the class launches
    }
    double4* rec2 = nullptr;     // resolve: the round's new records (exchanged with S.rec)
    uint8_t* dflag = nullptr;    // resolve: the pass that decided a particle
    int32_t* list_a = nullptr;   // resolve: pending lists (ping-pong)
    int32_t* list_b = nullptr;
    int32_t* seg_cnt = nullptr;  // resolve: entries per CTA segment of the pending lists (ping-pong)
    int2* rev = nullptr;         // half-stencil bricks: reverse entries (j, i) of a round
    int64_t rev_cap = 0;
    int32_t* ovf = nullptr;      // ... rows to rebuild from the full stencil
    static constexpr int resolve_ctas = kResolveMaxCtas;
    // opt-in (SRM_B200_WAVE=1 or SRM_B200_SWEEP=wave): measured no faster than the class
    // launches at cfg 4, so the class launches stay the default
    bool wave_default = [] {
        const char* v = std::getenv("SRM_B200_WAVE");
        return v && std::atoi(v) != 0;
    }();
    // unset: the wave on grids whose classes hold at most kWaveAutoLanes cells per resident
    // lane, where class launches run short of work and end in long tails (sweep per round at
    // cfg 4's density: 2 10^6 spheres 0.35 ms against 0.70 ms, 4 10^6 0.40 against 0.44; cfg 2
    // 0.41 against 0.48; at 10^7 the class launches win, 0.75 against 0.81: DESIGN.md §3.6)
    bool wave_auto = std::getenv("SRM_B200_WAVE") == nullptr;
    bool wave_fits(int64_t cells_per_class) const {
        return cells_per_class <= static_cast<int64_t>(kWaveAutoLanes) * queue_ctas * kSweepThreads;
    }
    static constexpr int kWaveAutoLanes = 6;
    WaveCtl* wave_ctl = nullptr;
    int32_t* wave_order = nullptr;  // rows in wave order (cell_cap entries)
    unsigned* wave_done = nullptr;  // per row: the epoch of the sweep that finished it
    // srm_generate: the device-resident graph loop (default) or the host-driven loop
    bool device_loop = std::getenv("SRM_B200_HOST_LOOP") == nullptr;
    uint8_t* acc = nullptr;

    uint32_t* count = nullptr;
    cell_t* cell_start = nullptr;
    uint64_t* partial = nullptr;
    int64_t cell_cap = 0;
    int64_t tile_cap = 0;

    GridParams* gp = nullptr;
    RoundParams* rp = nullptr;
    StatsDev* stats = nullptr;
    double* red_part_sum = nullptr;
    double* red_part_max = nullptr;
    double* red_out = nullptr;

    StatsDev* h_stats = nullptr;  // pinned
    double* h_red = nullptr;      // pinned [2]

    char* rec_stage = nullptr;
    size_t rec_stage_bytes = 0;

    int64_t launches = 0;

    bool timing = false;
    bool capturing = false;  // inside a graph capture: no timing events, no host syncs
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Pending {
        int fam;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
    double ms[SRM_B200_NPHASE] = {0, 0, 0, 0};
    int64_t calls[SRM_B200_NPHASE] = {0, 0, 0, 0};

    GridParams hg{};  // host copy of the grid currently in gp
    bool hg_set = false;

    cudaEvent_t sw_start = nullptr, sw_stop = nullptr;  // srm_b200_stopwatch
    int64_t last_nonmovers = 0;
    int64_t last_wave_waits = 0, last_wave_polls = 0, last_pair_tests = 0;

    // ---------------------------------------------------------------------------
    cudaEvent_t take_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            SRM_CUDA(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }
    struct FamScope {
        srm_b200_ctx* c;
        int fam;
        cudaEvent_t a = nullptr;
        FamScope(srm_b200_ctx* c_, int f) : c(c_), fam(f) {
            if (c->timing && !c->capturing) {
                a = c->take_event();
                SRM_CUDA(cudaEventRecord(a, c->stream));
            }
        }
        ~FamScope() {
            if (c->timing && a) {
                try {
                    cudaEvent_t b = c->take_event();
                    if (cudaEventRecord(b, c->stream) == cudaSuccess) c->pending.push_back({fam, a, b});
                } catch (...) {
                }
            }
        }
    };
    void harvest_timing() {
        if (pending.empty()) return;
        for (auto& p : pending) {
            float t = 0.f;
            SRM_CUDA(cudaEventSynchronize(p.b));
            SRM_CUDA(cudaEventElapsedTime(&t, p.a, p.b));
            ms[p.fam] += t;
            calls[p.fam] += 1;
        }
        pending.clear();
        ev_used = 0;
    }
    void sync() {
        SRM_CUDA(cudaStreamSynchronize(stream));
        SRM_CUDA(cudaGetLastError());
        if (timing && ev_used > 4096) harvest_timing();
    }
    void launched(int k = 1) {
        launches += k;
        SRM_CUDA(cudaPeekAtLastError());
    }

    // ---------------------------------------------------------------------------
    bool platelets() const { return shape == SRM_B200_PLATELET; }
    // crowded sphere grids (the 4x4x4-brick near kind) take the team sweep
    // SRM_B200_SWEEP=lane|trials|team forces one sweep kernel (tests: every kernel is
    // exact on any grid, the choice is only a matter of speed); unset: by the grid
    int sweep_force = [] {
        const char* v = std::getenv("SRM_B200_SWEEP");
        if (!v) return 0;
        const std::string s(v);
        return s == "lane" ? 1 : (s == "trials" ? 2 : (s == "team" ? 3 : (s == "wave" ? 4 : (s == "resolve" ? 5 : 0))));
    }();
    // the wavefront sweep replaces the class launches of k_sweep_warpq (sparse sphere grids)
    bool use_wave(const GridParams& g, int64_t class_cells_total) const {
        if (platelets() || !g.wave) return false;
        if (sweep_force) return sweep_force == 4;
        if (sphere_team(g) || trial_team(g, class_cells_total)) return false;
        return wave_default || (wave_auto && wave_fits(class_cells_total / std::max(1, g.ncls)));
    }
    // dependency resolution replaces the near-list kernel + class launches (the grid says where)
    bool use_resolve(const GridParams& g) const { return !platelets() && dim == 3 && g.resolve; }
    static int resolve_passes(const GridParams& g) { return g.ncls > 8 ? 20 : 12; }
    bool sphere_team(const GridParams& g) const {
        if (sweep_force) return sweep_force == 3 && dim == 3;
        return SRM_SPH_TEAM_ON && g.near_kind == 3;
    }
    // small grids (not crowded): a lane per cell would leave the GPU mostly idle; a
    // team per cell runs a particle's trials side by side (k_sweep_trials) while the
    // teams of a class launch still fit one wave of resident CTAs
    bool trial_team(const GridParams& g, int64_t class_cells_total) const {
        if (sweep_force) return sweep_force == 2;
        const int64_t per_class = class_cells_total / std::max(1, g.ncls);
        return SRM_TRIAL_TEAM_ON && g.near_kind != 3 && per_class * kTrialTeam <= 148LL * 8 * kSweepThreads;
    }
    void alloc_state(State& s) {
        s.rec = dalloc<double4>(cap);
        s.id = dalloc<int32_t>(cap);
        s.slot = dalloc<int32_t>(cap);
        if (platelets()) s.aux = dalloc<double4>(cap);
    }
    static void free_state(State& s) {
        cudaFree(s.rec);
        cudaFree(s.id);
        cudaFree(s.slot);
        cudaFree(s.aux);
    }
    // exchange the particle buffers of two states (the sorted state's fp32 copy stays)
    static void swap_state(State& a, State& b) {
        std::swap(a.rec, b.rec);
        std::swap(a.id, b.id);
        std::swap(a.slot, b.slot);
        std::swap(a.aux, b.aux);
    }

    void init() {
        SRM_CUDA(cudaSetDevice(device));
        SRM_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        if (platelets()) {  // spherodisk.cpp:60-66 rim seed angles 2 pi k / 32 through the host libm
            pl::SeedTable t;
            for (int k = 0; k < pl::kSeeds; ++k) {
                const double a = 2.0 * 3.141592653589793238462643383279502884 * k / pl::kSeeds;
                t.c[k] = std::cos(a);
                t.s[k] = std::sin(a);
            }
            SRM_CUDA(cudaMemcpyToSymbol(c_seed_table, &t, sizeof(t)));
        }
        if (platelets() || dim != 3) wave_mode &= ~6;  // (the dependency resolution: 3D spheres)
        alloc_state(P);
        alloc_state(Q);
        alloc_state(S);
        key = dalloc<uint32_t>(cap);
        skey = dalloc<uint32_t>(cap);
        perm = dalloc<int32_t>(cap);
        perm64 = dalloc<unsigned long long>(cap);
        acc = dalloc<uint8_t>(cap);
        gp = dalloc<GridParams>(1);
        rp = dalloc<RoundParams>(1);
        active = dalloc<int32_t>(cap);
        nbr = dalloc<int32_t>(cap * kNearRow);
        // crowded (polydisperse, platelet) states; offsets are int32 in the rows, so the
        // pool never exceeds 2^31 - 1 entries (a row that does not fit rescans its stencil)
        pool.cap = std::min<int64_t>(8 * cap + 32 * std::min<int64_t>(cap, 2000000), 2147483647LL);
        pool.e = dalloc<int32_t>(pool.cap);
        SRM_CUDA(cudaFuncSetAttribute(tiles::k_near_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(tiles::kTileSmem)));
        SRM_CUDA(cudaFuncSetAttribute(tiles::k_near_tiles, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        SRM_CUDA(cudaFuncSetAttribute(ctiles::k_near_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(ctiles::kTileSmem)));
        SRM_CUDA(cudaFuncSetAttribute(ctiles::k_near_tiles, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        {
            int per_sm = 0, sms = 0;
            SRM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_warpq<3>, kSweepThreads, 0));
            SRM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
            queue_ctas = std::max(1, per_sm) * std::max(1, sms);
        }
        S.xf = dalloc<float4>(cap);
#if SRM_NEAR_HALF
        if (dim == 3) {  // (expected: 0.35 reverse entries per particle at cfg 4's window, 0.9 at cfg 2's)
            rev_cap = 2 * cap + 1024;
            rev = dalloc<int2>(rev_cap);
            ovf = dalloc<int32_t>(cap + 1024);
        }
#endif
        if (!platelets() && dim == 3 && (wave_mode & 2)) {  // (the opt-in dependency resolution's buffers)
            rec2 = dalloc<double4>(cap);
            dflag = dalloc<uint8_t>(cap);
            // (a CTA's segment is its index range rounded up to whole chunks)
            list_a = dalloc<int32_t>(cap + static_cast<int64_t>(resolve_ctas) * kResolveThreads);
            list_b = dalloc<int32_t>(cap + static_cast<int64_t>(resolve_ctas) * kResolveThreads);
            seg_cnt = dalloc<int32_t>(2 * resolve_ctas);
            SRM_CUDA(cudaFuncSetAttribute(rtiles::k_near_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(rtiles::kTileSmem)));
            SRM_CUDA(cudaFuncSetAttribute(rtiles::k_near_tiles, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        }
        wave_ctl = dalloc<WaveCtl>(1);
        SRM_CUDA(cudaMemsetAsync(wave_ctl, 0, sizeof(WaveCtl), stream));
        stats = dalloc<StatsDev>(1);
        red_part_sum = dalloc<double>(kRedBlocks);
        red_part_max = dalloc<double>(kRedBlocks);
        red_out = dalloc<double>(2);
        SRM_CUDA(cudaMallocHost(&h_stats, sizeof(StatsDev)));
        SRM_CUDA(cudaMallocHost(&h_red, 2 * sizeof(double)));
    }

    ~srm_b200_ctx() {
        if (device >= 0) cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        free_state(P);
        free_state(Q);
        free_state(S);
        cudaFree(key); cudaFree(skey); cudaFree(perm); cudaFree(perm64); cudaFree(acc);
        cudaFree(count); cudaFree(cell_start); cudaFree(partial);
        cudaFree(gp); cudaFree(rp); cudaFree(active); cudaFree(stats); cudaFree(red_part_sum);
        cudaFree(nbr); cudaFree(pool.e); cudaFree(S.xf); cudaFree(wave_ctl); cudaFree(wave_order); cudaFree(wave_done);
        cudaFree(red_part_max); cudaFree(red_out); cudaFree(rec_stage);
        cudaFree(rec2); cudaFree(dflag); cudaFree(list_a); cudaFree(list_b); cudaFree(seg_cnt); cudaFree(rev); cudaFree(ovf);
        if (h_stats) cudaFreeHost(h_stats);
        if (h_red) cudaFreeHost(h_red);
        for (auto e : ev_pool) cudaEventDestroy(e);
        if (sw_start) cudaEventDestroy(sw_start);
        if (sw_stop) cudaEventDestroy(sw_stop);
        cudaFree(d_ctl);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (h_ring) cudaFreeHost(h_ring);
        if (h_ring_ctr) cudaFreeHost(h_ring_ctr);
        for (auto st : cap_streams)
            if (st) cudaStreamDestroy(st);
        if (stream) cudaStreamDestroy(stream);
    }

    // ---------------------------------------------------------------------------
    // CellGrid ctor (cell_grid.hpp:31-52) + the near-search stencil and the colouring
    // for a state whose largest radius is max_r_state and whose trial
    // moves have length c_m.  The colouring expression is the oracle's orc_colouring.
    GridParams make_grid(double cell_size, double max_r_state, double c_m) const {
        GridParams g{};
        const int st = grid_params(cell_size, max_r_state, c_m, box, dim, near_mode, &g, n, wave_mode);
        if (st == 1) throw Invalid{"CellGrid: cell_size must be positive"};
        if (st == 2) throw Invalid{"CellGrid: more than 2^32 cells (radius too small for the box)"};
        for (int a = 0; a < 3; ++a)
            for (const FastDiv& f : {g.fd_dims[a], g.fd_m[a]})  // cheap guard of the magic numbers
                for (uint32_t v : {0u, 1u, f.d - 1, f.d, f.d + 1, 2 * f.d + 1, 0x7fffffffu, 0xfffffffeu, 0xffffffffu})
                    if (fdiv(v, f) != v / f.d) throw std::logic_error("fast division self-check failed");
        return g;
    }

    void ensure_cells(int64_t ncells) {
        if (ncells <= cell_cap) return;
        cudaFree(count);
        cudaFree(cell_start);
        cudaFree(partial);
        cudaFree(wave_order);
        cudaFree(wave_done);
        count = nullptr; cell_start = nullptr; partial = nullptr; wave_order = nullptr; wave_done = nullptr;
        const int64_t c = ncells + ncells / 8 + 1024;
        count = dalloc<uint32_t>(c);
        cell_start = dalloc<cell_t>(c + 1);
        tile_cap = (c + kLbTile - 1) / kLbTile;
        partial = dalloc<uint64_t>(tile_cap + 1);  // look-back status words + the tile counter
        SRM_CUDA(cudaMemsetAsync(count, 0, sizeof(uint32_t) * c, stream));
        wave_order = dalloc<int32_t>(c);
        wave_done = dalloc<unsigned>(c);
        SRM_CUDA(cudaMemsetAsync(wave_done, 0, sizeof(unsigned) * c, stream));  // epochs start at 1
        cell_cap = c;
    }

    void set_grid(const GridParams& g) {
        ensure_cells(g.ncells);
        // cells per colour class: on each axis a body colour v < m has
        // floor(n / m) cells, a remainder colour one (sweep launch sizes)
        std::vector<int64_t> off(static_cast<size_t>(g.ncls) + 1, 0);
        for (int64_t k = 0; k < g.ncls; ++k) {
            int64_t rem = k, cells = 1;
            for (int a = 0; a < 3; ++a) {
                const int64_t v = rem % g.col_n[a];
                rem /= g.col_n[a];
                cells *= v < g.col_m[a] ? g.dims[a] / g.col_m[a] : 1;
            }
            off[k + 1] = off[k] + cells;
        }
        if (off[g.ncls] != g.ncells) throw std::logic_error("colour classes do not tile the grid");
        cls_cells_h.assign(off.begin(), off.end());
        k_set_grid<<<1, 1, 0, stream>>>(gp, g);
        launched();
        hg = g;
        hg_set = true;
    }

    void set_round(double c_m, int n_l, uint64_t seed, uint32_t round_id, uint32_t iteration, bool write_acc) {
        RoundParams v{};
        v.c_m = c_m;
        v.n_l = n_l;
        v.write_acc = write_acc ? 1 : 0;
        v.key.k0 = static_cast<uint32_t>(seed);
        v.key.k1 = static_cast<uint32_t>(seed >> 32);
        v.key.round_id = round_id & 0xFFFFFFu;
        v.key.iteration = iteration;
        v.cos_r = std::cos(c_r);  // spherodisk.hpp:50-51, host libm as the reference
        v.sin_r = std::sin(c_r);
        k_set_round<<<1, 1, 0, stream>>>(rp, v);
        launched();
    }

    // grid rebuild T -> S (sorted) + skey; gp must be set
    // ncells_bound: launch sizes for at least that many cells (graph capture: the largest
    // grid of the run; every kernel reads the actual grid from gp)
    void grid_build(State& T, int64_t ncells_bound = -1) {
        FamScope fs(this, 0);
        const int64_t nc = ncells_bound >= 0 ? ncells_bound : hg.ncells;
        const int nb = blocks_for(n, 256);
        const int cb = static_cast<int>(std::min<int64_t>(blocks_for(nc, 256), 148 * 64));
        if (dim == 2) k_keys<2><<<nb, 256, 0, stream>>>(n, T, gp, key, count);
        else k_keys<3><<<nb, 256, 0, stream>>>(n, T, gp, key, count);
        const int tiles = static_cast<int>((nc + kLbTile - 1) / kLbTile);
        SRM_CUDA(cudaMemsetAsync(partial, 0, sizeof(uint64_t) * (tiles + 1), stream));
        k_scan_lookback<<<tiles, kLbThreads, 0, stream>>>(count, gp, reinterpret_cast<unsigned long long*>(partial),
                                                         cell_start);
        k_scatter<<<nb, 256, 0, stream>>>(n, key, T.slot, cell_start, count, perm64);
        k_cellsort<<<cb, 256, 0, stream>>>(gp, cell_start, perm64);
        if (dim == 2) k_gather<2><<<nb, 256, 0, stream>>>(n, perm64, key, T, S, skey);
        else k_gather<3><<<nb, 256, 0, stream>>>(n, perm64, key, T, S, skey);
        launched(5);
    }

    void copy_state(State& A, State& B) {
        if (dim == 2) k_copy_state<2><<<blocks_for(n, 256), 256, 0, stream>>>(n, A, B);
        else k_copy_state<3><<<blocks_for(n, 256), 256, 0, stream>>>(n, A, B);
        launched();
    }

    // near lists of a sparse 3D grid: the shared-memory bricks (half stencil: each pair once)
    // and the merge of their reverse entries (every kernel tests the grid: GridParams::near_kind)
    void sparse_bricks(int ntiles) {
#if SRM_NEAR_HALF
        tiles::k_near_tiles<<<ntiles, tiles::kTileThreads, tiles::kTileSmem, stream>>>(S, gp, cell_start, skey, nbr, pool,
                                                                                       stats, rev, rev_cap, ovf);
        const int mb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 8));
        k_near_merge<<<mb, 256, 0, stream>>>(gp, rev, rev_cap, nbr, ovf, stats);
        k_near_rebuild<<<148, 128, 0, stream>>>(S, gp, cell_start, skey, nbr, pool, ovf, stats);
        launched(3);
#else
        tiles::k_near_tiles<<<ntiles, tiles::kTileThreads, tiles::kTileSmem, stream>>>(S, gp, cell_start, skey, nbr, pool,
                                                                                       stats);
        launched(1);
#endif
    }

    // passes 1 .. of the dependency resolution (srm_resolve.cuh); the last one finishes
    // whatever is left
    void resolve_passes_launch(const GridParams& g) {
        const int np = resolve_passes(g);
        // one contiguous range of particle indices per CTA, all CTAs resident
        const int grid = static_cast<int>(std::min<int64_t>(blocks_for(n, kResolveThreads), resolve_ctas));
        int64_t span = (n + grid - 1) / grid;
        span = (span + kResolveThreads - 1) / kResolveThreads * kResolveThreads;
        for (int pass = 1; pass <= np; ++pass)
            k_resolve_pass<3><<<grid, kResolveThreads, 0, stream>>>(pass, pass == np ? 1 : 0, n, span, S, rec2, dflag, box, gp,
                                                                    rp, cell_start, skey, nbr, pool.e, acc, active, list_a,
                                                                    list_b, seg_cnt, stats);
        launched(np);
    }

    // One round on T (T is rewritten in this round's sorted order); gp must be set.
    // grid rebuild, near lists, then the coloured Gauss-Seidel sweep (one launch per
    // colour class), then the overlap reduction (non-movers; all pairs for platelets).
    void round(State& T, double c_m, int n_l, uint64_t seed, uint32_t round_id, uint32_t iteration,
               bool with_stats, bool with_candidates, bool write_acc = false) {
        if (n_l > kMaxPhases) throw Invalid{"n_l > 254 is not supported by the B200 path"};
        set_round(c_m, n_l, seed, round_id, iteration, write_acc);
        grid_build(T);
        SRM_CUDA(cudaMemsetAsync(stats, 0, sizeof(StatsDev), stream));
        if (write_acc) SRM_CUDA(cudaMemsetAsync(acc, kNotAccepted, static_cast<size_t>(n), stream));
        const bool resolve = use_resolve(hg);
        if (resolve) {
            {  // pass 0: near lists + first trials + the particles nothing precedes
                FamScope fs(this, 2);
                rtiles::k_near_tiles<<<hg.ntiles, rtiles::kTileThreads, rtiles::kTileSmem, stream>>>(
                    S, gp, cell_start, skey, nbr, pool, stats, box, rp, rec2, dflag, acc);
                launched(1);
            }
            FamScope fs(this, 1);
            resolve_passes_launch(hg);
            std::swap(S.rec, rec2);  // the new records are the sorted state's
        } else {
            FamScope fs(this, 2);  // near lists
            const int nb = blocks_for(n, 256);
            if (hg.near_kind == 0) {  // shared-memory bricks
                sparse_bricks(hg.ntiles);
            } else if (hg.near_kind == 3) {  // crowded: small bricks, large staging
                ctiles::k_near_tiles<<<hg.ntiles, ctiles::kTileThreads, ctiles::kTileSmem, stream>>>(
                    S, gp, cell_start, skey, nbr, pool, stats);
                launched(1);
            } else {
                if (dim == 2) k_near_lists<2><<<nb, 256, 0, stream>>>(n, S, gp, cell_start, skey, nbr, pool, stats);
                else k_near_lists<3><<<nb, 256, 0, stream>>>(n, S, gp, cell_start, skey, nbr, pool, stats);
                launched(1);
            }
        }
        if (resolve) {
        } else if (use_wave(hg, cls_cells_h[hg.ncls] - cls_cells_h[0])) {  // one persistent launch
            FamScope fs(this, 1);
            k_wave_order<<<1, kWaveOrderThreads, 0, stream>>>(gp, wave_ctl, wave_order);
            if (dim == 2)
                k_sweep_wave<2><<<queue_ctas, kSweepThreads, 0, stream>>>(S, box, gp, rp, cell_start, skey, nbr, pool.e, acc,
                                                                          active, stats, wave_ctl, wave_order, wave_done);
            else
                k_sweep_wave<3><<<queue_ctas, kSweepThreads, 0, stream>>>(S, box, gp, rp, cell_start, skey, nbr, pool.e, acc,
                                                                          active, stats, wave_ctl, wave_order, wave_done);
            launched(2);
        } else {
            FamScope fs(this, 1);
            for (int cls = 0; cls < hg.ncls; ++cls) {
                const int64_t cells = cls_cells_h[cls + 1] - cls_cells_h[cls];
                // a cell per lane (the cells of a class are its parallelism: a cell's
                // particles are visited in order), at most one wave of resident CTAs
                const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks_for(cells, kSweepThreads), queue_ctas)));
                const int tgrid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(
                    blocks_for(cells * kTrialTeam, kSweepThreads), 148 * 32)));
                if (!platelets() && trial_team(hg, cls_cells_h[hg.ncls] - cls_cells_h[0])) {
                    if (dim == 2)
                        k_sweep_trials<2><<<tgrid, kSweepThreads, 0, stream>>>(cls, nullptr, S, box, gp, rp, cell_start, skey, nbr,
                                                                               pool.e, acc, active, stats);
                    else
                        k_sweep_trials<3><<<tgrid, kSweepThreads, 0, stream>>>(cls, nullptr, S, box, gp, rp, cell_start, skey, nbr,
                                                                               pool.e, acc, active, stats);
                } else if (dim == 2)
                    k_sweep_warpq<2><<<grid, kSweepThreads, 0, stream>>>(cls, nullptr, S, box, gp, rp, cell_start, skey, nbr, pool.e, acc,
                                                                         active, stats);
                else if (platelets())
                    k_sweep_pl_team<<<static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(
                                          blocks_for(cells * kPlTeam, kSweepThreads), 148 * 32))),
                                      kSweepThreads, 0, stream>>>(cls, nullptr, S, box, gp, rp, cell_start, skey, nbr, pool.e, acc,
                                                                  active, stats);
                else if (sphere_team(hg))
                    k_sweep_team<<<static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(
                                       blocks_for(cells * kSphTeam, kSweepThreads), 148 * 32))),
                                   kSweepThreads, 0, stream>>>(cls, nullptr, S, box, gp, rp, cell_start, skey, nbr, pool.e, acc,
                                                               active, stats);
                else
                    k_sweep_warpq<3><<<grid, kSweepThreads, 0, stream>>>(cls, nullptr, S, box, gp, rp, cell_start, skey, nbr, pool.e, acc,
                                                                         active, stats);
            }
            launched(hg.ncls);
        }
        if (with_stats) {
            FamScope fs(this, 3);
            const int lb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 8));
            if (platelets())
                k_overlap_pl<<<blocks_for(n * 32, kOverlapPlThreads), kOverlapPlThreads, 0, stream>>>(n, S, box, gp, cell_start, skey, stats);
            else if (dim == 2)
                k_stats_sweep<2><<<lb, 256, 0, stream>>>(S, box, gp, cell_start, skey, acc, active, stats);
            else
                k_stats_sweep<3><<<lb, 256, 0, stream>>>(S, box, gp, cell_start, skey, acc, active, stats);
            launched();
            if (with_candidates) {
                const int nb = blocks_for(n, 256);
                if (dim == 2) k_candidates<2><<<nb, 256, 0, stream>>>(n, gp, cell_start, skey, stats);
                else k_candidates<3><<<nb, 256, 0, stream>>>(n, gp, cell_start, skey, stats);
                launched();
            }
        }
        // the sweep updated the sorted state in place: it is the round's output
        swap_state(T, S);
    }

    // ---------------------------------------------------------------------------
    // Device-resident srm_generate: one CUDA graph, conditional nodes.
    //   WHILE(run) { k_gen_step; IF(active) { IF(copy) P->Q; IF(scale) Q *= factor;
    //     round on Q (grid build, near lists, WHILE(cls) sweep class, stats, S->Q);
    //     k_gen_after; IF(commit) Q->P; IF(f) volume fraction; IF(reorder) reorder P };
    //     k_gen_end }
    static cudaGraph_t add_conditional(cudaStream_t st, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
        cudaStreamCaptureStatus cst;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        cudaGraph_t g = nullptr;
        SRM_CUDA(cudaStreamGetCaptureInfo(st, &cst, nullptr, &g, &deps, &ndeps));
        cudaGraphNodeParams np{};
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = type;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        SRM_CUDA(cudaGraphAddNode(&node, g, deps, ndeps, &np));
        SRM_CUDA(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
        return np.conditional.phGraph_out[0];
    }
    static cudaGraphConditionalHandle new_handle(cudaStream_t st, unsigned dflt) {
        cudaStreamCaptureStatus cst;
        cudaGraph_t g = nullptr;
        SRM_CUDA(cudaStreamGetCaptureInfo(st, &cst, nullptr, &g, nullptr, nullptr));
        cudaGraphConditionalHandle h;
        SRM_CUDA(cudaGraphConditionalHandleCreate(&h, g, dflt, cudaGraphCondAssignDefault));
        return h;
    }
    // capture `body` into the (empty) graph `g` on stream st (which becomes `stream` meanwhile)
    template <typename F>
    void capture_into(cudaGraph_t g, cudaStream_t st, F&& body) {
        SRM_CUDA(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        cudaStream_t saved = stream;
        stream = st;
        body();
        stream = saved;
        cudaGraph_t out = nullptr;
        SRM_CUDA(cudaStreamEndCapture(st, &out));
    }

    GenCtl* d_ctl = nullptr;
    // live progress ring (pinned, host-mapped): records, published and consumed counters
    static constexpr int64_t kRing = 4096;
    GenProgress* h_ring = nullptr;
    int64_t* h_ring_ctr = nullptr;  // [0] published, [2] run start (device writes), [1] consumed (host writes)
    cudaStream_t cap_streams[4] = {nullptr, nullptr, nullptr, nullptr};
    // the instantiated generate graph, reused while everything baked into it is unchanged
    struct GraphKey {
        int64_t n, nc_max;
        int ntiles_max, ctiles_max, team0, trials0, queue_ctas, dim, plate, wave0, resolve0, resolve_np;
        const void* bufs[18];
        bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(GraphKey)) == 0; }
    };
    GraphKey gkey{};
    cudaGraphExec_t gexec = nullptr;
    int64_t graph_builds = 0;

    // Launch the generate graph and, with a progress sink, deliver the iteration records
    // while it runs (engine.hpp:251-254): poll the published counter of the mapped ring,
    // hand each record to the sink, report the consumed position back to the device.
    void launch_and_drain(const GenCtl& hc, srm_b200_progress_fn progress, void* user) {
        SRM_CUDA(cudaGraphLaunch(gexec, stream));
        if (!progress) {
            SRM_CUDA(cudaStreamSynchronize(stream));
            SRM_CUDA(cudaGetLastError());
            return;
        }
        volatile int64_t* ctr = reinterpret_cast<volatile int64_t*>(h_ring_ctr);
        int64_t consumed = 0;
        std::exception_ptr sink_error;
        for (;;) {
            const cudaError_t q = cudaStreamQuery(stream);
            if (q != cudaSuccess && q != cudaErrorNotReady) SRM_CUDA(q);
            const int64_t pub = ctr[0];
            std::atomic_thread_fence(std::memory_order_acquire);
            const uint64_t t0 = static_cast<uint64_t>(ctr[2]);  // the run's start (k_gen_t0)
            while (consumed < pub) {
                GenProgress r;
                std::memcpy(&r, const_cast<const GenProgress*>(h_ring + consumed % kRing), sizeof r);
                srm_b200_progress_record rec{r.iteration, r.volume_fraction, r.accepted, (r.t_ns - t0) * 1e-9, r.rounds};
                if (!sink_error) {
                    try {
                        progress(&rec, user);
                    } catch (...) {  // keep draining (the device may wait on the ring), rethrow after the run
                        sink_error = std::current_exception();
                    }
                }
                ++consumed;
                std::atomic_thread_fence(std::memory_order_release);
                ctr[1] = consumed;
            }
            if (q == cudaSuccess && consumed == ctr[0]) break;
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
        (void)hc;
        if (sink_error) std::rethrow_exception(sink_error);
    }

    // returns status; out counters filled from the controller
    int generate_graph(const srm_b200_params& p, int64_t it0, double f0, double max_r0, int64_t* done_out,
                       int64_t* acc_out, int64_t* rounds_out, int64_t* shakes_out, double* f_out,
                       srm_b200_progress_fn progress, void* user) {
        if (!d_ctl) d_ctl = dalloc<GenCtl>(1);
        GenProgress* d_ring = nullptr;
        int64_t* d_ctr = nullptr;
        if (progress) {
            if (!h_ring) {
                SRM_CUDA(cudaHostAlloc(&h_ring, sizeof(GenProgress) * kRing, cudaHostAllocMapped));
                SRM_CUDA(cudaHostAlloc(&h_ring_ctr, 3 * sizeof(int64_t), cudaHostAllocMapped));
            }
            SRM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_ring), h_ring, 0));
            SRM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_ctr), h_ring_ctr, 0));
            reinterpret_cast<volatile int64_t*>(h_ring_ctr)[0] = 0;
            reinterpret_cast<volatile int64_t*>(h_ring_ctr)[1] = 0;
        }
        for (auto& st : cap_streams)
            if (!st) SRM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        GenCtl hc{};
        hc.f_target = p.f_target;
        hc.stop = p.f_target * (1.0 - 1e-12);
        hc.c_w = p.c_w;
        hc.c_m = p.c_m;
        hc.box_measure = box_measure();
        hc.max_iter = p.max_iterations;
        hc.recs_cap = kRing;
        hc.pub = d_ctr;
        hc.cons = d_ctr ? d_ctr + 1 : nullptr;
        hc.it0 = it0;
        hc.n_k = p.n_k;
        hc.n_l = p.n_l;
        hc.reorder_period = p.reorder_period;
        hc.dim = dim;
        hc.near_mode = near_mode;
        hc.wave_mode = wave_mode;
        hc.n = n;
        hc.seed = p.seed;
        hc.cos_r = std::cos(p.c_r);
        hc.sin_r = std::sin(p.c_r);
        hc.f = f0;
        hc.max_r = max_r0;
        hc.recs = d_ring;
        // the largest grid of the run is the first one (radii only grow): launch bounds
        const GridParams g0 = make_grid(2.5 * max_r0 + p.c_m, max_r0, p.c_m);
        ensure_cells(g0.ncells);
        const int64_t nc_max = g0.ncells;
        // (brick count of the first grid, whether or not it takes the bricks: a later grid
        // of the run may, and its dims are no larger)
        const int ntiles_max = dim == 3 ? ((g0.dims[0] + kTX - 1) / kTX) * ((g0.dims[1] + kTY - 1) / kTY) *
                                              ((g0.dims[2] + kTZ - 1) / kTZ)
                                        : 1;
        const int ctiles_max = dim == 3 ? ((g0.dims[0] + kCTX - 1) / kCTX) * ((g0.dims[1] + kCTY - 1) / kCTY) *
                                              ((g0.dims[2] + kCTZ - 1) / kCTZ)
                                        : 1;
        const bool team0 = dim == 3 && !platelets() && sphere_team(g0);
        const bool trials0 = !platelets() && trial_team(g0, g0.ncells);
        // the wavefront sweep where a round's grid allows it (the kernels test the grid);
        // the class loop below runs otherwise
        const bool wave0 = !platelets() && !team0 && !trials0 &&
                           (sweep_force == 4 || (sweep_force == 0 && (wave_default || (wave_auto && wave_fits(g0.ncells / std::max(1, g0.ncls))))));
        // dependency resolution: captured whenever this context allows it; the grid of each
        // round (GridParams::resolve, set on the device) says whether it runs
        const bool resolve0 = !platelets() && dim == 3 && (wave_mode & 2) != 0;
        SRM_CUDA(cudaMemcpyAsync(d_ctl, &hc, sizeof(GenCtl), cudaMemcpyHostToDevice, stream));
        SRM_CUDA(cudaStreamSynchronize(stream));  // hc is a stack object

        GraphKey key{};
        key.n = n;
        key.nc_max = nc_max;
        key.ntiles_max = ntiles_max;
        key.ctiles_max = ctiles_max;
        key.team0 = team0;
        key.trials0 = trials0;
        key.queue_ctas = queue_ctas;
        key.dim = dim;
        key.plate = platelets();
        key.wave0 = wave0;
        key.resolve0 = resolve0;
        key.resolve_np = resolve_passes(g0);
        const void* bufs[18] = {P.rec, Q.rec, S.rec, P.aux, Q.aux, S.aux, count, cell_start, perm64, nbr, pool.e, S.xf,
                                wave_order, wave_done, rec2, dflag, list_a, list_b};
        (void)rev;  // (allocated with S.xf: the same lifetime)
        (void)seg_cnt;  // (allocated with list_a: the same lifetime)
        std::memcpy(key.bufs, bufs, sizeof bufs);
        if (gexec && key == gkey) {
            launch_and_drain(hc, progress, user);
        } else {
        if (gexec) {
            cudaGraphExecDestroy(gexec);
            gexec = nullptr;
        }
        cudaGraph_t G;
        SRM_CUDA(cudaGraphCreate(&G, 0));
        capturing = true;
        GenCtl* ctl = d_ctl;
        const int nb = blocks_for(n, 256);
        capture_into(G, cap_streams[0], [&]() {
            const cudaGraphConditionalHandle h_run = new_handle(stream, 1);
            k_gen_t0<<<1, 1, 0, stream>>>(ctl);
            cudaGraph_t B = add_conditional(stream, h_run, cudaGraphCondTypeWhile);
            capture_into(B, cap_streams[1], [&]() {
                const cudaGraphConditionalHandle h_active = new_handle(stream, 0);
                k_gen_step<<<1, 1, 0, stream>>>(ctl, gp, rp, stats, box, h_active);
                cudaGraph_t A = add_conditional(stream, h_active, cudaGraphCondTypeIf);
                capture_into(A, cap_streams[2], [&]() {
                    const cudaGraphConditionalHandle h_copy = new_handle(stream, 0), h_scale = new_handle(stream, 0);
                    const cudaGraphConditionalHandle h_cls = new_handle(stream, 0), h_commit = new_handle(stream, 0);
                    const cudaGraphConditionalHandle h_f = new_handle(stream, 0), h_reorder = new_handle(stream, 0);
                    k_gen_flags<<<1, 1, 0, stream>>>(ctl, h_copy, h_scale);
                    capture_into(add_conditional(stream, h_copy, cudaGraphCondTypeIf), cap_streams[3],
                                 [&]() { copy_state(P, Q); });
                    capture_into(add_conditional(stream, h_scale, cudaGraphCondTypeIf), cap_streams[3], [&]() {
                        k_scale_radius_ctl<<<nb, 256, 0, stream>>>(n, Q.rec, Q.aux, ctl);
                    });
                    // one round on Q
                    grid_build(Q, nc_max);
                    sparse_bricks(ntiles_max);
                    ctiles::k_near_tiles<<<ctiles_max, ctiles::kTileThreads, ctiles::kTileSmem, stream>>>(
                        S, gp, cell_start, skey, nbr, pool, stats);
                    if (dim == 2) k_near_lists<2><<<nb, 256, 0, stream>>>(n, S, gp, cell_start, skey, nbr, pool, stats);
                    else k_near_lists<3><<<nb, 256, 0, stream>>>(n, S, gp, cell_start, skey, nbr, pool, stats);
                    if (resolve0) {  // (each kernel tests the round's grid: GridParams::resolve)
                        rtiles::k_near_tiles<<<ntiles_max, rtiles::kTileThreads, rtiles::kTileSmem, stream>>>(
                            S, gp, cell_start, skey, nbr, pool, stats, box, rp, rec2, dflag, acc);
                        resolve_passes_launch(g0);
                    }
                    if (wave0) {
                        k_wave_order<<<1, kWaveOrderThreads, 0, stream>>>(gp, wave_ctl, wave_order);
                        if (dim == 2)
                            k_sweep_wave<2><<<queue_ctas, kSweepThreads, 0, stream>>>(S, box, gp, rp, cell_start, skey, nbr,
                                                                                      pool.e, acc, active, stats, wave_ctl,
                                                                                      wave_order, wave_done);
                        else
                            k_sweep_wave<3><<<queue_ctas, kSweepThreads, 0, stream>>>(S, box, gp, rp, cell_start, skey, nbr,
                                                                                      pool.e, acc, active, stats, wave_ctl,
                                                                                      wave_order, wave_done);
                    }
                    k_gen_cls_begin<<<1, 1, 0, stream>>>(ctl, gp, h_cls, wave0 ? 1 : 0);
                    capture_into(add_conditional(stream, h_cls, cudaGraphCondTypeWhile), cap_streams[3], [&]() {
                        if (trials0 && dim == 2)
                            k_sweep_trials<2><<<148 * 32, kSweepThreads, 0, stream>>>(0, &ctl->cls, S, box, gp, rp, cell_start,
                                                                                        skey, nbr, pool.e, acc, active, stats);
                        else if (trials0)
                            k_sweep_trials<3><<<148 * 32, kSweepThreads, 0, stream>>>(0, &ctl->cls, S, box, gp, rp, cell_start,
                                                                                        skey, nbr, pool.e, acc, active, stats);
                        else if (dim == 2)
                            k_sweep_warpq<2><<<queue_ctas, kSweepThreads, 0, stream>>>(0, &ctl->cls, S, box, gp, rp, cell_start,
                                                                                       skey, nbr, pool.e, acc, active, stats);
                        else if (platelets())
                            k_sweep_pl_team<<<148 * 32, kSweepThreads, 0, stream>>>(0, &ctl->cls, S, box, gp, rp,
                                                                                             cell_start, skey, nbr, pool.e, acc, active,
                                                                                             stats);
                        else if (team0)  // (the first grid's kind decides for the run; either is exact)
                            k_sweep_team<<<148 * 32, kSweepThreads, 0, stream>>>(0, &ctl->cls, S, box, gp, rp, cell_start,
                                                                                  skey, nbr, pool.e, acc, active, stats);
                        else
                            k_sweep_warpq<3><<<queue_ctas, kSweepThreads, 0, stream>>>(0, &ctl->cls, S, box, gp, rp, cell_start,
                                                                                       skey, nbr, pool.e, acc, active, stats);
                        k_gen_cls_next<<<1, 1, 0, stream>>>(ctl, gp, h_cls);
                    });
                    const int lb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 8));
                    if (dim == 2) k_stats_sweep<2><<<lb, 256, 0, stream>>>(S, box, gp, cell_start, skey, acc, active, stats);
                    else if (platelets())
                        k_overlap_pl<<<blocks_for(n * 32, kOverlapPlThreads), kOverlapPlThreads, 0, stream>>>(n, S, box, gp, cell_start, skey, stats);
                    else k_stats_sweep<3><<<lb, 256, 0, stream>>>(S, box, gp, cell_start, skey, acc, active, stats, rec2);
                    if (resolve0) {  // the round's records are in rec2 when the resolution swept it
                        k_copy_state<3><<<nb, 256, 0, stream>>>(n, S, Q, gp, rec2);
                        launched();
                    } else {
                        copy_state(S, Q);
                    }
                    k_gen_after<<<1, 1, 0, stream>>>(ctl, stats, h_commit, h_f, h_reorder);
                    capture_into(add_conditional(stream, h_commit, cudaGraphCondTypeIf), cap_streams[3],
                                 [&]() { copy_state(Q, P); });
                    capture_into(add_conditional(stream, h_f, cudaGraphCondTypeIf), cap_streams[3], [&]() {
                        if (dim == 2) k_reduce_partials<2><<<kRedBlocks, 256, 0, stream>>>(n, P.rec, red_part_sum, red_part_max, P.aux);
                        else k_reduce_partials<3><<<kRedBlocks, 256, 0, stream>>>(n, P.rec, red_part_sum, red_part_max, P.aux);
                        k_reduce_final<<<1, 256, 0, stream>>>(red_part_sum, red_part_max, red_out);
                        k_gen_f<<<1, 1, 0, stream>>>(ctl, red_out);
                    });
                    capture_into(add_conditional(stream, h_reorder, cudaGraphCondTypeIf), cap_streams[3], [&]() {
                        k_gen_grid_iter<<<1, 1, 0, stream>>>(ctl, gp);
                        grid_build(P, nc_max);
                        SRM_CUDA(cudaMemcpyAsync(Q.slot, S.slot, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, stream));
                        k_assign_slots<<<nb, 256, 0, stream>>>(n, S, nullptr, Q.slot);
                        copy_state(S, P);
                    });
                });
                k_gen_end<<<1, 1, 0, stream>>>(ctl, h_run);
            });
        });
        capturing = false;
        SRM_CUDA(cudaGraphInstantiate(&gexec, G, 0));
        cudaGraphDestroy(G);
        gkey = key;
        ++graph_builds;
        launch_and_drain(hc, progress, user);
        }
        SRM_CUDA(cudaMemcpy(&hc, d_ctl, sizeof(GenCtl), cudaMemcpyDeviceToHost));
        *done_out = hc.done;
        *acc_out = hc.accepted;
        *rounds_out = hc.rounds;
        *shakes_out = hc.shakes;
        *f_out = hc.f;
        if (hc.status == 2) throw Invalid{"CellGrid: cell_size below safety bound 2*maxR + slack"};
        return hc.status == 1 ? SRM_B200_ITERATION_LIMIT : SRM_B200_OK;
    }

    srm_b200_round_stats read_stats(bool with_candidates) {
        SRM_CUDA(cudaMemcpyAsync(h_stats, stats, sizeof(StatsDev), cudaMemcpyDeviceToHost, stream));
        sync();
        srm_b200_round_stats o{};
        o.overlap_pairs = static_cast<int64_t>(h_stats->overlap_pairs);
        double pen = 0.0;
        std::memcpy(&pen, &h_stats->pen_bits, sizeof(double));
        o.max_penetration = pen;
        o.candidate_pairs = with_candidates ? static_cast<int64_t>(h_stats->candidate_pairs) : -1;
        o.movers = n - static_cast<int64_t>(h_stats->active_count);
        last_nonmovers = static_cast<int64_t>(h_stats->active_count);
        last_wave_waits = static_cast<int64_t>(h_stats->wave_waits);
        last_wave_polls = static_cast<int64_t>(h_stats->wave_polls);
        last_pair_tests = static_cast<int64_t>(h_stats->pair_tests);
        return o;
    }

    // fixed-order reductions over the radii of T: {sum of measures, max radius}
    void reduce(const State& T, double* sum_measure, double* max_r) {
        if (dim == 2) k_reduce_partials<2><<<kRedBlocks, 256, 0, stream>>>(n, T.rec, red_part_sum, red_part_max, T.aux);
        else k_reduce_partials<3><<<kRedBlocks, 256, 0, stream>>>(n, T.rec, red_part_sum, red_part_max, T.aux);
        k_reduce_final<<<1, 256, 0, stream>>>(red_part_sum, red_part_max, red_out);
        launched(2);
        SRM_CUDA(cudaMemcpyAsync(h_red, red_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, stream));
        sync();
        if (sum_measure) *sum_measure = h_red[0];
        if (max_r) *max_r = h_red[1];
    }
    double box_measure() const {
        double m = 1.0;  // geometry.hpp:98-102
        for (int a = 0; a < dim; ++a) m *= box.L[a];
        return m;
    }
    double volume_fraction(const State& T) {
        double s = 0.0;
        reduce(T, &s, nullptr);
        return s / box_measure();
    }
    double max_radius(const State& T) {
        double m = 0.0;
        reduce(T, nullptr, &m);
        return m;
    }

    void scale_radius(State& T, double factor) {
        k_scale_radius<<<blocks_for(n, 256), 256, 0, stream>>>(n, T.rec, T.aux, factor);
        launched();
    }
};

namespace {

int fail(srm_b200_ctx* c, int code, const std::string& m) {
    if (c) c->err = m;
    return code;
}

template <typename F>
int guarded(srm_b200_ctx* c, F&& f) {
    if (!c) return SRM_B200_INVALID;
    try {
        c->err.clear();
        if (c->device >= 0) SRM_CUDA(cudaSetDevice(c->device));
        return f();
    } catch (const Invalid& e) {
        return fail(c, SRM_B200_INVALID, e.msg);
    } catch (const CudaError& e) {
        return fail(c, SRM_B200_CUDA_ERROR, e.msg);
    } catch (const std::bad_alloc&) {
        return fail(c, SRM_B200_CUDA_ERROR, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(c, SRM_B200_CUDA_ERROR, e.what());
    } catch (...) {  // (a caller's callback threw a non-standard exception: never across the ABI)
        return fail(c, SRM_B200_CUDA_ERROR, "unknown exception");
    }
}

// engine.hpp:38-49 validate_params, same order and messages
void validate_params(const srm_b200_params& p) {
    if (!(p.c_w >= 0.0)) throw Invalid{"params: c_w must be >= 0"};
    if (!(p.c_w <= 0.25)) throw Invalid{"params: c_w must be <= 0.25 (cell safety bound)"};
    if (!(p.c_m >= 0.0)) throw Invalid{"params: c_m must be >= 0"};
    if (!(p.c_r >= 0.0)) throw Invalid{"params: c_r must be >= 0"};
    if (p.n_k < 1) throw Invalid{"params: n_k must be >= 1"};
    if (p.n_l < 1) throw Invalid{"params: n_l must be >= 1"};
    if (!(p.f_target > 0.0 && p.f_target < 1.0)) throw Invalid{"params: f_target must lie in (0, 1)"};
    if (p.max_iterations < 1) throw Invalid{"params: max_iterations must be >= 1"};
    if (p.reorder_period < 0) throw Invalid{"params: reorder_period must be >= 0"};
    if (p.n_l > kMaxPhases) throw Invalid{"params: n_l > 254 is not supported by the B200 path"};
}

}  // namespace

extern "C" {

const char* srm_b200_create_error(void) { return g_create_error.c_str(); }

int srm_b200_create(int dim, int shape_kind, const double* box_lengths, int64_t capacity, int device,
                    srm_b200_ctx** out) {
    g_create_error.clear();
    if (!out) return SRM_B200_INVALID;
    *out = nullptr;
    if (dim != 2 && dim != 3) { g_create_error = "dim must be 2 or 3"; return SRM_B200_INVALID; }
    if (shape_kind != SRM_B200_SPHERE && shape_kind != SRM_B200_PLATELET) {
        g_create_error = "unsupported shape kind";
        return SRM_B200_INVALID;
    }
    if (shape_kind == SRM_B200_PLATELET && dim != 3) { g_create_error = "platelets are 3D"; return SRM_B200_INVALID; }
    if (capacity < 1) { g_create_error = "capacity must be >= 1"; return SRM_B200_INVALID; }
    if (capacity > 2147483647LL) {  // sorted indices and near-list entries are int32
        g_create_error = "capacity must be <= 2^31 - 1";
        return SRM_B200_INVALID;
    }
    for (int a = 0; a < dim; ++a)
        if (!(box_lengths[a] > 0.0)) {
            g_create_error = "PeriodicBox: axis length " + std::to_string(a) + " must be positive";
            return SRM_B200_INVALID;
        }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
        cudaGetLastError();
        g_create_error = "no CUDA device: the B200 SRM path has no CPU fallback";
        return SRM_B200_NO_DEVICE;
    }
    if (device < 0 || device >= ndev) { g_create_error = "bad device ordinal"; return SRM_B200_INVALID; }
    srm_b200_ctx* c = nullptr;
    try {
        c = new srm_b200_ctx();
        c->dim = dim;
        c->shape = shape_kind;
        c->device = device;
        c->cap = capacity;
        for (int a = 0; a < 3; ++a) {
            c->box.L[a] = a < dim ? box_lengths[a] : 1.0;
            c->box.half[a] = 0.5 * c->box.L[a];
        }
        c->init();
    } catch (const CudaError& e) {
        g_create_error = e.msg;
        delete c;
        return SRM_B200_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_create_error = e.what();
        delete c;
        return SRM_B200_CUDA_ERROR;
    }
    *out = c;
    return SRM_B200_OK;
}

void srm_b200_destroy(srm_b200_ctx* ctx) { delete ctx; }

const char* srm_b200_last_error(const srm_b200_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t srm_b200_count(const srm_b200_ctx* ctx) { return ctx ? ctx->n : 0; }

int srm_b200_describe(const srm_b200_ctx* ctx, int* dim, int* shape_kind, double* box_lengths) {
    if (!ctx) return SRM_B200_INVALID;
    if (dim) *dim = ctx->dim;
    if (shape_kind) *shape_kind = ctx->platelets() ? SRM_B200_PLATELET : SRM_B200_SPHERE;
    if (box_lengths)
        for (int a = 0; a < ctx->dim; ++a) box_lengths[a] = ctx->box.L[a];
    return SRM_B200_OK;
}

int srm_b200_upload(srm_b200_ctx* c, int64_t n, const double* pos, const double* radius, const int32_t* id) {
    return guarded(c, [&]() -> int {
        if (c->platelets()) throw Invalid{"upload: platelet context (use srm_b200_upload_platelets)"};
        if (n < 0 || n > c->cap) throw Invalid{"upload: n exceeds the context capacity"};
        if (n > 0 && (!pos || !radius)) throw Invalid{"upload: null pointer"};
        c->n = n;
        if (n == 0) return SRM_B200_OK;
        // stage through the sorted state's buffers (scratch outside a round):
        // positions at [0, dim n), radii at [3 cap, 3 cap + n) of S.rec viewed as doubles
        double* dpos = reinterpret_cast<double*>(c->S.rec);
        double* drad = dpos + 3 * c->cap;
        SRM_CUDA(cudaMemcpyAsync(dpos, pos, sizeof(double) * n * c->dim, cudaMemcpyHostToDevice, c->stream));
        SRM_CUDA(cudaMemcpyAsync(drad, radius, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        int32_t* did = nullptr;
        if (id) {
            SRM_CUDA(cudaMemcpyAsync(c->S.id, id, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
            did = c->S.id;
        }
        if (c->dim == 2) k_unpack_soa<2><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, dpos, drad, did, c->P);
        else k_unpack_soa<3><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, dpos, drad, did, c->P);
        c->launched();
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_download(srm_b200_ctx* c, double* pos, double* radius, int32_t* id) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        if (n == 0) return SRM_B200_OK;
        double* dpos = reinterpret_cast<double*>(c->S.rec);
        double* drad = dpos + 3 * c->cap;
        if (c->dim == 2) k_pack_soa<2><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->P, dpos, drad, c->S.id);
        else k_pack_soa<3><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->P, dpos, drad, c->S.id);
        c->launched();
        if (pos) SRM_CUDA(cudaMemcpyAsync(pos, dpos, sizeof(double) * n * c->dim, cudaMemcpyDeviceToHost, c->stream));
        if (radius) SRM_CUDA(cudaMemcpyAsync(radius, drad, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        if (id) SRM_CUDA(cudaMemcpyAsync(id, c->S.id, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_upload_platelets(srm_b200_ctx* c, int64_t n, const double* pos, const double* normal,
                              const double* diameter, const double* thickness, const int32_t* id) {
    return guarded(c, [&]() -> int {
        if (!c->platelets()) throw Invalid{"upload_platelets: not a platelet context"};
        if (n < 0 || n > c->cap) throw Invalid{"upload: n exceeds the context capacity"};
        if (n > 0 && (!pos || !normal || !diameter || !thickness)) throw Invalid{"upload: null pointer"};
        c->n = n;
        if (n == 0) return SRM_B200_OK;
        // stage through the sorted state's buffers: pos at [0, 3n), normal at [3 cap, ...)
        double* st = reinterpret_cast<double*>(c->S.rec);
        double* sa = reinterpret_cast<double*>(c->S.aux);
        SRM_CUDA(cudaMemcpyAsync(st, pos, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
        SRM_CUDA(cudaMemcpyAsync(st + 3 * c->cap, diameter, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        SRM_CUDA(cudaMemcpyAsync(sa, normal, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, c->stream));
        SRM_CUDA(cudaMemcpyAsync(sa + 3 * c->cap, thickness, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        int32_t* did = nullptr;
        if (id) {
            SRM_CUDA(cudaMemcpyAsync(c->S.id, id, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
            did = c->S.id;
        }
        k_unpack_pl<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, st, sa, st + 3 * c->cap, sa + 3 * c->cap, did, c->P);
        c->launched();
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_download_platelets(srm_b200_ctx* c, double* pos, double* normal, double* diameter, double* thickness,
                                int32_t* id) {
    return guarded(c, [&]() -> int {
        if (!c->platelets()) throw Invalid{"download_platelets: not a platelet context"};
        const int64_t n = c->n;
        if (n == 0) return SRM_B200_OK;
        double* st = reinterpret_cast<double*>(c->S.rec);
        double* sa = reinterpret_cast<double*>(c->S.aux);
        k_pack_pl<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->P, st, sa, st + 3 * c->cap, sa + 3 * c->cap, c->S.id);
        c->launched();
        if (pos) SRM_CUDA(cudaMemcpyAsync(pos, st, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
        if (normal) SRM_CUDA(cudaMemcpyAsync(normal, sa, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost, c->stream));
        if (diameter)
            SRM_CUDA(cudaMemcpyAsync(diameter, st + 3 * c->cap, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        if (thickness)
            SRM_CUDA(cudaMemcpyAsync(thickness, sa + 3 * c->cap, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        if (id) SRM_CUDA(cudaMemcpyAsync(id, c->S.id, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_set_rotation(srm_b200_ctx* c, double c_r) {
    return guarded(c, [&]() -> int {
        if (!(c_r >= 0.0)) throw Invalid{"params: c_r must be >= 0"};
        c->c_r = c_r;
        return SRM_B200_OK;
    });
}

// The reference's Particle<N> AoS layout (geometry.hpp:139-144) as the caller describes
// it: every field inside the record, doubles 8-byte aligned (a misaligned double load is
// a sticky CUDA error for the whole process), records of disks / spheres only (a
// platelet record also carries the normal and thickness: srm_b200_upload_platelets).
static void check_record_layout(const srm_b200_ctx* c, int64_t n, const void* records, int64_t stride, int64_t off_id,
                         int64_t off_pos, int64_t off_radius) {
    if (c->platelets()) throw Invalid{"records: platelet contexts take srm_b200_upload_platelets"};
    if (n > 0 && !records) throw Invalid{"records: null pointer"};
    if (stride < 1) throw Invalid{"records: bad stride"};
    if (off_id < 0 || off_id + 4 > stride) throw Invalid{"records: id field outside the record"};
    if (off_pos < 0 || off_pos + 8 * c->dim > stride) throw Invalid{"records: position field outside the record"};
    if (off_radius < 0 || off_radius + 8 > stride) throw Invalid{"records: radius field outside the record"};
    if (stride % 8 || off_pos % 8 || off_radius % 8 || off_id % 4 ||
        reinterpret_cast<uintptr_t>(records) % 8)
        throw Invalid{"records: doubles must be 8-byte aligned (stride, offsets and base address)"};
}

int srm_b200_upload_records(srm_b200_ctx* c, int64_t n, const void* records, int64_t stride, int64_t off_id,
                            int64_t off_pos, int64_t off_radius) {
    return guarded(c, [&]() -> int {
        if (n < 0 || n > c->cap) throw Invalid{"upload: n exceeds the context capacity"};
        check_record_layout(c, n, records, stride, off_id, off_pos, off_radius);
        c->n = n;
        if (n == 0) return SRM_B200_OK;
        const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(stride);
        if (bytes > c->rec_stage_bytes) {
            cudaFree(c->rec_stage);
            c->rec_stage = nullptr;
            c->rec_stage = dalloc<char>(static_cast<int64_t>(bytes));
            c->rec_stage_bytes = bytes;
        }
        SRM_CUDA(cudaMemcpyAsync(c->rec_stage, records, bytes, cudaMemcpyHostToDevice, c->stream));
        if (c->dim == 2)
            k_unpack_records<2><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->rec_stage, stride, off_id, off_pos, off_radius, c->P);
        else
            k_unpack_records<3><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->rec_stage, stride, off_id, off_pos, off_radius, c->P);
        c->launched();
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_download_records(srm_b200_ctx* c, void* records, int64_t stride, int64_t off_id, int64_t off_pos,
                              int64_t off_radius) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        check_record_layout(c, n, records, stride, off_id, off_pos, off_radius);
        if (n == 0) return SRM_B200_OK;
        const size_t bytes = static_cast<size_t>(n) * static_cast<size_t>(stride);
        if (bytes > c->rec_stage_bytes) {
            cudaFree(c->rec_stage);
            c->rec_stage = nullptr;
            c->rec_stage = dalloc<char>(static_cast<int64_t>(bytes));
            c->rec_stage_bytes = bytes;
        }
        // keep any bytes of the records we do not own (padding, extra fields)
        SRM_CUDA(cudaMemcpyAsync(c->rec_stage, records, bytes, cudaMemcpyHostToDevice, c->stream));
        if (c->dim == 2)
            k_pack_records<2><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->P, c->rec_stage, stride, off_id, off_pos, off_radius);
        else
            k_pack_records<3><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->P, c->rec_stage, stride, off_id, off_pos, off_radius);
        c->launched();
        SRM_CUDA(cudaMemcpyAsync(records, c->rec_stage, bytes, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_grid_dims(srm_b200_ctx* c, double cell_size, double max_radius, double slack, int32_t* dims_out,
                       double* edge_out, int64_t* ncells_out) {
    return guarded(c, [&]() -> int {
        const GridParams g = c->make_grid(cell_size, 0.0, 0.0);
        if (max_radius >= 0.0) {
            const double min_safe = 2.0 * max_radius + slack;  // cell_grid.hpp:33-35
            if (cell_size < min_safe) throw Invalid{"CellGrid: cell_size below safety bound 2*maxR + slack"};
        }
        for (int a = 0; a < c->dim; ++a) {
            if (dims_out) dims_out[a] = g.dims[a];
            if (edge_out) edge_out[a] = g.edge[a];
        }
        if (ncells_out) *ncells_out = g.ncells;
        return SRM_B200_OK;
    });
}

int srm_b200_grid_build(srm_b200_ctx* c, double cell_size, uint32_t* keys_out, int32_t* order_out,
                        int64_t* cell_start_out) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        const GridParams g = c->make_grid(cell_size, 0.0, 0.0);
        c->set_grid(g);
        if (n > 0) {
            c->grid_build(c->P);
            if (keys_out) {
                k_keys_by_slot<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->S.slot, c->skey, c->key);
                c->launched();
                SRM_CUDA(cudaMemcpyAsync(keys_out, c->key, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, c->stream));
            }
            if (order_out)
                SRM_CUDA(cudaMemcpyAsync(order_out, c->S.slot, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
            c->swap_state(c->S, c->P);  // keep the state physically sorted
        } else {
            SRM_CUDA(cudaMemsetAsync(c->cell_start, 0, sizeof(cell_t) * (g.ncells + 1), c->stream));
        }
        if (cell_start_out) {  // the device keeps 32-bit offsets; the ABI reports int64
            std::vector<cell_t> h(static_cast<size_t>(g.ncells) + 1);
            SRM_CUDA(cudaMemcpyAsync(h.data(), c->cell_start, sizeof(cell_t) * h.size(), cudaMemcpyDeviceToHost,
                                     c->stream));
            c->sync();
            for (size_t k = 0; k < h.size(); ++k) cell_start_out[k] = h[k];
        }
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_overlap_stats(srm_b200_ctx* c, double cell_size, srm_b200_round_stats* out) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        srm_b200_round_stats o{0, 0.0, 0, 0};
        if (n > 0) {
            const double mr = c->max_radius(c->P);
            const GridParams g = c->make_grid(cell_size, mr, 0.0);
            c->set_grid(g);
            c->grid_build(c->P);
            c->copy_state(c->S, c->P);
            SRM_CUDA(cudaMemsetAsync(c->stats, 0, sizeof(StatsDev), c->stream));
            {
                srm_b200_ctx::FamScope fs(c, 3);
                if (c->platelets())
                    k_overlap_pl<<<blocks_for(n * 32, kOverlapPlThreads), kOverlapPlThreads, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey,
                                                                          c->stats);
                else if (c->dim == 2)
                    k_overlap_full<2><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, 1, c->stats);
                else
                    k_overlap_full<3><<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, 1, c->stats);
                c->launched();
            }
            o = c->read_stats(true);
            o.movers = 0;
        }
        if (out) *out = o;
        return SRM_B200_OK;
    });
}

// ---- parity statistics on the device (srm_descriptors.cuh) ------------------------------
int srm_b200_nnd_histogram(srm_b200_ctx* c, int bins, double lo, double hi, int64_t* counts_out, int64_t* total_out,
                           int64_t* in_range_out, double* nnd_out) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        if (n < 2) throw Invalid{"nearest_neighbor_distances: need at least 2 particles"};
        if (counts_out && bins < 1) throw Invalid{"histogram: bin_count must be >= 1"};
        if (counts_out && !(hi > lo)) throw Invalid{"histogram: need hi > lo"};
        const double mr = c->max_radius(c->P);
        // any grid gives the exact answer; about one particle per cell, as descriptor_grid
        double vol = 1.0;
        for (int a = 0; a < c->dim; ++a) vol *= c->box.L[a];
        double cell = std::pow(vol / static_cast<double>(n), 1.0 / c->dim);
        cell = std::max(cell, 1e-3 * mr);
        c->set_grid(c->make_grid(cell, mr, 0.0));
        c->grid_build(c->P);
        DevBuf<double> d(n);
        const int nb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 16));
        if (c->dim == 2) k_nnd<2><<<nb, 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, d.p);
        else k_nnd<3><<<nb, 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, d.p);
        c->launched();
        if (counts_out) {
            DevBuf<unsigned long long> h(bins + 2);
            SRM_CUDA(cudaMemsetAsync(h.p, 0, sizeof(unsigned long long) * (bins + 2), c->stream));
            k_histogram<<<nb, 256, 0, c->stream>>>(n, d.p, bins, lo, hi, h.p, h.p + bins);
            c->launched();
            std::vector<unsigned long long> hh(static_cast<size_t>(bins) + 2);
            SRM_CUDA(cudaMemcpyAsync(hh.data(), h.p, sizeof(unsigned long long) * hh.size(), cudaMemcpyDeviceToHost,
                                     c->stream));
            SRM_CUDA(cudaStreamSynchronize(c->stream));
            for (int b = 0; b < bins; ++b) counts_out[b] = static_cast<int64_t>(hh[b]);
            if (total_out) *total_out = static_cast<int64_t>(hh[bins]);
            if (in_range_out) *in_range_out = static_cast<int64_t>(hh[bins + 1]);
        }
        if (nnd_out)
            SRM_CUDA(cudaMemcpyAsync(nnd_out, d.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
        SRM_CUDA(cudaStreamSynchronize(c->stream));
        return SRM_B200_OK;
    });
}

int srm_b200_rsa_device(srm_b200_ctx* c, int64_t n, const double* radii, uint64_t seed, int64_t max_rounds,
                        int64_t* placed_out, int64_t* rounds_out) {
    if (placed_out) *placed_out = 0;
    if (rounds_out) *rounds_out = 0;
    if (!c) return SRM_B200_INVALID;
    return guarded(c, [&]() -> int {
        if (c->platelets()) throw Invalid{"rsa_device: spheres and disks only"};
        if (n < 1 || n > c->cap || !radii) throw Invalid{"rsa_device: need 1 <= n <= capacity radii"};
        double max_r = 0.0, min_len = c->box.L[0];
        for (int64_t i = 0; i < n; ++i) {
            if (!(radii[i] > 0.0)) throw Invalid{"rsa_device: radii must be positive"};  // rsa.hpp:26-27
            max_r = std::max(max_r, radii[i]);
        }
        for (int a = 1; a < c->dim; ++a) min_len = std::min(min_len, c->box.L[a]);
        if (!(max_r < min_len / 4.0)) throw Invalid{"rsa_device: radius too large for the box"};  // rsa.hpp:28-29
        {
            std::vector<double> zero(static_cast<size_t>(n) * c->dim, 0.0);
            std::vector<int32_t> ids(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) ids[i] = static_cast<int32_t>(i);
            const int st = srm_b200_upload(c, n, zero.data(), radii, ids.data());
            if (st != SRM_B200_OK) return st;
        }
        // cells of at least 2 max_r: every overlapping pair is in the one-cell stencil
        c->set_grid(c->make_grid(2.0 * max_r * (1.0 + 1e-8), max_r, 0.0));
        DevBuf<uint8_t> placed(n);
        DevBuf<int8_t> state(n);
        DevBuf<int32_t> conf(n * kRsaConf), nconf(n);
        DevBuf<int64_t> where(n);
        DevBuf<unsigned long long> count(1);
        DevBuf<int> flag(1);
        SRM_CUDA(cudaMemsetAsync(placed.p, 0, static_cast<size_t>(n), c->stream));
        SRM_CUDA(cudaMemsetAsync(count.p, 0, sizeof(unsigned long long), c->stream));
        const int nb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 16));
        const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
        unsigned long long done = 0;
        int64_t r = 0;
        for (; r < max_rounds && static_cast<int64_t>(done) < n; ++r) {
            k_rsa_propose<<<nb, 256, 0, c->stream>>>(n, c->dim, c->P.rec, placed.p, c->box, k0, k1, static_cast<uint32_t>(r));
            c->grid_build(c->P);
            if (c->dim == 2)
                k_rsa_check<2><<<nb, 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, placed.p,
                                                          state.p, conf.p, nconf.p, where.p);
            else
                k_rsa_check<3><<<nb, 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, placed.p,
                                                          state.p, conf.p, nconf.p, where.p);
            c->launched(2);
            int h = 1;
            while (h > 0) {  // the resolution reaches its fixed point in a few sweeps
                SRM_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
                if (c->dim == 2)
                    k_rsa_resolve<2><<<nb, 256, 0, c->stream>>>(n, placed.p, state.p, conf.p, nconf.p, flag.p, c->S,
                                                                c->box, c->gp, c->cell_start, c->skey, where.p);
                else
                    k_rsa_resolve<3><<<nb, 256, 0, c->stream>>>(n, placed.p, state.p, conf.p, nconf.p, flag.p, c->S,
                                                                c->box, c->gp, c->cell_start, c->skey, where.p);
                c->launched();
                SRM_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
                SRM_CUDA(cudaStreamSynchronize(c->stream));
            }
            k_rsa_commit<<<nb, 256, 0, c->stream>>>(n, placed.p, state.p, count.p);
            c->launched();
            SRM_CUDA(cudaMemcpyAsync(&done, count.p, sizeof(done), cudaMemcpyDeviceToHost, c->stream));
            SRM_CUDA(cudaStreamSynchronize(c->stream));
        }
        if (placed_out) *placed_out = static_cast<int64_t>(done);
        if (rounds_out) *rounds_out = r;
        return static_cast<int64_t>(done) == n ? SRM_B200_OK : SRM_B200_PLACEMENT_FAILURE;
    });
}

// recipes.cpp:107-148 rsa_platelets, in rounds on the device
int srm_b200_rsa_platelets_device(srm_b200_ctx* c, int64_t n, double diameter, double aspect_ratio, uint64_t seed,
                                  int64_t max_rounds, int64_t* placed_out, int64_t* rounds_out) {
    if (placed_out) *placed_out = 0;
    if (rounds_out) *rounds_out = 0;
    if (!c) return SRM_B200_INVALID;
    return guarded(c, [&]() -> int {
        if (!c->platelets()) throw Invalid{"rsa_platelets_device: a platelet context is required"};
        if (n < 1 || n > c->cap) throw Invalid{"rsa_platelets: n must be >= 1"};  // recipes.cpp:109
        if (!(aspect_ratio > 1.0)) throw Invalid{"rsa_platelets: aspect ratio must exceed 1"};
        if (!(diameter > 0.0)) throw Invalid{"rsa_platelets: diameter must be positive"};
        const double thickness = diameter / aspect_ratio;  // recipes.cpp:112-117
        const double bound = 0.5 * (diameter + thickness);
        double min_len = c->box.L[0];
        for (int a = 1; a < 3; ++a) min_len = std::min(min_len, c->box.L[a]);
        if (!(bound < min_len / 4.0)) throw Invalid{"rsa_platelets: platelet too large for the box"};
        {
            std::vector<double> zero(static_cast<size_t>(n) * 3, 0.0), up(static_cast<size_t>(n) * 3, 0.0);
            for (int64_t i = 0; i < n; ++i) up[3 * i + 2] = 1.0;
            std::vector<double> D(static_cast<size_t>(n), diameter), t(static_cast<size_t>(n), thickness);
            std::vector<int32_t> ids(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) ids[i] = static_cast<int32_t>(i);
            const int st = srm_b200_upload_platelets(c, n, zero.data(), up.data(), D.data(), t.data(), ids.data());
            if (st != SRM_B200_OK) return st;
        }
        // cells of at least two bounding radii: every overlapping pair is in the one-cell stencil
        c->set_grid(c->make_grid(2.0 * bound * (1.0 + 1e-8), bound, 0.0));
        DevBuf<uint8_t> placed(n);
        DevBuf<int8_t> state(n);
        DevBuf<int32_t> conf(n * kRsaConf), nconf(n);
        DevBuf<int64_t> where(n);
        DevBuf<unsigned long long> count(1);
        DevBuf<int> flag(1);
        SRM_CUDA(cudaMemsetAsync(placed.p, 0, static_cast<size_t>(n), c->stream));
        SRM_CUDA(cudaMemsetAsync(count.p, 0, sizeof(unsigned long long), c->stream));
        const int nb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 16));
        const int nbc = static_cast<int>(std::min<int64_t>(blocks_for(n, 128), 148 * 16));
        const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
        unsigned long long done = 0;
        int64_t r = 0;
        for (; r < max_rounds && static_cast<int64_t>(done) < n; ++r) {
            k_rsa_pl_propose<<<nb, 256, 0, c->stream>>>(n, c->P.rec, c->P.aux, placed.p, c->box, k0, k1,
                                                        static_cast<uint32_t>(r));
            c->grid_build(c->P);
            k_rsa_pl_check<<<nbc, 128, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, placed.p,
                                                       state.p, conf.p, nconf.p, where.p);
            c->launched(2);
            int h = 1;
            while (h > 0) {
                SRM_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
                k_rsa_pl_resolve<<<nb, 256, 0, c->stream>>>(n, placed.p, state.p, conf.p, nconf.p, flag.p, c->S, c->box,
                                                            c->gp, c->cell_start, c->skey, where.p);
                c->launched();
                SRM_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
                SRM_CUDA(cudaStreamSynchronize(c->stream));
            }
            k_rsa_commit<<<nb, 256, 0, c->stream>>>(n, placed.p, state.p, count.p);
            c->launched();
            SRM_CUDA(cudaMemcpyAsync(&done, count.p, sizeof(done), cudaMemcpyDeviceToHost, c->stream));
            SRM_CUDA(cudaStreamSynchronize(c->stream));
        }
        if (placed_out) *placed_out = static_cast<int64_t>(done);
        if (rounds_out) *rounds_out = r;
        return static_cast<int64_t>(done) == n ? SRM_B200_OK : SRM_B200_PLACEMENT_FAILURE;
    });
}

int srm_b200_platelet_order(srm_b200_ctx* c, double cutoff, double* value_out, int32_t* count_out, double* nnd_out,
                            double* nn_align_out, double* q_out) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        if (!c->platelets()) throw Invalid{"platelet_order: a platelet context is required"};
        if ((value_out || count_out) && !(cutoff > 0.0))
            throw Invalid{"local_nematic_order: cutoff must be positive"};  // descriptors.hpp:183
        const double mr = c->max_radius(c->P);
        const int nb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 16));
        if (value_out || count_out) {
            c->set_grid(c->make_grid(cutoff, mr, 0.0));  // cells >= cutoff: a one-cell stencil
            c->grid_build(c->P);
            const GridParams& g = c->hg;
            int32_t sw[3];
            for (int a = 0; a < 3; ++a) sw[a] = g.dims[a] <= 3 ? -1 : 1;
            DevBuf<int32_t> dsw(3), cnt(n);
            DevBuf<double> val(n);
            SRM_CUDA(cudaMemcpyAsync(dsw.p, sw, sizeof(sw), cudaMemcpyHostToDevice, c->stream));
            k_local_nematic<<<nb, 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, dsw.p, cutoff, val.p,
                                                       cnt.p);
            c->launched();
            if (value_out) SRM_CUDA(cudaMemcpyAsync(value_out, val.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
            if (count_out) SRM_CUDA(cudaMemcpyAsync(count_out, cnt.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
            SRM_CUDA(cudaStreamSynchronize(c->stream));
        }
        if (nnd_out || nn_align_out) {
            if (n < 2) throw Invalid{"nearest_neighbor_distances: need at least 2 particles"};
            double cell = std::pow(c->box_measure() / static_cast<double>(n), 1.0 / 3.0);
            cell = std::max(cell, 1e-3 * mr);
            c->set_grid(c->make_grid(cell, mr, 0.0));
            c->grid_build(c->P);
            DevBuf<double> d(n), al(n);
            k_nnd<3><<<nb, 256, 0, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, d.p, al.p);
            c->launched();
            if (nnd_out) SRM_CUDA(cudaMemcpyAsync(nnd_out, d.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
            if (nn_align_out) SRM_CUDA(cudaMemcpyAsync(nn_align_out, al.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
            SRM_CUDA(cudaStreamSynchronize(c->stream));
        }
        if (q_out) {
            constexpr int kQBlocks = 296;
            DevBuf<double> part(kQBlocks * 6);
            k_q_tensor<<<kQBlocks, 256, 0, c->stream>>>(n, c->P.aux, part.p);
            c->launched();
            std::vector<double> hp(kQBlocks * 6);
            SRM_CUDA(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * hp.size(), cudaMemcpyDeviceToHost, c->stream));
            SRM_CUDA(cudaStreamSynchronize(c->stream));
            for (int k = 0; k < 6; ++k) {
                double s = 0.0;
                for (int b = 0; b < kQBlocks; ++b) s += hp[b * 6 + k];
                q_out[k] = s;
            }
        }
        return SRM_B200_OK;
    });
}

int srm_b200_pair_counts(srm_b200_ctx* c, const double* edges, int bins, int64_t* counts_out) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        if (bins < 1 || !(edges[bins] > edges[0]) || !(edges[0] >= 0.0)) throw Invalid{"pair_counts: bad edges"};
        std::vector<unsigned long long> hh(static_cast<size_t>(bins), 0ull);
        if (n >= 2) {
            const double hi = edges[bins];
            const double mr = c->max_radius(c->P);
            c->set_grid(c->make_grid(hi, mr, 0.0));
            c->grid_build(c->P);
            const GridParams& g = c->hg;
            int32_t sw[3] = {-1, -1, -1};
            for (int a = 0; a < c->dim; ++a) {  // the cells within hi, or the whole axis
                int s = 1;
                while (static_cast<double>(s) * g.edge[a] < hi && 2 * s + 1 < g.dims[a]) ++s;
                sw[a] = 2 * s + 1 >= g.dims[a] ? -1 : s;
            }
            DevBuf<int32_t> dsw(3);
            DevBuf<double> de(bins + 1);
            DevBuf<unsigned long long> h(bins);
            SRM_CUDA(cudaMemcpyAsync(dsw.p, sw, sizeof(sw), cudaMemcpyHostToDevice, c->stream));
            SRM_CUDA(cudaMemcpyAsync(de.p, edges, sizeof(double) * (bins + 1), cudaMemcpyHostToDevice, c->stream));
            SRM_CUDA(cudaMemsetAsync(h.p, 0, sizeof(unsigned long long) * bins, c->stream));
            const int nb = static_cast<int>(std::min<int64_t>(blocks_for(n, 256), 148 * 8));
            const size_t sh = sizeof(unsigned long long) * bins;
            if (sh > 48 * 1024) throw Invalid{"pair_counts: at most 6144 bins"};
            if (c->dim == 2)
                k_pair_counts<2><<<nb, 256, sh, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, de.p, bins,
                                                             dsw.p, h.p);
            else
                k_pair_counts<3><<<nb, 256, sh, c->stream>>>(n, c->S, c->box, c->gp, c->cell_start, c->skey, de.p, bins,
                                                             dsw.p, h.p);
            c->launched();
            SRM_CUDA(cudaMemcpyAsync(hh.data(), h.p, sizeof(unsigned long long) * bins, cudaMemcpyDeviceToHost, c->stream));
            SRM_CUDA(cudaStreamSynchronize(c->stream));
        }
        for (int b = 0; b < bins; ++b) counts_out[b] = static_cast<int64_t>(hh[b]);
        return SRM_B200_OK;
    });
}

int srm_b200_round(srm_b200_ctx* c, double cell_size, double c_m, int n_l, uint64_t key, uint32_t round_id,
                   uint32_t iteration, int with_candidates, uint8_t* accepted_out, srm_b200_round_stats* out) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        if (n_l < 1) throw Invalid{"params: n_l must be >= 1"};
        if (!(c_m >= 0.0)) throw Invalid{"params: c_m must be >= 0"};
        srm_b200_round_stats o{0, 0.0, with_candidates ? 0 : -1, 0};
        if (n > 0) {
            const double mr = c->max_radius(c->P);
            const GridParams g = c->make_grid(cell_size, mr, c_m);
            // the reference scans the 3^d cells of the trial position, which is only
            // complete under CellGrid's safety bound (cell_grid.hpp:31-36)
            if (cell_size < 2.0 * mr + c_m) throw Invalid{"CellGrid: cell_size below safety bound 2*maxR + slack"};
            c->set_grid(g);
            c->round(c->P, c_m, n_l, key, round_id, iteration, true, with_candidates != 0, accepted_out != nullptr);
            if (accepted_out) {
                k_acc_by_slot<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->P.slot, c->acc, reinterpret_cast<uint8_t*>(c->perm));
                c->launched();
                SRM_CUDA(cudaMemcpyAsync(accepted_out, c->perm, n, cudaMemcpyDeviceToHost, c->stream));
            }
            o = c->read_stats(with_candidates != 0);
        }
        if (out) *out = o;
        return SRM_B200_OK;
    });
}

int srm_b200_rounds(srm_b200_ctx* c, double cell_size, double c_m, int n_l, uint64_t key, uint32_t first_round,
                    uint32_t iteration, int rounds, srm_b200_round_stats* last) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        if (n_l < 1) throw Invalid{"params: n_l must be >= 1"};
        srm_b200_round_stats o{0, 0.0, -1, 0};
        if (n > 0 && rounds > 0) {
            const double mr = c->max_radius(c->P);
            if (cell_size < 2.0 * mr + c_m) throw Invalid{"CellGrid: cell_size below safety bound 2*maxR + slack"};
            const GridParams g = c->make_grid(cell_size, mr, c_m);
            c->set_grid(g);
            for (int k = 0; k < rounds; ++k) c->round(c->P, c_m, n_l, key, first_round + k, iteration, true, false);
            o = c->read_stats(false);
        }
        if (last) *last = o;
        return SRM_B200_OK;
    });
}

int srm_b200_relax_sweeps(srm_b200_ctx* c, double c_m, double c_r, int n_l, int sweeps, uint64_t key) {
    if (c) c->c_r = c_r;  // platelet rotation angle (ignored by disks/spheres)
    (void)c_r;  // rotation rate is ignored by disks/spheres (shape.hpp:27-28)
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        if (n == 0 || sweeps < 1) return SRM_B200_OK;  // engine.hpp:115
        if (n_l < 1) throw Invalid{"params: n_l must be >= 1"};
        const double max_r = c->max_radius(c->P);
        const double cs = 2.5 * max_r + c_m;  // engine.hpp:116-117
        const GridParams g = c->make_grid(cs, max_r, c_m);
        if (cs < 2.0 * max_r + c_m) throw Invalid{"CellGrid: cell_size below safety bound 2*maxR + slack"};
        c->set_grid(g);
        for (int k = 0; k < sweeps; ++k) c->round(c->P, c_m, n_l, key, static_cast<uint32_t>(k), 0u, false, false);
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_swell_all(srm_b200_ctx* c, double c_w) {
    return guarded(c, [&]() -> int {
        if (c->n > 0) c->scale_radius(c->P, 1.0 + c_w);  // engine.hpp:136
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_reorder_by_locality(srm_b200_ctx* c, double cell_size, int32_t* remap_out) {
    return guarded(c, [&]() -> int {
        const int64_t n = c->n;
        const GridParams g = c->make_grid(cell_size, 0.0, 0.0);
        if (n == 0) return SRM_B200_OK;
        c->set_grid(g);
        c->grid_build(c->P);
        // old slots of the sorted order are S.slot; remap[old] = new
        int32_t* remap_dev = c->perm;
        SRM_CUDA(cudaMemcpyAsync(c->Q.slot, c->S.slot, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, c->stream));
        k_assign_slots<<<blocks_for(n, 256), 256, 0, c->stream>>>(n, c->S, remap_dev, c->Q.slot);
        c->launched();
        c->swap_state(c->S, c->P);
        if (remap_out) SRM_CUDA(cudaMemcpyAsync(remap_out, remap_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_max_bounding_radius(srm_b200_ctx* c, double* out) {
    return guarded(c, [&]() -> int {
        *out = c->n > 0 ? c->max_radius(c->P) : 0.0;
        return SRM_B200_OK;
    });
}

int srm_b200_volume_fraction(srm_b200_ctx* c, double* out) {
    return guarded(c, [&]() -> int {
        *out = c->n > 0 ? c->volume_fraction(c->P) : 0.0;
        return SRM_B200_OK;
    });
}

// engine.hpp:176-260 srm_generate
int srm_b200_generate(srm_b200_ctx* c, const srm_b200_params* params, int64_t iteration_count_in,
                      srm_b200_progress_fn progress, void* user, srm_b200_generate_out* out) {
    return guarded(c, [&]() -> int {
        if (!params) throw Invalid{"params: null"};
        const srm_b200_params p = *params;
        c->c_r = p.c_r;
        validate_params(p);
        const int N = c->dim;
        double min_len = c->box.L[0];
        for (int a = 1; a < N; ++a) min_len = std::min(min_len, c->box.L[a]);
        if (!(p.c_m < 0.5 * min_len))
            throw Invalid{"srm_generate: c_m must be below half the shortest box length"};
        if (c->n == 0) throw Invalid{"srm_generate: initial snapshot has no particles"};

        double f = c->volume_fraction(c->P);
        const double stop = p.f_target * (1.0 - 1e-12);
        if (f < stop && p.c_w == 0.0)
            throw Invalid{"srm_generate: c_w must be positive to grow toward f_target"};

        const auto t_start = std::chrono::steady_clock::now();
        int64_t done = 0, accepted_iters = 0, rounds = 0, shakes = 0;
        int accepted_since_reorder = 0;
        int status = SRM_B200_OK;
        if (c->device_loop && f < stop) {  // one CUDA graph, no host round-trip per iteration
            status = c->generate_graph(p, iteration_count_in, f, c->max_radius(c->P), &done, &accepted_iters, &rounds,
                                       &shakes, &f, progress, user);
            if (out) {
                out->status = status;
                out->volume_fraction = f;
                out->iteration_count = iteration_count_in + done;
                out->accepted_iterations = accepted_iters;
                out->rounds = rounds;
                out->shake_rounds = shakes;
            }
            return status;
        }
        while (f < stop) {
            if (done >= p.max_iterations) {
                status = SRM_B200_ITERATION_LIMIT;
                break;
            }
            ++done;
            const int64_t it = iteration_count_in + done;
            double factor = 1.0 + p.c_w;
            if (f * std::pow(factor, N) > p.f_target) factor = std::pow(p.f_target / f, 1.0 / N);

            const double max_r = c->max_radius(c->P);
            const double cs = 2.5 * max_r + p.c_m;
            if (cs < 2.0 * (max_r * factor) + p.c_m)  // CellGrid(box, cs, max_r*factor, c_m)
                throw Invalid{"CellGrid: cell_size below safety bound 2*maxR + slack"};
            const GridParams gq = c->make_grid(cs, max_r * factor, p.c_m);
            c->set_grid(gq);

            c->copy_state(c->P, c->Q);
            c->scale_radius(c->Q, factor);

            bool success = false;
            int rounds_this = 0;
            for (int k = 0; k < p.n_k; ++k) {
                c->round(c->Q, p.c_m, p.n_l, p.seed, static_cast<uint32_t>(k), static_cast<uint32_t>(it), true, false);
                ++rounds;
                ++rounds_this;
                const srm_b200_round_stats st = c->read_stats(false);
                if (st.overlap_pairs == 0) {
                    success = true;
                    break;
                }
            }
            if (success) {
                c->swap_state(c->Q, c->P);  // commit (Q is rebuilt from P next iteration)
                f = c->volume_fraction(c->P);
                ++accepted_iters;
                if (p.reorder_period > 0 && ++accepted_since_reorder >= p.reorder_period) {
                    accepted_since_reorder = 0;
                    // reorder_by_locality(P, grid) (engine.hpp:239-243)
                    c->grid_build(c->P);
                    SRM_CUDA(cudaMemcpyAsync(c->Q.slot, c->S.slot, sizeof(int32_t) * c->n, cudaMemcpyDeviceToDevice, c->stream));
                    k_assign_slots<<<blocks_for(c->n, 256), 256, 0, c->stream>>>(c->n, c->S, nullptr, c->Q.slot);
                    c->launched();
                    c->swap_state(c->S, c->P);
                }
            } else {
                // shake: n_k sweeps on the pre-swell state with the same grid (engine.hpp:244-249)
                const GridParams gp_ = c->make_grid(cs, max_r, p.c_m);
                c->set_grid(gp_);
                for (int k = 0; k < p.n_k; ++k) {
                    c->round(c->P, p.c_m, p.n_l, p.seed, static_cast<uint32_t>(p.n_k + k), static_cast<uint32_t>(it), false, false);
                    ++shakes;
                }
                c->sync();
                rounds_this = p.n_k;
            }
            if (progress) {
                const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t_start;
                srm_b200_progress_record rec{it, f, success ? 1 : 0, dt.count(), rounds_this};
                progress(&rec, user);
            }
        }
        c->sync();
        if (out) {
            out->status = status;
            out->volume_fraction = f;
            out->iteration_count = iteration_count_in + done;
            out->accepted_iterations = accepted_iters;
            out->rounds = rounds;
            out->shake_rounds = shakes;
        }
        return status;
    });
}

int64_t srm_b200_launch_count(const srm_b200_ctx* c) { return c ? c->launches : 0; }
int64_t srm_b200_graph_builds(const srm_b200_ctx* c) { return c ? c->graph_builds : 0; }
void srm_b200_reset_launch_count(srm_b200_ctx* c) {
    if (c) c->launches = 0;
}

int srm_b200_timing_enable(srm_b200_ctx* c, int enable) {
    return guarded(c, [&]() -> int {
        c->sync();
        c->harvest_timing();
        c->timing = enable != 0;
        for (int k = 0; k < SRM_B200_NPHASE; ++k) {
            c->ms[k] = 0.0;
            c->calls[k] = 0;
        }
        return SRM_B200_OK;
    });
}

int srm_b200_timing_get(srm_b200_ctx* c, double* ms, int64_t* calls) {
    return guarded(c, [&]() -> int {
        c->sync();
        c->harvest_timing();
        for (int k = 0; k < SRM_B200_NPHASE; ++k) {
            if (ms) ms[k] = c->ms[k];
            if (calls) calls[k] = c->calls[k];
        }
        return SRM_B200_OK;
    });
}

int srm_b200_sync(srm_b200_ctx* c) {
    return guarded(c, [&]() -> int {
        c->sync();
        return SRM_B200_OK;
    });
}

int srm_b200_set_generate_mode(srm_b200_ctx* c, int device_loop) {
    return guarded(c, [&]() -> int {
        c->device_loop = device_loop != 0;
        return SRM_B200_OK;
    });
}

int srm_b200_last_round_info(srm_b200_ctx* c, int64_t* info) {
    return guarded(c, [&]() -> int {
        info[0] = c->last_nonmovers;
        info[1] = c->hg.ncls;
        info[2] = c->hg.cls_cells;
        info[3] = c->hg.near_s[0];
        info[4] = c->hg.col_m[0];
        info[5] = c->hg.ncells;
        info[6] = c->last_wave_waits;
        info[7] = c->last_wave_polls;
        info[8] = c->last_pair_tests;
        return SRM_B200_OK;
    });
}

int srm_b200_stopwatch(srm_b200_ctx* c, int op, double* ms) {
    return guarded(c, [&]() -> int {
        if (!c->sw_start) {
            SRM_CUDA(cudaEventCreate(&c->sw_start));
            SRM_CUDA(cudaEventCreate(&c->sw_stop));
        }
        if (op == 0) {
            SRM_CUDA(cudaEventRecord(c->sw_start, c->stream));
        } else {
            SRM_CUDA(cudaEventRecord(c->sw_stop, c->stream));
            SRM_CUDA(cudaEventSynchronize(c->sw_stop));
            float t = 0.f;
            SRM_CUDA(cudaEventElapsedTime(&t, c->sw_start, c->sw_stop));
            if (ms) *ms = t;
        }
        return SRM_B200_OK;
    });
}

}  // extern "C"
