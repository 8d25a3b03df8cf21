// random_access_bench.cu -- what the memory system of a B200 gives the access patterns of the
// SRM migrate step: 32-byte records read at random from an array larger than
// L2, independently and through one level of indirection (row -> neighbour record), at full
// occupancy and with the sweep's 18 resident warps per SM.  A ceiling for the class sweep,
// whose time is these accesses.
//
//   make microbench && tools/random_access_bench [records = 10000000]
//
// Prints, per pattern, reads/s, the useful GB/s (32 bytes per read) and -- from the ncu run in
// profiles/ -- the DRAM traffic is about twice that (the L2 fetches 64 bytes per miss).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                       \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h;
}

// streaming: every record once, in order
__global__ void k_stream(int64_t n, const double4* __restrict__ rec, double* __restrict__ out) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s += rec[i].x;
    if (s == 12345.678) out[0] = s;
}

// `reads` random records per thread, independent of one another (all in flight)
template <int kUnroll>
__global__ void k_random(int64_t n, int reads, const double4* __restrict__ rec, double* __restrict__ out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0.0;
    for (int r = 0; r < reads; r += kUnroll) {
        double4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) v[u] = rec[mix(t * 977u + (r + u) * 0x9e3779b9u) % static_cast<uint32_t>(n)];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) s += v[u].x;
    }
    if (s == 12345.678) out[0] = s;
}

// the sweep's chain: a random row (32 bytes, holding an index), then the record it names
__global__ void k_chain(int64_t n, int reads, const int4* __restrict__ row, const double4* __restrict__ rec,
                        double* __restrict__ out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0.0;
    for (int r = 0; r < reads; ++r) {
        const uint32_t i = mix(t * 977u + r * 0x9e3779b9u) % static_cast<uint32_t>(n);
        const int4 h = row[2 * static_cast<int64_t>(i)];  // (rows are 32 bytes: two int4)
        const double4 me = rec[i];
        const double4 v = rec[h.y];
        s += v.x + me.x;
    }
    if (s == 12345.678) out[0] = s;
}

__global__ void k_fill(int64_t n, double4* rec, int4* row) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        rec[i] = make_double4(1.0 * i, 0.0, 0.0, 1.0);
        // a neighbour a few thousand records away (the next plane of cells), as in the sorted state
        const int64_t j = (i + 45000 + (mix(static_cast<uint32_t>(i)) & 1023)) % n;
        row[2 * i] = make_int4(1, static_cast<int>(j), 0, 0);
        row[2 * i + 1] = make_int4(0, 0, 0, 0);
    }
}

template <typename F>
double time_ms(F&& launch, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    launch();  // warm-up
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    CK(cudaGetLastError());
    return ms / reps;
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? std::atoll(argv[1]) : 10000000;
    if (argc > 2) {  // L2 fetch granularity hint in bytes (32 / 64 / 128), before the context is used
        const cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(std::atoi(argv[2])));
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        std::printf("L2 fetch granularity: asked %s, %s, now %zu\n", argv[2], cudaGetErrorString(e), got);
    }
    double4* rec;
    int4* row;
    double* out;
    CK(cudaMalloc(&rec, sizeof(double4) * n));
    CK(cudaMalloc(&row, sizeof(int4) * 2 * n));
    CK(cudaMalloc(&out, 64));
    k_fill<<<148 * 8, 256>>>(n, rec, row);
    CK(cudaDeviceSynchronize());
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::printf("records %lld x 32 B (%.0f MB) + rows %.0f MB, %d SMs\n", (long long)n, n * 32e-6, n * 32e-6, sms);
    {
        const double ms = time_ms([&] { k_stream<<<sms * 16, 256>>>(n, rec, out); }, 10);
        std::printf("%-58s %8.3f ms  %7.1f GB/s\n", "stream, 32 B records in order", ms, n * 32e-6 / ms);
    }
    const int reads = 64;
    struct Cfg {
        const char* name;
        int ctas_per_sm, threads;
    };
    // 2048 / 1024 threads per SM, and the class sweep's residency: 10 CTAs x 64 threads
    const Cfg cfgs[] = {{"64 warps per SM", 8, 256}, {"32 warps per SM", 4, 256}, {"20 warps per SM (the class sweep)", 10, 64}};
    for (const Cfg& c : cfgs) {
        const int grid = sms * c.ctas_per_sm;
        const double total = static_cast<double>(grid) * c.threads * reads;
        char label[128];
        double ms = time_ms([&] { k_random<1><<<grid, c.threads>>>(n, reads, rec, out); }, 5);
        std::snprintf(label, sizeof label, "random 32 B reads, 1 in flight per thread, %s", c.name);
        std::printf("%-58s %8.3f ms  %7.2f Greads/s  %7.1f GB/s useful\n", label, ms, total / ms * 1e-6, total * 32e-6 / ms);
        ms = time_ms([&] { k_random<4><<<grid, c.threads>>>(n, reads, rec, out); }, 5);
        std::snprintf(label, sizeof label, "random 32 B reads, 4 in flight per thread, %s", c.name);
        std::printf("%-58s %8.3f ms  %7.2f Greads/s  %7.1f GB/s useful\n", label, ms, total / ms * 1e-6, total * 32e-6 / ms);
        ms = time_ms([&] { k_chain<<<grid, c.threads>>>(n, reads, row, rec, out); }, 5);
        std::snprintf(label, sizeof label, "row + record, then the record the row names, %s", c.name);
        std::printf("%-58s %8.3f ms  %7.2f Gvisits/s %7.1f GB/s useful (96 B per visit)\n", label, ms, total / ms * 1e-6,
                    total * 96e-6 / ms);
    }
    return 0;
}
