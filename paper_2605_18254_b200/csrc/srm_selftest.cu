// srm_selftest.cu -- device self-test entry points (parity of the device primitives).
//
// srm_b200_selftest_philox runs the hand-written Philox4x32-10 next to CUDA's own
// curand_Philox4x32_10 on the device; srm_b200_selftest_unit_vectors returns the
// device unit vectors so tests can compare them bit for bit with the oracle.
#include <cuda_runtime.h>
#include <curand_kernel.h>

#include "../../include/srm_b200.h"
#include "srm_device.cuh"

namespace {

__global__ void k_philox_pair(int64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* mine,
                              uint32_t* ref) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const srmb::U4 c{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]};
    const srmb::U4 o = srmb::philox4x32_10(c, key[2 * i], key[2 * i + 1]);
    mine[4 * i] = o.x;
    mine[4 * i + 1] = o.y;
    mine[4 * i + 2] = o.z;
    mine[4 * i + 3] = o.w;
    const uint4 r = curand_Philox4x32_10(make_uint4(c.x, c.y, c.z, c.w), make_uint2(key[2 * i], key[2 * i + 1]));
    ref[4 * i] = r.x;
    ref[4 * i + 1] = r.y;
    ref[4 * i + 2] = r.z;
    ref[4 * i + 3] = r.w;
}

template <int D>
__global__ void k_unit(int64_t n, srmb::RngKey key, const uint32_t* slot, const uint32_t* attempt,
                       uint32_t stream, double* out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double u[D];
    srmb::unit_vector<D>(key, slot[i], attempt[i], stream, u);
#pragma unroll
    for (int a = 0; a < D; ++a) out[i * D + a] = u[a];
}

template <typename T>
T* to_dev(const T* h, int64_t n) {
    T* d = nullptr;
    if (cudaMalloc(&d, sizeof(T) * (n > 0 ? n : 1)) != cudaSuccess) return nullptr;
    if (n > 0) cudaMemcpy(d, h, sizeof(T) * n, cudaMemcpyHostToDevice);
    return d;
}

}  // namespace

extern "C" {

int srm_b200_selftest_philox(int64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out_mine,
                             uint32_t* out_curand) {
    uint32_t *dc = to_dev(ctr, 4 * n), *dk = to_dev(key, 2 * n), *dm = nullptr, *dr = nullptr;
    cudaMalloc(&dm, sizeof(uint32_t) * 4 * (n > 0 ? n : 1));
    cudaMalloc(&dr, sizeof(uint32_t) * 4 * (n > 0 ? n : 1));
    int st = SRM_B200_OK;
    if (!dc || !dk || !dm || !dr) st = SRM_B200_CUDA_ERROR;
    if (st == SRM_B200_OK && n > 0) {
        k_philox_pair<<<(unsigned)((n + 255) / 256), 256>>>(n, dc, dk, dm, dr);
        if (cudaDeviceSynchronize() != cudaSuccess) st = SRM_B200_CUDA_ERROR;
        cudaMemcpy(out_mine, dm, sizeof(uint32_t) * 4 * n, cudaMemcpyDeviceToHost);
        cudaMemcpy(out_curand, dr, sizeof(uint32_t) * 4 * n, cudaMemcpyDeviceToHost);
    }
    cudaFree(dc); cudaFree(dk); cudaFree(dm); cudaFree(dr);
    return st;
}

int srm_b200_selftest_unit_vectors(int dim, uint64_t seed, int64_t n, const uint32_t* slot,
                                   const uint32_t* attempt, uint32_t stream, uint32_t round_id,
                                   uint32_t iteration, double* out) {
    if (dim != 2 && dim != 3) return SRM_B200_INVALID;
    uint32_t *ds = to_dev(slot, n), *da = to_dev(attempt, n);
    double* dout = nullptr;
    cudaMalloc(&dout, sizeof(double) * dim * (n > 0 ? n : 1));
    int st = SRM_B200_OK;
    if (!ds || !da || !dout) st = SRM_B200_CUDA_ERROR;
    const srmb::RngKey key{static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32), round_id & 0xFFFFFFu,
                           iteration};
    if (st == SRM_B200_OK && n > 0) {
        if (dim == 2) k_unit<2><<<(unsigned)((n + 255) / 256), 256>>>(n, key, ds, da, stream, dout);
        else k_unit<3><<<(unsigned)((n + 255) / 256), 256>>>(n, key, ds, da, stream, dout);
        if (cudaDeviceSynchronize() != cudaSuccess) st = SRM_B200_CUDA_ERROR;
        cudaMemcpy(out, dout, sizeof(double) * dim * n, cudaMemcpyDeviceToHost);
    }
    cudaFree(ds); cudaFree(da); cudaFree(dout);
    return st;
}

}  // extern "C"
