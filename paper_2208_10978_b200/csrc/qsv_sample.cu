// qsv_sample.cu -- shot sampling of a Z-basis parity (statevector.py:124-147).
//
// The reference draws `shots` outcomes with numpy's
//     Generator(Philox(seed)).choice(2^n, size=shots, p=|psi|^2 / sum)
// which is: cdf = cumsum(p); cdf /= cdf[-1]; u = random(shots) (53-bit
// uniforms of the Philox4x64-10 stream); idx = searchsorted(cdf, u, 'right').
// This file restates that on the device:
//   * p_i = hypot(re, im)^2 (numpy's abs(.)**2), normalised by the sum;
//   * cdf by a device-wide inclusive scan (CUB), normalised by its last entry;
//   * the same Philox4x64-10 stream (key from numpy's SeedSequence, passed in
//     by the host; counter of block b = b + 1, four outputs per block), so
//     every shot sees the reference's uniform bit for bit;
//   * upper-bound binary search per shot, parity of (idx & support), exact
//     int64 sum of +-1.
// Outcomes equal the reference's unless a uniform falls within the ~1e-16
// rounding difference between a parallel and a sequential prefix sum of a
// cdf boundary.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "qsv_internal.h"

namespace qsv {

namespace {

__global__ void probs_kernel(const double2 *__restrict__ psi, double *__restrict__ p, uint64_t dim)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < dim;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double2 a = psi[i];
        const double m = hypot(a.x, a.y);
        p[i] = m * m;
    }
}

__global__ void scale_kernel(double *__restrict__ p, uint64_t dim, const double *__restrict__ denom)
{
    const double d = *denom;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < dim;
         i += (uint64_t)gridDim.x * blockDim.x)
        p[i] /= d;
}

__global__ void copy_last_kernel(const double *__restrict__ cdf, uint64_t dim, double *__restrict__ out)
{
    *out = cdf[dim - 1];
}

__device__ __forceinline__ void philox4x64(uint64_t (&x)[4], uint64_t k0, uint64_t k1)
{
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t hi0 = __umul64hi(M0, x[0]), lo0 = M0 * x[0];
        const uint64_t hi1 = __umul64hi(M1, x[2]), lo1 = M1 * x[2];
        const uint64_t y0 = hi1 ^ x[1] ^ k0, y2 = hi0 ^ x[3] ^ k1;
        x[0] = y0;
        x[1] = lo1;
        x[2] = y2;
        x[3] = lo0;
        k0 += W0;
        k1 += W1;
    }
}

// one thread per Philox block (4 shots)
__global__ void sample_kernel(const double *__restrict__ cdf, uint64_t dim, int64_t shots,
                              uint64_t k0, uint64_t k1, uint64_t support,
                              unsigned long long *__restrict__ odd_count, int64_t *__restrict__ outcomes)
{
    unsigned int odd = 0;
    const int64_t nblk = (shots + 3) / 4;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nblk;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint64_t x[4] = {(uint64_t)b + 1ull, 0ull, 0ull, 0ull};
        philox4x64(x, k0, k1);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int64_t shot = 4 * b + w;
            if (shot >= shots) break;
            const double u = (double)(x[w] >> 11) * (1.0 / 9007199254740992.0);
            // searchsorted(cdf, u, side='right'): first index with cdf[idx] > u
            uint64_t lo = 0, hi = dim;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (cdf[mid] <= u) lo = mid + 1;
                else hi = mid;
            }
            if (outcomes) outcomes[shot] = (int64_t)lo;
            odd += __popcll(lo & support) & 1u;
        }
    }
    // warp + block reduction of the odd-parity count
    for (int o = 16; o > 0; o >>= 1) odd += __shfl_xor_sync(0xffffffffu, odd, o);
    if ((threadIdx.x & 31) == 0 && odd) atomicAdd(odd_count, (unsigned long long)odd);
}

int grid_for(uint64_t n, int device)
{
    uint64_t g = (n + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms(device) * 8;
    return (int)(g < cap ? (g ? g : 1) : cap);
}

}  // namespace

static inline size_t up256(size_t v) { return (v + 255) & ~(size_t)255; }

// Scratch layout (caller-provided device workspace of sample_scratch_bytes),
// every part 256 B aligned: [p, scanned in place into the cdf: 8*dim]
// [denom, last, odd count][cub temp] -- one 8-byte array per amplitude, so a
// 32-qubit state needs 32 GiB of scratch, not 64.
size_t sample_scratch_bytes(uint64_t dim)
{
    size_t t1 = 0, t2 = 0;
    cub::DeviceReduce::Sum(nullptr, t1, (const double *)nullptr, (double *)nullptr, (int64_t)dim);
    cub::DeviceScan::InclusiveSum(nullptr, t2, (double *)nullptr, (double *)nullptr, (int64_t)dim);
    const size_t temp = t1 > t2 ? t1 : t2;
    return up256(8 * dim) + 256 + up256(temp);
}

cudaError_t launch_sample_parity(const double2 *psi, uint64_t dim, int64_t shots, uint64_t k0,
                                 uint64_t k1, uint64_t support, void *scratch, size_t scratch_bytes,
                                 int64_t *d_outcomes, unsigned long long *h_odd, cudaStream_t st)
{
    int dev = 0;
    cudaGetDevice(&dev);
    char *base = (char *)scratch;
    double *p = (double *)base;
    double *cdf = p;  // inclusive scan in place (same additions in the same order)
    double *denom = (double *)(base + up256(8 * dim));
    double *last = denom + 1;
    unsigned long long *odd = (unsigned long long *)(denom + 2);
    void *temp = base + up256(8 * dim) + 256;
    size_t temp_bytes = scratch_bytes - up256(8 * dim) - 256;
    cudaError_t e;
    probs_kernel<<<grid_for(dim, dev), 256, 0, st>>>(psi, p, dim);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // probs /= probs.sum()
    if ((e = cub::DeviceReduce::Sum(temp, temp_bytes, p, denom, (int64_t)dim, st)) != cudaSuccess) return e;
    scale_kernel<<<grid_for(dim, dev), 256, 0, st>>>(p, dim, denom);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // cdf = cumsum(p); cdf /= cdf[-1]
    if ((e = cub::DeviceScan::InclusiveSum(temp, temp_bytes, p, cdf, (int64_t)dim, st)) != cudaSuccess)
        return e;
    copy_last_kernel<<<1, 1, 0, st>>>(cdf, dim, last);
    scale_kernel<<<grid_for(dim, dev), 256, 0, st>>>(cdf, dim, last);
    if ((e = cudaMemsetAsync(odd, 0, 8, st)) != cudaSuccess) return e;
    sample_kernel<<<grid_for((uint64_t)(shots + 3) / 4, dev), 256, 0, st>>>(cdf, dim, shots, k0, k1,
                                                                           support, odd, d_outcomes);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(h_odd, odd, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
}

}  // namespace qsv
