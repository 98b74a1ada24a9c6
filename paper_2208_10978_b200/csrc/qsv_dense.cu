// qsv_dense.cu -- general k-qubit dense gate (qsv_apply_matrix, k = 1..5).
//
// Generalises the reference's apply_1q / apply_2q (kernels/_cykernels.pyx:19-73)
// to a 2^k x 2^k complex matrix whose row index is formed from the target
// qubits with qubits[0] as the MOST significant bit (the apply_2q convention:
// rows = 2*bit(q0) + bit(q1), circuit.py:5-6).  One thread per coset of the
// 2^(n-k) index classes that differ only in the target bits: it loads the
// coset's 2^k amplitudes into registers (the matrix sits in shared memory)
// and writes the 2^k outputs straight back -- one HBM read + write of every
// amplitude (32 B), HBM-bound for k <= 4 (2^k / 4 FLOP/B vs a ridge of ~5),
// FP64-bound at k = 5.  Consecutive threads own consecutive cosets, so every
// load / store is coalesced across the warp whenever the low qubits are not
// targets.
#include <cuda_runtime.h>
#include <stdint.h>

#include "qsv_internal.h"

namespace qsv {
namespace {

template <int K>
__global__ void __launch_bounds__(256) dense_kernel(double2 *__restrict__ psi, uint64_t ncos,
                                                    const double2 *__restrict__ g_m, uint4 qlo, uint4 qhi)
{
    constexpr int D = 1 << K;
    __shared__ double2 m[D * D];
    for (int i = threadIdx.x; i < D * D; i += blockDim.x) m[i] = g_m[i];
    __syncthreads();
    int q[8] = {(int)qlo.x, (int)qlo.y, (int)qlo.z, (int)qlo.w, (int)qhi.x, (int)qhi.y, (int)qhi.z, (int)qhi.w};
    // sorted target bits for the zero insertions
    int srt[8];
#pragma unroll
    for (int i = 0; i < K; ++i) srt[i] = q[i];
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = 0; j + 1 < K - i; ++j)
            if (srt[j] > srt[j + 1]) { const int t = srt[j]; srt[j] = srt[j + 1]; srt[j + 1] = t; }
    uint64_t off[D];
#pragma unroll
    for (int r = 0; r < D; ++r) {  // row r: bit (K-1-i) of r is the bit of qubits[i]
        uint64_t o = 0;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if ((r >> (K - 1 - i)) & 1) o |= 1ull << q[i];
        off[r] = o;
    }
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < ncos;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = t;
#pragma unroll
        for (int i = 0; i < K; ++i)
            base = ((base >> srt[i]) << (srt[i] + 1)) | (base & ((1ull << srt[i]) - 1ull));
        double2 a[D];
#pragma unroll
        for (int c = 0; c < D; ++c) a[c] = psi[base | off[c]];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double re = 0.0, im = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double2 mm = m[r * D + c];
                re = fma(mm.x, a[c].x, fma(-mm.y, a[c].y, re));
                im = fma(mm.x, a[c].y, fma(mm.y, a[c].x, im));
            }
            psi[base | off[r]] = make_double2(re, im);
        }
    }
}

}  // namespace

cudaError_t launch_dense(double2 *psi, int n, int k, const int *qubits, const double2 *d_m, int sms,
                         cudaStream_t st)
{
    uint4 lo = {0, 0, 0, 0}, hi = {0, 0, 0, 0};
    for (int i = 0; i < k && i < 4; ++i) (&lo.x)[i] = (unsigned)qubits[i];
    for (int i = 4; i < k; ++i) (&hi.x)[i - 4] = (unsigned)qubits[i];
    const uint64_t ncos = 1ull << (n - k);
    const uint64_t want = (ncos + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    const int grid = (int)(want < cap ? (want ? want : 1) : cap);
    switch (k) {
        case 1: dense_kernel<1><<<grid, 256, 0, st>>>(psi, ncos, d_m, lo, hi); break;
        case 2: dense_kernel<2><<<grid, 256, 0, st>>>(psi, ncos, d_m, lo, hi); break;
        case 3: dense_kernel<3><<<grid, 256, 0, st>>>(psi, ncos, d_m, lo, hi); break;
        case 4: dense_kernel<4><<<grid, 256, 0, st>>>(psi, ncos, d_m, lo, hi); break;
        case 5: dense_kernel<5><<<grid, 256, 0, st>>>(psi, ncos, d_m, lo, hi); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace qsv
