// qsv_adjoint.cu -- reverse-mode (adjoint) gradient of a product of Pauli
// rotations, all on the device (statevector.py:153-211).
//
// For U = U_R ... U_1 with U_r = exp(-i theta_r/2 P_r) and E = <psi|H|psi>,
// |psi> = U|psi0>:
//     dE/dtheta_r = 2 Re <lam_r| (-i/2) P_r |phi_r> = Im <lam_r| P_r |phi_r>,
// phi_r = U_r...U_1 psi0 (the state after rotation r) and
// lam_r = U_{r+1}^dag ... U_R^dag H|psi>.  Walking r = R-1 .. 0 both vectors
// are un-rotated in place: phi <- U_r^dag phi, lam <- U_r^dag lam, with
// U_r^dag = exp(+i theta_r/2 P_r) = cos I + i sin P_r.
//
// P convention (kernels.apply_pauli, _cykernels.pyx:76-102):
//     (P a)_j = i^{|y|} (-1)^{popc((j ^ f) & (y | z))} a_{j ^ f},   f = x | y.
//
// Consecutive rotations with the same flip f (the strings of one excitation)
// act on the same amplitude pairs (j, j ^ f), so they are processed as a run:
// each thread keeps its pairs in registers across the run (per-rotation
// partial inner products, then the un-rotation) -- one read and one write of
// both vectors per run.  Default: one launch per run over every SM
// (partials into a [block][rotation] array, one deterministic column
// reduction at the end); QSV_ADJOINT=smem: for 2^n <= 4096 a single CTA runs
// the whole sweep in shared memory (no launches, but one SM of FP64: 2.2x
// slower at 12 qubits).  Either way the host reads the gradient once.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "qsv_internal.h"

namespace qsv {

namespace {

__device__ __forceinline__ double2 mul_ipow(double2 v, int k)  // v * i^k
{
    switch (k & 3) {
        case 0: return v;
        case 1: return make_double2(-v.y, v.x);
        case 2: return make_double2(-v.x, -v.y);
        default: return make_double2(v.y, -v.x);
    }
}

__device__ __forceinline__ uint64_t ins0_64(uint64_t i, int b)
{
    return ((i >> b) << (b + 1)) | (i & ((1ull << b) - 1ull));
}

// Im conj(l) * w
__device__ __forceinline__ double im_cdot(double2 l, double2 w) { return l.x * w.y - l.y * w.x; }

// a <- cos a + i sin (P a) on the pair (j0, j1 = j0 ^ f), f != 0
__device__ __forceinline__ void unrotate_pair(double2 &a0, double2 &a1, uint64_t j0, uint64_t j1,
                                              uint64_t s, int ny, double c, double sn)
{
    // (P a)_{j0} = i^ny sg(j1) a1 ; (P a)_{j1} = i^ny sg(j0) a0 ; then times i sn
    double2 p0 = mul_ipow(a1, ny + 1), p1 = mul_ipow(a0, ny + 1);
    if (__popcll(j1 & s) & 1) p0 = make_double2(-p0.x, -p0.y);
    if (__popcll(j0 & s) & 1) p1 = make_double2(-p1.x, -p1.y);
    const double2 n0 = make_double2(fma(sn, p0.x, c * a0.x), fma(sn, p0.y, c * a0.y));
    const double2 n1 = make_double2(fma(sn, p1.x, c * a1.x), fma(sn, p1.y, c * a1.y));
    a0 = n0;
    a1 = n1;
}

// a_j <- (cos + i sin i^ny sg(j)) a_j  (diagonal string, f == 0)
__device__ __forceinline__ double2 unrotate_diag(double2 a, uint64_t j, uint64_t s, int ny, double c,
                                                 double sn)
{
    double2 p = mul_ipow(a, ny + 1);
    if (__popcll(j & s) & 1) p = make_double2(-p.x, -p.y);
    return make_double2(fma(sn, p.x, c * a.x), fma(sn, p.y, c * a.y));
}

constexpr int kSmemT = 512;
constexpr int kPPT = 4;     // amplitude pairs per thread (2^12 / 2 / 512)
constexpr int kGroup = 8;   // rotations of one same-flip run handled in registers

// Block sum of v[0..g) (fixed order: lanes, then warps) into grad[r_top - k].
__device__ __forceinline__ void block_sums(double (&v)[kGroup], int g, double (*red)[kSmemT / 32],
                                           double *grad, int r_top)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
        if (k >= g) break;
        double a = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) red[k][warp] = a;
    }
    __syncthreads();
    if (threadIdx.x < g) {
        double a = 0.0;
        for (int w = 0; w < kSmemT / 32; ++w) a += red[threadIdx.x][w];
        grad[r_top - (int)threadIdx.x] = a;
    }
}

// Whole backward sweep in one CTA, both vectors in shared memory.  A run of
// consecutive rotations with the same flip f acts on the same amplitude
// pairs (j, j ^ f): each thread keeps its pairs in registers across the run
// (partial inner products per rotation, then the un-rotation), so a run
// costs one load / store of the pairs and one batched block reduction.
__global__ void __launch_bounds__(kSmemT, 1)
adjoint_smem_kernel(double2 *__restrict__ phi_g, double2 *__restrict__ lam_g, int n, int R,
                    const uint64_t *__restrict__ X, const uint64_t *__restrict__ Y,
                    const uint64_t *__restrict__ Z, const double2 *__restrict__ cs,
                    double *__restrict__ grad)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t dim = 1u << n;
    double2 *phi = reinterpret_cast<double2 *>(smem_raw);
    double2 *lam = phi + dim;
    __shared__ double red[kGroup][kSmemT / 32];
    const int tid = threadIdx.x;
    for (uint32_t j = tid; j < dim; j += kSmemT) {
        phi[j] = phi_g[j];
        lam[j] = lam_g[j];
    }
    __syncthreads();
    int r = R - 1;
    while (r >= 0) {
        const uint32_t f = (uint32_t)(__ldg(X + r) | __ldg(Y + r));
        int r_lo = r;
        while (r_lo > 0 && r - r_lo + 1 < kGroup &&
               (uint32_t)(__ldg(X + r_lo - 1) | __ldg(Y + r_lo - 1)) == f)
            --r_lo;
        const int g = r - r_lo + 1;
        double part[kGroup];
#pragma unroll
        for (int k = 0; k < kGroup; ++k) part[k] = 0.0;
        if (f != 0) {
            const int h = 31 - __clz(f);
#pragma unroll
            for (int q = 0; q < kPPT; ++q) {
                const uint32_t p = tid + q * kSmemT;
                if (p >= dim / 2) break;
                const uint32_t j0 = (uint32_t)ins0_64(p, h), j1 = j0 ^ f;
                double2 a0 = phi[j0], a1 = phi[j1], b0 = lam[j0], b1 = lam[j1];
                for (int k = 0; k < g; ++k) {
                    const int rr = r - k;
                    const uint64_t y = __ldg(Y + rr), sm = y | __ldg(Z + rr);
                    const int ny = __popcll(y) & 3;
                    // Im <lam|P|phi> over the pair: (P a)_{j0} = i^ny sg(j1) a1, ...
                    double2 w0 = mul_ipow(a1, ny), w1 = mul_ipow(a0, ny);
                    if (__popcll(j1 & sm) & 1) w0 = make_double2(-w0.x, -w0.y);
                    if (__popcll(j0 & sm) & 1) w1 = make_double2(-w1.x, -w1.y);
                    part[k] += im_cdot(b0, w0) + im_cdot(b1, w1);
                    const double2 csr = __ldg(cs + rr);
                    unrotate_pair(a0, a1, j0, j1, sm, ny, csr.x, csr.y);
                    unrotate_pair(b0, b1, j0, j1, sm, ny, csr.x, csr.y);
                }
                phi[j0] = a0;
                phi[j1] = a1;
                lam[j0] = b0;
                lam[j1] = b1;
            }
        } else {  // diagonal strings: every amplitude on its own
            for (uint32_t j = tid; j < dim; j += kSmemT) {
                double2 a = phi[j], b = lam[j];
                for (int k = 0; k < g; ++k) {
                    const int rr = r - k;
                    const uint64_t y = __ldg(Y + rr), sm = y | __ldg(Z + rr);
                    const int ny = __popcll(y) & 3;
                    double2 w = mul_ipow(a, ny);
                    if (__popcll((uint64_t)j & sm) & 1) w = make_double2(-w.x, -w.y);
                    part[k] += im_cdot(b, w);
                    const double2 csr = __ldg(cs + rr);
                    a = unrotate_diag(a, j, sm, ny, csr.x, csr.y);
                    b = unrotate_diag(b, j, sm, ny, csr.x, csr.y);
                }
                phi[j] = a;
                lam[j] = b;
            }
        }
        // grad[r - k] for k < g (the reduction's barrier also orders this
        // run's SMEM writes before the next run's reads)
        block_sums(part, g, red, grad, r);
        __syncthreads();
        r = r_lo - 1;
    }
    for (uint32_t j = tid; j < dim; j += kSmemT) {
        phi_g[j] = phi[j];
        lam_g[j] = lam[j];
    }
}

constexpr int kT = 128;

// One same-flip run (rotations r_top, r_top-1, .., r_top-g+1) over the whole
// vector: every thread takes pairs (j, j ^ f) grid-stride, accumulates each
// rotation's inner product and un-rotates the pair in registers; the block's
// per-rotation sums go to partial[block][rotation] (reduced at the end in a
// fixed order).  Diagonal runs (f == 0) take single amplitudes.
__global__ void __launch_bounds__(kT) adjoint_run_kernel(
    double2 *__restrict__ phi, double2 *__restrict__ lam, uint64_t dim, uint64_t f, int r_top, int g,
    const uint64_t *__restrict__ Y, const uint64_t *__restrict__ Z, const double2 *__restrict__ cs,
    int R, double *__restrict__ partial)
{
    __shared__ double red[kGroup][kT / 32];
    double part[kGroup];
#pragma unroll
    for (int k = 0; k < kGroup; ++k) part[k] = 0.0;
    uint64_t sm[kGroup];
    int ny[kGroup];
    double2 csr[kGroup];
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
        if (k >= g) break;
        const uint64_t y = __ldg(Y + r_top - k);
        sm[k] = y | __ldg(Z + r_top - k);
        ny[k] = __popcll(y) & 3;
        csr[k] = __ldg(cs + r_top - k);
    }
    const uint64_t stride = (uint64_t)gridDim.x * kT;
    if (f != 0) {
        const int h = 63 - __clzll(f);
        for (uint64_t p = (uint64_t)blockIdx.x * kT + threadIdx.x; p < dim / 2; p += stride) {
            const uint64_t j0 = ins0_64(p, h), j1 = j0 ^ f;
            double2 a0 = phi[j0], a1 = phi[j1], b0 = lam[j0], b1 = lam[j1];
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
                if (k >= g) break;
                double2 w0 = mul_ipow(a1, ny[k]), w1 = mul_ipow(a0, ny[k]);
                if (__popcll(j1 & sm[k]) & 1) w0 = make_double2(-w0.x, -w0.y);
                if (__popcll(j0 & sm[k]) & 1) w1 = make_double2(-w1.x, -w1.y);
                part[k] += im_cdot(b0, w0) + im_cdot(b1, w1);
                unrotate_pair(a0, a1, j0, j1, sm[k], ny[k], csr[k].x, csr[k].y);
                unrotate_pair(b0, b1, j0, j1, sm[k], ny[k], csr[k].x, csr[k].y);
            }
            phi[j0] = a0;
            phi[j1] = a1;
            lam[j0] = b0;
            lam[j1] = b1;
        }
    } else {
        for (uint64_t j = (uint64_t)blockIdx.x * kT + threadIdx.x; j < dim; j += stride) {
            double2 a = phi[j], b = lam[j];
#pragma unroll
            for (int k = 0; k < kGroup; ++k) {
                if (k >= g) break;
                double2 w = mul_ipow(a, ny[k]);
                if (__popcll(j & sm[k]) & 1) w = make_double2(-w.x, -w.y);
                part[k] += im_cdot(b, w);
                a = unrotate_diag(a, j, sm[k], ny[k], csr[k].x, csr[k].y);
                b = unrotate_diag(b, j, sm[k], ny[k], csr[k].x, csr[k].y);
            }
            phi[j] = a;
            lam[j] = b;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kGroup; ++k) {
        if (k >= g) break;
        double v = part[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[k][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x < g) {
        double v = 0.0;
        for (int w = 0; w < kT / 32; ++w) v += red[threadIdx.x][w];
        partial[(size_t)blockIdx.x * R + (r_top - (int)threadIdx.x)] = v;
    }
}

int run_grid(uint64_t dim, int device)
{
    const uint64_t want = (dim / 2 + kT - 1) / kT;
    const uint64_t cap = (uint64_t)num_sms(device) * 16;
    return (int)(want < cap ? (want ? want : 1) : cap);
}

bool use_smem_kernel(int n)
{
    // QSV_ADJOINT=smem|runs; default: runs (every SM works on each run)
    const char *e = getenv("QSV_ADJOINT");
    return e && e[0] == 's' && n <= 12;
}

}  // namespace

int adjoint_smem_max_qubits() { return 12; }

size_t adjoint_scratch_doubles(int n, int64_t R, int device)
{
    if (use_smem_kernel(n)) return (size_t)R;
    return (size_t)run_grid(1ull << n, device) * (size_t)R + (size_t)R;
}

// X/Y/Z/cs (cos, sin of theta/2): device arrays of R rotations in forward
// order (hX/hY/hZ: the same masks on the host, to form the same-flip runs);
// d_scratch of adjoint_scratch_doubles(); the gradient lands in d_grad[R].
cudaError_t launch_rotation_adjoint(double2 *phi, double2 *lam, int n, int64_t R, const uint64_t *X,
                                    const uint64_t *Y, const uint64_t *Z, const uint64_t *hX,
                                    const uint64_t *hY, const uint64_t *hZ, const double2 *cs,
                                    double *d_scratch, double *d_grad, cudaStream_t st)
{
    if (R <= 0) return cudaSuccess;
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t dim = 1ull << n;
    if (use_smem_kernel(n)) {
        const size_t smem = 32 * (size_t)dim;
        static PerDeviceOnce once;
        cudaError_t e = once.run([] {
            return cudaFuncSetAttribute(adjoint_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        32 << 12);  // 2 x 4096 amplitudes
        });
        if (e != cudaSuccess) return e;
        adjoint_smem_kernel<<<1, kSmemT, smem, st>>>(phi, lam, n, (int)R, X, Y, Z, cs, d_grad);
        return cudaGetLastError();
    }
    const int G = run_grid(dim, dev);
    for (int64_t r = R - 1; r >= 0;) {
        const uint64_t f = hX[r] | hY[r];
        int64_t lo = r;
        while (lo > 0 && r - lo + 1 < kGroup && (hX[lo - 1] | hY[lo - 1]) == f) --lo;
        adjoint_run_kernel<<<G, kT, 0, st>>>(phi, lam, dim, f, (int)r, (int)(r - lo + 1), Y, Z, cs,
                                             (int)R, d_scratch);
        r = lo - 1;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_reduce_columns(d_scratch, G, (int)R, nullptr, d_grad, st);
}

}  // namespace qsv
